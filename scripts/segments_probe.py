"""Probe: segments (runs of equal target rows after the CTA grouping) per
non-zero for every mode of a config, from MttkrpStats of the stats kernel.
Usage: segments_probe.py [delicious|amazon|nell2 ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"amazon": ([4821207, 1774269, 1805187], 1_741_809_018, 32, 0),
        "delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 16, 4),
        "nell2": ([12092, 9184, 28818], 76_879_419, 32, 0)}
for name in sys.argv[1:] or ["delicious"]:
    dims, nnz, R, skew = cfgs[name]
    dt = b.DeviceTensor.synthetic_draws(dims, nnz, 42, skew) if skew else b.DeviceTensor.synthetic(dims, nnz, 42)
    fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
    b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
    for m in range(len(dims)):
        out = torch.zeros((dims[m], R), dtype=torch.float64, device="cuda")
        st = b.MttkrpStats()
        dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out.data_ptr(), b.Strategy.Register, stats=st)
        torch.cuda.synchronize()
        print(f"{name} mode {m} ({dims[m]} rows): segments/nnz {st.segments / nnz:.3f}, commits {st.commit_events}, "
              f"processing {st.processing_cycles / max(1, st.processing_cycles + st.computing_cycles):.2f} of cycles",
              flush=True)
        del out
    del dt, fac
