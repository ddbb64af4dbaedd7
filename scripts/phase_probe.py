"""Probe: processing vs computing phase cycles of the sorted MTTKRP kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"nell2": ([12092, 9184, 28818], 76_879_419, 32, 0),
        "amazon": ([4821207, 1774269, 1805187], 1_741_809_018, 32, 0),
        "delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 16, 4)}
name = sys.argv[1] if len(sys.argv) > 1 else "nell2"
dims, nnz, R, skew = cfgs[name]
dt = (b.DeviceTensor.synthetic_draws(dims, nnz, 42, skew) if skew else b.DeviceTensor.synthetic(dims, nnz, 42))
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
out = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
cfg = b.ExecConfig(num_compute_units=148)
tiles = dt.nnz // 1024 + dt.nblocks
for m in range(len(dims)):
    st = b.MttkrpStats()
    dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out[m].data_ptr(), config=cfg, stats=st)
    dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out[m].data_ptr(), config=cfg, stats=st)
    print(f"{name} mode {m}: kernel {st.kernel_ms:.3f} ms, segments/nnz {st.segments / nnz:.3f}, "
          f"processing {st.processing_cycles / tiles:.0f} cyc/CTA, computing {st.computing_cycles / tiles / 8:.0f} cyc/warp")
