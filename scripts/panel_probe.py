"""Probe: panel-ordered tile dispatch (mttkrp.cu panel_plan) on an Amazon-shaped
(or Delicious-shaped, order 4) tensor.  For each BLCO_B200_PANEL setting: per-mode kernel ms (CUDA events,
L2 flushed between launches) and the relative difference from the ALTO-order
result.  Usage: panel_probe.py [amazon|amazon_small] [setting ...]"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"amazon": ([4821207, 1774269, 1805187], 1_741_809_018, 32, 0),
        "amazon_small": ([4821207, 1774269, 1805187], 200_000_000, 32, 0),
        "reddit_dev": ([8211298, 176962, 8116559], 1_000_000_000, 32, 0),
        "delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 16, 4)}
name = sys.argv[1] if len(sys.argv) > 1 else "amazon"
settings = sys.argv[2:] or ["0", "", "16,16", "17,17", "18,17", "17,18", "18,18", "16,18", "18,16"]
dims, nnz, R, skew = cfgs[name]
dt = b.DeviceTensor.synthetic_draws(dims, nnz, 42, skew) if skew else b.DeviceTensor.synthetic(dims, nnz, 42)
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
cfg = b.ExecConfig(num_compute_units=148)
modes = [int(x) for x in os.environ.get("PROBE_MODES", ",".join(map(str, range(len(dims))))).split(",")]
reps = int(os.environ.get("PROBE_REPS", "3"))
ref = [None] * len(dims)
for st in settings:
    # "VAR=value[,VAR=value]" sets library knobs (read per call); anything else is BLCO_B200_PANEL
    if "=" in st:
        for kv in st.split(";"):
            k, v = kv.split("=", 1)
            os.environ[k] = v
    else:
        os.environ["BLCO_B200_PANEL"] = st
    tot = 0.0
    row = []
    for m in modes:
        out = torch.zeros((dims[m], R), dtype=torch.float64, device="cuda")
        dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out.data_ptr(), b.Strategy.Register, cfg, stream=s)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out.data_ptr(), b.Strategy.Register, cfg, stream=s)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        if ref[m] is None:
            ref[m] = out.clone()
        err = float(torch.linalg.norm(out - ref[m]) / torch.linalg.norm(ref[m]))
        t = min(ts) if ts else float('nan')
        tot += t
        row.append(f"m{m} {t:.1f} ms ({err:.0e})")
        del out
    print(f"{name} {st if '=' in st else 'PANEL=' + (st or 'auto')}: all modes {tot:.1f} ms | " + " | ".join(row), flush=True)
