"""Probe: Register vs Hierarchical per mode on a tensor (kernel ms, CUDA events)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 16, 4),
        "nell2": ([12092, 9184, 28818], 76_879_419, 32, 0),
        "short": ([24, 200000, 100000], 20_000_000, 32, 0),
        "short16": ([100, 300000, 200000], 20_000_000, 16, 0)}
name = sys.argv[1] if len(sys.argv) > 1 else "delicious"
dims, nnz, R, skew = cfgs[name]
dt = b.DeviceTensor.synthetic_draws(dims, nnz, 42, skew) if skew else b.DeviceTensor.synthetic(dims, nnz, 42)
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
s = torch.cuda.current_stream().cuda_stream
for m in range(len(dims)):
    ref = None
    for strat in (b.Strategy.Register, b.Strategy.Hierarchical):
        for copies in ((1,) if strat == b.Strategy.Register else (1, 4)):
            out = torch.zeros((dims[m], R), dtype=torch.float64, device="cuda")
            cfg = b.ExecConfig(num_compute_units=148, num_factor_copies=copies)
            for _ in range(2):
                dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out.data_ptr(), strat, cfg, stream=s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                dt.mttkrp_device([a.data_ptr() for a in fac], R, m, out.data_ptr(), strat, cfg, stream=s)
            e1.record()
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            err = float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref))
            print(f"{name} mode {m} rows {dims[m]} {strat.name} copies {copies}: {e0.elapsed_time(e1) / 5:.3f} ms "
                  f"(rel diff {err:.1e})", flush=True)
