"""Probe: cost of the deterministic mode against the default kernels (NELL-2 shape)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

dims, nnz, R = [12092, 9184, 28818], 76_879_419, 32
dt = b.DeviceTensor.synthetic(dims, nnz, 42)
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
outs = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
fp = [a.data_ptr() for a in fac]
s = torch.cuda.current_stream().cuda_stream
for det in (False, True):
    cfg = b.ExecConfig(num_compute_units=148, deterministic=det)
    t0 = time.perf_counter()
    for m in range(3):
        dt.mttkrp_device(fp, R, m, outs[m].data_ptr(), config=cfg, stream=s)
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        for m in range(3):
            dt.mttkrp_device(fp, R, m, outs[m].data_ptr(), config=cfg, stream=s)
    e1.record()
    torch.cuda.synchronize()
    print(f"deterministic={det}: all-mode {e0.elapsed_time(e1) / 5:.2f} ms/iter; first call (index build) {first * 1e3:.1f} ms")
