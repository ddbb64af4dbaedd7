"""Probe: host-link rate of the all-mode host pipeline vs plain pinned H2D."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2201_12523_b200 as b

dims, nnz, R = [12092, 9184, 28818], 76_879_419, 32
dt = b.DeviceTensor.synthetic(dims, nnz, 42)
host = dt.to_host()
idx = b.api.pinned_empty(host.idx.size, np.uint64); idx[:] = host.idx
vals = b.api.pinned_empty(host.vals.size, np.float64); vals[:] = host.vals
ht = b.BlcoTensor(host.layout, host.max_nnz_per_block, host.keys, host.offsets, idx, vals)
f = b.FactorMatrices.random(dims, R, 7)
pf = []
for a in f.factors:
    p = b.api.pinned_empty(a.size, np.float64).reshape(a.shape); p[:] = a; pf.append(p)
f = b.FactorMatrices(R, pf)
outs = [b.api.pinned_empty(d * R, np.float64).reshape(d, R) for d in dims]

ti = torch.from_numpy(idx); tv = torch.from_numpy(vals)
print("pinned?", ti.is_pinned())
di = torch.empty_like(ti, device="cuda"); dv = torch.empty_like(tv, device="cuda")
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); di.copy_(ti, non_blocking=True); dv.copy_(tv, non_blocking=True); e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"plain H2D payload {nnz*16/1e9:.3f} GB: {ms:.2f} ms = {nnz*16/ms/1e6:.1f} GB/s")
src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True); dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dst.copy_(src, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print(f"torch pinned 1 GiB: {(1<<30)/e0.elapsed_time(e1)/1e6:.1f} GB/s")
rep = b.AllModesReport()
for chunk in [nnz, nnz // 4, nnz // 8, nnz // 16, nnz // 32, nnz // 64, nnz // 128]:
    ms = []
    for _ in range(4):
        b.mttkrp_all_modes(ht, f, outs=outs, chunk_elems=chunk, report=rep)
        ms.append(rep.device_ms)
    print(f"chunk {chunk}: chunks {rep.chunks} device_ms {min(ms[1:]):.2f} {ms}")
