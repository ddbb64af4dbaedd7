"""Single-GPU emulation of the per-rank compute of the multi-GPU strong-scaling
step (NOT a multi-GPU measurement): the Amazon-shaped tensor is cut into G
nnz-balanced span ranges exactly as blco_partition cuts it for G GPUs, and
every slice's all-mode MTTKRP (panel-ordered, full-size partial M_n) is timed
alone on this GPU.  max over slices = the compute part of a G-GPU step; the
NCCL reduce-scatter of M_n (overlapped with the next mode's kernel) comes on
top.  Usage: slice_probe.py [G ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

dims, nnz, R = [4821207, 1774269, 1805187], 1_741_809_018, 32
full = b.DeviceTensor.synthetic(dims, nnz, 42)
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
fp = [a.data_ptr() for a in fac]
outs = [torch.zeros((d, R), dtype=torch.float64, device="cuda") for d in dims]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def step_ms(dt, reps=3):
    for m in range(3):  # warm-up (builds the slice's panel tables)
        dt.mttkrp_device(fp, R, m, outs[m].data_ptr(), b.Strategy.Register, stream=s)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for m in range(3):
            dt.mttkrp_device(fp, R, m, outs[m].data_ptr(), b.Strategy.Register, stream=s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


one = step_ms(full)
print(f"G=1: {one:.1f} ms per all-mode step", flush=True)
for G in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    ranges = b.partition(full.block_nnz(), 1024, G)
    per = []
    for lo, hi in ranges:
        sl = full.slice(lo, hi, 0)
        per.append(step_ms(sl, 2))
        del sl
    mx = max(per)
    print(f"G={G}: slice steps {' '.join(f'{x:.1f}' for x in per)} ms; max {mx:.1f} ms = "
          f"{one / mx / G:.3f} of linear (compute only, one GPU emulating each rank)", flush=True)
