"""A/B probe on an L2-resident order-3 tensor: the fused all-mode kernel
(blco_mttkrp_all_device) against three per-mode launches, interleaved, L2
flushed before every step, nvidia-smi clocks sampled.  Usage:
fused_ab.py [nell2|cfg1] [rounds]"""
import subprocess
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"nell2": ([12092, 9184, 28818], 76_879_419, 32), "cfg1": ([1000, 1000, 1000], 1_000_000, 16),
        "nell2_r16": ([12092, 9184, 28818], 76_879_419, 16)}
name = sys.argv[1] if len(sys.argv) > 1 else "nell2"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims, nnz, R = cfgs[name]
dt = b.DeviceTensor.synthetic(dims, nnz, 42)
fac = [torch.empty((d, R), dtype=torch.float64, device="cuda") for d in dims]
b.factors_random_device(dims, R, 7, [a.data_ptr() for a in fac], 0)
outs = [torch.zeros((d, R), dtype=torch.float64, device="cuda") for d in dims]
ref = [torch.zeros((d, R), dtype=torch.float64, device="cuda") for d in dims]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
fp = [a.data_ptr() for a in fac]


def fused():
    assert dt.mttkrp_all_device(fp, R, [o.data_ptr() for o in outs], stream=s)


def per_mode():
    for m in range(3):
        dt.mttkrp_device(fp, R, m, ref[m].data_ptr(), b.Strategy.Register, stream=s)


def timed(fn):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "100"],
                       stdout=subprocess.PIPE, text=True)
for _ in range(3):
    fused(), per_mode()
tf, tp = [], []
for _ in range(rounds):
    tf.append(timed(fused))
    tp.append(timed(per_mode))
smi.terminate()
clk = [ln for ln in smi.communicate()[0].splitlines() if ln.strip()]
err = max(float(torch.linalg.norm(outs[m] - ref[m]) / torch.linalg.norm(ref[m])) for m in range(3))
tf.sort(), tp.sort()
print(f"{name} R={R}: fused median {tf[len(tf) // 2]:.3f} ms (min {tf[0]:.3f}) | per-mode median "
      f"{tp[len(tp) // 2]:.3f} ms (min {tp[0]:.3f}) | rel diff {err:.1e} | clocks {clk[len(clk) // 2] if clk else '?'}",
      flush=True)
