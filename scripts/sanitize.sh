# compute-sanitizer over small workloads of every kernel family (SURVEY.md 5:
# memcheck / racecheck / synccheck on configs 1 and 4, small).  Output -> gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/san_work.py <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2201_12523_b200 as b
dims = [120, 90, 150]
coo = b.synth_uniform_host(dims, 30000, 3)
t = b.build_blco(coo, 12, 5000)                      # device build, several blocks
f = b.FactorMatrices.random(dims, 32, 7)
for m in range(3):
    b.mttkrp(t, f, m)                                  # register path
    b.mttkrp(t, f, m, strategy=b.Strategy.Hierarchical)
    b.mttkrp(t, f, m, b.ExecConfig(deterministic=True))
b.mttkrp_all_modes(t, f, chunk_elems=4096)             # host pipeline
bud = b.DeviceBudget(capacity_bytes=1 << 28, num_queues=2, reservation_bytes=t.max_nnz_per_block * 16)
b.stream_mttkrp_all_modes(t, f, bud)                   # streaming
d4 = [40, 50, 30, 20]
t4 = b.DeviceTensor.synthetic_draws(d4, 20000, 42, 4)  # config-4 style draws
b.cp_als(t4, b.CpAlsOptions(rank=16, max_iters=2, tol=-1e300, seed=7))
# round 2: the fused all-mode kernel (opt-in), the device census, the library multi-GPU step (G = 1)
import torch
dt = b.DeviceTensor.synthetic([300, 250, 400], 40000, 5, 16, 4000)
fac = [torch.rand((d, 32), dtype=torch.float64, device="cuda") for d in (300, 250, 400)]
outs = [torch.zeros((d, 32), dtype=torch.float64, device="cuda") for d in (300, 250, 400)]
import os
os.environ["BLCO_B200_FUSED"] = "1"                    # the opt-in fused kernel
assert dt.mttkrp_all_device([a.data_ptr() for a in fac], 32, [o.data_ptr() for o in outs])
os.environ["BLCO_B200_FUSED"] = "0"
dt.census()
f3 = b.FactorMatrices.random([300, 250, 400], 32, 7)
b.MultiDeviceTensor(dt, [0]).mttkrp_all_modes(f3, reduce="reducescatter")
# panel-ordered dispatch (factors beyond L2: 307 MB), fp64 and fp32, orders 3 and 4
dp = [600000, 300000, 300000]
tp = b.DeviceTensor.synthetic(dp, 50000, 9, 48, 20000)
fp = b.FactorMatrices.random(dp, 32, 3)
for m in range(3):
    b.mttkrp(tp, fp, m)
    b.mttkrp_f32(tp, fp, m)
os.environ["BLCO_B200_PANEL"] = "10,12"
b.mttkrp(tp, fp, 0)
d5 = [300000, 200000, 150000, 50]
t5 = b.DeviceTensor.synthetic(d5, 30000, 4)
b.mttkrp(t5, b.FactorMatrices.random(d5, 32, 3), 1)
torch.cuda.synchronize()
print("sanitize workload done")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_work.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
