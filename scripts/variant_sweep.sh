# Kernel-variant sweep (build variants into paper_2201_12523_b200/lib/variants
# first); per variant: NELL-2 / config-1 / Amazon all-mode ms and the
# Delicious CP-ALS MTTKRP per-mode ms.  Output: gpurun_out/variants.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/variants.log
for v in base ${VARIANTS:-}; do
  if [ $v = base ]; then unset BLCO_B200_LIB; else export BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_b200_$v.so; fi
  for c in nell2 cfg1; do
    timeout 300 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-fp32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v $c', d['ms_per_step'], d['per_mode_ms'], d['segments_mode0'])" >> gpurun_out/variants.log
  done
  if [ -n "$AMAZON" ]; then timeout 600 python bench.py --config amazon --steps 3 --no-e2e --no-cpu-baseline --no-fp32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v amazon', d['ms_per_step'], d['per_mode_ms'])" >> gpurun_out/variants.log; fi
  timeout 600 python bench.py --config delicious_als --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v als', d['value'], d['mttkrp_per_mode_ms'])" >> gpurun_out/variants.log
done
cat gpurun_out/variants.log
