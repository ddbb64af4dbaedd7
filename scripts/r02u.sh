# round 2: solve kernel R = 16 at 3 vs 4 CTAs/SM (interleaved)
set -x
mkdir -p gpurun_out
for v in base s4 base s4; do
  if [ $v = base ]; then unset BLCO_B200_LIB; else export BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_b200_$v.so; fi
  echo "== $v" >> gpurun_out/r02u_probe.err
  BLCO_B200_ALS_PROBE=1 timeout 600 python bench.py --config delicious_als --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu 2>&1 >/dev/null | grep "mode 1" | tail -2 >> gpurun_out/r02u_probe.err
done
