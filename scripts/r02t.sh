# round 2: solve kernel at 168 registers (R = 16) -- parity and the ALS step
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cpals_exact.py tests/test_gpu_stream_cpals.py -m gpu -q -x > gpurun_out/r02t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02t_pytest.log
BLCO_B200_ALS_PROBE=1 timeout 600 python bench.py --config delicious_als --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu > gpurun_out/r02t_als_probe.json 2> gpurun_out/r02t_als_probe.err
timeout 900 python bench.py --config delicious_als --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02t_als.json 2> gpurun_out/r02t_als.err
