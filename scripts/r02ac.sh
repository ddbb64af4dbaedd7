# round 2: CP-ALS with the normalisation folded into the solves -- parity vs the reference goldens, the ALS step
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cpals_exact.py tests/test_gpu_stream_cpals.py tests/test_gpu_multirank.py tests/test_gpu_cxx.py -m gpu -q > gpurun_out/r02ac_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ac_pytest.log
BLCO_B200_ALS_PROBE=1 timeout 600 python bench.py --config delicious_als --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu > gpurun_out/r02ac_als_probe.json 2> gpurun_out/r02ac_als_probe.err
timeout 900 python bench.py --config delicious_als --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu > gpurun_out/r02ac_als.json 2> gpurun_out/r02ac_als.err
