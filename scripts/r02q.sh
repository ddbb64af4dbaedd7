# round 2: Stage<N>=4 row-in-record -- parity (orders 4-8), Delicious per-mode and CP-ALS
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_stress.py tests/test_gpu_cpals_exact.py -m gpu -q -x > gpurun_out/r02q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02q_pytest.log
timeout 900 python scripts/panel_probe.py delicious "" 0 "" 0 > gpurun_out/r02q_panel_delicious.log 2>&1
timeout 600 python bench.py --config delicious_als --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02q_als.json 2>> gpurun_out/r02q_als.err
