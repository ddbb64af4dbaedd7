# round 2: panel default (32 MB) -- parity, default bench, Delicious CP-ALS with/without panels, L2-resident gather microbench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_fullsize.py -m gpu -q -x -k "panel or fused or all_modes or amazon or delicious" > gpurun_out/r02n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02n_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
for p in 0 ""; do BLCO_B200_PANEL=$p timeout 600 python bench.py --config delicious_als --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02n_als_panel$p.json 2>> gpurun_out/r02n_als.err; done
for s in 100000 400000; do timeout 300 ./scripts/micro/dram_gather 3 7 $s >> gpurun_out/r02n_dram_gather.log 2>&1; done
