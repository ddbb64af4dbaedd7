set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
timeout 600 python bench.py --config amazon --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_amazon.json 2> gpurun_out/r02a_bench_amazon.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_mttkrp --launch-skip 3 --launch-count 3 --csv --log-file gpurun_out/r02a_ncu_amazon.csv python bench.py --config amazon --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fp32 > /dev/null 2>&1
tail -5 gpurun_out/r02a_pytest.log
