cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench3_sorted.json 2>&1
BLCO_B200_VARIANT=warp timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench3_warp.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 3 -c 1 -o gpurun_out/prof3_sorted python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/pytest_gpu3.log; cut -c1-400 gpurun_out/bench3_*.json
