cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench4_sorted.json 2>&1
BLCO_B200_VARIANT=warp timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench4_warp.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 3 -c 1 -o gpurun_out/prof4_sorted python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
BLCO_B200_VARIANT=warp timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_warp -s 3 -c 1 -o gpurun_out/prof4_warp python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu4w.log 2>&1
tail -3 gpurun_out/pytest_gpu4.log; cut -c1-300 gpurun_out/bench4_*.json
