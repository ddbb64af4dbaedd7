cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_stream_cpals.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_register -s 3 -c 1 -o gpurun_out/prof_nell2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu2.log; tail -5 gpurun_out/ncu_full.log
