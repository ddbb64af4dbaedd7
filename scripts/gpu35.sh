cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_mttkrp.py -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu35.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu35.log
tail -30 gpurun_out/pytest_gpu35.log | cut -c1-400
timeout 600 python bench.py --config reddit_stream_tiny --steps 2 > gpurun_out/bench35_tiny.json 2>&1; tail -2 gpurun_out/bench35_tiny.json | cut -c1-300
