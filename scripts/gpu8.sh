cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream_cpals.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu8.log
timeout 900 python bench.py --config delicious_als > gpurun_out/bench8_als.json 2> gpurun_out/bench8_als.err
timeout 1500 python bench.py --config reddit_stream > gpurun_out/bench8_stream.json 2> gpurun_out/bench8_stream.err
tail -3 gpurun_out/pytest_gpu8.log; cut -c1-400 gpurun_out/bench8_als.json; tail -3 gpurun_out/bench8_als.err; cut -c1-1800 gpurun_out/bench8_stream.json; tail -5 gpurun_out/bench8_stream.err; free -g
