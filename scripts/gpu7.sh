cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream_cpals.py tests/test_gpu_mttkrp.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu7.log
timeout 900 python bench.py --config reddit_stream_small > gpurun_out/bench7_stream_small.json 2> gpurun_out/bench7_stream_small.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench7_torchrun1.json 2> gpurun_out/bench7_torchrun1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7_als.csv python bench.py --config enron_als > gpurun_out/ncu7_als.log 2>&1
tail -3 gpurun_out/pytest_gpu7.log; cut -c1-1500 gpurun_out/bench7_stream_small.json; tail -5 gpurun_out/bench7_stream_small.err; cut -c1-300 gpurun_out/bench7_torchrun1.json; tail -3 gpurun_out/bench7_torchrun1.err
