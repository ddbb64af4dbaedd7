cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu13.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu13.log
timeout 900 python bench.py > gpurun_out/bench13.json 2> gpurun_out/bench13.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench13_ref.json 2> gpurun_out/bench13_ref.err
tail -3 gpurun_out/pytest_gpu13.log; tail -2 gpurun_out/smoke13.log
tail -1 gpurun_out/bench13.json | cut -c1-1500; tail -1 gpurun_out/bench13_ref.json | cut -c1-600
