cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu6.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu6.log
for v in mb2 mb3 packed; do
  BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench6_$v.json 2>&1
done
timeout 900 python bench.py --config delicious_als > gpurun_out/bench6_als.json 2> gpurun_out/bench6_als.err
tail -3 gpurun_out/pytest_gpu6.log; for v in mb2 mb3 packed; do echo $v; cut -c1-200 gpurun_out/bench6_$v.json; done; cut -c1-600 gpurun_out/bench6_als.json; tail -3 gpurun_out/bench6_als.err
