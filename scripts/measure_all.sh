# Round measurement on one B200 (run through gpurun from the repo root):
# smoke, the GPU test suite, every BASELINE configuration, the reference arm,
# and the ncu captures summarised under profiles/.  Outputs -> gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_nell2.json 2> gpurun_out/bench_nell2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> /dev/null
timeout 900 python bench.py --config cfg1 > gpurun_out/bench_cfg1.json 2> /dev/null
timeout 1500 python bench.py --config amazon --steps 3 > gpurun_out/bench_amazon.json 2> /dev/null
timeout 900 python bench.py --config delicious_als > gpurun_out/bench_als.json 2> /dev/null
timeout 1800 python bench.py --config reddit_stream > gpurun_out/bench_stream.json 2> /dev/null
for c in amazon delicious_als reddit_stream; do
  timeout 900 python bench.py --impl reference --config $c --steps 1 --warmup 1 > gpurun_out/bench_reference_$c.json 2> /dev/null
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mttkrp_sorted -s 4 -c 3 \
  -o gpurun_out/prof_nell2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_nell2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for f in bench_nell2 bench_reference bench_cfg1 bench_amazon bench_als bench_stream bench_reference_amazon bench_reference_delicious_als bench_reference_reddit_stream; do
  echo $f; tail -1 gpurun_out/$f.json | cut -c1-160
done
# then, here:  python scripts/ncu_summary.py full gpurun_out/prof_nell2.ncu-rep profiles/ncu_nell2.json
#              python scripts/ncu_summary.py launches gpurun_out/launches_nell2.csv profiles/r01_launches_nell2.json
