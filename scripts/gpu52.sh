cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke52.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu52.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu52.log
timeout 900 python bench.py > gpurun_out/bench52.json 2> gpurun_out/bench52.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench52_ref.json 2> gpurun_out/bench52_ref.err
timeout 900 python bench.py --config cfg1 > gpurun_out/bench52_cfg1.json 2> gpurun_out/bench52_cfg1.err
timeout 1200 python bench.py --config amazon --steps 3 --no-cpu-baseline > gpurun_out/bench52_amazon.json 2> gpurun_out/bench52_amazon.err
timeout 900 python bench.py --config delicious_als > gpurun_out/bench52_als.json 2> gpurun_out/bench52_als.err
timeout 1800 python bench.py --config reddit_stream > gpurun_out/bench52_stream.json 2> gpurun_out/bench52_stream.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mttkrp_sorted<" -s 3 -c 3 -o gpurun_out/prof52_nell2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches52.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu52.log; tail -1 gpurun_out/smoke52.log
for f in bench52 bench52_ref bench52_cfg1 bench52_amazon bench52_als bench52_stream; do echo $f; tail -1 gpurun_out/$f.json | cut -c1-150; done
