cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench36.json 2> gpurun_out/bench36.err
timeout 900 python bench.py --config cfg1 > gpurun_out/bench36_cfg1.json 2> gpurun_out/bench36_cfg1.err
timeout 1200 python bench.py --config amazon --steps 3 --no-cpu-baseline > gpurun_out/bench36_amazon.json 2> gpurun_out/bench36_amazon.err
timeout 900 python bench.py --config delicious_als > gpurun_out/bench36_als.json 2> gpurun_out/bench36_als.err
timeout 1800 python bench.py --config reddit_stream > gpurun_out/bench36_stream.json 2> gpurun_out/bench36_stream.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches36.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for f in bench36 bench36_cfg1 bench36_amazon bench36_als bench36_stream; do echo $f; tail -1 gpurun_out/$f.json | cut -c1-200; done
