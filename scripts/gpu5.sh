cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench5_full.json 2> gpurun_out/bench5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu5_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 1 -c 3 -o gpurun_out/prof5_modes python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu5_full.log 2>&1
timeout 1200 python bench.py --config amazon --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench5_amazon.json 2> gpurun_out/bench5_amazon.err
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 > gpurun_out/bench5_cfg1.json 2> gpurun_out/bench5_cfg1.err
cut -c1-300 gpurun_out/bench5_*.json; tail -3 gpurun_out/bench5_amazon.err
