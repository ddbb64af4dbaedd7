cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 4 -c 1 -o gpurun_out/prof64_amazon python bench.py --config amazon --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > gpurun_out/ncu64_amazon.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 5 -c 4 -o gpurun_out/prof64_delicious python bench.py --config delicious --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > gpurun_out/ncu64_del.log 2>&1
ls gpurun_out/prof64*
