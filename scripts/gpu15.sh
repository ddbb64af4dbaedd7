cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe15.log 2>&1
cat gpurun_out/e2e_probe15.log | tail -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 3 -c 1 -o gpurun_out/prof15_nell2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu15.log 2>&1
tail -3 gpurun_out/ncu15.log
