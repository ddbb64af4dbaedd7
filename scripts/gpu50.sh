cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mttkrp_sorted" -s 3 -c 1 -o gpurun_out/prof50_f64 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mttkrp_sorted_f32" -s 2 -c 1 -o gpurun_out/prof50_f32 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof50*
