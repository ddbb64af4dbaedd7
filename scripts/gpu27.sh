cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv -k regex:"k_solve_gram|k_scale_inner|k_gram" python bench.py --config delicious_als > gpurun_out/ncu27_als.csv 2>&1
grep -E '^"[0-9]' gpurun_out/ncu27_als.csv | awk -F'","' '{print $5, $13, $15}' | head -48
