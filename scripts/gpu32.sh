cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_solve_gram|k_scale_inner|k_reduce|k_gram" -c 40 python bench.py --config delicious_als > gpurun_out/ncu32_als.csv 2>&1
grep -E '^"[0-9]' gpurun_out/ncu32_als.csv | awk -F'","' '{print $5, $15}' | cut -c1-40,100-200 | head -40
