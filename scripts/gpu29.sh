cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_solve_gram" -s 1 -c 1 -o gpurun_out/prof29_solve python bench.py --config delicious_als > gpurun_out/ncu29.log 2>&1
tail -2 gpurun_out/ncu29.log
