# round 2: ncu full of the CP-ALS solve kernel (Delicious mode 1); ALS bench with live traffic
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:k_solve_gram --launch-skip 1 -c 1 -o gpurun_out/r02s_solve python bench.py --config delicious_als --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ncu > gpurun_out/r02s_ncu.log 2>&1
ncu -i gpurun_out/r02s_solve.ncu-rep --page details --csv > gpurun_out/r02s_details.csv 2>&1
ncu -i gpurun_out/r02s_solve.ncu-rep --page raw --csv > gpurun_out/r02s_raw.csv 2>&1
timeout 900 python bench.py --config delicious_als --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02s_als.json 2> gpurun_out/r02s_als.err
