cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config delicious_als > gpurun_out/bench11_als.json 2> gpurun_out/bench11_als.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 3 -c 1 -o gpurun_out/prof11_amazon python bench.py --config amazon --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu11_amazon.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 4 -c 4 -o gpurun_out/prof11_delicious python bench.py --config delicious --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu11_del.log 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench11_als.json').read().strip().splitlines()[-1]); print(d['value'], d['device_ms'], d['cp_als_call_ms'], d['mttkrp_per_mode_ms'])"; tail -2 gpurun_out/ncu11_amazon.log | cut -c1-300; tail -2 gpurun_out/ncu11_del.log | cut -c1-300
