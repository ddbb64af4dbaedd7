cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream_cpals.py tests/test_gpu_cxx.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -2
timeout 900 python bench.py --config delicious_als > gpurun_out/bench28_als.json 2> gpurun_out/bench28_als.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench28_als.json').read().strip().splitlines()[-1]); print(d['value'], d['device_ms'], d['mttkrp_per_mode_ms'], d['fit_history'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_solve_gram|k_scale_inner" -c 8 python bench.py --config delicious_als > gpurun_out/ncu28_als.csv 2>&1
grep -E '^"[0-9]' gpurun_out/ncu28_als.csv | awk -F'","' '{print $5, $13, $15}' | cut -c1-20,90-200 | head -24
