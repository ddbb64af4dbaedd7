cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_stream_cpals.py tests/test_gpu_cxx.py tests/test_gpu_fullsize.py -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench46.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench46.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['per_mode_ms'], d['fp32_variant']['ms_per_step'])"
timeout 900 python bench.py --config amazon --steps 2 --no-e2e --no-cpu-baseline --no-fp32 > gpurun_out/bench46_a.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench46_a.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['per_mode_ms'])"
timeout 900 python bench.py --config delicious_als > gpurun_out/bench46_als.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench46_als.json').read().strip().splitlines()[-1]); print(d['value'], d['mttkrp_per_mode_ms'])"
