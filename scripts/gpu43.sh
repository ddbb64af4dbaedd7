cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -q -k "fp32" --timeout 600 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench43.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench43.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['per_mode_ms'], d['fp32_variant'])"
timeout 900 python bench.py --config amazon --steps 2 --no-e2e --no-cpu-baseline > gpurun_out/bench43_a.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench43_a.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['per_mode_ms'], d['fp32_variant'])"
