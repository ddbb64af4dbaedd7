cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu25.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu25.log
timeout 900 python bench.py > gpurun_out/bench25.json 2> gpurun_out/bench25.err
timeout 300 python scripts/phase_probe.py nell2
tail -3 gpurun_out/pytest_gpu25.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu25.log | head
python3 -c "
import json; d=json.loads(open('gpurun_out/bench25.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['per_mode_ms'], d['e2e']['ms_per_step'], d.get('cpu_baseline'))"
