cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu31.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu31.log
tail -3 gpurun_out/pytest_gpu31.log; grep -E "^FAILED|^ERROR|Error:|assert " gpurun_out/pytest_gpu31.log | head -20
timeout 900 python bench.py --config delicious_als > gpurun_out/bench31_als.json 2> gpurun_out/bench31_als.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench31_als.json').read().strip().splitlines()[-1]); print(d['value'], d['device_ms'], d['mttkrp_per_mode_ms'], d['fit_history'][-1])"
