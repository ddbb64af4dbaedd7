cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu10.log
timeout 600 python bench.py --config delicious_als > gpurun_out/bench10_als.json 2> gpurun_out/bench10_als.err
tail -3 gpurun_out/pytest_gpu10.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu10.log | head; cut -c1-200 gpurun_out/bench10_als.json; python3 -c "
import json; d=json.loads(open('gpurun_out/bench10_als.json').read().strip().splitlines()[-1]); print(d['cp_als_call_ms'], d['mttkrp_per_mode_ms'])"
