cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu16.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu16.log
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe16.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench16.json 2> gpurun_out/bench16.err
timeout 1500 python bench.py --config reddit_stream > gpurun_out/bench16_stream.json 2> gpurun_out/bench16_stream.err
tail -4 gpurun_out/pytest_gpu16.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu16.log | head
tail -8 gpurun_out/e2e_probe16.log
python3 -c "
import json; d=json.loads(open('gpurun_out/bench16.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])
d=json.loads(open('gpurun_out/bench16_stream.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['stream'])"
tail -3 gpurun_out/bench16_stream.err
