cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu12.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu12.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench12.json 2>&1
timeout 900 python bench.py --config amazon --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench12_amazon.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches12.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu12.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu12.log | head -5
python3 -c "
import json
for f in ('gpurun_out/bench12.json','gpurun_out/bench12_amazon.json'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['build'])"
