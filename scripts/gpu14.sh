cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x --durations=8 > gpurun_out/pytest_gpu14.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu14.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench14.json 2> gpurun_out/bench14.err
tail -15 gpurun_out/pytest_gpu14.log
python3 -c "
import json; d=json.loads(open('gpurun_out/bench14.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
tail -3 gpurun_out/bench14.err
