cd $GRAFT_REPO_ROOT
BLCO_B200_TRACE=1 timeout 900 python bench.py --config delicious_als > gpurun_out/bench33_als.json 2> gpurun_out/bench33_als.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench33_als.json').read().strip().splitlines()[-1]); print(d['value'], d['device_ms'], d['cp_als_call_ms'])"
tail -3 gpurun_out/bench33_als.err
