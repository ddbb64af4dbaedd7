cd $GRAFT_REPO_ROOT
for V in 100 0 100 0 500 1000; do
BLCO_B200_CLOCK_MS=$V timeout 900 python bench.py --config delicious_als > gpurun_out/bench53.json 2> /dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/bench53.json').read().strip().splitlines()[-1]); print('clock_ms=$V', d['value'], d['device_ms'])"
done
