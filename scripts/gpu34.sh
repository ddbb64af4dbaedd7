cd $GRAFT_REPO_ROOT
for V in "" "CUDA_LAUNCH_BLOCKING=1" "BLCO_B200_TRACE=1"; do
env $V timeout 900 python bench.py --config delicious_als > gpurun_out/bench34.json 2> /dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/bench34.json').read().strip().splitlines()[-1]); print('$V', d['value'], d['device_ms'])"
done
