cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for T in 0 81 83 45 21 26; do
  BLCO_B200_TUNE=$T timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench22_t$T.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench22_t$T.json').read().strip().splitlines()[-1]); print('tune=$T', d['ms_per_step'], d['per_mode_ms'])"
done
