cd $GRAFT_REPO_ROOT
timeout 300 python scripts/phase_probe.py nell2
for T in 0 21; do
  BLCO_B200_TUNE=$T timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench23_t$T.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench23_t$T.json').read().strip().splitlines()[-1]); print('tune=$T', d['ms_per_step'], d['per_mode_ms'])"
done
