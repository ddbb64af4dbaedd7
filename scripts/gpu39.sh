cd $GRAFT_REPO_ROOT
for P in 0 2 3 4; do
  BLCO_B200_PIPE=$P timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench39_p$P.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench39_p$P.json').read().strip().splitlines()[-1]); print('pipe=$P', d['ms_per_step'], d['per_mode_ms'])"
done
for P in 0 2 3; do
  BLCO_B200_PIPE=$P timeout 900 python bench.py --config amazon --steps 2 --no-e2e --no-cpu-baseline > gpurun_out/bench39_a$P.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench39_a$P.json').read().strip().splitlines()[-1]); print('amazon pipe=$P', d['ms_per_step'], d['per_mode_ms'])"
done
