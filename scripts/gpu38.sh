cd $GRAFT_REPO_ROOT
for L in 0 1 2; do
  BLCO_B200_ROWLOAD=$L timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench38_l$L.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench38_l$L.json').read().strip().splitlines()[-1]); print('rowload=$L', d['ms_per_step'], d['per_mode_ms'])"
  BLCO_B200_ROWLOAD=$L timeout 900 python bench.py --config amazon --steps 2 --no-e2e --no-cpu-baseline > gpurun_out/bench38_a$L.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench38_a$L.json').read().strip().splitlines()[-1]); print('amazon rowload=$L', d['ms_per_step'], d['per_mode_ms'])"
done
