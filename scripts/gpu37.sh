cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for P in 0 45000 100000; do
  BLCO_B200_SMEM_PAD=$P timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench37_p$P.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench37_p$P.json').read().strip().splitlines()[-1]); print('pad=$P', d['ms_per_step'], d['per_mode_ms'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mttkrp_sorted -s 3 -c 3 -o gpurun_out/prof37_nell2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu37.log 2>&1
tail -1 gpurun_out/ncu37.log
