cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in 0 1 2; do
  BLCO_B200_LOADS=$L timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench20_l$L.json 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench20_l$L.json').read().strip().splitlines()[-1]); print('loads=$L', d['ms_per_step'], d['per_mode_ms'])"
done
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__lsu_writeback_active_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_red.sum,l1tex__data_pipe_lsu_wavefronts.sum
for L in 0 1; do
BLCO_B200_LOADS=$L timeout 600 ncu --metrics $M --csv -k regex:k_mttkrp_sorted -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu20_l$L.csv 2>&1
python3 - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/ncu20_l$L.csv")) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print("L$L", d["Metric Name"], d["Metric Value"])
PY
done
