cd $GRAFT_REPO_ROOT/scripts/micro
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__lsu_writeback_active_mem_lgds.sum,smsp__inst_executed_op_global_ld.sum,gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 300 ncu --metrics $M --csv -c 4 ./ldg_wavefronts > ../../gpurun_out/micro_ldg19.csv 2>&1
cd ../..
python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/micro_ldg19.csv")) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d["ID"], d["Kernel Name"][:18], d["Metric Name"], d["Metric Value"])
PY
