cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cd scripts/micro
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__lsu_writeback_active_mem_lgds.sum,smsp__inst_executed_op_global_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum
timeout 300 ncu --metrics $M --csv ./smem_wavefronts > ../../gpurun_out/micro_smem17.csv 2>&1
timeout 300 ncu --metrics $M --csv ./ldg_wavefronts > ../../gpurun_out/micro_ldg17.csv 2>&1
cd ../..
python3 - <<'PY'
import csv
for f in ("gpurun_out/micro_smem17.csv","gpurun_out/micro_ldg17.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]
    for r in rows[1:]:
        d=dict(zip(h,r)); print(d["Kernel Name"][:20], d["Metric Name"], d["Metric Value"])
PY
