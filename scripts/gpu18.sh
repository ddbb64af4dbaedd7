cd $GRAFT_REPO_ROOT/scripts/micro
./red_wavefronts > ../../gpurun_out/micro_red18.log 2>&1
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,lts__t_sectors.sum,l1tex__m_l1tex2xbar_write_bytes.sum,smsp__inst_executed.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --csv -c 3 ./red_wavefronts > ../../gpurun_out/micro_red18.csv 2>&1
cd ../..
cat gpurun_out/micro_red18.log
python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/micro_red18.csv")) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d["Kernel Name"][:10], d["Metric Name"], d["Metric Value"])
PY
