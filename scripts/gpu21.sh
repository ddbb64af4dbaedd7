cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__lsu_writeback_active_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed_op_global_red.sum,l1tex__data_pipe_lsu_wavefronts.sum,smsp__sass_inst_executed_op_global_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum
for L in 0 8; do
BLCO_B200_LOADS=$L timeout 600 ncu --metrics $M --csv -k regex:k_mttkrp_sorted -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu21_l$L.csv 2>&1
grep -E "lgds|wavefronts|duration|red" gpurun_out/ncu21_l$L.csv | awk -F'","' '{print "'L$L'", $13, $15}'
done
