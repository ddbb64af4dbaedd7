cd $GRAFT_REPO_ROOT/scripts/micro
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_global_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum
timeout 300 ncu --metrics $M --csv -c 4 ./red_wavefronts > ../../gpurun_out/micro_red24.csv 2>&1
timeout 300 ncu --metrics $M --csv ./smem_wavefronts > ../../gpurun_out/micro_smem24.csv 2>&1
cd ../..
for f in gpurun_out/micro_red24.csv gpurun_out/micro_smem24.csv; do grep -E '^"[0-9]' $f | awk -F'","' '{print $5, $13, $15}' | cut -c1-120; done
