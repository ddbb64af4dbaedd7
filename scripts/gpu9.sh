cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BLCO_B200_TRACE=1 timeout 900 python bench.py --config delicious_als > gpurun_out/bench9_als.json 2> gpurun_out/bench9_als.err
ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shfl.sum,gpu__time_duration.sum,sm__inst_executed.sum scripts/micro/shfl_cost > gpurun_out/micro_shfl.txt 2>&1
cut -c1-300 gpurun_out/bench9_als.json; grep trace gpurun_out/bench9_als.err; grep -E "shfl|lds|k_|wavefronts|duration|inst_executed" gpurun_out/micro_shfl.txt | head -30
