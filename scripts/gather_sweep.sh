cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in base g1 g2 g3; do
  if [ $v = base ]; then unset BLCO_B200_LIB; else export BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_b200_$v.so; fi
  echo "== $v" >> gpurun_out/sweep.log
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-fp32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('nell2', d['ms_per_step'], d['per_mode_ms'])" >> gpurun_out/sweep.log
  timeout 600 python bench.py --config amazon --steps 3 --no-e2e --no-cpu-baseline --no-fp32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('amazon', d['ms_per_step'], d['per_mode_ms'])" >> gpurun_out/sweep.log
  timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,lts__t_sectors.sum,gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_mttkrp_sorted -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 2>/dev/null | grep k_mttkrp >> gpurun_out/sweep.log
done
cat gpurun_out/sweep.log
