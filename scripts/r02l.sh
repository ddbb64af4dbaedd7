# round 2: Amazon gather L1 policy (ld.global.nc / .cg / L1::no_allocate) x panel order
set -x
mkdir -p gpurun_out
for v in base g1 g3; do
  if [ $v = base ]; then unset BLCO_B200_LIB; else export BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_b200_$v.so; fi
  echo "== $v" >> gpurun_out/r02l_gather.log
  timeout 900 python scripts/panel_probe.py amazon 0 16,16 >> gpurun_out/r02l_gather.log 2>&1
done
unset BLCO_B200_LIB
for v in base g1; do
  if [ $v = base ]; then unset BLCO_B200_LIB; else export BLCO_B200_LIB=$PWD/paper_2201_12523_b200/lib/variants/libblco_b200_$v.so; fi
  PROBE_MODES=0 PROBE_REPS=0 timeout 600 ncu --metrics l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_mttkrp_sorted --csv --log-file gpurun_out/r02l_ncu_$v.csv python scripts/panel_probe.py amazon 0 16,16 > /dev/null 2>&1
done
