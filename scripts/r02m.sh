# round 2: panel width sweep on Amazon (per-call knob build), ALTO-order controls interleaved; dram gather microbench
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/panel_probe.py amazon 0 16,16 15,15 0 17,17 16,15 15,16 0 17,16 16,17 14,14 0 18,16 16,31 31,16 0 15,17 17,15 16,16 0 > gpurun_out/r02m_panel.log 2>&1
for b in 2 3; do timeout 300 ./scripts/micro/dram_gather $b 7 >> gpurun_out/r02m_dram_gather.log 2>&1; done
timeout 600 ncu --metrics l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_mode -c 3 --csv ./scripts/micro/dram_gather 3 7 > gpurun_out/r02m_dram_gather_ncu.csv 2>&1
