# round 2: full-size Amazon DRAM bytes per launch under panel orders (ncu), gather microbench
set -x
mkdir -p gpurun_out
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum -k regex:k_mttkrp_sorted --launch-skip 3 --launch-count 100 --csv --log-file gpurun_out/r02j_ncu_panel.csv python scripts/panel_probe.py amazon 0 16,16 14,31 31,14 18,16 > gpurun_out/r02j_probe_under_ncu.log 2>&1
for b in 1 2 3; do timeout 120 ./scripts/micro/bulk_gather $b >> gpurun_out/r02j_bulk.log 2>&1; done
for k in k_ldg k_ring; do timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:$k -c 2 --csv ./scripts/micro/bulk_gather 2 >> gpurun_out/r02j_bulk_ncu.csv 2>&1; done
