# round 2: panel-ordered dispatch on Amazon (parity + width sweep), fused vs per-mode A/B on NELL-2
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mttkrp.py -m gpu -q -x -k "panel" > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
for c in nell2 nell2_r16 cfg1; do timeout 300 python scripts/fused_ab.py $c 10 >> gpurun_out/r02i_fused_ab.log 2>&1; done
timeout 1200 python scripts/panel_probe.py amazon 0 "" 16,16 17,17 18,17 17,18 18,18 16,18 18,16 15,15 > gpurun_out/r02i_panel.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed -k regex:k_mttkrp_sorted --csv --log-file gpurun_out/r02i_ncu_panel.csv python scripts/panel_probe.py amazon_small 0 "" > /dev/null 2>&1
