# round 2: ncu --set full of Amazon mode 0 under ALTO order vs 16,16 panels
set -x
mkdir -p gpurun_out
PROBE_MODES=0 PROBE_REPS=1 timeout 1500 ncu --set full --import-source on -k regex:k_mttkrp_sorted -o gpurun_out/r02k_amazon_panel python scripts/panel_probe.py amazon 0 16,16 > gpurun_out/r02k_probe.log 2>&1
ncu -i gpurun_out/r02k_amazon_panel.ncu-rep --page raw --csv > gpurun_out/r02k_raw.csv 2>&1
ncu -i gpurun_out/r02k_amazon_panel.ncu-rep --page details --csv > gpurun_out/r02k_details.csv 2>&1
