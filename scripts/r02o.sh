# round 2: panel parity (fp32 too); Delicious per-mode panel sweep; ncu full of the Delicious long mode
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -m gpu -q -x -k "panel" > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02o_pytest.log
timeout 900 python scripts/panel_probe.py delicious 0 "" 16,16 17,17 18,18 17,16 0 > gpurun_out/r02o_panel_delicious.log 2>&1
PROBE_MODES=1 PROBE_REPS=0 timeout 900 ncu --set full --import-source on -k regex:k_mttkrp_sorted -c 1 -o gpurun_out/r02o_delicious_m1 python scripts/panel_probe.py delicious "" > gpurun_out/r02o_ncu.log 2>&1
ncu -i gpurun_out/r02o_delicious_m1.ncu-rep --page raw --csv > gpurun_out/r02o_raw.csv 2>&1
ncu -i gpurun_out/r02o_delicious_m1.ncu-rep --page details --csv > gpurun_out/r02o_details.csv 2>&1
