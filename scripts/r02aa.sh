# round 2: tile-relative StageR record -- parity, then interleaved A/B (BLCO_B200_REL_STAGE) on Amazon and Delicious
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_stress.py tests/test_gpu_fullsize.py tests/test_gpu_cpals_exact.py -m gpu -q -x > gpurun_out/r02aa_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02aa_pytest.log
timeout 900 python scripts/panel_probe.py delicious BLCO_B200_REL_STAGE=0 BLCO_B200_REL_STAGE=1 BLCO_B200_REL_STAGE=0 BLCO_B200_REL_STAGE=1 > gpurun_out/r02aa_delicious.log 2>&1
timeout 900 python scripts/panel_probe.py amazon BLCO_B200_REL_STAGE=0 BLCO_B200_REL_STAGE=1 BLCO_B200_REL_STAGE=0 BLCO_B200_REL_STAGE=1 > gpurun_out/r02aa_amazon.log 2>&1
