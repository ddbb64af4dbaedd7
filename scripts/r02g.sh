# round 2: fused all-mode kernel parity + speed, skeleton probe, L2 window probe on Amazon, build timings
./scripts/micro/fused_skeleton > gpurun_out/r02g_skeleton.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or all_modes or multi or census or stress or build" > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02g_pytest.log
for cfg in u2m3 u4m2; do BLCO_B200_FUSED_CFG=$cfg timeout 600 python bench.py --config nell2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 --no-ncu > gpurun_out/r02g_nell2_$cfg.json 2>> gpurun_out/r02g_bench.err; done
timeout 600 python scripts/build_probe.py nell2 amazon > gpurun_out/r02g_build.log 2>&1
for w in 0 0.5 1.0; do BLCO_B200_L2WINDOW=$w timeout 600 python bench.py --config amazon --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 --no-ncu --no-extra > gpurun_out/r02g_amazon_l2w_$w.json 2>> gpurun_out/r02g_bench.err; done
