# round 2: library multi-GPU path (G = 1 on this box), C++ drop-in suite, multi-rank plumbing
timeout 1200 python -m pytest tests -m gpu -q -x -k "multi or cxx or stream" > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02d_pytest.log
