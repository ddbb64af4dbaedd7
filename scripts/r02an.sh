# round 2: byte-table ALTO encode -- build parity (bit-exact) and build times
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_build.py tests/test_gpu_stress.py tests/test_gpu_fullsize.py tests/test_gpu_container.py -m gpu -q -x > gpurun_out/r02an_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02an_pytest.log
timeout 600 python scripts/build_probe.py nell2 nell2 amazon > gpurun_out/r02an_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_encode -c 2 --csv --log-file gpurun_out/r02an_encode_ncu.csv python scripts/build_probe.py nell2 > /dev/null 2>&1
