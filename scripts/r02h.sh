# round 2 (re-entry): full GPU suite, default bench (driver command), reference arm, launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02h_smi.txt
nproc >> gpurun_out/r02h_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?" >> gpurun_out/r02h_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02h_ref.json 2> gpurun_out/r02h_ref.err; echo "ref rc=$?" >> gpurun_out/r02h_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/r02h_launch_bench.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1
