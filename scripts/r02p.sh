# round 2: full GPU suite (NCCL one-rank path included), default bench, reference arm, smoke
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02p_pytest.log
timeout 900 python bench.py > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err; echo "bench rc=$?" >> gpurun_out/r02p_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02p_ref.json 2> gpurun_out/r02p_ref.err; echo "ref rc=$?" >> gpurun_out/r02p_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.log 2>&1
