# round 2: final confirmation after the byte-table encode -- full GPU suite, smoke, default bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02ao_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ao_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ao_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02ao_bench.json 2> gpurun_out/r02ao_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02ao_ref.json 2> gpurun_out/r02ao_ref.err
tail -2 gpurun_out/r02ao_pytest.log; cat gpurun_out/r02ao_smoke.log
