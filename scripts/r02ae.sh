# round 2: final verification of the current build -- sanitizers, the full GPU suite, smoke,
# the driver's bench and reference arm, the launch list of the bench command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/sanitize.sh > /dev/null 2>&1
for t in memcheck racecheck synccheck; do mv gpurun_out/sanitize_$t.log gpurun_out/r02ae_sanitize_$t.log; done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02ae_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ae_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ae_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02ae_bench.json 2> gpurun_out/r02ae_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02ae_ref.json 2> gpurun_out/r02ae_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02ae_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ncu > /dev/null 2>&1
tail -3 gpurun_out/r02ae_pytest.log; cat gpurun_out/r02ae_smoke.log; tail -2 gpurun_out/r02ae_sanitize_*.log
