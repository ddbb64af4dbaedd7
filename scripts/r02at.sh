# round 2: last full verification -- sanitizers (byte-table encode, det kernel tables), the full GPU suite, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/sanitize.sh > /dev/null 2>&1
for t in memcheck racecheck synccheck; do mv gpurun_out/sanitize_$t.log gpurun_out/r02at_sanitize_$t.log; done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02at_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02at_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02at_smoke.log 2>&1
tail -2 gpurun_out/r02at_pytest.log; cat gpurun_out/r02at_smoke.log; tail -2 gpurun_out/r02at_sanitize_*.log
