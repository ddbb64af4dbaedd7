# round 2 (redo of r02x, ncu reports summarised on the box so gpurun_out stays small):
# every other BASELINE configuration, reference arms, ncu --set full of the mode kernels, tile span probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg1 > gpurun_out/r02y_cfg1.json 2> gpurun_out/r02y_cfg1.err
timeout 900 python bench.py --config nell2 > gpurun_out/r02y_nell2.json 2> gpurun_out/r02y_nell2.err
timeout 900 python bench.py --config delicious_als > gpurun_out/r02y_als.json 2> gpurun_out/r02y_als.err
timeout 2400 python bench.py --config reddit_stream > gpurun_out/r02y_stream.json 2> gpurun_out/r02y_stream.err
for c in nell2 delicious_als reddit_stream; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 1 > gpurun_out/r02y_reference_$c.json 2> /dev/null
done
PROBE_MODES=0,1,2 PROBE_REPS=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_mttkrp_sorted -o /tmp/prof_amazon python scripts/panel_probe.py amazon "" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mttkrp_sorted -s 4 -c 3 -o /tmp/prof_nell2 python bench.py --config nell2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 --no-ncu > /dev/null 2>&1
PROBE_REPS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mttkrp_sorted -o /tmp/prof_delicious python scripts/panel_probe.py delicious "" > /dev/null 2>&1
for c in amazon nell2 delicious; do python scripts/ncu_summary.py full /tmp/prof_$c.ncu-rep gpurun_out/r02y_ncu_$c.json; ncu -i /tmp/prof_$c.ncu-rep --page details --csv > gpurun_out/r02y_ncu_${c}_details.csv 2>&1; done
timeout 1500 python scripts/tile_span_probe.py nell2 delicious amazon > gpurun_out/r02y_tile_spans.log 2>&1
ls -la gpurun_out/
