cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_build.py tests/test_gpu_fullsize.py tests/test_gpu_container.py tests/test_gpu_stream_cpals.py tests/test_gpu_mttkrp.py -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench40.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench40.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['build'])"
timeout 900 python bench.py --config amazon --steps 1 --no-e2e --no-cpu-baseline > gpurun_out/bench40_a.json 2>&1
python3 -c "
import json; d=json.loads(open('gpurun_out/bench40_a.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['build'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_digit" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu40.csv 2>&1
grep -E '^"[0-9]' gpurun_out/ncu40.csv | awk -F'","' '{n=split($5,a,"("); print a[1], $13, $15}' | head -40
