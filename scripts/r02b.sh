# round 2: new parity tests + the reworked bench (Amazon headline, live ncu traffic, NELL-2 key)
python -m pytest tests -m gpu -x -q -k "census or refilling or escalation or two_rank_all_mode_streaming or amazon_full_size or nell2_full_size_build or synthetic_builds" > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?" >> gpurun_out/r02b_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?" >> gpurun_out/r02b_ref.err
