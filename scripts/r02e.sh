# round 2: micro-benchmark of factor-row gathers (LDG vs cp.async.bulk vs TMA gather4), library multi tests
for b in 1 2 3; do timeout 120 ./scripts/micro/bulk_gather $b >> gpurun_out/r02e_bulk.log 2>&1; done
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 6 --csv ./scripts/micro/bulk_gather 2 > gpurun_out/r02e_bulk_ncu.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "multi or cxx or stream" > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
