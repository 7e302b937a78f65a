#!/bin/bash
# ncu launch lists of the bench command itself (profiler window = the serving loop)
BENCH_NCU=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launch_bench_hbm.csv python bench.py --tier hbm --no-secondary --no-cpu --steps 2 --warmup 1 \
  > gpurun_out/ncu_bench_hbm.log 2>&1; echo "hbm rc=$?"
BENCH_NCU=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launch_bench_host.csv python bench.py --no-secondary --no-cpu --steps 2 --warmup 1 \
  > gpurun_out/ncu_bench_host.log 2>&1; echo "host rc=$?"
ls -la gpurun_out/launch_bench_*.csv
