set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | head -20
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err; echo "bench host rc=$?"; cat gpurun_out/bench_host.json; tail -5 gpurun_out/bench_host.err
timeout 900 python bench.py --tier hbm --no-cpu > gpurun_out/bench_hbm.json 2> gpurun_out/bench_hbm.err; echo "bench hbm rc=$?"; cat gpurun_out/bench_hbm.json; tail -5 gpurun_out/bench_hbm.err
for m in decode draft mixed; do timeout 600 python tools/profile_step.py --mode $m > gpurun_out/step_$m.log 2>&1; tail -1 gpurun_out/step_$m.log; done
for m in decode draft mixed; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launch_$m.csv $m; done
