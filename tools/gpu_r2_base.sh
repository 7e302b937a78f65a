# round-2 re-entry health check: all GPU tests, smoke, mixed-step launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/all_gpu.log; grep -E "^FAILED" gpurun_out/all_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
for m in draft mixed; do timeout 600 python tools/profile_step.py --mode $m > gpurun_out/step_$m.log 2>&1; tail -3 gpurun_out/step_$m.log; done
for m in mixed; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launch_$m.csv $m; done
