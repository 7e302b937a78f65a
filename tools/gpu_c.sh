timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:draft_attn_quant -s 600 -c 1 \
    -o gpurun_out/full_draft_b16 -f python tools/profile_step.py --mode draft > gpurun_out/ncu_draft_b16.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --tier hbm --no-cpu --steps 32 --warmup 8 > gpurun_out/bench_hbm.json 2> gpurun_out/bench_hbm.err; echo "bench rc=$?"; cat gpurun_out/bench_hbm.json; tail -3 gpurun_out/bench_hbm.err
