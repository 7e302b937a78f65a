timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:draft_attn_quant -s 40 -c 1 -o gpurun_out/full_draft_b16 -f python tools/profile_step.py --mode draft --x 1 > gpurun_out/ncu_draft_b16.log 2>&1; echo ncu rc=$?
