nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv
timeout 1500 python -m pytest tests/test_real_shapes.py tests/test_ref_boundary.py tests/test_drop_parity.py -m gpu -q -s -p no:cacheprovider > gpurun_out/new_tests.log 2>&1; echo "new rc=$?"
grep -E "MEASURED|passed|failed|Error" gpurun_out/new_tests.log | tail -60
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu.log 2>&1; echo "all rc=$?"; tail -15 gpurun_out/all_gpu.log
