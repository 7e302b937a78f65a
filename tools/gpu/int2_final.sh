timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f2_tests.log; grep -E "^FAILED" gpurun_out/f2_tests.log | head
timeout 1500 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/f2_hbm_int2.json 2> gpurun_out/f2_hbm_int2.err; echo "int2 rc=$?"
timeout 1500 python bench.py --config 4 > gpurun_out/f2_config4.json 2> gpurun_out/f2_config4.err; echo "c4 rc=$?"
