# int2 draft-kernel pass (gpurun -- bash tools/gpu/int2.sh): GPU suite, the int2 bench lines, one ncu capture of the int2 draft kernel.
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/i2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/i2_tests.log; grep -E "^FAILED" gpurun_out/i2_tests.log | head
timeout 1500 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/i2_hbm_int2.json 2> gpurun_out/i2_hbm_int2.err; echo "int2 rc=$?"
timeout 1500 python bench.py --config 4 > gpurun_out/i2_config4.json 2> gpurun_out/i2_config4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --capped --x 16 --bits 2 --no-cpu > gpurun_out/i2_capped16_int2.json 2> gpurun_out/i2_capped16_int2.err; echo "capped2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:draft_attn_quant_kernel -c 1 -o gpurun_out/m_draft_int2 python tools/kbench.py --bits 2 --batch 12 --ctx 65536 --dense 0 > /dev/null 2>&1; echo "ncu int2 rc=$?"
