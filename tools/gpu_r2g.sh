python tools/draft_batch_probe.py
timeout 1200 python -m pytest tests/test_real_shapes.py tests/test_attention_parity.py tests/test_composition.py tests/test_tier_placement.py -m gpu -q -s -p no:cacheprovider > gpurun_out/t_g.log 2>&1; echo "tests rc=$?"; grep -E "MEASURED (draft|compos)|passed|failed|Error" gpurun_out/t_g.log | tail -40
