timeout 900 python -m pytest tests/test_real_shapes.py -k batched tests/test_tier_placement.py tests/test_lossless.py -m gpu -q -s -p no:cacheprovider > gpurun_out/t_c.log 2>&1; echo "tests rc=$?"; grep -E "MEASURED|passed|failed|Error" gpurun_out/t_c.log | tail
timeout 900 python bench.py --capped --no-cpu --steps 6 --warmup 3 > gpurun_out/cap4.json 2> gpurun_out/cap4.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/cap4.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement'], d['step_roofline'])"
timeout 900 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/hbm2.json 2> gpurun_out/hbm2.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/hbm2.json')); print(d['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['tiers']['hbm']['step_roofline'], d['roofline'])"
