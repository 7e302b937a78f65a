#!/bin/bash
for x in 3 4 5; do
timeout 900 python bench.py --tier hbm --no-secondary --no-cpu --x $x > gpurun_out/hx$x.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/hx$x.json'));print('hbm x=$x', d['value'], d['full_kv_decode']['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['tokens_identical_to_full_kv'])"
done
for x in 2 3; do
timeout 900 python bench.py --config 4 --x $x > gpurun_out/rpx$x.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/rpx$x.json'));print('cfg4 x=$x', d['value'], d['full_kv']['value'], d['speedup_vs_full_kv'], d['vericache']['accepted_per_verify'], d['tokens_identical_to_full_kv'])"
done
