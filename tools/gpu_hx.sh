#!/bin/bash
for a in "5 0" "8 0" "6 32" "6 64" "7 0"; do set -- $a
timeout 900 python bench.py --tier hbm --no-secondary --no-cpu --x $1 --window $2 > gpurun_out/hx.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/hx.json'));print('x=$1 w=$2', d['value'], d['full_kv_decode']['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['config']['lookahead_window'], d['tokens_identical_to_full_kv'])"
done
