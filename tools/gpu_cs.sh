#!/bin/bash
timeout 300 python tools/rms_hash.py; timeout 300 python tools/rms_hash.py --big
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in "draft 1" "mixed 6" "mixed 47" "decode 1"; do set -- $m
  echo "$1 x=$2 $(timeout 300 python tools/profile_step.py --mode $1 --x $2 --steps 8 2>&1 | tail -1)"
done
timeout 900 python bench.py --tier hbm --no-secondary --no-cpu > gpurun_out/hb.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/hb.json'));print('hbm', d['value'], d['full_kv_decode']['value'], d['speedup_vs_full_kv'], d['tokens_identical_to_full_kv'], d['roofline']['achieved'])"
