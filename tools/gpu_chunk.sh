#!/bin/bash
for lib in libvericache.so libvc_k1.so libvc_k5.so; do
  for m in "mixed 6" "decode 1"; do set -- $m
    echo "$lib $1 x=$2 $(VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/profile_step.py --mode $1 --x $2 --steps 8 2>&1 | tail -1)"
  done
  VC_LIB=paper_2605_17613_b200/$lib timeout 600 python bench.py --tier hbm --no-secondary --no-cpu > gpurun_out/chunk_$lib.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/chunk_$lib.json'));print('$lib', d['value'], d['full_kv_decode']['value'], d['speedup_vs_full_kv'], d['tokens_identical_to_full_kv'])"
done
