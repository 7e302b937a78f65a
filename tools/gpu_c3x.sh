#!/bin/bash
for x in 3 4 6 10; do
timeout 900 python bench.py --config 3 --no-cpu --x $x > gpurun_out/c3_x$x.json 2> gpurun_out/c3_x$x.err; echo "x=$x rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c3_x$x.json'));print(d['value'], d['full_kv_decode']['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['tokens_identical_to_full_kv'])"
done
