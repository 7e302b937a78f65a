#!/bin/bash
for x in 4 6 12; do
timeout 600 python bench.py --config 4 --x $x > gpurun_out/rp_x$x.json 2> gpurun_out/rp_x$x.err; echo "x=$x rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/rp_x$x.json").read().strip().splitlines()[-1])
print(d["value"], d["speedup_vs_full_kv"], d["tokens_identical_to_full_kv"], d["vericache"], d["full_kv"]["value"], d["roofline"]["achieved"])
PY
done
