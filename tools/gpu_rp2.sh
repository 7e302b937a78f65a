#!/bin/bash
timeout 600 python -m pytest tests/test_remote_prefix.py -x -q 2>&1 | tail -3
for po in 0 1; do
timeout 600 python bench.py --config 4 --payload-order $po > gpurun_out/rp_po$po.json 2> gpurun_out/rp_po$po.err; echo "po=$po rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/rp_po$po.json").read().strip().splitlines()[-1])
print(d["value"], d["speedup_vs_full_kv"], d["tokens_identical_to_full_kv"], d["vericache"], d["full_kv"])
PY
done
