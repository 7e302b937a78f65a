# int2 HBM-tier horizon sweep (gpurun -- bash tools/gpu/int2_x.sh)
for x in 7 9 11; do
timeout 900 python bench.py --tier hbm --bits 2 --x $x --no-cpu --no-secondary > gpurun_out/i2x_$x.json 2>/dev/null; echo "x=$x rc=$?"
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/i2x_$x.json') if l.startswith('{')][-1])
t=d['tiers']['hbm']; print($x, t['value'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['tokens_identical_to_full_kv'], t['step_roofline']['ms_per_iteration'])
PY
done
