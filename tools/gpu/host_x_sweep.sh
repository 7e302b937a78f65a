# Host-tier draft-horizon sweep (bench.py --tier host --x N)
for x in ${XS:-31 47 63 95}; do
timeout 1200 python bench.py --tier host --x $x --no-cpu --no-secondary > gpurun_out/hx_$x.json 2> gpurun_out/hx_$x.err; echo "x=$x rc=$?"
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/hx_$x.json') if l.startswith('{')][0])
t=d['tiers']['host']; print($x, t['value'], t['accepted_per_verify'], t['tokens_identical_to_full_kv'], t['gpu_busy_frac'], t['swap']['link_busy_frac'], t['ms_per_step'])
PY
done
