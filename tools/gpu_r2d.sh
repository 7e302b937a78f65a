timeout 900 python -m pytest tests/test_tier_placement.py tests/test_lossless.py tests/test_remote_prefix.py tests/test_ref_boundary.py -m gpu -q -p no:cacheprovider > gpurun_out/t_d.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_d.log
VC_STEP_LOG=1 timeout 900 python bench.py --capped --no-cpu --steps 6 --warmup 3 > gpurun_out/cap4.json 2> gpurun_out/cap4.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/cap4.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement'], d['step_roofline'])"
grep STEP gpurun_out/cap4.err | tail -300 | python -c "
import sys,collections
d=collections.defaultdict(list)
for l in sys.stdin:
    f=dict(kv.split('=') for kv in l.split()[1:])
    d[(f['Mb'],f['verify'],f['rows_v'])].append(float(f['ms']))
for k,v in sorted(d.items(), key=lambda t:-len(t[1]))[:12]: print(k, len(v), round(sum(v)/len(v),3), round(max(v),2))
"
timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/host.json 2> gpurun_out/host.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/host.json')); print(d['value'], d['speedup_vs_full_kv'], d['tiers']['host']['gpu_busy_frac'], d['tiers']['host']['swap'], d['tiers']['host']['step_roofline'])"
