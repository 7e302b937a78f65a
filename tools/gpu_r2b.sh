# capped-regime diagnosis: per-step shapes and device times
VC_STEP_LOG=1 timeout 900 python bench.py --capped --no-cpu --steps 4 --warmup 3 > gpurun_out/cap_diag.json 2> gpurun_out/cap_diag.err; echo "rc=$?"
cat gpurun_out/cap_diag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['speedup_vs_full_kv'], d['placement'], d['step_roofline'])"
grep STEP gpurun_out/cap_diag.err | tail -400 | awk '{print $2, $3, $4, $5, $6, $7, $8}' | sort | uniq -c | sort -rn | head -40
grep STEP gpurun_out/cap_diag.err | tail -400 | python -c "
import sys,collections
d=collections.defaultdict(list)
for l in sys.stdin:
    f=dict(kv.split('=') for kv in l.split()[1:])
    d[(f['Mb'],f['verify'],f['rows_v'])].append(float(f['ms']))
for k,v in sorted(d.items(), key=lambda t:-len(t[1]))[:30]: print(k, len(v), round(sum(v)/len(v),3))
"
