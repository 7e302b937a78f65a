# full GPU suite + smoke + default bench line
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/all_gpu.log; grep -E "^FAILED" gpurun_out/all_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_default.json'))
print('headline', d['value'], d['e2e']['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['roofline']['frac'], d['gpu_launches'])
for k,t in d['tiers'].items(): print(k, t['value'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['step_roofline']['frac'], t['gpu_busy_frac'], t['tokens_identical_to_full_kv'], t.get('swap',{}).get('staging_hbm_bytes'))
print(d.get('knobs',{}).get('optimizer'), d.get('knobs',{}).get('constants'), d.get('cpu_baseline',{}).get('value'))
PY
