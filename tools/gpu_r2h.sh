timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/all_gpu.log; grep -E "^FAILED" gpurun_out/all_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json'))
print('headline', d['value'], d['e2e']['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['roofline']['frac'])
for k,t in d['tiers'].items(): print(k, t['value'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['step_roofline']['frac'], t['gpu_busy_frac'], t['tokens_identical_to_full_kv'])
print(d.get('knobs',{}).get('optimizer'))"
timeout 900 python bench.py --capped --x 16 --no-cpu > gpurun_out/bench_capped4.json 2> gpurun_out/bench_capped4.err; echo "capped rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_capped4.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement'], d['step_roofline']['frac'], d['tokens_identical_to_full_kv'])"
timeout 900 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/hbm2.json 2> gpurun_out/hbm2.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/hbm2.json')); print(d['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['tiers']['hbm']['step_roofline'], d['roofline']['frac'])"
