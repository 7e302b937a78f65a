timeout 900 python -m pytest tests/test_tier_placement.py tests/test_lossless.py -m gpu -q -p no:cacheprovider > gpurun_out/t_i.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_i.log; grep -E "^FAILED" gpurun_out/t_i.log | head
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json'))
print('headline', d['value'], d['e2e']['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])
for k,t in d['tiers'].items(): print(k, t['value'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['step_roofline']['frac'], t['gpu_busy_frac'], t['tokens_identical_to_full_kv'])
print(d.get('knobs',{}).get('optimizer'))"
timeout 900 python bench.py --capped --x 16 --no-cpu > gpurun_out/bench_capped4.json 2> gpurun_out/bench_capped4.err; echo "capped rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_capped4.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement'], d['step_roofline']['frac'], d['tokens_identical_to_full_kv'])"
