timeout 1500 python -m pytest tests/test_stream_ring.py tests/test_tier_placement.py tests/test_composition.py tests/test_lossless.py tests/test_drop_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_pack.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_pack.log; grep -E "^(FAILED|E )" gpurun_out/t_pack.log | head -20
timeout 1500 python bench.py > gpurun_out/f2_default.json 2> gpurun_out/f2_default.err; echo "default rc=$?"; tail -2 gpurun_out/f2_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/f2_default.json'))
print('headline', d['value'], d['e2e']['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['roofline']['frac'])
for k,t in d['tiers'].items(): print(k, t['value'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['step_roofline']['frac'], t['gpu_busy_frac'], t['tokens_identical_to_full_kv'], t.get('swap',{}).get('link_busy_frac'), t.get('swap',{}).get('h2d_gbs'))
print(d.get('knobs',{}).get('optimizer'))
PY
timeout 1500 python bench.py --capped --x 16 --no-cpu > gpurun_out/f2_capped16.json 2> gpurun_out/f2_capped16.err; echo "capped rc=$?"
python -c "import json; d=json.load(open('gpurun_out/f2_capped16.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement']['B_g_resident'], d['placement']['link_busy_frac'], d['tokens_identical_to_full_kv'])"
