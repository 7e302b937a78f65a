# SnapKV drop-topk: parity tests, then configs[2] lines (SnapKV vs L1 key norm)
timeout 900 python -m pytest tests/test_snapkv.py tests/test_drop_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_snap.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_snap.log; grep -E "^(FAILED|E )" gpurun_out/t_snap.log | head -20
for sc in snapkv norm; do
timeout 1500 python bench.py --config 3 --drop-score $sc > gpurun_out/bench_c3_$sc.json 2> gpurun_out/bench_c3_$sc.err; echo "c3 $sc rc=$?"; tail -2 gpurun_out/bench_c3_$sc.err
python - gpurun_out/bench_c3_$sc.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['accepted_per_verify'], d['tokens_identical_to_full_kv'], d['config']['draft_x'])
lh=d.get('long_horizon')
if lh: print('long', lh['value'], lh['speedup_vs_full_kv'], lh['accepted_per_verify'], lh['draft_x'], lh['tokens_identical_to_full_kv'])
print('cpu', d.get('cpu_baseline',{}) and d['cpu_baseline'].get('value'))
PY
done
