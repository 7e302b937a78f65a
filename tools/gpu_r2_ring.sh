# ring-mode host tier: new tests, then host-tier bench lines (chunk ring vs whole-request staging)
timeout 900 python -m pytest tests/test_stream_ring.py tests/test_tier_placement.py tests/test_lossless.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_ring.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_ring.log; grep -E "^(FAILED|E )" gpurun_out/t_ring.log | head -20
for cfg in "--ring 8 --streams 2" "--ring 8 --streams 3" "--ring 16 --streams 3" "--ring 0"; do
tag=$(echo $cfg | tr -d ' -')
timeout 1200 python bench.py --no-cpu --no-secondary $cfg > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench $cfg rc=$?"; tail -2 gpurun_out/bench_$tag.err
python - gpurun_out/bench_$tag.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
t=d['tiers']['host']
print('host', t['value'], t['e2e'], t['speedup_vs_full_kv'], t['accepted_per_verify'], t['gpu_busy_frac'], t['tokens_identical_to_full_kv'])
print(t['swap'])
PY
done
