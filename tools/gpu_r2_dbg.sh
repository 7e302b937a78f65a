timeout 900 python -m pytest tests/test_attention_parity.py tests/test_real_shapes.py tests/test_lossless.py tests/test_stream_ring.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_dbg.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_dbg.log; grep -E "^(FAILED|E )" gpurun_out/t_dbg.log | head -8
for i in 1 2; do
timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/rep_$i.json 2> gpurun_out/rep_$i.err
python -c "import json; d=json.load(open('gpurun_out/rep_$i.json')); t=d['tiers']['host']; print('run $i', t['value'], t['accepted_per_verify'], t['tokens_identical_to_full_kv'], t['tokens_compared'])"
done
