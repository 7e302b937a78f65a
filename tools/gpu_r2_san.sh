# compute-sanitizer over the extended smoke (round-2 code paths)
for t in racecheck memcheck synccheck; do
timeout 2400 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_smoke.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize smoke ok|Error" gpurun_out/san_$t.log | tail -3
done
timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/host_chk.json 2> gpurun_out/host_chk.err; echo "host rc=$?"
python -c "import json; d=json.load(open('gpurun_out/host_chk.json')); t=d['tiers']['host']; print(t['value'], t['accepted_per_verify'], t['swap'], t['tokens_identical_to_full_kv'])"
