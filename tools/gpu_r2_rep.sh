# reproduce the host-tier losslessness failure
for i in 1 2 3; do
timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/rep_$i.json 2> gpurun_out/rep_$i.err
python -c "import json; d=json.load(open('gpurun_out/rep_$i.json')); t=d['tiers']['host']; print('run $i', t['value'], t['accepted_per_verify'], t['tokens_identical_to_full_kv'], t['tokens_compared'])"
done
timeout 900 python bench.py --no-cpu --no-secondary --ring 0 > gpurun_out/rep_r0.json 2> gpurun_out/rep_r0.err
python -c "import json; d=json.load(open('gpurun_out/rep_r0.json')); t=d['tiers']['host']; print('ring0', t['value'], t['accepted_per_verify'], t['tokens_identical_to_full_kv'])"
