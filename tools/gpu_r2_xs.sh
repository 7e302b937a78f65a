# HBM-tier draft horizon sweep on the final kernels
for x in 4 5 6 7 8 10; do
timeout 900 python bench.py --tier hbm --no-cpu --no-secondary --x $x > gpurun_out/xs_$x.json 2> gpurun_out/xs_$x.err
python -c "import json,sys; d=json.load(open('gpurun_out/xs_$x.json')); print('x=$x', d['value'], d['speedup_vs_full_kv'], d['accepted_per_verify'], d['tiers']['hbm']['step_roofline']['frac'], d['tokens_identical_to_full_kv'])"
done
