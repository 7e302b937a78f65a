# capped-regime knob sweep: offloaded x, resident x, bits (short windows)
for cfg in "--x 47 --x-res 6" "--x 24 --x-res 6" "--x 16 --x-res 6" "--x 47 --x-res 8" "--x 24 --x-res 6 --bits 2" "--x 47 --x-res 6 --bits 2"; do
  timeout 900 python bench.py --capped --no-cpu --steps 4 --warmup 3 $cfg > gpurun_out/cap_sweep.json 2> gpurun_out/cap_sweep.err
  python -c "import json,sys; d=json.load(open('gpurun_out/cap_sweep.json')); p=d['placement']; print(sys.argv[1], d['value'], d['speedup_vs_full_kv'], p['B_g_resident'], p['resident_accepted_per_verify'], p['accepted_per_verify'], p['link_busy_frac'], d['step_roofline']['ms_per_iteration'])" "$cfg"
done
