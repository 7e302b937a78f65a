# A/B of the host-pool packing formats on one box (gpurun -- bash tools/gpu/pack_ab.sh):
# the default build vs tools/_trace/libvericache_pk76.so (the previous 4-bit-offset format), host tier only
for r in 1 2; do
for lib in paper_2605_17613_b200/libvericache.so tools/_trace/libvericache_pk76.so; do
VC_LIB=$lib timeout 900 python bench.py --tier host --no-cpu --no-secondary > gpurun_out/pab_$r_$(basename $lib .so).json 2>/dev/null
python - "$lib" <<PY
import json,sys
d=json.loads([l for l in open('gpurun_out/pab_$r_$(basename $lib .so).json') if l.startswith('{')][-1])
h=d['tiers']['host']; s=h['swap']; r=h['step_roofline']
print(sys.argv[1].split('/')[-1], d['value'], h['accepted_per_verify'], d['tokens_identical_to_full_kv'], 'h2d', s['h2d_gbs'], 'busy', s['link_busy_frac'], 'ratio', s['reload_bytes_over_full_kv'], 'ms/it', r['ms_per_iteration'], 'verifies', r['verifies'], 'gpu_busy', h['gpu_busy_frac'])
PY
done; done
