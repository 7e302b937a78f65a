# draft-kernel variant A/B without the suite (gpurun -- bash tools/gpu/qk_ab.sh): parity of the variants, then timings
for lib in tools/_trace/libvericache_*.so; do VC_LIB=$lib timeout 900 python -m pytest tests/test_attention_parity.py tests/test_real_shapes.py -m gpu -q -p no:cacheprovider -k draft 2>&1 | tail -1 | sed "s#^#$(basename $lib) parity #"; done
for r in 1 2; do
for lib in paper_2605_17613_b200/libvericache.so tools/_trace/libvericache_*.so; do
for b in 4 2; do VC_LIB=$lib timeout 600 python tools/kbench.py --bits $b --dense 0 2>&1 | tail -1 | sed "s#^#bits=$b #"; done
for m in "draft --x 6" "mixed --x 6"; do VC_LIB=$lib timeout 600 python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#$(basename $lib) $m #"; done
done; done
