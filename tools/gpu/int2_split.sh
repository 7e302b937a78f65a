# int2 bias variants (gpurun -- bash tools/gpu/int2_split.sh): default (bias MMA) vs tools/_trace/libvericache_split.so (per-lane sums)
VC_LIB=tools/_trace/libvericache_split.so timeout 900 python -m pytest tests/test_attention_parity.py tests/test_real_shapes.py -m gpu -q -p no:cacheprovider -k draft > gpurun_out/sp_tests.log 2>&1; echo "split parity rc=$?"; tail -1 gpurun_out/sp_tests.log
for r in 1 2 3; do for lib in paper_2605_17613_b200/libvericache.so tools/_trace/libvericache_split.so; do
VC_LIB=$lib timeout 600 python tools/kbench.py --bits 2 --dense 0 2>&1 | tail -1 | sed "s#^#int2 #"
done; done
