# A/B of the L2 evict-first policy: the default build vs a -DVC_L2_HINT=0 build at tools/_trace/libvericache_nohint.so
#   make -C paper_2605_17613_b200 -j8 OBJDIR=/tmp/nohint LIB=$PWD/tools/_trace/libvericache_nohint.so EXTRA=-DVC_L2_HINT=0
for r in 1 2; do
for lib in paper_2605_17613_b200/libvericache.so tools/_trace/libvericache_nohint.so; do
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do VC_LIB=$lib python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#$(basename $lib) $m #"; done
done; done
timeout 900 python -m pytest tests/test_gemm.py tests/test_attention_parity.py tests/test_lossless.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
