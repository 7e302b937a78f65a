# A/B of draft-kernel variants (gpurun -- bash tools/gpu/draft_ab.sh): the default build vs the
# variants under tools/_trace/ (built with EXTRA=-D... into tools/_trace/libvericache_<tag>.so).
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
for r in 1 2; do
for lib in paper_2605_17613_b200/libvericache.so tools/_trace/libvericache_*.so; do
for b in 4 2; do VC_LIB=$lib timeout 600 python tools/kbench.py --bits $b --dense 0 2>&1 | tail -1 | sed "s#^#bits=$b #"; done
for m in "draft --x 6" "mixed --x 6"; do VC_LIB=$lib timeout 600 python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#$(basename $lib) $m #"; done
done; done
