# Attention-combine diagnostics: phase trace (-DVC_COMBINE_TRACE build), and in-graph step times with the combine
# as built, as a no-op after its PDL wait (-DVC_COMBINE_NOOP build) and not launched (VC_SKIP=4).
make -C paper_2605_17613_b200 -j8 OBJDIR=/tmp/ctr LIB=$PWD/tools/_trace/libvericache_ctrace.so EXTRA=-DVC_COMBINE_TRACE > /dev/null
make -C paper_2605_17613_b200 -j8 OBJDIR=/tmp/cnoop LIB=$PWD/tools/_trace/libvericache_cnoop.so EXTRA=-DVC_COMBINE_NOOP > /dev/null
for m in decode draft mixed; do VC_LIB=tools/_trace/libvericache_ctrace.so python tools/comb_trace.py --mode $m 2>&1 | tail -2; done
for r in 1 2; do
for m in "decode" "draft --x 6" "mixed --x 6"; do
python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#full $m #"
VC_LIB=tools/_trace/libvericache_cnoop.so python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#noop $m #"
VC_SKIP=4 python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s#^#skip $m #"
done; done
