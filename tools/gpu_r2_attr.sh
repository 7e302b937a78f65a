# in-graph attribution of a step's time (VC_SKIP diagnostics: wrong results, timing only)
for m in "decode" "draft --x 6" "mixed --x 6"; do
for sk in 0 4 8 16 32 64 120 1 2; do
VC_SKIP=$sk python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/skip=$sk $m /"
done; done
