# chained-alone cost of each GEMM family (VC_SKIP keeps one family + the LM head; diagnostics only)
for m in "draft --x 6" "mixed --x 6"; do
for sk in 121 113 105 89 57 1; do
VC_SKIP=$sk python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/skip=$sk $m /"
done; done
