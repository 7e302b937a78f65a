# In-graph attribution of a step's time by removal (VC_SKIP diagnostics: results wrong, timing only).
# Part 1 removes one family; part 2 keeps one GEMM family (+ LM head) to time it chained alone.
for m in "decode" "draft --x 6" "mixed --x 6"; do
for sk in 0 4 8 16 32 64 120 1 2; do
VC_SKIP=$sk python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/skip=$sk $m /"
done; done
for m in "draft --x 6" "mixed --x 6"; do
for sk in 121 113 105 89 57 1; do
VC_SKIP=$sk python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/skip=$sk $m /"
done; done
