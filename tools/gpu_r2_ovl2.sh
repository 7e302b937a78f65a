for gd in off 0 20 28 36; do
if [ $gd = off ]; then e="VC_OVERLAP=0"; else e="VC_OVERLAP_GD=$gd"; fi
env $e VC_ATTN_TRACE=1 timeout 600 python tools/profile_step.py --mode mixed --steps 3 --x 6 --graphs 0 2>&1 | grep -E "ATTN" | tail -1 | sed "s/^/$gd /"
env $e timeout 600 python tools/profile_step.py --mode mixed --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/$gd x6 /"
env $e timeout 600 python tools/profile_step.py --mode mixed --steps 8 --x 16 2>&1 | tail -1 | sed "s/^/$gd x16 /"
done
