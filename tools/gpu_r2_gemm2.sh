# cluster size sweep (in-graph step times)
for c in 2 3 4 5 6; do for m in draft mixed; do
VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/cluster=$c /"
done; 
VC_SKIP=3 VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode mixed --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/cluster=$c gemm-only /"
done
