# auto cluster size vs uniform 5
for c in 0 5; do for m in draft mixed; do
VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/cluster=$c /"
VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 16 2>&1 | tail -1 | sed "s/^/cluster=$c x16 /"
done; done
