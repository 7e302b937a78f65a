# bisect the decode-step regression
for e in "X=1" "VC_FUSE_NORM=0" "VC_FUSE_NORM=0 VC_GEMM_CLUSTER_MIN=3" "VC_FUSE_NORM=0 VC_GEMM_CLUSTER_MIN=9"; do
env $e timeout 600 python tools/profile_step.py --mode decode --steps 8 2>&1 | tail -1 | sed "s|^|$e |"
env $e VC_SKIP=1 timeout 600 python tools/profile_step.py --mode decode --steps 8 2>&1 | tail -1 | sed "s|^|$e noattn |"
done
(cd paper_2605_17613_b200/build_ab/repo && VC_SKIP=1 timeout 600 python tools/profile_step.py --mode decode --steps 8 2>&1 | tail -1 | sed "s|^|old noattn |")
python tools/kbench.py 2>&1 | tail -4
(cd paper_2605_17613_b200/build_ab/repo && cp ../../../tools/kbench.py tools/ && python tools/kbench.py 2>&1 | tail -4 | sed "s|^|old |")
