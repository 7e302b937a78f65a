# A/B on one box: round-2 start (ring only, build_ab/repo) vs current library
for root in paper_2605_17613_b200/build_ab/repo .; do for m in decode draft mixed; do
(cd $root && timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1 | sed "s|^|$root |")
done; done
