for root in paper_2605_17613_b200/build_ab/r_8e3a389 paper_2605_17613_b200/build_ab/repo2 .; do
(cd $root && python tools/kbench.py 2>&1 | grep "kind=1\|kind=2 n=1" | sed "s|^|$root |")
done
