#!/bin/bash
for lib in libvericache.so libvc_t12.so libvc_t4.so; do
  VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/kbench.py --bits 4 --dense 1 2>&1 | grep -v "kind=0"
  for m in "mixed 6" "decode 1"; do set -- $m
    echo "$lib $1 x=$2 $(VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/profile_step.py --mode $1 --x $2 --steps 8 2>&1 | tail -1)"
  done
done
