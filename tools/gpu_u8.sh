#!/bin/bash
for lib in libvericache.so libvc_u8.so; do
for m in "draft 1" "mixed 6" "mixed 47" "decode 1"; do set -- $m
  echo "$lib $1 x=$2 $(VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/profile_step.py --mode $1 --x $2 --steps 8 2>&1 | tail -1)"
done; done
