#!/bin/bash
VC_LIB=paper_2605_17613_b200/libvc_f1.so timeout 300 python tools/rms_hash.py --big
VC_LIB=paper_2605_17613_b200/libvc_f1.so timeout 900 python -m pytest tests/test_gemm.py tests/test_lossless.py -x -q 2>&1 | tail -1
for lib in libvericache.so libvc_f1.so libvericache.so libvc_f1.so; do
for m in "draft 1" "mixed 6"; do set -- $m
  echo "$lib $1 x=$2 $(VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/profile_step.py --mode $1 --x $2 --steps 8 2>&1 | tail -1)"
done; done
