#!/bin/bash
for lib in libvericache.so libvc_ks.so; do
  for b in 4 2; do
    VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/kbench.py --bits $b --dense 0
  done
  VC_LIB=paper_2605_17613_b200/$lib timeout 300 python tools/kbench.py --bits 2 --dense 0 --batch 12 --ctx 65536
done
VC_LIB=paper_2605_17613_b200/libvc_ks.so timeout 600 python -m pytest tests/test_attention_parity.py tests/test_lossless.py -x -q 2>&1 | tail -2
