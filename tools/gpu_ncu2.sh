#!/bin/bash
# ncu --set full of the int2 draft attention at the configs[3] shape (12 x 64K)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:draft_attn_quant -s 40 -c 1 \
  -o gpurun_out/full_draft_int2 -f python tools/kbench.py --bits 2 --dense 0 --batch 12 --ctx 65536 > gpurun_out/ncu_int2.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_int2.log
