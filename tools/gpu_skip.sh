#!/bin/bash
for sk in 0 1 3; do
  for m in draft decode; do
    echo "VC_SKIP=$sk $(VC_SKIP=$sk timeout 300 python tools/profile_step.py --mode $m --x 1 --steps 8 2>&1 | tail -1)"
  done
done
