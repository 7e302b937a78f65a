#!/bin/bash
for sk in 0 1; do
  for x in 6 16 40; do
    echo "VC_SKIP=$sk x=$x $(VC_SKIP=$sk timeout 300 python tools/profile_step.py --mode mixed --x $x --steps 8 2>&1 | tail -1)"
  done
done
