#!/bin/bash
for m in "draft 1" "mixed 6"; do set -- $m
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launch_g_$1.csv python tools/profile_step.py --mode $1 --x $2 --steps 1 > /dev/null 2>&1; echo "ncu $1 rc=$?"
done
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_umma -s 5 -c 4 -o gpurun_out/full_gemm_nt32 -f python tools/profile_step.py --mode mixed --x 6 --steps 1 > /dev/null 2>&1; echo "ncu full rc=$?"
