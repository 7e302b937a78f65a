#!/bin/bash
# remote-prefix (configs[3]) tests + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_remote_prefix.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --config 4 --small > gpurun_out/rp_small.json 2> gpurun_out/rp_small.err; echo "small rc=$?"; tail -c 1500 gpurun_out/rp_small.json; tail -5 gpurun_out/rp_small.err
timeout 900 python bench.py --config 4 > gpurun_out/rp.json 2> gpurun_out/rp.err; echo "full rc=$?"; cat gpurun_out/rp.json; tail -5 gpurun_out/rp.err
