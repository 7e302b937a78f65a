# capacity-capped lines (gpurun -- bash tools/gpu/capped.sh)
timeout 1500 python bench.py --capped --x 16 --no-cpu > gpurun_out/c7_capped16.json 2> gpurun_out/c7_capped16.err; echo "capped rc=$?"
timeout 1500 python bench.py --capped --x 16 --bits 2 --no-cpu > gpurun_out/c7_capped16_int2.json 2> gpurun_out/c7_capped16_int2.err; echo "capped2 rc=$?"
