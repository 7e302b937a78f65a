timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -5
for m in "decode 16" "draft 16" "mixed 16" "mixed 96"; do set -- $m; timeout 300 python tools/profile_step.py --mode $1 --x $2 2>&1 | tail -1; done
timeout 300 python tools/kbench.py
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'], d['full_kv_decode'], d['tiers'], d['roofline']['achieved'])"; tail -2 gpurun_out/bench.err
