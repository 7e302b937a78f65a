# round 2 session A: full GPU suite, gamma(x) sweep, capacity-capped and default bench lines
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/all_gpu.log
timeout 1200 python tools/gamma_sweep.py --sensitivity --out gpurun_out/r02_gamma.json > gpurun_out/gamma.log 2>&1; echo "gamma rc=$?"; tail -40 gpurun_out/gamma.log
cp gpurun_out/r02_gamma.json profiles/r02_gamma.json 2>/dev/null
timeout 900 python bench.py --capped --no-cpu > gpurun_out/bench_capped4.json 2> gpurun_out/bench_capped4.err; echo "capped4 rc=$?"; cat gpurun_out/bench_capped4.json; tail -3 gpurun_out/bench_capped4.err
timeout 900 python bench.py --capped --bits 2 --no-cpu > gpurun_out/bench_capped2.json 2> gpurun_out/bench_capped2.err; echo "capped2 rc=$?"; cat gpurun_out/bench_capped2.json; tail -3 gpurun_out/bench_capped2.err
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
