# in-graph step breakdown (VC_SKIP: 1 = no attention+combine, 2 = no rms) + attention kernels alone + capped line on the ring
for m in draft mixed; do for sk in 0 1 3; do
VC_SKIP=$sk timeout 600 python tools/profile_step.py --mode $m --steps 6 --x 6 2>&1 | tail -1 | sed "s/^/skip=$sk /"
done; done
timeout 600 python tools/kbench.py 2>&1 | tail -4
timeout 1500 python bench.py --capped --no-cpu > gpurun_out/bench_capped_ring.json 2> gpurun_out/bench_capped_ring.err; echo "capped rc=$?"; tail -2 gpurun_out/bench_capped_ring.err
python -c "import json; d=json.load(open('gpurun_out/bench_capped_ring.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement'], d['tokens_identical_to_full_kv'])"
