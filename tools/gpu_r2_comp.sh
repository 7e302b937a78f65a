# composition report at the 8B shape + the int2 capacity-capped line
K=96 timeout 1500 python tools/ngram_bench.py > gpurun_out/ngram_bench.log 2>&1; echo "ngram rc=$?"; tail -8 gpurun_out/ngram_bench.log
timeout 1500 python bench.py --capped --x 16 --bits 2 --no-cpu > gpurun_out/f_capped16_int2.json 2> gpurun_out/f_capped16_int2.err; echo "capped2 rc=$?"; tail -2 gpurun_out/f_capped16_int2.err
python -c "import json; d=json.load(open('gpurun_out/f_capped16_int2.json')); print(d['value'], d['speedup_vs_full_kv'], d['full_kv_decode']['value'], d['placement']['B_g_resident'], d['tokens_identical_to_full_kv'])"
