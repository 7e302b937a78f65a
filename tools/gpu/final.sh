# Final measurement pass (run from the repo root on a GPU box: gpurun -- bash tools/gpu/final.sh):
# full GPU suite, smoke, every bench line, launch lists,
# in-graph step times, ncu --set full of the step's top kernels. Outputs land in gpurun_out/ (k_*.json, m_*.ncu-rep).
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu4.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/all_gpu4.log; grep -E "^FAILED" gpurun_out/all_gpu4.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke4.log
timeout 1500 python bench.py > gpurun_out/k_default.json 2> gpurun_out/k_default.err; echo "default rc=$?"
timeout 1500 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/k_hbm_int2.json 2> gpurun_out/k_hbm_int2.err; echo "int2 rc=$?"
timeout 1500 python bench.py --capped --x 16 --no-cpu > gpurun_out/k_capped16.json 2> gpurun_out/k_capped16.err; echo "capped rc=$?"
timeout 1500 python bench.py --capped --x 16 --bits 2 --no-cpu > gpurun_out/k_capped16_int2.json 2> gpurun_out/k_capped16_int2.err; echo "capped2 rc=$?"
timeout 1500 python bench.py --config 3 > gpurun_out/k_config3.json 2> gpurun_out/k_config3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config 4 > gpurun_out/k_config4.json 2> gpurun_out/k_config4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --config 5 --no-cpu > gpurun_out/k_config5.json 2> gpurun_out/k_config5.err; echo "c5 rc=$?"
for qr in "0.004 0.0004" "0.008 0.001" "0.02 0.002"; do set -- $qr
timeout 900 python bench.py --tier hbm --no-cpu --no-secondary --q-std $1 --resid-std $2 > gpurun_out/k_sens_$1.json 2> gpurun_out/k_sens_$1.err; echo "sens $1 rc=$?"
done
for m in decode draft mixed; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_launch_$m.csv python tools/profile_step.py --mode $m --x 6 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/k_launch_$m.csv $m > gpurun_out/k_launch_$m.txt; done
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done > gpurun_out/k_steps.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:draft_attn_quant_kernel -c 1 -o gpurun_out/m_draft python tools/profile_step.py --mode draft --x 6 --steps 1 > /dev/null 2>&1; echo "ncu draft rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:dense_umma_kernel -c 1 -o gpurun_out/m_dense python tools/profile_step.py --mode mixed --x 6 --steps 1 > /dev/null 2>&1; echo "ncu dense rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:dense_umma_kernel -c 1 -o gpurun_out/m_dense47 python tools/profile_step.py --mode mixed --x 47 --steps 1 > /dev/null 2>&1; echo "ncu dense47 rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_cluster_kernel -c 4 -o gpurun_out/m_gemm python tools/profile_step.py --mode mixed --x 6 --steps 1 > /dev/null 2>&1; echo "ncu gemm rc=$?"
