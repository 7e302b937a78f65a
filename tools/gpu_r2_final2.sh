# round-2 final measurement pass on the final code
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python bench.py > gpurun_out/g_default.json 2> gpurun_out/g_default.err; echo "default rc=$?"
timeout 1500 python bench.py --tier hbm --bits 2 --no-cpu --no-secondary > gpurun_out/g_hbm_int2.json 2> gpurun_out/g_hbm_int2.err; echo "int2 rc=$?"
timeout 1500 python bench.py --capped --x 16 --no-cpu > gpurun_out/g_capped16.json 2> gpurun_out/g_capped16.err; echo "capped rc=$?"
timeout 1500 python bench.py --capped --x 16 --bits 2 --no-cpu > gpurun_out/g_capped16_int2.json 2> gpurun_out/g_capped16_int2.err; echo "capped2 rc=$?"
timeout 1500 python bench.py --config 3 > gpurun_out/g_config3.json 2> gpurun_out/g_config3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config 4 > gpurun_out/g_config4.json 2> gpurun_out/g_config4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --config 5 --no-cpu > gpurun_out/g_config5.json 2> gpurun_out/g_config5.err; echo "c5 rc=$?"
for qr in "0.004 0.0004" "0.008 0.001" "0.02 0.002"; do set -- $qr
timeout 900 python bench.py --tier hbm --no-cpu --no-secondary --q-std $1 --resid-std $2 > gpurun_out/g_sens_$1.json 2> gpurun_out/g_sens_$1.err; echo "sens $1 rc=$?"
done
for m in decode draft mixed; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launch_$m.csv python tools/profile_step.py --mode $m --x 6 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/g_launch_$m.csv $m > gpurun_out/g_launch_$m.txt; done
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done > gpurun_out/g_steps.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:draft_attn_quant_kernel -c 1 -o gpurun_out/h_draft python tools/profile_step.py --mode draft --x 6 --steps 1 > /dev/null 2>&1; echo "ncu draft rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:dense_umma_kernel -c 1 -o gpurun_out/h_dense python tools/profile_step.py --mode mixed --x 6 --steps 1 > /dev/null 2>&1; echo "ncu dense rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_cluster_kernel -c 4 -o gpurun_out/h_gemm python tools/profile_step.py --mode mixed --x 6 --steps 1 > /dev/null 2>&1; echo "ncu gemm rc=$?"
