# one pytest -m gpu pass + ncu --set full captures of the top kernels (single GPU)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for k in draft_attn_quant_kernel:draft gemm_tma_kernel:draft dense_umma_kernel:decode dense_umma_kernel:mixed; do
  name=${k%%:*}; mode=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s 3 -c 1 \
    -o gpurun_out/full_${name}_${mode} -f python tools/profile_step.py --mode $mode > gpurun_out/ncu_${name}_${mode}.log 2>&1
  echo "ncu $name $mode rc=$?"
done
