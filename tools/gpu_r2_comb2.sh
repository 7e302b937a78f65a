# combine with pre-wait metadata + fused-norm load reorder: parity + step times
timeout 1500 python -m pytest tests/test_attention_parity.py tests/test_gemm.py tests/test_lossless.py tests/test_model_parity.py tests/test_real_shapes.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_comb2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_comb2.log
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done
for m in "draft --x 6"; do VC_SKIP=4 python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/skip4 $m /"; done
