# early epilogue operands: parity + step times + phase trace
timeout 1200 python -m pytest tests/test_gemm.py tests/test_lossless.py tests/test_model_parity.py tests/test_stream_ring.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_pre.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_pre.log
for r in 1 2; do
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done
done
for m in draft mixed; do VC_LIB=tools/_trace/libvericache_trace.so python tools/gemm_trace.py --mode $m --out gpurun_out/gt_$m.bin 2>&1 | tail -7; done
