# fused RMSNorm GEMM: bit identity + suites, then in-graph step times
timeout 1200 python -m pytest tests/test_gemm.py tests/test_lossless.py tests/test_model_parity.py tests/test_stream_ring.py tests/test_real_shapes.py tests/test_tp.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_fuse.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_fuse.log; grep -E "^(FAILED|E )" gpurun_out/t_fuse.log | head -20
for f in 0 1; do for m in draft mixed; do
VC_FUSE_NORM=$f timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/fuse=$f /"
done; done
