# cluster split-K GEMM: correctness, then in-graph step times vs stream-K (VC_GEMM_CLUSTER=1)
timeout 900 python -m pytest tests/test_gemm.py tests/test_lossless.py tests/test_model_parity.py tests/test_stream_ring.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gemm.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gemm.log; grep -E "^(FAILED|E )" gpurun_out/t_gemm.log | head -20
for c in 8 1 4; do for m in draft mixed; do
VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode $m --steps 6 --x 6 2>&1 | tail -1 | sed "s/^/cluster=$c /"
VC_SKIP=3 VC_GEMM_CLUSTER=$c timeout 600 python tools/profile_step.py --mode $m --steps 6 --x 6 2>&1 | tail -1 | sed "s/^/cluster=$c gemm-only /"
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_mixed_cl.csv python tools/profile_step.py --mode mixed --x 6 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launch_mixed_cl.csv mixed-cluster
