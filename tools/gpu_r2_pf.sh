timeout 1200 python -m pytest tests/test_attention_parity.py tests/test_lossless.py tests/test_stream_ring.py tests/test_drop_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_pf.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_pf.log
for m in decode draft mixed; do timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1; done
