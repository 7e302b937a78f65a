# verify/draft overlap: correctness (scheduled loops have mixed steps), then in-graph step times vs G_d
timeout 900 python -m pytest tests/test_lossless.py tests/test_tier_placement.py tests/test_stream_ring.py tests/test_attention_parity.py tests/test_real_shapes.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_ovl.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ovl.log; grep -E "^(FAILED|E )" gpurun_out/t_ovl.log | head -20
for x in 6 16; do
VC_OVERLAP=0 timeout 600 python tools/profile_step.py --mode mixed --steps 8 --x $x 2>&1 | tail -1 | sed "s/^/x=$x off /"
for gd in 0 16 24 32 48; do
VC_OVERLAP_GD=$gd timeout 600 python tools/profile_step.py --mode mixed --steps 8 --x $x 2>&1 | tail -1 | sed "s/^/x=$x gd=$gd /"
done; done
