# dense kernel with two softmax column groups: parity + A/B timing
timeout 1200 python -m pytest tests/test_attention_parity.py tests/test_real_shapes.py tests/test_lossless.py tests/test_stream_ring.py tests/test_drop_parity.py tests/test_snapkv.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_sg.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_sg.log; grep -E "^(FAILED|E )" gpurun_out/t_sg.log | head; grep "MEASURED dense" gpurun_out/t_sg.log | head -3
for i in 1 2; do for root in paper_2605_17613_b200/build_ab/base .; do
(cd $root && for m in "mixed --x 6" "mixed --x 16" "decode"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s|^|$root $m |"; done; python tools/kbench.py 2>&1 | grep "kind=[12]" | sed "s|^|$root |")
done; done
