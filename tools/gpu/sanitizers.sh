# compute-sanitizer (racecheck, memcheck, synccheck) over tools/sanitize_smoke.py, then racecheck over the
# multi-item dense attention and GEMM tests (profiles/r02_compute_sanitizer.txt)
for t in racecheck memcheck synccheck; do
timeout 2400 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_smoke.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize smoke ok|Error" gpurun_out/san_$t.log | tail -3
done
timeout 1800 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_attention_parity.py -m gpu -q -p no:cacheprovider -k "mixed_widths or many_items" > gpurun_out/race_dense2.log 2>&1; echo "racecheck dense rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/race_dense2.log | tail -3
timeout 1800 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gemm.py -m gpu -q -p no:cacheprovider -x > gpurun_out/race_gemm.log 2>&1; echo "racecheck gemm rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/race_gemm.log | tail -3
