# validation of the combine / GEMM epilogue changes: full GPU suite, smoke, steps, phase trace
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_gpu3.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/all_gpu3.log; grep -E "^FAILED" gpurun_out/all_gpu3.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done
for m in decode draft mixed; do VC_LIB=tools/_trace/libvericache_trace.so python tools/gemm_trace.py --mode $m --out gpurun_out/gt_$m.bin 2>&1 | tail -7; done > gpurun_out/gemm_trace.txt; cat gpurun_out/gemm_trace.txt
