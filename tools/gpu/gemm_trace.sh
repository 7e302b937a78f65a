# GEMM phase timeline: the -DVC_GEMM_TRACE build, then tools/gemm_trace.py per step kind (profiles/r02_gemm_phase_trace.txt)
make -C paper_2605_17613_b200 -j8 OBJDIR=/tmp/trbuild LIB=$PWD/tools/_trace/libvericache_trace.so EXTRA=-DVC_GEMM_TRACE > /dev/null
for m in decode draft mixed; do VC_LIB=tools/_trace/libvericache_trace.so python tools/gemm_trace.py --mode $m --out gpurun_out/gt_$m.bin 2>&1 | tail -7; done
