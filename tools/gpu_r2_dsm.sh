# DSMEM reduction with every rank's partial in flight: gemm tests + step times
timeout 900 python -m pytest tests/test_gemm.py tests/test_lossless.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_dsm.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_dsm.log
for r in 1 2; do
for m in "decode" "draft --x 6" "mixed --x 6" "mixed --x 16"; do python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/$m /"; done
done
for c in 3 4; do for m in "draft --x 6" "mixed --x 6"; do VC_GEMM_CLUSTER=$c python tools/profile_step.py --mode $m --steps 8 2>&1 | tail -1 | sed "s/^/cap$c $m /"; done; done
