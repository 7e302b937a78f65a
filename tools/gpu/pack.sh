# host-pool packing pass (gpurun -- bash tools/gpu/pack.sh): round trip + streamed-verify tests first, then the suite and the default bench line
timeout 900 python -m pytest tests/test_stream_ring.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pk_ring.log 2>&1; echo "ring tests rc=$?"; tail -3 gpurun_out/pk_ring.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pk_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pk_tests.log; grep -E "^FAILED" gpurun_out/pk_tests.log | head
timeout 900 python bench.py > gpurun_out/pk_default.json 2> gpurun_out/pk_default.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/pk_default.json
