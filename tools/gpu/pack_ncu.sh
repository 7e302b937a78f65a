# codec kernels (gpurun -- bash tools/gpu/pack_ncu.sh): the new overflow test, the codec alone, one ncu capture of each kernel
timeout 600 python -m pytest tests/test_stream_ring.py -m gpu -q -p no:cacheprovider -k pack > gpurun_out/pn_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pn_tests.log
timeout 300 python tools/pack_bench.py; echo "pack_bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|unpack_kernel" -c 2 -o gpurun_out/m_pack python tools/pack_bench.py > /dev/null 2>&1; echo "ncu rc=$?"
