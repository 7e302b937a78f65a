#!/bin/bash
for f in 0 1; do VC_FUSE_RMS=$f timeout 300 python tools/rms_hash.py; VC_FUSE_RMS=$f timeout 300 python tools/rms_hash.py --big; done
timeout 900 python -m pytest tests/test_model_parity.py tests/test_gemm.py tests/test_lossless.py tests/test_tp.py tests/test_ragged_batch.py -x -q 2>&1 | tail -3
for f in 0 1; do for m in draft decode mixed; do echo "FUSE=$f $(VC_FUSE_RMS=$f timeout 300 python tools/profile_step.py --mode $m --x 6 --steps 8 2>&1 | tail -1)"; done; done
