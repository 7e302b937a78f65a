#!/bin/bash
timeout 900 python -m pytest tests/test_attention_parity.py tests/test_lossless.py tests/test_ragged_batch.py tests/test_remote_prefix.py tests/test_tp.py -x -q 2>&1 | tail -4
timeout 300 python tools/kbench.py --bits 2 --dense 0
timeout 300 python tools/kbench.py --bits 2 --dense 0 --batch 12 --ctx 65536
timeout 300 python tools/kbench.py --bits 4 --dense 0
