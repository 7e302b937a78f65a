"""Repro harness for the baseline-decode part of bench.py (torch context + engine)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_17613_b200 as vc  # noqa: E402

B, ctx, K1, K2 = (int(v) for v in sys.argv[1:5])
torch.cuda.set_device(0)
for trial in range(int(os.environ.get("TRIALS", "1"))):
    eb = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=ctx + K1 + K2 + 8, max_x=1, quant_bits=0, max_verify=1)
    eb.init_weights(seed=0, std=0.02, resid_std=0.0002, q_std=0.002)
    for i in range(B):
        eb.add_synthetic(i, ctx, 100 + i, seed=1 + i)
    t, _ = eb.autoregress(list(range(B)), K1)
    eb.timing(reset=True)
    torch.cuda.synchronize()
    try:
        t, _ = eb.autoregress(list(range(B)), K2)
        print(trial, "ok", flush=True)
    except Exception as ex:
        print(trial, "FAILED", ex, flush=True)
    eb.close()
    del eb
    torch.cuda.empty_cache()
