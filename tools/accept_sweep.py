"""Accepted drafted tokens per verify (lock-step run_speculative, x=30, int4,
32K ctx, Llama-3-8B shape) as a function of the synthetic init knobs
q_std:resid_std -- calibrates the synthetic model to the paper's reported
acceptance (~19-23 accepted of x=30).  Args: q_std:resid_std ..."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

B, X, K = 4, 30, 124
ctx = int(os.environ.get("CTX", "32768"))
e = vc.Engine(vc.LLAMA3_8B, max_slots=2 * B, max_ctx=ctx + K + 2 * X + 8, max_x=X, quant_bits=4, max_verify=B)
for pair in sys.argv[1:]:
    q_std, rs = (float(v) for v in pair.split(":"))
    e.init_weights(0, 0.02, resid_std=rs, q_std=q_std)
    for i in range(B):
        e.add_synthetic(i, ctx, 100 + 37 * i, seed=1 + i)
        e.add_synthetic(B + i, ctx, 100 + 37 * i, seed=1 + i)
        e.compress(B + i)
    base, _ = e.autoregress(list(range(B)), K)
    spec, rounds, _ = e.run_speculative(list(range(B, 2 * B)), K, X)
    acc = [n - 1 for r in rounds for n in r[:-1]]  # drafted tokens accepted per verify (last round truncated)
    print(f"q_std={q_std} resid_std={rs}: accepted/verify {np.mean(acc):.2f} (x={X}, {len(acc)} verifies), "
          f"lossless={bool((spec == base).all())}", flush=True)
