"""Draft (int4 KV) vs full-KV top-1 agreement at 8B shape as a function of the
synthetic init (Q-projection std = attention temperature, residual-branch
std = depth-wise perturbation growth) -- calibrates the synthetic model's
acceptance.  Args: q_std:resid_std pairs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

shape = vc.LLAMA3_8B
ctx = int(os.environ.get("CTX", "32768"))
trials = int(os.environ.get("TRIALS", "12"))
e = vc.Engine(shape, max_slots=2, max_ctx=ctx + 64, max_x=8, quant_bits=int(os.environ.get("BITS", "4")))
for pair in sys.argv[1:]:
    q_std, rs = (float(v) for v in pair.split(":"))
    e.init_weights(0, 0.02, resid_std=rs, q_std=q_std)
    agree, diffs, gaps = 0, [], []
    for trial in range(trials):
        tok = 100 + 37 * trial
        e.add_synthetic(0, ctx, tok, seed=1 + trial)
        e.add_synthetic(1, ctx, tok, seed=1 + trial)
        e.compress(1)
        _, lf = e.step([(0, 0, [tok], -1)], want_logits=True)
        _, ld = e.step([(1, 1, [tok], -1)], want_logits=True)
        diffs.append(np.abs(lf[0] - ld[0]).max())
        top = np.sort(lf[0])[-2:]
        gaps.append(top[1] - top[0])
        agree += int(np.argmax(lf[0]) == np.argmax(ld[0]))
    print(f"q_std={q_std} resid_std={rs}: top-1 agreement {agree}/{trials}, median max|dlogit| "
          f"{np.median(diffs):.3f}, median top1-top2 gap {np.median(gaps):.3f}", flush=True)
