"""Which drafting rows differ between a batched draft step and single-row
steps?  (diagnosis of the large-batch draft-attention mismatch)"""
import sys
import numpy as np
sys.path[:0] = [".", "tests"]
import vc_testlib as T
from paper_2605_17613_b200 import Engine, ModelShape

s = ModelShape(vocab=512, hidden=512, layers=2, n_q=32, n_kv=8, d_head=128, ffn=512)
w = T.tiny_weights(s, seed=5, std=0.02)
for bits, n, ctx, step in [(4, 40, 2048, 263), (4, 24, 32768, 263), (4, 48, 8192, 0), (4, 48, 32768, 0), (4, 33, 2048, 0)]:
    e = Engine(s, max_slots=n, max_ctx=ctx + step * n + 64, max_x=8, quant_bits=bits)
    e.load_weights(w)
    for i in range(n):
        e.add_synthetic(i, ctx + step * i, 17 + i, seed=1 + i)
        e.compress(i)
    items = [(i, 1, [17 + i], -1) for i in range(n)]
    _, batched = e.step(items, want_logits=True)
    bad = []
    for i in range(n):
        _, one = e.step([items[i]], want_logits=True)
        err = float(np.abs(one[0] - batched[i]).max() / np.abs(one[0]).max())
        if err > 1e-6:
            bad.append((i, round(err, 3)))
    print(f"bits={bits} n={n} ctx={ctx}+{step}i: {len(bad)} rows differ: {bad[:12]}", flush=True)
    e.close()
