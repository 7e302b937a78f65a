"""Manual draft/verify/accept rounds on a tier-1 (host pool) engine vs tier 0."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T  # noqa: E402
from paper_2605_17613_b200 import TINY, Engine  # noqa: E402

w = T.tiny_weights(TINY, seed=7)
N = 2000
eng = {}
for tier in (0, 1):
    e = Engine(TINY, max_slots=2, max_ctx=N + 400, max_x=16, quant_bits=4, full_tier=tier, n_stage=2)
    e.load_weights(w)
    e.add_synthetic(0, N, 17, seed=1)
    e.compress(0)
    eng[tier] = e
# prefix rows equal?
k0, v0 = eng[0].kv_read(0, 0, 1, 1, 100, 4)
k1, v1 = eng[1].kv_read(2, 0, 1, 1, 100, 4)
print("prefix host==full", np.array_equal(k0, k1), np.array_equal(v0, v1))
x = eng[1].swap_begin(0, 0)
while not eng[1].swap_poll(x):
    pass
k2, v2 = eng[1].kv_read(1, 0, 1, 1, 100, 4)
print("prefix stage==full", np.array_equal(k0, k2), np.array_equal(v0, v2))
drafts = {}
for tier in (0, 1):
    drafts[tier] = [int(eng[tier].draft([0])[0]) for _ in range(3)]
print("drafts", drafts)
preds = {}
for tier in (0, 1):
    preds[tier] = eng[tier].verify([0], [0] if tier == 1 else None).tolist()
print("preds", preds)
for layer in range(2):
    for head in range(2):
        a = eng[0].kv_read(0, 0, layer, head, N, 4)
        b = eng[1].kv_read(1, 0, layer, head, N, 4)
        print("window KV layer", layer, "head", head, "k rows equal", [np.array_equal(a[0][i], b[0][i]) for i in range(4)],
              "v", [np.array_equal(a[1][i], b[1][i]) for i in range(4)])
