"""Run the same draft/verify sequence in fresh engines and compare (determinism)."""
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


def run(graphs, draft_first):
    e = Engine(TINY, max_slots=2, max_ctx=N + 400, max_x=16, quant_bits=4, use_graphs=graphs)
    e.load_weights(w)
    e.add_synthetic(0, N, 17, seed=1)
    e.compress(0)
    d = [int(e.draft([0])[0]) for _ in range(3)] if draft_first else []
    st = e.state(0)
    toks = [st["pending"]] + d
    out, lg = e.step([(0, 2, toks, -1)], want_logits=True)
    e.close()
    return d, out.tolist(), lg


for graphs in (False, True):
    for draft_first in (False, True):
        res = [run(graphs, draft_first) for _ in range(3)]
        print(f"graphs={graphs} drafts={draft_first}: drafts {[r[0] for r in res]} preds {[r[1] for r in res]}")
        print("   logits equal run0 vs 1,2:", [np.array_equal(res[0][2], res[i][2]) for i in (1, 2)])
