import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine
CTX = [1, 130, 2000, 4096, 700]; FIRST = [11, 23, 37, 41, 53]
w = T.tiny_weights(TINY, seed=5, std=0.02)
for bits in (4, 2):
    e = Engine(TINY, max_slots=5, max_ctx=4096 + 64, max_x=8, max_verify=2, quant_bits=bits)
    e.load_weights(w)
    for s, (n, f) in enumerate(zip(CTX, FIRST)):
        e.add_synthetic(s, n, f, seed=100 + s)
        e.compress(s)
    items = [(s, 1, [FIRST[s]], -1) for s in range(5)]
    _, batch = e.step(items, want_logits=True)
    for subset in ([0, 1, 2, 3, 4], [4], [3, 4], [2, 4], [1, 4], [0, 4]):
        _, part = e.step([items[s] for s in subset], want_logits=True)
        i = subset.index(4)
        print(bits, subset, "row4 err vs full batch", float(np.abs(part[i] - batch[4]).max()))
    e.close()
