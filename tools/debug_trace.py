"""Eager verify steps with VC_TRACE=1 (stage checksums to stderr)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T  # noqa: E402
from paper_2605_17613_b200 import TINY, Engine  # noqa: E402

w = T.tiny_weights(TINY, seed=7)
e = Engine(TINY, max_slots=2, max_ctx=2400, max_x=16, quant_bits=4, use_graphs=False)
e.load_weights(w)
e.add_synthetic(0, 2000, 17, seed=1)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    print("REP", rep, file=sys.stderr)
    out = e.step([(0, 2, [17], -1)])
    print("out", out.tolist(), file=sys.stderr)
