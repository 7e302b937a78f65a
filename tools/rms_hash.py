"""Hash of the logits of a few step shapes (decode 16 rows, verify window,
mixed) -- run under VC_FUSE_RMS=0 and =1 to check the fused RMSNorm is
bit-identical to the rms_apply launches."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

shape = vc.LLAMA3_8B if "--big" in sys.argv else vc.TINY
e = vc.Engine(shape, max_slots=20, max_ctx=2300, max_x=100, quant_bits=4, max_verify=2)
e.init_weights(0, 0.02)
for i in range(20):
    e.add_synthetic(i, 2000, 100 + i, seed=1 + i)
h = hashlib.sha256()
for items in ([(i, 0, [100 + i], -1) for i in range(16)], [(0, 2, list(range(5, 22)), -1)],
              [(i, 0, [100 + i], -1) for i in range(18)] + [(18, 2, list(range(3, 100)), -1),
                                                           (19, 2, list(range(7, 104)), -1)]):
    _, lg = e.step(items, want_logits=True)
    h.update(np.ascontiguousarray(lg).view(np.uint32).tobytes())
print("logits hash", h.hexdigest()[:16])
e.close()
