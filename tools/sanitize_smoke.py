"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
d=64 and d=128 head shapes; int4, int2 and drop-topk (key-norm and SnapKV)
tiers; tier 0, staged tier 1 and chunk-ring tier 1 (quant and drop) scheduled
loops; composition; the remote-prefix loop; no CUDA graphs (so every launch
is checked).  Every projection runs the cluster split-K GEMM with the fused
RMSNorm producer."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T  # noqa: E402
from paper_2605_17613_b200 import TINY, Engine, ModelShape  # noqa: E402

D128 = ModelShape(vocab=256, hidden=512, layers=2, n_q=8, n_kv=2, d_head=128, ffn=512)


def run(shape):
    w = T.tiny_weights(shape, seed=7)
    ref = Engine(shape, max_slots=2, max_ctx=700, max_x=8, quant_bits=0, use_graphs=False)
    ref.load_weights(w)
    for s in range(2):
        ref.add_synthetic(s, 500, 17 + s, seed=1 + s)
    base, _ = ref.autoregress([0, 1], 12)
    ref.close()
    for kw, sched in ((dict(quant_bits=4), {}), (dict(quant_bits=2), {}), (dict(quant_bits=0, drop_ratio=0.3), {}),
                      (dict(quant_bits=0, drop_ratio=0.3, drop_score="snapkv"), {}),
                      (dict(quant_bits=4, full_tier=1, n_stage=2), {}),
                      # round 2: the chunk ring (quant and drop tiers) and composition in the scheduled loop
                      (dict(quant_bits=4, full_tier=1, n_stage=0, ring_chunks=2), {}),
                      (dict(quant_bits=0, drop_ratio=0.3, full_tier=1, n_stage=0, ring_chunks=2), {}),
                      (dict(quant_bits=4, draft_depth=3), dict(ngram=1, depth=3))):
        e = Engine(shape, max_slots=2, max_ctx=700, max_x=8, max_verify=2, use_graphs=False, **kw)
        e.load_weights(w)
        for s in range(2):
            e.add_synthetic(s, 500, 17 + s, seed=1 + s)
            e.compress(s)
        out, st = e.run_scheduled([0, 1], 12, x=4, window=16, **sched)
        assert np.array_equal(out, base), (shape, kw)
        e.close()
    # remote prefix: the stored prefix streamed into fresh slots (int2 payload)
    e = Engine(shape, max_slots=3, max_ctx=700, max_x=8, max_verify=2, quant_bits=2, use_graphs=False)
    e.load_weights(w)
    e.add_synthetic(2, 500, 0, seed=1)
    e.compress(2)
    e.prefix_store(2)
    out, _ = e.run_remote_prefix([0, 1], 12, 4, [17, 18])
    assert np.array_equal(out[0], base[0]), (shape, "remote prefix")  # same prefix seed + first token
    e.close()


for shape in (TINY, D128):
    run(shape)
print("sanitize smoke ok")
