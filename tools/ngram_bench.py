"""Lock-step VeriCache vs VeriCache composed with n-gram drafts at configs[1]
shape (Llama-3-8B, 32K, int4, full KV in HBM, B=16), calibrated init: tokens/s
from host wall time of each loop, tokens checked against full-KV decode."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

B, CTX, K = 16, 32768, int(os.environ.get("K", "160"))
X = int(os.environ.get("X", "6"))
e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=CTX + K + 3 * (X + 1) + 8, max_x=X, quant_bits=4,
              max_verify=B)
e.init_weights(0, 0.02, resid_std=0.0002, q_std=0.002)
rng = np.random.default_rng(2)
first = [int(t) for t in rng.integers(0, vc.LLAMA3_8B.vocab, B)]
for i in range(B):
    e.add_synthetic(i, CTX, first[i], seed=1 + 1000 * i)
base, ms_b = e.autoregress(list(range(B)), K)
print(f"full-KV decode: {B * K / ms_b * 1e3:.1f} tok/s", flush=True)
for ngram in (0, 1, 2, 3):
    for i in range(B):  # same requests again, fresh state
        e.add_synthetic(i, CTX, first[i], seed=1 + 1000 * i)
        e.compress(i)
    slots = list(range(B))
    if ngram == 0:
        out, rounds, ms = e.run_speculative(slots, K, X)
        ng = [0] * B
    else:
        out, rounds, ng, ms = e.run_speculative_ngram(slots, K, X, ngram=ngram)
    ok = bool((out == base).all())
    nr = sum(len(r) for r in rounds)
    print(f"ngram={ngram}: {B * K / ms * 1e3:.1f} tok/s, rounds {nr}, n-gram rounds {sum(ng)}, "
          f"tokens/round {B * K / nr:.2f}, identical={ok}", flush=True)

# two-level composition inside the scheduled loop (HBM tier) against the
# reference's composed_accept_length with the measured gamma(x) (plain run)
# and gamma_e (auxiliary proposals confirmed / offered)
from paper_2605_17613_b200 import knobs  # noqa: E402
e.close()
D = int(os.environ.get("DEPTH", "3"))
res = {}
for depth in (1, D):
    ec = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=CTX + K + 3 * (X + 1) + 8, max_x=X * D, quant_bits=4,
                   max_verify=B, draft_depth=depth)
    ec.init_weights(0, 0.02, resid_std=0.0002, q_std=0.002)
    for i in range(B):
        ec.add_synthetic(i, CTX, first[i], seed=1 + 1000 * i)
        ec.compress(i)
    out, st = ec.run_scheduled(list(range(B)), K, x=X, window=48, ngram=2 if depth > 1 else 0, depth=depth)
    ok = bool((out == base).all())
    res[depth] = st
    print(f"scheduled depth={depth}: accepted/verify {st['mean_accept']:.3f}, drafted/verify "
          f"{st['drafted_tokens'] / max(st['verifies'], 1):.2f}, aux {st['aux_accepted']}/{st['aux_proposed']}, "
          f"{st['throughput']:.1f} tok/s, identical={ok}", flush=True)
    ec.close()
g = res[1]["mean_accept"] / X
ge = res[D]["aux_accepted"] / max(res[D]["aux_proposed"], 1)
print(f"composed_accept_length(x={X}, gamma={g:.3f}, d_e={D}, gamma_e={ge:.3f}) = "
      f"{knobs.composed_accept_length(X, g, D, ge):.3f} predicted vs {res[D]['mean_accept']:.3f} measured")

