"""Measured acceptance gamma(x) = accepted drafted tokens / x per verify, for
the configs[1] workload (Llama-3-8B shape, 32K context, calibrated synthetic
init q_std 2e-3 / resid_std 2e-4), int4 and int2 KIVI, lock-step
run_speculative over B requests; every emitted token is compared with full-KV
greedy decode.  Writes profiles/r02_gamma.json, the gamma table the knob
selection (paper_2605_17613_b200/knobs.py) and bench.py use.

With --sensitivity, also sweeps the synthetic init (q_std:resid_std pairs)
and reports gamma at x = 6 and x = 47 for each: acceptance, and so every
speed-up, is a property of the init (SURVEY.md §7 hard part 1).

    python tools/gamma_sweep.py [--sensitivity] [--out profiles/r02_gamma.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

XS = [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 47, 64]


def sweep(e, B, ctx, bits_label, xs, K, first):
    out = {}
    for x in xs:
        for i in range(B):
            e.add_synthetic(i, ctx, first[i], seed=1 + i)
            e.add_synthetic(B + i, ctx, first[i], seed=1 + i)
            e.compress(B + i)
        base, _ = e.autoregress(list(range(B)), K)
        spec, rounds, _ = e.run_speculative(list(range(B, 2 * B)), K, x)
        acc = [n - 1 for r in rounds for n in r[:-1]]  # last round may be truncated at K
        a = float(np.mean(acc)) if acc else 0.0
        out[x] = {"accepted_per_verify": round(a, 3), "gamma": round(a / x, 4), "verifies": len(acc),
                  "lossless": bool((spec == base).all())}
        print(f"{bits_label} x={x}: accepted/verify {a:.2f} gamma {a / x:.3f} ({len(acc)} verifies) "
              f"lossless={out[x]['lossless']}", flush=True)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_gamma.json"))
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--ctx", type=int, default=32768)
    p.add_argument("--tokens", type=int, default=160)
    p.add_argument("--sensitivity", action="store_true")
    a = p.parse_args()
    B, ctx, K = a.batch, a.ctx, a.tokens
    first = [100 + 37 * i for i in range(B)]
    res = {"workload": f"Llama-3-8B shape, {ctx} ctx, lock-step run_speculative, {B} requests x {K} tokens, "
                       "synthetic init q_std 2e-3 / resid_std 2e-4 (bench.py's calibration)", "tables": {}}
    t0 = time.time()
    for bits in (4, 2):
        e = vc.Engine(vc.LLAMA3_8B, max_slots=2 * B, max_ctx=ctx + K + 2 * 64 + 8, max_x=64, quant_bits=bits,
                      max_verify=B)
        e.init_weights(0, 0.02, resid_std=2e-4, q_std=2e-3)
        res["tables"][f"int{bits}"] = sweep(e, B, ctx, f"int{bits}", XS, K, first)
        if bits == 4 and a.sensitivity:
            sens = {}
            for q_std, rs in [(2e-3, 2e-4), (4e-3, 4e-4), (8e-3, 1e-3), (2e-2, 2e-3), (2e-2, 2e-2)]:
                e.init_weights(0, 0.02, resid_std=rs, q_std=q_std)
                sens[f"{q_std}:{rs}"] = sweep(e, B, ctx, f"int4 q_std={q_std} resid_std={rs}", [6, 47], K, first)
            res["sensitivity"] = sens
        e.close()
        del e
    res["seconds"] = round(time.time() - t0, 1)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
