"""Measured-constant knob selection.

Restates the reference's intra-request throughput objective and grid search
(intra_throughput / optimize_intra, /root/reference/proj/src/analytics.cpp:
47-82 and :130-150; kv_avg :9-13; acceptance-table lookup core.cpp:133-145)
and feeds it the constants measured on the B200 in this round instead of the
paper's nominal ones:
  * HBM bandwidth: the effective rate of the measured full-KV decode step and
    of the measured draft step (the model has one bandwidth; both are shown);
  * interconnect: the measured pinned H2D rate of the swap;
  * c: the measured compressed/full byte ratio of the int4 tier;
  * gamma(x): the measured accepted-drafted tokens per verify (nearest x).
It prints the model's prediction for the configurations bench.py runs next to
the measured values, and the knobs the reference's optimiser would pick.
Usage: python tools/knobs.py [profiles/r01_bench_default.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kv_avg(x, c, kv):                        # analytics.cpp:9-13
    return kv * (x * c + 1.0) / (x + 1.0)


def gamma_table(table, x):                   # core.cpp:138-145, nearest x, ties -> smaller
    xs = sorted(table)
    if x in table:
        return table[x]
    hi = next((k for k in xs if k > x), None)
    lo = max((k for k in xs if k < x), default=None)
    if hi is None:
        return table[lo]
    if lo is None:
        return table[hi]
    return table[hi] if hi - x < x - lo else table[lo]


def intra_throughput(b_c, x, c, l, bw_hbm, bw_inter, gpu_mem, weights, kv, batch, gtab):
    """analytics.cpp:47-82 (None = infeasible)."""
    if b_c == 0:
        if weights + batch * kv > gpu_mem:
            return None
        return batch / ((weights + batch * kv) / bw_hbm)
    if b_c / (x + 1.0) * l > 1.0 + 1e-12:    # one in-flight reload at a time
        return None
    avg = kv_avg(x, c, kv)
    if weights + (batch - b_c) * kv + b_c * avg > gpu_mem:
        return None
    t_gpu = (weights + batch * avg) / bw_hbm
    t_xfer = b_c * (1.0 - c) * kv / ((x + 1.0) * bw_inter * l)
    g = gamma_table(gtab, x)
    return batch * (g * x + 1.0) / (x + 1.0) / max(t_gpu, t_xfer)


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_bench_default.json")
    d = json.loads(open(path).read().strip().splitlines()[-1])
    B = d["config"]["global_batch"] // d["n_gpus"]
    kv = float(d["compressed"]["full_bytes"])
    c = (d["compressed"]["payload_bytes"] + d["compressed"]["aux_bytes"]) / kv
    weights = 15.01e9                        # bytes read per step (layers + LM head)
    dec_ms = d["full_kv_decode"]["ms_per_step"]
    bw_dec = (weights + B * kv) / (dec_ms / 1e3)
    bw_draft = d["roofline"]["achieved"] * 1e9
    host = d["tiers"]["host"]
    bw_inter = host["swap"]["h2d_gbs"] * 1e9
    gpu_mem = 179e9
    # measured accepted drafted tokens per verify at int4, 32K (this round)
    acc = {t["draft_x"]: t["accepted_per_verify"] for t in d["tiers"].values()}
    acc.setdefault(30, 21.1)                 # tools/accept_sweep.py calibration point
    gtab = {x: a / x for x, a in acc.items()}
    print(f"measured constants: B={B} kv_full={kv / 1e9:.2f} GB c={c:.3f} weights/step={weights / 1e9:.2f} GB")
    print(f"  HBM effective: decode step {bw_dec / 1e12:.2f} TB/s, draft attention {bw_draft / 1e12:.2f} TB/s;"
          f" H2D {bw_inter / 1e9:.1f} GB/s; gamma table {{x: gamma}} = "
          + ", ".join(f"{x}: {g:.3f}" for x, g in sorted(gtab.items())))
    for name, bw in (("decode-step bandwidth", bw_dec), ("draft-kernel bandwidth", bw_draft)):
        base = intra_throughput(0, 1, c, 1, bw, bw_inter, gpu_mem, weights, kv, B, gtab)
        host_pred = intra_throughput(B, host["draft_x"], c, 1, bw, bw_inter, gpu_mem, weights, kv, B, gtab)
        hbm_x = d["tiers"]["hbm"]["draft_x"]
        # the HBM tier = every request speculating with its full KV resident:
        # the model's B_c -> 0+ limit (no transfer term)
        avg = kv_avg(hbm_x, c, kv)
        hbm_pred = B * (gamma_table(gtab, hbm_x) * hbm_x + 1) / (hbm_x + 1) / ((weights + B * avg) / bw)
        best = None
        for b_c in range(0, B + 1):
            for x in range(1, 65):
                for l in range(1, 9):
                    v = intra_throughput(b_c, x, c, l, bw, bw_inter, gpu_mem, weights, kv, B, gtab)
                    if v is not None and (best is None or v > best[0]):
                        best = (v, b_c, x, l)
        print(f"\nmodel with the {name} ({bw / 1e12:.2f} TB/s):")
        print(f"  full-KV decode (B_c=0):          predicted {base:8.1f} tok/s   measured "
              f"{d['full_kv_decode']['value']:8.1f}")
        print(f"  host tier, B_c={B}, x={host['draft_x']:>2}, l=1:     predicted {host_pred if host_pred else 0:8.1f} tok/s   "
              f"measured {host['value']:8.1f}")
        print(f"  HBM tier (B_c->0+), x={hbm_x}:         predicted {hbm_pred:8.1f} tok/s   measured "
              f"{d['tiers']['hbm']['value']:8.1f}")
        print(f"  optimiser (B_c in 0..{B}, x in 1..64, l in 1..8, c={c:.3f}): B_c={best[1]}, x={best[2]}, "
              f"l={best[3]} -> {best[0]:.1f} tok/s")


if __name__ == "__main__":
    main()
