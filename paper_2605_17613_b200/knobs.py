"""Measured-constant knob selection: the reference's intra-request objective
and grid search, fed this engine's measured B200 constants.

Restates /root/reference/proj/src/analytics.cpp (same double operations in
the same order, so the results equal the compiled reference's bit for bit;
tests/test_knobs.py pins them against oracle/_ref):
  kv_avg            analytics.cpp:9-13
  intra_throughput  analytics.cpp:45-82   (B_c offloaded, x, c, l)
  optimize_intra    analytics.cpp:130-150 (lexicographic grid, strict >)
  expected_gamma    core.cpp:117-146, tabulated kind (nearest x, ties to the
                    smaller x)
bench.py uses it to pick the per-request tier placement B_c (how many
requests keep their full KV in the host tier) from the measured HBM and PCIe
bandwidths, the measured compression ratio and the measured acceptance
gamma(x) table (profiles/r02_gamma.json)."""
from __future__ import annotations

from dataclasses import dataclass


def kv_avg(x: int, c: float, kv_full: int) -> float:
    if x < 1:
        raise ValueError("kv_avg: x must be >= 1")
    if not (0.0 < c <= 1.0):
        raise ValueError("kv_avg: c out of (0,1]")
    return float(kv_full) * (x * c + 1.0) / (x + 1.0)


def expected_gamma(table: dict, x: int) -> float:
    """Tabulated gamma(x) for one c: nearest tabulated x, ties -> smaller x."""
    if x in table:
        return table[x]
    xs = sorted(table)
    hi = next((k for k in xs if k > x), None)
    if hi is None:
        return table[xs[-1]]
    if hi == xs[0]:
        return table[hi]
    lo = max(k for k in xs if k < x)
    return table[hi] if hi - x < x - lo else table[lo]


@dataclass(frozen=True)
class Hardware:
    hbm_bandwidth: float          # B/s
    interconnect_bandwidth: float  # B/s (host <-> GPU link)
    gpu_mem: int                  # bytes


def intra_throughput(b_c: int, x: int, c: float, l: int, hw: Hardware, weights: int, kv_full: int,
                     batch: int, gamma_table: dict):
    """Tokens/s of B requests with B_c offloaded (None = infeasible)."""
    if b_c < 0 or b_c > batch:
        raise ValueError("intra_throughput: B_c out of [0, B]")
    if x < 1 or l < 1:
        raise ValueError("intra_throughput: x and l must be >= 1")
    if b_c == 0:
        mem = float(weights) + float(batch) * kv_full
        if mem > float(hw.gpu_mem):
            return None
        t_gpu = (weights + float(batch) * kv_full) / hw.hbm_bandwidth
        return batch / t_gpu
    if not (0.0 < c < 1.0):
        raise ValueError("intra_throughput: c out of (0,1) for B_c > 0")
    if float(b_c) / (x + 1.0) * l > 1.0 + 1e-12:  # one in-flight reload at a time
        return None
    avg = kv_avg(x, c, kv_full)
    b_g = batch - b_c
    mem = float(weights) + float(b_g) * kv_full + b_c * avg
    if mem > float(hw.gpu_mem):
        return None
    t_gpu = (weights + batch * avg) / hw.hbm_bandwidth
    t_xfer = b_c * (1.0 - c) * float(kv_full) / ((x + 1.0) * hw.interconnect_bandwidth * l)
    gamma = expected_gamma(gamma_table, x)
    tokens_per_iter = batch * (gamma * x + 1.0) / (x + 1.0)
    return tokens_per_iter / max(t_gpu, t_xfer)


def optimize_intra(hw: Hardware, weights: int, kv_full: int, batch: int, gamma_table: dict, c: float,
                   x_max: int = 64, l_max: int = 8):
    """Best (throughput, B_c, x, l) over B_c in 0..B, x in 1..x_max, l in
    1..l_max at the measured c (the reference sweeps c too; here c is the
    compressor's measured ratio)."""
    best = None
    for b_c in range(0, batch + 1):
        for x in range(1, x_max + 1):
            for l in range(1, l_max + 1):
                v = intra_throughput(b_c, x, c, l, hw, weights, kv_full, batch, gamma_table)
                if v is None:
                    continue
                if best is None or v > best[0]:
                    best = (v, b_c, x, l)
    return best


def composed_accept_length(x: int, gamma_x: float, d_e: int, gamma_e: float) -> float:
    """Accepted tokens per verify of the two-level composition
    (composed_accept_length, /root/reference/proj/src/analytics.cpp:413-422):
    gamma * x * (1 + gamma_e * (d_e - 1)), gamma = the compressed model's
    acceptance at x (expected_gamma), gamma_e = the auxiliary drafter's."""
    if d_e < 1:
        raise ValueError("composed_accept_length: d_e must be >= 1")
    ge = 0.0 if d_e == 1 else gamma_e
    if d_e > 1 and not 0.0 <= ge <= 1.0:
        raise ValueError("composed_accept_length: gamma_e out of [0,1]")
    return gamma_x * x * (1.0 + ge * (d_e - 1.0))

