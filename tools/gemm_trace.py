"""Phase timeline of the cluster GEMM launches of one step (diagnostics).

Needs the -DVC_GEMM_TRACE build of the library (VC_LIB points at it):
  make -C paper_2605_17613_b200 OBJDIR=/tmp/trb LIB=$PWD/tools/_trace/libvericache_trace.so EXTRA=-DVC_GEMM_TRACE
  VC_LIB=tools/_trace/libvericache_trace.so python tools/gemm_trace.py --mode draft
Per launch of the measured (last captured) step: the span from the first CTA
start to the last CTA exit, and per-CTA medians of the phases -- start ->
PDL wait released (producer), -> accumulator complete, -> partials
exchanged, -> exit -- plus the gap from the previous launch's last exit.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_17613_b200 as vc  # noqa: E402
from paper_2605_17613_b200 import _lib  # noqa: E402

L, C, P = 512, 256, 7


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mode", default="draft", choices=["decode", "draft", "mixed"])
    p.add_argument("--x", type=int, default=6)
    p.add_argument("--out", default="gpurun_out/gemm_trace.bin")
    a = p.parse_args()
    B, x, ctx = 16, a.x, 32768
    comp = a.mode != "decode"
    e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=ctx + 256, max_x=x, quant_bits=4 if comp else 0,
                  max_verify=2, use_graphs=True)
    e.init_weights(0, 0.02)
    for i in range(B):
        e.add_synthetic(i, ctx, 100 + i, seed=1 + i)
        if comp:
            e.compress(i)
    if comp:
        for _ in range(x):
            e.draft([0])
    for _ in range(4):
        if a.mode == "decode":
            e.decode_step(list(range(B)))
        elif a.mode == "draft":
            e.step([(i, 1, [e.state(i)["pending"]], -1) for i in range(B)])
        else:
            st = e.state(0)
            e.step([(0, 2, [st["pending"]] + [1] * x, -1)] + [(i, 1, [e.state(i)["pending"]], -1) for i in range(1, B)])
    lib = _lib.load()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    rc = lib.vc_gemm_trace_dump(a.out.encode())
    e.close()
    assert rc == 0, rc
    raw = open(a.out, "rb").read()
    nk = np.frombuffer(raw[:L * 3 * 4], np.int32).reshape(L, 3)
    t = np.frombuffer(raw[L * 3 * 4:], np.uint64).reshape(L, C, P).astype(np.float64)
    used = [i for i in range(L) if nk[i, 0] > 0]
    # the measured step = the last captured graph: the last 4 * layers + 1 launches
    n = 4 * 32 + 1
    ids = used[-n:]
    prev_end = None
    rows = []
    for i in ids:
        N, K, S = nk[i]
        ctas = min(C, (N // 128) * max(S, 1))
        tt = t[i, :ctas]
        ok = tt[:, 0] > 0
        tt = tt[ok]
        if len(tt) == 0:
            continue
        start, end = tt[:, 0].min(), tt[:, 4].max() if S > 0 else tt[:, 0].max()
        ph = np.median(np.diff(tt[:, :5], axis=1), axis=0) / 1e3
        ep = tt[:, 5:7]
        eok = (ep > 0).all(axis=1)
        red = np.median(ep[eok, 0] - tt[eok, 3]) / 1e3 if eok.any() else float("nan")
        epi = np.median(ep[eok, 1] - ep[eok, 0]) / 1e3 if eok.any() else float("nan")
        gap = (tt[:, 1].min() - prev_end) / 1e3 if prev_end is not None else float("nan")
        rows.append((N, K, S, (end - start) / 1e3, gap, *ph, (tt[:, 1].min() - start) / 1e3, red, epi))
        prev_end = end
    rows = np.array(rows)
    names = {(6144, 4096): "qkv", (4096, 4096): "o", (28672, 4096): "gate/up", (4096, 14336): "down",
             (128256, 4096): "lm_head"}
    print(f"mode={a.mode} launches={len(rows)}  (us; medians over CTAs; gap = first PDL release - previous last exit)")
    print(f"{'gemm':8s} {'n':>3s} {'span':>7s} {'gap':>6s} {'st->pdl':>8s} {'pdl->acc':>9s} {'acc->xchg':>9s} {'xchg->end':>9s} {'first pdl-start':>15s} {'reduce':>7s} {'epi':>6s}")
    for key, nm in names.items():
        sel = (rows[:, 0] == key[0]) & (rows[:, 1] == key[1])
        if sel.any():
            m = rows[sel][:, 3:].mean(axis=0)
            print(f"{nm:8s} {sel.sum():3d} {m[0]:7.2f} {m[1]:6.2f} {m[2]:8.2f} {m[3]:9.2f} {m[4]:9.2f} {m[5]:9.2f} {m[6]:15.2f} {m[7]:7.2f} {m[8]:6.2f}")


if __name__ == "__main__":
    main()
