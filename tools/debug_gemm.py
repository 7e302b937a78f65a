"""Diagnose GEMM batch invariance: run the probe for several M, report diffs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T  # noqa: E402
from test_gemm import _gemm  # noqa: E402

rng = np.random.default_rng(0)
for K, N in ((4096, 6144), (512, 768), (4096, 1024)):
    X = T.f32_to_bf16(rng.standard_normal((200, K)).astype(np.float32))
    W = T.f32_to_bf16((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    ref = T.bf16_to_f32(X).astype(np.float64) @ T.bf16_to_f32(W).astype(np.float64).T
    full = _gemm(torch, X, W)
    print(f"K={K} N={N} full-vs-ref {np.abs(full - ref).max():.3e}")
    for m in (33, 48, 64):
        a = _gemm(torch, X[:m].copy(), W)
        b = _gemm(torch, X[:m].copy(), W)
        d = np.abs(a - ref[:m])
        bad = np.argwhere(np.abs(a - full[:m]) > 0)
        print(f"  m={m}: run-to-run {np.abs(a - b).max():.3e} vs-ref {d.max():.3e} vs-full nbad={len(bad)} "
              f"rows={sorted(set(bad[:, 0].tolist()))[:12]} tiles={sorted(set((bad[:, 1] // 128).tolist()))}")
