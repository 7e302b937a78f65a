"""GEMM determinism: StoreF32 vs SiLU epilogue on the same shapes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import vc_testlib as T  # noqa: E402
from paper_2605_17613_b200 import _lib  # noqa: E402

lib = _lib.load()


def run(X, W, epi):
    M, K = X.shape
    N = W.shape[0]
    xd = torch.from_numpy(X.view(np.int16).copy()).cuda()
    wd = torch.from_numpy(W.view(np.int16).copy()).cuda()
    y = torch.zeros(((M + 128) * N,), dtype=torch.float32, device="cuda")
    rc = lib.vc_gemm_probe_epi(xd.data_ptr(), M, K, wd.data_ptr(), N, epi, y.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.vc_last_error()
    torch.cuda.synchronize()
    return y.cpu().numpy()


rng = np.random.default_rng(0)
for M, N, K in ((16, 3072, 512), (16, 768, 512), (16, 28672, 4096)):
    X = T.f32_to_bf16(rng.standard_normal((M, K)).astype(np.float32))
    W = T.f32_to_bf16((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    for epi in (0, 3):
        outs = [run(X, W, epi) for _ in range(6)]
        same = [np.array_equal(o.view(np.uint32), outs[0].view(np.uint32)) for o in outs[1:]]
        print(f"M={M} N={N} K={K} epi={epi}: identical {same}")
