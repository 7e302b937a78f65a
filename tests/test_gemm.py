"""The stream-K projection GEMM: correct against an fp64 reference, and
batch-invariant -- a row's result is bit-identical for any number of rows
in the batch (the property the losslessness invariant rests on).
Tolerance: bf16 inputs, fp32 accumulate: |y - y64| <= 1e-3 * sqrt(K) * rms(y64) + 1e-5."""
import os

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import _lib

pytestmark = pytest.mark.gpu


def _gemm(torch, X, W):
    lib = _lib.load()
    M, K = X.shape
    N = W.shape[0]
    xd = torch.from_numpy(X.view(np.int16).copy()).cuda()
    wd = torch.from_numpy(W.view(np.int16).copy()).cuda()
    y = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    rc = lib.vc_gemm_probe(xd.data_ptr(), M, K, wd.data_ptr(), N, y.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.vc_last_error()
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(16, 6144, 4096), (3, 4096, 14336), (80, 768, 512), (200, 1024, 1024),
                                   (1, 128256 // 8 * 8 // 128 * 128, 4096)])
def test_gemm_matches_fp64(cuda, M, N, K):
    rng = np.random.default_rng(M + N + K)
    X = T.f32_to_bf16(rng.standard_normal((M, K)).astype(np.float32))
    W = T.f32_to_bf16((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    y = _gemm(cuda, X, W)
    ref = T.bf16_to_f32(X).astype(np.float64) @ T.bf16_to_f32(W).astype(np.float64).T
    tol = 1e-3 * np.sqrt(K) * np.sqrt((ref ** 2).mean()) + 1e-5
    assert np.abs(y - ref).max() <= tol


# (6144, 4096) qkv, (4096, 4096) o_proj and (4096, 14336) down_proj run the
# cluster split-K path (S = 6, 8, 8); (28672, 4096) gate/up the stream-K path
@pytest.mark.parametrize("N,K", [(6144, 4096), (4096, 4096), (4096, 14336), (28672, 4096)])
def test_gemm_batch_invariance(cuda, N, K):
    rng = np.random.default_rng(0)
    X = T.f32_to_bf16(rng.standard_normal((200, K)).astype(np.float32))
    W = T.f32_to_bf16((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    full = _gemm(cuda, X, W)
    for m in (1, 7, 16, 33, 80, 129):
        sub = _gemm(cuda, X[:m].copy(), W)
        np.testing.assert_array_equal(sub, full[:m])
    # a row in the middle of a batch == the same row alone
    np.testing.assert_array_equal(_gemm(cuda, X[150:151].copy(), W)[0], full[150])


_FUSE_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import os

import numpy as np
import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine
w = T.tiny_weights(TINY, seed=7, std=0.02)
e = Engine(TINY, max_slots=4, max_ctx=1200, max_x=16, quant_bits=4)
e.load_weights(w)
h = hashlib.sha256()
for s in range(4):
    e.add_synthetic(s, 700 + 50 * s, 17 + s, seed=1 + s)
for rows in (1, 9):  # one decode row per request (M=4) and verify windows (M=40)
    items = [(s, 2 if rows > 1 else 0, [17 + s + i for i in range(rows)], -1) for s in range(4)]
    out, logits = e.step(items, want_logits=True)
    h.update(logits.tobytes()); h.update(out.tobytes())
print(h.hexdigest())
"""


@pytest.mark.gpu
def test_fused_rmsnorm_gemm_is_bit_identical(cuda):
    """GemmNormIn (RMSNorm fused into the qkv and gate/up GEMMs) gives the
    same logits, bit for bit, as the separate rms_apply launches."""
    import subprocess
    import sys
    code = _FUSE_SCRIPT % (T.ROOT, os.path.join(T.ROOT, "tests"))
    digests = []
    for fuse in ("0", "1"):
        env = dict(os.environ, VC_FUSE_NORM=fuse)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
