"""Draft attention over the KIVI cache and dense (verify / full-KV decode)
attention match the CPU oracle within the stated tolerance.

Tolerance: draft attention feeds the tensor cores
fp16 q*kscale and fp16 p*vscale (fp32 accumulate), so per-output error is
bounded by  max|o - o_ref| <= 2e-2 * max|o_ref| + 2e-3;  dense attention
rounds P to bf16 (fp32 accumulate): same bound.  The reference for the
draft path is exact attention over the DEQUANTISED oracle cache, so the
bound covers kernel arithmetic only, not quantisation error."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import Engine, ModelShape

pytestmark = pytest.mark.gpu

SHAPES = {
    "d128_rep4": ModelShape(vocab=256, hidden=512, layers=2, n_q=8, n_kv=2, d_head=128, ffn=512),
    "d64_rep4": ModelShape(vocab=256, hidden=512, layers=2, n_q=8, n_kv=2, d_head=64, ffn=512),
}


def _tol_check(got, want, rel=2e-2, abs_=2e-3, name="attention"):
    err = np.abs(got - want).max()
    bound = rel * np.abs(want).max() + abs_
    print(f"MEASURED {name}: max_abs {err:.3e} rel {err / np.abs(want).max():.3e} bound {bound:.3e}")
    assert err <= bound, f"max err {err:.3e} > bound {bound:.3e}"


def _oracle_attn(q, k, v, lim=None):
    o = T.oracle()
    out = np.zeros_like(q)
    limp = T.ptr(np.ascontiguousarray(lim, np.int32), T.C.c_int) if lim is not None else None
    o.vco_attention(T.ptr(q, T.C.c_float), q.shape[0], T.ptr(k, T.C.c_float), T.ptr(v, T.C.c_float),
                    k.shape[0], q.shape[1], limp, T.ptr(out, T.C.c_float))
    return out


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("n_ctx,bits", [(4096, 4), (1000, 4), (2048 + 77, 2), (100, 4)])
def test_draft_attention(cuda, name, n_ctx, bits):
    torch = cuda
    s = SHAPES[name]
    e = Engine(s, max_slots=1, max_ctx=max(n_ctx + 64, 256), max_x=8, quant_bits=bits, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=11)
    e.add_kv(0, k, v, first_token=1)
    meta = e.compress(0)
    G = 128
    ng = n_ctx // G
    assert meta["n_groups"] == ng and meta["tail_tokens"] == n_ctx - ng * G
    rng = np.random.default_rng(3)
    q = T.f32_to_bf16(rng.standard_normal((1, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    rep = s.n_q // s.n_kv
    for layer in range(s.layers):
        got = T.bf16_to_f32(e.attention_probe(0, layer, 1, qd.data_ptr(), 1, n_ctx))[0]
        for h in range(s.n_kv):
            ck, sk, zk = T.quant_oracle(k[layer, h, : ng * G], G, bits, "rows")
            cv, sv, zv = T.quant_oracle(v[layer, h, : ng * G], s.d_head, bits, "cols")
            kk = np.zeros((n_ctx, s.d_head), np.float32)
            vv = np.zeros_like(kk)
            if ng:
                kk[: ng * G] = ck * np.repeat(T.f16_bits_to_f32(sk), G, 0) + np.repeat(T.f16_bits_to_f32(zk), G, 0)
                vv[: ng * G] = cv * T.f16_bits_to_f32(sv) + T.f16_bits_to_f32(zv)
            kk[ng * G:] = T.bf16_to_f32(k[layer, h, ng * G:])
            vv[ng * G:] = T.bf16_to_f32(v[layer, h, ng * G:])
            qf = T.bf16_to_f32(q[0, h * rep:(h + 1) * rep])
            want = _oracle_attn(np.ascontiguousarray(qf), kk, vv)
            _tol_check(got[h * rep:(h + 1) * rep], want, name=f"draft {name} T={n_ctx} int{bits}")
    e.close()


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("n_ctx,n_rows", [(4096, 1), (4096, 9), (333, 5), (300, 17), (1, 1)])
def test_dense_attention(cuda, name, n_ctx, n_rows):
    torch = cuda
    s = SHAPES[name]
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=16, quant_bits=0, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=5)
    e.add_kv(0, k, v, first_token=1)
    rng = np.random.default_rng(4)
    q = T.f32_to_bf16(rng.standard_normal((n_rows, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    rep = s.n_q // s.n_kv
    for layer in range(s.layers):
        got = T.bf16_to_f32(e.attention_probe(0, layer, 0, qd.data_ptr(), n_rows, n_ctx))
        for h in range(s.n_kv):
            kk = T.bf16_to_f32(k[layer, h])
            vv = T.bf16_to_f32(v[layer, h])
            qf = T.bf16_to_f32(q[:, h * rep:(h + 1) * rep]).reshape(n_rows * rep, s.d_head)
            lim = np.repeat(np.arange(n_rows) + n_ctx - n_rows + 1, rep)
            want = _oracle_attn(np.ascontiguousarray(qf), kk, vv, lim).reshape(n_rows, rep, s.d_head)
            _tol_check(got[:, h * rep:(h + 1) * rep], want, name=f"dense {name} T={n_ctx} rows={n_rows}")
    e.close()


def test_dense_attention_row_invariance(cuda):
    """A query row's output is bit-identical whether it is alone (decode) or
    the last row of a verify window (batch invariance -> losslessness)."""
    torch = cuda
    s = SHAPES["d128_rep4"]
    n_ctx = 3000
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=16, quant_bits=0, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=9)
    e.add_kv(0, k, v, first_token=1)
    rng = np.random.default_rng(5)
    q = T.f32_to_bf16(rng.standard_normal((9, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    many = e.attention_probe(0, 0, 2, qd.data_ptr(), 9, n_ctx)
    for i in range(9):
        one = e.attention_probe(0, 0, 0, qd[i:i + 1].data_ptr(), 1, n_ctx - 8 + i)
        np.testing.assert_array_equal(one[0], many[i])
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n_rows", [48, 20])
def test_dense_attention_row_invariance_many_items(cuda, n_rows):
    """Row invariance when every CTA runs several items (8 KV heads x 16
    chunks x up to 3 row blocks over 32K keys > 148 SMs) and the window's
    columns split across both softmax column groups: each row of a verify
    window equals the same row computed alone (the host tier's x=47 windows)."""
    torch = cuda
    s = ModelShape(vocab=256, hidden=1024, layers=1, n_q=32, n_kv=8, d_head=128, ffn=512)
    n_ctx = 32768
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=48, quant_bits=0, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=9)
    e.add_kv(0, k, v, first_token=1)
    rng = np.random.default_rng(n_rows)
    q = T.f32_to_bf16(rng.standard_normal((n_rows, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    many = e.attention_probe(0, 0, 2, qd.data_ptr(), n_rows, n_ctx)
    for i in range(n_rows):
        one = e.attention_probe(0, 0, 0, qd[i:i + 1].data_ptr(), 1, n_ctx - n_rows + 1 + i)
        np.testing.assert_array_equal(one[0], many[i], err_msg=f"row {i} of {n_rows}")
    e.close()


@pytest.mark.gpu
def test_verify_windows_of_mixed_widths_are_row_invariant(cuda):
    """Several verify windows of different widths in one step, over long
    contexts whose last chunks are short (items of 1-16 tiles, several per
    CTA, the softmax groups' column split changing from item to item): every
    row's logits equal that window verified alone.  (The two softmax column
    groups once shared per-column state across items -- a timing-dependent
    race this test does not reliably provoke; the full-scale host-tier bench
    line, 16 x 32K with 48-row windows, did, and checks it every run.)"""
    s = ModelShape(vocab=512, hidden=1024, layers=2, n_q=32, n_kv=8, d_head=128, ffn=1024)
    w = T.tiny_weights(s, seed=3, std=0.02)
    e = Engine(s, max_slots=3, max_ctx=33000, max_x=48, quant_bits=0, max_verify=3, use_graphs=False)
    e.load_weights(w)
    ctx = [32700, 30100, 2100]
    for i, n in enumerate(ctx):
        e.add_synthetic(i, n, 5 + i, seed=1 + i)
    rng = np.random.default_rng(0)
    wins = [[int(t) for t in rng.integers(0, s.vocab, n)] for n in (48, 7, 21)]
    items = [(i, 2, wins[i], -1) for i in range(3)]
    _, together = e.step(items, want_logits=True)
    off = 0
    for i in range(3):
        _, alone = e.step([items[i]], want_logits=True)
        np.testing.assert_array_equal(together[off:off + len(wins[i])], alone, err_msg=f"window {i}")
        off += len(wins[i])
    e.close()
