"""GPU vs the CPU oracle at the shapes the BASELINE.json configs actually run:

  * attention at 32K and 128K keys (configs[1] 32K, configs[2]/[4] 128K),
    where the draft kernel's stream-K split and the dense kernel's 2048-key
    chunk count differ from the 4K cases in test_attention_parity.py;
  * n_rep = 8 (Llama-3-70B: 64 Q / 8 KV heads, configs[4]): the
    draft_attn_quant_kernel<128, 4|2, 8> and dense_umma_kernel<128, 8>
    instantiations;
  * 8B-shape logits (hidden 4096, 32/8 heads, d 128, FFN 14336, vocabulary
    128256) at 32K context: decode, a verify window and a draft row;
  * the engine's logits against Hugging Face transformers directly
    (tests/golden/hf_tiny_logits.npz, a third-party forward);
  * a directed greedy-argmax test: ties, NaNs, -inf (specloop.cpp:256-263).

Tolerances are max|got - want| <= rel * max|want| + abs; each test prints its
measured error (`MEASURED ...`) and the bound; the bounds are about 2x the
largest value measured on a B200 (DESIGN.md §4 lists them)."""
import ctypes as C

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, ModelShape, _lib

pytestmark = pytest.mark.gpu

G = 128
REP8 = ModelShape(vocab=256, hidden=512, layers=2, n_q=16, n_kv=2, d_head=128, ffn=512)
REP4 = ModelShape(vocab=256, hidden=512, layers=1, n_q=8, n_kv=2, d_head=128, ffn=512)
L8B_2 = ModelShape(vocab=128256, hidden=4096, layers=2, n_q=32, n_kv=8, d_head=128, ffn=14336)

# bounds (rel, abs): max|got - want| <= rel * max|want| + abs, about 2x the
# largest error measured on a B200 (round 2, gpurun_out -> DESIGN.md §4):
#   draft int4 1.11e-2 (128K), draft int2 1.37e-2, dense 4.3e-3,
#   8B-shape logits 8.1e-3 (draft row), tiny engine vs HF fp64 6.2e-3
ATTN_DRAFT = {4: (2.2e-2, 0.0), 2: (2.8e-2, 0.0)}
ATTN_DENSE = (9e-3, 0.0)
LOGITS = (1.6e-2, 0.0)
LOGITS_HF = (1.3e-2, 0.0)


def _err(got, want, bound, name):
    err = float(np.abs(got - want).max())
    ref = float(np.abs(want).max())
    lim = bound[0] * ref + bound[1]
    print(f"MEASURED {name}: max_abs {err:.3e} rel {err / max(ref, 1e-30):.3e} bound {lim:.3e}")
    assert err <= lim, f"{name}: max err {err:.3e} > bound {lim:.3e}"
    return err


def _oracle_attn(q, k, v, lim=None):
    o = T.oracle()
    out = np.zeros_like(q)
    limp = T.ptr(np.ascontiguousarray(lim, np.int32), C.c_int) if lim is not None else None
    o.vco_attention(T.ptr(q, C.c_float), q.shape[0], T.ptr(k, C.c_float), T.ptr(v, C.c_float),
                    k.shape[0], q.shape[1], limp, T.ptr(out, C.c_float))
    return out


def _dequant(kb, vb, bits, d):
    """Dequantised (K, V) fp32 of one slice: groups from the oracle's codes,
    the residual (< G tokens) kept bf16 as the engine's tail."""
    n = kb.shape[0]
    ng = n // G
    kk = T.bf16_to_f32(kb).copy()
    vv = T.bf16_to_f32(vb).copy()
    if ng:
        ck, sk, zk = T.quant_oracle(kb[: ng * G], G, bits, "rows")
        cv, sv, zv = T.quant_oracle(vb[: ng * G], d, bits, "cols")
        kk[: ng * G] = ck * np.repeat(T.f16_bits_to_f32(sk), G, 0) + np.repeat(T.f16_bits_to_f32(zk), G, 0)
        vv[: ng * G] = cv * T.f16_bits_to_f32(sv) + T.f16_bits_to_f32(zv)
    return kk, vv


# ------------------------------------------------------------------ attention
@pytest.mark.parametrize("shape,n_ctx,bits", [(REP4, 32768, 4), (REP4, 131072, 4), (REP4, 32768 + 77, 2),
                                              (REP8, 4096 + 33, 4), (REP8, 4096, 2), (REP8, 32768, 4)])
def test_draft_attention_long_and_rep8(cuda, shape, n_ctx, bits):
    torch = cuda
    s = shape
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=8, quant_bits=bits, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=13)
    e.add_kv(0, k, v, first_token=1)
    e.compress(0)
    rep = s.n_q // s.n_kv
    q = T.f32_to_bf16(np.random.default_rng(7).standard_normal((1, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    layer = s.layers - 1
    got = T.bf16_to_f32(e.attention_probe(0, layer, 1, qd.data_ptr(), 1, n_ctx))[0]
    for h in range(s.n_kv):
        kk, vv = _dequant(k[layer, h], v[layer, h], bits, s.d_head)
        want = _oracle_attn(np.ascontiguousarray(T.bf16_to_f32(q[0, h * rep:(h + 1) * rep])), kk, vv)
        _err(got[h * rep:(h + 1) * rep], want, ATTN_DRAFT[bits], f"draft n_rep={rep} T={n_ctx} int{bits} head {h}")
    e.close()


@pytest.mark.parametrize("shape,n_ctx,n_rows", [(REP4, 32768, 17), (REP4, 131072, 17), (REP4, 131072, 1),
                                                (REP8, 4096 + 5, 9), (REP8, 32768, 1), (REP8, 32768, 17)])
def test_dense_attention_long_and_rep8(cuda, shape, n_ctx, n_rows):
    torch = cuda
    s = shape
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=16, quant_bits=0, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=17)
    e.add_kv(0, k, v, first_token=1)
    rep = s.n_q // s.n_kv
    q = T.f32_to_bf16(np.random.default_rng(8).standard_normal((n_rows, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    layer = s.layers - 1
    got = T.bf16_to_f32(e.attention_probe(0, layer, 0 if n_rows == 1 else 2, qd.data_ptr(), n_rows, n_ctx))
    for h in range(s.n_kv):
        qf = T.bf16_to_f32(q[:, h * rep:(h + 1) * rep]).reshape(n_rows * rep, s.d_head)
        lim = np.repeat(np.arange(n_rows) + n_ctx - n_rows + 1, rep)
        want = _oracle_attn(np.ascontiguousarray(qf), T.bf16_to_f32(k[layer, h]), T.bf16_to_f32(v[layer, h]),
                            lim).reshape(n_rows, rep, s.d_head)
        _err(got[:, h * rep:(h + 1) * rep], want, ATTN_DENSE, f"dense n_rep={rep} T={n_ctx} rows={n_rows} head {h}")
    e.close()


def test_dense_rep8_row_invariance(cuda):
    """n_rep 8: a row alone (decode) equals the same row inside a verify window."""
    torch = cuda
    s = REP8
    n_ctx = 5000
    e = Engine(s, max_slots=1, max_ctx=n_ctx + 64, max_x=16, quant_bits=0, use_graphs=False)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=19)
    e.add_kv(0, k, v, first_token=1)
    q = T.f32_to_bf16(np.random.default_rng(9).standard_normal((9, s.n_q, s.d_head)).astype(np.float32))
    qd = torch.from_numpy(q.view(np.int16).copy()).cuda()
    many = e.attention_probe(0, 1, 2, qd.data_ptr(), 9, n_ctx)
    for i in range(9):
        one = e.attention_probe(0, 1, 0, qd[i:i + 1].data_ptr(), 1, n_ctx - 8 + i)
        np.testing.assert_array_equal(one[0], many[i])
    e.close()


# ------------------------------------------------------------------ 8B-shape logits
@pytest.fixture(scope="module")
def l8b(cuda):
    """Two Llama-3-8B-shape layers with the full 128256-token vocabulary and
    a 32K-token synthetic prefix (the 8B geometry at configs[1]'s context;
    32 layers would only repeat the same kernels)."""
    s = L8B_2
    n_ctx = 32768
    w = T.tiny_weights(s, seed=11, std=0.02)
    k, v = T.synthetic_kv(s.layers, s.n_kv, n_ctx, s.d_head, seed=1)
    e = Engine(s, max_slots=2, max_ctx=n_ctx + 64, max_x=8, quant_bits=4)
    e.load_weights(w)
    om = T.OracleModel(s, w, cap=n_ctx + 64)
    yield s, e, om, k, v, n_ctx
    e.close()


def _top2_gap(row):
    t = np.sort(row)[-2:]
    return float(t[1] - t[0])


def _tokens_agree(got_tok, want_logits, bound, name):
    for i, row in enumerate(want_logits):
        if int(got_tok[i]) != int(np.argmax(row)):
            lim = bound[0] * np.abs(want_logits).max() + bound[1]
            assert _top2_gap(row) < 2 * lim, f"{name}: non-tie token mismatch at row {i}"


def test_8b_shape_decode_and_verify_logits_32k(l8b):
    s, e, om, k, v, n_ctx = l8b
    e.add_kv(0, k, v, first_token=17)
    toks = [17, 5, 900, 128255]
    st = om.new_kv(T.bf16_to_f32(k), T.bf16_to_f32(v))
    want = om.forward(st, toks)
    tok1, got1 = e.step([(0, 0, toks[:1], -1)], want_logits=True)  # decode row
    _err(got1[0], want[0], LOGITS, "8B-shape decode logits, 32K")
    _tokens_agree(tok1, want[:1], LOGITS, "8B decode")
    e.add_kv(0, k, v, first_token=17)  # fresh copy of the prefix
    tokv, gotv = e.step([(0, 2, toks, -1)], want_logits=True)  # 4-row verify window
    _err(gotv, want, LOGITS, "8B-shape verify-window logits, 32K")
    _tokens_agree(tokv, want, LOGITS, "8B verify")
    # the verify window's first row is the decode row, bit for bit (batch invariance)
    np.testing.assert_array_equal(gotv[0], got1[0])


def test_8b_shape_draft_logits_32k(l8b):
    s, e, om, k, v, n_ctx = l8b
    e.add_kv(1, k, v, first_token=17)
    e.compress(1)
    kq = np.zeros((s.layers, s.n_kv, n_ctx, s.d_head), np.float32)
    vq = np.zeros_like(kq)
    for l in range(s.layers):
        for h in range(s.n_kv):
            kq[l, h], vq[l, h] = _dequant(k[l, h], v[l, h], 4, s.d_head)
    want = om.forward(om.new_kv(kq, vq), [17])
    tok, got = e.step([(1, 1, [17], -1)], want_logits=True)
    _err(got[0], want[0], LOGITS, "8B-shape draft logits (int4 KV), 32K")
    _tokens_agree(tok, want, LOGITS, "8B draft")


def test_engine_logits_vs_hf_fixture(cuda):
    """The engine against Hugging Face transformers (fp64) directly: the
    third-party forward pins the GPU path, not just the oracle."""
    g = np.load(f"{T.GOLDEN}/hf_tiny_logits.npz")
    n_ctx = int(g["n_ctx"])
    toks = g["tokens"].tolist()
    w = T.tiny_weights(TINY, seed=7, std=0.02)
    k, v = T.synthetic_kv(TINY.layers, TINY.n_kv, n_ctx, TINY.d_head, seed=1)
    e = Engine(TINY, max_slots=1, max_ctx=n_ctx + 64, max_x=16, quant_bits=0)
    e.load_weights(w)
    e.add_kv(0, k, v, first_token=toks[0])
    tok, got = e.step([(0, 2, toks, -1)], want_logits=True)
    e.close()
    _err(got, g["logits"], LOGITS_HF, "tiny engine vs HF fp64 (9-row verify window)")
    _tokens_agree(tok, g["logits"], LOGITS_HF, "tiny vs HF")


# ------------------------------------------------------------------ argmax
def _max_element(row):
    """std::max_element over float (operator<), as speckv::greedy_oracle uses it."""
    best = 0
    for i in range(1, row.size):
        if row[best] < row[i]:
            best = i
    return best


def test_argmax_ties_nans_and_infs(cuda):
    torch = cuda
    V = 128256
    rows = []
    rng = np.random.default_rng(1)
    base = rng.standard_normal(V).astype(np.float32)
    r = base.copy(); r[[70000, 5, 127000, 33]] = 9.0; rows.append(r)           # tie: smallest index wins
    r = base.copy(); r[[4 * 1000 + 3, 4 * 1000 + 1]] = 7.5; rows.append(r)       # tie inside one float4
    r = base.copy(); r[[32 * 4 * 7 + 2, 32 * 4 * 3 + 2]] = 6.0; rows.append(r)   # tie across warps
    r = base.copy(); r[1000] = np.nan; r[2000] = 8.0; rows.append(r)             # NaN never wins
    r = base.copy(); r[0] = np.nan; r[2000] = 8.0; rows.append(r)                # NaN at 0 sticks
    r = np.full(V, -np.inf, np.float32); rows.append(r)                           # all -inf -> 0
    r = np.full(V, np.nan, np.float32); rows.append(r)                            # all NaN -> 0
    r = np.full(V, -np.inf, np.float32); r[V - 1] = -1e30; rows.append(r)        # last element wins
    r = np.zeros(V, np.float32); rows.append(r)                                   # all equal -> 0
    r = base.copy(); r[V - 1] = np.inf; r[V - 2] = np.inf; rows.append(r)        # +inf tie
    L = np.stack(rows)
    want = [_max_element(x) for x in L]
    o = T.oracle()
    oracle = [int(o.vco_argmax(T.ptr(np.ascontiguousarray(x), C.c_float), V)) for x in L]
    assert oracle == want
    ld = torch.from_numpy(L).cuda()
    out = torch.zeros(len(rows), dtype=torch.int32, device="cuda")
    lib = _lib.load()
    assert lib.vc_argmax_rows(ld.data_ptr(), len(rows), V, out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert out.cpu().tolist() == want
    # odd vocabulary (no float4 path)
    Lo = np.ascontiguousarray(L[:, :V - 1])
    want_o = [_max_element(x) for x in Lo]
    ld = torch.from_numpy(Lo).cuda()
    assert lib.vc_argmax_rows(ld.data_ptr(), len(rows), V - 1, out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert out.cpu().tolist() == want_o


@pytest.mark.parametrize("bits,n,ctx", [(4, 24, 2048), (2, 24, 2048), (2, 48, 32768), (4, 48, 32768)])
def test_draft_batched_equals_single(cuda, bits, n, ctx):
    """A drafting row's logits do not depend on how many other requests draft
    in the same step (the stream-K split of the draft kernel changes with the
    batch; partial boundaries move, the result stays within the draft
    tolerance) -- 24 requests of different lengths, 8B head geometry."""
    s = ModelShape(vocab=512, hidden=512, layers=2, n_q=32, n_kv=8, d_head=128, ffn=512)
    w = T.tiny_weights(s, seed=5, std=0.02)
    e = Engine(s, max_slots=n, max_ctx=ctx + 263 * n + 64, max_x=8, quant_bits=bits)
    e.load_weights(w)
    for i in range(n):
        e.add_synthetic(i, ctx + 256 * i + 7 * i, 17 + i, seed=1 + i)
        e.compress(i)
    items = [(i, 1, [17 + i], -1) for i in range(n)]
    _, batched = e.step(items, want_logits=True)
    worst = 0.0
    for i in range(n):
        _, one = e.step([items[i]], want_logits=True)
        err = float(np.abs(one[0] - batched[i]).max() / np.abs(one[0]).max())
        worst = max(worst, err)
    print(f"MEASURED draft batched vs single int{bits} n={n} ctx={ctx}: rel {worst:.3e}")
    assert worst <= 2e-2
    e.close()
