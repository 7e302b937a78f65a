"""Test-side helpers: the CPU oracle (oracle/liboracle.so), the compiled
reference (oracle/_ref/libspeckv_ref.so, optional), numpy twins of the
synthetic generators, and an independent decoder of the documented
compressed-KV fragment layout."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libspeckv_ref.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")

u8p, u16p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint16), C.POINTER(C.c_uint32)
i32p, i64p, f32p = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_float)


def ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ----------------------------------------------------------------- oracle
_oracle = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"],
                                  stdout=subprocess.DEVNULL)
        o = C.CDLL(ORACLE_SO)
        o.vco_splitmix64.restype = C.c_uint64
        o.vco_splitmix64.argtypes = [C.c_uint64]
        o.vco_mt64_next.restype = C.c_uint64
        o.vco_drop_indices.restype = C.c_int64
        o.vco_drop_indices.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_double, C.c_uint64,
                                       C.c_int, i64p]
        o.vco_argmax.restype = C.c_int32
        o.vco_fill_normal_bf16.argtypes = [C.c_uint64, C.c_uint64, C.c_size_t, C.c_float, u16p]
        o.vco_f32_to_f16.restype = C.c_uint16
        o.vco_f32_to_f16.argtypes = [C.c_float]
        o.vco_f16_to_f32.restype = C.c_float
        o.vco_f16_to_f32.argtypes = [C.c_uint16]
        o.vco_rope_tables.argtypes = [C.c_int, C.c_int, C.c_double, f32p, f32p]
        _oracle = o
    return _oracle


_ref = None


def ref():
    """The unmodified reference compiled by oracle/Makefile `ref` (None if absent)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            return None
        r = C.CDLL(REF_SO)
        r.ref_compress.restype = C.c_int64
        r.ref_compress.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_double,
                                   C.c_int, C.c_uint64, C.c_int, i64p, i64p, C.POINTER(C.c_int)]
        r.ref_random_table_next.restype = C.c_int32
        r.ref_random_table_next.argtypes = [C.c_int, C.c_uint64, i32p, C.c_int64]
        r.ref_soak.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64), C.POINTER(C.c_double), i64p]
        r.ref_reload_span.argtypes = [C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_int)]
        r.ref_last_error.restype = C.c_char_p
        _ref = r
    return _ref


# ------------------------------------------------------------ bit helpers
def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, np.uint32) << 16).view(np.float32)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


K_UNIT = np.float32(1.0 / (65536.0 * np.sqrt(1.0 / 3.0)))


def normal_bf16(seed: int, offset: int, n: int, std: float) -> np.ndarray:
    """Twin of vco_fill_normal_bf16 / the device fill kernel."""
    k = np.float32(std / (65536.0 * np.sqrt(1.0 / 3.0)))
    i = np.arange(n, dtype=np.uint64) + np.uint64(offset)
    h = splitmix64(np.uint64(seed) ^ splitmix64(i))
    s = sum(((h >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64) for j in range(4))
    z = (s - 131070).astype(np.float32) * k
    return f32_to_bf16(z)


def synthetic_kv(layers, n_kv, n_ctx, d, seed, outlier_channels=4, outlier_scale=10.0):
    """Twin of the engine's synthetic prefix KV: bf16 bits [layers][n_kv][n_ctx][d]."""
    n = layers * n_kv * n_ctx * d
    i = np.arange(n, dtype=np.uint64)
    hx = splitmix64(i)
    k_out = np.float32(outlier_scale / (65536.0 * np.sqrt(1.0 / 3.0)))

    def vals(s, kk):
        h = splitmix64(np.uint64(s) ^ hx)
        sm = sum(((h >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64) for j in range(4))
        return f32_to_bf16((sm - 131070).astype(np.float32) * kk)

    c = (i % np.uint64(d)).astype(np.int64)
    period = d // outlier_channels if outlier_channels > 0 else 0
    kk = np.full(n, K_UNIT, np.float32)
    if period:
        kk[(c % period) == period - 1] = k_out
    k = vals(seed, kk)
    v = vals(seed ^ 0x5555555555555555, np.full(n, K_UNIT, np.float32))
    shp = (layers, n_kv, n_ctx, d)
    return k.reshape(shp), v.reshape(shp)


# --------------------------------------------------------- KIVI oracle
def quant_oracle(x_bf16: np.ndarray, g: int, bits: int, axis: str):
    """axis 'rows' = per-channel over token groups (K), 'cols' = per-token (V)."""
    o = oracle()
    x = np.ascontiguousarray(x_bf16, np.uint16)
    rows, cols = x.shape
    codes = np.zeros((rows, cols), np.uint8)
    if axis == "rows":
        sc = np.zeros((rows // g, cols), np.uint16)
        fn = o.vco_quant_rows
    else:
        sc = np.zeros((rows, cols // g), np.uint16)
        fn = o.vco_quant_cols
    zr = np.zeros_like(sc)
    fn(ptr(x, C.c_uint16), rows, cols, g, bits, ptr(codes, C.c_uint8), ptr(sc, C.c_uint16),
       ptr(zr, C.c_uint16))
    return codes, sc, zr


_frag_cache = {}


def frag_map(d: int, bits: int, G: int = 128):
    """(word_index, field_shift, row_in_group, col) for every code of one group.
    K: row = token, col = channel.  V: row = channel, col = token (transposed tile)."""
    key = (d, bits, G)
    if key in _frag_cache:
        return _frag_cache[key]
    KS = d // 16
    W = KS if bits == 4 else KS // 2
    CH = min(W, 4)
    MT = G // 16
    widx, shift, a_r, a_c = [], [], [], []
    for m in range(MT):
        for w in range(W):
            wq, wl = divmod(w, CH)
            for lane in range(32):
                idx = ((m * (W // CH) + wq) * 32 + lane) * CH + wl
                for sub in range(1 if bits == 4 else 2):
                    s = w if bits == 4 else 2 * w + sub
                    for j in range(4):
                        for e in range(2):
                            r = lane // 4 + (8 if j & 1 else 0)
                            c = 2 * (lane % 4) + e + (8 if j & 2 else 0)
                            # int4: pairs 0,1 in low nibbles, 2,3 in high (vc_quant.cu kNibble)
                            sh = (0, 8, 4, 12)[j] + 16 * e if bits == 4 else 8 * sub + 2 * j + 16 * e
                            widx.append(idx)
                            shift.append(sh)
                            a_r.append(m * 16 + r)   # tile row -> token (K) / tok-step rows
                            a_c.append(s * 16 + c)   # tile col -> channel (K)
    res = tuple(np.array(v, np.int64) for v in (widx, shift, a_r, a_c))
    _frag_cache[key] = res
    return res


def unpack_group(words: np.ndarray, d: int, bits: int, kind: str, G: int = 128) -> np.ndarray:
    """Decode one group's u32 words into codes [G tokens][d channels]."""
    widx, shift, r, c = frag_map(d, bits, G)
    mask = (1 << bits) - 1
    vals = (words[widx] >> shift.astype(np.uint32)) & mask
    out = np.zeros((G, d), np.uint8)
    if kind == "k":
        out[r, c] = vals                 # K tile: rows = tokens, cols = channels
    else:
        # V^T tile of (tok-step m, channel tile s): element (row=channel, col=token)
        m, rr = np.divmod(r, 16)
        s, cc = np.divmod(c, 16)
        out[m * 16 + cc, s * 16 + rr] = vals
    return out


def pack_group(codes: np.ndarray, d: int, bits: int, kind: str, G: int = 128) -> np.ndarray:
    """Inverse of unpack_group: logical codes [G][d] -> u32 words (documented layout)."""
    widx, shift, r, c = frag_map(d, bits, G)
    if kind == "k":
        vals = codes[r, c].astype(np.uint64)
    else:
        m, rr = np.divmod(r, 16)
        s, cc = np.divmod(c, 16)
        vals = codes[m * 16 + cc, s * 16 + rr].astype(np.uint64)
    words = np.zeros(G * d * bits // 32, np.uint64)
    np.bitwise_or.at(words, widx, vals << shift.astype(np.uint64))
    return words.astype(np.uint32)


def pack_slice(codes: np.ndarray, d: int, bits: int, kind: str, G: int = 128) -> np.ndarray:
    return np.concatenate([pack_group(codes[g * G:(g + 1) * G], d, bits, kind, G)
                           for g in range(codes.shape[0] // G)])


def unpack_slice(words: np.ndarray, n_groups: int, d: int, bits: int, kind: str, G: int = 128):
    per = G * d * bits // 32
    return np.concatenate([unpack_group(words[g * per:(g + 1) * per], d, bits, kind, G)
                           for g in range(n_groups)], axis=0)


def f16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return np.asarray(h, np.uint16).view(np.float16).astype(np.float32)


# --------------------------------------------------------- tiny model
def tiny_weights(shape, seed=7, std=0.02):
    """Logical bf16 weights for the oracle and Engine.load_weights."""
    H, F, V, L, d = shape.hidden, shape.ffn, shape.vocab, shape.layers, shape.d_head
    qkv_n = (shape.n_q + 2 * shape.n_kv) * d
    off = [0]

    o = oracle()
    kf = np.float32(std / (65536.0 * np.sqrt(1.0 / 3.0)))

    def nrm(*dims):
        # vco_fill_normal_bf16: the C twin of normal_bf16 (same values, fast
        # enough for 8B-shape layers)
        n = int(np.prod(dims))
        a = np.empty(n, np.uint16)
        o.vco_fill_normal_bf16(seed, off[0], n, kf, ptr(a, C.c_uint16))
        off[0] += n
        return a.reshape(dims)

    ones = lambda n: np.full(n, 0x3F80, np.uint16)  # noqa: E731
    w = {"embed": nrm(V, H), "attn_norm": [], "wqkv": [], "wo": [], "mlp_norm": [], "wgate": [],
         "wup": [], "wdown": []}
    for _ in range(L):
        w["attn_norm"].append(ones(H))
        w["wqkv"].append(nrm(qkv_n, H))
        w["wo"].append(nrm(H, shape.n_q * d))
        w["mlp_norm"].append(ones(H))
        w["wgate"].append(nrm(F, H))
        w["wup"].append(nrm(F, H))
        w["wdown"].append(nrm(H, F))
    w["final_norm"] = ones(H)
    w["lm_head"] = nrm(V, H)
    return w


class VcoModelCfg(C.Structure):
    _fields_ = [("vocab", C.c_int), ("hidden", C.c_int), ("layers", C.c_int), ("n_q", C.c_int),
                ("n_kv", C.c_int), ("d", C.c_int), ("ffn", C.c_int), ("rope_theta", C.c_float),
                ("eps", C.c_float)]


class VcoWeights(C.Structure):
    _fields_ = [("embed", u16p)] + [(n, C.POINTER(u16p)) for n in
                                    ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate", "wup", "wdown")] + \
               [("final_norm", u16p), ("lm_head", u16p)]


class VcoKv(C.Structure):
    _fields_ = [("k", f32p), ("v", f32p), ("cap", C.c_int), ("len", C.c_int)]


class OracleModel:
    """CPU restatement of the forward (vco_forward) with its own fp32 KV views."""

    def __init__(self, shape, weights, cap):
        self.o = oracle()
        self.shape = shape
        self.cfg = VcoModelCfg(shape.vocab, shape.hidden, shape.layers, shape.n_q, shape.n_kv,
                               shape.d_head, shape.ffn, shape.rope_theta, shape.rms_eps)
        self.keep = []
        L = shape.layers

        def arr(a):
            a = np.ascontiguousarray(a, np.uint16)
            self.keep.append(a)
            return ptr(a, C.c_uint16)

        def lst(name):
            p = (u16p * L)(*[arr(weights[name][i]) for i in range(L)])
            self.keep.append(p)
            return p

        self.w = VcoWeights(arr(weights["embed"]), lst("attn_norm"), lst("wqkv"), lst("wo"),
                            lst("mlp_norm"), lst("wgate"), lst("wup"), lst("wdown"),
                            arr(weights["final_norm"]), arr(weights["lm_head"]))
        half = shape.d_head // 2
        self.cos = np.zeros((cap + 8, half), np.float32)
        self.sin = np.zeros_like(self.cos)
        self.o.vco_rope_tables(cap + 8, shape.d_head, float(shape.rope_theta), ptr(self.cos, C.c_float),
                               ptr(self.sin, C.c_float))
        self.cap = cap

    def new_kv(self, k_f32=None, v_f32=None):
        """fp32 KV [layers][n_kv][cap][d] pre-filled with a prefix."""
        s = self.shape
        k = np.zeros((s.layers, s.n_kv, self.cap, s.d_head), np.float32)
        v = np.zeros_like(k)
        n = 0
        if k_f32 is not None:
            n = k_f32.shape[2]
            k[:, :, :n] = k_f32
            v[:, :, :n] = v_f32
        kv = VcoKv(ptr(k, C.c_float), ptr(v, C.c_float), self.cap, n)
        return {"k": k, "v": v, "kv": kv}

    def forward(self, state, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        logits = np.zeros((t.size, self.shape.vocab), np.float32)
        self.o.vco_forward(C.byref(self.cfg), C.byref(self.w), C.byref(state["kv"]), ptr(t, C.c_int32),
                           t.size, ptr(self.cos, C.c_float), ptr(self.sin, C.c_float),
                           ptr(logits, C.c_float), None, None)
        return logits


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
