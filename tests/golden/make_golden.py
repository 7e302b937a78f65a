"""Regenerate tests/golden/* (run in a container that has /root/reference).

  make -C oracle all ref && python tests/golden/make_golden.py

reference_vectors.json -- vectors pinned by the REFERENCE library
  (oracle/_ref/libspeckv_ref.so, compiled unmodified from /root/reference):
  * accept(): the cases of proj/tests/test_specloop.cpp:86-115, outputs as
    the reference returns them;
  * drop-uniform index digests for seeded shapes (compressor.cpp:114-177);
  * the scheduler soak digest of acceptance_test.cpp:412-517 (seed 99,
    100k iterations) and a 20k-iteration seed-7 digest.
quant_kivi_d128_b4.npz -- the CPU oracle's KIVI codes for a seeded slice in
  the documented fragment layout (quantisation has no reference numerics:
  SPEC.md:560, so this fixture pins the oracle, "parity unpinned by the
  reference" as DESIGN.md states).
"""
import ctypes as C
import math
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import vc_testlib as T  # noqa: E402


def main():
    r = T.ref()
    if r is None:
        raise SystemExit("oracle/_ref/libspeckv_ref.so missing: make -C oracle ref")
    out = {"source": "oracle/_ref (unmodified /root/reference/proj compiled by oracle/Makefile)"}
    cases = [([1, 2, 3], [1, 2, 3, 9]), ([1, 2, 3], [1, 7, 3, 9]), ([4], [5, 6]),
             ([7, 7, 7, 7], [7, 7, 7, 7, 1]), ([2, 3], [2, 4, 0])]
    acc = []
    for d, p in cases:
        dd = np.array(d, np.int32)
        pp = np.array(p, np.int32)
        o = np.zeros(len(d) + 1, np.int32)
        n, fm, bonus = C.c_int(), C.c_int(), C.c_int()
        assert r.ref_accept(T.ptr(dd, C.c_int32), T.ptr(pp, C.c_int32), len(d), T.ptr(o, C.c_int32),
                            C.byref(n), C.byref(fm), C.byref(bonus)) == 0
        acc.append({"drafted": d, "preds": p, "accepted": o[: n.value].tolist(),
                    "first_mismatch": fm.value, "bonus": bool(bonus.value)})
    out["accept"] = acc
    dig = {}
    for tokens, ratio, seed in [(100, 0.25, 1), (4096, 0.2, 9), (777, 0.5, 123)]:
        drop = tokens - int(math.floor(ratio * tokens + 0.5))
        want = np.zeros((2, 3, drop), np.int64)
        pay, bs = C.c_int64(), C.c_int()
        assert r.ref_compress(0, 2, 3, tokens, 256, ratio, 4, seed, 0, T.ptr(want, C.c_int64),
                              C.byref(pay), C.byref(bs)) == drop
        dig[f"{tokens}_{ratio}_{seed}"] = int(np.bitwise_xor.reduce(want.reshape(-1) * 2654435761 % (1 << 61)))
    out["drop_uniform_digest"] = dig
    soak = {}
    for seed, iters in [(99, 100000), (7, 20000)]:
        d, em, cpl = C.c_uint64(), C.c_double(), C.c_int64()
        assert r.ref_soak(seed, iters, C.byref(d), C.byref(em), C.byref(cpl)) == 0
        soak[f"{seed}_{iters}"] = {"digest": f"{d.value:016x}", "emitted": em.value, "completed": cpl.value}
    out["soak"] = soak
    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(out, f, indent=1)

    # quant fixture from the oracle
    G, d, bits, ng = 128, 128, 4, 2
    k, v = T.synthetic_kv(1, 1, G * ng, d, seed=42)
    k, v = k[0, 0], v[0, 0]
    ck, sk, zk = T.quant_oracle(k, G, bits, "rows")
    cv, sv, zv = T.quant_oracle(v, d, bits, "cols")
    np.savez_compressed(
        os.path.join(HERE, "quant_kivi_d128_b4.npz"), k=k, v=v,
        kc=T.pack_slice(ck, d, bits, "k"), vc=T.pack_slice(cv, d, bits, "v"),
        ksz=(sk.reshape(-1).astype(np.uint32) | (zk.reshape(-1).astype(np.uint32) << 16)),
        vsz=(sv.reshape(-1).astype(np.uint32) | (zv.reshape(-1).astype(np.uint32) << 16)))
    print("wrote", HERE)


if __name__ == "__main__":
    main()
