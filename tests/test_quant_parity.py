"""quant_kivi (vc_quant.cu) is bit-exact with the CPU oracle: codes, fp16
scales and fp16 zeros, int4 and int2, d=128 and d=64, including degenerate
groups (constant channel -> scale 0) and outlier channels."""
import numpy as np
import pytest

import vc_testlib as T

pytestmark = pytest.mark.gpu


def _run(cuda, k_bits, v_bits, d, bits, n_groups):
    lib = __import__("paper_2605_17613_b200")._lib.load()
    torch = cuda
    G = 128
    kd = torch.from_numpy(k_bits.view(np.int16).copy()).cuda()
    vd = torch.from_numpy(v_bits.view(np.int16).copy()).cuda()
    words = G * d * bits // 32
    kc = torch.zeros(n_groups * words, dtype=torch.int32, device="cuda")
    vc = torch.zeros_like(kc)
    ksz = torch.zeros(n_groups * d, dtype=torch.int32, device="cuda")
    vsz = torch.zeros(n_groups * G, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.vc_quant_kivi_slice(kd.data_ptr(), vd.data_ptr(), n_groups, d, bits, kc.data_ptr(),
                                 ksz.data_ptr(), vc.data_ptr(), vsz.data_ptr(), s)
    assert rc == 0, lib.vc_last_error()
    torch.cuda.synchronize()
    g = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
    return g(kc), g(ksz), g(vc), g(vsz)


@pytest.mark.parametrize("d,bits", [(128, 4), (128, 2), (64, 4), (64, 2)])
@pytest.mark.parametrize("seed", [1, 2])
def test_quant_bit_exact(cuda, d, bits, seed):
    G, n_groups = 128, 3
    T_ = G * n_groups
    k, v = T.synthetic_kv(1, 1, T_, d, seed)
    k, v = k[0, 0], v[0, 0]
    # degenerate group: a constant channel and a constant token
    k[:G, 5] = k[0, 5]
    v[7, :] = v[7, 0]
    kc, ksz, vc, vsz = _run(cuda, k, v, d, bits, n_groups)
    codes_k, sk, zk = T.quant_oracle(k, G, bits, "rows")
    codes_v, sv, zv = T.quant_oracle(v, d, bits, "cols")
    got_k = T.unpack_slice(kc, n_groups, d, bits, "k")
    got_v = T.unpack_slice(vc, n_groups, d, bits, "v")
    np.testing.assert_array_equal(got_k, codes_k)
    np.testing.assert_array_equal(got_v, codes_v)
    np.testing.assert_array_equal((ksz & 0xFFFF).astype(np.uint16), sk.reshape(-1))
    np.testing.assert_array_equal((ksz >> 16).astype(np.uint16), zk.reshape(-1))
    np.testing.assert_array_equal((vsz & 0xFFFF).astype(np.uint16), sv.reshape(-1))
    np.testing.assert_array_equal((vsz >> 16).astype(np.uint16), zv.reshape(-1))
    assert (sk.reshape(n_groups, d)[0, 5]) == 0  # constant channel -> scale 0


def test_quant_golden_fixture(cuda):
    """The committed golden fixture (tests/golden/quant_kivi_d128_b4.npz)."""
    import os
    path = os.path.join(T.GOLDEN, "quant_kivi_d128_b4.npz")
    z = np.load(path)
    kc, ksz, vc, vsz = _run(cuda, z["k"], z["v"], 128, 4, z["k"].shape[0] // 128)
    np.testing.assert_array_equal(kc, z["kc"])
    np.testing.assert_array_equal(ksz, z["ksz"])
    np.testing.assert_array_equal(vc, z["vc"])
    np.testing.assert_array_equal(vsz, z["vsz"])
