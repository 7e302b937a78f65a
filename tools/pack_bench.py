"""Host-pool codec alone (vc_pack.cu) at one layer's K of a 32K request
(8 kv heads x 32768 rows x d=128, synthetic Gaussian KV): pack + unpack via
vc_pack_roundtrip, CUDA-event timed, and the packed/raw byte ratio.  The
target of the ncu capture of pack_kernel / unpack_kernel."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_17613_b200 import _lib  # noqa: E402


def packed_block_bytes(d):  # vc_gemm.h packed_block_bytes
    cap = 128 * d * 7 // 25 // 8 * 8
    return (d + 128 * d // 4 + 128 * d + 4 + cap // 2 + 4 + 4 * 60 + 15) // 16 * 16


slices, rows, d = 8, 32768, 128
x = torch.randn(slices, rows, d, device="cuda").to(torch.bfloat16).view(torch.int16)
out = torch.zeros_like(x)
lib = _lib.load()
ovf = C.c_int(0)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert lib.vc_pack_roundtrip(x.data_ptr(), rows, slices, d, out.data_ptr(), C.byref(ovf), st) == 0
assert ovf.value == 0 and torch.equal(out, x), "round trip"
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    lib.vc_pack_roundtrip(x.data_ptr(), rows, slices, d, out.data_ptr(), C.byref(ovf), st)
b.record()
b.synchronize()
ms = a.elapsed_time(b) / 5
raw = slices * rows * d * 2
print(f"pack+unpack {slices}x{rows}x{d}: {ms:.3f} ms per round trip (incl. alloc), raw {raw / 1e6:.1f} MB, "
      f"packed/raw {packed_block_bytes(d) * rows // 128 * slices / raw:.4f}")
