"""Combine-kernel phase timeline inside the step graph (needs the -DVC_COMBINE_TRACE build via VC_LIB; tools/gpu/combine.sh)."""
import argparse, ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa
from paper_2605_17613_b200 import _lib  # noqa

p = argparse.ArgumentParser(); p.add_argument("--mode", default="decode"); p.add_argument("--x", type=int, default=6)
a = p.parse_args()
B, x, ctx = 16, a.x, 32768
comp = a.mode != "decode"
e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=ctx + 256, max_x=x, quant_bits=4 if comp else 0, max_verify=2, use_graphs=True)
e.init_weights(0, 0.02)
for i in range(B):
    e.add_synthetic(i, ctx, 100 + i, seed=1 + i)
    if comp: e.compress(i)
if comp:
    for _ in range(x): e.draft([0])
for _ in range(4):
    if a.mode == "decode": e.decode_step(list(range(B)))
    elif a.mode == "draft": e.step([(i, 1, [e.state(i)["pending"]], -1) for i in range(B)])
    else:
        st = e.state(0)
        e.step([(0, 2, [st["pending"]] + [1] * x, -1)] + [(i, 1, [e.state(i)["pending"]], -1) for i in range(1, B)])
lib = _lib.load()
path = f"gpurun_out/ct_{a.mode}.bin"
assert lib.vc_combine_trace_dump(path.encode()) == 0
e.close()
t = np.fromfile(path, np.uint64).reshape(64, 4096, 6).astype(np.float64)
slots = [i for i in range(64) if (t[i, :, 5] > 0).any()]
slots.sort(key=lambda i: t[i, :, 5].max())
slots = slots[-32:]
rows = []
for i in slots:
    tt = t[i][(t[i] > 0).all(axis=1)]
    ph = np.median(np.diff(tt, axis=1), axis=0) / 1e3
    rel = tt[:, 2].min()
    rows.append([len(tt), (tt[:, 5].max() - tt[:, 0].min()) / 1e3, (tt[:, 5].max() - rel) / 1e3,
                 (tt[:, 2].max() - rel) / 1e3, *ph, np.percentile(tt[:, 5] - tt[:, 2], 90) / 1e3])
r = np.array(rows).mean(axis=0)
print(f"mode={a.mode} launches={len(rows)} ctas={r[0]:.0f}: span {r[1]:.2f} us, first release -> last exit {r[2]:.2f}, release skew {r[3]:.2f}")
print(f"  per-CTA medians: index {r[4]:.2f}  wait {r[5]:.2f}  (m,l) loads {r[6]:.2f}  M,l {r[7]:.2f}  O loads+store {r[8]:.2f}; p90 release->exit {r[9]:.2f}")
