"""Attention kernels alone at configs[1] shape (B requests x 32K, all 32
layers): draft (kind 0, int4 compressed) and dense (kind 1, full KV, 1 row).
Prints ms per launch-set and GB/s.  VC_LIB selects the library variant:
    VC_LIB=paper_2605_17613_b200/libvc_pf4.so python tools/kbench.py"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=16)
p.add_argument("--ctx", type=int, default=32768)
p.add_argument("--bits", type=int, default=4)
p.add_argument("--dense", type=int, default=1)
a = p.parse_args()
B = a.batch
e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=a.ctx + 256, max_x=16, quant_bits=a.bits, max_verify=2)
for i in range(B):
    e.add_synthetic(i, a.ctx, 100 + i, seed=1 + i)
    e.compress(i)
tag = os.path.basename(os.environ.get("VC_LIB", "libvericache.so"))
for kind, n in ([(0, B), (1, B), (2, 1), (2, 2)] if a.dense else [(0, B)]):
    ms, b = e.kernel_bench(kind, list(range(n)), reps=5)
    print(f"{tag} kind={kind} n={n} ms={ms:.3f} GB={b / 1e9:.2f} GB/s={b / ms / 1e6:.0f}", flush=True)
e.close()
