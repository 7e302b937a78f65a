"""Set up the configs[1] engine (Llama-3-8B shape, 32K ctx, batch 16) and run a
few steps of one kind, for ncu launch lists / full captures:
  --mode decode : full-KV greedy decode step (the baseline)
  --mode draft  : all 16 requests draft over the int4 cache
  --mode mixed  : 15 drafting rows + one verify window of x+1 rows
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/profile_step.py --mode mixed
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_17613_b200 as vc  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mode", default="mixed", choices=["decode", "draft", "mixed"])
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--ctx", type=int, default=32768)
    p.add_argument("--x", type=int, default=16)
    p.add_argument("--graphs", type=int, default=1)
    p.add_argument("--q-std", type=float, default=0.0)
    p.add_argument("--resid-std", type=float, default=0.0)
    p.add_argument("--reverse", action="store_true", help="draft items in reverse slot order")
    a = p.parse_args()
    B, x = a.batch, a.x
    comp = a.mode != "decode"
    e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=a.ctx + 256, max_x=x, quant_bits=4 if comp else 0,
                  max_verify=2, use_graphs=bool(a.graphs))
    e.init_weights(0, 0.02, resid_std=a.resid_std, q_std=a.q_std)
    for i in range(B):
        e.add_synthetic(i, a.ctx, 100 + i, seed=1 + i)
        if comp:
            e.compress(i)
    if comp:  # open a draft round of x tokens on request 0 so it can verify
        for _ in range(x):
            e.draft([0])
    e.timing(reset=True)
    # ncu --profile-from-start off: only the measured steps are profiled
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    cu.cuProfilerStart()
    for _ in range(a.steps):
        if a.mode == "decode":
            e.decode_step(list(range(B)))
        elif a.mode == "draft":
            order = range(B - 1, -1, -1) if a.reverse else range(B)
            e.step([(i, 1, [e.state(i)["pending"]], -1) for i in order])
        else:
            st = e.state(0)
            items = [(0, 2, [st["pending"]] + [1] * x, -1)]
            items += [(i, 1, [e.state(i)["pending"]], -1) for i in range(1, B)]
            e.step(items)
    cu.cuProfilerStop()
    ms, n = e.timing()
    print(f"mode={a.mode} steps={n} device_ms_per_step={ms / max(n, 1):.3f}")
    e.close()


if __name__ == "__main__":
    main()
