"""Dense verify attention (one request, 32K ctx, all 32 layers) vs the draft
window size: time per launch-set and GB/s -- separates per-tile softmax cost
(grows with the window's query rows) from K/V streaming (constant)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

for x in [int(v) for v in (sys.argv[1:] or ["0", "3", "7", "11", "15", "19", "31", "63", "95"])]:
    e = vc.Engine(vc.LLAMA3_8B, max_slots=1, max_ctx=32768 + 256, max_x=max(x, 1), quant_bits=0, max_verify=1)
    e.add_synthetic(0, 32768, 100, seed=1)
    ms, b = e.kernel_bench(2 if x > 0 else 1, [0], reps=5)
    print(f"x={x} rows={(x + 1) * 4} ms={ms:.3f} GB/s={b / ms / 1e6:.0f}", flush=True)
    e.close()
