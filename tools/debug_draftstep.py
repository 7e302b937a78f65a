"""Why is a draft step slower inside the bench than in profile_step?  Same
engine parameters as bench.py, draft steps via step() and via draft()."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_17613_b200 as vc  # noqa: E402

B, ctx = 16, 32768
max_ctx = int(sys.argv[1]) if len(sys.argv) > 1 else ctx + 16 + 64 + 51 + 8
n_stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=max_ctx, max_x=16, quant_bits=4, full_tier=0,
              n_stage=n_stage, max_verify=2)
e.init_weights(0, 0.02, resid_std=0.0005, q_std=0.005)
for i in range(B):
    e.add_synthetic(i, ctx, 100 + i, seed=1 + i)
    e.compress(i)
e.timing(reset=True)
for _ in range(6):
    e.step([(i, 1, [e.state(i)["pending"]], -1) for i in range(B)])
ms, n = e.timing(reset=True)
print(f"max_ctx={max_ctx} n_stage={n_stage}: step() draft {ms / n:.3f} ms")
for _ in range(6):
    e.draft(list(range(B)))
ms, n = e.timing(reset=True)
print(f"max_ctx={max_ctx} n_stage={n_stage}: draft() {ms / n:.3f} ms")
kms, kb = e.kernel_bench(0, list(range(B)), reps=3)
print(f"kernel_bench draft attention {kms:.3f} ms {kb / kms / 1e6:.0f} GB/s")
e.close()
e = vc.Engine(vc.LLAMA3_8B, max_slots=B, max_ctx=max_ctx, max_x=16, quant_bits=0, full_tier=0, max_verify=2)
e.init_weights(0, 0.02, resid_std=0.0005, q_std=0.005)
for i in range(B):
    e.add_synthetic(i, ctx, 100 + i, seed=1 + i)
kms, kb = e.kernel_bench(1, list(range(B)), reps=3)
print(f"kernel_bench dense (decode) attention {kms:.3f} ms {kb / kms / 1e6:.0f} GB/s")
for _ in range(3):
    e.decode_step(list(range(B)))
e.timing(reset=True)
for _ in range(6):
    e.decode_step(list(range(B)))
ms, n = e.timing(reset=True)
print(f"full-KV decode step {ms / n:.3f} ms")
