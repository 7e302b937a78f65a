"""Regenerate tests/golden/hf_tiny_logits.npz: Hugging Face transformers
LlamaForCausalLM (fp64, CPU) on the tiny configs[0] model -- weights
tiny_weights(TINY, seed=7), a 4096-token synthetic prefix (seed 1), first
token 17 -- over a 9-row window.  The GPU tests (tests/test_model_parity.py)
compare the engine's logits with this third-party output directly; the CPU
test tests/test_oracle_hf.py checks the fixture is still what HF computes.

    python tests/golden/make_hf_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import hf_llama as H  # noqa: E402
import vc_testlib as T  # noqa: E402
from paper_2605_17613_b200 import TINY  # noqa: E402

TOKENS = [17, 3, 99, 1024, 5, 6, 7, 8, 9]

if __name__ == "__main__":
    w = T.tiny_weights(TINY, seed=7, std=0.02)
    k, v = T.synthetic_kv(TINY.layers, TINY.n_kv, 4096, TINY.d_head, seed=1)
    hf = H.forward(H.build(TINY, w), TINY, k, v, TOKENS)
    np.savez_compressed(os.path.join(HERE, "hf_tiny_logits.npz"), tokens=np.array(TOKENS, np.int32),
                        logits=hf.astype(np.float32), n_ctx=np.int32(4096))
    print("wrote hf_tiny_logits.npz", hf.shape)
