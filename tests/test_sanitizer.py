"""compute-sanitizer memcheck over a small end-to-end run of every kernel
family (tools/sanitize_smoke.py): no out-of-bounds or misaligned access.
(sanitizers on the kernels.)"""
import os
import shutil
import subprocess
import sys

import pytest

import vc_testlib as T

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(shutil.which("compute-sanitizer") is None, reason="compute-sanitizer not on PATH")
def test_memcheck_clean(cuda):
    r = subprocess.run(["compute-sanitizer", "--tool", "memcheck", "--print-limit", "10", sys.executable,
                        os.path.join(T.ROOT, "tools", "sanitize_smoke.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "sanitize smoke ok" in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
