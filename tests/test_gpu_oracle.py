"""The drop-in boundary, end to end: the reference's protocol code drives the
B200 engine through include/speckv_gpu_oracle.hpp (TokenOracle adapters over
the C-ABI), and the speculative output is identical to full-KV greedy decode
(the losslessness property of proj/tests/acceptance_test.cpp:55-79, C1).

CPU: the adapter compiles against BOTH the reference's own headers
(/root/reference/proj/include, when present) and include/speckv_b200.hpp, and
the test program links against libvericache.so.  GPU: the program runs."""
import os
import subprocess

import pytest

import vc_testlib as T

BUILD = os.path.join(T.ROOT, "tests", "_build")
SRC = os.path.join(T.ROOT, "tests", "cpp", "gpu_oracle_run.cpp")
EXE = os.path.join(BUILD, "gpu_oracle_run")
LIBDIR = os.path.join(T.ROOT, "paper_2605_17613_b200")
REF_INC = "/root/reference/proj/include"


def _build():
    os.makedirs(BUILD, exist_ok=True)
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(T.ROOT, "include", "speckv_gpu_oracle.hpp")),
            os.path.getmtime(os.path.join(LIBDIR, "libvericache.so"))):
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(T.ROOT, "include"), SRC,
                               "-L", LIBDIR, "-lvericache", "-Wl,-rpath,$ORIGIN/../../paper_2605_17613_b200",
                               "-o", EXE])
    return EXE


def test_adapter_builds_and_links():
    assert os.path.exists(_build())


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_adapter_compiles_against_reference_headers(tmp_path):
    tu = tmp_path / "tu.cpp"
    tu.write_text('#include "speckv/specloop.hpp"\n#include "speckv/compressor.hpp"\n'
                  '#include "speckv_gpu_oracle.hpp"\n'
                  "speckv::TokenOracle f(vc_engine* e) {\n"
                  "  speckv::gpu::SlotOracles o(e, 0);\n"
                  "  return o.drafter<speckv::TokenOracle>();\n}\n"
                  "speckv::CompressedKVMeta g(vc_engine* e, const speckv::CompressorSpec& s) {\n"
                  "  return speckv::gpu::compress<speckv::CompressedKVMeta>(e, 0, s, 0.25, 7);\n}\n")
    subprocess.check_call(["g++", "-std=c++20", "-fsyntax-only", "-I", REF_INC, "-I",
                           os.path.join(T.ROOT, "include"), str(tu)])


@pytest.mark.gpu
@pytest.mark.parametrize("x,bits,tier", [(1, 4, 0), (4, 4, 0), (8, 2, 0), (16, 4, 0), (6, 4, 1)])
def test_reference_protocol_drives_engine_losslessly(cuda, x, bits, tier):
    r = subprocess.run([_build(), str(x), "40", str(bits), str(tier)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK"), r.stdout
