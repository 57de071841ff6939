"""The JIT emitter's straight-line codelets (jit.cpp, via fftc_jit_codelet_source) compiled
for the host with g++ and checked against the definition (the oracle's naive DFT): every
prime up to 61 (conjugate-pair form), Eq. 2 composites and the coprime splits that take
the Good-Thomas index maps (DESIGN reading 19).  No GPU needed."""
import os
import subprocess

import numpy as np
import pytest

import oracle

import paper_2207_06803_b200 as fftc

RADICES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 19, 20, 21, 22, 23, 25, 26, 27, 28, 29,
           30, 31, 32, 33, 35, 37, 39, 41, 43, 47, 53, 59, 61, 63, 64, 77, 121, 128]

PRELUDE = """#include <math.h>
#include <stdio.h>
#define __device__
#define __forceinline__ inline
struct cf { float x, y; };
"""


@pytest.fixture(scope="module")
def codelet_outputs(tmp_path_factory):
    d = tmp_path_factory.mktemp("jitcodelets")
    body = [PRELUDE]
    calls = []
    for R in RADICES:
        src = fftc.fftc_jit_codelet_source(R)
        assert src and ("void dft%d(cf* v)" % R) in src, R
        body.append(src)
        calls.append("""  { cf v[%d]; for (int n = 0; n < %d; ++n) { v[n].x = (float)sin(n + 1.0); v[n].y = (float)cos(2.0 * n + 1.0); }
    dft%d(v); for (int k = 0; k < %d; ++k) printf("%d %%d %%.9e %%.9e\\n", k, v[k].x, v[k].y); }""" % (R, R, R, R, R))
    body.append("int main() {\n" + "\n".join(calls) + "\n  return 0;\n}\n")
    c = d / "codelets.cpp"
    c.write_text("\n".join(body))
    exe = str(d / "codelets")
    r = subprocess.run(["g++", "-O1", "-o", exe, str(c), "-lm"], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail("g++ failed:\n" + r.stderr[-4000:])
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    res = {}
    for line in out.split("\n"):
        if line.strip():
            R, k, re, im = line.split()
            res.setdefault(int(R), {})[int(k)] = complex(float(re), float(im))
    return res


def test_codelet_source_domain():
    assert fftc.fftc_jit_codelet_source(1) is None
    assert fftc.fftc_jit_codelet_source(129) is None


@pytest.mark.parametrize("R", RADICES)
def test_jit_codelet_matches_definition(codelet_outputs, R):
    n = np.arange(R)
    x = (np.sin(n + 1.0).astype(np.float32) + 1j * np.cos(2.0 * n + 1.0).astype(np.float32)).astype(np.complex64)
    ref = oracle.dft_naive(x[None], -1)[0]
    y = np.array([codelet_outputs[R][k] for k in range(R)])
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err < 2e-6 * max(1.0, np.log2(R)), (R, err)

