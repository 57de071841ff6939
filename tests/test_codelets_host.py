"""Register codelets (codelets.cuh, __host__ __device__) compiled for the host and checked
against the definition (the oracle's naive DFT): every radix the schedules use.  Catches a
wrong index map / twiddle inside a codelet without a GPU."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "host", "codelet_host.cu")


@pytest.fixture(scope="module")
def codelet_output(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("codelets") / "codelet_host")
    r = subprocess.run(["nvcc", "-O2", "-std=c++17", "--expt-relaxed-constexpr", "-o", exe, SRC],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail("nvcc failed:\n" + r.stderr)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    res = {}
    for line in out.split("\n"):
        if not line.strip():
            continue
        R, k, re, im = line.split()
        res.setdefault(int(R), {})[int(k)] = complex(float(re), float(im))
    return res


def test_every_codelet_matches_the_definition(codelet_output):
    assert len(codelet_output) >= 17
    for R, ys in sorted(codelet_output.items()):
        n = np.arange(R)
        x = (np.sin(n + 1.0).astype(np.float32) + 1j * np.cos(2.0 * n + 1.0).astype(np.float32)).astype(np.complex64)
        ref = oracle.dft_naive(x[None], -1)[0]
        y = np.array([ys[k] for k in range(R)])
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        assert err < 1e-6, (R, err)
