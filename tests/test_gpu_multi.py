"""Multi-GPU tests (SURVEY §8(c) c8 tier T5): need >= 2 GPUs, skipped otherwise.

* batch shards over P = 2/4/8 NCCL ranks equal the unsharded 1-GPU output bit for bit and pass
  the oracle gate (tests/mp_check.py shards);
* the distributed six-step at N = 2^24 over NCCL (three all-to-alls, fused peer stores, fused +
  transposed output) matches the full fp64 O2 (tests/mp_check.py sixstep);
* bench.py --gpus P launches P ranks and reports gpus_active == P;
* a plan refuses to execute while another device is current (FFTC_ERROR_WRONG_DEVICE).
The host side of all of this runs on CPU in tests/test_dist_host.py (gloo, world size 2).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
import paper_2207_06803_b200 as fftc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(NDEV < 2, reason="needs >= 2 GPUs")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(P, *args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(P),
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + list(args)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    return r


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("mode", ["shards", "sixstep"])
def test_multi_gpu(P, mode):
    if NDEV < P:
        pytest.skip("needs %d GPUs" % P)
    r = _torchrun(P, os.path.join(ROOT, "tests", "mp_check.py"), mode)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["failures"] == 0 and line["world"] == P


def test_bench_launches_ranks():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--no-e2e", "--no-cpu",
                        "--no-extras"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["multi_gpu"]["gpus_active"] == 2 and line["multi_gpu"]["comm_nranks_ok"]


def test_wrong_device_rejected():
    torch.cuda.set_device(0)
    with fftc.Plan(64, 16, -1) as p:
        x = torch.zeros(64 * 16, dtype=torch.complex64, device="cuda:0")
        y = torch.empty_like(x)
        torch.cuda.set_device(1)
        try:
            assert fftc.fftc_execute(p.handle, x.data_ptr(), y.data_ptr(), 0) == fftc.FFTC_ERROR_WRONG_DEVICE
        finally:
            torch.cuda.set_device(0)
