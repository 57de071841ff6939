"""Multi-process host tests of the distributed paths (CPU, gloo, world size 2).

* The six-step chunk algebra of csrc/dist.cu (tests/dist_emulator.py), with the
  split chosen by libfftc's planner, exchanged by torch.distributed.all_to_all over
  gloo between two processes, matches the fp64 oracle.
* The same algebra with P = 4 and 8 virtual ranks in one process (list exchange).
* Batch sharding (weak scaling): each rank's seeded batch is distinct and
  reproducible, and per-rank oracle results combine by max over ranks.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
import paper_2207_06803_b200 as fftc
from tests.dist_emulator import six_step_rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, sign, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        split = fftc.fftc_dist_split(N, world)
        x = synth.uniform_c64(N, 1, seed=11)[0]
        slab = N // world
        x_p = x[rank * slab:(rank + 1) * slab].astype(np.complex128)

        def a2a(send):
            s = torch.from_numpy(np.ascontiguousarray(send).view(np.float64).reshape(world, -1))
            r = torch.empty_like(s)
            dist.all_to_all_single(r, s)
            return r.numpy().view(np.complex128).reshape(world, -1)

        X_p = six_step_rank(x_p, N, world, rank, split, a2a, sign)
        ref = oracle.fft_ct(x[None], sign)[0][rank * slab:(rank + 1) * slab]
        err = float(np.linalg.norm(X_p - ref) / np.linalg.norm(ref))
        errs = torch.tensor([err], dtype=torch.float64)
        dist.all_reduce(errs, op=dist.ReduceOp.MAX)
        q.put((rank, errs.item(), split))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,sign", [(1 << 16, -1), (1 << 20, 1), (1 << 22, -1)])
def test_six_step_gloo_world2(N, sign):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, sign, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, split in res:
        assert err < 1e-12, (rank, err, split)


@pytest.mark.parametrize("N,P", [(1 << 16, 4), (1 << 20, 8), (1 << 22, 4), (1 << 26, 8)])
def test_six_step_virtual_ranks(N, P):
    split = fftc.fftc_dist_split(N, P)
    assert split is not None and split[0] * split[1] == N and split[2] * split[3] == split[1]
    x = synth.uniform_c64(N, 1, seed=3)[0].astype(np.complex128)
    slab = N // P
    # run all ranks step by step with an in-process exchange
    import threading
    barrier = threading.Barrier(P)
    boxes = [None] * P
    outs = [None] * P

    def run(p):
        def a2a(send):
            boxes[p] = send
            barrier.wait()
            recv = np.stack([boxes[s][p] for s in range(P)])
            barrier.wait()
            return recv
        outs[p] = six_step_rank(x[p * slab:(p + 1) * slab], N, P, p, split, a2a, -1)

    th = [threading.Thread(target=run, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    X = np.concatenate(outs)
    ref = np.fft.fft(x) if N > (1 << 22) else oracle.fft_ct(x.astype(np.complex64)[None])[0]
    assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-12


def test_dist_split_properties():
    for N in [1 << k for k in range(16, 31)]:
        for P in (1, 2, 4, 8):
            s = fftc.fftc_dist_split(N, P)
            assert s is not None, (N, P)
            M, K, K1, K2 = s
            assert M * K == N and K1 * K2 == K and M % P == 0 and K % P == 0
            assert M <= 4096 and K1 <= 4096 and K2 <= 4096
    assert fftc.fftc_dist_split(1 << 30, 8) == (4096, 1 << 18, 512, 512)
    assert fftc.fftc_dist_split(11 * 4096, 2) is None


def test_shard_seeds_distinct_and_reproducible():
    a0 = synth.uniform_c64(64, 8, seed=synth.shard_seed(0, 0))
    a1 = synth.uniform_c64(64, 8, seed=synth.shard_seed(0, 1))
    assert np.array_equal(a0, synth.uniform_c64(64, 8, seed=0))
    assert not np.array_equal(a0, a1)
    assert np.array_equal(a1, synth.uniform_c64(64, 8, seed=synth.shard_seed(0, 1)))
