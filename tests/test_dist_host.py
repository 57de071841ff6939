"""Multi-process host tests of the distributed paths (CPU, gloo, world size 2).

* The six-step chunk algebra of csrc/dist.cu (tests/dist_emulator.py), with the
  split chosen by libfftc's planner, exchanged by torch.distributed.all_to_all over
  gloo between two processes, matches the fp64 oracle.
* The same algebra with P = 4 and 8 virtual ranks in one process (list exchange).
* Batch sharding: each rank's contiguous shard of the one seeded batch
  (drawn with PCG64.advance) equals the same rows of the one-GPU input, and the shards'
  transforms gathered over gloo equal the unsharded result bit for bit.
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


def test_shard_rows_equal_the_one_gpu_stream():
    """A rank's batch shard, drawn with PCG64.advance, is bit-identical to the same rows of the
    one-GPU input, for every partition used by bench.py --gpus P."""
    for N, B in [(8, 1 << 10), (60, 1000), (105, 639), (4096, 16)]:
        full = synth.uniform_c64(N, B, seed=0)
        for P in (1, 2, 3, 4, 8):
            parts = [synth.uniform_c64_rows(N, *synth.shard_range(B, r, P), seed=0) for r in range(P)]
            assert np.array_equal(np.concatenate(parts), full), (N, B, P)
    # a six-step slab is the same thing with N = 1 row element stride: elements [p N/P, (p+1) N/P)
    v = synth.uniform_c64(1 << 12, 1, seed=0)[0]
    for p in range(4):
        slab = synth.uniform_c64_rows(1, p << 10, (p + 1) << 10, seed=0).reshape(-1)
        assert np.array_equal(slab, v[p << 10:(p + 1) << 10])


def test_shard_range_partition():
    for B in (0, 1, 7, 16384, 1118481, 21474):
        for P in (1, 2, 3, 4, 8):
            r = [synth.shard_range(B, k, P) for k in range(P)]
            assert r[0][0] == 0 and r[-1][1] == B
            assert all(r[k][1] == r[k + 1][0] for k in range(P - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def _shard_worker(rank, world, port, N, B, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, b1 = synth.shard_range(B, rank, world)
        y = oracle.fft_ct(synth.uniform_c64_rows(N, b0, b1, seed=0), -1, nthreads=1)
        t = torch.from_numpy(np.ascontiguousarray(y).view(np.float64).reshape(-1))
        sizes = [(synth.shard_range(B, r, world)[1] - synth.shard_range(B, r, world)[0]) * N * 2
                 for r in range(world)]
        outs = [t if r == rank else torch.empty(n, dtype=torch.float64) for r, n in enumerate(sizes)]
        for r in range(world):  # shards may differ in size by one transform: broadcast each
            dist.broadcast(outs[r], r)
        if rank == 0:
            q.put(np.concatenate([o.numpy() for o in outs]).view(np.complex128).reshape(B, N))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,B", [(64, 96), (105, 37)])
def test_batch_shards_gloo_world2(N, B):
    """Batch sharding over two processes (gloo): each rank transforms its contiguous shard of the
    one seeded batch; the gathered result equals the unsharded transform bit for bit."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, N, B, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.fft_ct(synth.uniform_c64(N, B, seed=0), -1, nthreads=1)
    assert np.array_equal(got, ref)