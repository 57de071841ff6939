"""Multi-GPU checks run by tests/test_gpu_multi.py under torch.distributed.run (one process per
GPU, NCCL).  Exits non-zero on the first failure; rank 0 prints one JSON summary line.

    python -m torch.distributed.run --nproc-per-node P tests/mp_check.py shards|sixstep

shards : SURVEY §8(e) batch sharding -- rank r transforms its contiguous shard
         [floor(rB/P), floor((r+1)B/P)) of the seeded C2/C3 input (PCG64.advance); its output
         must equal, bit for bit, the same rows of the unsharded 1-GPU transform (every transform
         is computed the same way wherever it sits in the batch), and pass the oracle gate on
         sampled transforms.
sixstep: the distributed six-step over NCCL (default exchanges, fused peer stores, fused +
         transposed output) at N = 2^24 against the full fp64 O2 (Eq. 2: the
         all-to-alls realise the global permutation Pi^N_K).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    import torch
    import torch.distributed as dist
    import paper_2207_06803_b200 as fftc

    mode = sys.argv[1]
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    fails, report = [], []

    def gpu(x, N, b, sign):
        with fftc.Plan(N, b, sign) as p:
            y = p(torch.from_numpy(np.ascontiguousarray(x)).to(dev))
        torch.cuda.synchronize(dev)
        return y.cpu().numpy().reshape(b, N)

    if mode == "shards":
        for N, B, sign in [(8, 1 << 23, -1), (64, 1 << 20, 1), (4096, 1 << 14, -1), (1000, (1 << 26) // 1000, -1),
                           (3125, (1 << 26) // 3125, 1), (1 << 16, 64, -1)]:
            b0, b1 = synth.shard_range(B, rank, world)
            xs = synth.uniform_c64_rows(N, b0, b1, seed=0)
            ys = gpu(xs, N, b1 - b0, sign)
            # the unsharded transform (same kernels, this GPU) of the whole batch, rows [b0, b1)
            full = gpu(synth.uniform_c64(N, B, seed=0), N, B, sign)[b0:b1]
            if not np.array_equal(ys, full):
                fails.append("shard != unsharded rows: N=%d rank=%d" % (N, rank))
            idx = np.unique(np.r_[0, b1 - b0 - 1, np.random.default_rng(rank).integers(0, b1 - b0, 6)])
            err = float(oracle.rel_l2(ys[idx], oracle.fft_ct(xs[idx], sign)).max())
            if err > oracle.tolerance(N):
                fails.append("gate: N=%d rank=%d err=%.3e" % (N, rank, err))
            report.append({"N": N, "rank": rank, "rows": [b0, b1], "rel_l2": err})
    elif mode == "sixstep":
        N = 1 << 24
        slab = N // world
        x = synth.uniform_c64(N, 1, seed=5)[0]
        ref = {s: oracle.fft_ct(x[None], s)[0] for s in (-1, 1)}
        M, K, K1, K2 = fftc.fftc_dist_split(N, world)
        Mp = M // world
        for flags in (0, 2, 3):
            for sign in (-1, 1):
                idt = torch.zeros(fftc.FFTC_NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
                if rank == 0:
                    idt.copy_(torch.frombuffer(bytearray(fftc.fftc_dist_get_unique_id()), dtype=torch.uint8))
                dist.broadcast(idt, 0)
                with fftc.Plan.dist(N, sign, bytes(idt.cpu().numpy().tobytes()), rank, world, flags=flags) as p:
                    xd = torch.from_numpy(np.ascontiguousarray(x[rank * slab:(rank + 1) * slab])).to(dev)
                    yd = torch.empty_like(xd)
                    p.execute(xd, yd)
                    torch.cuda.synchronize(dev)
                    y = yd.cpu().numpy()
                if flags & 1:  # transposed output: out[k1*Mp + jl] = X[rank*Mp + jl + M*k1]
                    k1, jl = np.divmod(np.arange(slab), Mp)
                    want = ref[sign][rank * Mp + jl + M * k1]
                else:
                    want = ref[sign][rank * slab:(rank + 1) * slab]
                err = float(np.linalg.norm(y - want) / np.linalg.norm(want))
                if not err <= oracle.tolerance(N):
                    fails.append("six-step flags=%d sign=%d rank=%d err=%.3e" % (flags, sign, rank, err))
                report.append({"flags": flags, "sign": sign, "rank": rank, "rel_l2": err})
    else:
        raise SystemExit("unknown mode " + mode)

    nf = torch.tensor([len(fails)], device=dev)
    dist.all_reduce(nf)
    allrep = [None] * world
    dist.all_gather_object(allrep, {"fails": fails, "report": report})
    if rank == 0:
        print(json.dumps({"mode": mode, "world": world, "failures": int(nf.item()), "ranks": allrep}), flush=True)
    dist.destroy_process_group()
    sys.exit(1 if nf.item() else 0)


if __name__ == "__main__":
    main()
