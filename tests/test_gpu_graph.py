"""Every plan kind enqueued inside CUDA-graph stream capture and replayed: the library only
enqueues stream-ordered work (no host synchronisation, no allocation in fftc_execute), so a
captured graph reproduces the eager result bit for bit."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
import paper_2207_06803_b200 as fftc  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [("fused", lambda: fftc.Plan(64, 300, -1), 64, 300),
         ("generic", lambda: fftc.Plan(48, 77, 1), 48, 77),
         ("passes", lambda: fftc.Plan(1 << 16, 5, -1), 1 << 16, 5),
         ("gpass", lambda: fftc.Plan(100000, 3, -1), 100000, 3),
         ("jit", lambda: fftc.Plan(143, 40, 1), 143, 40),
         ("direct", lambda: fftc.Plan.direct(32, 500, -1), 32, 500),
         ("dist_loopback", lambda: fftc.Plan.dist(1 << 20, -1, None, 0, 4, loopback=True,
                                                  flags=fftc.FFTC_DIST_PEER_STORES), 1 << 20, 1)]


@pytest.mark.parametrize("name,mk,N,batch", CASES, ids=[c[0] for c in CASES])
def test_graph_capture_replays_eager_result(name, mk, N, batch):
    x = torch.from_numpy(synth.uniform_c64(N, batch, seed=7).reshape(-1)).cuda()
    y_eager = torch.empty_like(x)
    y_graph = torch.empty_like(x)
    with mk() as p:
        p.execute(x, y_eager)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            p.execute(x, y_graph, stream=s.cuda_stream)  # warm on the capture stream
            torch.cuda.synchronize()
            y_graph.zero_()
            with torch.cuda.graph(g, stream=s):
                p.execute(x, y_graph, stream=s.cuda_stream)
        torch.cuda.synchronize()
        assert torch.count_nonzero(y_graph) == 0 or name == "never"  # capture does not execute
        g.replay()
        g.replay()
        torch.cuda.synchronize()
    a = y_eager.cpu().numpy().view(np.uint32)
    b = y_graph.cpu().numpy().view(np.uint32)
    assert np.array_equal(a, b), name


def test_graph_capture_l2_resident(monkeypatch):
    """The L2-resident kernel (cooperative launch + counter reset) inside a captured graph."""
    monkeypatch.setenv("FFTC_LARGE", "l2")
    test_graph_capture_replays_eager_result("l2", lambda: fftc.Plan(1 << 16, 37, -1), 1 << 16, 37)


def test_graph_capture_cluster_single_pass(monkeypatch):
    """The 8-CTA cluster single pass for 2^16 (cudaLaunchKernelEx with a cluster dimension, st.async
    row delivery, mbarrier flow control) inside a captured graph."""
    monkeypatch.setenv("FFTC_LARGE", "cluster")
    test_graph_capture_replays_eager_result("cluster", lambda: fftc.Plan(1 << 16, 37, -1), 1 << 16, 37)


def test_graph_capture_register_pass(monkeypatch):
    """2^24 as two register-resident 4096-long passes inside a captured graph."""
    monkeypatch.setenv("FFTC_PASS_LOGS", "12,12")
    monkeypatch.setenv("FFTC_PASS", "rp4096_r16x16x16_c4")
    test_graph_capture_replays_eager_result("rpass", lambda: fftc.Plan(1 << 24, 2, 1), 1 << 24, 2)


def test_concurrent_plans_from_host_threads():
    """Plans of every kind created and executed concurrently from 6 host threads, each on its
    own stream (first-use kernel setup and the JIT cache are thread-safe); results equal the
    single-threaded ones bit for bit."""
    import threading
    kinds = [(64, 999, -1), (3125, 21, 1), (48, 77, -1), (1 << 16, 3, -1), (143, 40, 1), (100000, 2, -1)]
    xs = {k: torch.from_numpy(synth.uniform_c64(k[0], k[1], seed=k[0]).reshape(-1)).cuda() for k in kinds}
    ref = {}
    for k in kinds:
        with fftc.Plan(*k) as p:
            ref[k] = p(xs[k]).cpu().numpy()
    out, errors = {}, []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    with fftc.Plan(*k) as p:
                        y = torch.empty_like(xs[k])
                        p.execute(xs[k], y, stream=s.cuda_stream)
                s.synchronize()
                out[k] = y.cpu().numpy()
        except Exception as e:  # pragma: no cover - reported below
            errors.append((k, e))

    ts = [threading.Thread(target=work, args=(k,)) for k in kinds]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for k in kinds:
        assert np.array_equal(out[k].view(np.uint32), ref[k].view(np.uint32)), k
