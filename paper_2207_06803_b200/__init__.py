"""paper_2207_06803_b200 -- batched 1D complex DFT on B200 (sm_100a), Python binding.

Thin ctypes binding over ``libfftc.so`` (C ABI declared in ``include/fftc.h``).
Argument marshalling only: every step of the transform runs in the library's
CUDA kernels.  torch supplies device memory and streams.  There is no CPU
fallback: if the library or a CUDA device is missing, calls raise.

Functions keep the C names (``fftc_plan_create``, ``fftc_execute``,
``fftc_execute_host``, ``fftc_plan_destroy``, ``fftc_last_error``,
``fftc_status_string``, ``fftc_plan_describe``, ``fftc_plan_launches``,
``fftc_factorize``, ``fftc_plan_split``, ``fftc_dist_get_unique_id``,
``fftc_dist_plan_create``, ``fftc_dist_split``, ``fftc_candidates``, ``fftc_plan_passes``, ``fftc_plan_gpasses``); :class:`Plan` is a convenience wrapper that owns a
plan handle and takes contiguous ``torch.complex64`` CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# FFTC_LIB_PATH: an alternative in-tree build of the same library (A/B timing of build variants).
LIB_PATH = os.environ.get("FFTC_LIB_PATH") or os.path.join(_PKG, "libfftc.so")

FFTC_SUCCESS = 0
FFTC_ERROR_INVALID_VALUE = 1
FFTC_ERROR_UNSUPPORTED_SIZE = 2
FFTC_ERROR_MISALIGNED = 3
FFTC_ERROR_OUT_OF_MEMORY = 4
FFTC_ERROR_CUDA = 5
FFTC_ERROR_NCCL = 6
FFTC_ERROR_NO_DEVICE = 7
FFTC_ERROR_WRONG_DEVICE = 8
FFTC_NCCL_ID_BYTES = 128

_lib = None


class FFTCError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__("%s: %s" % (what or "fftc", fftc_status_string(status)))


def load(path: str = LIB_PATH):
    """Load libfftc.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libfftc.so not built: run `python -m paper_2207_06803_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    sig = {
        "fftc_plan_create": ([i64, i64, i32], vp),
        "fftc_execute": ([vp, vp, vp, vp], i32),
        "fftc_execute_host": ([vp, vp, vp], i32),
        "fftc_plan_destroy": ([vp], None),
        "fftc_last_error": ([], i32),
        "fftc_status_string": ([i32], ctypes.c_char_p),
        "fftc_plan_describe": ([vp, ctypes.c_char_p, sz], i32),
        "fftc_plan_launches": ([vp], i32),
        "fftc_factorize": ([i64, ctypes.POINTER(ctypes.c_int), i32], i32),
        "fftc_plan_split": ([i64, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)], i32),
        "fftc_dist_get_unique_id": ([vp], i32),
        "fftc_dist_plan_create": ([i64, i32, vp, i32, i32, i32], vp),
        "fftc_dist_plan_create_ex": ([i64, i32, vp, i32, i32, i32, i32], vp),
        "fftc_dist_split": ([i64, i32, ctypes.POINTER(ctypes.c_int64)], i32),
        "fftc_candidates": ([i64, ctypes.POINTER(ctypes.c_char_p), i32], i32),
        "fftc_plan_passes": ([i64, ctypes.POINTER(ctypes.c_int), i32], i32),
        "fftc_plan_gpasses": ([i64, ctypes.POINTER(ctypes.c_int), i32], i32),
        "fftc_expr_radices": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int), i32,
                               ctypes.c_char_p, sz], i32),
        "fftc_plan_create_radices": ([i64, i64, i32, ctypes.POINTER(ctypes.c_int), i32], vp),
        "fftc_plan_create_expr": ([ctypes.c_char_p, i64, i32], vp),
        "fftc_jit_source": ([i64, ctypes.c_char_p, sz], i32),
        "fftc_jit_codelet_source": ([ctypes.c_int, ctypes.c_char_p, sz], i32),
        "fftc_plan_create_direct": ([i64, i64, i32], vp),
        "fftc_jit_compile": ([i64, ctypes.c_char_p, sz], i32),
        "fftc_jit_pass_compile": ([i32, ctypes.c_char_p, sz], i32),
        "fftc_jit_pass_source": ([i32, ctypes.c_char_p, sz], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


# ---------------------------------------------------------------- C names
def fftc_plan_create(N: int, batch: int, sign: int) -> int:
    return load().fftc_plan_create(N, batch, sign) or 0


def fftc_execute(plan: int, d_in: int, d_out: int, stream: int = 0) -> int:
    return load().fftc_execute(plan, d_in, d_out, stream)


def fftc_execute_host(plan: int, h_in: int, h_out: int) -> int:
    return load().fftc_execute_host(plan, h_in, h_out)


def fftc_plan_destroy(plan: int) -> None:
    load().fftc_plan_destroy(plan)


def fftc_last_error() -> int:
    return load().fftc_last_error()


def fftc_status_string(s: int) -> str:
    return load().fftc_status_string(s).decode()


def fftc_plan_describe(plan: int) -> str:
    buf = ctypes.create_string_buffer(512)
    load().fftc_plan_describe(plan, buf, 512)
    return buf.value.decode()


def fftc_plan_launches(plan: int) -> int:
    return load().fftc_plan_launches(plan)


def fftc_factorize(N: int):
    arr = (ctypes.c_int * 32)()
    S = load().fftc_factorize(N, arr, 32)
    return None if S < 0 else [arr[i] for i in range(S)]


def fftc_candidates(N: int):
    arr = (ctypes.c_char_p * 64)()
    n = load().fftc_candidates(N, arr, 64)
    return [arr[i].decode() for i in range(min(n, 64))]


def fftc_plan_passes(N: int):
    arr = (ctypes.c_int * 8)()
    p = load().fftc_plan_passes(N, arr, 8)
    return None if p < 0 else [arr[i] for i in range(p)]


def fftc_plan_gpasses(N: int):
    arr = (ctypes.c_int * 8)()
    p = load().fftc_plan_gpasses(N, arr, 8)
    return None if p < 0 else [arr[i] for i in range(p)]


def fftc_expr_radices(expr: str):
    """Parse an FFTc factorization expression -> (N, radices); raises ValueError with the
    parser's message if it is not Eq. 2 applied recursively."""
    N = ctypes.c_int64()
    arr = (ctypes.c_int * 64)()
    err = ctypes.create_string_buffer(256)
    S = load().fftc_expr_radices(expr.encode(), ctypes.byref(N), arr, 64, err, 256)
    if S < 0:
        raise ValueError(err.value.decode())
    return N.value, [arr[i] for i in range(S)]


def fftc_plan_create_radices(N: int, batch: int, sign: int, radices) -> int:
    arr = (ctypes.c_int * max(1, len(radices)))(*radices)
    return load().fftc_plan_create_radices(N, batch, sign, arr, len(radices)) or 0


def fftc_plan_create_expr(expr: str, batch: int, sign: int) -> int:
    return load().fftc_plan_create_expr(expr.encode(), batch, sign) or 0


def fftc_jit_source(N: int):
    n = load().fftc_jit_source(N, None, 0)
    if n < 0:
        return None
    buf = ctypes.create_string_buffer(n + 1)
    load().fftc_jit_source(N, buf, n + 1)
    return buf.value.decode()


def fftc_jit_codelet_source(R: int):
    n = load().fftc_jit_codelet_source(R, None, 0)
    if n < 0:
        return None
    buf = ctypes.create_string_buffer(n + 1)
    load().fftc_jit_codelet_source(R, buf, n + 1)
    return buf.value.decode()


def fftc_jit_compile(N: int):
    """NVRTC-compile the JIT kernel for N (host only) -> (cubin bytes or error code, log)."""
    log = ctypes.create_string_buffer(1 << 16)
    r = load().fftc_jit_compile(N, log, 1 << 16)
    return r, log.value.decode(errors="replace")


def fftc_jit_pass_source(L: int):
    n = load().fftc_jit_pass_source(L, None, 0)
    if n < 0:
        return None
    buf = ctypes.create_string_buffer(n + 1)
    load().fftc_jit_pass_source(L, buf, n + 1)
    return buf.value.decode()


def fftc_jit_pass_compile(L: int):
    log = ctypes.create_string_buffer(1 << 16)
    r = load().fftc_jit_pass_compile(L, log, 1 << 16)
    return r, log.value.decode(errors="replace")


def fftc_plan_split(N: int):
    M, K = ctypes.c_int64(), ctypes.c_int64()
    r = load().fftc_plan_split(N, ctypes.byref(M), ctypes.byref(K))
    return (r, M.value, K.value)


def fftc_dist_split(N: int, nranks: int):
    out = (ctypes.c_int64 * 4)()
    r = load().fftc_dist_split(N, nranks, out)
    return None if r != 0 else tuple(out[i] for i in range(4))


def fftc_dist_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(FFTC_NCCL_ID_BYTES)
    s = load().fftc_dist_get_unique_id(buf)
    if s != FFTC_SUCCESS:
        raise FFTCError(s, "fftc_dist_get_unique_id")
    return buf.raw


FFTC_DIST_TRANSPOSED_OUT = 1
FFTC_DIST_PEER_STORES = 2


def fftc_dist_plan_create(N: int, sign: int, nccl_id: bytes | None, rank: int, nranks: int,
                          loopback: bool = False, flags: int = 0) -> int:
    idbuf = ctypes.create_string_buffer(nccl_id, FFTC_NCCL_ID_BYTES) if nccl_id else None
    return load().fftc_dist_plan_create_ex(N, sign, idbuf, rank, nranks, int(loopback), flags) or 0


# ---------------------------------------------------------------- convenience wrapper
class Plan:
    """Owns an fftc plan.  ``plan(x)`` transforms a contiguous complex64 CUDA tensor
    of ``batch*N`` elements on torch's current stream and returns a new tensor."""

    def __init__(self, N: int, batch: int, sign: int = -1, _handle: int | None = None):
        self.N, self.batch, self.sign = N, batch, sign
        self.elements = N * batch  # complex64 elements of in / out per execute
        self.device = _current_device()
        self.handle = _handle if _handle is not None else fftc_plan_create(N, batch, sign)
        if not self.handle:
            raise FFTCError(fftc_last_error(), "fftc_plan_create(N=%d, batch=%d, sign=%d)" % (N, batch, sign))

    @classmethod
    def from_expr(cls, expr: str, batch: int, sign: int = -1):
        """Plan from an FFTc factorization expression (Listing 1 syntax)."""
        N, _ = fftc_expr_radices(expr)
        h = fftc_plan_create_expr(expr, batch, sign)
        if not h:
            raise FFTCError(fftc_last_error(), "fftc_plan_create_expr(%r)" % expr)
        return cls(N, batch, sign, _handle=h)

    @classmethod
    def direct(cls, N: int, batch: int, sign: int = -1):
        """The paper's direct DFT as a batched dense product on the tensor cores (N = 16, 32)."""
        h = load().fftc_plan_create_direct(N, batch, sign) or 0
        if not h:
            raise FFTCError(fftc_last_error(), "fftc_plan_create_direct(N=%d)" % N)
        return cls(N, batch, sign, _handle=h)

    @classmethod
    def from_radices(cls, N: int, batch: int, sign: int, radices):
        h = fftc_plan_create_radices(N, batch, sign, list(radices))
        if not h:
            raise FFTCError(fftc_last_error(), "fftc_plan_create_radices(N=%d, %s)" % (N, list(radices)))
        return cls(N, batch, sign, _handle=h)

    @classmethod
    def dist(cls, N: int, sign: int, nccl_id: bytes | None, rank: int, nranks: int, loopback: bool = False,
             flags: int = 0):
        h = fftc_dist_plan_create(N, sign, nccl_id, rank, nranks, loopback, flags)
        if not h:
            raise FFTCError(fftc_last_error(), "fftc_dist_plan_create(N=%d, P=%d)" % (N, nranks))
        p = cls.__new__(cls)
        p.N, p.batch, p.sign, p.handle = N, 1, sign, h
        p.elements = N if (loopback or nranks == 1) else N // nranks  # this rank's slab
        p.device = _current_device()
        return p

    def describe(self) -> str:
        return fftc_plan_describe(self.handle)

    def launches(self) -> int:
        return fftc_plan_launches(self.handle)

    def _check(self, x, out, cuda: bool):
        import torch
        for name, t in (("input", x), ("output", out)):
            if hasattr(t, "data_ptr"):
                if t.dtype != torch.complex64 or not t.is_contiguous():
                    raise TypeError("%s: expected a contiguous complex64 tensor" % name)
                if t.is_cuda != cuda:
                    raise TypeError("%s: expected a %s tensor" % (name, "CUDA" if cuda else "host"))
                if cuda and t.device.index != self.device:
                    raise ValueError("%s is on cuda:%d, the plan on cuda:%d" % (name, t.device.index, self.device))
                n = t.numel()
            else:  # numpy array (host)
                if cuda:
                    raise TypeError("%s: expected a CUDA tensor" % name)
                if t.dtype.name != "complex64" or not t.flags["C_CONTIGUOUS"]:
                    raise TypeError("%s: expected a C-contiguous complex64 array" % name)
                n = t.size
            if n < self.elements:  # the kernels touch exactly the first `elements` elements
                raise ValueError("%s has %d elements, the plan needs %d" % (name, n, self.elements))

    def execute(self, x, out, stream=None):
        """Enqueue the transform of x into out on `stream` (default: torch's current stream of the
        plan's device).  Both must be contiguous complex64 tensors on the plan's device with at
        least N*batch elements (checked here: the C ABI receives bare pointers)."""
        # fast checks first (one call per property; the launch-bound small sizes feel every us)
        d = self.device
        if (x.dtype is not _c64() or out.dtype is not _c64() or x.get_device() != d or out.get_device() != d
                or not x.is_contiguous() or not out.is_contiguous() or x.numel() < self.elements
                or out.numel() < self.elements):
            self._check(x, out, cuda=True)  # raises with the precise message
            raise TypeError("invalid tensors")  # pragma: no cover  (_check always raises here)
        if stream is None:
            stream = _current_stream(d)
        s = _lib_fn("fftc_execute")(self.handle, x.data_ptr(), out.data_ptr(), stream)
        if s != FFTC_SUCCESS:
            raise FFTCError(s, "fftc_execute")
        return out

    def __call__(self, x, out=None):
        import torch
        if x.dtype != torch.complex64 or not x.is_cuda or not x.is_contiguous():
            raise TypeError("expected a contiguous complex64 CUDA tensor")
        if x.numel() < self.elements:
            raise ValueError("input has %d elements, the plan needs %d" % (x.numel(), self.elements))
        if out is None:
            out = torch.empty_like(x)
        return self.execute(x, out)

    def execute_host(self, x_host, out_host):
        """End to end on host (ideally pinned) tensors/arrays: H2D, transform, D2H."""
        self._check(x_host, out_host, cuda=False)
        s = fftc_execute_host(self.handle, _ptr(x_host), _ptr(out_host))
        if s != FFTC_SUCCESS:
            raise FFTCError(s, "fftc_execute_host")
        return out_host

    def close(self):
        if getattr(self, "handle", 0):
            fftc_plan_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


_C64 = None
_FNS = {}


def _c64():
    global _C64
    if _C64 is None:
        import torch
        _C64 = torch.complex64
    return _C64


def _lib_fn(name):
    f = _FNS.get(name)
    if f is None:
        f = _FNS[name] = getattr(load(), name)
    return f


def _current_stream(device: int) -> int:
    """Raw cudaStream_t of torch's current stream on `device`."""
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(device)
    return torch.cuda.current_stream(device).cuda_stream


def _current_device() -> int:
    try:
        import torch
        return torch.cuda.current_device() if torch.cuda.is_available() else -1
    except Exception:
        return -1


def _ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
