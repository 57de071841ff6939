/*
 * fftc.h -- C ABI of libfftc.so: batched 1D complex DFT on NVIDIA B200 (sm_100a).
 *
 * The operation (§Background): for each of `batch` independent
 * transforms,
 *     Y[b, k] = sum_{n=0}^{N-1} X[b, n] * w^{n k},   w = exp(sign * 2*pi*i / N),
 * unnormalised, natural order, out of place.  sign = -1 is the paper's DFT_N
 * (w_N = exp(-2*pi*i/N)); sign = +1 is the unnormalised inverse (our reading,
 * DESIGN.md §3 #1).  It is computed as the paper's general-radix
 * decimation-in-time Cooley-Tukey factorization (Eq. 2)
 *     DFT_N = (DFT_K (x) I_M) D^N_M (I_K (x) DFT_M) Pi^N_K,   N = M K,
 * applied recursively: each Stockham stage of the fused kernels is one level of
 * Eq. 2, the four-step path is Eq. 2 once at the top with M, K both large, and
 * the distributed six-step path realises Pi^N_K as NCCL all-to-alls.
 *
 * Data layout: `in` / `out` hold batch*N complex64 values, interleaved
 * (re, im) fp32; element (b, n) is at float offset 2*(b*N + n).
 * Device pointers unless the function says HOST.  All pointers must be
 * 16-byte aligned.  The caller owns in/out; `in` is never written.
 *
 * Errors: every call returns a status (never aborts).  A kernel fault is
 * reported by the next call that checks, as in CUDA.
 *
 * Thread safety: plans are immutable after create.  Single-pass plans are
 * re-entrant across streams.  Plans with a workspace (four-step, six-step,
 * host-staged execution) must not be executed concurrently on two streams.
 */
#ifndef FFTC_H_
#define FFTC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fftc_plan fftc_plan; /* opaque */

typedef enum {
  FFTC_SUCCESS = 0,
  FFTC_ERROR_INVALID_VALUE = 1,    /* N < 1, batch < 0, sign not in {-1,+1}, NULL pointer,
                                      in == out or overlapping buffers */
  FFTC_ERROR_UNSUPPORTED_SIZE = 2, /* N has a prime factor > 61, or one > 7 and NVRTC is unavailable
                                      (JIT sizes); N > 512^4; N*batch*8 overflows;
                                      dist: nranks does not divide M and K */
  FFTC_ERROR_MISALIGNED = 3,       /* in / out not 16-byte aligned */
  FFTC_ERROR_OUT_OF_MEMORY = 4,    /* twiddle table / workspace allocation failed */
  FFTC_ERROR_CUDA = 5,             /* CUDA launch / runtime error (cudaGetLastError captured) */
  FFTC_ERROR_NCCL = 6,             /* distributed plan: NCCL failure */
  FFTC_ERROR_NO_DEVICE = 7,        /* no CUDA device / not an sm_100 device */
  FFTC_ERROR_WRONG_DEVICE = 8      /* execute called while a device other than the plan's is
                                      current (a plan is bound to the device current at create) */
} fftc_status;

/* Create a plan for `batch` transforms of length N with direction `sign`.
 * Factors N into the radix schedule (planner, "N = MK" applied
 * recursively), builds fp32 twiddle tables from double on the host and
 * uploads them to the current device; allocates the four-step workspace
 * (N*batch*8 bytes) when N exceeds the single-pass limit (4096).
 * batch == 0 is valid (execute is then a no-op).  N == 1 is a copy.
 * Returns NULL on failure; the reason is fftc_last_error().               */
fftc_plan* fftc_plan_create(int64_t N, int64_t batch, int sign);

/* Enqueue the transform on `stream` (a cudaStream_t; NULL = legacy default
 * stream).  Asynchronous: never synchronises the host.  in/out: device
 * pointers as described above, out-of-place (in != out, no overlap).
 * The device current on the calling thread must be the one the plan was
 * created on (else FFTC_ERROR_WRONG_DEVICE, nothing enqueued).            */
fftc_status fftc_execute(const fftc_plan* plan, const void* in, void* out, void* stream);

/* End-to-end form of fftc_execute on HOST buffers (pinned or pageable;
 * the plan's device must be current, as for fftc_execute):
 * copies in -> device, runs the transform, copies the result back, in
 * chunks of transforms pipelined over two streams so host<->device copies
 * overlap the kernels.  Synchronous: returns after `out` is written.
 * Uses a plan-owned device staging area (allocated on first use).         */
fftc_status fftc_execute_host(fftc_plan* plan, const void* host_in, void* host_out);

/* Free tables and workspace.  NULL-safe. */
void fftc_plan_destroy(fftc_plan* plan);

/* Status of the last fftc_plan_create on this thread. */
fftc_status fftc_last_error(void);
const char* fftc_status_string(fftc_status s);

/* Human-readable plan summary into buf (radices, passes, kernel, workspace
 * bytes, launches per execute).  Returns the number of characters written
 * (excluding NUL), or -1 if plan is NULL.                                  */
int fftc_plan_describe(const fftc_plan* plan, char* buf, size_t len);

/* Number of kernel launches one fftc_execute of this plan enqueues. */
int fftc_plan_launches(const fftc_plan* plan);

/* Planner, host only (no device needed): the radix schedule R_0..R_{S-1}
 * (R_0 = innermost, leaf DFT; prod R_s = N) the single-pass path uses for N.
 * Writes up to `max` radices, returns the stage count S (0 for N == 1), or
 * -1 if N < 1 or N has a prime factor > 7.  For N above the single-pass
 * limit this is the schedule of the whole length; the executed path is
 * given by fftc_plan_split().                                              */
int fftc_factorize(int64_t N, int* radices, int max);

/* Planner introspection (host only): names of the compiled single-pass
 * schedules for N, default first; writes up to `max` pointers to static
 * strings, returns the count.  Setting the environment variable
 * FFTC_KERNEL=<name> before fftc_plan_create pins the planner to that
 * candidate (used by the tuner, tools/tune.py, and the per-candidate tests). */
int fftc_candidates(int64_t N, const char** names, int max);

/* Two-level split for N: returns 1 (single pass: *M = N, *K = 1),
 * 2 (four-step: N = M*K, column DFT_M then row DFT_K), or -1 unsupported.
 * Powers of two above 4096 run the multi-pass path instead (fftc_plan_passes)
 * unless the environment variable FFTC_LARGE selects another large-N path at
 * plan creation: fourstep (the classic two-kernel four-step), l2 (all passes
 * in one L2-resident kernel, 2^13..2^21), gpass (runtime-schedule passes) or
 * cluster (N = 65536 only: one HBM round trip on a cluster of eight CTAs).  */
int fftc_plan_split(int64_t N, int64_t* M, int64_t* K);

/* Multi-pass split (host only): power-of-two N in [2^9, 2^48] as p passes
 * of lengths L_s (product N), each one level of Eq. 2 in Stockham form over
 * HBM: 2^17..2^20 two passes of <= 1024, 2^21..2^23 two passes with a
 * 2048/4096-long first pass, 2^25..2^28 three passes ending in 256, every
 * other N ceil(log2 N / 8) passes of lengths in [16, 256].  Writes up to `max`
 * lengths, returns p, or -1 if N is not such a power of two.              */
int fftc_plan_passes(int64_t N, int* lengths, int max);

/* Runtime-schedule multi-pass split (host only): for a 7-smooth N > 4096
 * that is not a power of two (those run fftc_plan_passes), the fewest
 * passes p in [2, 4] with lengths L_s <= 512 (each pass a JIT kernel
 * specialised to its length; <= 256 without NVRTC or with
 * FFTC_GPASS_JIT=0), product N, longest first;
 * each pass is one level of Eq. 2 in Stockham form over HBM, its
 * DFT_{L_s} built from the generic radices {16, 8, 4, 2, 9, 3, 25, 5, 7}.
 * Writes up to `max` lengths, returns p, or -1 (N <= 4096, a prime
 * factor > 7, or N > 256^4).                                               */
int fftc_plan_gpasses(int64_t N, int* lengths, int max);

/* ---------------------------------------------------------------------
 * FFTc factorization expressions (the paper's DSL front end, P:100-121,
 * Listing 1 / Table 1): e.g.
 *   (DFT(2) ⊗ I(2)) · twiddle(4,2) · (I(2) ⊗ DFT(2)) · Permute(4,2)
 * '⊗' (U+2297) or '&' is the Kronecker product, '·' (U+00B7), '*' or '@'
 * the matrix product; DFT(n), I(n), twiddle(N,M) = D^N_M, Permute(N,K) =
 * Pi^N_K.  The expression must be Eq. 2 applied recursively,
 *   (DFT_K ⊗ I_M) · twiddle(N,M) · (I_K ⊗ X_M) · Permute(N,K),  N = M K,
 * X_M = DFT(M) or again such a factorization (a factored outer DFT_K is
 * flattened into consecutive stages); or a bare DFT(N) (planner's choice).
 * An optional "var name =" prefix, trailing ';' and trailing input
 * identifier (Listing 1's "· InputComplex") are ignored.
 * ------------------------------------------------------------------- */

/* Host only: parse `expr`, write N and its radix schedule R_0..R_{S-1}
 * (R_0 = innermost DFT, the executed Stockham stage order).  Returns S
 * (0 for a bare DFT(N)), or -1 with a message in err (NUL-terminated,
 * truncated to errlen; err may be NULL).                                  */
int fftc_expr_radices(const char* expr, int64_t* N, int* radices, int max, char* err, size_t errlen);

/* Plan with an explicit radix schedule (product = N, each >= 2; S = 0:
 * planner's choice).  N <= 4096: a compiled schedule with exactly these
 * stages if there is one, else the runtime-schedule kernel (radices from
 * {16, 8, 4, 2, 9, 3, 25, 5, 7}); N > 4096: consecutive stages grouped
 * into at most 4 passes of length <= 256.  NULL on failure: INVALID_VALUE
 * (bad product / arguments), UNSUPPORTED_SIZE (a radix outside the
 * runtime set with no compiled schedule, or too many passes).           */
fftc_plan* fftc_plan_create_radices(int64_t N, int64_t batch, int sign, const int* radices, int S);

/* fftc_expr_radices + fftc_plan_create_radices.  INVALID_VALUE if the
 * expression does not parse or is not an Eq. 2 factorization.            */
fftc_plan* fftc_plan_create_expr(const char* expr, int64_t batch, int sign);

/* ---------------------------------------------------------------------
 * JIT mode: an N <= 4096 with prime factors above 7 (up to 61)
 * gets a single-pass kernel generated for that N (larger such N: runtime
 * passes, each a kernel generated for its length) -- Stockham stages, each
 * DFT_R a straight-line codelet emitted by Eq. 2 (primes: conjugate-pair
 * form of the definition) -- compiled by NVRTC for sm_100a when the plan
 * is created (fftc_plan_create; cached per N for the process).  Without
 * libnvrtc such sizes return FFTC_ERROR_UNSUPPORTED_SIZE.
 * ------------------------------------------------------------------- */

/* Host only: the generated CUDA source for N (NUL-terminated, truncated to
 * len).  Returns its length, or -1 if N is not a JIT size.                 */
int fftc_jit_source(int64_t N, char* buf, size_t len);

/* Host only: the straight-line codelet `dft<R>(cf* v)` (in-place forward DFT_R
 * of R complex values, cf = {float x, y}) that the emitter generates -- Eq. 2
 * for composite R (Good-Thomas index maps when the split is coprime), the
 * conjugate-pair form for primes.  2 <= R <= 128; returns its length, or -1.
 * Truncation and NUL termination as fftc_jit_source.                       */
int fftc_jit_codelet_source(int R, char* buf, size_t len);

/* Host only (no device needed): compile the generated source with NVRTC for
 * sm_100a.  Returns the cubin size (> 0), or < 0 (-1 no NVRTC / not a JIT
 * size, -4 compile error); the NVRTC log goes to log (may be NULL).        */
int fftc_jit_compile(int64_t N, char* log, size_t loglen);

/* Host only: the generated CUDA source of the pass kernel for pass length L (the kernel
 * fftc_jit_pass_compile compiles).  Returns its length, or -1 if L is not a JIT pass
 * length.  Truncation and NUL termination as fftc_jit_source.             */
int fftc_jit_pass_source(int L, char* buf, size_t len);

/* Host only: compile the JIT pass kernel for pass length L (<= 4096, prime factors <= 61;
 * the runtime multi-pass path above 4096 specialises each pass this way).  Returns the
 * cubin size, or < 0 as fftc_jit_compile.                                 */
int fftc_jit_pass_compile(int L, char* log, size_t loglen);

/* The paper's "direct" DFT: y = DFT_N x as one dense
 * product per transform, batched into a GEMM on the tcgen05 tensor cores
 * (kind::tf32, 3xTF32 split for fp32-level accuracy), for N in {16, 32}.
 * Same layout, signs and errors as fftc_plan_create; UNSUPPORTED_SIZE for
 * other N.  Opt-in: fftc_plan_create never selects it.                     */
fftc_plan* fftc_plan_create_direct(int64_t N, int64_t batch, int sign);

/* ---------------------------------------------------------------------
 * Distributed six-step (one process per GPU, NCCL over NVLink/NVSwitch).
 * A single transform of length N is block-distributed: rank p holds
 * elements [p*N/P, (p+1)*N/P) of the input and of the output, both in
 * natural order.  N = M*K with P | M and P | K; the three all-to-alls
 * realise the global stride permutations of Eq. 2 (Pi^N_K).
 * ------------------------------------------------------------------- */

/* Size of the opaque NCCL unique id blob. */
#define FFTC_NCCL_ID_BYTES 128

/* Rank 0 calls this and broadcasts the 128 bytes to the other ranks
 * (e.g. over torch.distributed).  Returns FFTC_SUCCESS or FFTC_ERROR_NCCL. */
fftc_status fftc_dist_get_unique_id(void* id_out);

/* Collective over `nranks` processes; each calls it with the same N, sign
 * and id and its own rank, with its GPU current.  nranks == 1 without
 * loopback returns the single-GPU plan for N (the all-to-alls would be
 * identities).  Returns NULL on failure.
 * `loopback` != 0 runs all nranks virtual ranks inside this one process on
 * the current GPU (the all-to-alls become device copies; id/rank ignored):
 * in/out then hold the whole N-element vector.                            */
fftc_plan* fftc_dist_plan_create(int64_t N, int sign, const void* nccl_id, int rank, int nranks,
                                 int loopback);

/* Options of fftc_dist_plan_create_ex (bit flags):
 * FFTC_DIST_TRANSPOSED_OUT: drop all-to-all #3 -- rank p's out holds
 *   out[k1*Mp + jl] = X[p*Mp + jl + M*k1] (k1 < K, jl < Mp = M/P), the
 *   natural output of the last local DFT.
 * FFTC_DIST_PEER_STORES: fuse the exchanges into the kernels around them:
 *   the pack kernel stores each chunk straight into the receiving rank's
 *   buffer and the DFT_M kernel's epilogue does the same for exchange #2
 *   (and the DFT_K epilogue for exchange #3 when DFT_K is one pass)
 *   (P2P stores over NVLink into buffers mapped by CUDA IPC, handles
 *   all-gathered over NCCL at create; a 1-int NCCL all-reduce orders each
 *   exchange).  nranks <= 8.                                               */
#define FFTC_DIST_TRANSPOSED_OUT 1
#define FFTC_DIST_PEER_STORES 2
fftc_plan* fftc_dist_plan_create_ex(int64_t N, int sign, const void* nccl_id, int rank, int nranks,
                                    int loopback, int flags);

/* fftc_execute on a distributed plan: in / out are this rank's
 * N/nranks-element natural-order slabs (device); in loopback mode the whole
 * N-element vectors.  Enqueues 4-5 kernels and 3 all-to-alls per call. */

/* Host only (no device): the split the six-step uses for (N, nranks):
 * out[0..3] = M, K, K1, K2 (K = K1*K2; K2 == 1 when DFT_K is single pass).
 * Returns 0, or -1 if no supported split exists.                           */
int fftc_dist_split(int64_t N, int nranks, int64_t* out4);

#ifdef __cplusplus
}
#endif
#endif /* FFTC_H_ */
