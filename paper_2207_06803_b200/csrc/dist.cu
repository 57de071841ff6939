// dist.cu -- distributed six-step DFT over P GPUs (product path).
//
// One transform of length N = M K is block-distributed over P ranks (rank p holds
// x[pN/P, (p+1)N/P), and the same slab of X at the end), P | M, P | K,
// Mp = M/P, Kp = K/P.  In the M x K view A[q][r] = x[qK + r] rank p owns rows
// [p Mp, (p+1) Mp).  Eq. 2 at the top level, with its global
// stride permutation Pi^N_K realised as all-to-alls:
//   1. pack      send[d][ql][rl]   = x_p[ql K + d Kp + rl]            (Mp x Kp blocks)
//   2. a2a #1    recv[s][ql][rl]   = A[s Mp + ql][p Kp + rl]   ->  recv = B[q][rl], M x Kp
//   3. DFT_M     down each local column rl (stride Kp), times w_N^{(p Kp + rl) j}  (D^N_M),
//                written transposed into send[d][rl][jl] for j = d Mp + jl
//   4. a2a #2    recv[s][rl][jl]   = Y[p Mp + jl][s Kp + rl]   ->  recv = V[r][jl], K x Mp
//   5. DFT_K     down each local column jl (stride Mp) -> send[k1][jl] = Z[jl][k1]
//                (K > 4096: K = K1 K2, Eq. 2 again as two strided column passes,
//                 DFT_K1 with twiddle w_K^{b ja}, then DFT_K2)
//   6. a2a #3    recv[s][k1l][jl]  = Z_s[jl][p Kp + k1l]
//   7. unpack    X_p[k1l M + s Mp + jl] = recv[s][k1l][jl]   (natural order: X[j + M k1])
// All-to-alls are NCCL grouped send/recv on the plan stream (NVLink / NVSwitch);
// in loopback mode all P virtual ranks live on the current GPU and every
// all-to-all is P^2 device-to-device copies (used to parity-test the kernels and
// layouts on one GPU).  The inverse (sign = +1) conjugates in pack and unpack.
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "dist.h"
#include "fourstep.h"
#include "plan.h"
#include "planner.h"

namespace fftc {

struct DistState {
  int64_t N = 0, M = 0, K = 0, Mp = 0, Kp = 0, K1 = 0, K2 = 1;
  int P = 1, rank = 0, sign = -1, nloc = 1;
  bool loopback = false;
  const ColEntry* cM = nullptr;
  const ColEntry* cK1 = nullptr;  // DFT_K (K <= 4096) or DFT_K1
  const ColEntry* cK2 = nullptr;  // DFT_K2 (K > 4096)
  float2 *twM = nullptr, *twK1 = nullptr, *twK2 = nullptr;
  float2 *twA_N = nullptr, *twB_N = nullptr, *twA_K = nullptr, *twB_K = nullptr;
  float2 *send = nullptr, *recv = nullptr, *work = nullptr;  // nloc * N/P each
  ncclComm_t comm = nullptr;
  int launches = 0;
  int flags = 0;                 // FFTC_DIST_TRANSPOSED_OUT | FFTC_DIST_PEER_STORES
  // peer-store exchange: a second receive buffer (exchange #2) and every rank's receive
  // buffers mapped into this process (CUDA IPC over NVLink; in loopback, this GPU's slabs)
  float2* recv2 = nullptr;
  float2* peerA[8] = {};         // rank q's receive buffer of exchange #1
  float2* peerB[8] = {};         // rank q's receive buffer of exchange #2
  bool ipc_opened[8] = {};
  int* bar = nullptr;            // 1-int NCCL barrier buffer
};

namespace {

// dst[i0*s0 + i1*s1 + i2] = src[(i0*n1 + i1)*n2 + i2] (src contiguous [n0][n1][n2]), optional conj.
// Index decomposition in 32-bit unsigned arithmetic (a rank's slab holds < 2^32 elements).
__global__ void k_permute3(const float2* __restrict__ src, float2* __restrict__ dst, unsigned n0, unsigned n1,
                           unsigned n2, long long s0, long long s1, float csign) {
  const unsigned total = n0 * n1 * n2;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned r = t / n2, i2 = t - r * n2;
    const unsigned i0 = r / n1, i1 = r - i0 * n1;
    float2 a = __ldcs(src + t);
    __stcs(dst + i0 * s0 + i1 * s1 + i2, make_float2(a.x, csign * a.y));
  }
}
// same with 128-bit element pairs (n2, s0, s1 even; 16-byte aligned buffers)
__global__ void k_permute3_v2(const float4* __restrict__ src, float2* __restrict__ dst, unsigned n0, unsigned n1,
                              unsigned n2h, long long s0, long long s1, float csign) {
  const unsigned total = n0 * n1 * n2h;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned r = t / n2h, i2 = 2 * (t - r * n2h);
    const unsigned i0 = r / n1, i1 = r - i0 * n1;
    float4 a = __ldcs(src + t);
    __stcs(reinterpret_cast<float4*>(dst + i0 * s0 + i1 * s1 + i2), make_float4(a.x, csign * a.y, a.z, csign * a.w));
  }
}

// Fused pack + exchange #1: dst_{i1}[i0*s0 + i2] = src[(i0*n1 + i1)*n2 + i2], the destination
// base chosen per i1 (= the receiving rank) from a table of peer pointers.
struct PeerTable {
  float2* p[8];
};
__global__ void k_permute3_peer(const float2* __restrict__ src, PeerTable dst, unsigned n0, unsigned n1, unsigned n2,
                                long long s0, float csign) {
  const unsigned total = n0 * n1 * n2;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned r = t / n2, i2 = t - r * n2;
    const unsigned i0 = r / n1, i1 = r - i0 * n1;
    float2 a = __ldcs(src + t);
    __stcs(dst.p[i1] + i0 * s0 + i2, make_float2(a.x, csign * a.y));
  }
}

cudaError_t permute3_peer(const float2* src, const PeerTable& dst, long long n0, long long n1, long long n2,
                          long long s0, int conj, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (n0 * n1 * n2 >= (1LL << 32) || n1 > 8) return cudaErrorInvalidValue;
  const long long total = n0 * n1 * n2;
  long long blocks = (total + 255) / 256;
  if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
  k_permute3_peer<<<(unsigned)blocks, 256, 0, st>>>(src, dst, (unsigned)n0, (unsigned)n1, (unsigned)n2, s0,
                                                    conj ? -1.f : 1.f);
  return cudaGetLastError();
}

cudaError_t permute3(const float2* src, float2* dst, long long n0, long long n1, long long n2, long long s0,
                     long long s1, int conj, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const float cs = conj ? -1.f : 1.f;
  if (n0 * n1 * n2 >= (1LL << 32)) return cudaErrorInvalidValue;  // slab beyond 32-bit indexing
  if (n2 % 2 == 0 && s0 % 2 == 0 && s1 % 2 == 0) {
    const long long total = n0 * n1 * (n2 / 2);
    long long blocks = (total + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    k_permute3_v2<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(src), dst, (unsigned)n0,
                                                    (unsigned)n1, (unsigned)(n2 / 2), s0, s1, cs);
  } else {
    const long long total = n0 * n1 * n2;
    long long blocks = (total + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    k_permute3<<<(unsigned)blocks, 256, 0, st>>>(src, dst, (unsigned)n0, (unsigned)n1, (unsigned)n2, s0, s1, cs);
  }
  return cudaGetLastError();
}

int ilog2ll(long long v) {
  int l = 0;
  while ((1LL << (l + 1)) <= v) ++l;
  return l;
}
bool pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

// Split N = M K for P ranks (single-pass DFT_M with a transposed-output column
// kernel; DFT_K single pass or K = K1 K2).  Returns false if no split fits.
bool dist_split(int64_t N, int P, DistState* d) {
  for (int mi = col_count() - 1; mi >= 0; --mi) {  // largest M first
    const ColEntry* cm = col_at(mi);
    const int64_t M = cm->M;
    if (N % M || M % P || !cm->launch_t) continue;
    const int64_t K = N / M;
    if (K % P) continue;
    const int64_t Mp = M / P, Kp = K / P;
    if (!pow2(Mp) || Kp % cm->cols) continue;
    if (K <= 4096) {
      const ColEntry* ck = find_col((int)K);
      if (!ck || Mp % ck->cols) continue;
      d->M = M, d->K = K, d->Mp = Mp, d->Kp = Kp, d->K1 = K, d->K2 = 1, d->cM = cm, d->cK1 = ck, d->cK2 = nullptr;
      return true;
    }
    // K = K1 K2, most balanced pair of compiled column sizes
    const ColEntry *b1 = nullptr, *b2 = nullptr;
    for (int i = 0; i < col_count(); ++i)
      for (int j = 0; j < col_count(); ++j) {
        const ColEntry *c1 = col_at(i), *c2 = col_at(j);
        if ((int64_t)c1->M * c2->M != K) continue;
        if ((c2->M * Mp) % c1->cols || Mp % c2->cols) continue;
        if (!b1 || llabs((long long)c1->M - c2->M) < llabs((long long)b1->M - b2->M)) b1 = c1, b2 = c2;
      }
    if (!b1) continue;
    d->M = M, d->K = K, d->Mp = Mp, d->Kp = Kp, d->K1 = b1->M, d->K2 = b2->M, d->cM = cm, d->cK1 = b1, d->cK2 = b2;
    return true;
  }
  return false;
}

cudaError_t all_to_all(DistState* d, cudaStream_t st, fftc_status* ns) {
  const int64_t chunk = d->Mp * d->Kp;  // complex elements per peer
  const int64_t slab = d->N / d->P;
  if (d->loopback || d->P == 1) {
    for (int p = 0; p < d->nloc; ++p)
      for (int s = 0; s < d->P; ++s) {
        cudaError_t e = cudaMemcpyAsync(d->recv + p * slab + s * chunk, d->send + s * slab + p * chunk,
                                        chunk * sizeof(float2), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
      }
    return cudaSuccess;
  }
  const size_t count = (size_t)chunk * 2;  // floats
  ncclResult_t r = ncclGroupStart();
  for (int s = 0; s < d->P && r == ncclSuccess; ++s) {
    if (s == d->rank) continue;
    r = ncclSend(d->send + s * chunk, count, ncclFloat, s, d->comm, st);
    if (r == ncclSuccess) r = ncclRecv(d->recv + s * chunk, count, ncclFloat, s, d->comm, st);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    *ns = FFTC_ERROR_NCCL;
    return cudaErrorUnknown;
  }
  return cudaMemcpyAsync(d->recv + d->rank * chunk, d->send + d->rank * chunk, chunk * sizeof(float2),
                         cudaMemcpyDeviceToDevice, st);
}

// Cross-rank barrier on the stream (a 1-int NCCL all-reduce): every rank's earlier kernels,
// including their stores into this rank's buffers, are complete when it returns.
cudaError_t barrier(DistState* d, cudaStream_t st, fftc_status* ns) {
  if (d->loopback || d->P == 1) return cudaSuccess;
  if (ncclAllReduce(d->bar, d->bar, 1, ncclInt, ncclSum, d->comm, st) != ncclSuccess) {
    *ns = FFTC_ERROR_NCCL;
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace

fftc_status dist_execute(DistState* d, const void* in, void* out, cudaStream_t st) {
  if (!d) return FFTC_ERROR_INVALID_VALUE;
  if (((uintptr_t)in & 15u) || ((uintptr_t)out & 15u)) return FFTC_ERROR_MISALIGNED;
  const int64_t slab = d->N / d->P;
  if (in == out) return FFTC_ERROR_INVALID_VALUE;
  const float2* x = (const float2*)in;
  float2* X = (float2*)out;
  const int conj = d->sign > 0;
  fftc_status ns = FFTC_SUCCESS;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return FFTC_ERROR_CUDA;
  const int64_t M = d->M, K = d->K, Mp = d->Mp, Kp = d->Kp, P = d->P;
  const bool peer = (d->flags & FFTC_DIST_PEER_STORES) != 0;
  const bool tout = (d->flags & FFTC_DIST_TRANSPOSED_OUT) != 0;
  const int64_t chunk = Mp * Kp;
  float2* recvA = d->recv;                 // exchange #1 lands here
  float2* recvB = peer ? d->recv2 : d->recv;  // exchange #2 lands here
  const bool fuse3 = peer && !tout && d->K2 == 1;  // exchange #3 fused into the DFT_K epilogue
  if (peer) {
    // 1+2. pack fused with exchange #1: x_p[ql][d][rl] -> rank d's recvA[p][ql][rl] (NVLink stores)
    e = barrier(d, st, &ns);  // every rank is done reading its receive buffers (previous call)
    for (int p = 0; p < d->nloc && e == cudaSuccess; ++p) {
      const int prank = d->loopback ? p : d->rank;
      PeerTable t{};
      for (int q = 0; q < P; ++q) t.p[q] = d->peerA[q] + prank * chunk;
      e = permute3_peer(x + p * slab, t, Mp, P, Kp, Kp, conj, st);
    }
    if (e == cudaSuccess) e = barrier(d, st, &ns);
  } else {
    // 1. pack: src x_p viewed as [ql][d][rl] (Mp, P, Kp) -> send[d][ql][rl]
    for (int p = 0; p < d->nloc && e == cudaSuccess; ++p)
      e = permute3(x + p * slab, d->send + p * slab, Mp, P, Kp, Kp, Mp * Kp, conj, st);
    // 2. a2a #1
    if (e == cudaSuccess) e = all_to_all(d, st, &ns);
  }
  // 3. DFT_M down columns rl of B[q][rl] (stride Kp), twiddle w_N^{(p Kp + rl) j}, transposed out
  //    (peer mode: chunk j / Mp goes straight to that rank's recvB[p] -- exchange #2 fused)
  for (int p = 0; p < d->nloc && e == cudaSuccess; ++p) {
    const int prank = d->loopback ? p : d->rank;
    ColGeom g{};
    g.tiles = (int)(Kp / d->cM->cols);
    g.in_g = 0;
    g.in_s = Kp;
    g.out_g = 0;
    g.out_c = Mp;
    g.out_s = 1;
    g.out_cs = Kp * Mp;
    g.ocl = ilog2ll(Mp);
    g.tw = 1;
    g.tw_shift = 0;
    g.tw_off = (long long)prank * Kp;
    if (peer) {
      g.npeer = (int)P;
      for (int q = 0; q < P; ++q) g.peer[q] = (unsigned long long)(d->peerB[q] + prank * chunk);
    }
    e = d->cM->launch_t(recvA + p * slab, d->send + p * slab, d->twM, d->twA_N, d->twB_N, g, 1, 0, 0, st);
  }
  // 4. a2a #2
  if (e == cudaSuccess) e = peer ? barrier(d, st, &ns) : all_to_all(d, st, &ns);
  // 5. DFT_K down columns jl of V[r][jl] (stride Mp) -> send[k1][jl]
  //    (transposed-output mode: straight into out, with the inverse's output conjugation)
  for (int p = 0; p < d->nloc && e == cudaSuccess; ++p) {
    float2* kout = tout ? X + p * slab : d->send + p * slab;
    const int cj = tout ? conj : 0;
    if (d->K2 == 1) {
      ColGeom g{};
      g.tiles = (int)(Mp / d->cK1->cols);
      g.in_s = Mp;
      g.out_c = 1;
      g.out_s = Mp;
      g.ocl = 62;
      if (fuse3) {
        // exchange #3 fused: output k1 goes to rank k1 / Kp's recvA[p][k1 mod Kp][jl] (recvA is
        // free: every rank passed the barrier after its DFT_M, the last reader of recvA)
        const int prank = d->loopback ? p : d->rank;
        g.ocl = ilog2ll(Kp);
        g.npeer = (int)P;
        for (int q = 0; q < P; ++q) g.peer[q] = (unsigned long long)(d->peerA[q] + prank * chunk);
      }
      e = d->cK1->launch(recvB + p * slab, kout, d->twK1, nullptr, nullptr, g, 1, 0, cj, st);
    } else {
      const int64_t K1 = d->K1, K2 = d->K2;
      // pass A: columns (b, jl) -> c = b Mp + jl, DFT_K1 over a (stride K2 Mp), twiddle w_K^{b ja}
      ColGeom a{};
      a.tiles = (int)(K2 * Mp / d->cK1->cols);
      a.in_s = K2 * Mp;
      a.out_c = 1;
      a.out_s = K2 * Mp;
      a.ocl = 62;
      a.tw = 1;
      a.tw_shift = ilog2ll(Mp);
      e = d->cK1->launch(recvB + p * slab, d->work + p * slab, d->twK1, d->twA_K, d->twB_K, a, 1, 0, 0, st);
      // pass B: groups ja, columns jl, DFT_K2 over b (stride Mp), out X[(ja + K1 kb) Mp + jl]
      ColGeom b{};
      b.tiles = (int)(Mp / d->cK2->cols);
      b.in_g = K2 * Mp;
      b.in_s = Mp;
      b.out_g = Mp;
      b.out_c = 1;
      b.out_s = K1 * Mp;
      b.ocl = 62;
      if (e == cudaSuccess) e = d->cK2->launch(d->work + p * slab, kout, d->twK2, nullptr, nullptr, b, K1, 0, cj, st);
    }
  }
  if (!tout) {
    // 6. a2a #3 (fused: the barrier after the peer stores)
    if (e == cudaSuccess) e = fuse3 ? barrier(d, st, &ns) : all_to_all(d, st, &ns);
    // 7. unpack: recv viewed as [s][k1l][jl] (P, Kp, Mp) -> X_p[k1l M + s Mp + jl]
    for (int p = 0; p < d->nloc && e == cudaSuccess; ++p)
      e = permute3(d->recv + p * slab, X + p * slab, P, Kp, Mp, Mp, M, conj, st);
  }
  (void)K;
  if (ns != FFTC_SUCCESS) return ns;
  return e == cudaSuccess ? FFTC_SUCCESS : FFTC_ERROR_CUDA;
}

void dist_destroy(DistState* d) {
  if (!d) return;
  cudaFree(d->twM);
  cudaFree(d->twK1);
  cudaFree(d->twK2);
  cudaFree(d->twA_N);
  cudaFree(d->twB_N);
  cudaFree(d->twA_K);
  cudaFree(d->twB_K);
  for (int q = 0; q < 8; ++q) {
    if (d->ipc_opened[q]) {
      cudaIpcCloseMemHandle(d->peerA[q]);
      cudaIpcCloseMemHandle(d->peerB[q]);
    }
  }
  cudaFree(d->send);
  cudaFree(d->recv);
  cudaFree(d->recv2);
  cudaFree(d->bar);
  cudaFree(d->work);
  if (d->comm) ncclCommDestroy(d->comm);
  delete d;
}

int dist_launches(const DistState* d) { return d ? d->launches : -1; }

int dist_describe(const DistState* d, char* buf, size_t len) {
  if (!d) return -1;
  return snprintf(buf, len,
                  "kind=dist N=%lld P=%d rank=%d sign=%d M=%lld K=%lld K1=%lld K2=%lld Mp=%lld Kp=%lld loopback=%d "
                  "launches=%d a2a=%d exchange=%s output=%s chunk_bytes=%lld",
                  (long long)d->N, d->P, d->rank, d->sign, (long long)d->M, (long long)d->K, (long long)d->K1,
                  (long long)d->K2, (long long)d->Mp, (long long)d->Kp, (int)d->loopback, d->launches,
                  (d->flags & FFTC_DIST_TRANSPOSED_OUT) ? 2 : 3,
                  (d->flags & FFTC_DIST_PEER_STORES)
                      ? (((d->flags & FFTC_DIST_TRANSPOSED_OUT) || d->K2 != 1) ? "peer-stores(#1,#2 fused)"
                                                                                : "peer-stores(#1,#2,#3 fused)")
                      : "nccl",
                  (d->flags & FFTC_DIST_TRANSPOSED_OUT) ? "transposed" : "natural",
                  (long long)(d->Mp * d->Kp * (int64_t)sizeof(float2)));
}

}  // namespace fftc

using namespace fftc;

extern "C" fftc_status fftc_check_device(int* dev);
extern "C" void fftc_set_last_error(fftc_status s);

extern "C" int fftc_dist_split(int64_t N, int nranks, int64_t* out4) {
  if (!out4 || N < 2 || nranks < 1) return -1;
  DistState d;
  if (!dist_split(N, nranks, &d)) return -1;
  out4[0] = d.M;
  out4[1] = d.K;
  out4[2] = d.K1;
  out4[3] = d.K2;
  return 0;
}

extern "C" fftc_status fftc_dist_get_unique_id(void* id_out) {
  if (!id_out) return FFTC_ERROR_INVALID_VALUE;
  static_assert(sizeof(ncclUniqueId) == FFTC_NCCL_ID_BYTES, "NCCL id size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FFTC_ERROR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return FFTC_SUCCESS;
}

extern "C" fftc_plan* fftc_dist_plan_create_ex(int64_t N, int sign, const void* nccl_id, int rank, int nranks,
                                               int loopback, int flags);

extern "C" fftc_plan* fftc_dist_plan_create(int64_t N, int sign, const void* nccl_id, int rank, int nranks,
                                            int loopback) {
  return fftc_dist_plan_create_ex(N, sign, nccl_id, rank, nranks, loopback, 0);
}

extern "C" fftc_plan* fftc_dist_plan_create_ex(int64_t N, int sign, const void* nccl_id, int rank, int nranks,
                                               int loopback, int flags) {
  auto fail = [&](fftc_status s, DistState* d) -> fftc_plan* {
    dist_destroy(d);
    fftc_set_last_error(s);
    return nullptr;
  };
  if (N < 2 || (sign != -1 && sign != 1) || nranks < 1 || (!loopback && (rank < 0 || rank >= nranks)))
    return fail(FFTC_ERROR_INVALID_VALUE, nullptr);
  if (!loopback && nranks > 1 && !nccl_id) return fail(FFTC_ERROR_INVALID_VALUE, nullptr);
  if (flags & ~(FFTC_DIST_TRANSPOSED_OUT | FFTC_DIST_PEER_STORES)) return fail(FFTC_ERROR_INVALID_VALUE, nullptr);
  if ((flags & FFTC_DIST_PEER_STORES) && nranks > 8) return fail(FFTC_ERROR_UNSUPPORTED_SIZE, nullptr);
  // One rank without loopback: every all-to-all is the identity, so the transform is
  // the single-GPU plan (multi-pass / four-step / fused) -- no copies, no extra passes.
  if (nranks == 1 && !loopback && !flags && !getenv("FFTC_DIST_SIXSTEP")) return fftc_plan_create(N, 1, sign);
  int dev = 0;
  fftc_status ds = fftc_check_device(&dev);
  if (ds != FFTC_SUCCESS) return fail(ds, nullptr);
  DistState* d = new DistState();
  d->N = N;
  d->P = nranks;
  d->rank = loopback ? 0 : rank;
  d->sign = sign;
  d->loopback = loopback != 0;
  d->nloc = d->loopback ? nranks : 1;
  d->flags = flags;
  if (!dist_split(N, nranks, d)) return fail(FFTC_ERROR_UNSUPPORTED_SIZE, d);
  cudaError_t err = cudaSuccess;
  d->twM = upload_stage_table(d->M, d->cM->R, d->cM->S, &err);
  if (err == cudaSuccess) d->twK1 = upload_stage_table(d->K1, d->cK1->R, d->cK1->S, &err);
  if (err == cudaSuccess && d->cK2) d->twK2 = upload_stage_table(d->K2, d->cK2->R, d->cK2->S, &err);
  if (err == cudaSuccess) d->twA_N = upload_root_table(N, N < 4096 ? N : 4096, 1, &err);
  if (err == cudaSuccess) d->twB_N = upload_root_table(N, (N + 4095) / 4096, 4096, &err);
  if (err == cudaSuccess && d->cK2) d->twA_K = upload_root_table(d->K, d->K < 4096 ? d->K : 4096, 1, &err);
  if (err == cudaSuccess && d->cK2) d->twB_K = upload_root_table(d->K, (d->K + 4095) / 4096, 4096, &err);
  const size_t bytes = (size_t)(N / nranks) * d->nloc * sizeof(float2);
  if (err == cudaSuccess) err = cudaMalloc(&d->send, bytes);
  if (err == cudaSuccess) err = cudaMalloc(&d->recv, bytes);
  if (err == cudaSuccess && d->cK2) err = cudaMalloc(&d->work, bytes);
  if (err != cudaSuccess)
    return fail(err == cudaErrorMemoryAllocation ? FFTC_ERROR_OUT_OF_MEMORY : FFTC_ERROR_CUDA, d);
  const bool peer = (flags & FFTC_DIST_PEER_STORES) != 0;
  if (err == cudaSuccess && peer) err = cudaMalloc(&d->recv2, bytes);
  if (err == cudaSuccess && peer) err = cudaMalloc(&d->bar, 256);
  if (err == cudaSuccess && peer) err = cudaMemset(d->bar, 0, 256);
  if (err != cudaSuccess)
    return fail(err == cudaErrorMemoryAllocation ? FFTC_ERROR_OUT_OF_MEMORY : FFTC_ERROR_CUDA, d);
  if (!d->loopback && nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    if (ncclCommInitRank(&d->comm, nranks, id, rank) != ncclSuccess) return fail(FFTC_ERROR_NCCL, d);
  }
  const int64_t slab = N / nranks;
  if (peer && (d->loopback || nranks == 1)) {
    for (int q = 0; q < nranks; ++q) {  // the virtual ranks' slabs on this GPU
      d->peerA[q] = d->recv + q * slab;
      d->peerB[q] = d->recv2 + q * slab;
    }
  } else if (peer) {
    // map every rank's receive buffers: CUDA IPC handles all-gathered over NCCL
    cudaIpcMemHandle_t h[2];
    if (cudaIpcGetMemHandle(&h[0], d->recv) != cudaSuccess || cudaIpcGetMemHandle(&h[1], d->recv2) != cudaSuccess)
      return fail(FFTC_ERROR_CUDA, d);
    const size_t hb = sizeof(h);
    char* dh = nullptr;
    std::vector<char> all((size_t)nranks * hb);
    cudaStream_t cs = nullptr;
    bool ok = cudaMalloc(&dh, (size_t)(nranks + 1) * hb) == cudaSuccess &&
              cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMemcpy(dh + (size_t)nranks * hb, h, hb, cudaMemcpyHostToDevice) == cudaSuccess &&
              ncclAllGather(dh + (size_t)nranks * hb, dh, hb, ncclChar, d->comm, cs) == ncclSuccess &&
              cudaStreamSynchronize(cs) == cudaSuccess &&
              cudaMemcpy(all.data(), dh, all.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (cs) cudaStreamDestroy(cs);
    cudaFree(dh);
    for (int q = 0; ok && q < nranks; ++q) {
      if (q == rank) {
        d->peerA[q] = d->recv;
        d->peerB[q] = d->recv2;
        continue;
      }
      cudaIpcMemHandle_t hq[2];
      memcpy(hq, all.data() + (size_t)q * hb, hb);
      void *pa = nullptr, *pb = nullptr;
      ok = cudaIpcOpenMemHandle(&pa, hq[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess &&
           cudaIpcOpenMemHandle(&pb, hq[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      d->peerA[q] = (float2*)pa;
      d->peerB[q] = (float2*)pb;
      d->ipc_opened[q] = ok;
    }
    if (!ok) return fail(FFTC_ERROR_CUDA, d);
  }
  d->launches = d->nloc * (d->cK2 ? 5 : 4) - ((flags & FFTC_DIST_TRANSPOSED_OUT) ? d->nloc : 0);
  fftc_plan* p = new fftc_plan();
  p->N = N;
  p->batch = 1;
  p->sign = sign;
  p->device = dev;
  p->kind = KIND_DIST;
  p->dist = d;
  return p;
}
