// common.cuh -- device-side building blocks shared by the libils kernels (sm_100a only).
//
// Index stream: implemented from the normative text in include/ils.h ("Index stream").
// The CPU oracle (oracle/index_stream.py) implements the same text independently.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libils targets sm_100a only"
#endif

namespace ils {

constexpr int kTagRkRgs = 1;
constexpr int kTagScdA = 2;
constexpr int kTagScdB = 3;
constexpr int kTagScdC = 4;
constexpr int kTagRcd = 6;
constexpr int kFeistelRounds = 8;

// ---------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// draw(seed, k, t, tag): counter (t_lo, t_hi, k, tag), key (seed_lo, seed_hi)
__host__ __device__ __forceinline__ U4 draw(uint64_t seed, uint32_t k, uint64_t t, uint32_t tag) {
  return philox10(U4{(uint32_t)t, (uint32_t)(t >> 32), k, tag}, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
}

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// j = min{ j : S[j] > v }, v = floor(U * S[n-1] / 2^64). S in shared or global memory.
__device__ __forceinline__ int sample_weighted(uint64_t U, const uint64_t* S, int n) {
  const uint64_t v = mulhi64(U, S[n - 1]);
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S[mid] > v) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// The same index for n <= 32 without a data-dependent loop: j = #{k < n-1 : S_k <= v} (S is
// strictly increasing and S_{n-1} > v), by five fixed halving steps with selects.
__device__ __forceinline__ int sample_weighted_small(uint64_t U, const uint64_t* S, int n) {
  const uint64_t v = mulhi64(U, S[n - 1]);
  int j = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int k = j + step - 1;
    const uint64_t sk = S[k < n - 1 ? k : 0];
    j = (k < n - 1 && sk <= v) ? j + step : j;
  }
  return j;
}

// ---------------------------------------------------------------- Feistel permutation of [n]
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

struct Feistel {
  uint32_t h, mask, n;
  uint32_t key[kFeistelRounds];
};

__host__ __device__ __forceinline__ uint32_t feistel_half_bits(uint32_t n) {
  uint32_t b = 0;
  while ((1u << b) < n) ++b;
  return (b + 1) >> 1;
}

// inverse of one 8-round encryption: undo rounds 7..0; round r was (L,R)->(R, L^F(R,K_r))
__device__ __forceinline__ uint32_t feistel_decrypt_once(uint32_t y, const uint32_t* key, uint32_t h,
                                                         uint32_t mask) {
  uint32_t L = y >> h, R = y & mask;
#pragma unroll
  for (int r = kFeistelRounds - 1; r >= 0; --r) {
    const uint32_t Lp = R ^ (mix32(L ^ key[r]) & mask);  // previous L
    R = L;                                                // previous R
    L = Lp;
  }
  return (L << h) | R;
}

// pi^{-1}(s) for s in [0, n): cycle-walk the inverse until the value lies in [0, n).
__device__ __forceinline__ uint32_t feistel_inverse(uint32_t s, const uint32_t* key, uint32_t h,
                                                    uint32_t mask, uint32_t n) {
  if (n == 1) return 0;
  uint32_t y = feistel_decrypt_once(s, key, h, mask);
  while (y >= n) y = feistel_decrypt_once(y, key, h, mask);
  return y;
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// (val, idx, payload) argmax with ties to the smallest idx; invalid entries have idx = INT_MAX.
struct ArgMax { double val; int idx; double pay; };

__device__ __forceinline__ bool argmax_better(double v1, int i1, double v2, int i2) {
  return (v1 > v2) || (v1 == v2 && i1 < i2);
}

// Warp argmax of a non-negative double key with ties to the smallest index, by integer warp
// reductions (redux.sync): the bit pattern of a double >= 0 orders like the value, so the max is
// taken on the high word, then on the low word among the lanes that hold the high max, then the
// min index among the lanes that hold both. Lanes without a candidate pass key 0 and idx INT_MAX
// (a valid key 0 then wins by its index). Returns the winning index in every lane (INT_MAX: none).
__device__ __forceinline__ int warp_argmax_redux(double key, int idx) {
  const unsigned long long kb = (unsigned long long)__double_as_longlong(key);
  const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const unsigned cand = (hi == mhi && lo == mlo) ? (unsigned)idx : 0xffffffffu;
  return (int)min(__reduce_min_sync(0xffffffffu, cand), (unsigned)INT_MAX);
}

__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_xor_sync(0xffffffffu, a.val, o);
    const int i = __shfl_xor_sync(0xffffffffu, a.idx, o);
    const double p = __shfl_xor_sync(0xffffffffu, a.pay, o);
    if (argmax_better(v, i, a.val, a.idx)) { a.val = v; a.idx = i; a.pay = p; }
  }
  return a;
}

// ---------------------------------------------------------------- mbarrier / bulk copy PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {   // release.cta
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 1D bulk copy global -> shared (TMA engine), completion signalled on bar (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- cluster / DSMEM PTX
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t map_shared_rank(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

// Asynchronous DSMEM stores whose arrival is counted on the destination CTA's mbarrier
// (complete_tx): a one-hop all-to-all without a cluster-wide barrier.
__device__ __forceinline__ void st_async_v2f64(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}

// wait on a local mbarrier phase whose completion may come from other CTAs of the cluster
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}

// named barrier over the first nthreads threads of the CTA
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// ---------------------------------------------------------------- blocked RK-RGS helpers (rk_rgs.cu, sparse.cu)
template <int B>
struct RkBlk {
  static constexpr int NV = (3 * B * B + 3 * B) / 2;
  __host__ __device__ static constexpr int P(int i) { return i; }
  __host__ __device__ static constexpr int Q(int i) { return B + i; }
  __host__ __device__ static constexpr int AA(int i, int k) { return 2 * B + i * (i - 1) / 2 + k; }
  __host__ __device__ static constexpr int BA(int i, int k) { return 2 * B + B * (B - 1) / 2 + i * (i + 1) / 2 + k; }
  __host__ __device__ static constexpr int BB(int i, int k) {
    return 2 * B + B * (B - 1) / 2 + B * (B + 1) / 2 + i * (i - 1) / 2 + k;
  }
};

// butterfly reduce-scatter of NVP (power of two <= 32) values over the warp: on return lane l
// holds the warp sum of value l & (NVP - 1) (NVP - 1 + log2(32 / NVP) shuffles of doubles)
// the butterfly levels of warp_reduce_scatter only: lane l holds value l & (NVP - 1) summed over its
// NVP-lane group (the cross-group sum is left to the consumer)
template <int NVP>
__device__ __forceinline__ double warp_reduce_scatter_groups(double (&x)[NVP], int lane) {
#pragma unroll
  for (int half = NVP / 2; half >= 1; half /= 2) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double lo_v = x[i], hi_v = x[i + half];
      const double send = hi ? lo_v : hi_v;
      const double keep = hi ? hi_v : lo_v;
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return x[0];
}

template <int NVP>
__device__ __forceinline__ double warp_reduce_scatter(double (&x)[NVP], int lane) {
#pragma unroll
  for (int half = NVP / 2; half >= 1; half /= 2) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double lo_v = x[i], hi_v = x[i + half];
      const double send = hi ? lo_v : hi_v;
      const double keep = hi ? hi_v : lo_v;
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  double v = x[0];
#pragma unroll
  for (int o = NVP; o < 32; o *= 2) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t ld_acquire_cta_s64(const int64_t* a) {
  int64_t v;
  asm volatile("ld.acquire.cta.shared::cta.s64 %0, [%1];" : "=l"(v) : "r"(smem_u32(a)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_s64(int64_t* a, int64_t v) {
  asm volatile("st.release.cta.shared::cta.s64 [%0], %1;" ::"r"(smem_u32(a)), "l"(v) : "memory");
}
// Progress counter written after a CTA barrier that every reader of the guarded buffer took part in:
// the readers' loads have returned (their values were consumed) before the barrier completes, so the
// counter only has to become visible after it, which program order behind bar.sync gives. The release
// form above compiles to MEMBAR.ALL.CTA + STS and cost ~250 cycles per block on the compute chain of
// the look-ahead RK-RGS kernels (ILS_RK_PROF: loop-top 253 cycles).
__device__ __forceinline__ void st_relaxed_cta_s64(int64_t* a, int64_t v) {
  asm volatile("st.relaxed.cta.shared::cta.s64 [%0], %1;" ::"r"(smem_u32(a)), "l"(v) : "memory");
}

// ---------------------------------------------------------------- cp.async (LDGSTS)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- DMMA (fp64 tensor core)
// D(8x8) += A(8x4, row) * B(4x8, col). Lane l holds A[l>>2][l&3], B[l&3][l>>2],
// D[l>>2][2*(l&3) + {0,1}].  SASS: DMMA.8x8x4.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace ils
