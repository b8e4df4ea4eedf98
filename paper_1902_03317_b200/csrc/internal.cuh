// Internal helpers shared by the sm_100a kernels behind include/spten_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/spten_b200.h"

// ---------------------------------------------------------------------------
// Host side: context, errors, scratch.

struct spt_ctx {
  int device = 0;
  int num_sms = 148;
  size_t l2_bytes = 0;
  // Sticky device error words (min entry index of the first failure), reset
  // to all-ones. [0] tew_eq pattern mismatch, [1] tew_eq div-by-zero,
  // [2] mttkrp unsorted input, [3] spare.
  unsigned long long* d_err = nullptr;
  // Growable scratch (sort temp storage, counts, ...).
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // Decoupled look-back state: per-tile status words tagged with an epoch,
  // a self-resetting tile-id counter and R-wide fp64 payloads.
  uint32_t* d_status = nullptr;
  size_t status_cap = 0;  // tiles
  double* d_payload = nullptr;
  size_t payload_cap = 0;  // doubles
  unsigned long long* d_tile_ctr = nullptr;
  uint32_t epoch = 0;
  // 64-bit look-back words (epoch | flag | u32 count) for count scans.
  unsigned long long* d_status64 = nullptr;
  size_t status64_cap = 0;
  // Pinned host words for count read-back.
  unsigned long long* h_pinned = nullptr;
  // Private stream-ordered pool for the library's temporaries (its release
  // threshold is raised here only, never the device's default pool's).
  cudaMemPool_t pool = nullptr;
  // L2 flush buffer.
  void* l2buf = nullptr;
  size_t l2buf_bytes = 0;
  uint64_t launches = 0;
};

namespace spt {

int set_error(int status, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
// Grow-only scratch; may synchronise the device when it grows.
int ctx_scratch(spt_ctx* ctx, size_t bytes, void** out);
// Look-back state sized for `tiles` tiles and `payload_doubles` doubles;
// returns the epoch to pass to the kernel (never 0).
int ctx_lookback(spt_ctx* ctx, size_t tiles, size_t payload_doubles, uint32_t* epoch);
// 64-bit status words for `tiles` tiles (zeroed on growth); use with an epoch
// from ctx_lookback.
int ctx_status64(spt_ctx* ctx, size_t tiles, unsigned long long** out);
// Validate a descriptor (order range, nnz limit, non-null pointers when nnz>0).
int check_coo(const spt_coo* t, const char* who, bool need_values = true);
// Synchronise `stream` and decode the sticky error words.
int sync_and_check(spt_ctx* ctx, cudaStream_t stream);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Stream-ordered temporaries from the context's private pool.
template <typename T>
inline cudaError_t tmp_alloc(spt_ctx* ctx, T** p, size_t bytes, cudaStream_t st) {
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, ctx->pool, st);
}

__host__ __device__ inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline unsigned grid_for(uint64_t work_items, unsigned block, unsigned max_blocks) {
  uint64_t g = (work_items + block - 1) / block;
  if (g == 0) g = 1;
  if (g > max_blocks) g = max_blocks;
  return static_cast<unsigned>(g);
}

#define SPT_CUDA(call)                                               \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return ::spt::cuda_status(_e, #call);     \
  } while (0)

#define SPT_LAUNCHED(ctx)                                                           \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) return ::spt::cuda_status(_e, "kernel launch");          \
    (ctx)->launches++;                                                              \
  } while (0)

#define SPT_TRY(expr)              \
  do {                             \
    int _s = (expr);               \
    if (_s != SPT_OK) return _s;   \
  } while (0)

// Internal entry points implemented in the other translation units.
// Stable; d_perm receives the permutation. nkeys < order sorts by the first
// nkeys modes of mode_order only (ties keep the input order).
int sort_tuples(spt_ctx* ctx, const spt_coo* x, const uint32_t* mode_order, uint32_t* d_perm,
                cudaStream_t stream, uint32_t nkeys = SPT_MAX_ORDER);
int gather_coo(spt_ctx* ctx, spt_coo* x, const uint32_t* d_perm, cudaStream_t stream);
// MTTKRP plans (mttkrp_plan.cu) serve this input / rank.
bool plan_supported(const spt_coo* x, uint64_t R);
int mttkrp_sorted_copy(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors,
                       const uint64_t* rows, const uint64_t* cols, uint32_t mode, float* d_out,
                       unsigned flags, void* stream);

// One-wave segmented MTTKRP for small mode-sorted inputs (mttkrp_ow.cu).
bool mttkrp_onewave_ok(const spt_coo* x, uint64_t R, const float* const* d_factors, uint32_t mode,
                       const float* d_out);
int mttkrp_onewave(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors, uint32_t mode,
                   uint32_t R, float* d_out, cudaStream_t st);

}  // namespace spt

// ---------------------------------------------------------------------------
// Device side.

namespace spt {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Streaming (evict-first) 128-bit loads/stores for data touched once.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) { __stcs(p, v); }
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  return __ldcs(reinterpret_cast<const unsigned int*>(p));
}
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t v) {
  __stcs(reinterpret_cast<unsigned int*>(p), v);
}

// Acquire/release on a status word (gpu scope) for decoupled look-back.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Release-only fence (MEMBAR.ALL.GPU): orders this thread's payload writes
// before a later flag store, without the L1 invalidation (CCTL.IVALL) that
// __threadfence() adds -- which would evict the L1-resident factor rows.
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }
// Relaxed polling loads (no L1 invalidation per poll, unlike ld.acquire).
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mbarrier + bulk async copy (TMA engine, non-tensor form): global -> shared
// runs of 16-byte-aligned bytes, completion counted in the barrier's tx-count.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// try_wait's suspend-time hint: a waiting warp sleeps until the phase flips
// (or this many ns pass) instead of re-issuing the test in a tight loop.
#ifndef SPT_MBAR_SUSPEND_NS
#define SPT_MBAR_SUSPEND_NS 0x10000
#endif
constexpr uint32_t kMbarSuspendNs = SPT_MBAR_SUSPEND_NS;
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
#if SPT_MBAR_SUSPEND_NS == 0
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SPT_MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SPT_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SPT_MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra SPT_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(kMbarSuspendNs)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// Named barrier over the first `n` threads (warp multiples) of the CTA.
__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Warp-parallel decoupled look-back over epoch-tagged u32 status words
// (word = epoch << 3 | flags, flags & 3 == 1: aggregate A, == 2: inclusive P).
// Called by one full warp for tile `tile` > 0. Polls (never blocks on) the 32
// nearest predecessors at a time and returns n such that the chain of tiles
// [tile-n, tile-1] ends in a P at tile-n with only A's nearer: the caller sums
// payload[tile-n .. tile-1]. Tiles further back than the first P are never
// waited for, so predecessors that publish nothing (their row did not
// continue) cannot stall it.
__device__ __forceinline__ uint32_t lookback_chain(const uint32_t* status, uint32_t tile,
                                                   uint32_t epoch) {
  const unsigned lane = threadIdx.x & 31u;
  uint32_t base = 0;  // predecessors already known to be A
  while (true) {
    const int64_t j = (int64_t)tile - 1 - base - lane;
    uint32_t flag = 2;  // before tile 0: behave as a terminating P
    if (j >= 0) {
      const uint32_t s = ld_relaxed(status + j);
      flag = ((s >> 3) == epoch) ? (s & 3u) : 0u;
    }
    const unsigned ready = __ballot_sync(0xffffffffu, flag != 0);
    const unsigned isP = __ballot_sync(0xffffffffu, flag == 2);
    // length of the ready prefix (lanes 0..k-1 all published)
    const int prefix = (~ready) ? __ffs(~ready) - 1 : 32;
    const unsigned pmask = isP & (prefix == 32 ? 0xffffffffu : ((1u << prefix) - 1));
    if (pmask) {
      __threadfence();  // acquire: payloads written before the flags are visible
      return base + __ffs(pmask);  // includes the P tile
    }
    if (prefix == 32) base += 32;  // all A: slide the window
    else __nanosleep(32);
  }
}

// Same over 64-bit words (epoch << 34 | flag << 32 | u32 count): returns the
// exclusive prefix count for `tile` (sum of A counts up to and including the
// nearest P's inclusive count). One full warp; result valid in all lanes.
__device__ __forceinline__ unsigned long long lookback_count64(const unsigned long long* status,
                                                               uint32_t tile, uint32_t epoch) {
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long acc = 0;
  uint32_t base = 0;
  while (true) {
    const int64_t j = (int64_t)tile - 1 - base - lane;
    uint32_t flag = 2, cnt = 0;
    if (j >= 0) {
      // relaxed: the count lives in the flag word itself, no payload to order
      const unsigned long long w = ld_relaxed64(status + j);
      flag = ((w >> 34) == epoch) ? (uint32_t)((w >> 32) & 3u) : 0u;
      cnt = (uint32_t)w;
    }
    const unsigned ready = __ballot_sync(0xffffffffu, flag != 0);
    const unsigned isP = __ballot_sync(0xffffffffu, flag == 2);
    const int prefix = (~ready) ? __ffs(~ready) - 1 : 32;
    const unsigned pmask = isP & (prefix == 32 ? 0xffffffffu : ((1u << prefix) - 1));
    const int upto = pmask ? __ffs(pmask) : (prefix == 32 ? 32 : 0);
    unsigned long long v = (lane < (unsigned)upto) ? cnt : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc += v;
    if (pmask) return acc;
    if (prefix == 32) base += 32;
    else __nanosleep(32);
  }
}

// Wide-window lookback_count64: one warp polls 32*W predecessors per round
// trip (lane L owns tiles tile-1-W*L-k, k < W; all W loads in flight). For
// persistent kernels where a whole wave of ~#CTAs tiles publishes A at once
// and the nearest P sits a wave back, this turns ~wave/32 sequential round
// trips into one or two.
template <int W, int SH = 0>
__device__ __forceinline__ unsigned long long lookback_count64_wide(
    const unsigned long long* status, uint32_t tile, uint32_t epoch) {
  // Predecessor at distance 32*k + lane + 1 sits in lane `lane`, slot k, so
  // each of the W loads is one coalesced 256-byte request.
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long acc = 0;
  uint32_t base = 0;
  while (true) {
    uint32_t cnt[W];
    unsigned ready[W], isP[W];
    unsigned long long w[W];
    // all W loads in flight before the first use (the asm is volatile, so
    // they must be issued ahead of the ballots explicitly)
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t j = (int64_t)tile - 1 - base - (int64_t)(32 * k + lane);
      w[k] = j >= 0 ? ld_relaxed64(status + (j << SH)) : ((unsigned long long)epoch << 34) | (2ull << 32);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t flag = ((w[k] >> 34) == epoch) ? (uint32_t)((w[k] >> 32) & 3u) : 0u;
      cnt[k] = (uint32_t)w[k];
      ready[k] = __ballot_sync(0xffffffffu, flag != 0);
      isP[k] = __ballot_sync(0xffffffffu, flag == 2);
    }
    // walk the sub-windows nearest-first (warp-uniform)
    int ks = W, ls = 31;  // take sub-windows < ks fully, sub-window ks up to lane ls
    bool found = false, blocked = false;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (found || blocked) continue;
      const int prefix = (~ready[k]) ? __ffs(~ready[k]) - 1 : 32;
      const unsigned pm = isP[k] & (prefix == 32 ? 0xffffffffu : ((1u << prefix) - 1u));
      if (pm) {
        found = true;
        ks = k;
        ls = __ffs(pm) - 1;
      } else if (prefix < 32) {
        blocked = true;
      }
    }
    if (blocked) {
      __nanosleep(32);
      continue;
    }
    unsigned long long v = 0;
#pragma unroll
    for (int k = 0; k < W; ++k)
      v += (k < ks || (k == ks && static_cast<int>(lane) <= ls)) ? cnt[k] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc += v;
    if (found) return acc;
    base += 32 * W;
  }
}


// Philox4x32-10 counter-based RNG (Salmon et al., SC'11).
struct Philox {
  static __host__ __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi_compat(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi_compat(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  static __host__ __device__ __forceinline__ uint32_t __umulhi_compat(uint32_t a, uint32_t b) {
    return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
  }
  static __host__ __device__ __forceinline__ uint4 gen(uint64_t counter, uint64_t stream,
                                                       uint64_t seed) {
    uint4 c = make_uint4(static_cast<uint32_t>(counter), static_cast<uint32_t>(counter >> 32),
                         static_cast<uint32_t>(stream), static_cast<uint32_t>(stream >> 32));
    uint2 k = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    for (int i = 0; i < 10; ++i) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// 24-bit mantissa uniform in [0,1).
__host__ __device__ __forceinline__ float u01(uint32_t r) {
  return static_cast<float>(r >> 8) * (1.0f / 16777216.0f);
}
// 53-bit uniform in [0,1).
__host__ __device__ __forceinline__ double u01d(uint32_t a, uint32_t b) {
  return static_cast<double>((static_cast<uint64_t>(a) << 21) ^ (b >> 11)) *
         (1.0 / 9007199254740992.0);
}

}  // namespace spt
