// K8b MTTKRP on a plan: prefix-reuse traversal of a mode-leading sorted copy
// with a shared-memory cache of the most-gathered factor rows.
//
// Reference: seq::mttkrp P/src/kernels_seq.cpp:153-174 (out(i_n,r) +=
// val * prod_{d != n} F_d(i_d, r), the term formed in mttkrp_row,
// P/src/kernel_detail.hpp:176-188), par::mttkrp P/src/kernels_par.cpp:275-337.
//
// Why a plan. A COO traversal gathers N-1 factor rows per nonzero; at the
// BASELINE configs those gathers, not the COO stream, are the traffic: C5
// (1B nnz, R=32) moves 2 x 1B x 128 B = 256 GB of rows from L2 per mode,
// ~20 ms at the ~12 TB/s L2 slice cap, against 16 GB of COO. The plan is the
// preprocessing (timed apart, like the reference's sort_s, P/src/bench.cpp:
// 363-368) that cuts the gathers:
//   * entries are sorted (mode, l_0, .., l_{K-1}) with the non-output modes
//     ordered by decreasing extent, so the factor with the most rows (the one
//     that misses L2) sits nearest the root of the implied CSF tree;
//   * the kernel detects on the fly where a prefix (i_n, l_0..l_j) changes and
//     gathers F_{l_j} only then, keeping the current prefix's rows in
//     registers. C5: 1.42 row gathers per nonzero instead of 2 (measured: 42%
//     of entries start a new (i_n, i_a) prefix); C4: 1.9 instead of 3
//     (tune/probe_reuse.py);
//   * ids whose rows are gathered most (per-level gather counts from the
//     sorted copy, top-H by count over all levels, H = what shared memory
//     holds at this R) are re-encoded as slots (bit 31 | slot) of a per-CTA
//     shared-memory copy of those rows, loaded once per launch by bulk
//     copies. C5: the 1024 hottest ids serve 52% of the leaf gathers;
//   * the copy is stored blocked (AoSoA): per block of CH entries the row
//     index, each level's ids and the values lie contiguous, so one bulk copy
//     (TMA engine, L2 evict-first) stages a lane group's next CH entries.
// Each term val * F_mid.. * F_leaf is formed in fp32 (like mttkrp_row's
// product, but not in its d-ascending order), at most U terms are summed in
// fp32 before an fp64 fold, and each output element is rounded once: every
// entry stays within the 1e-5 tolerance against an fp64 recomputation
// (DESIGN.md).
//
// Kernel shape: one persistent CTA per SM, 16 warps, lane groups of G = CB/4
// lanes (a float4 per lane: R=32 -> 8 lanes cover a 128-byte row). The nnz
// are split into equal, block-aligned contiguous ranges, one per lane group
// (no tickets, no look-back chains). Per iteration a group decodes U staged
// entries, issues all their gathers (a predicated LDS from the hot copy or
// LDG from the factor, no branch), then folds them in order. Rows complete
// inside a group are stored directly; each group's first and last row become
// partials folded per CTA in shared memory, then across CTAs by the last CTA
// to finish (an arrival counter), in fixed order: deterministic. Empty rows
// are zero-filled by the group whose range spans them, so the output needs no
// memset and every element is written exactly once.
#include <cub/cub.cuh>

#include <type_traits>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

struct spt_mttkrp_plan {
  int device = 0;
  uint32_t N = 0, mode = 0, nm1 = 0, R = 0, CB = 0, CH = 0, NA = 0;
  uint64_t nnz = 0, nblk = 0;
  uint32_t dims[SPT_MAX_ORDER] = {};
  uint32_t lvl_mode[SPT_MAX_ORDER - 1] = {};  // tensor mode of level k (outermost first)
  uint32_t* blk = nullptr;  // [nblk][NA][CH]: row index, level ids (hot ones encoded), value bits
  uint32_t nhot = 0;
  uint2* hot = nullptr;  // [nhot] (level, id)
  uint32_t hot_per_level[SPT_MAX_ORDER - 1] = {};
  double* part = nullptr;  // [2 * grid][CB] CTA first/last-row partials
  uint32_t* part_row = nullptr;
  double* gpart = nullptr;  // [2 * groups][CB] lane-group first/last-row partials
  uint32_t* gprow = nullptr;
  unsigned int* done = nullptr;
  uint32_t grid = 0;
  // The arrays come from the context's stream-ordered pool and are released
  // on the stream that used the plan last: creating and destroying a plan
  // never synchronises the device (a host caller's copies on other streams
  // keep running under the plan builds).
  mutable cudaStream_t last = nullptr;
};

namespace {

constexpr uint32_t kHot = 0x80000000u;  // id field holds a shared-memory slot
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
#ifndef SPT_PLAN_WARPS
#define SPT_PLAN_WARPS 16
#endif
constexpr int kW = SPT_PLAN_WARPS;  // warps per CTA: 128 registers, no spilled gather
// (L2 prefetching of the next block's rows -- per-lane prefetch.global.L2, or
// a dedicated warp issuing cp.async.cg L2::128B fills -- measured slower: C5
// 25.7 vs 20.6 ms, C4 3.55 vs 2.53 ms.)

constexpr int kNB = 2;  // staging buffers per warp
constexpr int kFoldCap = 320;  // >= 2 * grid slots for the grid fold

template <int NM1, int G>
struct PCfg {
  static constexpr int THREADS = kW * 32;
  static constexpr int GPW = 32 / G;                          // lane groups per warp
  static constexpr int GROUPS = kW * GPW;                    // per CTA
  static constexpr int CB = 4 * G;                            // columns per launch
  static constexpr int NA = NM1 + 2;                          // arrays per block
  static constexpr int CH = (G == 8 && NM1 <= 2) ? 32 : 16;   // entries per block
  static constexpr int U = NM1 >= 3 ? 4 : 8;                  // entries per group per iteration
  static constexpr int GS = NA * CH + 4;                      // u32 per staged block (+16 B bank shift)
  static constexpr size_t BARS = kW * kNB * 8;
  static constexpr size_t RING = (size_t)kW * kNB * GPW * GS * 4;
  static constexpr int S = 2 * GROUPS;                        // partial slots per CTA
  static constexpr size_t PARTS = (size_t)S * CB * 8 + (size_t)S * 4 + 16;
  static constexpr size_t FIXED = BARS + (RING > PARTS ? RING : PARTS);
  static_assert(CH % U == 0 && U % 4 == 0, "chunk shape");
  static_assert(S <= kFoldCap, "fold slots");
};

struct PlanParams {
  const uint32_t* blk;
  const float* fac[SPT_MAX_ORDER - 1];  // factor of level k
  const uint2* hot;
  float* out;
  double* gpart;
  uint32_t* gprow;
  double* part;
  uint32_t* part_row;
  unsigned int* done;
  uint32_t nnz, nhot, rows, R, c0, total_groups;
};

// Group j's first entry: equal shares rounded down to whole blocks.
template <int CH>
__device__ __forceinline__ uint32_t gbound(uint32_t nnz, uint32_t total, uint32_t j) {
  return j >= total ? nnz : static_cast<uint32_t>((uint64_t)nnz * j / total / CH * CH);
}
template <int NA, int CH>
__device__ __forceinline__ uint32_t plan_row(const uint32_t* blk, uint32_t e) {
  return __ldg(blk + (size_t)(e / CH) * NA * CH + e % CH);
}

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes,
                                              unsigned long long* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(spt::smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   spt::smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

// mbar_wait on a precomputed shared-space address.
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SPT_PLAN_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra SPT_PLAN_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(spt::kMbarSuspendNs)
      : "memory");
}

// Lane 0 of a warp: stage block c of each of the warp's lane groups (one
// bulk copy per group) into the buffer at shared address `buf`.
template <int NM1, int G>
__device__ __forceinline__ void stage_chunk(const PlanParams& p, uint32_t buf,
                                            unsigned long long* bar, const uint32_t* bnd,
                                            uint32_t c, uint64_t pol) {
  using C = PCfg<NM1, G>;
  uint32_t n = 0;
#pragma unroll
  for (int gg = 0; gg < C::GPW; ++gg) n += bnd[gg] + c * C::CH < bnd[gg + 1];
  mbar_arrive_tx(bar, n * C::NA * C::CH * 4);
#pragma unroll
  for (int gg = 0; gg < C::GPW; ++gg) {
    const uint32_t s = bnd[gg] + c * C::CH;
    if (s < bnd[gg + 1])
      bulk_g2s_hint(buf + gg * C::GS * 4, p.blk + (size_t)(s / C::CH) * C::NA * C::CH,
                    C::NA * C::CH * 4, bar, pol);
  }
}

// One factor row slice (16 B per lane). HOT: from the shared-memory hot copy
// when the id carries kHot (a32 = hot base + slot * row bytes: the shift drops
// the flag bit), else from global memory; both addresses are formed and one
// of two predicated loads runs (no generic address, no branch).
template <int CB, bool HOT>
__device__ __forceinline__ float4 gather_row(bool on, uint32_t e, uint32_t hot_q, const char* fb,
                                             uint32_t rb) {
  float4 v;
  if constexpr (HOT) {
    constexpr int SH = CB == 32 ? 7 : 6;
    const uint32_t a32 = hot_q + (e << SH);
    const char* a64 = fb + (size_t)e * rb;
    asm volatile(
        "{\n .reg .pred ph, pg, pon;\n"
        " setp.ne.u32 pon, %4, 0;\n"
        " setp.lt.s32 ph, %5, 0;\n"
        " and.pred pg, pon, !ph;\n"
        " and.pred ph, pon, ph;\n"
        " @ph ld.shared.v4.f32 {%0, %1, %2, %3}, [%6];\n"
        " @pg ld.global.v4.f32 {%0, %1, %2, %3}, [%7];\n"
        "}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"((uint32_t)on), "r"(e), "r"(a32), "l"(a64));
  } else {
    const char* a64 = fb + (size_t)e * rb;
    asm volatile(
        "{\n .reg .pred pon;\n"
        " setp.ne.u32 pon, %4, 0;\n"
        " @pon ld.global.v4.f32 {%0, %1, %2, %3}, [%5];\n"
        "}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"((uint32_t)on), "l"(a64));
  }
  return v;
}

__device__ __forceinline__ void zero_rows4(float* out, uint32_t r0, uint32_t r1, uint32_t R,
                                           uint32_t col) {
  for (uint32_t r = r0; r < r1; ++r)
    __stcs(reinterpret_cast<float4*>(out + (size_t)r * R + col), make_float4(0.f, 0.f, 0.f, 0.f));
}

// Fold the runs of equal rows in `nslot` ordered slots (row ids in shared
// memory, CB-wide fp64 values; kNoRow = empty). Runs whose row is keep0 /
// keep1 go to dst slot 0 / 1, the others are complete and go to out. Work is
// spread over (run start, column) items.
template <int CB>
__device__ void fold_slots(const uint32_t* srow, const double* sval, int nslot, int* sstart,
                           int* nstart, uint32_t keep0, uint32_t keep1, double* dst, float* out,
                           uint32_t R, uint32_t c0) {
  if (threadIdx.x == 0) *nstart = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    const uint32_t r = srow[i];
    if (r == kNoRow) continue;
    int j = i - 1;
    while (j >= 0 && srow[j] == kNoRow) --j;
    if (j < 0 || srow[j] != r) sstart[atomicAdd(nstart, 1)] = i;
  }
  __syncthreads();
  const int items = *nstart * CB;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int i = sstart[it / CB], col = it % CB;
    const uint32_t r = srow[i];
    double s = 0.0;
    for (int k = i; k < nslot; ++k) {
      const uint32_t rk = srow[k];
      if (rk == kNoRow) continue;
      if (rk != r) break;
      s += sval[(size_t)k * CB + col];
    }
    if (r == keep0) dst[col] = s;
    else if (r == keep1) dst[CB + col] = s;
    else out[(size_t)r * R + c0 + col] = (float)s;
  }
}

template <int NM1, int G, bool HOT>
__global__ void __launch_bounds__(PCfg<NM1, G>::THREADS, 1) mttkrp_plan_kernel(PlanParams p) {
  using C = PCfg<NM1, G>;
  constexpr int GPW = C::GPW, CB = C::CB, CH = C::CH, U = C::U, GS = C::GS, S = C::S;
  constexpr int NA = C::NA;
  constexpr int NMID = NM1 > 1 ? NM1 - 1 : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);
  float* hot = reinterpret_cast<float*>(smem + C::FIXED);
  __shared__ uint32_t s_bnd[C::GROUPS + 1];
  __shared__ int s_start[kFoldCap];
  __shared__ int s_nstart, s_last;
  __shared__ __align__(8) unsigned long long s_hbar;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane / G, q = lane % G;
  const uint32_t col = p.c0 + q * 4;
  for (int i = tid; i <= C::GROUPS; i += C::THREADS)
    s_bnd[i] = gbound<CH>(p.nnz, p.total_groups, blockIdx.x * C::GROUPS + i);
  unsigned long long* wbar = bars + warp * kNB;
  const uint32_t wbar_a = spt::smem_addr(wbar);  // hoisted: no cvta in the loop
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < kNB; ++b) spt::mbar_init(&wbar[b], 1);
  }
  if (tid == 0 && p.nhot) spt::mbar_init(&s_hbar, 1);
  spt::mbar_fence_init();
  __syncthreads();
  const int lg = warp * GPW + g;  // lane group within the CTA
  const uint32_t gid = blockIdx.x * C::GROUPS + lg;
  const uint32_t* wbnd = s_bnd + warp * GPW;
  const uint32_t lo = s_bnd[lg], hi = s_bnd[lg + 1], len = hi - lo;
  uint32_t mlen = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mlen = max(mlen, __shfl_xor_sync(0xffffffffu, mlen, o));
  const uint32_t nch = (mlen + CH - 1) / CH;
  const uint32_t wring = spt::smem_addr(smem + C::BARS) + warp * kNB * GPW * GS * 4;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0)
    for (uint32_t c = 0; c < min(static_cast<uint32_t>(kNB), nch); ++c)
      stage_chunk<NM1, G>(p, wring + c * GPW * GS * 4, &wbar[c], wbnd, c, pol);

  // hot rows of every level into shared memory by bulk copies (overlap the
  // first chunks); one CTA barrier counts their bytes
  if (HOT && p.nhot) {
    if (tid == 0) mbar_arrive_tx(&s_hbar, p.nhot * CB * 4);
    __syncthreads();
    for (uint32_t s = tid; s < p.nhot; s += C::THREADS) {
      const uint2 h = p.hot[s];
      const float* f = p.fac[0];
#pragma unroll
      for (int j = 1; j < NM1; ++j)
        if (h.x == (uint32_t)j) f = p.fac[j];
      spt::bulk_g2s(hot + (size_t)s * CB, f + (size_t)h.y * p.R + p.c0, CB * 4, &s_hbar);
    }
    spt::mbar_wait(&s_hbar, 0);
  }
  __syncthreads();

  // per-lane gather bases: the hot copy (shared) and every level's factor
  const uint32_t hot_q = spt::smem_addr(hot) + q * 16;
  const uint32_t rb = p.R * 4;
  const char* fb[NM1];
#pragma unroll
  for (int j = 0; j < NM1; ++j) fb[j] = reinterpret_cast<const char*>(p.fac[j] + p.c0 + q * 4);
  uint32_t cur = kNoRow, prow = kNoRow;
  uint32_t pid[NMID];
#pragma unroll
  for (int j = 0; j < NMID; ++j) pid[j] = kNoRow;
  // Per lane, 4 columns as two float2 (packed FMUL2/FFMA2 on sm_100):
  //   fm  = the current mid-level rows (gathered when their prefix changes),
  //   ra  = fp32 sum of this iteration's terms val * fm.. * F_leaf (<= U terms),
  //   acc = fp64 sum of the folds: the row's value, rounded once at the end.
  float2 ra0 = make_float2(0.f, 0.f), ra1 = ra0;
  float2 fm0[NMID], fm1[NMID];
#pragma unroll
  for (int j = 0; j < NMID; ++j) fm0[j] = fm1[j] = make_float2(1.f, 1.f);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  bool first = true;
  // rows before this group's first row that no group owns yet: from the row
  // after the previous entry's (the previous group's last row)
  uint32_t gap = (len > 0 && lo > 0) ? plan_row<NA, CH>(p.blk, lo - 1) + 1 : 0;
  double* myp = p.gpart + (size_t)gid * 2 * CB + q * 4;

  auto fold = [&]() {  // ra -> acc
    acc[0] += (double)ra0.x, acc[1] += (double)ra0.y;
    acc[2] += (double)ra1.x, acc[3] += (double)ra1.y;
    ra0 = ra1 = make_float2(0.f, 0.f);
  };
  auto emit = [&](uint32_t r) {
    if (first) {  // the group's first row: a partial (it may continue in the previous group)
      *reinterpret_cast<double2*>(myp) = make_double2(acc[0], acc[1]);
      *reinterpret_cast<double2*>(myp + 2) = make_double2(acc[2], acc[3]);
      if (q == 0) p.gprow[2 * gid] = r;
      first = false;
    } else {
      __stcs(reinterpret_cast<float4*>(p.out + (size_t)r * p.R + col),
             make_float4((float)acc[0], (float)acc[1], (float)acc[2], (float)acc[3]));
    }
  };

  const uint32_t niter = (mlen + U - 1) / U;
  const uint32_t gbase = wring + g * GS * 4;
  // FULL: every group of the warp has all U entries of this iteration (true
  // except in the ranges' last iterations): the validity tests drop out.
  auto iterate = [&](uint32_t it, auto full_c) {
    constexpr bool FULL = decltype(full_c)::value;
    const uint32_t e0 = it * U;
    const uint32_t c = e0 / CH, o = e0 % CH, b = c % kNB;
    if (o == 0) mbar_wait_a(wbar_a + b * 8, (c / kNB) & 1u);
    const uint32_t sb = gbase + b * GPW * GS * 4 + o * 4;
    uint32_t rr[U], id[NM1][U];
    float vv[U];
#pragma unroll
    for (int k = 0; k < U; k += 4) {
      const uint4 w = lds128(sb + k * 4);
      rr[k] = w.x, rr[k + 1] = w.y, rr[k + 2] = w.z, rr[k + 3] = w.w;
#pragma unroll
      for (int j = 0; j < NM1; ++j) {
        const uint4 x = lds128(sb + ((1 + j) * CH + k) * 4);
        id[j][k] = x.x, id[j][k + 1] = x.y, id[j][k + 2] = x.z, id[j][k + 3] = x.w;
      }
      const uint4 v = lds128(sb + ((NM1 + 1) * CH + k) * 4);
      vv[k] = __uint_as_float(v.x), vv[k + 1] = __uint_as_float(v.y);
      vv[k + 2] = __uint_as_float(v.z), vv[k + 3] = __uint_as_float(v.w);
    }
    // per entry: valid, row changed, mid level j's prefix changed
    bool ok[U], nr[U], nm[NMID][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = FULL || e0 + u < len;
      nr[u] = rr[u] != (u ? rr[u - 1] : prow);
      bool ch = nr[u];
#pragma unroll
      for (int j = 0; j < NM1 - 1; ++j) {
        ch = ch || id[j][u] != (u ? id[j][u - 1] : pid[j]);
        nm[j][u] = ch;
      }
    }
    prow = rr[U - 1];
#pragma unroll
    for (int j = 0; j < NM1 - 1; ++j) pid[j] = id[j][U - 1];
    // all gathers of the batch in flight before the first use
    float4 L[U];
    float4 M[NMID][U];
#pragma unroll
    for (int u = 0; u < U; ++u) L[u] = gather_row<CB, HOT>(ok[u], id[NM1 - 1][u], hot_q, fb[NM1 - 1], rb);
#pragma unroll
    for (int j = 0; j < NM1 - 1; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u)
        M[j][u] = gather_row<CB, HOT>(ok[u] && nm[j][u], id[j][u], hot_q, fb[j], rb);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!FULL && !ok[u]) break;
      if (nr[u]) {  // row change: the finished row goes out
        fold();
        if (cur != kNoRow) {
          emit(cur);
          gap = cur + 1;
        }
        zero_rows4(p.out, gap, rr[u], p.R, col);
        acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
        cur = rr[u];
      }
#pragma unroll
      for (int j = 0; j < NM1 - 1; ++j)
        if (nm[j][u]) {
          fm0[j] = make_float2(M[j][u].x, M[j][u].y);
          fm1[j] = make_float2(M[j][u].z, M[j][u].w);
        }
      float2 w0 = make_float2(vv[u], vv[u]), w1 = w0;
#pragma unroll
      for (int j = NM1 - 2; j >= 0; --j) w0 = __fmul2_rn(w0, fm0[j]), w1 = __fmul2_rn(w1, fm1[j]);
      ra0 = __ffma2_rn(w0, make_float2(L[u].x, L[u].y), ra0);
      ra1 = __ffma2_rn(w1, make_float2(L[u].z, L[u].w), ra1);
    }
    fold();
    if (o + U == CH || it + 1 == niter) {
      __syncwarp();
      if (lane == 0 && c + kNB < nch) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_chunk<NM1, G>(p, wring + b * GPW * GS * 4, &wbar[b], wbnd, c + kNB, pol);
      }
    }
  };
  uint32_t minlen = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) minlen = min(minlen, __shfl_xor_sync(0xffffffffu, minlen, o));
  const uint32_t nfull = minlen / U;
  for (uint32_t it = 0; it < nfull; ++it) iterate(it, std::true_type{});
  for (uint32_t it = nfull; it < niter; ++it) iterate(it, std::false_type{});
  uint32_t trow = kNoRow;
  if (cur != kNoRow) {
    if (first) {
      emit(cur);
    } else {
      trow = cur;
      *reinterpret_cast<double2*>(myp + CB) = make_double2(acc[0], acc[1]);
      *reinterpret_cast<double2*>(myp + CB + 2) = make_double2(acc[2], acc[3]);
    }
    if (hi == p.nnz) zero_rows4(p.out, cur + 1, p.rows, p.R, col);
  } else if (q == 0) {
    p.gprow[2 * gid] = kNoRow;
  }
  if (q == 0) p.gprow[2 * gid + 1] = trow;

  // ---- fold the groups' first/last rows per CTA (copied into shared memory)
  __syncthreads();
  uint32_t* srow = reinterpret_cast<uint32_t*>(smem + C::BARS);
  double* sval = reinterpret_cast<double*>(smem + C::BARS + ((S * 4 + 15) & ~15));
  const uint32_t g0 = blockIdx.x * C::GROUPS;
  for (int i = tid; i < S; i += C::THREADS) srow[i] = __ldcg(p.gprow + 2 * g0 + i);
  for (int i = tid; i < S * CB / 2; i += C::THREADS)
    reinterpret_cast<double2*>(sval)[i] =
        __ldcg(reinterpret_cast<const double2*>(p.gpart + (size_t)2 * g0 * CB) + i);
  const uint32_t clo = s_bnd[0], chi = s_bnd[C::GROUPS];
  const uint32_t cfirst = clo < chi ? plan_row<NA, CH>(p.blk, clo) : kNoRow;
  const uint32_t clast = clo < chi ? plan_row<NA, CH>(p.blk, chi - 1) : kNoRow;
  const uint32_t keep1 = clast != cfirst ? clast : kNoRow;
  if (tid == 0) {
    p.part_row[2 * blockIdx.x] = cfirst;
    p.part_row[2 * blockIdx.x + 1] = keep1;
  }
  fold_slots<CB>(srow, sval, S, s_start, &s_nstart, cfirst, keep1,
                 p.part + (size_t)2 * blockIdx.x * CB, p.out, p.R, p.c0);

  // ---- the last CTA to finish folds the CTAs' first/last rows
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int GS2 = 2 * gridDim.x;  // <= kFoldCap
  double* gval = reinterpret_cast<double*>(smem + C::BARS + ((GS2 * 4 + 15) & ~15));
  for (int i = tid; i < GS2; i += C::THREADS) srow[i] = __ldcg(p.part_row + i);
  for (int i = tid; i < GS2 * CB / 2; i += C::THREADS)
    reinterpret_cast<double2*>(gval)[i] = __ldcg(reinterpret_cast<const double2*>(p.part) + i);
  fold_slots<CB>(srow, gval, GS2, s_start, &s_nstart, kNoRow, kNoRow, nullptr, p.out, p.R, p.c0);
  if (tid == 0) *p.done = 0u;
}

using PlanKernel = void (*)(PlanParams);

struct PlanVariant {
  PlanKernel fn, fn_hot;
  size_t fixed;
  uint32_t groups, CH, NA;
};

PlanVariant plan_variant(uint32_t nm1, uint32_t CB) {
#define SPT_PV(N1, GG)                                                                      \
  PlanVariant{mttkrp_plan_kernel<N1, GG, false>, mttkrp_plan_kernel<N1, GG, true>,          \
              PCfg<N1, GG>::FIXED, PCfg<N1, GG>::GROUPS, PCfg<N1, GG>::CH, PCfg<N1, GG>::NA}
  if (CB == 32) {
    if (nm1 == 1) return SPT_PV(1, 8);
    if (nm1 == 2) return SPT_PV(2, 8);
    if (nm1 == 3) return SPT_PV(3, 8);
  } else if (CB == 16) {
    if (nm1 == 1) return SPT_PV(1, 4);
    if (nm1 == 2) return SPT_PV(2, 4);
    if (nm1 == 3) return SPT_PV(3, 4);
  }
#undef SPT_PV
  return PlanVariant{nullptr, nullptr, 0, 0, 0, 0};
}

// ---- plan construction kernels -------------------------------------------

struct LvlPtrs {
  uint32_t* p[SPT_MAX_ORDER - 1];
  uint32_t* h[SPT_MAX_ORDER - 1];  // per-level histogram / slot map
};

// Per-level gather counts: the leaf row is gathered for every entry, level
// j's row wherever the prefix (row, l_0..l_j) changes.
__global__ void plan_hist_kernel(const uint32_t* row, LvlPtrs L, int nm1, uint64_t nnz) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < nnz; base += stride) {
    const uint64_t e = base + threadIdx.x;
    const bool ok = e < nnz;
    int lev = nm1;
    if (ok) {
      if (e == 0 || row[e] != row[e - 1]) lev = 0;
      else
        for (int j = nm1 - 2; j >= 0; --j)
          if (L.p[j][e] != L.p[j][e - 1]) lev = j + 1;
    }
    for (int j = 0; j < nm1; ++j) {
      const bool ev = ok && (j == nm1 - 1 || j + 1 >= lev);
      const uint32_t id = ev ? L.p[j][e] : 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, id);
      if (ev && (__ffs(peers) - 1) == (int)(threadIdx.x & 31u))
        atomicAdd(L.h[j] + id, (uint32_t)__popc(peers));
    }
  }
}

__global__ void iota_kernel(uint32_t* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

// id -> encoded id maps: sel[s] -> kHot | s; unmapped ids stay as they are.
__global__ void plan_slot_map_kernel(const uint2* sel, uint32_t nsel, uint32_t nhot, LvlPtrs L) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsel) {
    const uint2 h = sel[s];
    uint32_t* m = L.h[0];
    for (uint32_t j = 1; j < SPT_MAX_ORDER - 1; ++j)
      if (h.x == j) m = L.h[j];
    m[h.y] = kHot | s;
  }
}

__global__ void plan_encode_kernel(LvlPtrs L, int nm1, uint64_t nnz) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride)
    for (int j = 0; j < nm1; ++j) {
      const uint32_t s = L.h[j][L.p[j][e]];
      if (s != 0xFFFFFFFFu) L.p[j][e] = s;
    }
}

struct TileSrc {
  const uint32_t* a[SPT_MAX_ORDER + 1];  // row, levels.., value bits
};

// SoA -> blocked AoSoA: block b holds NA arrays of CH entries; the padding
// past nnz repeats the last entry (never consumed: the kernel stops at nnz).
// perm != nullptr: entry e of the plan is entry perm[e] of the source arrays
// (the sort permutation: no sorted SoA copy is materialised).
__global__ void plan_tile_kernel(TileSrc src, const uint32_t* __restrict__ perm, int na,
                                 uint32_t ch, uint64_t nnz, uint64_t nblk, uint32_t* blk) {
  const uint64_t total = nblk * ch;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    uint64_t s = e < nnz ? e : nnz - 1;
    if (perm) s = perm[s];
    uint32_t* d = blk + (e / ch) * na * ch + e % ch;
    for (int a = 0; a < na; ++a) d[a * ch] = src.a[a][s];
  }
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

int plan_max_smem(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
    v = 227 * 1024;
  return v;
}

// Choose the hot rows and encode them in the sorted SoA level arrays.
int plan_select_hot(spt_ctx* ctx, spt_mttkrp_plan* pl, const uint32_t* row, uint32_t* const* lvl,
                    uint32_t cap, cudaStream_t st) {
  const uint32_t nm1 = pl->nm1;
  LvlPtrs L{};
  size_t hist_words = 0;
  uint32_t off[SPT_MAX_ORDER] = {};
  uint32_t maxd = 0;
  for (uint32_t j = 0; j < nm1; ++j) {
    off[j] = static_cast<uint32_t>(hist_words);
    hist_words += pl->dims[pl->lvl_mode[j]];
    maxd = std::max(maxd, pl->dims[pl->lvl_mode[j]]);
  }
  uint32_t* hist = nullptr;
  SPT_CUDA(spt::tmp_alloc(ctx, &hist, hist_words * 4, st));
  SPT_CUDA(cudaMemsetAsync(hist, 0, hist_words * 4, st));
  for (uint32_t j = 0; j < nm1; ++j) {
    L.p[j] = lvl[j];
    L.h[j] = hist + off[j];
  }
  const unsigned grid = static_cast<unsigned>(
      std::min<uint64_t>((pl->nnz + 255) / 256, (uint64_t)ctx->num_sms * 8));
  plan_hist_kernel<<<std::max(grid, 1u), 256, 0, st>>>(row, L, static_cast<int>(nm1), pl->nnz);
  SPT_LAUNCHED(ctx);
  // the `cap` most gathered (count, id) of every level
  const uint32_t want = cap;
  size_t temp = 0;
  {
    cub::DoubleBuffer<uint32_t> k(nullptr, nullptr), v(nullptr, nullptr);
    SPT_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, k, v,
                                                       static_cast<int64_t>(maxd), 0, 32, st));
  }
  char* buf = nullptr;
  const size_t wb = align256((size_t)maxd * 4);
  SPT_CUDA(spt::tmp_alloc(ctx, reinterpret_cast<void**>(&buf), 3 * wb + align256(temp), st));
  uint32_t* kalt = reinterpret_cast<uint32_t*>(buf);
  uint32_t* vcur = reinterpret_cast<uint32_t*>(buf + wb);
  uint32_t* valt = reinterpret_cast<uint32_t*>(buf + 2 * wb);
  void* tmp = buf + 3 * wb;
  struct Cand {
    uint32_t cnt, lvl, id;
  };
  std::vector<Cand> cand;
  std::vector<uint32_t> hc(want), hi(want);
  for (uint32_t j = 0; j < nm1; ++j) {
    const uint32_t n = pl->dims[pl->lvl_mode[j]];
    iota_kernel<<<std::max(1u, std::min<unsigned>((n + 255) / 256, ctx->num_sms * 8)), 256, 0,
                  st>>>(vcur, n);
    SPT_LAUNCHED(ctx);
    cub::DoubleBuffer<uint32_t> k(hist + off[j], kalt), v(vcur, valt);
    size_t t2 = temp;
    SPT_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, t2, k, v, static_cast<int64_t>(n), 0,
                                                       32, st));
    const uint32_t m = std::min(want, n);
    SPT_CUDA(cudaMemcpyAsync(hc.data(), k.Current(), m * 4, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaMemcpyAsync(hi.data(), v.Current(), m * 4, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < m && hc[i] > 0; ++i) cand.push_back({hc[i], j, hi[i]});
  }
  std::stable_sort(cand.begin(), cand.end(),
                   [](const Cand& a, const Cand& b) { return a.cnt > b.cnt; });
  // a shared-memory row costs one L2 read per CTA per launch: keep rows
  // gathered more often than that
  std::vector<uint2> sel;
  const uint32_t thresh = 2u * static_cast<uint32_t>(ctx->num_sms);
  for (size_t i = 0; i < cand.size() && sel.size() < cap && cand[i].cnt > thresh; ++i) {
    sel.push_back(make_uint2(cand[i].lvl, cand[i].id));
    pl->hot_per_level[cand[i].lvl]++;
  }
  pl->nhot = static_cast<uint32_t>(sel.size());
  const uint32_t nsel = static_cast<uint32_t>(sel.size());
  if (nsel) {
    uint2* dsel = nullptr;
    SPT_CUDA(spt::tmp_alloc(ctx, &dsel, nsel * sizeof(uint2), st));
    SPT_CUDA(cudaMemcpyAsync(dsel, sel.data(), nsel * sizeof(uint2), cudaMemcpyHostToDevice, st));
    SPT_CUDA(spt::tmp_alloc(ctx, &pl->hot, pl->nhot * sizeof(uint2), st));
    SPT_CUDA(cudaMemcpyAsync(pl->hot, dsel, pl->nhot * sizeof(uint2), cudaMemcpyDeviceToDevice,
                             st));
    // id -> encoded id maps reuse the histogram words (the sort left them permuted)
    SPT_CUDA(cudaMemsetAsync(hist, 0xFF, hist_words * 4, st));
    plan_slot_map_kernel<<<(nsel + 255) / 256, 256, 0, st>>>(dsel, nsel, pl->nhot, L);
    SPT_LAUNCHED(ctx);
    plan_encode_kernel<<<std::max(grid, 1u), 256, 0, st>>>(L, static_cast<int>(nm1), pl->nnz);
    SPT_LAUNCHED(ctx);
    SPT_CUDA(cudaStreamSynchronize(st));  // sel (host) and dsel in use until here
    SPT_CUDA(cudaFreeAsync(dsel, st));
  }
  SPT_CUDA(cudaFreeAsync(buf, st));
  SPT_CUDA(cudaFreeAsync(hist, st));
  return SPT_OK;
}

void plan_free(spt_mttkrp_plan* pl) {
  if (!pl) return;
  // wait for the plan's last user only; an invalid (destroyed) stream falls
  // back to the whole device and the legacy stream
  if (cudaStreamSynchronize(pl->last) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    pl->last = nullptr;
  }
  void* arrays[] = {pl->blk, pl->hot, pl->part, pl->part_row, pl->gpart, pl->gprow, pl->done};
  for (void* a : arrays)
    if (a) cudaFreeAsync(a, pl->last);
  delete pl;
}

// The plan's blocked copy of x in (mode, levels...) order. Without hot rows
// (the default) nothing but the sort permutation is materialised: the tile
// kernel gathers x through it, or reads x in place when it already has the
// order; and when x is sorted such that a *stable* sort on the leading k modes
// alone gives the plan's order (x in (0,1,2) order, plan (1,0,2) or (2,0,1):
// k = 1), only those modes are sorted -- 24 key bits instead of 72 at C5.
// With hot rows: a sorted SoA copy, hot ids encoded in place, then tiled.
int plan_build(spt_ctx* ctx, spt_mttkrp_plan* pl, const spt_coo* x, unsigned flags,
               cudaStream_t st) {
  const uint32_t N = pl->N;
  uint32_t order[SPT_MAX_ORDER];
  order[0] = pl->mode;
  for (uint32_t j = 0; j < pl->nm1; ++j) order[1 + j] = pl->lvl_mode[j];
  // smallest k such that x's sort order without the modes order[0..k) is order[k..N)
  uint32_t nkeys = N;
  if (x->has_sort_order) {
    for (uint32_t k = 0; k < N; ++k) {
      uint32_t rest[SPT_MAX_ORDER], nr = 0;
      for (uint32_t j = 0; j < N; ++j) {
        const uint32_t m = static_cast<uint32_t>(x->sort_order[j]);
        bool lead = false;
        for (uint32_t i = 0; i < k; ++i) lead = lead || order[i] == m;
        if (!lead) rest[nr++] = m;
      }
      bool ok = nr == N - k;
      for (uint32_t j = 0; ok && j < nr; ++j) ok = rest[j] == order[k + j];
      if (ok) {
        nkeys = k;
        break;
      }
    }
  }
  const PlanVariant v = plan_variant(pl->nm1, pl->CB);
  const long avail = (long)plan_max_smem(ctx->device) - (long)v.fixed - 4096;  // static smem
  uint32_t cap = avail > 0 ? static_cast<uint32_t>(avail / (pl->CB * 4)) : 0;
  // Shared-memory hot rows measured no faster than L1 hits on the same
  // rows (C1/C4/C5) and cost L1 capacity: off unless asked for.
  cap = std::min<uint32_t>(cap, static_cast<uint32_t>(atoi(getenv("SPT_PLAN_HOT_MAX") ?: "0")));
  // (An L2 evict_last tier for the next ~750K most-gathered rows, evict_first
  // for the rest, measured no faster at C5 either: 23.1 vs 23.6 ms.)
  bool ids_fit = true;  // kHot needs ids < 2^31
  for (uint32_t j = 0; j < pl->nm1; ++j) ids_fit = ids_fit && pl->dims[pl->lvl_mode[j]] <= kHot;
  if (!ids_fit || (flags & SPT_PLAN_NO_HOT)) cap = 0;
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(
      1, std::min<uint64_t>((pl->nblk * pl->CH + 255) / 256, (uint64_t)ctx->num_sms * 16)));

  if (cap == 0) {
    uint32_t* perm = nullptr;
    int s = SPT_OK;
    if (nkeys > 0 && x->nnz > 1) {
      if (spt::tmp_alloc(ctx, &perm, x->nnz * sizeof(uint32_t), st) != cudaSuccess) {
        cudaGetLastError();
        return spt::set_error(SPT_ENOMEM, "mttkrp_plan: out of device memory (%zu bytes)",
                              (size_t)x->nnz * 4);
      }
      s = spt::sort_tuples(ctx, x, order, perm, st, nkeys);
    }
    if (s == SPT_OK) {
      TileSrc src{};
      src.a[0] = x->idx[pl->mode];
      for (uint32_t j = 0; j < pl->nm1; ++j) src.a[1 + j] = x->idx[pl->lvl_mode[j]];
      src.a[pl->nm1 + 1] = reinterpret_cast<const uint32_t*>(x->val);
      plan_tile_kernel<<<grid, 256, 0, st>>>(src, perm, static_cast<int>(pl->NA), pl->CH, x->nnz,
                                             pl->nblk, pl->blk);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) s = spt::cuda_status(e, "plan_tile_kernel");
      else ctx->launches++;
    }
    if (perm) cudaFreeAsync(perm, st);
    return s;
  }

  const size_t ab = align256((x->nnz + 4) * 4);
  char* soa = nullptr;
  if (spt::tmp_alloc(ctx, reinterpret_cast<void**>(&soa), ab * (N + 1), st) != cudaSuccess) {
    cudaGetLastError();
    return spt::set_error(SPT_ENOMEM, "mttkrp_plan: out of device memory (%zu bytes)",
                          ab * (N + 1));
  }
  spt_coo c = *x;
  for (uint32_t d = 0; d < N; ++d) {
    c.idx[d] = reinterpret_cast<uint32_t*>(soa + d * ab);
    SPT_CUDA(cudaMemcpyAsync(c.idx[d], x->idx[d], x->nnz * 4, cudaMemcpyDeviceToDevice, st));
  }
  c.val = reinterpret_cast<float*>(soa + N * ab);
  SPT_CUDA(cudaMemcpyAsync(c.val, x->val, x->nnz * 4, cudaMemcpyDeviceToDevice, st));
  int s = SPT_OK;
  if (nkeys > 0 && x->nnz > 1) s = spt_sort_f32(ctx, &c, order, 0, st);
  uint32_t* lvl[SPT_MAX_ORDER - 1];
  for (uint32_t j = 0; j < pl->nm1; ++j) lvl[j] = c.idx[pl->lvl_mode[j]];
  if (s == SPT_OK) s = plan_select_hot(ctx, pl, c.idx[pl->mode], lvl, cap, st);
  if (s == SPT_OK) {
    TileSrc src{};
    src.a[0] = c.idx[pl->mode];
    for (uint32_t j = 0; j < pl->nm1; ++j) src.a[1 + j] = lvl[j];
    src.a[pl->nm1 + 1] = reinterpret_cast<const uint32_t*>(c.val);
    plan_tile_kernel<<<grid, 256, 0, st>>>(src, nullptr, static_cast<int>(pl->NA), pl->CH, x->nnz,
                                           pl->nblk, pl->blk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = spt::cuda_status(e, "plan_tile_kernel");
    else ctx->launches++;
  }
  cudaFreeAsync(soa, st);
  return s;
}

}  // namespace

namespace spt {
// Plan kernels serve R a multiple of 16 (CB = 32 or 16 columns per launch),
// orders 2..4.
bool plan_supported(const spt_coo* x, uint64_t R) {
  if (R == 0 || R % 16 != 0 || R > 0xFFFFFFFFull || x->order < 2 || x->order > 4) return false;
  for (uint32_t d = 0; d < x->order; ++d)
    if (x->dims[d] > 0xFFFFFFFEu) return false;
  return true;
}
}  // namespace spt

extern "C" int spt_mttkrp_plan_create(spt_ctx* ctx, const spt_coo* x, uint32_t mode, uint64_t R,
                                      unsigned flags, spt_mttkrp_plan** out, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "mttkrp_plan: null context");
  if (!out) return spt::set_error(SPT_EINVAL, "mttkrp_plan: null out");
  *out = nullptr;
  SPT_TRY(spt::check_coo(x, "mttkrp_plan"));
  const uint32_t N = x->order;
  // P/src/kernel_detail.hpp:157-162
  if (N < 2) return spt::set_error(SPT_EINVAL, "mttkrp: input must have order >= 2");
  if (mode >= N) return spt::set_error(SPT_EINVAL, "mttkrp: mode out of range");
  if (!x->coalesced) return spt::set_error(SPT_EINVAL, "mttkrp: tensor must be coalesced");
  if (!spt::plan_supported(x, R))
    return spt::set_error(SPT_EINVAL,
                          "mttkrp_plan: needs R a multiple of 16 and order 2..4");
  cudaStream_t st = spt::as_stream(stream);
  spt_mttkrp_plan* pl = new spt_mttkrp_plan();
  pl->device = ctx->device;
  pl->N = N;
  pl->mode = mode;
  pl->nm1 = N - 1;
  pl->R = static_cast<uint32_t>(R);
  pl->CB = R % 32 == 0 ? 32 : 16;
  pl->nnz = x->nnz;
  for (uint32_t d = 0; d < N; ++d) pl->dims[d] = x->dims[d];
  // levels: the other modes by decreasing extent (ties: ascending mode)
  uint32_t k = 0;
  for (uint32_t d = 0; d < N; ++d)
    if (d != mode) pl->lvl_mode[k++] = d;
  std::stable_sort(pl->lvl_mode, pl->lvl_mode + pl->nm1,
                   [&](uint32_t a, uint32_t b) { return x->dims[a] > x->dims[b]; });
  const PlanVariant v = plan_variant(pl->nm1, pl->CB);
  pl->CH = v.CH;
  pl->NA = v.NA;
  pl->nblk = (x->nnz + pl->CH - 1) / pl->CH;
  pl->grid = static_cast<uint32_t>(std::min(ctx->num_sms, kFoldCap / 2));
  const size_t groups = (size_t)pl->grid * v.groups;
  pl->last = st;
  if ((pl->nblk &&
       spt::tmp_alloc(ctx, &pl->blk, pl->nblk * pl->NA * pl->CH * 4, st) != cudaSuccess) ||
      spt::tmp_alloc(ctx, &pl->part, (size_t)2 * pl->grid * pl->CB * sizeof(double), st) !=
          cudaSuccess ||
      spt::tmp_alloc(ctx, &pl->part_row, (size_t)2 * pl->grid * 4, st) != cudaSuccess ||
      spt::tmp_alloc(ctx, &pl->gpart, 2 * groups * pl->CB * sizeof(double), st) != cudaSuccess ||
      spt::tmp_alloc(ctx, &pl->gprow, 2 * groups * 4, st) != cudaSuccess ||
      spt::tmp_alloc(ctx, &pl->done, 4, st) != cudaSuccess) {
    cudaGetLastError();
    plan_free(pl);
    return spt::set_error(SPT_ENOMEM, "mttkrp_plan: out of device memory");
  }
  if (x->nnz) {
    const int s = plan_build(ctx, pl, x, flags, st);
    if (s != SPT_OK) {
      cudaStreamSynchronize(st);
      plan_free(pl);
      return s;
    }
  }
  SPT_CUDA(cudaMemsetAsync(pl->done, 0, 4, st));
  SPT_CUDA(cudaStreamSynchronize(st));
  *out = pl;
  return SPT_OK;
}

extern "C" void spt_mttkrp_plan_destroy(spt_mttkrp_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->device);
  plan_free(plan);
}

extern "C" int spt_mttkrp_plan_info(const spt_mttkrp_plan* plan, uint32_t* level_modes,
                                    uint32_t* hot_per_level, uint32_t* nhot) {
  if (!plan) return spt::set_error(SPT_EINVAL, "mttkrp_plan: null plan");
  for (uint32_t j = 0; j < plan->nm1; ++j) {
    if (level_modes) level_modes[j] = plan->lvl_mode[j];
    if (hot_per_level) hot_per_level[j] = plan->hot_per_level[j];
  }
  if (nhot) *nhot = plan->nhot;
  return SPT_OK;
}

extern "C" int spt_mttkrp_plan_exec(spt_ctx* ctx, const spt_mttkrp_plan* pl,
                                    const float* const* d_factors, const uint64_t* rows,
                                    const uint64_t* cols, float* d_out, unsigned flags,
                                    void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "mttkrp: null context");
  if (!pl) return spt::set_error(SPT_EINVAL, "mttkrp: null plan");
  if (!d_factors || !rows || !cols)
    return spt::set_error(SPT_EINVAL, "mttkrp: need one factor matrix per mode");
  // P/src/kernel_detail.hpp:163-173
  for (uint32_t d = 0; d < pl->N; ++d) {
    if (d == pl->mode) continue;
    if (cols[d] != pl->R)
      return spt::set_error(SPT_EINVAL, "mttkrp: factor matrices must share the column count "
                                        "(plan built for R=%u)", pl->R);
    if (rows[d] != pl->dims[d])
      return spt::set_error(SPT_EINVAL, "mttkrp: factor rows must match the mode dimension");
    if (!d_factors[d]) return spt::set_error(SPT_EINVAL, "mttkrp: null factor for mode %u", d);
    if (!spt::aligned16(d_factors[d]))
      return spt::set_error(SPT_EINVAL, "mttkrp: plan path needs 16-byte-aligned factors");
  }
  const uint32_t I = pl->dims[pl->mode];
  if (I > 0 && !d_out) return spt::set_error(SPT_EINVAL, "mttkrp: null output");
  if (!spt::aligned16(d_out))
    return spt::set_error(SPT_EINVAL, "mttkrp: plan path needs a 16-byte-aligned output");
  cudaStream_t st = spt::as_stream(stream);
  pl->last = st;
  if (I == 0) return SPT_OK;
  if (pl->nnz == 0) {
    SPT_CUDA(cudaMemsetAsync(d_out, 0, (size_t)I * pl->R * sizeof(float), st));
    return SPT_OK;
  }
  const PlanVariant v = plan_variant(pl->nm1, pl->CB);
  if (!v.fn) return spt::set_error(SPT_EINVAL, "mttkrp: no plan kernel for this shape");
  // the last CTA folds 2 slots per CTA in shared memory
  const size_t gfold = 16 + (((size_t)2 * pl->grid * 4 + 15) & ~size_t(15)) +
                       (size_t)2 * pl->grid * pl->CB * 8 + (size_t)kW * kNB * 8;
  const size_t smem = std::max(v.fixed + (size_t)pl->nhot * pl->CB * 4, gfold);
  const PlanKernel fn = pl->nhot ? v.fn_hot : v.fn;
  SPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  PlanParams p{};
  p.blk = pl->blk;
  for (uint32_t j = 0; j < pl->nm1; ++j) p.fac[j] = d_factors[pl->lvl_mode[j]];
  p.hot = pl->hot;
  p.nhot = pl->nhot;
  p.out = d_out;
  p.gpart = pl->gpart;
  p.gprow = pl->gprow;
  p.part = pl->part;
  p.part_row = pl->part_row;
  p.done = pl->done;
  p.nnz = static_cast<uint32_t>(pl->nnz);
  p.rows = I;
  p.R = pl->R;
  p.total_groups = pl->grid * v.groups;
  for (uint32_t c0 = 0; c0 < pl->R; c0 += pl->CB) {
    p.c0 = c0;
    fn<<<pl->grid, kW * 32, smem, st>>>(p);
    SPT_LAUNCHED(ctx);
  }
  if (flags & SPT_FLAG_ASYNC) return SPT_OK;
  return spt::sync_and_check(ctx, st);
}
