// One-wave segmented MTTKRP for small and medium inputs (C1: 1M nonzeros,
// R = 16; used up to 32M entries when rows average >= 16 entries).
//
// Reference: seq::mttkrp / par::mttkrp (P/src/kernels_seq.cpp:153-174,
// P/src/kernel_detail.hpp:176-188), input sorted with the output mode leading.
//
// At this size the tiled kernels of mttkrp.cu are a latency chain (ticket ->
// staging -> 8 dependent gather batches -> fold -> look-back, ~28 us for a
// 5 us transfer). Here the whole grid is one resident wave and every warp owns
// one contiguous, equal share of the entries -- no tickets, no tile look-back:
//   * a warp first pulls its whole share of entry words into shared memory
//     with cp.async (every word in flight at once: one DRAM round trip instead
//     of one per iteration), in chunks of kOwChunk entries for larger inputs;
//   * a warp step covers 32/G entries (G lanes per factor row, one or two
//     float4 slices each); U steps are gathered at once (one L1/L2 round trip
//     per iteration);
//   * each term is val * F_d0 * F_d1 ... in fp32, d ascending, exactly the
//     reference's product; a lane group accumulates its entries of the current
//     row in fp64 (fp32 across the <= U terms of one iteration);
//   * when a step's entries are not all of the current row (rare: a warp's
//     share holds a few rows), the step is replayed entry by entry and finished
//     rows are reduced over the lane groups by a fixed shuffle tree;
//   * rows strictly inside a warp's share are written once; its first and last
//     row go to two fp64 partial slots in shared memory (slot 0 flagged when
//     the row continues the previous share's); the CTA folds its warps' slots
//     into two global slots, and a second small kernel sums each row's run of
//     CTA slots in slot order. Rows without entries are zero-filled
//     by the warp whose share spans the gap. Deterministic: the split and both
//     summation orders are fixed by (nnz, grid).
#include <algorithm>

#include "internal.cuh"

namespace {

#ifndef SPT_OW_THREADS
#define SPT_OW_THREADS 384
#endif
constexpr int kOwThreads = SPT_OW_THREADS;
constexpr int kOwWarps = kOwThreads / 32;
constexpr int kOwU = 4;
constexpr int kOwChunk = 288;  // entries of a share staged at a time (C1's share: 282)
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr uint32_t kContinues = 0x80000000u;  // slot-0 row id flag: the row began in an earlier share

struct OwParams {
  const uint32_t* out_idx;
  const uint32_t* oidx[SPT_MAX_ORDER - 1];
  const float* ofac[SPT_MAX_ORDER - 1];
  const float* val;
  float* out;
  uint32_t nnz, rows, R, nwarps, share_q, share_r;
  double* part;    // [2 * nwarps][R]
  uint32_t* prow;  // [2 * nwarps]
  unsigned long long* err;
};

// Share w starts at w*q + min(w, r) (q, r = nnz / shares, nnz % shares),
// rounded down to a multiple of 4.
__device__ __forceinline__ uint32_t share_cut(uint32_t nnz, uint32_t shares, uint32_t q,
                                              uint32_t r, uint32_t w) {
  if (w >= shares) return nnz;
  return (w * q + min(w, r)) & ~3u;
}

__device__ __forceinline__ void ow_zero_rows(float* out, uint32_t r0, uint32_t r1, uint32_t R,
                                             unsigned lane) {
  if (r0 >= r1) return;
  float4* o = reinterpret_cast<float4*>(out + static_cast<size_t>(r0) * R);
  const size_t n4 = static_cast<size_t>(r1 - r0) * R / 4;
  for (size_t i = lane; i < n4; i += 32) __stcs(o + i, make_float4(0.f, 0.f, 0.f, 0.f));
}

// One warp's share. G lanes per factor row, V float4 slices (4V columns) per
// lane: R = 4 G V. myrow[2] / myslots[2][R]: the share's first-row and
// last-row partials (in shared memory; the CTA folds them afterwards); sw: the
// warp's staging area.
template <int NM1, int G, int V>
__device__ __forceinline__ void ow_share(const OwParams& p, uint32_t w, uint32_t* myrow,
                                         double* myslots, uint32_t* sw) {
  constexpr int EPW = 32 / G;  // entries per warp step
  constexpr int U = kOwU / V;  // steps gathered at once
  constexpr int C2 = 2 * V;    // float2 pairs per lane
  const unsigned lane = threadIdx.x & 31u, g = lane / G, q = lane % G;
  // equal shares cut at multiples of 4 entries: every array's piece of a share
  // starts 16-byte aligned (16-byte cp.async.cg, which also keeps the entry
  // stream out of L1 -- that is for the factor rows)
  const uint32_t lo = share_cut(p.nnz, p.nwarps, p.share_q, p.share_r, w);
  const uint32_t hi = share_cut(p.nnz, p.nwarps, p.share_q, p.share_r, w + 1);
  double* mypart = myslots + q * 4 * V;
  if (lo >= hi) {
    if (lane == 0) myrow[0] = myrow[1] = kNoRow;
    return;
  }
  const float* fq[NM1];
#pragma unroll
  for (int j = 0; j < NM1; ++j) fq[j] = p.ofac[j] + q * 4 * V;
  const uint32_t rb = p.R * 4;  // row bytes

  uint32_t cur = kNoRow;       // current row (warp-uniform)
  int flushed = 0;             // rows finished so far
  double acc[2 * C2];
  float2 ra[C2];
#pragma unroll
  for (int c = 0; c < C2; ++c) {
    acc[2 * c] = acc[2 * c + 1] = 0.0;
    ra[c] = make_float2(0.f, 0.f);
  }
  // rows before the share's first row that no earlier share ends in
  const uint32_t prev_row = lo ? __ldg(p.out_idx + lo - 1) : kNoRow;
  uint32_t gap = lo ? prev_row + 1 : 0;
  const bool first_continues = lo && prev_row == __ldg(p.out_idx + lo);

  auto fold = [&]() {
#pragma unroll
    for (int c = 0; c < C2; ++c) {
      acc[2 * c] += static_cast<double>(ra[c].x), acc[2 * c + 1] += static_cast<double>(ra[c].y);
      ra[c] = make_float2(0.f, 0.f);
    }
  };
  // The finished row `cur`: sum the lane groups' parts (fixed xor tree) and
  // write it -- the share's first row to slot 0 (it may continue an earlier
  // share's last row), later ones to the output.
  auto finish = [&](bool last) {
    fold();
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
#pragma unroll
      for (int c = 0; c < 2 * C2; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    }
    if (flushed == 0 || last) {
      const int slot = flushed == 0 ? 0 : 1;
      if (g == 0) {
        double* d = mypart + static_cast<size_t>(slot) * p.R;
#pragma unroll
        for (int c = 0; c < C2; ++c)
          *reinterpret_cast<double2*>(d + 2 * c) = make_double2(acc[2 * c], acc[2 * c + 1]);
      }
      if (lane == 0) myrow[slot] = (slot == 0 && first_continues) ? (cur | kContinues) : cur;
    } else if (g == 0) {
      float* o = p.out + static_cast<size_t>(cur) * p.R + q * 4 * V;
#pragma unroll
      for (int k = 0; k < V; ++k)
        __stcs(reinterpret_cast<float4*>(o) + k,
               make_float4(static_cast<float>(acc[4 * k]), static_cast<float>(acc[4 * k + 1]),
                           static_cast<float>(acc[4 * k + 2]),
                           static_cast<float>(acc[4 * k + 3])));
    }
    ++flushed;
#pragma unroll
    for (int c = 0; c < 2 * C2; ++c) acc[c] = 0.0;
  };

  // the share's entry words, staged per warp: [row | ids.. | val][kOwChunk]
  const uint32_t sw_a = spt::smem_addr(sw);
  for (uint32_t c0 = lo; c0 < hi; c0 += kOwChunk) {
    const uint32_t n = min(static_cast<uint32_t>(kOwChunk), hi - c0);
    __syncwarp();  // the previous chunk is consumed
    for (uint32_t i = lane * 4; i < n; i += 128) {
      const uint32_t d = sw_a + i * 4;
      if (i + 4 <= n) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                     "l"(p.out_idx + c0 + i));
#pragma unroll
        for (int j = 0; j < NM1; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           d + (1 + j) * kOwChunk * 4),
                       "l"(p.oidx[j] + c0 + i));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         d + (NM1 + 1) * kOwChunk * 4),
                     "l"(p.val + c0 + i));
      } else {
        for (uint32_t k = i; k < n; ++k) {
          const uint32_t dk = sw_a + k * 4;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dk),
                       "l"(p.out_idx + c0 + k));
#pragma unroll
          for (int j = 0; j < NM1; ++j)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             dk + (1 + j) * kOwChunk * 4),
                         "l"(p.oidx[j] + c0 + k));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           dk + (NM1 + 1) * kOwChunk * 4),
                       "l"(p.val + c0 + k));
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    for (uint32_t b0 = 0; b0 < n; b0 += U * EPW) {
      float4 F[NM1][U][V];
      uint32_t r[U];
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = b0 + u * EPW + g;
        const bool ok = i < n;
        r[u] = ok ? sw[i] : kNoRow;
        v[u] = ok ? __uint_as_float(sw[(NM1 + 1) * kOwChunk + i]) : 0.f;
#pragma unroll
        for (int j = 0; j < NM1; ++j) {
          // byte address = base + id * row bytes: one IMAD.WIDE
          const float4* row = reinterpret_cast<const float4*>(
              reinterpret_cast<const char*>(fq[j]) +
              static_cast<size_t>(ok ? sw[(1 + j) * kOwChunk + i] : 0u) * rb);
#pragma unroll
          for (int k = 0; k < V; ++k)
            F[j][u][k] = ok ? __ldg(row + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // val * F_d0 * F_d1 ... (d ascending): each term is bit-identical to
        // the reference's (packed FMUL2/FFMA2 measured no faster here)
        float2 t[C2];
#pragma unroll
        for (int c = 0; c < C2; ++c) t[c] = make_float2(v[u], v[u]);
#pragma unroll
        for (int j = 0; j < NM1; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k) {
            t[2 * k].x *= F[j][u][k].x, t[2 * k].y *= F[j][u][k].y;
            t[2 * k + 1].x *= F[j][u][k].z, t[2 * k + 1].y *= F[j][u][k].w;
          }
        const bool valid = r[u] != kNoRow;
        if (__all_sync(0xffffffffu, !valid || r[u] == cur)) {
          // invalid entries carry zero terms
#pragma unroll
          for (int c = 0; c < C2; ++c) ra[c].x += t[c].x, ra[c].y += t[c].y;
        } else {
          // a row boundary (or the share's first entry) inside this step:
          // one round per row present in the step, found by ballot
          uint32_t todo = __ballot_sync(0xffffffffu, valid);  // lanes still to add
          while (todo) {
            const int e = (__ffs(todo) - 1) / G;  // first group not added yet
            const uint32_t re = __shfl_sync(0xffffffffu, r[u], e * G);
            if (re != cur) {
              if (cur != kNoRow) {
                if (re < cur && lane == 0)
                  atomicMin(p.err + 2, static_cast<unsigned long long>(c0 + b0 + u * EPW + e));
                finish(false);
                gap = cur + 1;
              } else if (gap > re + 1 && lane == 0) {  // the previous share ends in a later row
                atomicMin(p.err + 2, static_cast<unsigned long long>(lo));
              }
              ow_zero_rows(p.out, gap, re, p.R, lane);
              cur = re;
            }
            // every group of this row in the step (they are consecutive)
            const bool mine = valid && r[u] == cur && ((todo >> lane) & 1u);
            if (mine) {
#pragma unroll
              for (int c = 0; c < C2; ++c) ra[c].x += t[c].x, ra[c].y += t[c].y;
            }
            todo &= ~__ballot_sync(0xffffffffu, mine);
          }
        }
      }
      fold();
    }
  }
  finish(true);
  if (flushed == 1 && lane == 0) myrow[1] = kNoRow;  // the whole share was one row
  if (hi == p.nnz) ow_zero_rows(p.out, cur + 1, p.rows, p.R, lane);
}

// The kernel: every warp does its share, then the CTA folds its warps' 2 x 8
// slots in shared memory: runs of equal rows are summed in slot order; the
// CTA's first run (it may continue the previous CTA's last row: the flag of
// its first slot is kept) and last run go to the CTA's two global slots, runs
// in between are complete and go to the output. The fold kernel then only
// sees 2 slots per CTA: a heavy row spanning most of the tensor is a run of a
// few hundred CTA slots, not thousands of warp slots.
template <int NM1, int G, int V>
__global__ void __launch_bounds__(kOwThreads, 768 / kOwThreads) mttkrp_ow_kernel(OwParams p) {
  constexpr int S = 2 * kOwWarps;
  extern __shared__ __align__(16) uint32_t ow_smem[];
  const unsigned warp = threadIdx.x >> 5;
  // let the fold kernel's CTAs become resident now (they block in
  // griddepcontrol.wait until this grid has finished and flushed its writes)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  double* sval = reinterpret_cast<double*>(ow_smem + kOwWarps * (NM1 + 2) * kOwChunk);  // [S][R]
  uint32_t* srow = reinterpret_cast<uint32_t*>(sval + static_cast<size_t>(S) * p.R);   // [S]
  ow_share<NM1, G, V>(p, blockIdx.x * kOwWarps + warp, srow + 2 * warp,
                      sval + static_cast<size_t>(2 * warp) * p.R,
                      ow_smem + warp * (NM1 + 2) * kOwChunk);
  uint32_t* grow = p.prow + 2 * blockIdx.x;
  double* gpart = p.part + static_cast<size_t>(2 * blockIdx.x) * p.R;
  if (threadIdx.x == 0) grow[0] = grow[1] = kNoRow;
  __syncthreads();
  for (uint32_t item = threadIdx.x; item < S * p.R; item += kOwThreads) {
    const int i = static_cast<int>(item / p.R);
    const uint32_t c = item % p.R;
    const uint32_t tag = srow[i];
    if (tag == kNoRow) continue;
    const uint32_t row = tag & ~kContinues;
    int j = i - 1;
    while (j >= 0 && srow[j] == kNoRow) --j;
    if (j >= 0 && (srow[j] & ~kContinues) == row) continue;  // not the run's first slot
    double s = 0.0;
    int k = i;
    bool last_run = true;
    for (; k < S; ++k) {
      const uint32_t t = srow[k];
      if (t == kNoRow) continue;
      if ((t & ~kContinues) != row) {
        last_run = false;
        break;
      }
      s += sval[static_cast<size_t>(k) * p.R + c];
    }
    if (j < 0) {  // the CTA's first run: tag with its continuation flag
      gpart[c] = s;
      if (c == 0) grow[0] = tag;
    } else if (last_run) {
      gpart[p.R + c] = s;
      if (c == 0) grow[1] = row;
    } else {
      p.out[static_cast<size_t>(row) * p.R + c] = static_cast<float>(s);
    }
  }
}

// Sum each row's run of partial slots in slot order. One thread per (slot,
// column); the run's first slot -- a slot 1, or a slot 0 whose row does not
// continue the previous share's -- does the work: its own part plus the slot 0
// of the following shares for as long as they continue the row (a share whose
// slot 1 is used ends the run: its last row is another one). The GL = min(R,
// 32) lanes of a slot walk the run together: each reads the tags of one of the
// next GL shares, ballots find where the run stops, then every lane adds its
// column of the member slots in slot order -- a heavy row spanning hundreds of
// shares costs a dozen round trips instead of one per four shares.
__global__ void ow_fold_kernel(const double* __restrict__ part, const uint32_t* __restrict__ prow,
                               uint32_t nslots, uint32_t R, float* __restrict__ out) {
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t i = gt / R, c = gt % R;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t GL = R < 32u ? R : 32u;
  const unsigned base = lane & ~(GL - 1u), l = lane - base;
  const uint32_t gmask = GL == 32u ? 0xffffffffu : ((1u << GL) - 1u);
  // launched with programmatic stream serialization: the grid is resident
  // before the main kernel ends; wait for its writes here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tag = i < nslots ? prow[i] : kNoRow;
  const bool start = tag != kNoRow && !(tag & kContinues);
  const uint32_t row = tag;
  double s = start ? part[static_cast<size_t>(i) * R + c] : 0.0;
  // a slot 0 with its share's slot 1 in use is a complete run by itself
  bool walk = start && ((i & 1u) || prow[i + 1] == kNoRow);
  uint32_t k0 = (i | 1u) + 1;
  while (__any_sync(0xffffffffu, walk)) {
    // lane l of the slot's group looks at share l of the next GL
    const uint32_t k = k0 + 2 * l;
    const bool in = walk && k < nslots;
    const uint32_t t0 = in ? prow[k] : 0u;  // 0 carries no flag: ends the run
    const uint32_t t1 = in ? prow[k + 1] : 0u;
    const bool empty = t0 == kNoRow && t1 == kNoRow;  // an empty share (nnz < shares)
    const bool member = t0 == (row | kContinues);
    const uint32_t bad_m = (__ballot_sync(0xffffffffu, !empty && !member) >> base) & gmask;
    const uint32_t end_m = (__ballot_sync(0xffffffffu, member && t1 != kNoRow) >> base) & gmask;
    const uint32_t mem_m = (__ballot_sync(0xffffffffu, member) >> base) & gmask;
    const uint32_t first_bad = bad_m ? __ffs(bad_m) - 1 : GL;
    const uint32_t first_end = end_m ? __ffs(end_m) - 1 : GL;
    const uint32_t ntake = min(first_bad, first_end + 1);
    if (walk) {
      uint32_t take = mem_m & (ntake >= 32u ? 0xffffffffu : ((1u << ntake) - 1u));
      // slot order; all of the round's loads in flight (absent ones add 0.0)
      double v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u)
        v[u] = (take >> u) & 1u ? part[static_cast<size_t>(k0 + 2 * u) * R + c] : 0.0;
#pragma unroll
      for (int u = 0; u < 32; ++u) s += v[u];
      if (first_bad < GL || first_end < GL) walk = false;
      k0 += 2 * GL;
    }
  }
  if (start) out[static_cast<size_t>(row) * R + c] = static_cast<float>(s);
}

using OwFn = void (*)(OwParams);
template <int G, int V>
OwFn pick_ow(int nm1) {
  switch (nm1) {
    case 1: return mttkrp_ow_kernel<1, G, V>;
    case 2: return mttkrp_ow_kernel<2, G, V>;
    case 3: return mttkrp_ow_kernel<3, G, V>;
    default: return nullptr;
  }
}

}  // namespace

namespace spt {

// Inputs this path serves: R = 4G with G a power of two <= 32, orders 2..4,
// 16-byte-aligned factors and output, at most kOwMaxNnz entries.
bool mttkrp_onewave_ok(const spt_coo* x, uint64_t R, const float* const* d_factors, uint32_t mode,
                       const float* d_out) {
  // Measured against the tiled kernels (tune/probe_c1_times.py, uniform rows):
  // 16 vs 20 us at 0.5M, 21 vs 29 at 1M, 38 vs 61 at 3M, 94 vs 138 at 10M,
  // 175 vs 250 at 20M entries (R = 16, 1000 rows); 701 vs 812 us with 20
  // entries per row, but 1232 vs 1114 with 4: every row end costs a reduction
  // over the lane groups, so short rows stay with the tiled kernels.
#ifndef SPT_OW_MAX_NNZ
#define SPT_OW_MAX_NNZ 32000000ull
#endif
#ifndef SPT_OW_MIN_ROW
#define SPT_OW_MIN_ROW 16ull
#endif
  if (x->nnz == 0 || x->nnz > SPT_OW_MAX_NNZ) return false;
  if (x->nnz < SPT_OW_MIN_ROW * x->dims[mode]) return false;
  if (x->order < 2 || x->order > 4) return false;
  if (x->dims[mode] >= kContinues) return false;  // the slot tag's top bit is a flag
  if (!(R == 8 || R == 16 || R == 32 || R == 64 || R == 128)) return false;
  if (!aligned16(d_out) || !aligned16(x->val)) return false;
  for (uint32_t d = 0; d < x->order; ++d) {
    if (!aligned16(x->idx[d])) return false;
    if (d != mode && !aligned16(d_factors[d])) return false;
  }
  return true;
}

int mttkrp_onewave(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors, uint32_t mode,
                   uint32_t R, float* d_out, cudaStream_t st) {
  const int nm1 = static_cast<int>(x->order) - 1;
  // One float4 slice per lane. (Two slices per lane, V = 2, halve the index
  // and address work per column but make the fp64 reduction over the lane
  // groups at a row's end 5x longer -- 24 vs 16 us at C1.)
  OwFn fn = nullptr;
  switch (R) {
    case 8: fn = pick_ow<2, 1>(nm1); break;
    case 16: fn = pick_ow<4, 1>(nm1); break;
    case 32: fn = pick_ow<8, 1>(nm1); break;
    case 64: fn = pick_ow<16, 1>(nm1); break;
    case 128: fn = pick_ow<32, 1>(nm1); break;
  }
  if (!fn) return set_error(SPT_EINVAL, "mttkrp: no one-wave kernel for this shape");
  const size_t smem = static_cast<size_t>(kOwWarps) * (nm1 + 2) * kOwChunk * 4 +
                      static_cast<size_t>(2 * kOwWarps) * R * 8 + 2 * kOwWarps * 4;
  // attribute + occupancy once per (kernel, device): a 20 us op should not pay
  // two runtime queries per call
  struct Cached {
    OwFn fn;
    int device, per_sm;
  };
  static thread_local Cached cache[8] = {};
  int per_sm = 0;
  for (const Cached& c : cache)
    if (c.fn == fn && c.device == ctx->device) per_sm = c.per_sm;
  if (per_sm == 0) {
    SPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    SPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kOwThreads, smem));
    per_sm = std::max(per_sm, 1);
    static thread_local int next = 0;
    cache[next++ % 8] = Cached{fn, ctx->device, per_sm};
  }
  const uint32_t grid = static_cast<uint32_t>(std::max(per_sm, 1) * ctx->num_sms);
  OwParams p{};
  p.out_idx = x->idx[mode];
  int j = 0;
  for (uint32_t d = 0; d < x->order; ++d) {
    if (d == mode) continue;
    p.oidx[j] = x->idx[d];
    p.ofac[j] = d_factors[d];
    ++j;
  }
  p.val = x->val;
  p.out = d_out;
  p.nnz = static_cast<uint32_t>(x->nnz);
  p.rows = x->dims[mode];
  p.R = R;
  p.nwarps = grid * kOwWarps;
  p.share_q = p.nnz / p.nwarps;
  p.share_r = p.nnz % p.nwarps;
  p.err = ctx->d_err;
  const size_t slots = static_cast<size_t>(2) * grid;  // two per CTA
  const size_t pbytes = ((slots * R * sizeof(double) + 255) / 256) * 256;
  void* scratch;
  SPT_TRY(ctx_scratch(ctx, pbytes + slots * sizeof(uint32_t), &scratch));
  p.part = static_cast<double*>(scratch);
  p.prow = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + pbytes);
  fn<<<grid, kOwThreads, smem, st>>>(p);
  SPT_LAUNCHED(ctx);
  const uint32_t threads = static_cast<uint32_t>(slots) * R;
  // the fold's launch overlaps the main kernel's tail (programmatic dependent
  // launch); it waits on griddepcontrol.wait before reading the slots
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((threads + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  SPT_CUDA(cudaLaunchKernelEx(&cfg, ow_fold_kernel, static_cast<const double*>(p.part),
                              static_cast<const uint32_t*>(p.prow),
                              static_cast<uint32_t>(slots), R, d_out));
  ctx->launches++;
  return SPT_OK;
}

}  // namespace spt
