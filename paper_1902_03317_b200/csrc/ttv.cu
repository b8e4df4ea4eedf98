// K6 TTV: one output entry per fiber, value = sum over the fiber of val*v[k].
//
// Reference: seq::ttv P/src/kernels_seq.cpp:69-101, par::ttv
// P/src/kernels_par.cpp:179-216, ttv_fiber_value P/src/kernel_detail.hpp:121-128,
// check_fiber_kernel_inputs P/src/kernel_detail.hpp:106-119, drop_mode :142-149.
//
// x is sorted with `mode` last, so a fiber is a contiguous entry range
// [fptr[f], fptr[f+1]). The kernel is nnz-balanced, not fiber-balanced: a CTA
// owns 2048 consecutive entries (256 threads x 8, blocked), forms each term
// val*v[k] in fp32 (bit-identical to the reference's term), and reduces the
// terms by fiber with a block-wide segmented scan in fp64 (cub::BlockScan over
// (head-flag, sum) pairs). Fibers that cross a tile boundary are completed by
// the tile holding their last entry, using the same epoch-tagged decoupled
// look-back as MTTKRP (scalar fp64 payloads). The fiber index enters as the
// u32 offsets plus a per-tile "first fiber" map built by a streaming pass
// over fptr, so no tile ever binary-searches global memory. Output index
// tuples are written by the tile holding the fiber head (gathered from the
// head entry, P/src/kernels_seq.cpp:89-94).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace {

constexpr int kThreads = 256;
#ifndef SPT_TTV_EPT
#define SPT_TTV_EPT 8
#endif
#ifndef SPT_TTV_TICKET
#define SPT_TTV_TICKET 0
#endif
#ifndef SPT_TTV_MINB
#define SPT_TTV_MINB 4
#endif
constexpr int kEPT = SPT_TTV_EPT;
constexpr int kTile = kThreads * kEPT;
constexpr uint32_t kFlagA = 1, kFlagP = 2;

struct SegPair {
  int head;
  double v;
};
struct SegOp {
  __device__ __forceinline__ SegPair operator()(const SegPair& a, const SegPair& b) const {
    return {a.head | b.head, b.head ? b.v : a.v + b.v};
  }
};

struct TtvParams {
  const uint32_t* kidx;  // x.indices[mode]
  const float* val;
  const float* v;
  const uint32_t* fptr;
  const uint32_t* tile_fiber;
  const uint32_t* hidx[SPT_MAX_ORDER - 1];  // x.indices[d], d != mode ascending
  uint32_t* zidx[SPT_MAX_ORDER - 1];
  float* zval;
  uint64_t nnz;
  uint32_t nfibs;
  uint32_t ntiles;
  uint32_t epoch;
  uint32_t* status;
  double* payA;
  double* payP;
  unsigned long long* tile_ctr;
  int vec_ok;  // mode-index and value arrays 16-byte aligned (vector loads)
};

template <int NO>
__global__ void __launch_bounds__(kThreads, SPT_TTV_MINB) ttv_kernel(TtvParams p) {
  using Scan = cub::BlockScan<SegPair, kThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_fptr[kTile + 2];
  __shared__ uint32_t s_tile;
  __shared__ int s_meta[3];
  __shared__ double s_carry;

  const int tid = threadIdx.x;
  if (tid == 0) {
    const unsigned long long t = atomicAdd(p.tile_ctr, 1ull);
    if (t == p.ntiles - 1) atomicExch(p.tile_ctr, 0ull);
    s_tile = static_cast<uint32_t>(t);
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * kTile;
  const int cnt = (p.nnz - t0 < (uint64_t)kTile) ? static_cast<int>(p.nnz - t0) : kTile;
  const uint32_t f_lo = p.tile_fiber[tile];
  const uint32_t f_end = (tile + 1 < p.ntiles) ? p.tile_fiber[tile + 1] + 1 : p.nfibs;
  const uint32_t nstage = f_end - f_lo + 1;  // fptr[f_lo .. f_end]
  for (uint32_t i = tid; i < nstage; i += kThreads) s_fptr[i] = p.fptr[f_lo + i];

  // Terms (fp32, as the reference forms them), blocked: entries tid*8 .. +7.
  const int e0 = tid * kEPT;
  float val[kEPT];
  uint32_t kk[kEPT];
  // The other modes' indices are read up front (fiber heads take their output
  // tuple from here), so the emission needs no second dependent round trip.
  uint32_t oi[NO][kEPT];
  if (cnt == kTile && p.vec_ok) {
#pragma unroll
    for (int c = 0; c < kEPT / 4; ++c) {
#pragma unroll
      for (int d = 0; d < NO; ++d) {
        const uint4 a = spt::ld_stream(reinterpret_cast<const uint4*>(p.hidx[d] + t0 + e0) + c);
        oi[d][4 * c] = a.x, oi[d][4 * c + 1] = a.y, oi[d][4 * c + 2] = a.z, oi[d][4 * c + 3] = a.w;
      }
      const uint4 k0 = spt::ld_stream(reinterpret_cast<const uint4*>(p.kidx + t0 + e0) + c);
      const uint4 v0 = spt::ld_stream(reinterpret_cast<const uint4*>(p.val + t0 + e0) + c);
      kk[4 * c] = k0.x, kk[4 * c + 1] = k0.y, kk[4 * c + 2] = k0.z, kk[4 * c + 3] = k0.w;
      val[4 * c] = __uint_as_float(v0.x), val[4 * c + 1] = __uint_as_float(v0.y);
      val[4 * c + 2] = __uint_as_float(v0.z), val[4 * c + 3] = __uint_as_float(v0.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kEPT; ++i) {
      const bool ok = e0 + i < cnt;
      kk[i] = ok ? p.kidx[t0 + e0 + i] : 0;
      val[i] = ok ? p.val[t0 + e0 + i] : 0.0f;
#pragma unroll
      for (int d = 0; d < NO; ++d) oi[d][i] = ok ? p.hidx[d][t0 + e0 + i] : 0;
    }
  }
  float term[kEPT];
#pragma unroll
  for (int i = 0; i < kEPT; ++i) term[i] = (e0 + i < cnt) ? __fmul_rn(val[i], __ldg(p.v + kk[i])) : 0.0f;
  __syncthreads();

  // Local fiber of each item: binary search once, then walk.
  int lf[kEPT];
  bool head[kEPT];
  {
    const uint64_t m0 = t0 + e0;
    int lo = 0, hi = static_cast<int>(nstage) - 1;  // largest j with s_fptr[j] <= m0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_fptr[mid] <= m0) lo = mid;
      else hi = mid - 1;
    }
    int j = lo;
#pragma unroll
    for (int i = 0; i < kEPT; ++i) {
      const uint64_t m = m0 + i;
      while (j + 1 < static_cast<int>(nstage) && s_fptr[j + 1] <= m) ++j;
      lf[i] = j;
      head[i] = (e0 + i < cnt) && s_fptr[j] == m;
    }
  }
  SegPair agg{0, 0.0};
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    if (e0 + i >= cnt) break;
    if (head[i]) agg = {1, (double)term[i]};
    else agg.v += (double)term[i];
  }
  SegPair excl, block_agg;
  Scan(scan_tmp).ExclusiveScan(agg, excl, SegOp(), block_agg);
  if (tid == 0) excl = {0, 0.0};

  if (tid == 0) {
    const bool cont_prev = s_fptr[0] < t0;
    // fiber of the last entry
    const uint64_t ml = t0 + cnt - 1;
    int lo = 0, hi = static_cast<int>(nstage) - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_fptr[mid] <= ml) lo = mid;
      else hi = mid - 1;
    }
    s_meta[0] = cont_prev;
    s_meta[1] = s_fptr[lo + 1] > ml + 1;  // last fiber continues into the next tile
    s_meta[2] = lo;                        // local id of the last fiber
  }
  __syncthreads();
  const bool cont_prev = s_meta[0], cont_next = s_meta[1];
  const bool single = s_meta[2] == 0;
  const uint32_t tag = p.epoch << 3;

  // Publish the tail partial for successors (only when one needs it).
  if (cont_next && tid == 0) {
    if (!single || !cont_prev) {
      p.payP[tile] = block_agg.v;
      spt::st_release(p.status + tile, tag | kFlagP);
    } else {
      p.payA[tile] = block_agg.v;
      spt::st_release(p.status + tile, tag | kFlagA);
    }
  }
  // Look-back for the first fiber's carry-in: warp 0 finds the chain of A's
  // ending in a P (32 predecessors per poll) and sums its scalar payloads.
  // Only a tile that completes its first fiber walks back; tiles strictly
  // inside a long fiber publish their aggregate and never wait.
  if (tid < 32) {
    double carry = 0.0;
    if (cont_prev && !(single && cont_next)) {
      const uint32_t n = spt::lookback_chain(p.status, tile, p.epoch);
      for (uint32_t q = 1 + tid; q <= n && q <= tile; q += 32)
        carry += spt::ld_cg((q == n ? p.payP : p.payA) + (tile - q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) carry += __shfl_xor_sync(0xffffffffu, carry, o);
    }
    if (tid == 0) s_carry = carry;
  }
  __syncthreads();
  const double carry = s_carry;

  // Fibers ending here get their value, fibers starting here their index
  // tuple (gathered from the head entry), staged by local fiber id and then
  // written with coalesced stores (consecutive fibers -> consecutive slots).
  extern __shared__ uint32_t s_dyn[];
  float* s_zv = reinterpret_cast<float*>(s_dyn);  // [kTile + 2]
  uint32_t* s_zi = s_dyn + (kTile + 2);           // [NO][kTile + 2]
  double run = excl.v;
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    const int e = e0 + i;
    if (e >= cnt) break;
    const uint64_t m = t0 + e;
    run = head[i] ? (double)term[i] : run + (double)term[i];
    if (head[i]) {
#pragma unroll
      for (int d = 0; d < NO; ++d) s_zi[d * (kTile + 2) + lf[i]] = oi[d][i];
    }
    if (s_fptr[lf[i] + 1] == m + 1) s_zv[lf[i]] = (float)(run + (lf[i] == 0 ? carry : 0.0));
  }
  __syncthreads();
  const int last = s_meta[2];
  const int end_hi = cont_next ? last : last + 1;  // fibers [0, end_hi) end here
  const int head_lo = cont_prev ? 1 : 0;           // fibers [head_lo, last] start here
  for (int o = tid; o < end_hi; o += kThreads) spt::st_stream(
      reinterpret_cast<uint32_t*>(p.zval) + f_lo + o, __float_as_uint(s_zv[o]));
#pragma unroll
  for (int d = 0; d < NO; ++d)
    for (int o = head_lo + tid; o <= last; o += kThreads)
      spt::st_stream(p.zidx[d] + f_lo + o, s_zi[d * (kTile + 2) + o]);
}

// map[t] = fiber containing entry t*tile = the largest f < nfibs with
// fptr[f] <= t*tile (fptr is non-decreasing, fptr[0] = 0). G = 8 lanes per
// tile run a 9-ary search over fptr: ~8 dependent rounds for 5e7 fibers, all
// tiles in parallel -- instead of a streaming pass over every fiber.
constexpr int kMapG = 8;
__global__ void tile_fiber_kernel(const uint32_t* fptr, uint32_t nfibs, uint32_t tile,
                                  uint32_t ntiles, uint32_t* map) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) / kMapG;
  const unsigned lane = threadIdx.x & 31u, gl = lane % kMapG, g0 = lane - gl;
  const unsigned gmask = ((1u << kMapG) - 1u) << g0;
  const bool live = t < ntiles;
  const uint64_t target = (uint64_t)t * tile;
  uint32_t lo = 0, hi = live ? nfibs : 0;  // answer in [lo, hi): fptr[lo] <= target
  while (__any_sync(0xffffffffu, hi - lo > kMapG)) {
    const uint32_t span = hi - lo;
    const bool act = span > kMapG;
    const uint32_t m = lo + (uint32_t)(((uint64_t)span * (gl + 1)) / (kMapG + 1));
    const bool pred = act && fptr[m] <= target;
    const int ntrue = __popc((__ballot_sync(0xffffffffu, pred) & gmask) >> g0);
    const uint32_t m_last = __shfl_sync(0xffffffffu, m, g0 + (ntrue > 0 ? ntrue - 1 : 0));
    const uint32_t m_first_false =
        __shfl_sync(0xffffffffu, m, g0 + (ntrue < kMapG ? ntrue : kMapG - 1));
    if (act) {
      if (ntrue > 0) lo = m_last;
      if (ntrue < kMapG) hi = m_first_false;
    }
  }
  // final: the last m in [lo, hi) with fptr[m] <= target (fptr[lo] <= target holds)
  const uint32_t m = lo + gl;
  const bool pred = m < hi && fptr[m] <= target;
  const int ntrue = __popc((__ballot_sync(0xffffffffu, pred) & gmask) >> g0);
  if (gl == 0 && live) map[t] = lo + (ntrue > 0 ? ntrue - 1 : 0);
}

// ---------------------------------------------------------------------------
// Warp-tile TTV: every warp owns a tile of kWT = 128 or 256 consecutive entries (4 or 8
// per lane) and does everything itself -- head flags from its slice of fptr,
// fp32 terms, an fp64 segmented warp scan, staging of its fibers' outputs in
// its own shared-memory slice, coalesced stores -- so no warp ever waits at a
// CTA barrier. A fiber crossing a warp-tile boundary is completed by the tile
// holding its last entry through the same epoch-tagged decoupled look-back
// (scalar fp64 payloads); C3's short fibers rarely cross one. A CTA draws one
// ticket for its 8 consecutive warp tiles, so predecessors are resident.

// Per-tile phase timeline for tune/probe_ttv_trace.py (-DSPT_TTV_TRACE).
#ifdef SPT_TTV_TRACE
__device__ unsigned long long g_ttv_trace[65536 * 8];
__device__ __forceinline__ unsigned long long tgtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TV_TR(k) do { if (lane == 0 && wt < 65536) g_ttv_trace[wt * 8 + (k)] = tgtime(); } while (0)
#else
#define TV_TR(k) do {} while (0)
#endif

template <int NO, int kWT>
constexpr size_t ttv_wt_slice() {
  return (size_t)(kWT + 8) + (size_t)(kWT + 1) * 4 * (1 + NO);  // heads | zv | zi[NO]
}

// kWT entries per warp tile (128 or 256); 128-entry tiles hold half the
// registers (8 CTAs per SM instead of 4) and win when fibers are ~1 entry
// long (C3 mode 0: 202 vs 232 us at 20M), 256 wins once fibers are longer
// (fewer tiles split a fiber: mode 2 239 vs 249 us).
template <int NO, int kWT>
__global__ void __launch_bounds__(kThreads, kWT == 128 ? 8 : 4) ttv_wt_kernel(TtvParams p) {
  constexpr int kWE = kWT / 32;  // entries per lane (blocked)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#if SPT_TTV_TICKET
  __shared__ uint32_t s_ticket;
  if (tid == 0) {
    const unsigned long long t = atomicAdd(p.tile_ctr, 1ull);
    if (t == gridDim.x - 1) atomicExch(p.tile_ctr, 0ull);
    s_ticket = static_cast<uint32_t>(t);
  }
  __syncthreads();
  const uint32_t cta = s_ticket;
#else
  // tiles in launch order (as CUB's single-pass scans do): CTAs are dispatched
  // in blockIdx order, so a tile's predecessors are resident or done
  const uint32_t cta = blockIdx.x;
#endif
  const uint32_t wt = cta * (kThreads / 32) + warp;
  if (wt >= p.ntiles) return;
  unsigned char* base = smem_raw + warp * ((ttv_wt_slice<NO, kWT>() + 15) & ~size_t(15));
  uint8_t* s_head = base;                                             // [kWT + 8]
  float* s_zv = reinterpret_cast<float*>(base + kWT + 8);             // [kWT + 1]
  uint32_t* s_zi = reinterpret_cast<uint32_t*>(s_zv + (kWT + 1));      // [NO][kWT + 1]
  const uint64_t t0 = (uint64_t)wt * kWT;
  const int cnt = (p.nnz - t0 < (uint64_t)kWT) ? static_cast<int>(p.nnz - t0) : kWT;
  const uint32_t f_lo = __ldg(p.tile_fiber + wt);  // fiber containing entry t0
  TV_TR(0);

  // ---- entries (issued first: the longest round trip)
  const int e0 = lane * kWE;
  uint32_t kk[kWE], oi[NO][kWE];
  float val[kWE];
  if (cnt == kWT && p.vec_ok) {
#pragma unroll
    for (int c = 0; c < kWE / 4; ++c) {
      const uint4 k4 = spt::ld_stream(reinterpret_cast<const uint4*>(p.kidx + t0 + e0) + c);
      const uint4 v4 = spt::ld_stream(reinterpret_cast<const uint4*>(p.val + t0 + e0) + c);
      kk[4 * c] = k4.x, kk[4 * c + 1] = k4.y, kk[4 * c + 2] = k4.z, kk[4 * c + 3] = k4.w;
      val[4 * c] = __uint_as_float(v4.x), val[4 * c + 1] = __uint_as_float(v4.y);
      val[4 * c + 2] = __uint_as_float(v4.z), val[4 * c + 3] = __uint_as_float(v4.w);
#pragma unroll
      for (int d = 0; d < NO; ++d) {
        const uint4 a = spt::ld_stream(reinterpret_cast<const uint4*>(p.hidx[d] + t0 + e0) + c);
        oi[d][4 * c] = a.x, oi[d][4 * c + 1] = a.y, oi[d][4 * c + 2] = a.z, oi[d][4 * c + 3] = a.w;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kWE; ++i) {
      const bool ok = e0 + i < cnt;
      kk[i] = ok ? p.kidx[t0 + e0 + i] : 0u;
      val[i] = ok ? p.val[t0 + e0 + i] : 0.0f;
#pragma unroll
      for (int d = 0; d < NO; ++d) oi[d][i] = ok ? p.hidx[d][t0 + e0 + i] : 0u;
    }
  }

  TV_TR(1);
  // ---- head flags. x is coalesced and sorted with `mode` last, so a fiber
  // starts exactly where a non-mode index changes (build_fiber_index,
  // P/src/tensor.cpp:92-120): compare each entry's tuple with its
  // predecessor's (previous lane by shuffle, entry t0-1 / t_end loaded by
  // lanes 0 / 31) -- no fptr reads on the tile's critical path.
  const uint64_t t_end = t0 + cnt;
  uint32_t prv[NO], nxt[NO];
#pragma unroll
  for (int d = 0; d < NO; ++d) {
    prv[d] = (lane == 0 && t0 > 0) ? p.hidx[d][t0 - 1] : 0u;
    nxt[d] = (lane == 31 && t_end < p.nnz) ? p.hidx[d][t_end] : 0u;
  }
  bool hd[kWE];
  {
    bool diff0 = (lane == 0 && t0 == 0);
#pragma unroll
    for (int d = 0; d < NO; ++d) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, oi[d][kWE - 1], 1);
      const uint32_t before = lane == 0 ? prv[d] : up;
      diff0 = diff0 || oi[d][0] != before;
    }
    hd[0] = diff0;
#pragma unroll
    for (int i = 1; i < kWE; ++i) {
      bool df = false;
#pragma unroll
      for (int d = 0; d < NO; ++d) df = df || oi[d][i] != oi[d][i - 1];
      hd[i] = df;
    }
  }
  // does the tile's last fiber go on past t_end?
  bool cont_nx_l = false;
  if (lane == 31 && t_end < p.nnz) {
    // entry t_end - 1 is lane 31's last valid entry only for full tiles; the
    // partial tile is the last one (t_end == nnz), so this branch sees a full tile
    cont_nx_l = true;
#pragma unroll
    for (int d = 0; d < NO; ++d) cont_nx_l = cont_nx_l && nxt[d] == oi[d][kWE - 1];
  }
  const bool cont_nx = __shfl_sync(0xffffffffu, cont_nx_l ? 1 : 0, 31) != 0;
#pragma unroll
  for (int i = 0; i < kWE; ++i) s_head[e0 + i] = (e0 + i < cnt && hd[i]) ? 1 : 0;
  __syncwarp();

  TV_TR(2);
  // ---- terms, segmented warp scan (fp64), local fiber ids
  float term[kWE];
  bool head[kWE];
#pragma unroll
  for (int i = 0; i < kWE; ++i) {
    const bool ok = e0 + i < cnt;
    term[i] = ok ? __fmul_rn(val[i], __ldg(p.v + kk[i])) : 0.0f;
    head[i] = ok && s_head[e0 + i];
  }
  int nh = 0;  // heads in this lane
  bool any = false;
  double lsum = 0.0;  // sum since this lane's last head (or lane start)
#pragma unroll
  for (int i = 0; i < kWE; ++i) {
    nh += head[i] ? 1 : 0;
    if (head[i]) {
      any = true;
      lsum = (double)term[i];
    } else {
      lsum += (double)term[i];
    }
  }
  // exclusive scan of (any-head, sum) and of the head counts
  int hx = nh;
  bool fx = any;
  double sx = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int hv = __shfl_up_sync(0xffffffffu, hx, o);
    const bool fv = __shfl_up_sync(0xffffffffu, fx ? 1 : 0, o) != 0;
    const double sv = __shfl_up_sync(0xffffffffu, sx, o);
    if (lane >= o) {
      hx += hv;
      if (!fx) sx += sv;  // combine(prev, mine): mine has no head -> prev + mine
      fx = fx || fv;
    }
  }
  // exclusive values for this lane = inclusive of lane - 1
  int h_before = __shfl_up_sync(0xffffffffu, hx, 1);
  double s_before = __shfl_up_sync(0xffffffffu, sx, 1);
  if (lane == 0) {
    h_before = 0;
    s_before = 0.0;
  }
  const bool head0 = __shfl_sync(0xffffffffu, head[0] ? 1 : 0, 0) != 0;  // entry t0 starts a fiber
  const bool cont_prev = !head0;
  const int hc0 = head0 ? 1 : 0;
  const int total_h = __shfl_sync(0xffffffffu, hx, 31);
  const int last_lf = total_h - hc0;  // local id of the tile's last fiber
  const bool single = last_lf == 0;
  const double tile_tail = __shfl_sync(0xffffffffu, sx, 31);  // sum of the last fiber in this tile

  TV_TR(3);
  // ---- publish the tail partial, then look back for the first fiber's carry
  const uint32_t tag = p.epoch << 3;
  if (cont_nx && lane == 0) {
    if (!single || !cont_prev) {
      p.payP[wt] = tile_tail;
      spt::st_release(p.status + wt, tag | kFlagP);
    } else {
      p.payA[wt] = tile_tail;
      spt::st_release(p.status + wt, tag | kFlagA);
    }
  }
  double carry = 0.0;
  if (cont_prev && !(single && cont_nx)) {
    const uint32_t n = spt::lookback_chain(p.status, wt, p.epoch);
    for (uint32_t q = 1 + lane; q <= n && q <= wt; q += 32)
      carry += spt::ld_cg((q == n ? p.payP : p.payA) + (wt - q));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) carry += __shfl_xor_sync(0xffffffffu, carry, o);
  }

  TV_TR(4);
  // ---- stage outputs by local fiber id, then coalesced stores
  int hcount = h_before;
  double run = s_before;
#pragma unroll
  for (int i = 0; i < kWE; ++i) {
    const int e = e0 + i;
    if (e >= cnt) break;
    hcount += head[i] ? 1 : 0;
    run = head[i] ? (double)term[i] : run + (double)term[i];
    const int lf = hcount - hc0;
    if (head[i]) {
#pragma unroll
      for (int d = 0; d < NO; ++d) s_zi[d * (kWT + 1) + lf] = oi[d][i];
    }
    const bool ends = (e + 1 < cnt) ? s_head[e + 1] != 0 : !cont_nx;
    if (ends) s_zv[lf] = (float)(run + (lf == 0 ? carry : 0.0));
  }
  __syncwarp();
  const int end_hi = cont_nx ? last_lf : last_lf + 1;  // fibers [0, end_hi) end here
  const int head_lo = cont_prev ? 1 : 0;            // fibers [head_lo, last_lf] start here
  for (int o = lane; o < end_hi; o += 32)
    spt::st_stream(reinterpret_cast<uint32_t*>(p.zval) + f_lo + o, __float_as_uint(s_zv[o]));
#pragma unroll
  for (int d = 0; d < NO; ++d)
    for (int o = head_lo + lane; o <= last_lf; o += 32)
      spt::st_stream(p.zidx[d] + f_lo + o, s_zi[d * (kWT + 1) + o]);
  TV_TR(5);
}

template <int NO, int kWT>
int launch_ttv_wt(spt_ctx* ctx, const TtvParams& p, cudaStream_t st) {
  const size_t smem = (size_t)(kThreads / 32) * ((ttv_wt_slice<NO, kWT>() + 15) & ~size_t(15));
  SPT_CUDA(cudaFuncSetAttribute(ttv_wt_kernel<NO, kWT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  const unsigned grid = static_cast<unsigned>((p.ntiles + kThreads / 32 - 1) / (kThreads / 32));
  ttv_wt_kernel<NO, kWT><<<grid, kThreads, smem, st>>>(p);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

template <int NO>
int launch_ttv_wt_any(spt_ctx* ctx, const TtvParams& p, cudaStream_t st, uint32_t wt_entries) {
  return wt_entries == 128 ? launch_ttv_wt<NO, 128>(ctx, p, st) : launch_ttv_wt<NO, 256>(ctx, p, st);
}

template <int NO>
int launch_ttv(spt_ctx* ctx, const TtvParams& p, unsigned grid, cudaStream_t st) {
  const size_t smem = (size_t)(NO + 1) * (kTile + 2) * sizeof(uint32_t);
  SPT_CUDA(cudaFuncSetAttribute(ttv_kernel<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  ttv_kernel<NO><<<grid, kThreads, smem, st>>>(p);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

}  // namespace

namespace spt {

int build_tile_fiber_map(spt_ctx* ctx, const uint32_t* d_fptr, uint32_t nfibs, uint32_t tile,
                         uint32_t ntiles, uint32_t* d_map, cudaStream_t st) {
  const uint64_t threads = (uint64_t)ntiles * kMapG;
  tile_fiber_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      d_fptr, nfibs, tile, ntiles, d_map);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

int check_fiber_inputs(const spt_coo* x, uint32_t mode, const uint32_t* d_fptr, uint64_t nfibs,
                       const char* k) {
  SPT_TRY(check_coo(x, k));
  // P/src/kernel_detail.hpp:110-118
  if (x->order < 2) return set_error(SPT_EINVAL, "%s: input must have order >= 2", k);
  if (mode >= x->order) return set_error(SPT_EINVAL, "%s: mode out of range", k);
  if (!x->coalesced) return set_error(SPT_EINVAL, "%s: tensor must be coalesced", k);
  if (!x->has_sort_order || static_cast<uint32_t>(x->sort_order[x->order - 1]) != mode)
    return set_error(SPT_EINVAL, "%s: tensor must be sorted with the target mode last", k);
  if (!d_fptr || nfibs > x->nnz || (x->nnz > 0 && nfibs == 0))
    return set_error(SPT_EINVAL, "%s: fiber index does not match the tensor", k);
  return SPT_OK;
}

}  // namespace spt

extern "C" int spt_ttv_f32(spt_ctx* ctx, const spt_coo* x, const float* d_v, uint64_t v_len,
                           uint32_t mode, const uint32_t* d_fptr, uint64_t nfibs, spt_coo* z,
                           unsigned flags, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "ttv: null context");
  SPT_TRY(spt::check_fiber_inputs(x, mode, d_fptr, nfibs, "ttv"));
  if (v_len != x->dims[mode])
    return spt::set_error(SPT_EINVAL, "ttv: vector length must match the mode dimension");
  if (!z) return spt::set_error(SPT_EINVAL, "ttv: null output");
  const uint32_t N = x->order;
  // Output metadata: dims without `mode`, sort order drop_mode(...), coalesced.
  z->order = N - 1;
  z->nnz = nfibs;
  uint32_t dz = 0;
  for (uint32_t d = 0; d < N; ++d)
    if (d != mode) z->dims[dz++] = x->dims[d];
  for (uint32_t d = dz; d < SPT_MAX_ORDER; ++d) z->dims[d] = 0;
  uint32_t k = 0;
  for (uint32_t j = 0; j < N; ++j) {
    const uint32_t d = x->sort_order[j];
    if (d != mode) z->sort_order[k++] = d < mode ? d : d - 1;
  }
  z->has_sort_order = 1;
  z->coalesced = 1;
  if (nfibs == 0) return SPT_OK;
  for (uint32_t d = 0; d < N - 1; ++d)
    if (!z->idx[d]) return spt::set_error(SPT_EINVAL, "ttv: null output index array");
  if (!z->val || !d_v) return spt::set_error(SPT_EINVAL, "ttv: null vector or output values");

  cudaStream_t st = spt::as_stream(stream);
#ifndef SPT_TTV_WARP_TILES
#define SPT_TTV_WARP_TILES 1
#endif
  // warp tiles of 128 entries for ~1-entry fibers, 256 otherwise
  const uint32_t wt_entries = x->nnz <= nfibs + nfibs / 2 ? 128u : 256u;
  const uint32_t tile_entries = SPT_TTV_WARP_TILES ? wt_entries : kTile;
  const uint64_t ntiles = (x->nnz + tile_entries - 1) / tile_entries;
  uint32_t* map;
  SPT_TRY(spt::ctx_scratch(ctx, ntiles * sizeof(uint32_t), reinterpret_cast<void**>(&map)));
  SPT_TRY(spt::build_tile_fiber_map(ctx, d_fptr, static_cast<uint32_t>(nfibs), tile_entries,
                                    static_cast<uint32_t>(ntiles), map, st));
  uint32_t epoch;
  SPT_TRY(spt::ctx_lookback(ctx, ntiles, 2 * ntiles, &epoch));
  TtvParams p{};
  p.kidx = x->idx[mode];
  p.val = x->val;
  p.v = d_v;
  p.fptr = d_fptr;
  p.tile_fiber = map;
  uint32_t j = 0;
  for (uint32_t d = 0; d < N; ++d) {
    if (d == mode) continue;
    p.hidx[j] = x->idx[d];
    p.zidx[j] = z->idx[j];
    ++j;
  }
  p.zval = z->val;
  p.nnz = x->nnz;
  p.nfibs = static_cast<uint32_t>(nfibs);
  p.ntiles = static_cast<uint32_t>(ntiles);
  p.epoch = epoch;
  p.status = ctx->d_status;
  p.payA = ctx->d_payload;
  p.payP = ctx->d_payload + ntiles;
  p.tile_ctr = ctx->d_tile_ctr;
  p.vec_ok = 1;
  for (uint32_t d = 0; d < N; ++d) p.vec_ok = p.vec_ok && spt::aligned16(x->idx[d]);
  p.vec_ok = p.vec_ok && spt::aligned16(x->val);
  if (SPT_TTV_WARP_TILES) {
    switch (N - 1) {
      case 1: SPT_TRY(launch_ttv_wt_any<1>(ctx, p, st, wt_entries)); break;
      case 2: SPT_TRY(launch_ttv_wt_any<2>(ctx, p, st, wt_entries)); break;
      case 3: SPT_TRY(launch_ttv_wt_any<3>(ctx, p, st, wt_entries)); break;
      case 4: SPT_TRY(launch_ttv_wt_any<4>(ctx, p, st, wt_entries)); break;
      case 5: SPT_TRY(launch_ttv_wt_any<5>(ctx, p, st, wt_entries)); break;
      case 6: SPT_TRY(launch_ttv_wt_any<6>(ctx, p, st, wt_entries)); break;
      default: SPT_TRY(launch_ttv_wt_any<7>(ctx, p, st, wt_entries)); break;
    }
    (void)flags;
    return SPT_OK;
  }
  const unsigned grid = static_cast<unsigned>(ntiles);
  switch (N - 1) {
    case 1: SPT_TRY(launch_ttv<1>(ctx, p, grid, st)); break;
    case 2: SPT_TRY(launch_ttv<2>(ctx, p, grid, st)); break;
    case 3: SPT_TRY(launch_ttv<3>(ctx, p, grid, st)); break;
    case 4: SPT_TRY(launch_ttv<4>(ctx, p, grid, st)); break;
    case 5: SPT_TRY(launch_ttv<5>(ctx, p, grid, st)); break;
    case 6: SPT_TRY(launch_ttv<6>(ctx, p, grid, st)); break;
    default: SPT_TRY(launch_ttv<7>(ctx, p, grid, st)); break;
  }
  (void)flags;
  return SPT_OK;
}

#ifdef SPT_TTV_TRACE
extern "C" __attribute__((visibility("default"))) int spt_debug_ttv_trace(void* dst) {
  return cudaMemcpyFromSymbol(dst, g_ttv_trace, sizeof(g_ttv_trace)) == cudaSuccess ? 0 : 5;
}
#endif
