// K3 TEW: general elementwise op of two coalesced tensors by sorted merge.
//
// Reference: seq::tew P/src/kernels_seq.cpp:41-53, merge_range
// P/src/kernel_detail.hpp:47-84 (matched -> op(x, y); unmatched x -> x for
// add/sub; unmatched y -> y (add) or -y (sub); mul keeps matches only),
// tew_output_dims :97-102, par::tew P/src/kernels_par.cpp:144-177.
//
// Two launches, no host round trip:
//   * a partition kernel places every 2048-item tile boundary on the merge
//     path of x and y ((G+1)-ary search on the diagonal; ties take x first,
//     so a matched pair is always "x then y" and each tuple is emitted once);
//   * when the N index widths fit 64 bits (the usual case) a persistent,
//     warp-specialised kernel (merge64p_kernel, below) streams the tiles:
//     bulk-async staging, u64-key merge of 8 items per thread, block scan,
//     decoupled look-back over 64-bit epoch-tagged tile counts, coalesced
//     emission (tuple + value, one IEEE op, bit-identical to the reference);
//   * otherwise merge_kernel does the same per CTA with N-word compares.
// The merge order equals the reference's two-pointer merge order, so the
// output is entry-for-entry identical to seq::tew's.
#include <cub/cub.cuh>

#include <algorithm>

#include "internal.cuh"

namespace {

constexpr int kThreads = 256;
#ifndef SPT_MERGE_IPT
#define SPT_MERGE_IPT 8
#endif
constexpr int kIPT = SPT_MERGE_IPT;
constexpr int kTile = kThreads * kIPT;
// Key arrays in shared memory get one pad word per 32 entries: the threads'
// merge-path positions advance ~4 entries apart, which would otherwise fold
// onto 8 banks.
constexpr int kTP = kTile + kTile / 32;
__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }
constexpr unsigned long long kFlagA = 1, kFlagP = 2;

struct MergeParams {
  const uint32_t* xi[SPT_MAX_ORDER];  // in sort order (k-th = mode ord[k])
  const uint32_t* yi[SPT_MAX_ORDER];
  uint32_t* zi[SPT_MAX_ORDER];        // in sort order
  const float* xv;
  const float* yv;
  float* zv;
  uint64_t nx, ny;
  const uint32_t* split;  // [ntiles+1] x-count at each tile diagonal
  uint32_t ntiles;
  uint32_t epoch;
  int op;
  unsigned long long* status;
  unsigned long long* tile_ctr;
  unsigned long long* total;  // device: output count
  // Packed-key path: position k of the sort order occupies bits
  // [shift[k], shift[k] + width) of a u64 key (sort-order significance).
  uint32_t shift[SPT_MAX_ORDER];
  uint32_t mask[SPT_MAX_ORDER];
};

template <int N>
__device__ __forceinline__ unsigned long long pack_g(const uint32_t* const* idx, const MergeParams& p,
                                                     uint64_t m) {
  unsigned long long k = 0;
#pragma unroll
  for (int q = 0; q < N; ++q) k |= (unsigned long long)idx[q][m] << p.shift[q];
  return k;
}

template <int N>
__device__ __forceinline__ int cmp_g(const MergeParams& p, uint64_t i, uint64_t j) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t a = p.xi[k][i], b = p.yi[k][j];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

// Tile boundaries on the merge path (x-first on ties): split[t] = number of x
// items among the first t*kTile merged items = the first m in [lo, hi) where
// x[m] <= y[diag-1-m] fails. G lanes per diagonal run a (G+1)-ary search.
// Each probe is a random sector pair, so the total sector traffic (rounds x
// G) -- not the round count -- bounds this kernel; G = 8 balances traffic
// against the number of dependent round trips (measured: 17.6 us vs 21.9 us
// for G = 32 at 10M + 10M).
#ifndef SPT_PART_G
#define SPT_PART_G 8
#endif
template <int N, int G>
__global__ void partition_g_kernel(MergeParams p, uint32_t* split) {
  // the merge kernel's CTAs may become resident now (they wait for this grid)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t gid = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const unsigned lane = threadIdx.x & 31u, gl = lane % G;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane - gl);
  const uint32_t t = gid;
  const bool live = t <= p.ntiles;
  const uint64_t total = p.nx + p.ny;
  const uint64_t diag = live ? std::min<uint64_t>((uint64_t)t * kTile, total) : 0;
  uint64_t lo = diag > p.ny ? diag - p.ny : 0;
  uint64_t hi = std::min<uint64_t>(diag, p.nx);
  while (__any_sync(0xffffffffu, hi - lo > G)) {
    const uint64_t span = hi - lo;
    const bool act = span > G;
    const uint64_t m = lo + (span * (gl + 1)) / (G + 1);
    const bool pred = act && cmp_g<N>(p, m, diag - 1 - m) <= 0;
    const unsigned bal = (__ballot_sync(0xffffffffu, pred) & gmask) >> (lane - gl);
    const int ntrue = __popc(bal);
    const uint64_t m_last = __shfl_sync(0xffffffffu, m, (lane - gl) + (ntrue > 0 ? ntrue - 1 : 0));
    const uint64_t m_first_false =
        __shfl_sync(0xffffffffu, m, (lane - gl) + (ntrue < G ? ntrue : G - 1));
    if (act) {
      if (ntrue > 0) lo = m_last + 1;
      if (ntrue < G) hi = m_first_false;
    }
  }
  const uint64_t m = lo + gl;
  const bool pred = m < hi && cmp_g<N>(p, m, diag - 1 - m) <= 0;
  const int ntrue = __popc((__ballot_sync(0xffffffffu, pred) & gmask));
  if (gl == 0 && live) split[t] = static_cast<uint32_t>(lo + ntrue);
}

template <int N>
__device__ __forceinline__ int cmp_s(const uint32_t* sx, int i, const uint32_t* sy, int j) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t a = sx[k * kTP + pad(i)], b = sy[k * kTP + pad(j)];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

__device__ __forceinline__ float apply(int op, float a, float b) {
  return op == SPT_ADD ? a + b : (op == SPT_SUB ? a - b : a * b);
}

template <int N>
__global__ void __launch_bounds__(kThreads) merge_kernel(MergeParams p) {
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sx = smem;              // [N][kTP] keys (padded)
  uint32_t* sy = smem + N * kTP;    // [N][kTP]
  float* sxv = reinterpret_cast<float*>(sy + N * kTP);  // [kTP] values
  float* syv = sxv + kTP;                               // [kTP]
  uint32_t* s_obuf = reinterpret_cast<uint32_t*>(syv + kTP);  // [kTile] output staging
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_base;

  const int tid = threadIdx.x;
  if (tid == 0) {
    const unsigned long long t = atomicAdd(p.tile_ctr, 1ull);
    if (t == p.ntiles - 1) atomicExch(p.tile_ctr, 0ull);
    s_tile = static_cast<uint32_t>(t);
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t total = p.nx + p.ny;
  const uint64_t d0 = (uint64_t)tile * kTile;
  const uint64_t d1 = std::min<uint64_t>(d0 + kTile, total);
  const uint64_t a0 = p.split[tile], a1 = p.split[tile + 1];
  const uint64_t b0 = d0 - a0, b1 = d1 - a1;
  const int nxt = static_cast<int>(a1 - a0), nyt = static_cast<int>(b1 - b0);
  for (int i = tid; i < nxt; i += kThreads) {
#pragma unroll
    for (int k = 0; k < N; ++k) sx[k * kTP + pad(i)] = spt::ld_stream(p.xi[k] + a0 + i);
    sxv[pad(i)] = __ldcs(p.xv + a0 + i);
  }
  for (int j = tid; j < nyt; j += kThreads) {
#pragma unroll
    for (int k = 0; k < N; ++k) sy[k * kTP + pad(j)] = spt::ld_stream(p.yi[k] + b0 + j);
    syv[pad(j)] = __ldcs(p.yv + b0 + j);
  }
  __syncthreads();

  // Thread-local merge path split.
  const int len = nxt + nyt;
  const int dg = std::min(tid * kIPT, len);
  int lo = std::max(0, dg - nyt), hi = std::min(dg, nxt);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cmp_s<N>(sx, mid, sy, dg - 1 - mid) <= 0) lo = mid + 1;
    else hi = mid;
  }
  int i = lo, j = dg - lo;
  // Serial merge of up to 8 items: record (source, local index, matched).
  uint8_t src[kIPT];  // 0 none, 1 x, 2 y
  uint8_t matched[kIPT];
  int li[kIPT];
  uint32_t cnt = 0;
#pragma unroll
  for (int k = 0; k < kIPT; ++k) {
    src[k] = 0;
    matched[k] = 0;
    li[k] = 0;
    if (dg + k >= len) continue;
    const bool take_x = j >= nyt || (i < nxt && cmp_s<N>(sx, i, sy, j) <= 0);
    if (take_x) {
      // matched iff the next y (global b0+j) equals x[i]
      bool m = false;
      if (j < nyt) m = cmp_s<N>(sx, i, sy, j) == 0;
      else if (b0 + j < p.ny) m = cmp_g<N>(p, a0 + i, b0 + j) == 0;
      src[k] = 1;
      matched[k] = m;
      li[k] = i;
      ++i;
      cnt += (p.op == SPT_MUL) ? (m ? 1u : 0u) : 1u;
    } else {
      // matched iff the previous x (global a0+i-1) equals y[j]
      bool m = false;
      if (i > 0) m = cmp_s<N>(sx, i - 1, sy, j) == 0;
      else if (a0 > 0) m = cmp_g<N>(p, a0 - 1, b0 + j) == 0;
      src[k] = 2;
      matched[k] = m;
      li[k] = j;
      ++j;
      cnt += (p.op != SPT_MUL && !m) ? 1u : 0u;
    }
  }
  uint32_t excl, tile_total;
  Scan(scan_tmp).ExclusiveSum(cnt, excl, tile_total);

  // Decoupled look-back over tile counts (word = epoch<<34 | flag<<32 | count),
  // warp-parallel: 32 predecessors per poll.
  // Decoupled look-back over the tile counts. The count travels inside the
  // status word itself, so publication is a relaxed store (no MEMBAR) and
  // polling is relaxed (no L1 invalidation).
  if (tid < 32) {
    const unsigned long long tag = (unsigned long long)p.epoch << 34;
    unsigned long long base = 0;
    if (tile == 0) {
      if (tid == 0) spt::st_relaxed64(p.status + tile, tag | (kFlagP << 32) | tile_total);
    } else {
      if (tid == 0) spt::st_relaxed64(p.status + tile, tag | (kFlagA << 32) | tile_total);
      base = spt::lookback_count64(p.status, tile, p.epoch);
      if (tid == 0)
        spt::st_relaxed64(p.status + tile, tag | (kFlagP << 32) | (base + tile_total));
    }
    if (tid == 0) {
      s_base = base;
      if (tile == p.ntiles - 1) *p.total = base + tile_total;
    }
  }
  __syncthreads();

  // Emission: every emitted item gets a tile-local slot; each of the N index
  // arrays and the value array is assembled in shared memory and written out
  // with fully coalesced stores (the thread-strided direct scatter would cost
  // one 32-byte sector transaction per 4-byte element).
  int lslot[kIPT];
  uint32_t vbits[kIPT];
  {
    int lp = static_cast<int>(excl);
#pragma unroll
    for (int k = 0; k < kIPT; ++k) {
      lslot[k] = -1;
      vbits[k] = 0;
      if (src[k] == 0) continue;
      const bool m = matched[k];
      if (src[k] == 1) {
        if (p.op == SPT_MUL && !m) continue;
        float v = sxv[pad(li[k])];
        if (m) {
          // the matching y is the next y in merge order: local index = number of
          // y items before this x item = (dg + k) - li[k]; it may sit just past
          // this tile's y run.
          const int yl = dg + k - li[k];
          v = apply(p.op, v, yl < nyt ? syv[pad(yl)] : __ldg(p.yv + b0 + yl));
        }
        vbits[k] = __float_as_uint(v);
      } else {
        if (p.op == SPT_MUL || m) continue;
        const float yv = syv[pad(li[k])];
        vbits[k] = __float_as_uint(p.op == SPT_SUB ? -yv : yv);
      }
      lslot[k] = lp++;
    }
  }
  const uint64_t base = s_base;
#pragma unroll 1
  for (int q = 0; q <= N; ++q) {
#pragma unroll
    for (int k = 0; k < kIPT; ++k) {
      if (lslot[k] < 0) continue;
      uint32_t w;
      if (q == N) w = vbits[k];
      else w = (src[k] == 1 ? sx : sy)[q * kTP + pad(li[k])];
      s_obuf[lslot[k]] = w;
    }
    __syncthreads();
    uint32_t* dst = q == N ? reinterpret_cast<uint32_t*>(p.zv) : p.zi[q];
    for (uint32_t o = tid; o < tile_total; o += kThreads) spt::st_stream(dst + base + o, s_obuf[o]);
    __syncthreads();
  }
}

// Packed-key variant (sum of per-mode index widths <= 64 bits, e.g. C2's
// 3 x 14 bits): every comparison is one u64 compare on a key staged once per
// entry; indices are unpacked from the key on emission. u64 smem arrays get
// one pad element per 16 so the ~4-apart merge positions of a half-warp hit
// distinct banks.
// Packed keys: one pad slot per 32 (measured best of 8/16/32/64/XOR for the
// data-dependent merge-path positions).
constexpr int kPad64Shift = 5;
__device__ __forceinline__ int pad64(int i) { return i + (i >> kPad64Shift); }

// ---------------------------------------------------------------------------
// Persistent, pipelined, warp-specialised merge (packed u64 keys).
//
// A CTA (resident for the whole merge) = 8 merge warps + 1 emitter warp + 1
// producer warp:
//   * producer: takes tile tickets in order, reads the tile's merge-path split
//     and moves the tile's x and y runs (N index arrays + values per side)
//     into a shared-memory stage with bulk async copies (the TMA engine;
//     16-byte-aligned body per run, <= 3 scalar head/tail words by lanes);
//   * merge warps: pack u64 keys from the stage and free it (the producer
//     refills it with the next tile at once), merge 8 items per thread, block
//     scan, publish the tile's count (A), and leave the emitted (key, value)
//     pairs in an emission buffer -- they never wait for other tiles;
//   * emitter: decoupled look-back for that tile (wide window), publishes its
//     inclusive count (P), writes the tile's output with coalesced streaming
//     stores, frees the emission buffer.
// So load latency hides behind the previous tile's merge, and look-back
// latency behind the next tile's merge.
#ifndef SPT_MERGE_STAGES
#define SPT_MERGE_STAGES 1
#endif
constexpr int kStages = SPT_MERGE_STAGES;
#ifndef SPT_STATUS_SHIFT
#define SPT_STATUS_SHIFT 2
#endif
constexpr int kSS = SPT_STATUS_SHIFT;  // status word of tile t at t << kSS
constexpr int kSeg = kTile + 16;  // words per staged array (x run + y run + alignment slack)
constexpr uint32_t kDone = 0xFFFFFFFFu;
constexpr int kLB = 2;                      // look-back warps (alternate tiles)
constexpr int kPThreads = kThreads + 32 * (kLB + 2);  // + look-back x2, emitter, producer
constexpr int kSlots = 4;                   // tile hand-off ring (merge -> look-back -> emitter)
// Emission buffers: threads write their emitted items ~8 apart, so pad one
// slot per 16 (u64 keys) / per 8 (u32 values) to spread those rows over all
// banks; the emitter reads them back consecutively.
constexpr int kEK = kTile + kTile / 16;
constexpr int kEV = kTile + kTile / 8;
__device__ __forceinline__ int epad64(int o) { return o + (o >> 4); }
__device__ __forceinline__ int epad(int o) { return o + (o >> 3); }

struct StageInfo {
  uint32_t tile, nxt, nyt, _pad;
  uint32_t xoff[SPT_MAX_ORDER + 1], yoff[SPT_MAX_ORDER + 1];
  unsigned long long x_before, y_after;
  unsigned long long a0, b0;  // the tile's first x / y entry
  uint32_t yv_after, _pad2;  // value of the first y after the tile (matches across the edge)
};

// Packed tile in shared memory: x keys at key slots [0, nxt), a sentinel slot
// at nxt, y keys at [nxt+1, nxt+1+nyt), a sentinel slot after them whose value
// is the first y after the tile. Clamped head reads land on the sentinels, so
// the merge loop has no bounds branches.
constexpr int kSK = (kTile + 2 + ((kTile + 2) >> kPad64Shift) + 4) & ~3;  // >= pad64(kTile+1)+1
constexpr int kSV = (kTile + 2 + (kTile + 2) / 32 + 8) & ~3;  // >= pad(kTile + 2) + 1, 16B multiple
// smem: stages [kStages][(N+1) * kSeg] u32 | sk [kSK] u64 | ek [2][kEK] u64 |
//       sv [kSV] u32 | ev [2][kEV] u32 | info [kStages] | barriers | scalars
template <int N>
constexpr size_t pers_smem() {
  return (size_t)kStages * (N + 1) * kSeg * 4 + (size_t)kSK * 8 + (size_t)2 * kEK * 8 +
         (size_t)kSV * 4 + (size_t)2 * kEV * 4 + kStages * sizeof(StageInfo) +
         (2 * kStages + 4 + 3 * kSlots) * 8 + kSlots * 16 + 16 * 8;
}

// One run [e0, e0+n) of array `src` into stage words starting at `dst`, where
// dst and src+e0 share their 16-byte phase: scalar head/tail, bulk body.
__device__ __forceinline__ void copy_run(uint32_t* dst, const uint32_t* src, uint64_t e0,
                                         uint32_t n, uint32_t head, uint32_t body,
                                         unsigned long long* bar) {
  if (body) spt::bulk_g2s(dst + head, src + e0 + head, body * 4, bar);
  // <= 3 head and <= 3 tail words: all six loads in flight, then the stores
  const uint32_t tail = n - head - body;
  uint32_t hv[3], tv[3];
#pragma unroll
  for (uint32_t k = 0; k < 3; ++k) {
    if (k < head) hv[k] = __ldg(src + e0 + k);
    if (k < tail) tv[k] = __ldg(src + e0 + head + body + k);
  }
#pragma unroll
  for (uint32_t k = 0; k < 3; ++k) {
    if (k < head) dst[k] = hv[k];
    if (k < tail) dst[head + body + k] = tv[k];
  }
}

__device__ __forceinline__ uint32_t word_phase(const uint32_t* p) {
  return (static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p)) >> 2) & 3u;
}

// Per-tile phase timeline for tune/probe_merge_trace.py (-DSPT_MERGE_TRACE).
#ifdef SPT_MERGE_TRACE
__device__ unsigned long long g_mtrace[16384 * 8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MT_TR(tile, k) do { if ((tile) < 16384) g_mtrace[(tile) * 8 + (k)] = gtime(); } while (0)
#else
#define MT_TR(tile, k) do {} while (0)
#endif

template <int N, int OP>
__global__ void __launch_bounds__(kPThreads, 2) merge64p_kernel(MergeParams p, uint32_t nctas) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* stages = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned long long* sk =
      reinterpret_cast<unsigned long long*>(stages + (size_t)kStages * (N + 1) * kSeg);
  unsigned long long* ek0 = sk + kSK;  // [2][kEK] emission buffers
  uint32_t* sv = reinterpret_cast<uint32_t*>(ek0 + 2 * kEK);
  uint32_t* ev0 = sv + kSV;  // [2][kEV]
  StageInfo* info = reinterpret_cast<StageInfo*>(ev0 + 2 * kEV);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(info + kStages);
  unsigned long long* empty = full + kStages;
  unsigned long long* efull = empty + kStages;  // [2]
  unsigned long long* eempty = efull + 2;       // [2]
  unsigned long long* lbfull = eempty + 2;      // [kSlots] merge -> look-back
  unsigned long long* bfull = lbfull + kSlots;  // [kSlots] look-back -> emitter
  unsigned long long* sempty = bfull + kSlots;  // [kSlots] emitter -> merge
  struct Slot {
    uint32_t tile, total;
    unsigned long long base;
  };
  Slot* slot = reinterpret_cast<Slot*>(sempty + kSlots);
  uint32_t* s_wsum = reinterpret_cast<uint32_t*>(slot + kSlots);  // [8]

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      spt::mbar_init(full + s, 32);
      spt::mbar_init(empty + s, kThreads / 32);
    }
    for (int b = 0; b < 2; ++b) {
      spt::mbar_init(efull + b, kThreads);
      spt::mbar_init(eempty + b, 32);
    }
    for (int r = 0; r < kSlots; ++r) {
      spt::mbar_init(lbfull + r, 1);
      spt::mbar_init(bfull + r, 1);
      spt::mbar_init(sempty + r, 1);
    }
    spt::mbar_fence_init();
  }
  // launched as a programmatic dependent of the partition kernel: the CTAs are
  // resident and their barriers set up while it runs; its splits are read
  // only after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  const uint64_t total = p.nx + p.ny;
  const unsigned lane = tid & 31u;
  const unsigned long long tag = (unsigned long long)p.epoch << 34;

  if (tid >= kThreads + 32 * (kLB + 1)) {
    // ---- producer warp ----
    for (uint32_t it = 0;; ++it) {
      const int s = it % kStages;
      unsigned long long t = 0;
      if (lane == 0) {
        t = atomicAdd(p.tile_ctr, 1ull);
        if (t == (unsigned long long)p.ntiles + nctas - 1) atomicExch(p.tile_ctr, 0ull);
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      uint64_t a0 = 0, a1 = 0;
      if (t < p.ntiles) {
        a0 = p.split[t];
        a1 = p.split[t + 1];
      }
      if (lane == 0 && t < p.ntiles) MT_TR(t, 0);
      if (it >= kStages) spt::mbar_wait(empty + s, ((it / kStages) - 1) & 1u);
      if (lane == 0 && t < p.ntiles) MT_TR(t, 1);
      StageInfo& inf = info[s];
      if (t >= p.ntiles) {
        if (lane == 0) inf.tile = kDone;
        __syncwarp();
        spt::mbar_arrive(full + s);
        break;
      }
      const uint64_t d0 = t * (uint64_t)kTile;
      const uint64_t d1 = std::min<uint64_t>(d0 + kTile, total);
      const uint64_t b0 = d0 - a0, b1 = d1 - a1;
      const uint32_t nxt = static_cast<uint32_t>(a1 - a0), nyt = static_cast<uint32_t>(b1 - b0);
      // lane q <= N: x run of array q (q == N: values); lane 16+q: y run.
      const bool is_y = lane >= 16;
      const uint32_t q = lane & 15u;
      // mul stages no values: only its (few) matches read them, from global
      if (q < static_cast<uint32_t>(N) || (q == static_cast<uint32_t>(N) && OP != SPT_MUL)) {
        const uint32_t* xs =
            q < static_cast<uint32_t>(N) ? p.xi[q] : reinterpret_cast<const uint32_t*>(p.xv);
        const uint32_t* ys =
            q < static_cast<uint32_t>(N) ? p.yi[q] : reinterpret_cast<const uint32_t*>(p.yv);
        const uint32_t* src = is_y ? ys : xs;
        const uint64_t e0 = is_y ? b0 : a0;
        const uint32_t n = is_y ? nyt : nxt;
        // x run at word xp (the 16-byte phase of xs+a0); y run after it, in
        // its own phase.
        const uint32_t xp = word_phase(xs + a0);
        const uint32_t off = is_y ? ((xp + nxt + 3u) & ~3u) + word_phase(ys + b0) : xp;
        if (is_y) inf.yoff[q] = off;
        else inf.xoff[q] = off;
        const uint32_t head = std::min<uint32_t>(n, (4u - word_phase(src + e0)) & 3u);
        const uint32_t body = (n - head) & ~3u;
        // announce this lane's bytes before its copy can complete
        if (body) spt::mbar_expect_tx(full + s, body * 4);
        copy_run(stages + ((size_t)s * (N + 1) + q) * kSeg + off, src, e0, n, head, body,
                 full + s);
      }
      if (lane == 31) {
        inf.tile = static_cast<uint32_t>(t);
        inf.nxt = nxt;
        inf.nyt = nyt;
        inf.a0 = a0;
        inf.b0 = b0;
        inf.y_after = (b1 < p.ny) ? pack_g<N>(p.yi, p, b1) : ~0ull;
        inf.x_before = (a0 > 0) ? pack_g<N>(p.xi, p, a0 - 1) : ~0ull;
        inf.yv_after = (b1 < p.ny) ? __float_as_uint(__ldg(p.yv + b1)) : 0u;
      }
      spt::mbar_arrive(full + s);
    }
    return;
  }

  if (tid >= kThreads + 32 * kLB) {
    // ---- emitter warp: coalesced output of each tile at its base ----
    for (uint32_t it = 0;; ++it) {
      const int r = it % kSlots, b = it & 1;
      spt::mbar_wait(bfull + r, (it / kSlots) & 1u);
      const uint32_t tile = slot[r].tile, tile_total = slot[r].total;
      const unsigned long long base = slot[r].base;
      __syncwarp();
      if (lane == 0) spt::mbar_arrive(sempty + r);
      if (tile == kDone) break;
      spt::mbar_wait(efull + b, (it >> 1) & 1u);
      const unsigned long long* ek = ek0 + b * kEK;
      const uint32_t* ev = ev0 + b * kEV;
      for (uint32_t o = lane; o < tile_total; o += 32) {
        const unsigned long long k = ek[epad64(o)];
#pragma unroll
        for (int q = 0; q < N; ++q)
          spt::st_stream(p.zi[q] + base + o, (uint32_t)((k >> p.shift[q]) & p.mask[q]));
        spt::st_stream(reinterpret_cast<uint32_t*>(p.zv) + base + o, ev[epad(o)]);
      }
      spt::mbar_arrive(eempty + b);
    }
    return;
  }

  if (tid >= kThreads) {
    // ---- look-back warps: exclusive output offset of each tile, publish P.
    // kLB warps take the CTA's tiles round-robin, so a look-back that waits
    // on a slow predecessor does not hold up the next tile's.
    for (uint32_t it = (tid - kThreads) >> 5;; it += kLB) {
      const int r = it % kSlots;
      spt::mbar_wait(lbfull + r, (it / kSlots) & 1u);
      const uint32_t tile = slot[r].tile, tile_total = slot[r].total;
      unsigned long long base = 0;
      if (tile != kDone) {
        if (tile != 0) {
          base = spt::lookback_count64_wide<8, kSS>(p.status, tile, p.epoch);
          if (lane == 0)
            spt::st_relaxed64(p.status + ((size_t)tile << kSS),
                              tag | (kFlagP << 32) | (base + tile_total));
        }
        if (lane == 0 && tile == p.ntiles - 1) *p.total = base + tile_total;
      }
      if (lane == 0) {
        slot[r].base = base;
        spt::mbar_arrive(bfull + r);
      }
      if (tile == kDone) break;
    }
    return;
  }

  // ---- merge warps ----
  using spt::bar_sync;
  const int warp = tid >> 5;
  // A tile's emitted items stay in registers until the next tile has been
  // merged, and only then go to an emission buffer: by that time the tile's
  // look-back has mostly resolved, so each buffer is held only for the
  // emission itself (two buffers + this register stage = three in flight).
  unsigned long long pkey[kIPT];
  uint32_t pvb[kIPT];
  uint32_t pmask = 0, pexcl = 0;
  auto flush = [&](uint32_t eseq) {
    const int b = eseq & 1;
    if (eseq >= 2) spt::mbar_wait(eempty + b, ((eseq >> 1) - 1) & 1u);
    unsigned long long* ek = ek0 + b * kEK;
    uint32_t* ev = ev0 + b * kEV;
    int lp = static_cast<int>(pexcl);
#pragma unroll
    for (int k = 0; k < kIPT; ++k) {
      if (!((pmask >> k) & 1u)) continue;
      ek[epad64(lp)] = pkey[k];
      ev[epad(lp)] = pvb[k];
      ++lp;
    }
    spt::mbar_arrive(efull + b);
  };
  for (uint32_t it = 0;; ++it) {
    const int s = it % kStages;
#ifdef SPT_MERGE_TRACE
    const unsigned long long tw0 = gtime();
#endif
    spt::mbar_wait(full + s, (it / kStages) & 1u);
    const StageInfo& inf = info[s];
    const uint32_t tile = inf.tile;
#ifdef SPT_MERGE_TRACE
    if (tid == 0 && tile != kDone && tile < 16384) {
      g_mtrace[tile * 8 + 2] = tw0;
      MT_TR(tile, 3);
    }
#endif
    const int r = it % kSlots;
    if (tile == kDone) {
      if (it > 0) flush(it - 1);
      if (tid == 0) {
        // one kDone per look-back warp (each waits on its own slots)
        for (uint32_t d = it; d < it + kLB; ++d) {
          const int rd = d % kSlots;
          if (d >= kSlots) spt::mbar_wait(sempty + rd, ((d / kSlots) - 1) & 1u);
          slot[rd].tile = kDone;
          spt::mbar_arrive(lbfull + rd);
        }
      }
      break;
    }
    const int nxt = static_cast<int>(inf.nxt), nyt = static_cast<int>(inf.nyt);
    const unsigned long long x_before = inf.x_before, y_after = inf.y_after;
    const unsigned long long inf_a0 = inf.a0, inf_b0 = inf.b0;
    const uint32_t yv_after = inf.yv_after;
    const int len = nxt + nyt;
    const int Y0 = nxt + 1;  // key slot of y entry 0
    {
      const uint32_t* st0 = stages + (size_t)s * (N + 1) * kSeg;
      uint32_t xo[N + 1], yo[N + 1];
#pragma unroll
      for (int q = 0; q <= N; ++q) {
        xo[q] = inf.xoff[q];
        yo[q] = inf.yoff[q] - nxt;  // y entry j sits at word yoff + j = (yoff - nxt) + i
      }
      for (int i = tid; i < len; i += kThreads) {
        const bool isx = i < nxt;
        unsigned long long k = 0;
#pragma unroll
        for (int q = 0; q < N; ++q)
          k |= (unsigned long long)st0[q * kSeg + (isx ? xo[q] : yo[q]) + i] << p.shift[q];
        const int slot_i = isx ? i : i + 1;
        sk[pad64(slot_i)] = k;
        if (OP != SPT_MUL) sv[pad(slot_i)] = st0[N * kSeg + (isx ? xo[N] : yo[N]) + i];
      }
      if (tid == 0) {
        sk[pad64(nxt)] = ~0ull;
        sk[pad64(Y0 + nyt)] = ~0ull;
        if (OP != SPT_MUL) sv[pad(Y0 + nyt)] = inf.yv_after;
      }
    }
    __syncwarp();
    if (lane == 0) spt::mbar_arrive(empty + s);  // this warp is done with the stage
    bar_sync(1, kThreads);
    if (tid == 0) MT_TR(tile, 4);

    const int dg = std::min(tid * kIPT, len);
    int lo = std::max(0, dg - nyt), hi = std::min(dg, nxt);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sk[pad64(mid)] <= sk[pad64(Y0 + dg - 1 - mid)]) lo = mid + 1;
      else hi = mid;
    }
    // Branch-free serial merge: per item one key load (the new head of the
    // side just consumed, clamped onto the sentinels) and one value load; the
    // previous x and the next y that decide matches ride in registers.
    int i = lo, j = dg - lo;
    unsigned long long kx = sk[pad64(i)];
    unsigned long long ky = sk[pad64(Y0 + j)];
    unsigned long long px = i > 0 ? sk[pad64(i - 1)] : x_before;  // last x before item
    unsigned long long key[kIPT];
    uint32_t vbits[kIPT];
    uint32_t emitm = 0;
#pragma unroll
    for (int k = 0; k < kIPT; ++k) {
      const bool valid = dg + k < len;
      const bool xin = i < nxt, yin = j < nyt;
      const bool take_x = xin && (!yin || kx <= ky);
      const bool mx = kx == (yin ? ky : y_after);  // x matched by the following y
      const bool my = px == ky;                    // y matched by the preceding x
      float v = 0.f;
      if (OP == SPT_MUL) {
        if (take_x && mx)  // the y head; past the run, the first y after the tile
          v = __ldg(p.xv + inf_a0 + i) *
              (j < nyt ? __ldg(p.yv + inf_b0 + j) : __uint_as_float(yv_after));
      } else {
        v = __uint_as_float(sv[take_x ? pad(i) : pad(Y0 + j)]);
        if (take_x && mx) {
          // the y head's value; past the run, the sentinel slot holds the next y's
          const float w = __uint_as_float(sv[pad(Y0 + j)]);
          v = OP == SPT_ADD ? v + w : v - w;
        }
      }
      if (OP == SPT_SUB && !take_x) v = -v;
      const bool e = valid && (take_x ? (OP != SPT_MUL || mx) : (OP != SPT_MUL && !my));
      emitm |= e ? (1u << k) : 0u;
      key[k] = take_x ? kx : ky;
      vbits[k] = __float_as_uint(v);
      px = take_x ? kx : px;
      i += take_x ? 1 : 0;
      j += take_x ? 0 : 1;
      const unsigned long long nk =
          sk[take_x ? pad64(min(i, nxt)) : pad64(Y0 + min(j, nyt))];
      kx = take_x ? nk : kx;
      ky = take_x ? ky : nk;
    }
    const uint32_t cnt = __popc(emitm);
    // block exclusive scan of cnt over the 256 merge threads
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<unsigned>(o)) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    bar_sync(1, kThreads);
    uint32_t wpre = 0, tile_total = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint32_t v = s_wsum[w];
      wpre += w < warp ? v : 0u;
      tile_total += v;
    }
    const uint32_t excl = wpre + incl - cnt;
    if (tid == 0) MT_TR(tile, 5);
    if (tid == 0) {
      spt::st_relaxed64(p.status + ((size_t)tile << kSS),
                        tag | ((tile == 0 ? kFlagP : kFlagA) << 32) | tile_total);
      // hand the tile to the look-back warp at once (before the emission
      // buffer is free), so its look-back overlaps everything after
      if (it >= kSlots) spt::mbar_wait(sempty + r, ((it / kSlots) - 1) & 1u);
      slot[r].tile = tile;
      slot[r].total = tile_total;
      spt::mbar_arrive(lbfull + r);
    }
    if (it > 0) flush(it - 1);
    if (tid == 0) MT_TR(tile, 6);
#pragma unroll
    for (int k = 0; k < kIPT; ++k) {
      pkey[k] = key[k];
      pvb[k] = vbits[k];
    }
    pmask = emitm;
    pexcl = excl;
    // s_wsum[0..7] are rewritten only after the next pack barrier, which every
    // thread reaches after its reads above.
  }
}

template <int N, int OP>
int launch64p_op(spt_ctx* ctx, MergeParams& p, cudaStream_t st) {
  constexpr size_t smem = pers_smem<N>();
  static int per_sm = -1;
  if (per_sm < 0) {
    SPT_CUDA(cudaFuncSetAttribute(merge64p_kernel<N, OP>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    SPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge64p_kernel<N, OP>,
                                                           kPThreads, smem));
    per_sm = std::max(per_sm, 1);
  }
  const uint32_t nctas = std::min<uint32_t>(p.ntiles, (uint32_t)(per_sm * ctx->num_sms));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nctas);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  SPT_CUDA(cudaLaunchKernelEx(&cfg, merge64p_kernel<N, OP>, p, nctas));
  ctx->launches++;
  return SPT_OK;
}

template <int N>
int launch64p(spt_ctx* ctx, MergeParams& p, cudaStream_t st) {
  const uint32_t nt = p.ntiles;
  partition_g_kernel<N, SPT_PART_G><<<((uint64_t)(nt + 1) * SPT_PART_G + 255) / 256, 256, 0, st>>>(p, const_cast<uint32_t*>(p.split));
  SPT_LAUNCHED(ctx);
  switch (p.op) {
    case SPT_ADD: return launch64p_op<N, SPT_ADD>(ctx, p, st);
    case SPT_SUB: return launch64p_op<N, SPT_SUB>(ctx, p, st);
    default: return launch64p_op<N, SPT_MUL>(ctx, p, st);
  }
}

template <int N>
int launch(spt_ctx* ctx, MergeParams& p, cudaStream_t st) {
  const uint32_t nt = p.ntiles;
  partition_g_kernel<N, SPT_PART_G><<<((uint64_t)(nt + 1) * SPT_PART_G + 255) / 256, 256, 0, st>>>(p, const_cast<uint32_t*>(p.split));
  SPT_LAUNCHED(ctx);
  const size_t smem = (size_t)(2 * N + 2) * kTP * sizeof(uint32_t) + kTile * sizeof(uint32_t);
  SPT_CUDA(cudaFuncSetAttribute(merge_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  merge_kernel<N><<<nt, kThreads, smem, st>>>(p);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

}  // namespace

extern "C" int spt_tew_f32(spt_ctx* ctx, const spt_coo* x, const spt_coo* y, int op, spt_coo* z,
                           uint64_t z_capacity, uint64_t* h_nnz, uint64_t* d_nnz, unsigned flags,
                           void* stream) {
  (void)flags;
  if (!ctx) return spt::set_error(SPT_EINVAL, "tew: null context");
  SPT_TRY(spt::check_coo(x, "tew"));
  SPT_TRY(spt::check_coo(y, "tew"));
  if (!z) return spt::set_error(SPT_EINVAL, "tew: null output");
  // check_tew_inputs, P/src/kernel_detail.hpp:36-45
  if (op == SPT_DIV)
    return spt::set_error(SPT_EINVAL,
                          "tew: div is not defined for mismatched patterns (unmatched entries "
                          "divide by zero)");
  if (op < SPT_ADD || op > SPT_MUL) return spt::set_error(SPT_EINVAL, "tew: unknown op %d", op);
  if (x->order != y->order)
    return spt::set_error(SPT_EINVAL, "tew: tensors must have the same order");
  if (!x->coalesced || !y->coalesced)
    return spt::set_error(SPT_EINVAL, "tew: both inputs must be coalesced");
  const uint32_t N = x->order;
  bool same = x->has_sort_order && y->has_sort_order;
  for (uint32_t k = 0; same && k < N; ++k) same = x->sort_order[k] == y->sort_order[k];
  if (!same)
    return spt::set_error(SPT_EINVAL,
                          "tew: inputs must share a sort order (sort both ascending first, as "
                          "unify_tew_sort does)");
  const uint64_t need = op == SPT_MUL ? std::min(x->nnz, y->nnz) : x->nnz + y->nnz;
  if (z_capacity < need)
    return spt::set_error(SPT_EINVAL, "tew: output capacity %llu < %llu",
                          (unsigned long long)z_capacity, (unsigned long long)need);
  if (x->nnz + y->nnz >= (1ull << 32))
    return spt::set_error(SPT_EOVERFLOW, "tew: nnz_x + nnz_y exceeds the u32 device range");
  cudaStream_t st = spt::as_stream(stream);
  z->order = N;
  for (uint32_t d = 0; d < SPT_MAX_ORDER; ++d) {
    z->dims[d] = d < N ? std::max(x->dims[d], y->dims[d]) : 0;
    z->sort_order[d] = x->sort_order[d];
  }
  z->has_sort_order = 1;
  z->coalesced = 1;
  const uint64_t total = x->nnz + y->nnz;
  void* scratch;
  const uint64_t ntiles = std::max<uint64_t>(1, (total + kTile - 1) / kTile);
  SPT_TRY(spt::ctx_scratch(ctx, (ntiles + 1) * 4 + 64, &scratch));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch);
  uint32_t* split = reinterpret_cast<uint32_t*>(cnt + 2);
  if (total == 0) {
    SPT_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
  } else {
    for (uint32_t d = 0; d < N && need; ++d)
      if (!z->idx[d]) return spt::set_error(SPT_EINVAL, "tew: null output index array");
    if (!z->val && need) return spt::set_error(SPT_EINVAL, "tew: null output values");
    MergeParams p{};
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t d = x->sort_order[k];
      p.xi[k] = x->idx[d];
      p.yi[k] = y->idx[d];
      p.zi[k] = z->idx[d];
    }
    p.xv = x->val;
    p.yv = y->val;
    p.zv = z->val;
    p.nx = x->nnz;
    p.ny = y->nnz;
    p.split = split;
    p.ntiles = static_cast<uint32_t>(ntiles);
    p.op = op;
    p.tile_ctr = ctx->d_tile_ctr;
    p.total = cnt;
    uint32_t epoch;
    SPT_TRY(spt::ctx_lookback(ctx, 1, 1, &epoch));
    SPT_TRY(spt::ctx_status64(ctx, ntiles << 3, &p.status));  // room for strided layouts
    p.epoch = epoch;
    // Packed u64 keys when the per-mode index widths fit (sort order = key
    // significance; indices are < dims as validate() requires).
    uint32_t width[SPT_MAX_ORDER], bits = 0;
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t d = x->sort_order[k];
      const uint32_t ext = std::max(x->dims[d], y->dims[d]);
      uint32_t w = 0;
      while (w < 32 && (1ull << w) < ext) ++w;
      width[k] = w;
      bits += w;
    }
    if (bits <= 64) {
      uint32_t sh = 0;
      for (int k = static_cast<int>(N) - 1; k >= 0; --k) {
        p.shift[k] = sh;
        p.mask[k] = width[k] >= 32 ? 0xFFFFFFFFu : ((1u << width[k]) - 1u);
        sh += width[k];
      }
      switch (N) {
        case 1: SPT_TRY(launch64p<1>(ctx, p, st)); break;
        case 2: SPT_TRY(launch64p<2>(ctx, p, st)); break;
        case 3: SPT_TRY(launch64p<3>(ctx, p, st)); break;
        case 4: SPT_TRY(launch64p<4>(ctx, p, st)); break;
        case 5: SPT_TRY(launch64p<5>(ctx, p, st)); break;
        case 6: SPT_TRY(launch64p<6>(ctx, p, st)); break;
        case 7: SPT_TRY(launch64p<7>(ctx, p, st)); break;
        default: SPT_TRY(launch64p<8>(ctx, p, st)); break;
      }
    } else switch (N) {
      case 1: SPT_TRY(launch<1>(ctx, p, st)); break;
      case 2: SPT_TRY(launch<2>(ctx, p, st)); break;
      case 3: SPT_TRY(launch<3>(ctx, p, st)); break;
      case 4: SPT_TRY(launch<4>(ctx, p, st)); break;
      case 5: SPT_TRY(launch<5>(ctx, p, st)); break;
      case 6: SPT_TRY(launch<6>(ctx, p, st)); break;
      case 7: SPT_TRY(launch<7>(ctx, p, st)); break;
      default: SPT_TRY(launch<8>(ctx, p, st)); break;
    }
  }
  if (d_nnz)
    SPT_CUDA(cudaMemcpyAsync(d_nnz, cnt, 8, cudaMemcpyDeviceToDevice, st));
  if (h_nnz) {
    SPT_CUDA(cudaMemcpyAsync(ctx->h_pinned, cnt, 8, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
    *h_nnz = ctx->h_pinned[0];
    z->nnz = *h_nnz;
  }
  return SPT_OK;
}

#ifdef SPT_MERGE_TRACE
extern "C" __attribute__((visibility("default"))) int spt_debug_merge_trace(void* dst) {
  return cudaMemcpyFromSymbol(dst, g_mtrace, sizeof(g_mtrace)) == cudaSuccess ? 0 : 5;
}
#endif
