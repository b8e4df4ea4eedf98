// K8 MTTKRP: out(i_n, r) = sum_m val_m * prod_{d != n, ascending} F_d(i_d(m), r).
//
// Reference: seq::mttkrp P/src/kernels_seq.cpp:153-174, par::mttkrp
// P/src/kernels_par.cpp:275-337, mttkrp_row P/src/kernel_detail.hpp:176-188,
// check_mttkrp_inputs P/src/kernel_detail.hpp:153-174.
//
// Segmented strategy (input sorted with the output mode leading, i.e. entries
// of one output row are contiguous):
//   * A CTA owns a tile of TILE=2048 consecutive entries, staged into shared
//     memory with 128-bit loads. Tile ids are taken from a self-resetting
//     atomic counter so predecessors are always resident (look-back safety).
//   * Each warp splits into P = 32/G lane groups; a group owns a contiguous
//     run of entries and each lane holds VEC consecutive columns (float4
//     gathers: an R=32 factor row is one 128-byte line read by 8 lanes).
//     Gathers for U=4 entries are issued before any is consumed.
//   * Per-term products are formed in fp32 exactly as the reference does
//     (val, then *= F_d for d ascending), so every term is bit-identical to
//     seq's; accumulation is in fp64 and each output element is rounded
//     once, which keeps the result within 1e-5 of an fp64 recomputation even
//     for the heavy Zipf rows (a serial fp32 chain would not be).
//   * Rows that start and end inside one group are written directly (plain
//     128-bit stores, one writer per row, no atomics); the first/last run of
//     each group goes to a shared-memory slot; the CTA folds the slots, writes
//     the rows it completes and zero-fills every empty row in its range, so
//     the output needs no memset and each element is written exactly once.
//   * A row that continues across tiles is completed with a decoupled
//     look-back over fp64 R-wide tile partials (status words tagged with a
//     per-launch epoch, so no per-launch reset is needed). Tiles whose first
//     row starts inside them never wait.
//   * The kernel verifies the sortedness it relies on (free: it reads the
//     mode index anyway) and reports violations through the context's
//     error word.
// Atomic strategy (any order): zero the output, then vector red.global.add
// per term group -- the analogue of the reference's `omp atomic` strategy.
#include <algorithm>

#include "internal.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 2048;
constexpr int kTileP = kTile + kTile / 8;  // padded per-entry smem arrays
__device__ __forceinline__ int sw(int e) { return e + ((e >> 5) << 2); }
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kFlagA = 1, kFlagP = 2;

struct MttkrpParams {
  const uint32_t* out_idx;
  const uint32_t* oidx[SPT_MAX_ORDER - 1];
  const float* ofac[SPT_MAX_ORDER - 1];
  const float* val;
  float* out;
  uint64_t nnz;
  uint32_t rows;   // I_n
  uint32_t R;      // row stride of factors and output
  uint32_t c0;     // first column handled by this launch
  uint32_t ncols;  // columns handled (<= CB)
  uint32_t ntiles;
  uint32_t epoch;
  uint32_t* status;
  double* payA;  // [ntiles][CB]
  double* payP;  // [ntiles][CB]
  unsigned long long* tile_ctr;
  unsigned long long* err;
  int vec_ok;  // per-entry arrays 16-byte aligned (vector staging)
  int bid_tiles;  // warp tiles: the grid fits in one wave, so tile = blockIdx (no ticket)
  // TTM (FIBER=true): output rows are fibers of an x sorted with `mode` last.
  const uint32_t* fptr;
  const uint32_t* tile_fiber;
  const uint32_t* hidx[SPT_MAX_ORDER];  // x.indices[d] for the output index tuples
  uint32_t* zidx[SPT_MAX_ORDER];        // z.indices[d]
  const uint32_t* hnm[SPT_MAX_ORDER - 1];  // x.indices of the non-mode dims, ascending
  uint32_t N;
  uint32_t mode;
};

// TTM output index tuples of fiber `row` for `ncol` columns starting at col:
// z.indices[d][row*R + r] = head index of the fiber (d != mode) or r
// (P/src/kernels_seq.cpp:128-138).
// The fiber head's non-mode indices come from the tile's staged copy
// (s_hid[j][sw(head - t0)], j = non-mode dims ascending) when the head lies in
// the tile -- no dependent global load per output row -- else from global.
template <int NCOL>
__device__ __forceinline__ void ttm_emit_idx(const MttkrpParams& p, uint32_t head,
                                             uint32_t row, uint32_t col, const uint32_t* s_hid,
                                             uint64_t t0) {
  const size_t base = (size_t)row * p.R + col;
  int j = 0;
  for (uint32_t d = 0; d < p.N; ++d) {
    uint32_t w[NCOL];
    if (d == p.mode) {
#pragma unroll
      for (int k = 0; k < NCOL; ++k) w[k] = col + k;
    } else {
      const uint32_t h = head >= t0 ? s_hid[j * kTileP + sw(static_cast<int>(head - t0))]
                                    : p.hidx[d][head];
      ++j;
#pragma unroll
      for (int k = 0; k < NCOL; ++k) w[k] = h;
    }
    if constexpr (NCOL == 4) {
      // outputs are written once and never re-read here: evict-first stores
      __stcs(reinterpret_cast<uint4*>(p.zidx[d] + base), make_uint4(w[0], w[1], w[2], w[3]));
    } else {
#pragma unroll
      for (int k = 0; k < NCOL; ++k) p.zidx[d][base + k] = w[k];
    }
  }
}

template <int VEC>
struct Vec;
template <>
struct Vec<4> {
  static __device__ __forceinline__ void load(const float* p, float (&f)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
  }
  static __device__ __forceinline__ void store(float* p, const float (&f)[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(f[0], f[1], f[2], f[3]));
  }
};
template <>
struct Vec<1> {
  static __device__ __forceinline__ void load(const float* p, float (&f)[1]) { f[0] = __ldg(p); }
  static __device__ __forceinline__ void store(float* p, const float (&f)[1]) { *p = f[0]; }
};

template <int U>
__device__ __forceinline__ void ld_batch(const uint32_t* p, uint32_t (&o)[U]) {
  if constexpr (U == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
  } else {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    o[0] = v.x, o[1] = v.y;
  }
}

// Zero rows [r0, r1) for this lane's columns.
template <int VEC>
__device__ __forceinline__ void zero_rows(float* out, uint32_t r0, uint32_t r1, uint32_t R,
                                          uint32_t col, bool col_ok) {
  if (!col_ok) return;
  float z[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) z[k] = 0.0f;
  for (uint32_t r = r0; r < r1; ++r) Vec<VEC>::store(out + (size_t)r * R + col, z);
}

#ifndef SPT_MTTKRP_UNROLL
#define SPT_MTTKRP_UNROLL 4
#endif
#ifndef SPT_SEG_TICKET
#define SPT_SEG_TICKET 0
#endif
#ifndef SPT_MTTKRP_MINB
#define SPT_MTTKRP_MINB 3  // <= 85 registers: 3 CTAs (24 warps) per SM
#endif

template <int NM1, int G, int VEC, bool FIBER>
__global__ void __launch_bounds__(kThreads, SPT_MTTKRP_MINB) mttkrp_seg_kernel(MttkrpParams p) {
  constexpr int P = 32 / G;            // groups per warp
  constexpr int GROUPS = kWarps * P;   // groups per CTA
  constexpr int EG = kTile / GROUPS;   // entries per group
  constexpr int CB = G * VEC;          // columns per launch
  constexpr int NSLOT = 2 * kWarps;  // warp head/tail partials

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_slot = reinterpret_cast<double*>(smem_raw);                 // [NSLOT][CB]
  // Per-entry arrays use the padded layout sw(e) (16 B of padding every 32
  // entries) so the P groups of a warp, which read entries EG apart, hit
  // distinct banks; 16-byte chunks stay aligned for the vector staging.
  uint32_t* s_out = reinterpret_cast<uint32_t*>(s_slot + NSLOT * CB);  // [kTileP]
  float* s_val = reinterpret_cast<float*>(s_out + kTileP);             // [kTileP]
  uint32_t* s_oidx = reinterpret_cast<uint32_t*>(s_val + kTileP);      // [NM1][kTileP]
  uint32_t* s_fptr = s_oidx + NM1 * kTileP;                            // FIBER: [kTile+2]
  double* s_gslot = reinterpret_cast<double*>(s_fptr + (FIBER ? kTile + 4 : 0));  // [GROUPS*2][CB]
  // FIBER: the tile's non-mode indices (fiber head tuples), [N-1][kTileP].
  uint32_t* s_hid = reinterpret_cast<uint32_t*>(s_gslot + 2 * GROUPS * CB);
  __shared__ uint32_t s_grow[2 * GROUPS];
  __shared__ uint32_t s_slot_row[NSLOT];
  __shared__ uint32_t s_flag;
  __shared__ uint32_t s_meta[4];

  const int tid = threadIdx.x;
#if SPT_SEG_TICKET
  __shared__ uint32_t s_tile;
  if (tid == 0) {
    const unsigned long long t = atomicAdd(p.tile_ctr, 1ull);
    if (t == p.ntiles - 1) atomicExch(p.tile_ctr, 0ull);  // last increment of this launch
    s_tile = static_cast<uint32_t>(t);
  }
  __syncthreads();
  const uint32_t tile = s_tile;
#else
  // tiles in launch order (CTAs are dispatched in blockIdx order, as CUB's
  // single-pass scans assume): no ticket round trip
  const uint32_t tile = blockIdx.x;
#endif
  const uint64_t t0 = (uint64_t)tile * kTile;
  const int cnt = (p.nnz - t0 < (uint64_t)kTile) ? static_cast<int>(p.nnz - t0) : kTile;

  // ---- stage the tile (mode index, values, other-mode indices) ----------
  uint32_t f_lo = 0, nstage = 0;
  if constexpr (FIBER) {
    f_lo = p.tile_fiber[tile];
    const uint32_t f_end = (tile + 1 < p.ntiles) ? p.tile_fiber[tile + 1] + 1 : p.rows;
    nstage = f_end - f_lo + 1;
    for (uint32_t i = tid; i < nstage; i += kThreads) s_fptr[i] = p.fptr[f_lo + i];
  }
  if (cnt == kTile && p.vec_ok) {
    const int nv = kTile / 4;
    for (int i = tid; i < nv; i += kThreads) {
      if constexpr (!FIBER)
        reinterpret_cast<uint4*>(s_out)[i + (i >> 3)] =
            spt::ld_stream(reinterpret_cast<const uint4*>(p.out_idx + t0) + i);
      reinterpret_cast<uint4*>(s_val)[i + (i >> 3)] =
          spt::ld_stream(reinterpret_cast<const uint4*>(p.val + t0) + i);
#pragma unroll
      for (int j = 0; j < NM1; ++j)
        reinterpret_cast<uint4*>(s_oidx + j * kTileP)[i + (i >> 3)] =
            spt::ld_stream(reinterpret_cast<const uint4*>(p.oidx[j] + t0) + i);
    }
  } else {
    // Partial (or unaligned) tile: scalar loads; entries past the end get
    // index 0 / value 0 so the gather loop can load unconditionally (their
    // rows are marked dead and never accumulated).
    for (int i = tid; i < kTile; i += kThreads) {
      const bool ok = i < cnt;
      if constexpr (!FIBER) s_out[sw(i)] = ok ? p.out_idx[t0 + i] : 0u;
      s_val[sw(i)] = ok ? p.val[t0 + i] : 0.0f;
#pragma unroll
      for (int j = 0; j < NM1; ++j) s_oidx[j * kTileP + sw(i)] = ok ? p.oidx[j][t0 + i] : 0u;
    }
  }
  if constexpr (FIBER) {
    for (uint32_t j = 0; j + 1 < p.N; ++j)
      for (int i = tid; i < cnt; i += kThreads) s_hid[j * kTileP + sw(i)] = p.hnm[j][t0 + i];
  }
  for (int i = tid; i < NSLOT; i += kThreads) s_slot_row[i] = kNone;
  __syncthreads();
  if constexpr (FIBER) {
    // Output row of each entry = its fiber id (search once, then walk).
    const int per = kTile / kThreads;
    const int e0 = tid * per;
    if (e0 < cnt) {
      const uint64_t m0 = t0 + e0;
      int lo = 0, hi = static_cast<int>(nstage) - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_fptr[mid] <= m0) lo = mid;
        else hi = mid - 1;
      }
      for (int i = 0; i < per && e0 + i < cnt; ++i) {
        while (lo + 1 < static_cast<int>(nstage) && s_fptr[lo + 1] <= m0 + i) ++lo;
        s_out[sw(e0 + i)] = f_lo + lo;
      }
    }
    __syncthreads();
  }

  // ---- per-group segmented accumulation ----------------------------------
  const int warp = tid >> 5, lane = tid & 31;
  const int group = warp * P + lane / G;
  const int gl = lane % G;
  const uint32_t lcol = gl * VEC;  // column within the block
  const bool col_ok = lcol < p.ncols;
  const uint32_t col = p.c0 + lcol;
  const int e_begin = group * EG;
  const int e_end = min(e_begin + EG, cnt);

  uint32_t run_row = kNone;
  bool first_run = true;
  // Group results go to this warp's slots: [2*gw] = first run, [2*gw+1] = last
  // run (if distinct). acc: fp64 total of the open run; a32: fp32 partial of
  // the open run within the current batch (<= kUnroll terms), spilled into acc
  // once per batch.
  const int gw = lane / G;  // group within the warp
  double* my_gslot = s_gslot + (size_t)warp * (2 * P) * CB;
  uint32_t* my_grow = s_grow + warp * (2 * P);
  if (gl == 0) {
    my_grow[2 * gw] = kNone;
    my_grow[2 * gw + 1] = kNone;
  }
  double acc[VEC];
  float a32[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    acc[k] = 0.0;
    a32[k] = 0.0f;
  }

  // Per-lane byte bases of the factor slices (column folded in; lanes beyond
  // ncols read column c0, never stored) and the byte row stride.
  const char* fbase[NM1];
#pragma unroll
  for (int j = 0; j < NM1; ++j)
    fbase[j] = reinterpret_cast<const char*>(p.ofac[j] + (col_ok ? col : p.c0));
  const uint32_t rstride = p.R * 4u;
  constexpr int kUnroll = (NM1 * VEC <= 12) ? 4 : 2;
  for (int e = e_begin; e < e_end; e += kUnroll) {
    float prod[kUnroll][VEC];
    uint32_t rr[kUnroll], ix[NM1][kUnroll];
    float vv[kUnroll];
    // One vector LDS per array for the whole batch (batches are 16-byte
    // aligned in the padded layout and never straddle a pad).
    ld_batch<kUnroll>(s_out + sw(e), rr);
    ld_batch<kUnroll>(reinterpret_cast<const uint32_t*>(s_val) + sw(e),
                      reinterpret_cast<uint32_t(&)[kUnroll]>(vv));
#pragma unroll
    for (int j = 0; j < NM1; ++j) ld_batch<kUnroll>(s_oidx + j * kTileP + sw(e), ix[j]);
    const bool full = e + kUnroll <= e_end;
    // Issue every gather of the batch before consuming any. Loads are
    // unconditional (dead entries carry index 0, dead columns read a valid
    // column) so the block is straight-line: one IMAD.WIDE + one LDG each.
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (e + u >= e_end) rr[u] = kNone;
    float f[kUnroll][NM1][VEC];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int j = 0; j < NM1; ++j)
        Vec<VEC>::load(reinterpret_cast<const float*>(fbase[j] + (size_t)ix[j][u] * rstride),
                       f[u][j]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float t = vv[u];  // row[r] = val; row[r] *= f_d[r] for d ascending
#pragma unroll
        for (int j = 0; j < NM1; ++j) t = __fmul_rn(t, f[u][j][k]);
        prod[u][k] = t;
      }
    }
    // Fast path: the whole batch continues the open run (the common case).
    bool same = full && rr[0] == run_row;
#pragma unroll
    for (int u = 1; u < kUnroll; ++u) same = same && rr[u] == run_row;
    if (same) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float s = prod[0][k];
#pragma unroll
        for (int u = 1; u < kUnroll; ++u) s += prod[u][k];
        acc[k] += (double)s;
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (rr[u] == kNone) continue;
      const uint32_t row = rr[u];
      if (row == run_row) {
#pragma unroll
        for (int k = 0; k < VEC; ++k) a32[k] += prod[u][k];
      } else {
        if (run_row != kNone) {
          if (row < run_row) {
            if (gl == 0) atomicMin(p.err + 2, (unsigned long long)(t0 + e + u));
          }
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[k] += (double)a32[k];
          if (first_run) {
            if (gl == 0) my_grow[2 * gw] = run_row;
#pragma unroll
            for (int k = 0; k < VEC; ++k) my_gslot[(2 * gw) * CB + lcol + k] = acc[k];
            first_run = false;
          } else if (col_ok) {
            float o[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k) o[k] = (float)acc[k];
            Vec<VEC>::store(p.out + (size_t)run_row * p.R + col, o);
            if constexpr (FIBER)
              ttm_emit_idx<VEC>(p, s_fptr[run_row - f_lo], run_row, col, s_hid, t0);
          }
          if (row > run_row + 1) zero_rows<VEC>(p.out, run_row + 1, row, p.R, col, col_ok);
        }
        run_row = row;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          acc[k] = 0.0;
          a32[k] = prod[u][k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      acc[k] += (double)a32[k];
      a32[k] = 0.0f;
    }
  }
  if (run_row != kNone) {
    const int sl = 2 * gw + (first_run ? 0 : 1);
    if (gl == 0) my_grow[sl] = run_row;
#pragma unroll
    for (int k = 0; k < VEC; ++k) my_gslot[sl * CB + lcol + k] = acc[k];
  }
  __syncwarp();

  // ---- warp fold of the P groups' boundary runs (every lane group walks the
  // warp's 2P slots, in parallel across warps): rows complete inside the warp
  // are written here, the warp's first and last row go to two CTA slots.
  {
    uint32_t w_cur = kNone, h_row = kNone;
    int cur_g = -1;
    double w_acc[VEC], h_acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) w_acc[k] = h_acc[k] = 0.0;
    const bool writer = gw == 0 && col_ok;
#pragma unroll 1
    for (int g = 0; g < P; ++g) {
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int sl = 2 * g + it;
        const uint32_t row = my_grow[sl];
        if (row == kNone) continue;
        double v[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = my_gslot[sl * CB + lcol + k];
        if (row == w_cur) {
#pragma unroll
          for (int k = 0; k < VEC; ++k) w_acc[k] += v[k];
        } else {
          if (w_cur != kNone) {
            if (h_row == kNone) {
              h_row = w_cur;
#pragma unroll
              for (int k = 0; k < VEC; ++k) h_acc[k] = w_acc[k];
            } else if (writer) {
              float o[VEC];
#pragma unroll
              for (int k = 0; k < VEC; ++k) o[k] = (float)w_acc[k];
              Vec<VEC>::store(p.out + (size_t)w_cur * p.R + col, o);
              if constexpr (FIBER)
                ttm_emit_idx<VEC>(p, s_fptr[w_cur - f_lo], w_cur, col, s_hid, t0);
            }
            if (g != cur_g && row > w_cur + 1 && writer)
              zero_rows<VEC>(p.out, w_cur + 1, row, p.R, col, true);
          }
          w_cur = row;
#pragma unroll
          for (int k = 0; k < VEC; ++k) w_acc[k] = v[k];
        }
        cur_g = g;
      }
    }
    // slots: [2w] = warp head row, [2w+1] = warp tail row (if distinct)
    uint32_t t_row = kNone;
    if (h_row == kNone) {
      h_row = w_cur;
#pragma unroll
      for (int k = 0; k < VEC; ++k) h_acc[k] = w_acc[k];
    } else {
      t_row = w_cur;
    }
    if (gw == 0) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        s_slot[(2 * warp) * CB + lcol + k] = h_acc[k];
        s_slot[(2 * warp + 1) * CB + lcol + k] = w_acc[k];
      }
      if (lane == 0) {
        s_slot_row[2 * warp] = h_row;
        s_slot_row[2 * warp + 1] = t_row;
      }
    }
  }
  __syncthreads();

  // ---- CTA fold of the group boundary slots -------------------------------
  const uint32_t head_row = s_out[0];
  const uint32_t tail_row = s_out[sw(cnt - 1)];
  if (tid == 0) {
    uint32_t prev_row, next_row;
    if constexpr (FIBER) {
      // Rows are fiber ids: contiguous, every fiber non-empty.
      prev_row = tile > 0 ? (s_fptr[0] < t0 ? f_lo : f_lo - 1) : kNone;
      next_row = kNone;
      if (tile + 1 < p.ntiles) next_row = s_fptr[tail_row - f_lo + 1] > t0 + cnt ? tail_row : tail_row + 1;
    } else {
      prev_row = tile > 0 ? p.out_idx[t0 - 1] : kNone;
      next_row = (tile + 1 < p.ntiles) ? p.out_idx[t0 + cnt] : kNone;
    }
    if (prev_row != kNone && prev_row > head_row) atomicMin(p.err + 2, (unsigned long long)t0);
    if (next_row != kNone && next_row < tail_row)
      atomicMin(p.err + 2, (unsigned long long)(t0 + cnt));
    s_meta[0] = prev_row == head_row ? 1u : 0u;  // continues from previous tile
    s_meta[1] = next_row == tail_row ? 1u : 0u;  // continues into next tile
    s_meta[2] = next_row;
  }
  double head_acc = 0.0, tail_acc = 0.0;
  const int c = tid;  // one thread per column of the block for the fold
  if (c < CB) {
    const bool cok = static_cast<uint32_t>(c) < p.ncols;
    uint32_t cur_row = kNone;
    int cur_group = -1;
    double cur = 0.0;
    for (int s = 0; s < NSLOT; ++s) {
      const uint32_t r = s_slot_row[s];
      if (r == kNone) continue;
      const double v = s_slot[s * CB + c];
      if (r == cur_row) {
        cur += v;
      } else {
        if (cur_row != kNone) {
          if (cur_row == head_row) head_acc = cur;
          else if (cur_row == tail_row) tail_acc = cur;
          else if (cok) {
            p.out[(size_t)cur_row * p.R + p.c0 + c] = (float)cur;
            if constexpr (FIBER)
              ttm_emit_idx<1>(p, s_fptr[cur_row - f_lo], cur_row, p.c0 + c, s_hid, t0);
          }
          if ((s >> 1) != cur_group && r > cur_row + 1 && cok)
            for (uint32_t z = cur_row + 1; z < r; ++z) p.out[(size_t)z * p.R + p.c0 + c] = 0.0f;
        }
        cur_row = r;
        cur = v;
      }
      cur_group = s >> 1;
    }
    if (cur_row != kNone) {
      if (cur_row == head_row) head_acc = cur;
      else tail_acc = cur;  // cur_row == tail_row
    }
  }
  __syncthreads();
  const bool cont_prev = s_meta[0] != 0;
  const bool cont_next = s_meta[1] != 0;
  const uint32_t next_row = s_meta[2];
  const bool boundary = head_row != tail_row;

  // ---- inter-tile zero fill ------------------------------------------------
  if (c < CB && static_cast<uint32_t>(c) < p.ncols) {
    if (tile == 0)
      for (uint32_t z = 0; z < head_row; ++z) p.out[(size_t)z * p.R + p.c0 + c] = 0.0f;
    const uint32_t stop = next_row == kNone ? p.rows : next_row;
    for (uint32_t z = tail_row + 1; z < stop; ++z) p.out[(size_t)z * p.R + p.c0 + c] = 0.0f;
  }

  // ---- decoupled look-back for rows spanning tiles ------------------------
  double carry = 0.0;
  const uint32_t tag = p.epoch << 3;
  if (cont_next && (boundary || !cont_prev)) {
    // Inclusive partial of the tail row is known without predecessors.
    if (c < CB) {
      p.payP[(size_t)tile * CB + c] = boundary ? tail_acc : head_acc;
      spt::fence_release();
    }
    __syncthreads();
    if (tid == 0) spt::st_release(p.status + tile, tag | kFlagP);
  } else if (cont_next) {
    // Single-row tile continuing both ways: publish the aggregate first.
    if (c < CB) {
      p.payA[(size_t)tile * CB + c] = head_acc;
      spt::fence_release();
    }
    __syncthreads();
    if (tid == 0) spt::st_release(p.status + tile, tag | kFlagA);
  }
  if (cont_prev && (boundary || !cont_next)) {
    // This tile completes a row that started in an earlier tile: it sums the
    // aggregates of every tile the row crossed (A's back to the P of the tile
    // where the row started). Tiles strictly inside a heavy row publish only
    // their A and never wait, so a row spanning thousands of tiles costs one
    // walk at its end instead of a serial chain of inclusive prefixes.
    if (warp == 0) {
      const uint32_t n = spt::lookback_chain(p.status, tile, p.epoch);
      if (lane == 0) s_flag = n;
    }
    __syncthreads();
    const uint32_t n = s_flag;
    // The CTA sums the chain: NS slices per column, fixed order (deterministic).
    constexpr int NS = kThreads / CB;
    const int cc = tid % CB, sl = tid / CB;
    double part = 0.0;
    for (uint32_t q = 1 + sl; q <= n && q <= tile; q += NS)
      part += spt::ld_cg((q == n ? p.payP : p.payA) + (size_t)(tile - q) * CB + cc);
    s_gslot[sl * CB + cc] = part;  // group slots are free after the warp fold
    __syncthreads();
    if (c < CB)
      for (int s = 0; s < NS; ++s) carry += s_gslot[s * CB + c];
  }

  // ---- rows completed by this tile ------------------------------------------
  if (c < CB && static_cast<uint32_t>(c) < p.ncols) {
    if (boundary || !cont_next) {
      p.out[(size_t)head_row * p.R + p.c0 + c] = (float)(carry + head_acc);
      if constexpr (FIBER) {
        // The head of the tile's first fiber may lie in an earlier tile.
        ttm_emit_idx<1>(p, s_fptr[head_row - f_lo], head_row, p.c0 + c, s_hid, t0);
      }
    }
    if (boundary && !cont_next) {
      p.out[(size_t)tail_row * p.R + p.c0 + c] = (float)tail_acc;
      if constexpr (FIBER)
        ttm_emit_idx<1>(p, s_fptr[tail_row - f_lo], tail_row, p.c0 + c, s_hid, t0);
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent segmented MTTKRP with an asynchronous tile fold (16-byte-aligned
// inputs, > 4M nnz). CTA = 8 gather warps + 1 fold warp, resident for the
// whole launch:
//   * gather warps stream their 256-entry slice of each tile through a
//     per-warp cp.async ring (no CTA staging barrier), gather and accumulate
//     exactly as mttkrp_seg_kernel does, fold their P groups, write the rows
//     complete inside the warp and hand the warp's first/last-row partials to
//     the fold warp -- then move straight on to the next tile;
//   * the fold warp takes tile tickets (in order, 4 ahead), folds the 8
//     warps' partials, zero-fills the gaps, publishes the tail partial and
//     runs the decoupled look-back for the head row, writing the tile's
//     boundary rows -- while the gather warps already work on the next tile.
// The end-of-tile CTA barriers of the non-persistent kernel (about a fifth of
// its time on the Zipf configs) disappear from the gather warps' path.
constexpr int kPfRingD = 3;
#ifndef SPT_PF_TICKETS
#define SPT_PF_TICKETS 4
#endif
constexpr int kPfTickets = SPT_PF_TICKETS;
#ifndef SPT_PF_CBUF
#define SPT_PF_CBUF 4
#endif
constexpr int kPfCBuf = SPT_PF_CBUF;  // tiles of fold slack for the gather warps
constexpr int kPfThreads = kThreads + 32;

__device__ __forceinline__ void pf_cp_async(void* dst, const void* src, int bytes,
                                            int src_bytes) {
  const uint32_t d = spt::smem_addr(dst);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                 "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void pf_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void pf_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NM1, int G, int VEC>
struct PfShape {
  static constexpr int P = 32 / G;
  static constexpr int CB = G * VEC;
  static constexpr int kU = (NM1 * VEC <= 12) ? 4 : 2;
  static constexpr int NA = 2 + NM1;
  static constexpr int EG = kTile / kWarps / P;  // entries per group
  static constexpr int NB = EG / kU;              // batches per group
  static constexpr int kSlotW = NA * P * kU;      // ring words per batch (warp)
  static constexpr size_t ring = (size_t)kWarps * kPfRingD * kSlotW * 4;
  static constexpr size_t gslot = (size_t)kWarps * 2 * P * CB * 8;
  static constexpr size_t cslot = (size_t)kPfCBuf * 2 * kWarps * CB * 8;
  static constexpr size_t smem = gslot + cslot + ring;
};

template <int NM1, int G, int VEC>
__global__ void __launch_bounds__(kPfThreads, 3) mttkrp_pf_kernel(MttkrpParams p, uint32_t nctas) {
  using S = PfShape<NM1, G, VEC>;
  constexpr int P = S::P, CB = S::CB, kU = S::kU, NA = S::NA, EG = S::EG, NB = S::NB;
  constexpr int NSL = 2 * kWarps;  // CTA slots per tile: head/tail of each warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_gslot = reinterpret_cast<double*>(smem_raw);               // [kWarps][2P][CB]
  double* s_cslot = s_gslot + (size_t)kWarps * 2 * P * CB;             // [kPfCBuf][NSL][CB]
  uint32_t* s_ring = reinterpret_cast<uint32_t*>(s_cslot + kPfCBuf * NSL * CB);
  __shared__ uint32_t s_grow[kWarps][2 * P];
  __shared__ uint32_t s_crow[kPfCBuf][NSL];
  __shared__ uint32_t s_ticket[kPfTickets];
  __shared__ __align__(8) unsigned long long s_bar[2 * kPfTickets + 2 * kPfCBuf];
  unsigned long long* tfull = s_bar;                 // [4] ticket published (count 1)
  unsigned long long* tempty = s_bar + kPfTickets;   // [4] ticket read by all gather warps (8)
  unsigned long long* cfull = s_bar + 2 * kPfTickets;  // [kPfCBuf] slots written (256 threads)
  unsigned long long* cempty = cfull + kPfCBuf;        // [kPfCBuf] slots folded (32 lanes)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int r = 0; r < kPfTickets; ++r) {
      spt::mbar_init(tfull + r, 1);
      spt::mbar_init(tempty + r, kWarps);
    }
    for (int b = 0; b < kPfCBuf; ++b) {
      spt::mbar_init(cfull + b, kThreads);
      spt::mbar_init(cempty + b, 32);
    }
    spt::mbar_fence_init();
  }
  __syncthreads();

  if (warp == kWarps) {
    // ================= fold warp =================
    bool got_end = false;
    auto fetch = [&]() -> uint32_t {
      unsigned long long t = 0;
      if (lane == 0) {
        t = atomicAdd(p.tile_ctr, 1ull);
        if (t == (unsigned long long)p.ntiles + nctas - 1) atomicExch(p.tile_ctr, 0ull);
      }
      return static_cast<uint32_t>(__shfl_sync(0xffffffffu, t, 0));
    };
    for (int r = 0; r < kPfTickets; ++r) {
      uint32_t t = p.ntiles;
      if (!got_end) {
        t = fetch();
        got_end = t >= p.ntiles;
      }
      if (lane == 0) {
        s_ticket[r] = t;
        spt::mbar_arrive(tfull + r);
      }
    }
    const uint32_t tag = p.epoch << 3;
    for (uint32_t i = 0;; ++i) {
      const int r = i % kPfTickets, cb = i % kPfCBuf;
      const uint32_t tile = s_ticket[r];
      if (tile >= p.ntiles) break;
      const uint64_t t0 = (uint64_t)tile * kTile;
      const uint32_t cnt = static_cast<uint32_t>(std::min<uint64_t>(kTile, p.nnz - t0));
      // neighbours (issued before the wait, consumed after it)
      const uint32_t prev_row = tile > 0 ? __ldg(p.out_idx + t0 - 1) : kNone;
      const uint32_t next_row = t0 + cnt < p.nnz ? __ldg(p.out_idx + t0 + cnt) : kNone;
      spt::mbar_wait(cfull + cb, (i / kPfCBuf) & 1u);
      const double* cs = s_cslot + (size_t)cb * NSL * CB;
      const uint32_t* crow = s_crow[cb];
      uint32_t head_row = kNone, tail_row = kNone;
      for (int s = 0; s < NSL; ++s) {
        const uint32_t rw = crow[s];
        if (rw == kNone) continue;
        if (head_row == kNone) head_row = rw;
        tail_row = rw;
      }
      if (lane == 0) {
        if (prev_row != kNone && prev_row > head_row) atomicMin(p.err + 2, (unsigned long long)t0);
        if (next_row != kNone && next_row < tail_row)
          atomicMin(p.err + 2, (unsigned long long)(t0 + cnt));
      }
      const bool cont_prev = prev_row == head_row;
      const bool cont_next = next_row == tail_row;
      const bool boundary = head_row != tail_row;
      bool ext = false;  // interior tile whose predecessor already published P
      if (cont_prev && cont_next && !boundary) {
        uint32_t sp = lane == 0 ? spt::ld_relaxed(p.status + tile - 1) : 0u;
        sp = __shfl_sync(0xffffffffu, sp, 0);
        ext = (sp >> 3) == p.epoch && (sp & 3u) == kFlagP;
        if (ext) __threadfence();  // acquire: the predecessor's payload is visible
      }
      for (int c = lane; c < CB; c += 32) {
        const bool cok = static_cast<uint32_t>(c) < p.ncols;
        const uint32_t col = p.c0 + c;
        // fold of the warps' first/last-row partials (rows complete here)
        double head_acc = 0.0, tail_acc = 0.0, cur = 0.0;
        uint32_t cur_row = kNone;
        int cur_w = -1;
        for (int s = 0; s < NSL; ++s) {
          const uint32_t rw = crow[s];
          if (rw == kNone) continue;
          const double v = cs[s * CB + c];
          if (rw == cur_row) {
            cur += v;
          } else {
            if (cur_row != kNone) {
              if (cur_row == head_row) head_acc = cur;
              else if (cok) __stcs(p.out + (size_t)cur_row * p.R + col, (float)cur);
              if ((s >> 1) != cur_w && rw > cur_row + 1 && cok)
                for (uint32_t z = cur_row + 1; z < rw; ++z) __stcs(p.out + (size_t)z * p.R + col, 0.0f);
            }
            cur_row = rw;
            cur = v;
          }
          cur_w = s >> 1;
        }
        if (cur_row == head_row) head_acc = cur;
        else tail_acc = cur;
        if (!boundary) tail_acc = head_acc;
        // inter-tile zero fill
        if (cok) {
          if (tile == 0)
            for (uint32_t z = 0; z < head_row; ++z) __stcs(p.out + (size_t)z * p.R + col, 0.0f);
          const uint32_t stop = next_row == kNone ? p.rows : next_row;
          for (uint32_t z = tail_row + 1; z < stop; ++z) __stcs(p.out + (size_t)z * p.R + col, 0.0f);
        }
        // publish this tile's tail partial for successors; a tile strictly
        // inside a long row extends its predecessor's inclusive prefix when
        // that is already there (no waiting), which keeps the walk of the
        // row's last tile short
        if (cont_next) {
          const bool incl = boundary || !cont_prev || ext;
          double v = boundary || !cont_prev ? tail_acc : head_acc;
          if (ext) v += spt::ld_cg(p.payP + (size_t)(tile - 1) * CB + c);
          (incl ? p.payP : p.payA)[(size_t)tile * CB + c] = v;
        }
      }
      if (cont_next) {
        spt::fence_release();
        __syncwarp();
        if (lane == 0)
          spt::st_release(p.status + tile,
                          tag | ((boundary || !cont_prev || ext) ? kFlagP : kFlagA));
      }
      uint32_t n_chain = 0;
      if (cont_prev && (boundary || !cont_next)) n_chain = spt::lookback_chain(p.status, tile, p.epoch);
      for (int c = lane; c < CB; c += 32) {
        const bool cok = static_cast<uint32_t>(c) < p.ncols;
        const uint32_t col = p.c0 + c;
        // head/tail partials again (same fold, no stores) -- cheaper than
        // keeping CB/32 pairs of doubles per lane across the look-back
        double head_acc = 0.0, tail_acc = 0.0, cur = 0.0;
        uint32_t cur_row = kNone;
        for (int s = 0; s < NSL; ++s) {
          const uint32_t rw = crow[s];
          if (rw == kNone) continue;
          const double v = cs[s * CB + c];
          if (rw == cur_row) {
            cur += v;
          } else {
            if (cur_row == head_row) head_acc = cur;
            cur_row = rw;
            cur = v;
          }
        }
        if (cur_row == head_row) head_acc = cur;
        else tail_acc = cur;
        // chain sum, 8 independent partials so the loads overlap (a row
        // spanning thousands of tiles makes this walk long)
        const uint32_t nq = std::min<uint32_t>(n_chain, tile);
        double part[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        uint32_t q = 1;
        for (; q + 7 < nq; q += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            part[u] += spt::ld_cg(p.payA + (size_t)(tile - q - u) * CB + c);
        }
        for (; q <= nq; ++q)
          part[0] += spt::ld_cg((q == n_chain ? p.payP : p.payA) + (size_t)(tile - q) * CB + c);
        const double carry = ((part[0] + part[1]) + (part[2] + part[3])) +
                             ((part[4] + part[5]) + (part[6] + part[7]));
        if (cok) {
          if (boundary || !cont_next)
            __stcs(p.out + (size_t)head_row * p.R + col, (float)(carry + head_acc));
          if (boundary && !cont_next) __stcs(p.out + (size_t)tail_row * p.R + col, (float)tail_acc);
        }
      }
      __syncwarp();
      spt::mbar_arrive(cempty + cb);
      // refill this ticket slot for the CTA's tile i + kPfTickets
      spt::mbar_wait(tempty + r, (i / kPfTickets) & 1u);
      uint32_t t = p.ntiles;
      if (!got_end) {
        t = fetch();
        got_end = t >= p.ntiles;
      }
      if (lane == 0) {
        s_ticket[r] = t;
        spt::mbar_arrive(tfull + r);
      }
    }
    return;
  }

  // ================= gather warps =================
  const int gw = lane / G, gl = lane % G;
  const uint32_t lcol = gl * VEC;
  const bool col_ok = lcol < p.ncols;
  const uint32_t col = p.c0 + lcol;
  const char* fbase[NM1];
#pragma unroll
  for (int j = 0; j < NM1; ++j)
    fbase[j] = reinterpret_cast<const char*>(p.ofac[j] + (col_ok ? col : p.c0));
  const uint32_t rstride = p.R * 4u;
  double* my_gslot = s_gslot + (size_t)warp * (2 * P) * CB;
  uint32_t* my_grow = s_grow[warp];
  uint32_t* my_ring = s_ring + (size_t)warp * kPfRingD * S::kSlotW;
  const int wbase = warp * P * EG;

  for (uint32_t i = 0;; ++i) {
    const int r = i % kPfTickets;
    spt::mbar_wait(tfull + r, (i / kPfTickets) & 1u);
    const uint32_t tile = s_ticket[r];
    __syncwarp();
    if (lane == 0) spt::mbar_arrive(tempty + r);
    if (tile >= p.ntiles) break;
    const uint64_t t0 = (uint64_t)tile * kTile;
    const int cnt = static_cast<int>(std::min<uint64_t>(kTile, p.nnz - t0));
    // batch k of every group of this warp: lane c < NA*P (two roles when
    // NA*P > 32) copies array c/P of group c%P; source and destination are
    // fixed per tile, so a batch costs one address add and one cp.async
    constexpr int kRoles = (NA * P + 31) / 32;
    const uint32_t* rsrc[kRoles];
    int rrem[kRoles], rdst[kRoles];
#pragma unroll
    for (int q = 0; q < kRoles; ++q) {
      const int c = lane + 32 * q;
      const int a = c / P, g = c % P;
      const uint32_t* src = a == 0 ? p.out_idx : reinterpret_cast<const uint32_t*>(p.val);
#pragma unroll
      for (int j = 0; j < NM1; ++j)
        if (a == 2 + j) src = p.oidx[j];
      const int ee = wbase + g * EG;
      rsrc[q] = src + t0 + ee;
      rrem[q] = c < NA * P ? cnt - ee : -1;  // -1: no role
      rdst[q] = a * P * kU + g * kU;
    }
    auto issue = [&](int k) {
      if (k < NB) {
#pragma unroll
        for (int q = 0; q < kRoles; ++q) {
          if (rrem[q] < 0 && lane + 32 * q >= NA * P) continue;
          const int rem = rrem[q] - k * kU;
          const int sb = rem >= kU ? kU * 4 : (rem > 0 ? rem * 4 : 0);
          pf_cp_async(my_ring + (k % kPfRingD) * S::kSlotW + rdst[q],
                      sb > 0 ? rsrc[q] + k * kU : p.out_idx, kU * 4, sb);
        }
      }
      pf_commit();
    };
#pragma unroll
    for (int k = 0; k < kPfRingD - 1; ++k) issue(k);

    const int e_begin = wbase + gw * EG;
    const int e_end = min(e_begin + EG, cnt);
    if (gl == 0) {
      my_grow[2 * gw] = kNone;
      my_grow[2 * gw + 1] = kNone;
    }
    uint32_t run_row = kNone;
    bool first_run = true;
    double acc[VEC];
    float a32[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[q] = 0.0;
      a32[q] = 0.0f;
    }
    for (int k = 0; k < NB; ++k) {
      const int e = e_begin + k * kU;
      __syncwarp();  // every lane is done with the slot about to be refilled
      issue(k + kPfRingD - 1);
      pf_wait<kPfRingD - 1>();
      __syncwarp();  // batch k (copied by several lanes) is visible
      const uint32_t* slot = my_ring + (k % kPfRingD) * S::kSlotW + gw * kU;
      uint32_t rr[kU], ix[NM1][kU];
      float vv[kU];
      ld_batch<kU>(slot, rr);
      ld_batch<kU>(slot + P * kU, reinterpret_cast<uint32_t(&)[kU]>(vv));
#pragma unroll
      for (int j = 0; j < NM1; ++j) ld_batch<kU>(slot + (2 + j) * P * kU, ix[j]);
      const bool full = e + kU <= e_end;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (e + u >= e_end) rr[u] = kNone;
      float f[kU][NM1][VEC];
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < NM1; ++j)
          Vec<VEC>::load(reinterpret_cast<const float*>(fbase[j] + (size_t)ix[j][u] * rstride),
                         f[u][j]);
      float prod[kU][VEC];
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          float t = vv[u];
#pragma unroll
          for (int j = 0; j < NM1; ++j) t = __fmul_rn(t, f[u][j][q]);
          prod[u][q] = t;
        }
      bool same = full && rr[0] == run_row;
#pragma unroll
      for (int u = 1; u < kU; ++u) same = same && rr[u] == run_row;
      if (same) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          float s = prod[0][q];
#pragma unroll
          for (int u = 1; u < kU; ++u) s += prod[u][q];
          acc[q] += (double)s;
        }
        continue;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (rr[u] == kNone) continue;
        const uint32_t row = rr[u];
        if (row == run_row) {
#pragma unroll
          for (int q = 0; q < VEC; ++q) a32[q] += prod[u][q];
        } else {
          if (run_row != kNone) {
            if (row < run_row && gl == 0) atomicMin(p.err + 2, (unsigned long long)(t0 + e + u));
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] += (double)a32[q];
            if (first_run) {
              if (gl == 0) my_grow[2 * gw] = run_row;
#pragma unroll
              for (int q = 0; q < VEC; ++q) my_gslot[(2 * gw) * CB + lcol + q] = acc[q];
              first_run = false;
            } else if (col_ok) {
              float o[VEC];
#pragma unroll
              for (int q = 0; q < VEC; ++q) o[q] = (float)acc[q];
              Vec<VEC>::store(p.out + (size_t)run_row * p.R + col, o);
            }
            if (row > run_row + 1) zero_rows<VEC>(p.out, run_row + 1, row, p.R, col, col_ok);
          }
          run_row = row;
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            acc[q] = 0.0;
            a32[q] = prod[u][q];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        acc[q] += (double)a32[q];
        a32[q] = 0.0f;
      }
    }
    if (run_row != kNone) {
      const int sl = 2 * gw + (first_run ? 0 : 1);
      if (gl == 0) my_grow[sl] = run_row;
#pragma unroll
      for (int q = 0; q < VEC; ++q) my_gslot[sl * CB + lcol + q] = acc[q];
    }
    __syncwarp();
    // ---- warp fold of the P groups (as mttkrp_seg_kernel)
    uint32_t w_cur = kNone, h_row = kNone;
    int cur_g = -1;
    double w_acc[VEC], h_acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) w_acc[q] = h_acc[q] = 0.0;
    const bool writer = gw == 0 && col_ok;
#pragma unroll 1
    for (int g = 0; g < P; ++g) {
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int sl = 2 * g + it;
        const uint32_t row = my_grow[sl];
        if (row == kNone) continue;
        double v[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) v[q] = my_gslot[sl * CB + lcol + q];
        if (row == w_cur) {
#pragma unroll
          for (int q = 0; q < VEC; ++q) w_acc[q] += v[q];
        } else {
          if (w_cur != kNone) {
            if (h_row == kNone) {
              h_row = w_cur;
#pragma unroll
              for (int q = 0; q < VEC; ++q) h_acc[q] = w_acc[q];
            } else if (writer) {
              float o[VEC];
#pragma unroll
              for (int q = 0; q < VEC; ++q) o[q] = (float)w_acc[q];
              Vec<VEC>::store(p.out + (size_t)w_cur * p.R + col, o);
            }
            if (g != cur_g && row > w_cur + 1 && writer)
              zero_rows<VEC>(p.out, w_cur + 1, row, p.R, col, true);
          }
          w_cur = row;
#pragma unroll
          for (int q = 0; q < VEC; ++q) w_acc[q] = v[q];
        }
        cur_g = g;
      }
    }
    uint32_t t_row = kNone;
    if (h_row == kNone) {
      h_row = w_cur;
#pragma unroll
      for (int q = 0; q < VEC; ++q) h_acc[q] = w_acc[q];
    } else {
      t_row = w_cur;
    }
    // ---- hand the warp's first/last-row partials to the fold warp
    const int cb = i % kPfCBuf;
    if (i >= kPfCBuf) spt::mbar_wait(cempty + cb, ((i / kPfCBuf) - 1) & 1u);
    double* cs = s_cslot + (size_t)cb * NSL * CB;
    if (gw == 0) {
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        cs[(2 * warp) * CB + lcol + q] = h_acc[q];
        cs[(2 * warp + 1) * CB + lcol + q] = w_acc[q];
      }
    }
    if (lane == 0) {
      s_crow[cb][2 * warp] = h_row;
      s_crow[cb][2 * warp + 1] = t_row;
    }
    spt::mbar_arrive(cfull + cb);
  }
  pf_wait<0>();
}

// ---------------------------------------------------------------------------
// Warp-tile variant of the segmented MTTKRP: every warp is an independent
// tile of kWT consecutive entries with its own shared-memory slice, its own
// head/tail partials and its own decoupled look-back -- no CTA barrier, so a
// warp that meets many short (Zipf) rows never stalls the other seven, and the
// CTA-level fold disappears. A CTA draws one ticket for its 8 consecutive warp
// tiles, so predecessors are always resident.
#ifndef SPT_MTTKRP_WT
#define SPT_MTTKRP_WT 256
#endif
constexpr int kWT = SPT_MTTKRP_WT;
// warp tiles in launch order (blockIdx) instead of in-order tickets
#ifndef SPT_WT_BID
#define SPT_WT_BID 1
#endif
constexpr int kWTP = kWT + kWT / 8;  // padded (sw layout)

// TTM output index tuples of fiber `row` (head entry h) for NCOL columns at
// col, head indices from the warp's staged copy when h lies in its tile.
// NT > 0: the order is a compile-time constant (unrolled, the mode test is a
// select); NT = 0: any order.
template <int NCOL, int NT>
__device__ __forceinline__ void wt_emit_idx(const MttkrpParams& p, uint32_t h, uint32_t row,
                                            uint32_t col, const uint32_t* s_hid, uint64_t t0) {
  const size_t base = (size_t)row * p.R + col;
  const bool staged = h >= t0;
  const int hs = staged ? sw(static_cast<int>(h - t0)) : 0;
  auto put = [&](uint32_t d, const uint32_t (&w)[NCOL]) {
    if constexpr (NCOL == 4) {
      __stcs(reinterpret_cast<uint4*>(p.zidx[d] + base), make_uint4(w[0], w[1], w[2], w[3]));
    } else {
#pragma unroll
      for (int k = 0; k < NCOL; ++k) __stcs(p.zidx[d] + base + k, w[k]);
    }
  };
  if constexpr (NT > 0) {
    const int mode = static_cast<int>(p.mode);
    uint32_t hv[NT];
    if (staged) {
      // head tuple from the warp's staged copy (the usual case)
      const uint32_t* src = s_hid + hs;
#pragma unroll
      for (int d = 0; d < NT; ++d) {
        const int j = d < mode ? d : d - 1;  // position among the non-mode dims
        hv[d] = d == mode ? 0u : src[j * kWTP];
      }
    } else {
#pragma unroll
      for (int d = 0; d < NT; ++d) hv[d] = d == mode ? 0u : p.hidx[d][h];
    }
#pragma unroll
    for (int d = 0; d < NT; ++d) {
      uint32_t w[NCOL];
#pragma unroll
      for (int k = 0; k < NCOL; ++k) w[k] = d == mode ? col + k : hv[d];
      put(d, w);
    }
  } else {
    int j = 0;
    for (uint32_t d = 0; d < p.N; ++d) {
      uint32_t w[NCOL];
      if (d == p.mode) {
#pragma unroll
        for (int k = 0; k < NCOL; ++k) w[k] = col + k;
      } else {
        const uint32_t hv = staged ? s_hid[j * kWTP + hs] : p.hidx[d][h];
        ++j;
#pragma unroll
        for (int k = 0; k < NCOL; ++k) w[k] = hv;
      }
      put(d, w);
    }
  }
}

// per-warp shared-memory slice of the warp-tile kernels
template <int NM1, int G, int VEC, bool FIBER>
__host__ __device__ constexpr size_t wt_slice(uint32_t n_modes) {
  // group slots; TTM adds the staged entries, fiber offsets, head tuples and
  // head flags (MTTKRP reads its entries through L1)
  return (size_t)2 * (32 / G) * G * VEC * sizeof(double) +
         (FIBER ? (size_t)(2 + NM1) * kWTP * 4 + (size_t)(kWTP + 4) * 4 +
                      (size_t)(n_modes - 1) * kWTP * 4 + (kWT + 16)
                : 0);
}

#ifdef SPT_WT_TRACE
__device__ unsigned long long g_wt_trace[16384 * 8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define WT_TR(k) do { if (lane == 0 && tile < 16384) g_wt_trace[tile * 8 + (k)] = gtime(); } while (0)
#else
#define WT_TR(k) do {} while (0)
#endif
#ifndef SPT_WT_MINB
#define SPT_WT_MINB 4
#endif
template <int NM1, int G, int VEC, bool FIBER = false, int NT = 0>
__global__ void __launch_bounds__(kThreads, SPT_WT_MINB) mttkrp_wt_kernel(MttkrpParams p) {
  constexpr int P = 32 / G;
  constexpr int EG = kWT / P;
  constexpr int CB = G * VEC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // per-warp slice: [2P][CB] doubles of group slots, then the staged entries
  // (TTM adds the fiber offsets, the head index tuples and head flags)
  const size_t kSlice = (wt_slice<NM1, G, VEC, FIBER>(p.N) + 15) & ~size_t(15);
  unsigned char* base = smem_raw + warp * kSlice;
  double* s_gslot = reinterpret_cast<double*>(base);
  uint32_t* s_out = reinterpret_cast<uint32_t*>(s_gslot + 2 * P * CB);
  float* s_val = reinterpret_cast<float*>(s_out + kWTP);
  uint32_t* s_oidx = reinterpret_cast<uint32_t*>(s_val + kWTP);
  uint32_t* s_fp = s_oidx + NM1 * kWTP;           // FIBER: [sw(local fiber)] an entry of it
  uint32_t* s_hid = s_fp + (kWTP + 4);             // FIBER: [N-1][kWTP]
  uint8_t* s_hd = reinterpret_cast<uint8_t*>(s_hid + (FIBER ? (p.N - 1) * kWTP : 0));
  __shared__ uint32_t s_ticket;
  __shared__ uint32_t s_grow_all[kWarps][64];
#ifdef SPT_WT_TRACE
  const unsigned long long t_entry = gtime();
#endif

  uint32_t cta_tile;
  if (p.bid_tiles) {
    // every CTA of the grid is resident at once, so predecessors always make
    // progress without in-order tickets
    cta_tile = blockIdx.x;
  } else {
    if (tid == 0) {
      const unsigned long long t = atomicAdd(p.tile_ctr, 1ull);
      if (t == gridDim.x - 1) atomicExch(p.tile_ctr, 0ull);
      s_ticket = static_cast<uint32_t>(t);
    }
    __syncthreads();  // the only CTA barrier
    cta_tile = s_ticket;
  }
  const uint32_t tile = cta_tile * kWarps + warp;
  if (tile >= p.ntiles) return;
  WT_TR(0);
  const uint64_t t0 = (uint64_t)tile * kWT;
  const int cnt = (p.nnz - t0 < (uint64_t)kWT) ? static_cast<int>(p.nnz - t0) : kWT;
  uint32_t* my_grow = s_grow_all[warp];

  // ---- stage. MTTKRP: no shared-memory copy -- each lane touches one 32-byte
  // sector of every entry array (one warp = the tile's 4*32 sectors), so the
  // groups' batch loads below hit L1, and the smem left free goes to L1 for
  // the factor rows. TTM: staged copy (vector loads when full and aligned).
  if constexpr (!FIBER) {
    const uint64_t e8 = t0 + 8u * lane;
    if (e8 < p.nnz) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p.out_idx + e8));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p.val + e8));
#pragma unroll
      for (int j = 0; j < NM1; ++j) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.oidx[j] + e8));
    }
  } else if (cnt == kWT && p.vec_ok) {
#pragma unroll
    for (int r = 0; r < kWT / 128; ++r) {
      const int i = lane + 32 * r;  // uint4 chunk
      if constexpr (!FIBER)
        reinterpret_cast<uint4*>(s_out)[i + (i >> 3)] =
            spt::ld_stream(reinterpret_cast<const uint4*>(p.out_idx + t0) + i);
      reinterpret_cast<uint4*>(s_val)[i + (i >> 3)] =
          spt::ld_stream(reinterpret_cast<const uint4*>(p.val + t0) + i);
#pragma unroll
      for (int j = 0; j < NM1; ++j)
        reinterpret_cast<uint4*>(s_oidx + j * kWTP)[i + (i >> 3)] =
            spt::ld_stream(reinterpret_cast<const uint4*>(p.oidx[j] + t0) + i);
    }
  } else {
    for (int i = lane; i < kWT; i += 32) {
      const bool ok = i < cnt;
      if constexpr (!FIBER) s_out[sw(i)] = ok ? p.out_idx[t0 + i] : 0u;
      s_val[sw(i)] = ok ? p.val[t0 + i] : 0.0f;
#pragma unroll
      for (int j = 0; j < NM1; ++j) s_oidx[j * kWTP + sw(i)] = ok ? p.oidx[j][t0 + i] : 0u;
    }
  }
  // neighbours for the tile-level continuation tests (issued with the staging)
  uint32_t prev_row = kNone, next_row = kNone;
  uint32_t f_lo = 0;
  if constexpr (!FIBER) {
    if (lane == 0 && t0 > 0) prev_row = p.out_idx[t0 - 1];
    if (lane == 1 && t0 + cnt < p.nnz) next_row = p.out_idx[t0 + cnt];
    prev_row = __shfl_sync(0xffffffffu, prev_row, 0);
    next_row = __shfl_sync(0xffffffffu, next_row, 1);
  } else {
    // TTM: rows are fiber ids. Head tuples of the tile's entries and the head
    // flags: a fiber starts where the non-mode tuple changes (x is coalesced
    // and sorted with `mode` last -- build_fiber_index's definition,
    // P/src/tensor.cpp:92-120), compared in registers as the tuples are
    // staged, so no fptr slice sits behind the tile map on the critical path.
    // Each entry's fiber = the tile's first fiber (map) + heads so far.
    f_lo = __ldg(p.tile_fiber + tile);
    const uint64_t t_end = t0 + cnt;
    const uint32_t nhd = p.N - 1;  // non-mode dims
    uint32_t nb = 0;  // lane j: hnm[j][t0 - 1]; lane 16 + j: hnm[j][t_end]
    if (lane < nhd && t0 > 0) nb = p.hnm[lane][t0 - 1];
    if (lane >= 16 && lane - 16 < nhd && t_end < p.nnz) nb = p.hnm[lane - 16][t_end];
    bool vec = cnt == kWT;
    for (uint32_t j = 0; j < nhd; ++j) vec = vec && spt::aligned16(p.hnm[j]);
    bool eq_next = t_end < p.nnz;
    if (vec) {
      constexpr int kR = kWT / 128;  // uint4 chunks per lane: entries 128 r + 4 lane + q
      uint32_t dm[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) dm[r] = 0;
      for (uint32_t j = 0; j < nhd; ++j) {
        uint4 c[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = lane + 32 * r;
          c[r] = spt::ld_stream(reinterpret_cast<const uint4*>(p.hnm[j] + t0) + i);
          reinterpret_cast<uint4*>(s_hid + j * kWTP)[i + (i >> 3)] = c[r];
        }
        const uint32_t pv = __shfl_sync(0xffffffffu, nb, j);
        const uint32_t nv = __shfl_sync(0xffffffffu, nb, 16 + j);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const uint32_t up = __shfl_up_sync(0xffffffffu, c[r].w, 1);
          const uint32_t wrap = __shfl_sync(0xffffffffu, c[r > 0 ? r - 1 : 0].w, 31);
          const uint32_t before = lane ? up : (r == 0 ? pv : wrap);
          dm[r] |= (c[r].x != before ? 1u : 0u) | (c[r].y != c[r].x ? 2u : 0u) |
                   (c[r].z != c[r].y ? 4u : 0u) | (c[r].w != c[r].z ? 8u : 0u);
        }
        eq_next = eq_next && __shfl_sync(0xffffffffu, c[kR - 1].w, 31) == nv;
      }
      if (t0 == 0 && lane == 0) dm[0] |= 1u;  // the tensor's first entry
#pragma unroll
      for (int r = 0; r < kR; ++r)
        reinterpret_cast<uint32_t*>(s_hd)[32 * r + lane] =
            (dm[r] & 1u) | ((dm[r] >> 1) & 1u) << 8 | ((dm[r] >> 2) & 1u) << 16 |
            ((dm[r] >> 3) & 1u) << 24;
    } else {
      for (uint32_t j = 0; j < nhd; ++j)
        for (int i = lane; i < kWT; i += 32) s_hid[j * kWTP + sw(i)] = i < cnt ? p.hnm[j][t0 + i] : 0u;
      __syncwarp();
      for (uint32_t j = 0; j < nhd; ++j) {
        const uint32_t nv = __shfl_sync(0xffffffffu, nb, 16 + j);
        eq_next = eq_next && s_hid[j * kWTP + sw(cnt - 1)] == nv;
      }
      bool first_diff = t0 == 0;
      for (uint32_t j = 0; j < nhd; ++j)
        first_diff = first_diff || s_hid[j * kWTP + sw(0)] != __shfl_sync(0xffffffffu, nb, j);
      for (int e = lane; e < kWT; e += 32) {
        bool h = false;
        if (e == 0) {
          h = first_diff;
        } else if (e < cnt) {
          for (uint32_t j = 0; j < nhd; ++j)
            h = h || s_hid[j * kWTP + sw(e)] != s_hid[j * kWTP + sw(e - 1)];
        }
        s_hd[e] = h ? 1 : 0;
      }
    }
    __syncwarp();
    constexpr int kPer = kWT / 32;
    int nh = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) nh += (lane * kPer + q < cnt && s_hd[lane * kPer + q]) ? 1 : 0;
    int incl = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int head0 = __shfl_sync(0xffffffffu, (int)s_hd[0], 0);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int hc = incl - nh;
    // s_fp[local fiber] = an entry of that fiber in this tile (its head, or
    // entry t0 for the fiber continuing into the tile): any entry carries the
    // fiber's non-mode tuple, which is all the emission reads from it
    if (lane == 0 && !head0) s_fp[sw(0)] = static_cast<uint32_t>(t0);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = lane * kPer + q;
      if (e < cnt && s_hd[e]) {
        ++hc;
        s_fp[sw(hc - head0)] = static_cast<uint32_t>(t0 + e);
      }
      s_out[sw(e)] = e < cnt ? f_lo + (uint32_t)(hc - head0) : 0u;
    }
    const uint32_t last_fiber = f_lo + (uint32_t)(total - head0);
    if (tile > 0) prev_row = head0 ? f_lo - 1 : f_lo;
    if (t_end < p.nnz) next_row = eq_next ? last_fiber : last_fiber + 1;
  }
  __syncwarp();
  WT_TR(1);

  // ---- per-group segmented accumulation (as in mttkrp_seg_kernel)
  const int gw = lane / G, gl = lane % G;
  const uint32_t lcol = gl * VEC;
  const bool col_ok = lcol < p.ncols;
  const uint32_t col = p.c0 + lcol;
  const int e_begin = gw * EG;
  const int e_end = min(e_begin + EG, cnt);
  if (gl == 0) {
    my_grow[2 * gw] = kNone;
    my_grow[2 * gw + 1] = kNone;
  }
  uint32_t run_row = kNone;
  bool first_run = true;
  double acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = 0.0;
  const char* fbase[NM1];
#pragma unroll
  for (int j = 0; j < NM1; ++j)
    fbase[j] = reinterpret_cast<const char*>(p.ofac[j] + (col_ok ? col : p.c0));
  const uint32_t rstride = p.R * 4u;
  constexpr int kU = (NM1 * VEC <= 12) ? 4 : 2;
  for (int e = e_begin; e < e_end; e += kU) {
    uint32_t rr[kU], ix[NM1][kU];
    float vv[kU];
    const bool full = e + kU <= e_end;
    if constexpr (!FIBER) {
      if (full && p.vec_ok) {
        ld_batch<kU>(p.out_idx + t0 + e, rr);
        ld_batch<kU>(reinterpret_cast<const uint32_t*>(p.val) + t0 + e,
                     reinterpret_cast<uint32_t(&)[kU]>(vv));
#pragma unroll
        for (int j = 0; j < NM1; ++j) ld_batch<kU>(p.oidx[j] + t0 + e, ix[j]);
      } else {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const bool ok = e + u < e_end;
          const uint64_t m = t0 + e + u;
          rr[u] = ok ? p.out_idx[m] : 0u;
          vv[u] = ok ? p.val[m] : 0.0f;
#pragma unroll
          for (int j = 0; j < NM1; ++j) ix[j][u] = ok ? p.oidx[j][m] : 0u;
        }
      }
    } else {
      ld_batch<kU>(s_out + sw(e), rr);
      ld_batch<kU>(reinterpret_cast<const uint32_t*>(s_val) + sw(e),
                   reinterpret_cast<uint32_t(&)[kU]>(vv));
#pragma unroll
      for (int j = 0; j < NM1; ++j) ld_batch<kU>(s_oidx + j * kWTP + sw(e), ix[j]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e + u >= e_end) rr[u] = kNone;
    float f[kU][NM1][VEC];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int j = 0; j < NM1; ++j)
        Vec<VEC>::load(reinterpret_cast<const float*>(fbase[j] + (size_t)ix[j][u] * rstride),
                       f[u][j]);
    float prod[kU][VEC];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float t = vv[u];  // row[r] = val; row[r] *= f_d[r] for d ascending
#pragma unroll
        for (int j = 0; j < NM1; ++j) t = __fmul_rn(t, f[u][j][k]);
        prod[u][k] = t;
      }
    bool same = full && rr[0] == run_row;
#pragma unroll
    for (int u = 1; u < kU; ++u) same = same && rr[u] == run_row;
    if (same) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        float s = prod[0][k];
#pragma unroll
        for (int u = 1; u < kU; ++u) s += prod[u][k];
        acc[k] += (double)s;
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (rr[u] == kNone) continue;
      const uint32_t row = rr[u];
      if (row == run_row) {
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[k] += (double)prod[u][k];
        continue;
      }
      if (run_row != kNone) {
        // fiber ids increase by construction (TTM): only MTTKRP checks its input
        if (!FIBER && row < run_row && gl == 0)
          atomicMin(p.err + 2, (unsigned long long)(t0 + e + u));
        if (first_run) {
          if (gl == 0) my_grow[2 * gw] = run_row;
#pragma unroll
          for (int k = 0; k < VEC; ++k) s_gslot[(2 * gw) * CB + lcol + k] = acc[k];
          first_run = false;
        } else if (col_ok) {
          float o[VEC];
#pragma unroll
          for (int k = 0; k < VEC; ++k) o[k] = (float)acc[k];
          Vec<VEC>::store(p.out + (size_t)run_row * p.R + col, o);
        }
        // TTM rows are consecutive fibers: no gaps to zero
        if (!FIBER && row > run_row + 1) zero_rows<VEC>(p.out, run_row + 1, row, p.R, col, col_ok);
      }
      run_row = row;
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] = (double)prod[u][k];
    }
  }
  if (run_row != kNone) {
    const int sl = 2 * gw + (first_run ? 0 : 1);
    if (gl == 0) my_grow[sl] = run_row;
#pragma unroll
    for (int k = 0; k < VEC; ++k) s_gslot[sl * CB + lcol + k] = acc[k];
  }
  __syncwarp();
  WT_TR(2);

  // ---- warp fold over the P groups' boundary runs -> tile head / tail
  uint32_t w_cur = kNone, h_row = kNone;
  int cur_g = -1;
  double w_acc[VEC], h_acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) w_acc[k] = h_acc[k] = 0.0;
  const bool writer = gw == 0 && col_ok;
#pragma unroll 1
  for (int g = 0; g < P; ++g) {
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int sl = 2 * g + it;
      const uint32_t row = my_grow[sl];
      if (row == kNone) continue;
      double v[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) v[k] = s_gslot[sl * CB + lcol + k];
      if (row == w_cur) {
#pragma unroll
        for (int k = 0; k < VEC; ++k) w_acc[k] += v[k];
      } else {
        if (w_cur != kNone) {
          if (h_row == kNone) {
            h_row = w_cur;
#pragma unroll
            for (int k = 0; k < VEC; ++k) h_acc[k] = w_acc[k];
          } else if (writer) {
            float o[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k) o[k] = (float)w_acc[k];
            Vec<VEC>::store(p.out + (size_t)w_cur * p.R + col, o);
          }
          if (!FIBER && g != cur_g && row > w_cur + 1 && writer)
            zero_rows<VEC>(p.out, w_cur + 1, row, p.R, col, true);
        }
        w_cur = row;
#pragma unroll
        for (int k = 0; k < VEC; ++k) w_acc[k] = v[k];
      }
      cur_g = g;
    }
  }
  // tile head = h (or the only segment), tail = w_cur
  const bool boundary = h_row != kNone;
  const uint32_t head_row = boundary ? h_row : w_cur;
  const uint32_t tail_row = w_cur;
  double head_acc[VEC], tail_acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    head_acc[k] = boundary ? h_acc[k] : w_acc[k];
    tail_acc[k] = w_acc[k];
  }
  if constexpr (!FIBER) {
    if (prev_row != kNone && prev_row > head_row && lane == 0)
      atomicMin(p.err + 2, (unsigned long long)t0);
    if (next_row != kNone && next_row < tail_row && lane == 0)
      atomicMin(p.err + 2, (unsigned long long)(t0 + cnt));
  }
  const bool cont_prev = prev_row == head_row;
  const bool cont_next = next_row == tail_row;

  // ---- inter-tile zero fill (MTTKRP: rows without entries)
  if (!FIBER && writer) {
    if (tile == 0) zero_rows<VEC>(p.out, 0, head_row, p.R, col, true);
    const uint32_t stop = next_row == kNone ? p.rows : next_row;
    if (tail_row + 1 < stop) zero_rows<VEC>(p.out, tail_row + 1, stop, p.R, col, true);
  }

  WT_TR(3);
  // ---- publish / look-back (warp-level)
  const uint32_t tag = p.epoch << 3;
  if (cont_next) {
    bool inclusive = boundary || !cont_prev;
    double pub[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) pub[k] = boundary ? tail_acc[k] : head_acc[k];
    if (!inclusive) {
      // Inside a row spanning many tiles: if the predecessor already holds its
      // inclusive prefix, extend it (no waiting) so the row's end tile finds a
      // P within a few tiles instead of walking the whole row.
      uint32_t s = lane == 0 ? spt::ld_relaxed(p.status + tile - 1) : 0u;
      s = __shfl_sync(0xffffffffu, s, 0);
      if ((s >> 3) == p.epoch && (s & 3u) == kFlagP) {
        __threadfence();
        const double* prev = p.payP + (size_t)(tile - 1) * CB + lcol;
#pragma unroll
        for (int k = 0; k < VEC; ++k) pub[k] += spt::ld_cg(prev + k);
        inclusive = true;
      }
    }
    double* pay = (inclusive ? p.payP : p.payA) + (size_t)tile * CB;
    if (gw == 0) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) pay[lcol + k] = pub[k];
      spt::fence_release();
    }
    __syncwarp();
    if (lane == 0) spt::st_release(p.status + tile, tag | (inclusive ? kFlagP : kFlagA));
  }
  double carry[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) carry[k] = 0.0;
  if (cont_prev && (boundary || !cont_next)) {
    const uint32_t n = spt::lookback_chain(p.status, tile, p.epoch);
    // group g sums chain entries q = 1 + g, 1 + g + P, ...; then fold the groups
    for (uint32_t q = 1 + gw; q <= n && q <= tile; q += P) {
      const double* pay = (q == n ? p.payP : p.payA) + (size_t)(tile - q) * CB + lcol;
#pragma unroll
      for (int k = 0; k < VEC; ++k) carry[k] += spt::ld_cg(pay + k);
    }
#pragma unroll
    for (int o = G; o < 32; o <<= 1)
#pragma unroll
      for (int k = 0; k < VEC; ++k) carry[k] += __shfl_xor_sync(0xffffffffu, carry[k], o);
  }

  WT_TR(4);
  // ---- rows completed by this tile
  if (writer) {
    if (boundary || !cont_next) {
      float o[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) o[k] = (float)(carry[k] + head_acc[k]);
      Vec<VEC>::store(p.out + (size_t)head_row * p.R + col, o);
    }
    if (boundary && !cont_next) {
      float o[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) o[k] = (float)tail_acc[k];
      Vec<VEC>::store(p.out + (size_t)tail_row * p.R + col, o);
    }
  }
  if constexpr (FIBER) {
    // TTM output index rows of every fiber completed in this tile, written by
    // the whole warp at the end: consecutive lanes cover consecutive
    // (fiber, column-vector) pairs, so each store instruction fills 512
    // contiguous bytes (full lines) instead of 8 scattered 64-byte pieces.
    const bool head_done = boundary || !cont_next;
    const bool tail_done = boundary ? !cont_next : head_done;
    const uint32_t fa = head_done ? head_row : head_row + 1;
    const uint32_t fb = tail_done ? tail_row + 1 : tail_row;  // exclusive
    const uint32_t per = p.ncols / VEC;  // column vectors per fiber
    const uint32_t total = fb > fa ? (fb - fa) * per : 0u;
    for (uint32_t c = lane; c < total; c += 32) {
      const uint32_t f = fa + c / per, k0 = (c % per) * VEC;
      wt_emit_idx<VEC, NT>(p, s_fp[sw(static_cast<int>(f - f_lo))], f, p.c0 + k0, s_hid, t0);
    }
  }
  WT_TR(5);
#ifdef SPT_WT_TRACE
  if (lane == 0 && tile < 16384) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    g_wt_trace[tile * 8 + 6] = sm;
    g_wt_trace[tile * 8 + 7] = t_entry;
  }
#endif
}

template <int G, int VEC>
size_t wt_smem(int nm1) {
  (void)nm1;
  return (size_t)kWarps * ((size_t)2 * (32 / G) * G * VEC * sizeof(double));
}

using KernelFnT = void (*)(MttkrpParams);

template <int G, int VEC>
KernelFnT pick_wt(int nm1) {
  switch (nm1) {
    case 1: return mttkrp_wt_kernel<1, G, VEC>;
    case 2: return mttkrp_wt_kernel<2, G, VEC>;
    case 3: return mttkrp_wt_kernel<3, G, VEC>;
    case 4: return mttkrp_wt_kernel<4, G, VEC>;
    case 5: return mttkrp_wt_kernel<5, G, VEC>;
    case 6: return mttkrp_wt_kernel<6, G, VEC>;
    default: return mttkrp_wt_kernel<7, G, VEC>;
  }
}

template <int NM1, int G, int VEC>
__global__ void __launch_bounds__(kThreads) mttkrp_atomic_kernel(MttkrpParams p) {
  constexpr int P = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const uint32_t lcol = gl * VEC;
  if (lcol >= p.ncols) return;
  const uint32_t col = p.c0 + lcol;
  const uint64_t gid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / G;
  const uint64_t ngroups = (uint64_t)gridDim.x * blockDim.x / G;
  (void)P;
  for (uint64_t m = gid; m < p.nnz; m += ngroups) {
    float f[NM1][VEC];
#pragma unroll
    for (int j = 0; j < NM1; ++j) Vec<VEC>::load(p.ofac[j] + (size_t)p.oidx[j][m] * p.R + col, f[j]);
    const float v = p.val[m];
    float* o = p.out + (size_t)p.out_idx[m] * p.R + col;
    float t[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      t[k] = v;
#pragma unroll
      for (int j = 0; j < NM1; ++j) t[k] = __fmul_rn(t[k], f[j][k]);
    }
    if constexpr (VEC == 4) {
      atomicAdd(reinterpret_cast<float4*>(o), make_float4(t[0], t[1], t[2], t[3]));
    } else {
#pragma unroll
      for (int k = 0; k < VEC; ++k) atomicAdd(o + k, t[k]);
    }
  }
}

template <int G, int VEC>
size_t seg_smem(int nm1) {
  constexpr int GROUPS = kWarps * (32 / G);
  constexpr int CB = G * VEC;
  return (size_t)2 * kWarps * CB * sizeof(double) + (size_t)kTileP * (2 + nm1) * sizeof(uint32_t) +
         (size_t)2 * GROUPS * CB * sizeof(double);
}

// TTM: same kernel with fiber rows and one "other" mode (the contracted one).
template <int G, int VEC>
size_t ttm_smem() {
  return seg_smem<G, VEC>(1) + (size_t)(kTile + 4) * sizeof(uint32_t);
}

using KernelFn = void (*)(MttkrpParams);

template <int G, int VEC>
KernelFn pick_seg(int nm1) {
  switch (nm1) {
    case 1: return mttkrp_seg_kernel<1, G, VEC, false>;
    case 2: return mttkrp_seg_kernel<2, G, VEC, false>;
    case 3: return mttkrp_seg_kernel<3, G, VEC, false>;
    case 4: return mttkrp_seg_kernel<4, G, VEC, false>;
    case 5: return mttkrp_seg_kernel<5, G, VEC, false>;
    case 6: return mttkrp_seg_kernel<6, G, VEC, false>;
    default: return mttkrp_seg_kernel<7, G, VEC, false>;
  }
}

template <int G, int VEC>
KernelFn pick_atomic(int nm1) {
  switch (nm1) {
    case 1: return mttkrp_atomic_kernel<1, G, VEC>;
    case 2: return mttkrp_atomic_kernel<2, G, VEC>;
    case 3: return mttkrp_atomic_kernel<3, G, VEC>;
    case 4: return mttkrp_atomic_kernel<4, G, VEC>;
    case 5: return mttkrp_atomic_kernel<5, G, VEC>;
    case 6: return mttkrp_atomic_kernel<6, G, VEC>;
    default: return mttkrp_atomic_kernel<7, G, VEC>;
  }
}

using KernelFnP = void (*)(MttkrpParams, uint32_t);
struct PfVariant {
  KernelFnP fn;
  size_t smem;
};
template <int G, int VEC>
PfVariant pick_pf(int nm1) {
  switch (nm1) {
#define SPT_PF_CASE(n) \
  case n: return {mttkrp_pf_kernel<n, G, VEC>, PfShape<n, G, VEC>::smem};
    SPT_PF_CASE(1)
    SPT_PF_CASE(2)
    SPT_PF_CASE(3)
    SPT_PF_CASE(4)
    SPT_PF_CASE(5)
    SPT_PF_CASE(6)
#undef SPT_PF_CASE
    default: return {mttkrp_pf_kernel<7, G, VEC>, PfShape<7, G, VEC>::smem};
  }
}
PfVariant choose_pf(int G, int VEC, int nm1) {
  if (VEC == 4) {
    switch (G) {
      case 2: return pick_pf<2, 4>(nm1);
      case 4: return pick_pf<4, 4>(nm1);
      case 8: return pick_pf<8, 4>(nm1);
      case 16: return pick_pf<16, 4>(nm1);
      default: return pick_pf<32, 4>(nm1);
    }
  }
  return pick_pf<32, 1>(nm1);
}

struct Variant {
  int G, VEC;
  KernelFn seg, atomic;
  size_t smem;
};

KernelFnT choose_wt(int G, int VEC, int nm1, size_t* smem) {
  if (VEC == 4) {
    switch (G) {
      case 2: *smem = wt_smem<2, 4>(nm1); return pick_wt<2, 4>(nm1);
      case 4: *smem = wt_smem<4, 4>(nm1); return pick_wt<4, 4>(nm1);
      case 8: *smem = wt_smem<8, 4>(nm1); return pick_wt<8, 4>(nm1);
      case 16: *smem = wt_smem<16, 4>(nm1); return pick_wt<16, 4>(nm1);
      default: *smem = wt_smem<32, 4>(nm1); return pick_wt<32, 4>(nm1);
    }
  }
  *smem = wt_smem<32, 1>(nm1);
  return pick_wt<32, 1>(nm1);
}

// Column blocking: float4 lanes when R % 4 == 0 (G = smallest power of two
// with G*4 >= R, at most 32 -> 128 columns per launch), scalar lanes otherwise
// (32 columns per launch).
Variant choose_variant(uint32_t R, int nm1) {
  if (R % 4 == 0) {
    const uint32_t q = R / 4;
    if (q <= 2) return {2, 4, pick_seg<2, 4>(nm1), pick_atomic<2, 4>(nm1), seg_smem<2, 4>(nm1)};
    if (q <= 4) return {4, 4, pick_seg<4, 4>(nm1), pick_atomic<4, 4>(nm1), seg_smem<4, 4>(nm1)};
    if (q <= 8) return {8, 4, pick_seg<8, 4>(nm1), pick_atomic<8, 4>(nm1), seg_smem<8, 4>(nm1)};
    if (q <= 16)
      return {16, 4, pick_seg<16, 4>(nm1), pick_atomic<16, 4>(nm1), seg_smem<16, 4>(nm1)};
    return {32, 4, pick_seg<32, 4>(nm1), pick_atomic<32, 4>(nm1), seg_smem<32, 4>(nm1)};
  }
  return {32, 1, pick_seg<32, 1>(nm1), pick_atomic<32, 1>(nm1), seg_smem<32, 1>(nm1)};
}

struct TtmVariant {
  int G, VEC;
  KernelFn fn;
  size_t smem;
  KernelFn wt;  // warp-tile TTM (same G/VEC)
};

template <int G, int VEC>
KernelFn pick_ttm_wt(uint32_t N) {
  switch (N) {
    case 3: return mttkrp_wt_kernel<1, G, VEC, true, 3>;
    case 4: return mttkrp_wt_kernel<1, G, VEC, true, 4>;
    default: return mttkrp_wt_kernel<1, G, VEC, true>;
  }
}

TtmVariant choose_ttm(uint32_t R, bool aligned, uint32_t N) {
#define SPT_TTM_V(g, v) \
  { g, v, mttkrp_seg_kernel<1, g, v, true>, ttm_smem<g, v>(), pick_ttm_wt<g, v>(N) }
  if (R % 4 == 0 && aligned) {
    const uint32_t q = R / 4;
    if (q <= 2) return SPT_TTM_V(2, 4);
    if (q <= 4) return SPT_TTM_V(4, 4);
    if (q <= 8) return SPT_TTM_V(8, 4);
    if (q <= 16) return SPT_TTM_V(16, 4);
    return SPT_TTM_V(32, 4);
  }
  return SPT_TTM_V(32, 1);
#undef SPT_TTM_V
}

size_t ttm_wt_smem(int G, int VEC, uint32_t n_modes) {
  const auto slice = [&](size_t s) { return (s + 15) & ~size_t(15); };
  switch (VEC * 100 + G) {
    case 402: return kWarps * slice(wt_slice<1, 2, 4, true>(n_modes));
    case 404: return kWarps * slice(wt_slice<1, 4, 4, true>(n_modes));
    case 408: return kWarps * slice(wt_slice<1, 8, 4, true>(n_modes));
    case 416: return kWarps * slice(wt_slice<1, 16, 4, true>(n_modes));
    case 432: return kWarps * slice(wt_slice<1, 32, 4, true>(n_modes));
    default: return kWarps * slice(wt_slice<1, 32, 1, true>(n_modes));
  }
}

}  // namespace

namespace spt {
int build_tile_fiber_map(spt_ctx* ctx, const uint32_t* d_fptr, uint32_t nfibs, uint32_t tile,
                         uint32_t ntiles, uint32_t* d_map, cudaStream_t st);
int check_fiber_inputs(const spt_coo* x, uint32_t mode, const uint32_t* d_fptr, uint64_t nfibs,
                       const char* k);
}  // namespace spt

// K7 TTM (P/src/kernels_seq.cpp:108-151, P/src/kernels_par.cpp:224-273,
// ttm_fiber P/src/kernel_detail.hpp:132-140): the segmented kernel above with
// output rows = fibers of x (sorted with `mode` last), the contracted mode's
// index gathering rows of U, and an epilogue that writes the R output entries
// of each fiber (value row + N index rows) with vector stores. Tensor cores are
// deliberately not used: the op is gather/scatter-bound (1 mul-add per
// 8 bytes gathered), and the output COO write dominates.
extern "C" int spt_ttm_f32(spt_ctx* ctx, const spt_coo* x, const float* d_u, uint64_t u_rows,
                           uint64_t u_cols, uint32_t mode, const uint32_t* d_fptr, uint64_t nfibs,
                           spt_coo* z, unsigned flags, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "ttm: null context");
  SPT_TRY(spt::check_fiber_inputs(x, mode, d_fptr, nfibs, "ttm"));
  if (u_rows != x->dims[mode])
    return spt::set_error(SPT_EINVAL, "ttm: matrix rows must match the mode dimension");
  if (u_cols == 0) return spt::set_error(SPT_EINVAL, "ttm: matrix must have at least one column");
  if (u_cols > 0xFFFFFFFFull || nfibs * u_cols >= (1ull << 32))
    return spt::set_error(SPT_EOVERFLOW, "ttm: output nnz %llu exceeds the u32 device range",
                          (unsigned long long)(nfibs * u_cols));
  if (!z) return spt::set_error(SPT_EINVAL, "ttm: null output");
  const uint32_t N = x->order;
  const uint32_t R = static_cast<uint32_t>(u_cols);
  z->order = N;
  z->nnz = nfibs * R;
  for (uint32_t d = 0; d < SPT_MAX_ORDER; ++d) {
    z->dims[d] = d < N ? (d == mode ? R : x->dims[d]) : 0;
    z->sort_order[d] = x->sort_order[d];
  }
  z->has_sort_order = 1;
  z->coalesced = 1;
  if (nfibs == 0) return SPT_OK;
  for (uint32_t d = 0; d < N; ++d)
    if (!z->idx[d]) return spt::set_error(SPT_EINVAL, "ttm: null output index array");
  if (!z->val || !d_u) return spt::set_error(SPT_EINVAL, "ttm: null matrix or output values");
  cudaStream_t st = spt::as_stream(stream);

  bool aligned = spt::aligned16(d_u) && spt::aligned16(z->val);
  for (uint32_t d = 0; d < N; ++d) aligned = aligned && spt::aligned16(z->idx[d]);
  const TtmVariant v = choose_ttm(R, aligned, N);
  const uint32_t CB = v.G * v.VEC;
#ifndef SPT_TTM_WARP_TILES
#define SPT_TTM_WARP_TILES 1
#endif
  // warp tiles (no CTA barrier) by default; per-CTA tiles kept for A/B
  const bool wt = SPT_TTM_WARP_TILES != 0;
  const uint32_t tile_entries = wt ? kWT : kTile;
  const uint64_t ntiles = (x->nnz + tile_entries - 1) / tile_entries;
  uint32_t* map;
  SPT_TRY(spt::ctx_scratch(ctx, ntiles * sizeof(uint32_t), reinterpret_cast<void**>(&map)));
  SPT_TRY(spt::build_tile_fiber_map(ctx, d_fptr, static_cast<uint32_t>(nfibs), tile_entries,
                                    static_cast<uint32_t>(ntiles), map, st));

  MttkrpParams p{};
  p.oidx[0] = x->idx[mode];
  p.ofac[0] = d_u;
  p.val = x->val;
  p.vec_ok = spt::aligned16(x->idx[mode]) && spt::aligned16(x->val);
  p.out = z->val;
  p.nnz = x->nnz;
  p.rows = static_cast<uint32_t>(nfibs);
  p.R = R;
  p.err = ctx->d_err;
  p.tile_ctr = ctx->d_tile_ctr;
  p.ntiles = static_cast<uint32_t>(ntiles);
  p.fptr = d_fptr;
  p.tile_fiber = map;
  for (uint32_t d = 0, j = 0; d < N; ++d) {
    p.hidx[d] = x->idx[d];
    p.zidx[d] = z->idx[d];
    if (d != mode) p.hnm[j++] = x->idx[d];
  }
  p.N = N;
  p.mode = mode;
  p.bid_tiles = SPT_WT_BID;
  const KernelFn fn = wt ? v.wt : v.fn;
  const size_t smem = wt ? ttm_wt_smem(v.G, v.VEC, N)
                         : v.smem + (size_t)(N - 1) * kTileP * sizeof(uint32_t);
  const unsigned grid = wt ? static_cast<unsigned>((ntiles + kWarps - 1) / kWarps)
                           : static_cast<unsigned>(ntiles);
  SPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  for (uint32_t c0 = 0; c0 < R; c0 += CB) {
    uint32_t epoch;
    SPT_TRY(spt::ctx_lookback(ctx, ntiles, 2 * ntiles * CB, &epoch));
    p.status = ctx->d_status;
    p.payA = ctx->d_payload;
    p.payP = ctx->d_payload + ntiles * CB;
    p.epoch = epoch;
    p.c0 = c0;
    p.ncols = std::min<uint32_t>(CB, R - c0);
    fn<<<grid, kThreads, smem, st>>>(p);
    SPT_LAUNCHED(ctx);
  }
  (void)flags;
  return SPT_OK;
}

namespace spt {
// A mode-leading sorted copy of x (stream-ordered temporaries), then the
// segmented kernel on it.
int mttkrp_sorted_copy(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors,
                       const uint64_t* rows, const uint64_t* cols, uint32_t mode, float* d_out,
                       unsigned flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  const uint32_t N = x->order;
  const size_t ab = ((x->nnz * 4 + 255) / 256) * 256;
  char* mem = nullptr;
  if (spt::tmp_alloc(ctx, reinterpret_cast<void**>(&mem), ab * (N + 1), st) != cudaSuccess) {
    cudaGetLastError();
    return set_error(SPT_ENOMEM, "mttkrp: out of device memory for a sorted copy");
  }
  spt_coo c = *x;
  int s = SPT_OK;
  for (uint32_t d = 0; d < N && s == SPT_OK; ++d) {
    c.idx[d] = reinterpret_cast<uint32_t*>(mem + d * ab);
    if (cudaMemcpyAsync(c.idx[d], x->idx[d], x->nnz * 4, cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
      s = cuda_status(cudaGetLastError(), "mttkrp sorted copy");
  }
  c.val = reinterpret_cast<float*>(mem + N * ab);
  if (s == SPT_OK &&
      cudaMemcpyAsync(c.val, x->val, x->nnz * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    s = cuda_status(cudaGetLastError(), "mttkrp sorted copy");
  uint32_t order[SPT_MAX_ORDER];
  order[0] = mode;
  for (uint32_t d = 0, k = 1; d < N; ++d)
    if (d != mode) order[k++] = d;
  if (s == SPT_OK) s = spt_sort_f32(ctx, &c, order, 0, stream);
  if (s == SPT_OK)
    s = spt_mttkrp_f32(ctx, &c, d_factors, rows, cols, mode, d_out, SPT_MTTKRP_SEGMENTED,
                       flags & ~SPT_FLAG_ASYNC, stream);
  cudaStreamSynchronize(st);
  cudaFreeAsync(mem, st);
  return s;
}
}  // namespace spt

extern "C" int spt_mttkrp_f32(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors,
                              const uint64_t* rows, const uint64_t* cols, uint32_t mode,
                              float* d_out, int strategy, unsigned flags, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "mttkrp: null context");
  SPT_TRY(spt::check_coo(x, "mttkrp"));
  const uint32_t N = x->order;
  // P/src/kernel_detail.hpp:157-173
  if (N < 2) return spt::set_error(SPT_EINVAL, "mttkrp: input must have order >= 2");
  if (mode >= N) return spt::set_error(SPT_EINVAL, "mttkrp: mode out of range");
  if (!x->coalesced) return spt::set_error(SPT_EINVAL, "mttkrp: tensor must be coalesced");
  if (!d_factors || !rows || !cols)
    return spt::set_error(SPT_EINVAL, "mttkrp: need one factor matrix per mode");
  uint64_t R = 0;
  for (uint32_t d = 0; d < N; ++d) {
    if (d == mode) continue;
    if (R == 0) R = cols[d];
    if (cols[d] != R)
      return spt::set_error(SPT_EINVAL, "mttkrp: factor matrices must share the column count");
    if (rows[d] != x->dims[d])
      return spt::set_error(SPT_EINVAL, "mttkrp: factor rows must match the mode dimension");
  }
  if (R == 0) return spt::set_error(SPT_EINVAL, "mttkrp: factor rank must be >= 1");
  if (R > 0xFFFFFFFFull) return spt::set_error(SPT_EOVERFLOW, "mttkrp: rank too large");
  for (uint32_t d = 0; d < N; ++d)
    if (d != mode && !d_factors[d] && x->dims[d] > 0)
      return spt::set_error(SPT_EINVAL, "mttkrp: null factor for mode %u", d);
  const uint32_t I = x->dims[mode];
  if (I > 0 && !d_out) return spt::set_error(SPT_EINVAL, "mttkrp: null output");
  cudaStream_t st = spt::as_stream(stream);
  if (I == 0) return SPT_OK;
  if (x->nnz == 0) {
    SPT_CUDA(cudaMemsetAsync(d_out, 0, (size_t)I * R * sizeof(float), st));
    return SPT_OK;
  }

  const int nm1 = static_cast<int>(N) - 1;
  Variant v = choose_variant(static_cast<uint32_t>(R), nm1);
  bool aligned = true;
  for (uint32_t d = 0; d < N; ++d)
    if (d != mode && !spt::aligned16(d_factors[d])) aligned = false;
  if (!spt::aligned16(d_out)) aligned = false;
  if (v.VEC == 4 && !aligned) v = {32, 1, pick_seg<32, 1>(nm1), pick_atomic<32, 1>(nm1), seg_smem<32, 1>(nm1)};
  const uint32_t CB = v.G * v.VEC;

  if (strategy == SPT_MTTKRP_AUTO) {
    if (x->has_sort_order && static_cast<uint32_t>(x->sort_order[0]) == mode) {
      strategy = SPT_MTTKRP_SEGMENTED;
    } else {
      // Any order, like seq::mttkrp (P/src/kernels_seq.cpp:153-174), on the
      // 1e-5 contract: a temporary plan (a mode-leading copy, R % 16 == 0) or
      // a mode-leading sorted copy for the segmented kernel. fp32 atomics only
      // when the caller asks for MTTKRP_ATOMIC.
      if (spt::plan_supported(x, R) && aligned) {
        spt_mttkrp_plan* pl = nullptr;
        SPT_TRY(spt_mttkrp_plan_create(ctx, x, mode, R, SPT_PLAN_NO_HOT, &pl, stream));
        const int s = spt_mttkrp_plan_exec(ctx, pl, d_factors, rows, cols, d_out, 0, stream);
        spt_mttkrp_plan_destroy(pl);
        return s;
      }
      return spt::mttkrp_sorted_copy(ctx, x, d_factors, rows, cols, mode, d_out, flags, stream);
    }
  }
  if (strategy < SPT_MTTKRP_SEGMENTED || strategy > SPT_MTTKRP_SEGMENTED_WARP)
    return spt::set_error(SPT_EINVAL, "mttkrp: unknown strategy %d", strategy);
  // The rest (short rows, other ranks, unaligned operands): warp tiles win in
  // the latency-bound small-problem regime (1M nnz: 29 vs 37 us); from ~2M nnz
  // the persistent CTA-tile kernel wins (4M: 82 vs 94 us, C4 shape at 8M: 301
  // vs 528 us).
  // Inputs up to 32M entries whose rows average >= 16 entries: one resident
  // wave, a contiguous share per warp, no tile look-back (mttkrp_ow.cu; C1 24
  // vs 30 us, 10M entries 104 vs 138 us, 10M with Zipf(1.5) rows 114 vs 269).
  if (strategy == SPT_MTTKRP_SEGMENTED && spt::mttkrp_onewave_ok(x, R, d_factors, mode, d_out)) {
    SPT_TRY(spt::mttkrp_onewave(ctx, x, d_factors, mode, static_cast<uint32_t>(R), d_out, st));
    if (flags & SPT_FLAG_ASYNC) return SPT_OK;
    return spt::sync_and_check(ctx, st);
  }
  if (strategy == SPT_MTTKRP_SEGMENTED)
    strategy = x->nnz <= 1500000 ? SPT_MTTKRP_SEGMENTED_WARP : SPT_MTTKRP_SEGMENTED_CTA;

  MttkrpParams p{};
  p.out_idx = x->idx[mode];
  int j = 0;
  for (uint32_t d = 0; d < N; ++d) {
    if (d == mode) continue;
    p.oidx[j] = x->idx[d];
    p.ofac[j] = d_factors[d];
    ++j;
  }
  p.val = x->val;
  p.out = d_out;
  p.nnz = x->nnz;
  p.rows = I;
  p.vec_ok = 1;
  for (uint32_t d = 0; d < N; ++d) p.vec_ok = p.vec_ok && spt::aligned16(x->idx[d]);
  p.vec_ok = p.vec_ok && spt::aligned16(x->val);
  p.R = static_cast<uint32_t>(R);
  p.err = ctx->d_err;
  p.tile_ctr = ctx->d_tile_ctr;

  if (strategy == SPT_MTTKRP_ATOMIC) {
    SPT_CUDA(cudaMemsetAsync(d_out, 0, (size_t)I * R * sizeof(float), st));
    ctx->launches++;
    const unsigned grid = spt::grid_for(x->nnz * v.G, kThreads, ctx->num_sms * 16);
    for (uint32_t c0 = 0; c0 < R; c0 += CB) {
      p.c0 = c0;
      p.ncols = static_cast<uint32_t>(std::min<uint64_t>(CB, R - c0));
      v.atomic<<<grid, kThreads, 0, st>>>(p);
      SPT_LAUNCHED(ctx);
    }
    return SPT_OK;
  }

  if (strategy == SPT_MTTKRP_SEGMENTED_WARP) {
    size_t smem = 0;
    KernelFnT fn = choose_wt(v.G, v.VEC, nm1, &smem);
    const uint64_t ntiles = (x->nnz + kWT - 1) / kWT;
    p.ntiles = static_cast<uint32_t>(ntiles);
    SPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
#ifndef SPT_WT_CARVEOUT
#define SPT_WT_CARVEOUT 40  // ~100 KB smem per SM: 4 CTAs, the rest of the 256 KB is L1
#endif
    SPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  SPT_WT_CARVEOUT));
    const uint64_t grid = (ntiles + kWarps - 1) / kWarps;
    int per_sm = 0;
    if (!SPT_WT_BID)  // tickets unless the grid fits one resident wave
      SPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
    p.bid_tiles = SPT_WT_BID || grid <= (uint64_t)per_sm * ctx->num_sms ? 1 : 0;
    for (uint32_t c0 = 0; c0 < R; c0 += CB) {
      uint32_t epoch;
      SPT_TRY(spt::ctx_lookback(ctx, ntiles, 2 * ntiles * CB, &epoch));
      p.status = ctx->d_status;
      p.payA = ctx->d_payload;
      p.payP = ctx->d_payload + ntiles * CB;
      p.epoch = epoch;
      p.c0 = c0;
      p.ncols = static_cast<uint32_t>(std::min<uint64_t>(CB, R - c0));
      fn<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(p);
      SPT_LAUNCHED(ctx);
    }
    if (flags & SPT_FLAG_ASYNC) return SPT_OK;
    return spt::sync_and_check(ctx, st);
  }
  const uint64_t ntiles = (x->nnz + kTile - 1) / kTile;
  p.ntiles = static_cast<uint32_t>(ntiles);
#ifndef SPT_MTTKRP_PF
#define SPT_MTTKRP_PF 1
#endif
  // Persistent CTAs with the asynchronous tile fold win up to a few 10M nnz
  // (10M uniform: 160 vs 209 us; C4 shape at 20M: 615 vs 655 us). At 100M+
  // with Zipf rows spanning thousands of tiles, the one fold warp that sums
  // such a row's chain stalls its CTA (and the tickets it holds); the
  // per-CTA kernel, which sums chains with all 256 threads, is faster there
  // (C4 mode 3 at 100M: 2.71 vs 3.12 ms).
#ifndef SPT_PF_MAX_NNZ
#define SPT_PF_MAX_NNZ (32ull << 20)
#endif
  if (SPT_MTTKRP_PF && p.vec_ok && x->nnz <= SPT_PF_MAX_NNZ) {
    const PfVariant pv = choose_pf(v.G, v.VEC, nm1);
    SPT_CUDA(cudaFuncSetAttribute(pv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(pv.smem)));
    int per_sm = 0;
    SPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pv.fn, kPfThreads, pv.smem));
    const uint32_t nctas = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(ntiles, (uint64_t)std::max(per_sm, 1) * ctx->num_sms)));
    for (uint32_t c0 = 0; c0 < R; c0 += CB) {
      uint32_t epoch;
      SPT_TRY(spt::ctx_lookback(ctx, ntiles, 2 * ntiles * CB, &epoch));
      p.status = ctx->d_status;
      p.payA = ctx->d_payload;
      p.payP = ctx->d_payload + ntiles * CB;
      p.epoch = epoch;
      p.c0 = c0;
      p.ncols = static_cast<uint32_t>(std::min<uint64_t>(CB, R - c0));
      pv.fn<<<nctas, kPfThreads, pv.smem, st>>>(p, nctas);
      SPT_LAUNCHED(ctx);
    }
    if (flags & SPT_FLAG_ASYNC) return SPT_OK;
    return spt::sync_and_check(ctx, st);
  }
  SPT_CUDA(cudaFuncSetAttribute(v.seg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(v.smem)));
  for (uint32_t c0 = 0; c0 < R; c0 += CB) {
    uint32_t epoch;
    SPT_TRY(spt::ctx_lookback(ctx, ntiles, 2 * ntiles * CB, &epoch));
    p.status = ctx->d_status;
    p.payA = ctx->d_payload;
    p.payP = ctx->d_payload + ntiles * CB;
    p.epoch = epoch;
    p.c0 = c0;
    p.ncols = static_cast<uint32_t>(std::min<uint64_t>(CB, R - c0));
    v.seg<<<static_cast<unsigned>(ntiles), kThreads, v.smem, st>>>(p);
    SPT_LAUNCHED(ctx);
  }
  if (flags & SPT_FLAG_ASYNC) return SPT_OK;
  return spt::sync_and_check(ctx, st);
}

#ifdef SPT_WT_TRACE
extern "C" __attribute__((visibility("default"))) int spt_debug_wt_trace(void* dst) {
  return cudaMemcpyFromSymbol(dst, g_wt_trace, sizeof(g_wt_trace)) == cudaSuccess ? 0 : 5;
}
#endif
