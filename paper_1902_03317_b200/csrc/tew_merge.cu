// K3 TEW: general elementwise op of two coalesced tensors by sorted merge.
//
// Reference: seq::tew P/src/kernels_seq.cpp:41-53, merge_range
// P/src/kernel_detail.hpp:47-84 (matched -> op(x, y); unmatched x -> x for
// add/sub; unmatched y -> y (add) or -y (sub); mul keeps matches only),
// tew_output_dims :97-102, par::tew P/src/kernels_par.cpp:144-177.
//
// One pass, no host round trip:
//   * a partition kernel places every 2048-item tile boundary on the merge
//     path of x and y (binary search on the diagonal; ties take x first, so
//     a matched pair is always "x then y" and each tuple is emitted once);
//   * a CTA stages its x and y key runs (N u32 arrays each, permuted into sort
//     order) in shared memory, each thread merges 8 items serially, decides
//     what it emits, counts, and the CTA gets its global output offset from a
//     block scan plus a decoupled look-back over 64-bit epoch-tagged tile
//     counts; then every thread scatters its entries (tuple + value, one IEEE
//     op, bit-identical to the reference).
// The merge order equals the reference's two-pointer merge order, so the
// output is entry-for-entry identical to seq::tew's.
#include <cub/cub.cuh>

#include <algorithm>

#include "internal.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kIPT = 8;
constexpr int kTile = kThreads * kIPT;
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
};

template <int N>
__device__ __forceinline__ int cmp_g(const MergeParams& p, uint64_t i, uint64_t j) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t a = p.xi[k][i], b = p.yi[k][j];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

// Tile boundaries on the merge path (x-first on ties).
template <int N>
__global__ void partition_kernel(MergeParams p, uint32_t* split) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > p.ntiles) return;
  const uint64_t total = p.nx + p.ny;
  const uint64_t diag = std::min<uint64_t>((uint64_t)t * kTile, total);
  uint64_t lo = diag > p.ny ? diag - p.ny : 0;
  uint64_t hi = std::min<uint64_t>(diag, p.nx);
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    // take x[mid] before y[diag-1-mid] iff x[mid] <= y[diag-1-mid]
    if (cmp_g<N>(p, mid, diag - 1 - mid) <= 0) lo = mid + 1;
    else hi = mid;
  }
  split[t] = static_cast<uint32_t>(lo);
}

template <int N>
__device__ __forceinline__ int cmp_s(const uint32_t* sx, int i, const uint32_t* sy, int j) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t a = sx[k * kTile + i], b = sy[k * kTile + j];
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
  uint32_t* sx = smem;              // [N][kTile]
  uint32_t* sy = smem + N * kTile;  // [N][kTile]
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
  for (int i = tid; i < nxt; i += kThreads)
#pragma unroll
    for (int k = 0; k < N; ++k) sx[k * kTile + i] = p.xi[k][a0 + i];
  for (int j = tid; j < nyt; j += kThreads)
#pragma unroll
    for (int k = 0; k < N; ++k) sy[k * kTile + j] = p.yi[k][b0 + j];
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

  // Decoupled look-back over tile counts: word = epoch<<34 | flag<<32 | count.
  if (tid == 0) {
    const unsigned long long tag = (unsigned long long)p.epoch << 34;
    unsigned long long base = 0;
    if (tile == 0) {
      spt::st_release64(p.status + tile, tag | (kFlagP << 32) | tile_total);
    } else {
      spt::st_release64(p.status + tile, tag | (kFlagA << 32) | tile_total);
      uint32_t t = tile - 1;
      while (true) {
        unsigned long long w;
        do {
          w = spt::ld_acquire64(p.status + t);
        } while ((w >> 34) != p.epoch || ((w >> 32) & 3ull) == 0);
        base += w & 0xFFFFFFFFull;
        if (((w >> 32) & 3ull) == kFlagP || t == 0) break;
        --t;
      }
      spt::st_release64(p.status + tile, tag | (kFlagP << 32) | (base + tile_total));
    }
    s_base = base;
    if (tile == p.ntiles - 1) *p.total = base + tile_total;
  }
  __syncthreads();
  uint64_t pos = s_base + excl;

#pragma unroll
  for (int k = 0; k < kIPT; ++k) {
    if (src[k] == 0) continue;
    const bool m = matched[k];
    if (src[k] == 1) {
      if (p.op == SPT_MUL && !m) continue;
      const uint64_t gx = a0 + li[k];
      float v = __ldg(p.xv + gx);
      if (m) {
        // the matching y is the next y in merge order: global b0 + (#y consumed)
        // recomputed from the tuple position: y index = number of y items before
        // this x item in merge order.
        const uint64_t gy = b0 + (static_cast<uint64_t>(dg + k) - li[k]);
        v = apply(p.op, v, __ldg(p.yv + gy));
      }
#pragma unroll
      for (int q = 0; q < N; ++q) p.zi[q][pos] = sx[q * kTile + li[k]];
      p.zv[pos] = v;
      ++pos;
    } else {
      if (p.op == SPT_MUL || m) continue;
      const uint64_t gy = b0 + li[k];
      const float yv = __ldg(p.yv + gy);
#pragma unroll
      for (int q = 0; q < N; ++q) p.zi[q][pos] = sy[q * kTile + li[k]];
      p.zv[pos] = p.op == SPT_SUB ? -yv : yv;
      ++pos;
    }
  }
}

template <int N>
int launch(spt_ctx* ctx, MergeParams& p, cudaStream_t st) {
  const uint32_t nt = p.ntiles;
  partition_kernel<N><<<(nt + 1 + 255) / 256, 256, 0, st>>>(p, const_cast<uint32_t*>(p.split));
  SPT_LAUNCHED(ctx);
  const size_t smem = (size_t)2 * N * kTile * sizeof(uint32_t);
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
    SPT_TRY(spt::ctx_status64(ctx, ntiles, &p.status));
    p.epoch = epoch;
    // An empty side makes every key lookup on it invalid; give it a dummy.
    switch (N) {
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
