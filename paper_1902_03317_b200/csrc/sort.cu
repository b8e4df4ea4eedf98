// K4/K5 preprocessing: stable lexicographic sort, coalesce, fiber index.
//
// Reference: sort_lexicographic P/src/tensor.cpp:54-64 (std::stable_sort of a
// permutation under compare_entries, then gather_entries :39-50), coalesce
// P/src/tensor.cpp:66-90, build_fiber_index P/src/tensor.cpp:92-120.
//
// Sort = stable LSD radix over the modes of the sort order (the hand-written
// single-sweep passes of radix.cu). Modes are packed,
// least significant first, into <=64-bit chunk keys using log2(dims[d]) bits
// each (indices must be < dims, as validate() requires, P/src/tensor.cpp:190-215);
// each chunk is one stable radix sort of (key, permutation) pairs over only
// its significant bits, the permutation is carried into the next chunk, and
// finally the N index arrays and the value array are gathered through it.
// A stable sort of the (tuple, original position) order is exactly what
// std::stable_sort produces, so the result is bit-identical to the reference,
// duplicates included. Keys wider than 64 bits (C4: 67 bits, C5: 72 bits)
// simply take a second chunk.

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"
#include "radix.cuh"

namespace {

using spt::radix::PackSpec;
using spt::radix::UnpackSpec;

__host__ __device__ inline uint32_t bits_for(uint32_t extent) {
  if (extent <= 1) return 0;
  uint32_t v = extent - 1, b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ src, const uint32_t* __restrict__ perm,
                              T* __restrict__ dst, uint64_t n) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[perm[i]];
}

struct TupleCmp {
  const uint32_t* idx[SPT_MAX_ORDER];
  int n;
};

__global__ void fptr_tail_kernel(uint32_t* fptr, const uint32_t* d_count32,
                                 unsigned long long* d_count64, uint64_t n) {
  const uint32_t nf = *d_count32;
  fptr[nf] = static_cast<uint32_t>(n);
  if (d_count64) *d_count64 = nf;
}

// build_fiber_index in one launch (P/src/tensor.cpp:92-120). The grid is a
// few CTAs per SM; CTA r (ticket order) owns a contiguous range of 4096-entry
// tiles, and inside a tile each of the 8 warps owns 512 consecutive entries
// (four 128-entry quads read as 128-bit loads over each non-mode index array;
// a lane's first entry is compared with the previous lane's last by shuffle).
// Sweep 1 counts the fiber heads per (tile, warp) into shared memory -- the
// head masks of the range's first 8 tiles stay in registers -- then the CTA
// publishes its total, gets its offset from one decoupled look-back over
// epoch-tagged 64-bit count words (a per-tile look-back chain held 54% of the
// warps at the barrier) and scans the (tile, warp) counts once. Sweep 2 is
// warp-local: every warp knows where its heads of every tile go, compacts
// them in its own shared-memory slice and writes them out coalesced -- no CTA
// barrier per tile (they were 43% of the stall samples). The last range
// appends fptr[nfibs] = nnz.
constexpr int kFibThreads = 256, kFibQuads = 4, kFibWarps = kFibThreads / 32;
constexpr int kFibWarpEntries = kFibQuads * 128, kFibTile = kFibWarps * kFibWarpEntries;
constexpr int kFibKeep = 8;  // tiles of a range whose head masks stay in registers

template <bool VEC>
__device__ __forceinline__ void fiber_tile_heads(const TupleCmp& t, uint64_t n, uint64_t wbase,
                                                 unsigned lane, uint32_t (&hd)[kFibQuads]) {
  // wbase: the warp's first entry of the tile; quad q, lane l: wbase + q*128 + l*4
#pragma unroll
  for (int q = 0; q < kFibQuads; ++q) hd[q] = 0;
#pragma unroll
  for (int j = 0; j < SPT_MAX_ORDER; ++j) {
    if (j >= t.n) continue;
    const uint32_t* a = t.idx[j];
    uint32_t v[kFibQuads][4];
#pragma unroll
    for (int q = 0; q < kFibQuads; ++q) {
      const uint64_t e0 = wbase + q * 128 + lane * 4;
      if (VEC && e0 + 4 <= n) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(a + e0));
        v[q][0] = u.x, v[q][1] = u.y, v[q][2] = u.z, v[q][3] = u.w;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) v[q][c] = e0 + c < n ? a[e0 + c] : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < kFibQuads; ++q) {
      const uint64_t e0 = wbase + q * 128 + lane * 4;
      uint32_t prev = __shfl_up_sync(0xffffffffu, v[q][3], 1);
      if (lane == 0) {
        // the previous quad's last entry sits in lane 31 of the same warp
        prev = q ? 0u : ((e0 > 0 && e0 < n) ? __ldg(a + e0 - 1) : ~v[q][0]);
      }
      if (q) {
        const uint32_t last = __shfl_sync(0xffffffffu, v[q - 1][3], 31);
        if (lane == 0) prev = last;
      }
      hd[q] |= (v[q][0] != prev ? 1u : 0u) | (v[q][1] != v[q][0] ? 2u : 0u) |
               (v[q][2] != v[q][1] ? 4u : 0u) | (v[q][3] != v[q][2] ? 8u : 0u);
    }
  }
#pragma unroll
  for (int q = 0; q < kFibQuads; ++q) {
    const uint64_t e0 = wbase + q * 128 + lane * 4;
    const uint32_t vq = e0 >= n ? 0u : (n - e0 < 4 ? static_cast<uint32_t>(n - e0) : 4u);
    if (e0 == 0 && vq) hd[q] |= 1u;  // entry 0 always starts a fiber
    hd[q] &= (1u << vq) - 1u;
  }
}

template <bool VEC>
__global__ void __launch_bounds__(kFibThreads)
    fiber_index_kernel(TupleCmp t, uint64_t n, uint32_t ntiles, uint32_t tiles_per_cta,
                       uint32_t* __restrict__ fptr, unsigned long long* status, uint32_t epoch,
                       unsigned long long* tile_ctr, unsigned long long* d_count,
                       unsigned long long* h_count) {
  constexpr int WARPS = kFibWarps;
  __shared__ uint32_t s_rank;
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_part[kFibThreads / 32];
  __shared__ uint32_t out_s[kFibTile];            // a 512-word slice per warp
  extern __shared__ uint32_t s_cnt[];             // [tiles_per_cta][WARPS] head counts
  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) {
    const unsigned long long tk = atomicAdd(tile_ctr, 1ull);
    if (tk == gridDim.x - 1) atomicExch(tile_ctr, 0ull);  // last ticket of this launch
    s_rank = static_cast<uint32_t>(tk);
  }
  __syncthreads();
  const uint32_t r = s_rank;
  const uint32_t tile_lo = min(r * tiles_per_cta, ntiles);
  const uint32_t tile_hi = min(tile_lo + tiles_per_cta, ntiles);
  const uint32_t nt = tile_hi - tile_lo;
  uint32_t hd[kFibQuads];

  // sweep 1: head counts per (tile, warp); masks of the first kFibKeep tiles
  // stay in registers (16 bits per thread and tile)
  uint32_t keep[kFibKeep / 2];
#pragma unroll
  for (int k = 0; k < kFibKeep / 2; ++k) keep[k] = 0;
#pragma unroll 1
  for (uint32_t k = 0; k < nt; ++k) {
    const uint64_t wbase =
        static_cast<uint64_t>(tile_lo + k) * kFibTile + warp * kFibWarpEntries;
    fiber_tile_heads<VEC>(t, n, wbase, lane, hd);
    uint32_t m16 = 0, c = 0;
#pragma unroll
    for (int q = 0; q < kFibQuads; ++q) {
      c += __popc(hd[q]);
      m16 |= hd[q] << (4 * q);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) s_cnt[k * WARPS + warp] = c;
#pragma unroll
    for (int kk = 0; kk < kFibKeep; ++kk)
      if (k == static_cast<uint32_t>(kk)) keep[kk / 2] |= m16 << (16 * (kk & 1));
  }
  __syncthreads();
  // exclusive scan of the nt*WARPS counts (tile-major = entry order): a
  // contiguous chunk per thread, then the chunks' sums over the CTA
  const uint32_t M = nt * WARPS;
  const uint32_t chunk = (M + kFibThreads - 1) / kFibThreads;
  const uint32_t c_lo = min(tid * chunk, M), c_hi = min(c_lo + chunk, M);
  uint32_t mine = 0;
  for (uint32_t i = c_lo; i < c_hi; ++i) mine += s_cnt[i];
  uint32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_part[warp] = inc;
  __syncthreads();
  uint32_t pre = inc - mine, range_total = 0;
#pragma unroll
  for (int w = 0; w < kFibThreads / 32; ++w) {
    if (w < static_cast<int>(warp)) pre += s_part[w];
    range_total += s_part[w];
  }
  for (uint32_t i = c_lo; i < c_hi; ++i) {
    const uint32_t v = s_cnt[i];
    s_cnt[i] = pre;
    pre += v;
  }
  if (warp == 0) {
    const unsigned long long ep = static_cast<unsigned long long>(epoch) << 34;
    if (lane == 0)
      spt::st_relaxed64(status + r, ep | ((r == 0 ? 2ull : 1ull) << 32) | range_total);
    unsigned long long base = 0;
    if (r > 0) {
      base = spt::lookback_count64_wide<8>(status, r, epoch);
      if (lane == 0) spt::st_relaxed64(status + r, ep | (2ull << 32) | (base + range_total));
    }
    if (lane == 0) {
      s_base = base;
      if (r == gridDim.x - 1) {
        fptr[base + range_total] = static_cast<uint32_t>(n);
        if (d_count) *d_count = base + range_total;
        if (h_count) {  // pinned host word (UVA): no copy, the caller only synchronises
          *h_count = base + range_total;
          __threadfence_system();
        }
      }
    }
  }
  __syncthreads();
  const unsigned long long base = s_base;

  // sweep 2, warp-local: the warp's heads of tile k go to fptr[base + s_cnt[k][warp] ...]
  uint32_t* wout = out_s + warp * kFibWarpEntries;
#pragma unroll 1
  for (uint32_t k = 0; k < nt; ++k) {
    const uint64_t wbase =
        static_cast<uint64_t>(tile_lo + k) * kFibTile + warp * kFibWarpEntries;
    if (k < kFibKeep) {
      uint32_t m16 = 0;
#pragma unroll
      for (int kk = 0; kk < kFibKeep; ++kk)
        if (k == static_cast<uint32_t>(kk)) m16 = (keep[kk / 2] >> (16 * (kk & 1))) & 0xffffu;
#pragma unroll
      for (int q = 0; q < kFibQuads; ++q) hd[q] = (m16 >> (4 * q)) & 0xfu;
    } else {
      fiber_tile_heads<VEC>(t, n, wbase, lane, hd);
    }
    uint32_t run = 0;  // heads of the warp's earlier quads
#pragma unroll
    for (int q = 0; q < kFibQuads; ++q) {
      const uint32_t c = __popc(hd[q]);
      uint32_t in = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, in, o);
        if (lane >= o) in += u;
      }
      uint32_t pos = run + in - c;
      const uint32_t e0 = static_cast<uint32_t>(wbase) + q * 128 + lane * 4;
      uint32_t h = hd[q];
      while (h) {
        wout[pos++] = e0 + (__ffs(h) - 1);
        h &= h - 1;
      }
      run += __shfl_sync(0xffffffffu, in, 31);
    }
    __syncwarp();
    uint32_t* dst = fptr + base + s_cnt[k * WARPS + warp];
    for (uint32_t i = lane; i < run; i += 32) spt::st_stream(dst + i, wout[i]);
    __syncwarp();  // the slice is reused by the next tile
  }
}

// Positions of the entries that start a new group of equal tuples over the
// arrays of `t` (in order), then n as the sentinel; the count goes to *d_count
// and, when h_count is given, into that pinned host word.
int launch_heads(spt_ctx* ctx, const TupleCmp& t, uint64_t n, uint32_t* d_heads,
                 unsigned long long* d_count, unsigned long long* h_count, cudaStream_t st) {
  const uint32_t ntiles = static_cast<uint32_t>((n + kFibTile - 1) / kFibTile);
  // a few CTAs per SM; more when a range's (tile, warp) counts would not fit
  // 24 KB of shared memory (ticket order keeps a larger grid safe)
  const uint32_t grid = std::min<uint32_t>(
      ntiles, std::max<uint32_t>(static_cast<uint32_t>(ctx->num_sms) * 5u, (ntiles + 767) / 768));
  const uint32_t tpc = (ntiles + grid - 1) / grid;
  unsigned long long* status;
  SPT_TRY(spt::ctx_status64(ctx, grid, &status));
  uint32_t epoch;
  SPT_TRY(spt::ctx_lookback(ctx, 0, 0, &epoch));
  bool vec = true;
  for (int j = 0; j < t.n; ++j) vec = vec && spt::aligned16(t.idx[j]);
  const size_t dsm = static_cast<size_t>(tpc) * kFibWarps * sizeof(uint32_t);  // <= 24 KB
  if (vec)
    fiber_index_kernel<true><<<grid, kFibThreads, dsm, st>>>(
        t, n, ntiles, tpc, d_heads, status, epoch, ctx->d_tile_ctr, d_count, h_count);
  else
    fiber_index_kernel<false><<<grid, kFibThreads, dsm, st>>>(
        t, n, ntiles, tpc, d_heads, status, epoch, ctx->d_tile_ctr, d_count, h_count);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

// Coalesce: output p is the tuple at heads[p] with the sequential fp32 sum of
// its group in storage order (acc = v[m]; acc += v[e] ...; P/src/tensor.cpp:79-88
// -- the order is the contract, so a group is one thread's chain).
__global__ void coalesce_runs_kernel(TupleCmp t, const float* __restrict__ vals,
                                     const uint32_t* __restrict__ heads,
                                     const unsigned long long* __restrict__ count, TupleCmp out,
                                     float* __restrict__ out_val) {
  const uint64_t cnt = *count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < cnt;
       p += stride) {
    const uint32_t m = heads[p], e = heads[p + 1];
    float acc = vals[m];
    for (uint32_t k = m + 1; k < e; ++k) acc += vals[k];
#pragma unroll
    for (int j = 0; j < SPT_MAX_ORDER; ++j)
      if (j < t.n) const_cast<uint32_t*>(out.idx[j])[p] = t.idx[j][m];
    out_val[p] = acc;
  }
}

inline unsigned grid_of(spt_ctx* ctx, uint64_t n) {
  return spt::grid_for(n, 256, ctx->num_sms * 16);
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

namespace spt {

int sort_tuples(spt_ctx* ctx, const spt_coo* x, const uint32_t* mo, uint32_t* d_perm_out,
                cudaStream_t st, uint32_t nkeys) {
  const uint64_t n = x->nnz;
  const uint32_t N = std::min(x->order, nkeys);
  // Chunks from least significant mode (mo[N-1]) upward, each <= 64 bits.
  std::vector<PackSpec> chunks;
  std::vector<uint32_t> chunk_bits;
  {
    PackSpec cur{};
    uint32_t used = 0;
    for (int k = static_cast<int>(N) - 1; k >= 0; --k) {
      const uint32_t d = mo[k];
      const uint32_t b = bits_for(x->dims[d]);
      if (b == 0) continue;  // constant mode
      if (used + b > 64) {
        chunks.push_back(cur);
        chunk_bits.push_back(used);
        cur = PackSpec{};
        used = 0;
      }
      cur.idx[cur.n] = x->idx[d];
      cur.shift[cur.n] = used;
      cur.n++;
      used += b;
    }
    if (cur.n) {
      chunks.push_back(cur);
      chunk_bits.push_back(used);
    }
  }
  if (chunks.empty()) {  // every mode has extent <= 1: already sorted
    chunks.push_back(PackSpec{});
    chunk_bits.push_back(1);
  }
  // One stable radix sort per chunk; the first packs its keys from the index
  // arrays in entry order, the later ones through the running permutation.
  for (size_t c = 0; c < chunks.size(); ++c)
    SPT_TRY(radix::sort_chunk_perm(ctx, chunks[c], c == 0 ? nullptr : d_perm_out, d_perm_out, n,
                                   chunk_bits[c], st));
  return SPT_OK;
}

}  // namespace spt

extern "C" {

int spt_sort_f32(spt_ctx* ctx, spt_coo* x, const uint32_t* mode_order, unsigned flags,
                 void* stream) {
  (void)flags;
  if (!ctx) return spt::set_error(SPT_EINVAL, "sort_lexicographic: null context");
  SPT_TRY(spt::check_coo(x, "sort_lexicographic"));
  if (!mode_order) return spt::set_error(SPT_EINVAL, "sort_lexicographic: null mode order");
  // check_mode_order, P/src/tensor.cpp:28-37
  bool seen[SPT_MAX_ORDER] = {false};
  for (uint32_t k = 0; k < x->order; ++k) {
    if (mode_order[k] >= x->order || seen[mode_order[k]])
      return spt::set_error(SPT_EINVAL, "sort_lexicographic: mode order is not a permutation");
    seen[mode_order[k]] = true;
  }
  cudaStream_t st = spt::as_stream(stream);
  const uint64_t n = x->nnz;
  // Whole tuple in one key (the common case: C2 42 bits, C3 48): sort
  // (packed key, value) pairs and unpack the indices from the sorted keys --
  // no permutation and no gather pass.
  uint32_t total_bits = 0;
  for (uint32_t d = 0; d < x->order; ++d) total_bits += bits_for(x->dims[d]);
  if (n > 1 && total_bits <= 64) {
    PackSpec spec{};
    UnpackSpec un{};
    uint32_t used = 0;
    for (int k = static_cast<int>(x->order) - 1; k >= 0; --k) {
      const uint32_t d = mode_order[k];
      const uint32_t b = bits_for(x->dims[d]);
      un.idx[un.n] = x->idx[d];
      un.shift[un.n] = used;
      un.mask[un.n] = b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
      un.n++;
      if (b == 0) continue;
      spec.idx[spec.n] = x->idx[d];
      spec.shift[spec.n] = used;
      spec.n++;
      used += b;
    }
    SPT_TRY(spt::radix::sort_tuple_inplace(ctx, spec, un, reinterpret_cast<uint32_t*>(x->val), n,
                                           std::max<uint32_t>(used, 1), st));
  } else if (n > 1) {
    // perm lives in its own allocation (sort_tuples uses the ctx scratch).
    uint32_t* perm = nullptr;
    uint32_t* tmp = nullptr;
    SPT_CUDA(spt::tmp_alloc(ctx, &perm, n * sizeof(uint32_t), st));
    int s = spt::sort_tuples(ctx, x, mode_order, perm, st);
    if (s == SPT_OK) {
      cudaError_t e = spt::tmp_alloc(ctx, &tmp, n * sizeof(uint32_t), st);
      if (e != cudaSuccess) s = spt::cuda_status(e, "sort gather buffer");
    }
    if (s == SPT_OK) {
      const unsigned g = grid_of(ctx, n);
      for (uint32_t d = 0; d <= x->order && s == SPT_OK; ++d) {
        uint32_t* arr = d < x->order ? x->idx[d] : reinterpret_cast<uint32_t*>(x->val);
        gather_kernel<uint32_t><<<g, 256, 0, st>>>(arr, perm, tmp, n);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(arr, tmp, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) s = spt::cuda_status(e, "sort gather");
        ctx->launches++;
      }
    }
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(perm, st);
    if (s != SPT_OK) return s;
  }
  x->has_sort_order = 1;
  for (uint32_t k = 0; k < SPT_MAX_ORDER; ++k)
    x->sort_order[k] = k < x->order ? static_cast<int32_t>(mode_order[k]) : 0;
  return SPT_OK;
}

int spt_coalesce_f32(spt_ctx* ctx, const spt_coo* x, spt_coo* z, uint64_t* h_nnz,
                     uint64_t* d_nnz, unsigned flags, void* stream) {
  (void)flags;
  if (!ctx) return spt::set_error(SPT_EINVAL, "coalesce: null context");
  SPT_TRY(spt::check_coo(x, "coalesce"));
  if (!z) return spt::set_error(SPT_EINVAL, "coalesce: null output");
  if (!x->has_sort_order)
    return spt::set_error(SPT_EINVAL, "coalesce: input must be sorted (sort it first)");
  cudaStream_t st = spt::as_stream(stream);
  const uint64_t n = x->nnz;
  // metadata: dims of x, sort order of x, coalesced
  z->order = x->order;
  for (uint32_t d = 0; d < SPT_MAX_ORDER; ++d) {
    z->dims[d] = d < x->order ? x->dims[d] : 0;
    z->sort_order[d] = x->sort_order[d];
  }
  z->has_sort_order = 1;
  z->coalesced = 1;
  if (n == 0) {
    z->nnz = 0;
    if (h_nnz) *h_nnz = 0;
    if (d_nnz) SPT_CUDA(cudaMemsetAsync(d_nnz, 0, sizeof(uint64_t), st));
    return SPT_OK;
  }
  // group heads by the single-launch head-position kernel (the fiber index's,
  // over all N index arrays), then one thread per output sums its group
  void* scratch;
  SPT_TRY(spt::ctx_scratch(ctx, 256 + align_up((n + 1) * 4), &scratch));
  unsigned long long* cnt = static_cast<unsigned long long*>(scratch);
  uint32_t* heads = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + 256);
  unsigned long long* count_out = d_nnz ? reinterpret_cast<unsigned long long*>(d_nnz) : cnt;
  TupleCmp t{};
  TupleCmp o{};
  for (uint32_t d = 0; d < x->order; ++d) {
    t.idx[d] = x->idx[d];
    o.idx[d] = z->idx[d];
  }
  t.n = o.n = static_cast<int>(x->order);
  SPT_TRY(launch_heads(ctx, t, n, heads, count_out, h_nnz ? ctx->h_pinned : nullptr, st));
  coalesce_runs_kernel<<<grid_of(ctx, n), 256, 0, st>>>(t, x->val, heads, count_out, o, z->val);
  SPT_LAUNCHED(ctx);
  if (h_nnz) {
    SPT_CUDA(cudaStreamSynchronize(st));
    *h_nnz = ctx->h_pinned[0];
    z->nnz = *h_nnz;
  }
  return SPT_OK;
}

int spt_fiber_index(spt_ctx* ctx, const spt_coo* x, uint32_t mode, uint32_t* d_fptr,
                    uint64_t* h_nfibs, uint64_t* d_nfibs, unsigned flags, void* stream) {
  (void)flags;
  if (!ctx) return spt::set_error(SPT_EINVAL, "build_fiber_index: null context");
  SPT_TRY(spt::check_coo(x, "build_fiber_index", false));
  // P/src/tensor.cpp:94-99
  if (mode >= x->order) return spt::set_error(SPT_EINVAL, "build_fiber_index: mode out of range");
  if (!x->has_sort_order || static_cast<uint32_t>(x->sort_order[x->order - 1]) != mode)
    return spt::set_error(SPT_EINVAL,
                          "build_fiber_index: tensor must be sorted with the target mode as "
                          "the last key");
  if (!d_fptr) return spt::set_error(SPT_EINVAL, "build_fiber_index: null fptr");
  cudaStream_t st = spt::as_stream(stream);
  const uint64_t n = x->nnz;
  TupleCmp t{};
  for (uint32_t d = 0; d < x->order; ++d)
    if (d != mode) t.idx[t.n++] = x->idx[d];
  void* scratch;
  SPT_TRY(spt::ctx_scratch(ctx, 256, &scratch));
  uint32_t* cnt32 = static_cast<uint32_t*>(scratch);
  unsigned long long* cnt64 = reinterpret_cast<unsigned long long*>(cnt32 + 2);
  unsigned long long* count_out =
      d_nfibs ? reinterpret_cast<unsigned long long*>(d_nfibs) : cnt64;
  if (n > 0) {
    SPT_TRY(launch_heads(ctx, t, n, d_fptr, count_out, h_nfibs ? ctx->h_pinned : nullptr, st));
  } else {
    SPT_CUDA(cudaMemsetAsync(cnt32, 0, 4, st));
    fptr_tail_kernel<<<1, 1, 0, st>>>(d_fptr, cnt32, count_out, n);
    SPT_LAUNCHED(ctx);
  }
  if (h_nfibs) {
    if (n == 0)
      SPT_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_nfibs ? (void*)d_nfibs : (void*)cnt64, 8,
                               cudaMemcpyDeviceToHost, st));
    // n > 0: the kernel's last range wrote the count into the pinned word itself
    SPT_CUDA(cudaStreamSynchronize(st));
    *h_nfibs = ctx->h_pinned[0];
  }
  return SPT_OK;
}

}  // extern "C"
