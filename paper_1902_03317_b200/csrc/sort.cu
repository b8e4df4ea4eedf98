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
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
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

// flag[m] = 1 iff entry m starts a new group of equal (selected-mode) tuples.
__global__ void head_flags_kernel(TupleCmp t, uint32_t* flags, uint64_t n) {
  uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; m < n; m += stride) {
    uint32_t f = (m == 0);
    for (int j = 0; j < t.n && !f; ++j) f = t.idx[j][m] != t.idx[j][m - 1];
    flags[m] = f;
  }
}

// Coalesce: heads write the tuple and the sequential fp32 sum of their group
// in storage order (acc = v[m]; acc += v[e] ...; P/src/tensor.cpp:79-88).
__global__ void coalesce_write_kernel(TupleCmp t, const float* vals, const uint32_t* flags,
                                      const uint32_t* pos, uint64_t n, TupleCmp out,
                                      float* out_val) {
  uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; m < n; m += stride) {
    if (!flags[m]) continue;
    const uint32_t p = pos[m];
    float acc = vals[m];
    for (uint64_t e = m + 1; e < n && !flags[e]; ++e) acc += vals[e];
    for (int j = 0; j < t.n; ++j) const_cast<uint32_t*>(out.idx[j])[p] = t.idx[j][m];
    out_val[p] = acc;
  }
}

__global__ void fptr_tail_kernel(uint32_t* fptr, const uint32_t* d_count32,
                                 unsigned long long* d_count64, uint64_t n) {
  const uint32_t nf = *d_count32;
  fptr[nf] = static_cast<uint32_t>(n);
  if (d_count64) *d_count64 = nf;
}

__global__ void count_from_scan_kernel(const uint32_t* flags, const uint32_t* pos, uint64_t n,
                                       unsigned long long* out) {
  *out = n ? (unsigned long long)pos[n - 1] + flags[n - 1] : 0ull;
}

inline unsigned grid_of(spt_ctx* ctx, uint64_t n) {
  return spt::grid_for(n, 256, ctx->num_sms * 16);
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

namespace spt {

int sort_tuples(spt_ctx* ctx, const spt_coo* x, const uint32_t* mo, uint32_t* d_perm_out,
                cudaStream_t st) {
  const uint64_t n = x->nnz;
  const uint32_t N = x->order;
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
  size_t temp = 0;
  SPT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                         static_cast<int64_t>(n), st));
  const size_t fb = align_up(n * 4);
  void* scratch;
  SPT_TRY(spt::ctx_scratch(ctx, 2 * fb + align_up(temp) + 256, &scratch));
  char* base = static_cast<char*>(scratch);
  uint32_t* flags_d = reinterpret_cast<uint32_t*>(base);
  uint32_t* pos = reinterpret_cast<uint32_t*>(base + fb);
  void* tmp = base + 2 * fb;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(base + 2 * fb + align_up(temp));
  TupleCmp t{};
  TupleCmp o{};
  for (uint32_t d = 0; d < x->order; ++d) {
    t.idx[d] = x->idx[d];
    o.idx[d] = z->idx[d];
  }
  t.n = o.n = static_cast<int>(x->order);
  const unsigned g = grid_of(ctx, n);
  head_flags_kernel<<<g, 256, 0, st>>>(t, flags_d, n);
  SPT_LAUNCHED(ctx);
  SPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, temp, flags_d, pos, static_cast<int64_t>(n), st));
  ctx->launches += 2;
  coalesce_write_kernel<<<g, 256, 0, st>>>(t, x->val, flags_d, pos, n, o, z->val);
  SPT_LAUNCHED(ctx);
  count_from_scan_kernel<<<1, 1, 0, st>>>(flags_d, pos, n,
                                          d_nnz ? reinterpret_cast<unsigned long long*>(d_nnz)
                                                : cnt);
  SPT_LAUNCHED(ctx);
  if (h_nnz) {
    SPT_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_nnz ? (void*)d_nnz : (void*)cnt, 8,
                             cudaMemcpyDeviceToHost, st));
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
  size_t temp = 0;
  thrust::counting_iterator<uint32_t> it(0);
  SPT_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, it, (uint32_t*)nullptr, d_fptr,
                                      (uint32_t*)nullptr, static_cast<int64_t>(n), st));
  const size_t fb = align_up((n ? n : 1) * 4);
  void* scratch;
  SPT_TRY(spt::ctx_scratch(ctx, fb + align_up(temp) + 256, &scratch));
  char* base = static_cast<char*>(scratch);
  uint32_t* flags_d = reinterpret_cast<uint32_t*>(base);
  void* tmp = base + fb;
  uint32_t* cnt32 = reinterpret_cast<uint32_t*>(base + fb + align_up(temp));
  unsigned long long* cnt64 = reinterpret_cast<unsigned long long*>(cnt32 + 2);
  if (n > 0) {
    head_flags_kernel<<<grid_of(ctx, n), 256, 0, st>>>(t, flags_d, n);
    SPT_LAUNCHED(ctx);
    SPT_CUDA(cub::DeviceSelect::Flagged(tmp, temp, it, flags_d, d_fptr, cnt32,
                                        static_cast<int64_t>(n), st));
    ctx->launches += 2;
  } else {
    SPT_CUDA(cudaMemsetAsync(cnt32, 0, 4, st));
  }
  fptr_tail_kernel<<<1, 1, 0, st>>>(d_fptr, cnt32,
                                    d_nfibs ? reinterpret_cast<unsigned long long*>(d_nfibs)
                                            : cnt64,
                                    n);
  SPT_LAUNCHED(ctx);
  if (h_nfibs) {
    SPT_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_nfibs ? (void*)d_nfibs : (void*)cnt64, 8,
                             cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
    *h_nfibs = ctx->h_pinned[0];
  }
  return SPT_OK;
}

}  // extern "C"
