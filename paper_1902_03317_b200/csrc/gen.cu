// K10 seeded synthetic COO generator (bench/test inputs; not a reference path).
//
// The reference's gen_synthetic (P/src/io.cpp:151-244) draws uniform tuples
// with rejection of duplicates and U[1,2) values; it cannot express the
// BASELINE configs (Zipf modes, other value ranges) and overflows its u64
// linearisation for C4/C5 (P/src/io.cpp:157-166). This generator keeps its
// contract -- exactly nnz distinct tuples, duplicates rejected in draw order
// -- on the device:
//   1. draw M >= nnz candidate tuples, mode d from Philox(c, d): uniform
//      (multiply-high) or Zipf(s) by inverse CDF (fp64 prefix table + guide
//      table) mapped through a seeded Feistel permutation of [0, dims[d]);
//   2. stable-sort candidates by tuple (the library's own radix sort), flag
//      the first occurrence of each tuple;
//   3. keep the nnz first occurrences with the smallest draw index (what
//      sequential rejection sampling would keep), in draw order;
//   4. values U[lo,hi) from Philox(position); optionally sort.
// If fewer than nnz distinct tuples were drawn, M grows and the (counter-based,
// hence prefix-stable) draw is repeated.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "internal.cuh"

namespace {

constexpr int kGuideBits = 16;

__device__ __forceinline__ uint32_t mix32(uint32_t x, uint32_t k) {
  x ^= k;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Seeded bijection on [0, n) (Feistel on 2h bits + cycle walking).
struct Perm {
  uint32_t n, h, mask;
  uint32_t k[4];
  __device__ uint32_t operator()(uint32_t v) const {
    if (n <= 1) return 0;
    do {
      uint32_t L = v >> h, R = v & mask;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t t = L ^ (mix32(R, k[r]) & mask);
        L = R;
        R = t;
      }
      v = (L << h) | R;
    } while (v >= n);
    return v;
  }
};

struct ModeDist {
  uint32_t dim;
  int zipf;            // 0 uniform, 1 zipf
  const double* cdf;   // [dim], inclusive, cdf[dim-1] == 1
  const uint32_t* guide;  // [2^kGuideBits + 1]
  Perm perm;
};

struct DrawParams {
  ModeDist m[SPT_MAX_ORDER];
  uint32_t* out[SPT_MAX_ORDER];
  int N;
  uint64_t M;
  uint64_t seed;
};

__global__ void zipf_weights_kernel(double* w, uint32_t n, double s) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += gridDim.x * blockDim.x) w[i] = pow((double)(i + 1), -s);
}

__global__ void normalize_kernel(double* c, uint32_t n) {
  const double tot = c[n - 1];
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += gridDim.x * blockDim.x) c[i] = (i + 1 == n) ? 1.0 : c[i] / tot;
}

// guide[b] = first k with cdf[k] >= b / 2^G.
__global__ void guide_kernel(const double* cdf, uint32_t n, uint32_t* guide) {
  const uint32_t B = 1u << kGuideBits;
  uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  for (; b <= B; b += gridDim.x * blockDim.x) {
    const double t = (double)b / B;
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (cdf[mid] >= t) hi = mid;
      else lo = mid + 1;
    }
    guide[b] = lo;
  }
}

__global__ void draw_kernel(DrawParams p) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; c < p.M; c += stride) {
    for (int d = 0; d < p.N; ++d) {
      const ModeDist& md = p.m[d];
      const uint4 r = spt::Philox::gen(c, 0x1000 + d, p.seed);
      uint32_t v;
      if (!md.zipf) {
        v = static_cast<uint32_t>(((uint64_t)r.x * md.dim) >> 32);
      } else {
        const double u = spt::u01d(r.x, r.y);
        const uint32_t b = static_cast<uint32_t>(u * (1u << kGuideBits));
        uint32_t lo = md.guide[b], hi = md.guide[b + 1];
        // first k in [lo, hi] with cdf[k] > u
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (md.cdf[mid] > u) hi = mid;
          else lo = mid + 1;
        }
        v = md.perm(lo);
      }
      p.out[d][c] = v;
    }
  }
}

struct TupleRef {
  const uint32_t* idx[SPT_MAX_ORDER];
  int n;
};

// keep[perm[i]] = 1 iff sorted position i starts a new tuple (first occurrence).
__global__ void first_occurrence_kernel(TupleRef t, const uint32_t* perm, uint32_t* keep,
                                        uint64_t M) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < M; i += stride) {
    const uint32_t a = perm[i];
    uint32_t f = 1;
    if (i > 0) {
      const uint32_t b = perm[i - 1];
      f = 0;
      for (int d = 0; d < t.n && !f; ++d) f = t.idx[d][a] != t.idx[d][b];
    }
    keep[a] = f;
  }
}

__global__ void compact_kernel(TupleRef cand, const uint32_t* keep, const uint32_t* pos,
                               uint64_t M, uint64_t nnz, TupleRef out) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; c < M; c += stride) {
    if (!keep[c] || pos[c] >= nnz) continue;
    for (int d = 0; d < cand.n; ++d) const_cast<uint32_t*>(out.idx[d])[pos[c]] = cand.idx[d][c];
  }
}

__global__ void values_kernel(float* v, uint64_t n, uint64_t seed, float lo, float hi) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float w = hi - lo;
  for (; i < n; i += stride) {
    const uint4 r = spt::Philox::gen(i, 0x2000, seed);
    const float x = lo + w * spt::u01(r.x);
    v[i] = x < hi ? x : lo;
  }
}

uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" int spt_gen_coo_f32(spt_ctx* ctx, spt_coo* x, uint64_t seed, const double* zipf_s,
                               float lo, float hi, const uint32_t* sort_order, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "gen: null context");
  SPT_TRY(spt::check_coo(x, "gen"));
  const int N = static_cast<int>(x->order);
  const uint64_t nnz = x->nnz;
  long double cap = 1;
  for (int d = 0; d < N; ++d) cap *= x->dims[d];
  if ((long double)nnz > cap)
    return spt::set_error(SPT_EINVAL, "gen: nnz %llu exceeds the index-space capacity",
                          (unsigned long long)nnz);
  if (!(hi > lo)) return spt::set_error(SPT_EINVAL, "gen: need lo < hi");
  cudaStream_t st = spt::as_stream(stream);
  x->coalesced = 1;
  x->has_sort_order = 0;
  if (nnz == 0) return SPT_OK;

  // Per-mode distributions.
  DrawParams dp{};
  dp.N = N;
  dp.seed = seed;
  std::vector<void*> allocs;
  auto cleanup = [&]() {
    for (void* a : allocs) cudaFreeAsync(a, st);
    allocs.clear();
  };
  uint64_t ks = seed ^ 0x5eedf00dull;
  for (int d = 0; d < N; ++d) {
    ModeDist& md = dp.m[d];
    md.dim = x->dims[d];
    const double s = zipf_s ? zipf_s[d] : 0.0;
    md.zipf = s > 0.0 && md.dim > 1;
    uint32_t h = 1;
    while ((1ull << (2 * h)) < md.dim) ++h;
    md.perm.n = md.dim;
    md.perm.h = h;
    md.perm.mask = (1u << h) - 1;
    for (int r = 0; r < 4; ++r) md.perm.k[r] = static_cast<uint32_t>(splitmix(ks));
    if (!md.zipf) continue;
    double* cdf;
    uint32_t* guide;
    SPT_CUDA(spt::tmp_alloc(ctx, &cdf, (size_t)md.dim * sizeof(double), st));
    allocs.push_back(cdf);
    SPT_CUDA(spt::tmp_alloc(ctx, &guide, ((1u << kGuideBits) + 1) * sizeof(uint32_t), st));
    allocs.push_back(guide);
    zipf_weights_kernel<<<spt::grid_for(md.dim, 256, 4096), 256, 0, st>>>(cdf, md.dim, s);
    SPT_LAUNCHED(ctx);
    size_t tb = 0;
    SPT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cdf, cdf, (int64_t)md.dim, st));
    void* tmp;
    SPT_CUDA(spt::tmp_alloc(ctx, &tmp, tb, st));
    SPT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, cdf, cdf, (int64_t)md.dim, st));
    cudaFreeAsync(tmp, st);
    normalize_kernel<<<spt::grid_for(md.dim, 256, 4096), 256, 0, st>>>(cdf, md.dim);
    SPT_LAUNCHED(ctx);
    guide_kernel<<<spt::grid_for((1u << kGuideBits) + 1, 256, 4096), 256, 0, st>>>(cdf, md.dim,
                                                                                    guide);
    SPT_LAUNCHED(ctx);
    md.cdf = cdf;
    md.guide = guide;
  }

  uint64_t M = nnz + nnz / 16 + 1024;
  int status = SPT_OK;
  bool done = false;
  for (int attempt = 0; attempt < 12; ++attempt) {
    if (M >= (1ull << 32)) M = (1ull << 32) - 1;
    std::vector<uint32_t*> cand(N, nullptr);
    uint32_t *perm = nullptr, *keep = nullptr, *pos = nullptr;
    void* tmp = nullptr;
    auto free_round = [&]() {
      for (auto* c : cand) cudaFreeAsync(c, st);
      cudaFreeAsync(perm, st);
      cudaFreeAsync(keep, st);
      cudaFreeAsync(pos, st);
      cudaFreeAsync(tmp, st);
    };
#define GEN_CUDA(call)                                \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) {                          \
      free_round();                                   \
      cleanup();                                      \
      return spt::cuda_status(_e, #call);             \
    }                                                 \
  } while (0)
    for (int d = 0; d < N; ++d) GEN_CUDA(spt::tmp_alloc(ctx, &cand[d], M * 4, st));
    GEN_CUDA(spt::tmp_alloc(ctx, &perm, M * 4, st));
    GEN_CUDA(spt::tmp_alloc(ctx, &keep, M * 4, st));
    GEN_CUDA(spt::tmp_alloc(ctx, &pos, M * 4, st));
    for (int d = 0; d < N; ++d) dp.out[d] = cand[d];
    dp.M = M;
    draw_kernel<<<spt::grid_for(M, 256, ctx->num_sms * 16), 256, 0, st>>>(dp);
    GEN_CUDA(cudaGetLastError());
    ctx->launches++;
    spt_coo c{};
    c.order = N;
    c.nnz = M;
    for (int d = 0; d < N; ++d) {
      c.dims[d] = x->dims[d];
      c.idx[d] = cand[d];
    }
    uint32_t asc[SPT_MAX_ORDER];
    for (int d = 0; d < N; ++d) asc[d] = d;
    status = spt::sort_tuples(ctx, &c, asc, perm, st);
    if (status != SPT_OK) {
      free_round();
      cleanup();
      return status;
    }
    TupleRef t{};
    t.n = N;
    for (int d = 0; d < N; ++d) t.idx[d] = cand[d];
    first_occurrence_kernel<<<spt::grid_for(M, 256, ctx->num_sms * 16), 256, 0, st>>>(t, perm,
                                                                                      keep, M);
    GEN_CUDA(cudaGetLastError());
    ctx->launches++;
    size_t tb = 0;
    GEN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, pos, (int64_t)M, st));
    GEN_CUDA(spt::tmp_alloc(ctx, &tmp, tb, st));
    GEN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, keep, pos, (int64_t)M, st));
    uint32_t last[2];
    GEN_CUDA(cudaMemcpyAsync(&last[0], pos + M - 1, 4, cudaMemcpyDeviceToHost, st));
    GEN_CUDA(cudaMemcpyAsync(&last[1], keep + M - 1, 4, cudaMemcpyDeviceToHost, st));
    GEN_CUDA(cudaStreamSynchronize(st));
    const uint64_t uniq = (uint64_t)last[0] + last[1];
    if (uniq >= nnz) {
      TupleRef o{};
      o.n = N;
      for (int d = 0; d < N; ++d) o.idx[d] = x->idx[d];
      compact_kernel<<<spt::grid_for(M, 256, ctx->num_sms * 16), 256, 0, st>>>(t, keep, pos, M,
                                                                              nnz, o);
      GEN_CUDA(cudaGetLastError());
      ctx->launches++;
      free_round();
      done = true;
      break;
    }
    free_round();
    if (M == (1ull << 32) - 1) {
      cleanup();
      return spt::set_error(SPT_EOVERFLOW,
                            "gen: could not draw %llu distinct tuples within 2^32 candidates",
                            (unsigned long long)nnz);
    }
    // Grow by the observed duplicate rate (with margin).
    const double rate = uniq > 0 ? (double)uniq / (double)M : 0.5;
    M = static_cast<uint64_t>(std::ceil((double)nnz / std::max(rate, 0.05) * 1.1)) + 4096;
#undef GEN_CUDA
  }
  cleanup();
  if (!done)
    return spt::set_error(SPT_ERUNTIME, "gen: too many duplicate draws for %llu distinct tuples",
                          (unsigned long long)nnz);
  values_kernel<<<spt::grid_for(nnz, 256, ctx->num_sms * 16), 256, 0, st>>>(x->val, nnz, seed,
                                                                            lo, hi);
  SPT_LAUNCHED(ctx);
  if (sort_order) return spt_sort_f32(ctx, x, sort_order, 0, stream);
  return SPT_OK;
}
