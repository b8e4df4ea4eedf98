// K1 TS and K2 TEW-eq: pure HBM streaming kernels.
//
// Reference semantics:
//   ts      P/src/kernels_seq.cpp:55-67, P/src/kernels_par.cpp:69-91,
//           apply_scalar P/src/kernel_detail.hpp:29-32
//   tew_eq  P/src/kernels_seq.cpp:11-39, P/src/kernels_par.cpp:19-67,
//           apply_elem P/src/kernel_detail.hpp:19-27
// Both copy x's index arrays into z (the output is a freshly materialised
// COO, exactly as the reference returns it by value) and apply one IEEE fp32
// op per stored value (no FMA contraction possible, no fast-math), so values
// are bit-identical to the reference.
//
// Layout: each thread moves one 16-byte vector (4 entries) of every one of the
// N index arrays and the value array(s): (N+1) independent 128-bit loads in
// flight per thread for TS, 2(N+1) for TEW-eq, streamed with evict-first
// hints since nothing is re-read.
#include "internal.cuh"

namespace {

struct EwPtrs {
  const uint32_t* xi[SPT_MAX_ORDER];
  const uint32_t* yi[SPT_MAX_ORDER];
  uint32_t* zi[SPT_MAX_ORDER];
  const float* xv;
  const float* yv;
  float* zv;
};

__device__ __forceinline__ float scalar_op(int op, float a, float s) {
  return op == SPT_SCALAR_ADD ? a + s : a * s;
}

__device__ __forceinline__ float elem_op(int op, float a, float b) {
  switch (op) {
    case SPT_ADD: return a + b;
    case SPT_SUB: return a - b;
    case SPT_MUL: return a * b;
    default: return a / b;
  }
}

template <int N>
__global__ void __launch_bounds__(256) ts_vec_kernel(EwPtrs p, uint64_t nvec, float s, int op) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < nvec; i += stride) {
    uint4 ix[N];
#pragma unroll
    for (int d = 0; d < N; ++d) ix[d] = spt::ld_stream(reinterpret_cast<const uint4*>(p.xi[d]) + i);
    uint4 v = spt::ld_stream(reinterpret_cast<const uint4*>(p.xv) + i);
#pragma unroll
    for (int d = 0; d < N; ++d) spt::st_stream(reinterpret_cast<uint4*>(p.zi[d]) + i, ix[d]);
    float4 f = *reinterpret_cast<float4*>(&v);
    f.x = scalar_op(op, f.x, s);
    f.y = scalar_op(op, f.y, s);
    f.z = scalar_op(op, f.z, s);
    f.w = scalar_op(op, f.w, s);
    spt::st_stream(reinterpret_cast<uint4*>(p.zv) + i, *reinterpret_cast<uint4*>(&f));
  }
}

// Scalar path for the tail (and for unaligned arrays).
__global__ void ts_scalar_kernel(EwPtrs p, uint32_t order, uint64_t begin, uint64_t end, float s,
                                 int op) {
  uint64_t m = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; m < end; m += stride) {
    for (uint32_t d = 0; d < order; ++d) p.zi[d][m] = p.xi[d][m];
    p.zv[m] = scalar_op(op, p.xv[m], s);
  }
}

template <int N>
__global__ void __launch_bounds__(256)
    tew_eq_vec_kernel(EwPtrs p, uint64_t nvec, int op, unsigned long long* err) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < nvec; i += stride) {
    uint4 xi[N], yi[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
      xi[d] = spt::ld_stream(reinterpret_cast<const uint4*>(p.xi[d]) + i);
      yi[d] = spt::ld_stream(reinterpret_cast<const uint4*>(p.yi[d]) + i);
    }
    uint4 xv = spt::ld_stream(reinterpret_cast<const uint4*>(p.xv) + i);
    uint4 yv = spt::ld_stream(reinterpret_cast<const uint4*>(p.yv) + i);
#pragma unroll
    for (int d = 0; d < N; ++d) spt::st_stream(reinterpret_cast<uint4*>(p.zi[d]) + i, xi[d]);
    // Per-lane mismatch mask over the 4 entries.
    unsigned bad = 0;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      bad |= (xi[d].x != yi[d].x) ? 1u : 0u;
      bad |= (xi[d].y != yi[d].y) ? 2u : 0u;
      bad |= (xi[d].z != yi[d].z) ? 4u : 0u;
      bad |= (xi[d].w != yi[d].w) ? 8u : 0u;
    }
    const float4 a = *reinterpret_cast<float4*>(&xv);
    const float4 b = *reinterpret_cast<float4*>(&yv);
    unsigned dz = 0;
    if (op == SPT_DIV) {
      dz |= (b.x == 0.0f) ? 1u : 0u;
      dz |= (b.y == 0.0f) ? 2u : 0u;
      dz |= (b.z == 0.0f) ? 4u : 0u;
      dz |= (b.w == 0.0f) ? 8u : 0u;
    }
    float4 z;
    z.x = elem_op(op, a.x, b.x);
    z.y = elem_op(op, a.y, b.y);
    z.z = elem_op(op, a.z, b.z);
    z.w = elem_op(op, a.w, b.w);
    spt::st_stream(reinterpret_cast<uint4*>(p.zv) + i, *reinterpret_cast<uint4*>(&z));
    if (bad) atomicMin(&err[0], (unsigned long long)(i * 4 + __ffs(bad) - 1));
    if (dz) atomicMin(&err[1], (unsigned long long)(i * 4 + __ffs(dz) - 1));
  }
}

__global__ void tew_eq_scalar_kernel(EwPtrs p, uint32_t order, uint64_t begin, uint64_t end,
                                     int op, unsigned long long* err) {
  uint64_t m = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; m < end; m += stride) {
    bool bad = false;
    for (uint32_t d = 0; d < order; ++d) {
      const uint32_t a = p.xi[d][m];
      bad |= a != p.yi[d][m];
      p.zi[d][m] = a;
    }
    const float b = p.yv[m];
    p.zv[m] = elem_op(op, p.xv[m], b);
    if (bad) atomicMin(&err[0], (unsigned long long)m);
    if (op == SPT_DIV && b == 0.0f) atomicMin(&err[1], (unsigned long long)m);
  }
}

bool all_aligned(const spt_coo* t) {
  for (uint32_t d = 0; d < t->order; ++d)
    if (!spt::aligned16(t->idx[d])) return false;
  return spt::aligned16(t->val);
}

void copy_meta(const spt_coo* x, spt_coo* z) {
  z->order = x->order;
  z->nnz = x->nnz;
  for (uint32_t d = 0; d < SPT_MAX_ORDER; ++d) {
    z->dims[d] = d < x->order ? x->dims[d] : 0;
    z->sort_order[d] = x->sort_order[d];
  }
  z->has_sort_order = x->has_sort_order;
  z->coalesced = x->coalesced;
}

#define SPT_ORDER_SWITCH(ORDER, KERNEL, GRID, STREAM, ...)                        \
  switch (ORDER) {                                                                \
    case 1: KERNEL<1><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 2: KERNEL<2><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 3: KERNEL<3><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 4: KERNEL<4><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 5: KERNEL<5><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 6: KERNEL<6><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    case 7: KERNEL<7><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;             \
    default: KERNEL<8><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;            \
  }

}  // namespace

extern "C" {

int spt_ts_f32(spt_ctx* ctx, const spt_coo* x, float s, int op, spt_coo* z, unsigned flags,
               void* stream) {
  (void)flags;
  if (!ctx) return spt::set_error(SPT_EINVAL, "ts: null context");
  SPT_TRY(spt::check_coo(x, "ts"));
  if (!z) return spt::set_error(SPT_EINVAL, "ts: null output descriptor");
  if (op != SPT_SCALAR_ADD && op != SPT_SCALAR_MUL)
    return spt::set_error(SPT_EINVAL, "ts: unknown scalar op %d", op);
  const uint64_t n = x->nnz;
  if (n > 0) {
    for (uint32_t d = 0; d < x->order; ++d)
      if (!z->idx[d]) return spt::set_error(SPT_EINVAL, "ts: null output index array");
    if (!z->val) return spt::set_error(SPT_EINVAL, "ts: null output value array");
  }
  copy_meta(x, z);
  if (n == 0) return SPT_OK;
  cudaStream_t st = spt::as_stream(stream);
  EwPtrs p{};
  for (uint32_t d = 0; d < x->order; ++d) {
    p.xi[d] = x->idx[d];
    p.zi[d] = z->idx[d];
  }
  p.xv = x->val;
  p.zv = z->val;
  uint64_t nvec = (all_aligned(x) && all_aligned(z)) ? n / 4 : 0;
  if (nvec) {
    unsigned grid = spt::grid_for(nvec, 256, 1u << 30);
    SPT_ORDER_SWITCH(x->order, ts_vec_kernel, grid, st, p, nvec, s, op);
    SPT_LAUNCHED(ctx);
  }
  if (nvec * 4 < n) {
    unsigned grid = spt::grid_for(n - nvec * 4, 256, ctx->num_sms * 8);
    ts_scalar_kernel<<<grid, 256, 0, st>>>(p, x->order, nvec * 4, n, s, op);
    SPT_LAUNCHED(ctx);
  }
  return SPT_OK;
}

int spt_tew_eq_f32(spt_ctx* ctx, const spt_coo* x, const spt_coo* y, int op, spt_coo* z,
                   unsigned flags, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "tew_eq: null context");
  SPT_TRY(spt::check_coo(x, "tew_eq"));
  SPT_TRY(spt::check_coo(y, "tew_eq"));
  if (!z) return spt::set_error(SPT_EINVAL, "tew_eq: null output descriptor");
  if (op < SPT_ADD || op > SPT_DIV) return spt::set_error(SPT_EINVAL, "tew_eq: unknown op %d", op);
  // P/src/kernels_seq.cpp:14-17
  bool same_dims = x->order == y->order;
  for (uint32_t d = 0; same_dims && d < x->order; ++d) same_dims = x->dims[d] == y->dims[d];
  if (!same_dims)
    return spt::set_error(SPT_EINVAL, "tew_eq: tensors must have identical dimensions");
  if (x->nnz != y->nnz)
    return spt::set_error(SPT_EINVAL, "tew_eq: tensors must have identical nonzero counts");
  const uint64_t n = x->nnz;
  if (n > 0) {
    for (uint32_t d = 0; d < x->order; ++d)
      if (!z->idx[d]) return spt::set_error(SPT_EINVAL, "tew_eq: null output index array");
    if (!z->val) return spt::set_error(SPT_EINVAL, "tew_eq: null output value array");
  }
  copy_meta(x, z);
  if (n == 0) return SPT_OK;
  cudaStream_t st = spt::as_stream(stream);
  EwPtrs p{};
  for (uint32_t d = 0; d < x->order; ++d) {
    p.xi[d] = x->idx[d];
    p.yi[d] = y->idx[d];
    p.zi[d] = z->idx[d];
  }
  p.xv = x->val;
  p.yv = y->val;
  p.zv = z->val;
  uint64_t nvec = (all_aligned(x) && all_aligned(y) && all_aligned(z)) ? n / 4 : 0;
  if (nvec) {
    unsigned grid = spt::grid_for(nvec, 256, 1u << 30);
    SPT_ORDER_SWITCH(x->order, tew_eq_vec_kernel, grid, st, p, nvec, op, ctx->d_err);
    SPT_LAUNCHED(ctx);
  }
  if (nvec * 4 < n) {
    unsigned grid = spt::grid_for(n - nvec * 4, 256, ctx->num_sms * 8);
    tew_eq_scalar_kernel<<<grid, 256, 0, st>>>(p, x->order, nvec * 4, n, op, ctx->d_err);
    SPT_LAUNCHED(ctx);
  }
  if (flags & SPT_FLAG_ASYNC) return SPT_OK;
  return spt::sync_and_check(ctx, st);
}

}  // extern "C"
