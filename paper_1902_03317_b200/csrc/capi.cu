// Library plumbing behind include/spten_b200.h: contexts, errors, scratch,
// deferred error decoding, L2 flush and the uniform generator.
#include <cstring>
#include <mutex>

#include "internal.cuh"

namespace {
thread_local std::string g_last_error;
}

namespace spt {

int set_error(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_error(SPT_ENOMEM, "CUDA out of memory in %s", what);
  }
  return set_error(SPT_ERUNTIME, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

int ctx_scratch(spt_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->scratch) {
      SPT_CUDA(cudaDeviceSynchronize());
      SPT_CUDA(cudaFree(ctx->scratch));
      ctx->scratch = nullptr;
      ctx->scratch_bytes = 0;
    }
    size_t want = bytes + bytes / 4 + 256;
    SPT_CUDA(cudaMalloc(&ctx->scratch, want));
    ctx->scratch_bytes = want;
  }
  *out = ctx->scratch;
  return SPT_OK;
}

int ctx_lookback(spt_ctx* ctx, size_t tiles, size_t payload_doubles, uint32_t* epoch) {
  if (tiles > ctx->status_cap) {
    if (ctx->d_status) {
      SPT_CUDA(cudaDeviceSynchronize());
      SPT_CUDA(cudaFree(ctx->d_status));
      ctx->d_status = nullptr;
    }
    size_t cap = tiles + tiles / 4 + 64;
    SPT_CUDA(cudaMalloc(&ctx->d_status, cap * sizeof(uint32_t)));
    SPT_CUDA(cudaMemset(ctx->d_status, 0, cap * sizeof(uint32_t)));
    ctx->status_cap = cap;  // fresh words are epoch 0, which is never issued
  }
  if (payload_doubles > ctx->payload_cap) {
    if (ctx->d_payload) {
      SPT_CUDA(cudaDeviceSynchronize());
      SPT_CUDA(cudaFree(ctx->d_payload));
      ctx->d_payload = nullptr;
    }
    size_t cap = payload_doubles + payload_doubles / 4 + 256;
    SPT_CUDA(cudaMalloc(&ctx->d_payload, cap * sizeof(double)));
    ctx->payload_cap = cap;
  }
  // Status word = (epoch << 3) | flags; 29-bit epoch, 0 reserved for "never".
  ctx->epoch = (ctx->epoch + 1) & 0x1FFFFFFFu;
  if (ctx->epoch == 0) {
    SPT_CUDA(cudaDeviceSynchronize());
    SPT_CUDA(cudaMemset(ctx->d_status, 0, ctx->status_cap * sizeof(uint32_t)));
    if (ctx->d_status64)
      SPT_CUDA(cudaMemset(ctx->d_status64, 0, ctx->status64_cap * sizeof(unsigned long long)));
    ctx->epoch = 1;
  }
  *epoch = ctx->epoch;
  return SPT_OK;
}

int ctx_status64(spt_ctx* ctx, size_t tiles, unsigned long long** out) {
  if (tiles > ctx->status64_cap) {
    if (ctx->d_status64) {
      SPT_CUDA(cudaDeviceSynchronize());
      SPT_CUDA(cudaFree(ctx->d_status64));
      ctx->d_status64 = nullptr;
    }
    size_t cap = tiles + tiles / 4 + 64;
    SPT_CUDA(cudaMalloc(&ctx->d_status64, cap * sizeof(unsigned long long)));
    SPT_CUDA(cudaMemset(ctx->d_status64, 0, cap * sizeof(unsigned long long)));
    ctx->status64_cap = cap;
  }
  *out = ctx->d_status64;
  return SPT_OK;
}

int check_coo(const spt_coo* t, const char* who, bool need_values) {
  if (!t) return set_error(SPT_EINVAL, "%s: null tensor descriptor", who);
  if (t->order < 1 || t->order > SPT_MAX_ORDER)
    return set_error(SPT_EINVAL, "%s: order %u outside 1..%d", who, t->order, SPT_MAX_ORDER);
  if (t->nnz >= (1ull << 32))
    return set_error(SPT_EOVERFLOW, "%s: nnz %llu exceeds the u32 device offset range; shard it",
                     who, (unsigned long long)t->nnz);
  if (t->nnz > 0) {
    for (uint32_t d = 0; d < t->order; ++d)
      if (!t->idx[d]) return set_error(SPT_EINVAL, "%s: null index array for mode %u", who, d);
    if (need_values && !t->val) return set_error(SPT_EINVAL, "%s: null value array", who);
  }
  if (t->has_sort_order) {
    bool seen[SPT_MAX_ORDER] = {false};
    for (uint32_t d = 0; d < t->order; ++d) {
      int32_t m = t->sort_order[d];
      if (m < 0 || static_cast<uint32_t>(m) >= t->order || seen[m])
        return set_error(SPT_EINVAL, "%s: sort_order is not a permutation", who);
      seen[m] = true;
    }
  }
  return SPT_OK;
}

int sync_and_check(spt_ctx* ctx, cudaStream_t stream) {
  SPT_CUDA(cudaStreamSynchronize(stream));
  unsigned long long err[4];
  SPT_CUDA(cudaMemcpy(err, ctx->d_err, sizeof err, cudaMemcpyDeviceToHost));
  const unsigned long long none = ~0ull;
  if (err[0] == none && err[1] == none && err[2] == none && err[3] == none) return SPT_OK;
  SPT_CUDA(cudaMemset(ctx->d_err, 0xFF, sizeof err));
  // tew_eq: seq throws at the first failing entry, checking the pattern
  // before the divisor (P/src/kernels_seq.cpp:27-36).
  if (err[0] != none && err[0] <= err[1])
    return set_error(SPT_EINVAL, "tew_eq: nonzero patterns differ at entry %llu", err[0]);
  if (err[1] != none)
    return set_error(SPT_EDOMAIN, "tew_eq: division by a stored zero at entry %llu", err[1]);
  if (err[2] != none)
    return set_error(SPT_EINVAL,
                     "mttkrp: segmented strategy needs entries sorted by the output mode "
                     "(violation at entry %llu)",
                     err[2]);
  return set_error(SPT_EINVAL, "device check failed at entry %llu", err[3]);
}

}  // namespace spt

// ---------------------------------------------------------------------------

namespace {

// Evicts the L2 by *reading* a buffer twice its size, so it is left full of
// clean lines: a write-based flush would leave ~126 MB of dirty lines whose
// write-back the next (timed) kernel would pay for.
__global__ void l2_flush_kernel(const uint4* buf, size_t n16, uint32_t salt, uint32_t* sink) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (; i < n16; i += stride) {
    const uint4 v = __ldcg(buf + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == salt) sink[threadIdx.x] = acc;  // practically never; keeps the loads live
}

__global__ void uniform_kernel(float* out, uint64_t n, uint64_t seed, uint64_t sid, float lo,
                               float hi) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float w = hi - lo;
  for (uint64_t q = i; q * 4 < n; q += stride) {
    uint4 r = spt::Philox::gen(q, sid, seed);
    uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint64_t m = q * 4 + k;
      if (m < n) {
        float v = lo + w * spt::u01(rr[k]);
        out[m] = v < hi ? v : lo;  // keep [lo, hi) under rounding
      }
    }
  }
}

}  // namespace

extern "C" {

int spt_abi_version(void) { return SPT_ABI_VERSION; }

const char* spt_last_error(void) { return g_last_error.c_str(); }

int spt_ctx_create(int device, spt_ctx** out) {
  if (!out) return spt::set_error(SPT_EINVAL, "spt_ctx_create: null out");
  *out = nullptr;
  SPT_CUDA(cudaSetDevice(device));
  spt_ctx* c = new spt_ctx();
  c->device = device;
  cudaDeviceProp prop;
  SPT_CUDA(cudaGetDeviceProperties(&prop, device));
  c->num_sms = prop.multiProcessorCount;
  c->l2_bytes = prop.l2CacheSize;
  SPT_CUDA(cudaMalloc(&c->d_err, 4 * sizeof(unsigned long long)));
  SPT_CUDA(cudaMemset(c->d_err, 0xFF, 4 * sizeof(unsigned long long)));
  SPT_CUDA(cudaMalloc(&c->d_tile_ctr, 4 * sizeof(unsigned long long)));
  SPT_CUDA(cudaMemset(c->d_tile_ctr, 0, 4 * sizeof(unsigned long long)));
  SPT_CUDA(cudaMallocHost(&c->h_pinned, 8 * sizeof(unsigned long long)));
  // Stream-ordered temporaries (sort permutations, plan copies) come from a
  // private pool that keeps its freed memory mapped (no unmap/remap of tens
  // of MB per call); spt_ctx_trim hands it back. The device's default pool
  // -- the caller's -- is left alone.
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  SPT_CUDA(cudaMemPoolCreate(&c->pool, &props));
  uint64_t keep = ~0ull;
  SPT_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  *out = c;
  return SPT_OK;
}

void spt_ctx_destroy(spt_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  cudaFree(c->d_err);
  cudaFree(c->d_tile_ctr);
  cudaFree(c->scratch);
  cudaFree(c->d_status);
  cudaFree(c->d_payload);
  cudaFree(c->d_status64);
  cudaFree(c->l2buf);
  cudaFreeHost(c->h_pinned);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  delete c;
}

int spt_ctx_trim(spt_ctx* c) {
  if (!c) return spt::set_error(SPT_EINVAL, "spt_ctx_trim: null context");
  SPT_CUDA(cudaSetDevice(c->device));
  SPT_CUDA(cudaDeviceSynchronize());
  cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_bytes = 0;
  cudaFree(c->d_status);
  c->d_status = nullptr;
  c->status_cap = 0;
  cudaFree(c->d_payload);
  c->d_payload = nullptr;
  c->payload_cap = 0;
  cudaFree(c->d_status64);
  c->d_status64 = nullptr;
  c->status64_cap = 0;
  cudaFree(c->l2buf);
  c->l2buf = nullptr;
  c->l2buf_bytes = 0;
  SPT_CUDA(cudaMemPoolTrimTo(c->pool, 0));
  return SPT_OK;
}

uint64_t spt_ctx_launches(const spt_ctx* c) { return c ? c->launches : 0; }

int spt_ctx_check(spt_ctx* ctx, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "spt_ctx_check: null context");
  return spt::sync_and_check(ctx, spt::as_stream(stream));
}

int spt_l2_flush(spt_ctx* ctx, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "spt_l2_flush: null context");
  size_t want = (ctx->l2_bytes ? ctx->l2_bytes : (126u << 20)) * 2;
  if (ctx->l2buf_bytes < want) {
    cudaFree(ctx->l2buf);
    ctx->l2buf = nullptr;
    SPT_CUDA(cudaMalloc(&ctx->l2buf, want + 4096));
    SPT_CUDA(cudaMemset(ctx->l2buf, 0x5a, want + 4096));
    SPT_CUDA(cudaDeviceSynchronize());
    ctx->l2buf_bytes = want;
  }
  l2_flush_kernel<<<ctx->num_sms * 4, 512, 0, spt::as_stream(stream)>>>(
      static_cast<const uint4*>(ctx->l2buf), ctx->l2buf_bytes / 16, 0x12345678u,
      reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->l2buf) + ctx->l2buf_bytes));
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

int spt_gen_uniform_f32(spt_ctx* ctx, float* d_out, uint64_t n, uint64_t seed, uint64_t sid,
                        float lo, float hi, void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "spt_gen_uniform_f32: null context");
  if (n == 0) return SPT_OK;
  if (!d_out) return spt::set_error(SPT_EINVAL, "spt_gen_uniform_f32: null output");
  unsigned grid = spt::grid_for((n + 3) / 4, 256, ctx->num_sms * 8);
  uniform_kernel<<<grid, 256, 0, spt::as_stream(stream)>>>(d_out, n, seed, sid, lo, hi);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

}  // extern "C"
