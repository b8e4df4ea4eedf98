// Single-process multi-GPU MTTKRP through the C-ABI.
//
// The reference's only parallel reduction of MTTKRP is the private-buffer
// sum of par::mttkrp's privatize strategy (P/src/kernels_par.cpp:290-319).
// Across GPUs the tensor is split into row-aligned shards instead: the entry
// ranges of the mode-leading sorted tensor are cut at row starts
// (spt_row_aligned_cuts), so every output row is computed whole, by one
// device, in the single-GPU entry order. Each device writes its shard's
// I_n x R result into its own buffer -- exact on the row block it owns, zero
// elsewhere -- and one NCCL group of in-place broadcasts (root k sends rows
// [row_lo[k], row_lo[k+1])) leaves the whole result on every device: each
// device receives (G-1)/G of the output, half of an all-reduce's traffic, and
// no partial sums cross devices (bit-identical to one GPU on the same shards).
// NCCL is loaded on first use (dlopen), so single-GPU callers never need it.
#include <dlfcn.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace {

// The few NCCL entry points used (nccl.h types as plain ints/pointers).
struct Nccl {
  using Comm = void*;
  int (*CommInitAll)(Comm*, int, const int*) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
  static Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return;
      n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(h, "ncclBroadcast"));
      n.GetErrorString =
          reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      n.ok = n.CommInitAll && n.GroupStart && n.GroupEnd && n.Broadcast && n.GetErrorString;
    });
    return n;
  }
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32 in nccl.h

// One communicator set per device list, kept for the process.
std::vector<Nccl::Comm>* comms_for(const std::vector<int>& devs, int* status) {
  static std::mutex m;
  static std::map<std::vector<int>, std::vector<Nccl::Comm>> cache;
  std::lock_guard<std::mutex> lk(m);
  auto it = cache.find(devs);
  if (it != cache.end()) return &it->second;
  Nccl& n = Nccl::get();
  if (!n.ok) {
    *status = spt::set_error(SPT_ERUNTIME, "mttkrp_multi: NCCL (libnccl.so.2) not available");
    return nullptr;
  }
  std::vector<Nccl::Comm> c(devs.size(), nullptr);
  const int r = n.CommInitAll(c.data(), static_cast<int>(devs.size()), devs.data());
  if (r != 0) {
    *status = spt::set_error(SPT_ERUNTIME, "ncclCommInitAll: %s", n.GetErrorString(r));
    return nullptr;
  }
  return &cache.emplace(devs, std::move(c)).first->second;
}

// cuts[p] for p = 1..parts-1: the row start at or below the equal-nnz point
// p*nnz/parts, or that row's end when it started before the previous cut
// (sequential over p: parts is the device count).
__global__ void row_cuts_kernel(const uint32_t* rows, uint64_t nnz, uint32_t parts,
                                uint64_t* cuts, uint32_t* row_lo, uint32_t I) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  auto lower = [&](uint32_t v) {  // first entry with row >= v
    uint64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (rows[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  cuts[0] = 0;
  for (uint32_t p = 1; p < parts; ++p) {
    const uint64_t t = nnz * p / parts;
    uint64_t c = nnz;
    if (t < nnz) {
      const uint32_t r = rows[t];
      c = lower(r);
      if (c <= cuts[p - 1]) c = r == 0xFFFFFFFFu ? nnz : lower(r + 1);
    }
    cuts[p] = c > cuts[p - 1] ? c : cuts[p - 1];
  }
  cuts[parts] = nnz;
  // owned row blocks (parallel.row_blocks): from a shard's first row to the
  // next non-empty shard's first row; the first non-empty shard from row 0
  uint32_t next = I;
  for (int p = static_cast<int>(parts) - 1; p >= 0; --p) {
    if (cuts[p] < cuts[p + 1]) next = rows[cuts[p]];
    row_lo[p] = next;
  }
  row_lo[0] = 0;
  row_lo[parts] = I;
}

}  // namespace

extern "C" int spt_row_aligned_cuts(spt_ctx* ctx, const spt_coo* x, uint32_t mode,
                                    uint32_t parts, uint64_t* entry_cuts, uint32_t* row_lo,
                                    void* stream) {
  if (!ctx) return spt::set_error(SPT_EINVAL, "row_aligned_cuts: null context");
  SPT_TRY(spt::check_coo(x, "row_aligned_cuts", false));
  if (mode >= x->order) return spt::set_error(SPT_EINVAL, "row_aligned_cuts: mode out of range");
  if (parts < 1) return spt::set_error(SPT_EINVAL, "row_aligned_cuts: parts must be >= 1");
  if (!x->has_sort_order || static_cast<uint32_t>(x->sort_order[0]) != mode)
    return spt::set_error(SPT_EINVAL, "row_aligned_cuts: x must be sorted with the mode leading");
  if (!entry_cuts || !row_lo) return spt::set_error(SPT_EINVAL, "row_aligned_cuts: null output");
  cudaStream_t st = spt::as_stream(stream);
  uint64_t* dcuts;
  SPT_CUDA(spt::tmp_alloc(ctx, &dcuts, (parts + 1) * (sizeof(uint64_t) + sizeof(uint32_t)), st));
  uint32_t* drow = reinterpret_cast<uint32_t*>(dcuts + parts + 1);
  row_cuts_kernel<<<1, 32, 0, st>>>(x->idx[mode], x->nnz, parts, dcuts, drow, x->dims[mode]);
  SPT_LAUNCHED(ctx);
  SPT_CUDA(cudaMemcpyAsync(entry_cuts, dcuts, (parts + 1) * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, st));
  SPT_CUDA(cudaMemcpyAsync(row_lo, drow, (parts + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           st));
  SPT_CUDA(cudaFreeAsync(dcuts, st));
  SPT_CUDA(cudaStreamSynchronize(st));
  return SPT_OK;
}

extern "C" int spt_mttkrp_f32_multi(int ndev, spt_ctx* const* ctxs, const spt_coo* shards,
                                    const uint32_t* row_lo, const float* const* d_factors,
                                    const uint64_t* rows, const uint64_t* cols, uint32_t mode,
                                    float* const* d_out, void* const* streams) {
  if (ndev < 1 || !ctxs || !shards || !row_lo || !d_factors || !d_out || !streams)
    return spt::set_error(SPT_EINVAL, "mttkrp_multi: null argument or ndev < 1");
  const uint32_t N = shards[0].order;
  std::vector<int> devs(ndev);
  uint64_t R = 0;
  for (uint32_t d = 0; d < N; ++d)
    if (d != mode) R = R ? R : cols[d];
  for (int k = 0; k < ndev; ++k) {
    if (!ctxs[k]) return spt::set_error(SPT_EINVAL, "mttkrp_multi: null context %d", k);
    devs[k] = ctxs[k]->device;
    if (shards[k].order != N || shards[k].dims[mode] != shards[0].dims[mode])
      return spt::set_error(SPT_EINVAL, "mttkrp_multi: shards must share order and dims");
    if (k && row_lo[k] < row_lo[k - 1])
      return spt::set_error(SPT_EINVAL, "mttkrp_multi: row blocks must be increasing");
  }
  for (int a = 0; a < ndev; ++a)
    for (int b = a + 1; b < ndev; ++b)
      if (devs[a] == devs[b])
        return spt::set_error(SPT_EINVAL, "mttkrp_multi: one context per distinct device");
  const uint32_t I = shards[0].dims[mode];
  if (row_lo[0] != 0 || row_lo[ndev] != I)
    return spt::set_error(SPT_EINVAL, "mttkrp_multi: row blocks must cover [0, dims[mode])");
  // every device: its shard's rows, exact; zero outside them
  for (int k = 0; k < ndev; ++k) {
    SPT_CUDA(cudaSetDevice(devs[k]));
    const int s = spt_mttkrp_f32(ctxs[k], &shards[k], d_factors + (size_t)k * N, rows, cols, mode,
                                 d_out[k], SPT_MTTKRP_AUTO, SPT_FLAG_ASYNC, streams[k]);
    if (s != SPT_OK) return s;
  }
  if (ndev > 1) {
    int status = SPT_OK;
    auto* comms = comms_for(devs, &status);
    if (!comms) return status;
    Nccl& n = Nccl::get();
    n.GroupStart();
    for (int root = 0; root < ndev; ++root) {
      const size_t off = (size_t)row_lo[root] * R;
      const size_t count = (size_t)(row_lo[root + 1] - row_lo[root]) * R;
      if (!count) continue;
      for (int k = 0; k < ndev; ++k)
        n.Broadcast(d_out[k] + off, d_out[k] + off, count, kNcclFloat32, root, (*comms)[k],
                    spt::as_stream(streams[k]));
    }
    const int r = n.GroupEnd();
    if (r != 0) return spt::set_error(SPT_ERUNTIME, "nccl broadcast group: %s", n.GetErrorString(r));
  }
  for (int k = 0; k < ndev; ++k) {
    SPT_CUDA(cudaSetDevice(devs[k]));
    SPT_TRY(spt::sync_and_check(ctxs[k], spt::as_stream(streams[k])));
  }
  return SPT_OK;
}
