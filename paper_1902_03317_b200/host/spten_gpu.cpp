// C++ drop-in layer (include/spten/gpu.hpp): the reference's signatures and
// types on top of the C-ABI (include/spten_b200.h). Host glue only -- every
// element of work runs in the sm_100a kernels behind the C-ABI; there is no
// CPU fallback. Built against the reference's headers (P/include); the
// spten::flops symbols resolve against the reference library the caller
// already links (P/src/flop_counter.cpp).
#include "spten/gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "spten/flop_counter.hpp"
#include "spten_b200.h"

namespace spten::gpu {
namespace {

[[noreturn]] void raise(int status) {
  const std::string msg = spt_last_error();
  switch (status) {
    case SPT_EINVAL: throw std::invalid_argument(msg);
    case SPT_EDOMAIN: throw std::domain_error(msg);
    case SPT_EOVERFLOW: throw std::overflow_error(msg);
    case SPT_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

inline void check(int status) {
  if (status != SPT_OK) raise(status);
}

inline void cuda(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// One context + stream per host thread and device (contexts are not
// thread-safe; streams keep concurrent callers independent).
struct Session {
  int device = -1;
  spt_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  ~Session() {
    if (ctx) spt_ctx_destroy(ctx);
    if (stream) cudaStreamDestroy(stream);
  }
};

Session& session() {
  thread_local Session s;
  int dev = 0;
  cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (s.device != dev) {
    if (s.ctx) spt_ctx_destroy(s.ctx);
    if (s.stream) cudaStreamDestroy(s.stream);
    s.ctx = nullptr;
    s.stream = nullptr;
    check(spt_ctx_create(dev, &s.ctx));
    cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    s.device = dev;
  }
  return s;
}

// Stream-ordered device buffer.
struct DBuf {
  void* p = nullptr;
  cudaStream_t st;
  DBuf(size_t bytes, cudaStream_t s) : st(s) {
    cuda(cudaMallocAsync(&p, bytes ? bytes : 16, st), "cudaMallocAsync");
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { cudaFreeAsync(p, st); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Device copy of a SparseTensorCOO<float> plus its C-ABI descriptor.
struct DevCoo {
  spt_coo d{};
  std::vector<DBuf*> bufs;
  cudaStream_t st;
  DevCoo(unsigned order, const std::vector<Index>& dims, size_t nnz, cudaStream_t s) : st(s) {
    if (order > SPT_MAX_ORDER)
      throw std::invalid_argument("spten::gpu: order exceeds " + std::to_string(SPT_MAX_ORDER));
    d.order = order;
    d.nnz = nnz;
    for (unsigned m = 0; m < order; ++m) {
      d.dims[m] = m < dims.size() ? dims[m] : 0;
      bufs.push_back(new DBuf(nnz * sizeof(Index), st));
      d.idx[m] = bufs.back()->as<uint32_t>();
    }
    bufs.push_back(new DBuf(nnz * sizeof(float), st));
    d.val = bufs.back()->as<float>();
  }
  ~DevCoo() {
    for (auto* b : bufs) delete b;
  }
  static DevCoo* upload(const SparseTensorCOO<float>& t, cudaStream_t s) {
    for (unsigned m = 0; m < t.order(); ++m)
      if (t.indices[m].size() != t.nnz())
        throw std::invalid_argument("spten::gpu: index array length != nnz");
    auto* dc = new DevCoo(t.order(), t.dims, t.nnz(), s);
    const size_t n = t.nnz();
    for (unsigned m = 0; m < t.order(); ++m)
      if (n) cuda(cudaMemcpyAsync(dc->d.idx[m], t.indices[m].data(), n * 4, cudaMemcpyHostToDevice, s), "H2D");
    if (n) cuda(cudaMemcpyAsync(dc->d.val, t.values.data(), n * 4, cudaMemcpyHostToDevice, s), "H2D");
    if (t.sort_order) {
      dc->d.has_sort_order = 1;
      for (unsigned m = 0; m < t.order(); ++m) dc->d.sort_order[m] = static_cast<int32_t>((*t.sort_order)[m]);
    }
    dc->d.coalesced = t.coalesced ? 1 : 0;
    return dc;
  }
  // Copy the first n entries and the metadata of descriptor `meta` back.
  void download(SparseTensorCOO<float>& t, const spt_coo& meta, size_t n) const {
    t.dims.assign(meta.dims, meta.dims + meta.order);
    t.indices.assign(meta.order, std::vector<Index>(n));
    t.values.resize(n);
    for (unsigned m = 0; m < meta.order; ++m)
      if (n) cuda(cudaMemcpyAsync(t.indices[m].data(), meta.idx[m], n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (n) cuda(cudaMemcpyAsync(t.values.data(), meta.val, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    cuda(cudaStreamSynchronize(st), "sync");
    if (meta.has_sort_order) t.sort_order = std::vector<unsigned>(meta.sort_order, meta.sort_order + meta.order);
    else t.sort_order.reset();
    t.coalesced = meta.coalesced != 0;
  }
};

struct Owned {
  DevCoo* p;
  explicit Owned(DevCoo* q) : p(q) {}
  ~Owned() { delete p; }
  DevCoo* operator->() const { return p; }
};

// check_fiber_kernel_inputs, P/src/kernel_detail.hpp:106-119 (host-side part)
void check_fiber(const SparseTensorCOO<float>& x, unsigned mode, const FiberIndex& fib,
                 const char* kernel) {
  const std::string k = kernel;
  if (x.order() < 2) throw std::invalid_argument(k + ": input must have order >= 2");
  if (mode >= x.order()) throw std::invalid_argument(k + ": mode out of range");
  if (!x.coalesced) throw std::invalid_argument(k + ": tensor must be coalesced");
  if (!x.sort_order || x.sort_order->back() != mode)
    throw std::invalid_argument(k + ": tensor must be sorted with the target mode last");
  if (fib.mode != mode || fib.fptr.empty() || fib.fptr.back() != x.nnz() ||
      fib.nfibs + 1 != fib.fptr.size())
    throw std::invalid_argument(k + ": fiber index does not match the tensor");
}

DBuf* upload_fptr(const FiberIndex& fib, cudaStream_t st) {
  std::vector<uint32_t> f(fib.fptr.size());
  for (size_t i = 0; i < f.size(); ++i) {
    if (fib.fptr[i] >= (size_t{1} << 32))
      throw std::overflow_error("spten::gpu: fiber offsets exceed the u32 device range");
    f[i] = static_cast<uint32_t>(fib.fptr[i]);
  }
  auto* b = new DBuf(f.size() * 4, st);
  cuda(cudaMemcpyAsync(b->p, f.data(), f.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
  cuda(cudaStreamSynchronize(st), "sync");  // f is a temporary
  return b;
}

}  // namespace

SparseTensorCOO<float> ts(const SparseTensorCOO<float>& x, float s, ScalarOp op) {
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  DevCoo dz(x.order(), x.dims, x.nnz(), S.stream);
  check(spt_ts_f32(S.ctx, &dx->d, s, static_cast<int>(op), &dz.d, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, x.nnz());
  flops::record(x.nnz());
  return z;
}

SparseTensorCOO<float> tew_eq(const SparseTensorCOO<float>& x, const SparseTensorCOO<float>& y,
                              ElemOp op) {
  // P/src/kernels_seq.cpp:14-17 (checked before any transfer)
  if (x.order() != y.order() || x.dims != y.dims)
    throw std::invalid_argument("tew_eq: tensors must have identical dimensions");
  if (x.nnz() != y.nnz())
    throw std::invalid_argument("tew_eq: tensors must have identical nonzero counts");
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  Owned dy(DevCoo::upload(y, S.stream));
  DevCoo dz(x.order(), x.dims, x.nnz(), S.stream);
  check(spt_tew_eq_f32(S.ctx, &dx->d, &dy->d, static_cast<int>(op), &dz.d, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, x.nnz());
  flops::record(x.nnz());
  return z;
}

SparseTensorCOO<float> tew(SparseTensorCOO<float>& x, SparseTensorCOO<float>& y, ElemOp op) {
  // check_tew_inputs, P/src/kernel_detail.hpp:36-45
  if (op == ElemOp::div)
    throw std::invalid_argument(
        "tew: div is not defined for mismatched patterns (unmatched entries divide by zero)");
  if (x.order() != y.order()) throw std::invalid_argument("tew: tensors must have the same order");
  if (!x.coalesced || !y.coalesced)
    throw std::invalid_argument("tew: both inputs must be coalesced");
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  Owned dy(DevCoo::upload(y, S.stream));
  // unify_tew_sort, P/src/kernel_detail.hpp:88-95: sort both ascending in
  // place unless they already share an order (and hand the sorted operands
  // back, as the reference's non-const references do).
  if (!(x.sort_order && y.sort_order && *x.sort_order == *y.sort_order)) {
    std::vector<uint32_t> asc(x.order());
    for (unsigned m = 0; m < x.order(); ++m) asc[m] = m;
    check(spt_sort_f32(S.ctx, &dx->d, asc.data(), 0, S.stream));
    check(spt_sort_f32(S.ctx, &dy->d, asc.data(), 0, S.stream));
    dx->download(x, dx->d, x.nnz());
    dy->download(y, dy->d, y.nnz());
  }
  const size_t cap = op == ElemOp::mul ? std::min(x.nnz(), y.nnz()) : x.nnz() + y.nnz();
  std::vector<Index> dims(x.order());
  for (unsigned m = 0; m < x.order(); ++m) dims[m] = std::max(x.dims[m], y.dims[m]);
  DevCoo dz(x.order(), dims, cap, S.stream);
  uint64_t nz = 0;
  check(spt_tew_f32(S.ctx, &dx->d, &dy->d, static_cast<int>(op), &dz.d, cap, &nz, nullptr, 0,
                    S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, nz);
  // matches + sub negations, P/src/kernel_detail.hpp:55-83
  flops::record(op == ElemOp::add ? x.nnz() + y.nnz() - nz : (op == ElemOp::sub ? y.nnz() : nz));
  return z;
}

SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, const FiberIndex& fib) {
  check_fiber(x, mode, fib, "ttv");
  if (v.len() != x.dims[mode])
    throw std::invalid_argument("ttv: vector length must match the mode dimension");
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  std::unique_ptr<DBuf> df(upload_fptr(fib, S.stream));
  DBuf dv(v.len() * 4, S.stream);
  if (v.len()) cuda(cudaMemcpyAsync(dv.p, v.data.data(), v.len() * 4, cudaMemcpyHostToDevice, S.stream), "H2D");
  std::vector<Index> od;
  for (unsigned d = 0; d < x.order(); ++d)
    if (d != mode) od.push_back(x.dims[d]);
  DevCoo dz(x.order() - 1, od, fib.nfibs, S.stream);
  check(spt_ttv_f32(S.ctx, &dx->d, dv.as<float>(), v.len(), mode, df->as<uint32_t>(), fib.nfibs,
                    &dz.d, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, fib.nfibs);
  flops::record(2 * x.nnz());
  return z;
}

SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode) {
  return ttv(x, v, mode, build_fiber_index(x, mode));
}

SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, const FiberIndex& fib) {
  check_fiber(x, mode, fib, "ttm");
  if (u.rows != x.dims[mode])
    throw std::invalid_argument("ttm: matrix rows must match the mode dimension");
  const size_t R = u.cols;
  if (R == 0) throw std::invalid_argument("ttm: matrix must have at least one column");
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  std::unique_ptr<DBuf> df(upload_fptr(fib, S.stream));
  DBuf du(u.data.size() * 4, S.stream);
  if (!u.data.empty())
    cuda(cudaMemcpyAsync(du.p, u.data.data(), u.data.size() * 4, cudaMemcpyHostToDevice, S.stream), "H2D");
  std::vector<Index> od = x.dims;
  od[mode] = static_cast<Index>(R);
  DevCoo dz(x.order(), od, fib.nfibs * R, S.stream);
  check(spt_ttm_f32(S.ctx, &dx->d, du.as<float>(), u.rows, R, mode, df->as<uint32_t>(),
                    fib.nfibs, &dz.d, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, fib.nfibs * R);
  flops::record(2 * R * x.nnz());
  return z;
}

SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode) {
  return ttm(x, u, mode, build_fiber_index(x, mode));
}

DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode,
                          MttkrpStrategy strategy) {
  // check_mttkrp_inputs, P/src/kernel_detail.hpp:153-174
  const unsigned N = x.order();
  if (N < 2) throw std::invalid_argument("mttkrp: input must have order >= 2");
  if (mode >= N) throw std::invalid_argument("mttkrp: mode out of range");
  if (!x.coalesced) throw std::invalid_argument("mttkrp: tensor must be coalesced");
  if (factors.size() != N) throw std::invalid_argument("mttkrp: need one factor matrix per mode");
  size_t R = 0;
  for (unsigned d = 0; d < N; ++d) {
    if (d == mode) continue;
    if (R == 0) R = factors[d].cols;
    if (factors[d].cols != R)
      throw std::invalid_argument("mttkrp: factor matrices must share the column count");
    if (factors[d].rows != x.dims[d])
      throw std::invalid_argument("mttkrp: factor rows must match the mode dimension");
  }
  if (R == 0) throw std::invalid_argument("mttkrp: factor rank must be >= 1");
  Session& S = session();
  Owned dx(DevCoo::upload(x, S.stream));
  int strat = SPT_MTTKRP_ATOMIC;
  if (strategy == MttkrpStrategy::privatize) {
    strat = SPT_MTTKRP_SEGMENTED;
    const bool leading = x.sort_order && (*x.sort_order)[0] == mode;
    if (!leading) {  // mode-leading copy (device sort, bit-exact permutation)
      std::vector<uint32_t> mo{mode};
      for (unsigned d = 0; d < N; ++d)
        if (d != mode) mo.push_back(d);
      check(spt_sort_f32(S.ctx, &dx->d, mo.data(), 0, S.stream));
    }
  }
  std::vector<DBuf*> fb;
  std::vector<const float*> fp(N, nullptr);
  std::vector<uint64_t> rows(N, 0), cols(N, 0);
  for (unsigned d = 0; d < N; ++d) {
    if (d == mode) continue;
    fb.push_back(new DBuf(factors[d].data.size() * 4, S.stream));
    if (!factors[d].data.empty())
      cuda(cudaMemcpyAsync(fb.back()->p, factors[d].data.data(), factors[d].data.size() * 4,
                           cudaMemcpyHostToDevice, S.stream), "H2D");
    fp[d] = fb.back()->as<float>();
    rows[d] = factors[d].rows;
    cols[d] = factors[d].cols;
  }
  DenseMatrix<float> out(x.dims[mode], R);
  DBuf dout(out.data.size() * 4, S.stream);
  int st = spt_mttkrp_f32(S.ctx, &dx->d, fp.data(), rows.data(), cols.data(), mode,
                          dout.as<float>(), strat, 0, S.stream);
  if (st == SPT_OK && !out.data.empty())
    cuda(cudaMemcpyAsync(out.data.data(), dout.p, out.data.size() * 4, cudaMemcpyDeviceToHost,
                         S.stream), "D2H");
  if (st == SPT_OK) cuda(cudaStreamSynchronize(S.stream), "sync");
  for (auto* b : fb) delete b;
  check(st);
  flops::record(static_cast<std::uint64_t>(x.nnz()) * N * R);
  return out;
}

DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode) {
  return mttkrp(x, factors, mode, MttkrpStrategy::privatize);
}

void sort_lexicographic(SparseTensorCOO<float>& t, std::span<const unsigned> mode_order) {
  // check_mode_order, P/src/tensor.cpp:28-37
  if (mode_order.size() != t.order())
    throw std::invalid_argument("sort_lexicographic: mode order has wrong length");
  std::vector<bool> seen(t.order(), false);
  for (unsigned d : mode_order) {
    if (d >= t.order() || seen[d])
      throw std::invalid_argument("sort_lexicographic: mode order is not a permutation");
    seen[d] = true;
  }
  Session& S = session();
  Owned dt(DevCoo::upload(t, S.stream));
  std::vector<uint32_t> mo(mode_order.begin(), mode_order.end());
  check(spt_sort_f32(S.ctx, &dt->d, mo.data(), 0, S.stream));
  dt->download(t, dt->d, t.nnz());
}

SparseTensorCOO<float> coalesce(const SparseTensorCOO<float>& t) {
  Session& S = session();
  Owned dt(DevCoo::upload(t, S.stream));
  if (!t.sort_order) {
    std::vector<uint32_t> asc(t.order());
    for (unsigned m = 0; m < t.order(); ++m) asc[m] = m;
    check(spt_sort_f32(S.ctx, &dt->d, asc.data(), 0, S.stream));
  }
  DevCoo dz(t.order(), t.dims, t.nnz(), S.stream);
  uint64_t n = 0;
  check(spt_coalesce_f32(S.ctx, &dt->d, &dz.d, &n, nullptr, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, n);
  return z;
}

FiberIndex build_fiber_index(const SparseTensorCOO<float>& t, unsigned mode) {
  // P/src/tensor.cpp:94-99 (checked before any transfer)
  if (mode >= t.order()) throw std::invalid_argument("build_fiber_index: mode out of range");
  if (!t.sort_order || t.sort_order->back() != mode)
    throw std::invalid_argument(
        "build_fiber_index: tensor must be sorted with the target mode as the last key");
  Session& S = session();
  Owned dt(DevCoo::upload(t, S.stream));
  DBuf fptr((t.nnz() + 1) * 4, S.stream);
  uint64_t nf = 0;
  check(spt_fiber_index(S.ctx, &dt->d, mode, fptr.as<uint32_t>(), &nf, nullptr, 0, S.stream));
  std::vector<uint32_t> f(nf + 1);
  cuda(cudaMemcpyAsync(f.data(), fptr.p, (nf + 1) * 4, cudaMemcpyDeviceToHost, S.stream), "D2H");
  cuda(cudaStreamSynchronize(S.stream), "sync");
  FiberIndex fib;
  fib.mode = mode;
  fib.nfibs = nf;
  fib.fptr.assign(f.begin(), f.end());
  return fib;
}

}  // namespace spten::gpu
