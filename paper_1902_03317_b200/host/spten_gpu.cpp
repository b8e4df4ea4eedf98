// C++ drop-in layer (include/spten/gpu.hpp): the reference's signatures and
// types on top of the C-ABI (include/spten_b200.h). Host glue only -- every
// element of work runs in the sm_100a kernels behind the C-ABI; there is no
// CPU fallback. Built against the reference's headers (P/include); the
// spten::flops symbols resolve against the reference library the caller
// already links (P/src/flop_counter.cpp).
#include "spten/gpu.hpp"

#include <cuda_runtime.h>

#include <fcntl.h>
#include <pthread.h>
#include <sys/stat.h>
#include <unistd.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <optional>
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

// Per host thread and device: a context, a compute stream and two copy
// streams, grow-only device buffers reused across calls (no allocation in the
// steady state) and pinned bounce buffers, so host <-> device traffic from the
// caller's pageable std::vectors runs at PCIe speed: the host copies chunk k
// into a pinned buffer (several threads) while the DMA engine moves chunk k-1.
constexpr size_t kChunk = size_t(32) << 20;  // bytes per pinned bounce buffer

// SPT_DROPIN_TRACE=1: per-phase host times of every call on stderr (tuning).
struct Trace {
  const bool on = std::getenv("SPT_DROPIN_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dropin] %-12s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// Host copies between the caller's pageable vectors and the pinned buffers,
// split over a small persistent thread pool (std::thread: independent of the
// caller's OpenMP settings -- OMP_PROC_BIND=close, set for the reference's
// kernels, packed OpenMP copies onto a few cores at ~8 GB/s).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool p;
    return p;
  }
  void memcpy(void* dst, const void* src, size_t n) {
    constexpr size_t kPiece = size_t(1) << 20;
    if (n <= 2 * kPiece || workers_.empty()) {
      std::memcpy(dst, src, n);
      return;
    }
    run(static_cast<char*>(dst), static_cast<const char*>(src), -1, 0, n);
  }
  // n bytes of file fd from offset off into dst, in parallel pieces; false on
  // a read error or a short file.
  bool pread(void* dst, int fd, uint64_t off, size_t n) {
    read_error_.store(false);
    run(static_cast<char*>(dst), nullptr, fd, off, n);
    return !read_error_.load();
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  void run(char* dst, const char* src, int fd, uint64_t off, size_t n) {
    std::unique_lock<std::mutex> lk(m_);
    dst_ = dst;
    src_ = src;
    fd_ = fd;
    foff_ = off;
    n_ = n;
    next_.store(0);
    busy_ = static_cast<int>(workers_.size());
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    work();
    lk.lock();
    done_.wait(lk, [&] { return busy_ == 0; });
  }
  CopyPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    for (unsigned i = 0; i < std::min(hw, 8u) - 1; ++i)
      workers_.emplace_back([this, hw] {
        // a thread inherits its creator's CPU mask: a caller whose OpenMP
        // runtime pinned the main thread (OMP_PROC_BIND) would put every
        // copy worker on that one core
        cpu_set_t all;
        CPU_ZERO(&all);
        for (unsigned c = 0; c < hw && c < CPU_SETSIZE; ++c) CPU_SET(c, &all);
        pthread_setaffinity_np(pthread_self(), sizeof all, &all);
        uint64_t seen = 0;
        while (true) {
          {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            if (stop_) return;
          }
          work();
          std::lock_guard<std::mutex> lk(m_);
          if (--busy_ == 0) done_.notify_one();
        }
      });
  }
  void work() {
    constexpr size_t kPiece = size_t(1) << 20;
    for (size_t o; (o = next_.fetch_add(kPiece)) < n_;) {
      const size_t c = std::min(kPiece, n_ - o);
      if (fd_ < 0) {
        std::memcpy(dst_ + o, src_ + o, c);
        continue;
      }
      for (size_t got = 0; got < c;) {
        const ssize_t r = ::pread(fd_, dst_ + o + got, c - got, static_cast<off_t>(foff_ + o + got));
        if (r <= 0) {
          read_error_.store(true);
          break;
        }
        got += static_cast<size_t>(r);
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  int busy_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0};
  int fd_ = -1;
  uint64_t foff_ = 0;
  std::atomic<bool> read_error_{false};
};

void par_memcpy(void* dst, const void* src, size_t n) { CopyPool::get().memcpy(dst, src, n); }

struct Session {
  int device = -1;
  spt_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr, h2d = nullptr, d2h = nullptr;
  void* pin[4] = {};  // [0,1] upload, [2,3] download
  cudaEvent_t ev[4] = {}, done_h2d = nullptr, done_cmp = nullptr;
  std::vector<std::pair<void*, size_t>> slots;  // grow-only device buffers
  int next = 0;  // round robin over the two upload buffers
  ~Session() { release(); }
  void release() {
    if (device < 0) return;
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    if (ctx) spt_ctx_destroy(ctx);
    for (auto& s : slots) cudaFree(s.first);
    for (int i = 0; i < 4; ++i) {
      if (pin[i]) cudaFreeHost(pin[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    for (cudaStream_t s : {stream, h2d, d2h})
      if (s) cudaStreamDestroy(s);
    if (done_h2d) cudaEventDestroy(done_h2d);
    if (done_cmp) cudaEventDestroy(done_cmp);
    *this = Session();
    device = -1;
  }
  Session& operator=(const Session&) = default;

  // Device buffer `slot`, at least `bytes`, kept across calls.
  void* buf(size_t slot, size_t bytes) {
    if (slots.size() <= slot) slots.resize(slot + 1, {nullptr, 0});
    auto& s = slots[slot];
    if (s.second < bytes || !s.first) {
      cuda(cudaStreamSynchronize(stream), "sync");
      if (s.first) cudaFree(s.first);
      s = {nullptr, 0};
      const size_t want = std::max<size_t>(bytes + bytes / 8, 256);
      cuda(cudaMalloc(&s.first, want), "cudaMalloc");
      s.second = want;
    }
    return s.first;
  }

  // Pageable host -> device through the pinned ring (stream h2d).
  double t_wait = 0, t_copy = 0;  // SPT_DROPIN_TRACE accounting
  void upload(void* dst, const void* src, size_t n) {
    if (!n) return;
    for (size_t o = 0; o < n; o += kChunk) {
      const size_t c = std::min(kChunk, n - o);
      const int k = next;
      next ^= 1;
      const auto t0 = std::chrono::steady_clock::now();
      cuda(cudaEventSynchronize(ev[k]), "sync");  // the DMA out of this buffer is done
      const auto t1 = std::chrono::steady_clock::now();
      par_memcpy(pin[k], static_cast<const char*>(src) + o, c);
      t_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
      t_copy += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
      cuda(cudaMemcpyAsync(static_cast<char*>(dst) + o, pin[k], c, cudaMemcpyHostToDevice, h2d),
           "H2D");
      cuda(cudaEventRecord(ev[k], h2d), "event");
    }
  }
  // Compute stream waits for every upload issued so far.
  void uploads_done() {
    cuda(cudaEventRecord(done_h2d, h2d), "event");
    cuda(cudaStreamWaitEvent(stream, done_h2d, 0), "wait");
  }
  // Device -> pageable host after the compute stream's work so far: DMA of
  // chunk k overlaps the host copy of chunk k-1.
  void download(void* dst, const void* src, size_t n) {
    if (!n) return;
    cuda(cudaEventRecord(done_cmp, stream), "event");
    cuda(cudaStreamWaitEvent(d2h, done_cmp, 0), "wait");
    size_t prev_o = 0, prev_c = 0;
    int prev_k = -1, k = 2;
    for (size_t o = 0; o < n; o += kChunk) {
      const size_t c = std::min(kChunk, n - o);
      cuda(cudaMemcpyAsync(pin[k], static_cast<const char*>(src) + o, c, cudaMemcpyDeviceToHost,
                           d2h), "D2H");
      cuda(cudaEventRecord(ev[k], d2h), "event");
      if (prev_k >= 0) {
        cuda(cudaEventSynchronize(ev[prev_k]), "sync");
        par_memcpy(static_cast<char*>(dst) + prev_o, pin[prev_k], prev_c);
      }
      prev_k = k, prev_o = o, prev_c = c;
      k = k == 2 ? 3 : 2;
    }
    cuda(cudaEventSynchronize(ev[prev_k]), "sync");
    par_memcpy(static_cast<char*>(dst) + prev_o, pin[prev_k], prev_c);
  }
};

Session& session() {
  thread_local Session s;
  int dev = 0;
  cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (s.device != dev) {
    s.release();
    check(spt_ctx_create(dev, &s.ctx));
    for (cudaStream_t* p : {&s.stream, &s.h2d, &s.d2h})
      cuda(cudaStreamCreateWithFlags(p, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < 4; ++i) {
      cuda(cudaMallocHost(&s.pin[i], kChunk), "cudaMallocHost");
      cuda(cudaEventCreateWithFlags(&s.ev[i], cudaEventDisableTiming), "event");
    }
    cuda(cudaEventCreateWithFlags(&s.done_h2d, cudaEventDisableTiming), "event");
    cuda(cudaEventCreateWithFlags(&s.done_cmp, cudaEventDisableTiming), "event");
    s.device = dev;
  }
  return s;
}

// Device buffer slots of one call: tensors take 9 slots each (N <= 8 index
// arrays + values).
enum Slot : size_t { kX = 0, kY = 9, kZ = 18, kF = 27, kOut = 36, kAux = 37, kAux2 = 38 };

// A SparseTensorCOO<float> in session slots, with its C-ABI descriptor.
struct DevCoo {
  spt_coo d{};
  Session* S;
  DevCoo(Session& s, size_t base, unsigned order, const std::vector<Index>& dims, size_t nnz)
      : S(&s) {
    if (order > SPT_MAX_ORDER)
      throw std::invalid_argument("spten::gpu: order exceeds " + std::to_string(SPT_MAX_ORDER));
    d.order = order;
    d.nnz = nnz;
    for (unsigned m = 0; m < order; ++m) {
      d.dims[m] = m < dims.size() ? dims[m] : 0;
      d.idx[m] = static_cast<uint32_t*>(s.buf(base + m, nnz * sizeof(Index)));
    }
    d.val = static_cast<float*>(s.buf(base + 8, nnz * sizeof(float)));
  }
  static DevCoo upload(Session& s, size_t base, const SparseTensorCOO<float>& t) {
    for (unsigned m = 0; m < t.order(); ++m)
      if (t.indices[m].size() != t.nnz())
        throw std::invalid_argument("spten::gpu: index array length != nnz");
    DevCoo dc(s, base, t.order(), t.dims, t.nnz());
    const size_t n = t.nnz();
    for (unsigned m = 0; m < t.order(); ++m) s.upload(dc.d.idx[m], t.indices[m].data(), n * 4);
    s.upload(dc.d.val, t.values.data(), n * 4);
    if (t.sort_order) {
      dc.d.has_sort_order = 1;
      for (unsigned m = 0; m < t.order(); ++m)
        dc.d.sort_order[m] = static_cast<int32_t>((*t.sort_order)[m]);
    }
    dc.d.coalesced = t.coalesced ? 1 : 0;
    return dc;
  }
  // Copy the first n entries and the metadata of descriptor `meta` back.
  void download(SparseTensorCOO<float>& t, const spt_coo& meta, size_t n) const {
    Trace tr;
    t.dims.assign(meta.dims, meta.dims + meta.order);
    t.indices.resize(meta.order);  // by-value outputs (the reference API): one
    for (auto& ix : t.indices) ix.resize(n);  // value-init pass each, no copies
    t.values.resize(n);
    tr.mark("  alloc");
    for (unsigned m = 0; m < meta.order; ++m) S->download(t.indices[m].data(), meta.idx[m], n * 4);
    S->download(t.values.data(), meta.val, n * 4);
    if (meta.has_sort_order)
      t.sort_order = std::vector<unsigned>(meta.sort_order, meta.sort_order + meta.order);
    else
      t.sort_order.reset();
    t.coalesced = meta.coalesced != 0;
  }
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

uint32_t* upload_fptr(Session& S, const FiberIndex& fib) {
  std::vector<uint32_t> f(fib.fptr.size());
  for (size_t i = 0; i < f.size(); ++i) {
    if (fib.fptr[i] >= (size_t{1} << 32))
      throw std::overflow_error("spten::gpu: fiber offsets exceed the u32 device range");
    f[i] = static_cast<uint32_t>(fib.fptr[i]);
  }
  auto* d = static_cast<uint32_t*>(S.buf(kAux, f.size() * 4));
  S.upload(d, f.data(), f.size() * 4);
  cuda(cudaStreamSynchronize(S.h2d), "sync");  // f is a temporary
  return d;
}

}  // namespace

SparseTensorCOO<float> read_tns(const std::string& path, std::optional<std::vector<Index>> dims) {
  struct Fd {
    int fd;
    ~Fd() {
      if (fd >= 0) ::close(fd);
    }
  } f{::open(path.c_str(), O_RDONLY)};
  if (f.fd < 0) throw std::runtime_error("read_tns: cannot open " + path);  // P/src/io.cpp:45
  if (dims && dims->empty())  // P/src/io.cpp:52
    throw std::invalid_argument("read_tns: dims override must not be empty");
  if (dims && dims->size() > SPT_MAX_ORDER)
    throw std::overflow_error("read_tns: order exceeds " + std::to_string(SPT_MAX_ORDER));
  struct stat sb;
  if (::fstat(f.fd, &sb) != 0) throw std::runtime_error("read_tns: I/O error reading " + path);
  Session& S = session();
  // the file's bytes straight into the pinned ring (parallel preads), DMA of
  // chunk k under the read of chunk k+1
  const size_t bytes = static_cast<size_t>(sb.st_size);
  char* d_text = static_cast<char*>(S.buf(kAux2, bytes + 1));
  for (size_t o = 0; o < bytes; o += kChunk) {
    const size_t c = std::min(kChunk, bytes - o);
    const int k = S.next;
    S.next ^= 1;
    cuda(cudaEventSynchronize(S.ev[k]), "sync");
    if (!CopyPool::get().pread(S.pin[k], f.fd, o, c))
      throw std::runtime_error("read_tns: I/O error reading " + path);
    cuda(cudaMemcpyAsync(d_text + o, S.pin[k], c, cudaMemcpyHostToDevice, S.h2d), "H2D");
    cuda(cudaEventRecord(S.ev[k], S.h2d), "event");
  }
  S.uploads_done();
  // errors: the reference's "path:line: msg" (P/src/io.cpp:37-39)
  uint64_t line = 0;
  auto fail = [&](int status) {
    const std::string msg = spt_last_error();
    if (status == SPT_ERUNTIME && line)
      throw std::runtime_error(path + ":" + std::to_string(line) + ": " + msg);
    if (status == SPT_ERUNTIME && msg.find("order is unknown") != std::string::npos)
      throw std::runtime_error("read_tns: " + path + " " + msg);  // P/src/io.cpp:112-114
    raise(status);
  };
  std::vector<uint32_t> ov;
  if (dims) ov.assign(dims->begin(), dims->end());
  spt_tns* scan = nullptr;
  uint32_t order = 0;
  uint64_t nnz = 0;
  int st = spt_tns_scan(S.ctx, d_text, bytes, dims ? ov.data() : nullptr,
                        static_cast<uint32_t>(ov.size()), &scan, &order, &nnz, &line, S.stream);
  if (st != SPT_OK) fail(st);
  std::unique_ptr<spt_tns, void (*)(spt_tns*)> own(scan, spt_tns_destroy);
  DevCoo dz(S, kZ, order, ov, nnz);
  st = spt_tns_parse(S.ctx, scan, &dz.d, &line, S.stream);
  if (st != SPT_OK) fail(st);
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, nnz);
  return z;
}

SparseTensorCOO<float> ts(const SparseTensorCOO<float>& x, float s, ScalarOp op) {
  Session& S = session();
  DevCoo dx = DevCoo::upload(S, kX, x);
  S.uploads_done();
  DevCoo dz(S, kZ, x.order(), x.dims, x.nnz());
  check(spt_ts_f32(S.ctx, &dx.d, s, static_cast<int>(op), &dz.d, SPT_FLAG_ASYNC, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, x.nnz());
  check(spt_ctx_check(S.ctx, S.stream));
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
  Trace tr;
  Session& S = session();
  tr.mark("session");
  S.t_wait = S.t_copy = 0;
  DevCoo dx = DevCoo::upload(S, kX, x);
  DevCoo dy = DevCoo::upload(S, kY, y);
  S.uploads_done();
  tr.mark("upload");
  if (tr.on) std::fprintf(stderr, "[dropin]   wait %.3f copy %.3f ms\n", S.t_wait, S.t_copy);
  DevCoo dz(S, kZ, x.order(), x.dims, x.nnz());
  // data-dependent errors (pattern mismatch, stored-zero divisor) are raised
  // by spt_ctx_check before the result is handed out
  check(spt_tew_eq_f32(S.ctx, &dx.d, &dy.d, static_cast<int>(op), &dz.d, SPT_FLAG_ASYNC,
                       S.stream));
  tr.mark("launch");
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, x.nnz());
  tr.mark("download");
  check(spt_ctx_check(S.ctx, S.stream));
  tr.mark("check");
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
  DevCoo dx = DevCoo::upload(S, kX, x);
  DevCoo dy = DevCoo::upload(S, kY, y);
  S.uploads_done();
  // unify_tew_sort, P/src/kernel_detail.hpp:88-95: sort both ascending in
  // place unless they already share an order (and hand the sorted operands
  // back, as the reference's non-const references do).
  if (!(x.sort_order && y.sort_order && *x.sort_order == *y.sort_order)) {
    std::vector<uint32_t> asc(x.order());
    for (unsigned m = 0; m < x.order(); ++m) asc[m] = m;
    check(spt_sort_f32(S.ctx, &dx.d, asc.data(), 0, S.stream));
    check(spt_sort_f32(S.ctx, &dy.d, asc.data(), 0, S.stream));
    dx.download(x, dx.d, x.nnz());
    dy.download(y, dy.d, y.nnz());
  }
  const size_t cap = op == ElemOp::mul ? std::min(x.nnz(), y.nnz()) : x.nnz() + y.nnz();
  std::vector<Index> dims(x.order());
  for (unsigned m = 0; m < x.order(); ++m) dims[m] = std::max(x.dims[m], y.dims[m]);
  DevCoo dz(S, kZ, x.order(), dims, cap);
  uint64_t nz = 0;
  check(spt_tew_f32(S.ctx, &dx.d, &dy.d, static_cast<int>(op), &dz.d, cap, &nz, nullptr, 0,
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
  DevCoo dx = DevCoo::upload(S, kX, x);
  uint32_t* df = upload_fptr(S, fib);
  auto* dv = static_cast<float*>(S.buf(kAux2, v.len() * 4));
  S.upload(dv, v.data.data(), v.len() * 4);
  S.uploads_done();
  std::vector<Index> od;
  for (unsigned d = 0; d < x.order(); ++d)
    if (d != mode) od.push_back(x.dims[d]);
  DevCoo dz(S, kZ, x.order() - 1, od, fib.nfibs);
  check(spt_ttv_f32(S.ctx, &dx.d, dv, v.len(), mode, df, fib.nfibs, &dz.d, 0, S.stream));
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
  DevCoo dx = DevCoo::upload(S, kX, x);
  uint32_t* df = upload_fptr(S, fib);
  auto* du = static_cast<float*>(S.buf(kAux2, u.data.size() * 4));
  S.upload(du, u.data.data(), u.data.size() * 4);
  S.uploads_done();
  std::vector<Index> od = x.dims;
  od[mode] = static_cast<Index>(R);
  DevCoo dz(S, kZ, x.order(), od, fib.nfibs * R);
  check(spt_ttm_f32(S.ctx, &dx.d, du, u.rows, R, mode, df, fib.nfibs, &dz.d, 0, S.stream));
  SparseTensorCOO<float> z;
  dz.download(z, dz.d, fib.nfibs * R);
  flops::record(2 * R * x.nnz());
  return z;
}

SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode) {
  return ttm(x, u, mode, build_fiber_index(x, mode));
}

namespace {
// check_mttkrp_inputs, P/src/kernel_detail.hpp:153-174; returns R
size_t check_mttkrp(const SparseTensorCOO<float>& x,
                    const std::vector<DenseMatrix<float>>& factors, unsigned mode) {
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
  return R;
}
}  // namespace

DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode,
                          MttkrpStrategy strategy) {
  const unsigned N = x.order();
  const size_t R = check_mttkrp(x, factors, mode);
  Session& S = session();
  DevCoo dx = DevCoo::upload(S, kX, x);
  std::vector<const float*> fp(N, nullptr);
  std::vector<uint64_t> rows(N, 0), cols(N, 0);
  for (unsigned d = 0; d < N; ++d) {
    if (d == mode) continue;
    auto* f = static_cast<float*>(S.buf(kF + d, factors[d].data.size() * 4));
    S.upload(f, factors[d].data.data(), factors[d].data.size() * 4);
    fp[d] = f;
    rows[d] = factors[d].rows;
    cols[d] = factors[d].cols;
  }
  S.uploads_done();
  DenseMatrix<float> out(x.dims[mode], R);
  auto* dout = static_cast<float*>(S.buf(kOut, out.data.size() * 4));
  // privatize (the reference's deterministic strategy) -> AUTO: the segmented
  // kernel on a mode-leading input, else a device-side plan / sorted copy;
  // atomic -> vector red.global.add
  const int strat = strategy == MttkrpStrategy::atomic ? SPT_MTTKRP_ATOMIC : SPT_MTTKRP_AUTO;
  check(spt_mttkrp_f32(S.ctx, &dx.d, fp.data(), rows.data(), cols.data(), mode, dout, strat, 0,
                       S.stream));
  S.download(out.data.data(), dout, out.data.size() * 4);
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
  DevCoo dt = DevCoo::upload(S, kX, t);
  S.uploads_done();
  std::vector<uint32_t> mo(mode_order.begin(), mode_order.end());
  check(spt_sort_f32(S.ctx, &dt.d, mo.data(), 0, S.stream));
  dt.download(t, dt.d, t.nnz());
}

SparseTensorCOO<float> coalesce(const SparseTensorCOO<float>& t) {
  Session& S = session();
  DevCoo dt = DevCoo::upload(S, kX, t);
  S.uploads_done();
  if (!t.sort_order) {
    std::vector<uint32_t> asc(t.order());
    for (unsigned m = 0; m < t.order(); ++m) asc[m] = m;
    check(spt_sort_f32(S.ctx, &dt.d, asc.data(), 0, S.stream));
  }
  DevCoo dz(S, kZ, t.order(), t.dims, t.nnz());
  uint64_t n = 0;
  check(spt_coalesce_f32(S.ctx, &dt.d, &dz.d, &n, nullptr, 0, S.stream));
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
  DevCoo dt = DevCoo::upload(S, kX, t);
  S.uploads_done();
  auto* fptr = static_cast<uint32_t*>(S.buf(kAux, (t.nnz() + 1) * 4));
  uint64_t nf = 0;
  check(spt_fiber_index(S.ctx, &dt.d, mode, fptr, &nf, nullptr, 0, S.stream));
  std::vector<uint32_t> f(nf + 1);
  S.download(f.data(), fptr, (nf + 1) * 4);
  FiberIndex fib;
  fib.mode = mode;
  fib.nfibs = nf;
  fib.fptr.assign(f.begin(), f.end());
  return fib;
}

// ---- par:: twins (P/include/spten/kernels_par.hpp:35-72) --------------------
namespace par {
SparseTensorCOO<float> tew_eq(const SparseTensorCOO<float>& x, const SparseTensorCOO<float>& y,
                              ElemOp op, int) {
  return gpu::tew_eq(x, y, op);
}
SparseTensorCOO<float> tew(SparseTensorCOO<float>& x, SparseTensorCOO<float>& y, ElemOp op, int) {
  return gpu::tew(x, y, op);
}
SparseTensorCOO<float> ts(const SparseTensorCOO<float>& x, float s, ScalarOp op, int) {
  return gpu::ts(x, s, op);
}
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, const FiberIndex& fib, int) {
  return gpu::ttv(x, v, mode, fib);
}
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, int) {
  return gpu::ttv(x, v, mode);
}
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, const FiberIndex& fib, int) {
  return gpu::ttm(x, u, mode, fib);
}
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, int) {
  return gpu::ttm(x, u, mode);
}
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode, int,
                          MttkrpStrategy strategy) {
  return gpu::mttkrp(x, factors, mode, strategy);
}
}  // namespace par

}  // namespace spten::gpu

// Tuning hook (tune/ only): GB/s of the drop-in's host copy from `src` into
// its pinned upload buffer.
extern "C" double spten_gpu_copy_probe(const void* src, size_t n) {
  using namespace spten::gpu;
  Session& S = session();
  const auto t0 = std::chrono::steady_clock::now();
  for (size_t o = 0; o < n; o += kChunk)
    par_memcpy(S.pin[0], static_cast<const char*>(src) + o, std::min(kChunk, n - o));
  return n / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9;
}
