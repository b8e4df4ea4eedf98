// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the *real* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libspten_ref.so;
// the sources are never copied into this repo). It lets Python tests, the
// golden-vector generator (tests/golden/make_golden.py) and bench.py's
// reference arm / cpu_baseline call spten::seq / spten::par on host arrays.
// Inputs are converted once into opaque SparseTensorCOO<float> handles so
// that timed calls measure the reference kernel (including its by-value
// output allocation), not the conversion.
#include <cstdint>
#include <cstring>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "spten/flop_counter.hpp"
#include "spten/io.hpp"
#include "spten/kernels_par.hpp"
#include "spten/kernels_seq.hpp"
#include "spten/tensor.hpp"

using namespace spten;
using Coo = SparseTensorCOO<float>;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

struct Dense {
  DenseMatrix<float> m;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_flops_reset() { flops::reset(); }
uint64_t ref_flops_count() { return flops::count(); }

// ---- tensor handles --------------------------------------------------------
void* ref_coo_new(uint32_t order, const uint32_t* dims, uint64_t nnz, const uint32_t* const* idx,
                  const float* vals, const int32_t* sort_order, int has_sort, int coalesced) {
  auto* t = new Coo(std::vector<Index>(dims, dims + order));
  for (uint32_t d = 0; d < order; ++d) t->indices[d].assign(idx[d], idx[d] + nnz);
  t->values.assign(vals, vals + nnz);
  if (has_sort) t->sort_order = std::vector<unsigned>(sort_order, sort_order + order);
  t->coalesced = coalesced != 0;
  return t;
}

void ref_coo_free(void* h) { delete static_cast<Coo*>(h); }

uint32_t ref_coo_order(void* h) { return static_cast<Coo*>(h)->order(); }
uint64_t ref_coo_nnz(void* h) { return static_cast<Coo*>(h)->nnz(); }

// Copy out: dims[order], idx[order][nnz], vals[nnz], sort_order[order].
// Returns has_sort_order | coalesced << 1.
int ref_coo_read(void* h, uint32_t* dims, uint32_t** idx, float* vals, int32_t* sort_order) {
  const Coo& t = *static_cast<Coo*>(h);
  for (uint32_t d = 0; d < t.order(); ++d) {
    dims[d] = t.dims[d];
    if (t.nnz()) std::memcpy(idx[d], t.indices[d].data(), t.nnz() * sizeof(Index));
  }
  if (t.nnz()) std::memcpy(vals, t.values.data(), t.nnz() * sizeof(float));
  if (t.sort_order)
    for (uint32_t d = 0; d < t.order(); ++d) sort_order[d] = static_cast<int32_t>((*t.sort_order)[d]);
  return (t.sort_order ? 1 : 0) | (t.coalesced ? 2 : 0);
}

void* ref_gen_synthetic(uint32_t order, const uint32_t* dims, uint64_t nnz, uint64_t seed) {
  void* out = nullptr;
  if (guard([&] {
        out = new Coo(gen_synthetic<float>(std::vector<Index>(dims, dims + order), nnz, seed));
      }))
    return nullptr;
  return out;
}

// ---- kernels: variant 0 = seq, 1 = par(nthreads) ----------------------------
int ref_ts(void* x, float s, int op, int variant, int nthreads, void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    *out = new Coo(variant ? par::ts(a, s, static_cast<ScalarOp>(op), nthreads)
                           : seq::ts(a, s, static_cast<ScalarOp>(op)));
  });
}

int ref_tew_eq(void* x, void* y, int op, int variant, int nthreads, void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    const Coo& b = *static_cast<Coo*>(y);
    *out = new Coo(variant ? par::tew_eq(a, b, static_cast<ElemOp>(op), nthreads)
                           : seq::tew_eq(a, b, static_cast<ElemOp>(op)));
  });
}

// tew sorts its operands in place (P/src/kernel_detail.hpp:88-95); the
// handles x and y observe that, read them back with ref_coo_read.
int ref_tew(void* x, void* y, int op, int variant, int nthreads, void** out) {
  return guard([&] {
    Coo& a = *static_cast<Coo*>(x);
    Coo& b = *static_cast<Coo*>(y);
    *out = new Coo(variant ? par::tew(a, b, static_cast<ElemOp>(op), nthreads)
                           : seq::tew(a, b, static_cast<ElemOp>(op)));
  });
}

int ref_sort(void* x, const uint32_t* mode_order) {
  return guard([&] {
    Coo& a = *static_cast<Coo*>(x);
    std::vector<unsigned> mo(mode_order, mode_order + a.order());
    sort_lexicographic(a, std::span<const unsigned>(mo));
  });
}

int ref_coalesce(void* x, void** out) {
  return guard([&] { *out = new Coo(coalesce(*static_cast<Coo*>(x))); });
}

// fptr receives nfibs+1 offsets (capacity nnz+1).
int ref_fiber_index(void* x, uint32_t mode, uint64_t* fptr, uint64_t* nfibs) {
  return guard([&] {
    FiberIndex f = build_fiber_index(*static_cast<Coo*>(x), mode);
    for (std::size_t i = 0; i < f.fptr.size(); ++i) fptr[i] = f.fptr[i];
    *nfibs = f.nfibs;
  });
}

int ref_ttv(void* x, const float* v, uint64_t vlen, uint32_t mode, int variant, int nthreads,
            void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    DenseVector<float> dv(vlen);
    std::memcpy(dv.data.data(), v, vlen * sizeof(float));
    *out = new Coo(variant ? par::ttv(a, dv, mode, nthreads) : seq::ttv(a, dv, mode));
  });
}

// With a prebuilt fiber index (timed path: the fiber index is preprocessing).
void* ref_fiber_new(void* x, uint32_t mode) {
  FiberIndex* f = nullptr;
  if (guard([&] { f = new FiberIndex(build_fiber_index(*static_cast<Coo*>(x), mode)); }))
    return nullptr;
  return f;
}
void ref_fiber_free(void* f) { delete static_cast<FiberIndex*>(f); }

void* ref_vector_new(const float* v, uint64_t n) {
  auto* dv = new DenseVector<float>(n);
  std::memcpy(dv->data.data(), v, n * sizeof(float));
  return dv;
}
void ref_vector_free(void* v) { delete static_cast<DenseVector<float>*>(v); }

void* ref_matrix_new(const float* m, uint64_t rows, uint64_t cols) {
  auto* dm = new DenseMatrix<float>(rows, cols);
  if (rows * cols) std::memcpy(dm->data.data(), m, rows * cols * sizeof(float));
  return dm;
}
void ref_matrix_free(void* m) { delete static_cast<DenseMatrix<float>*>(m); }
void ref_matrix_read(void* m, float* out) {
  auto* dm = static_cast<DenseMatrix<float>*>(m);
  if (!dm->data.empty()) std::memcpy(out, dm->data.data(), dm->data.size() * sizeof(float));
}

int ref_ttv_fib(void* x, void* v, uint32_t mode, void* fib, int variant, int nthreads,
                void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    const auto& dv = *static_cast<DenseVector<float>*>(v);
    const auto& f = *static_cast<FiberIndex*>(fib);
    *out = new Coo(variant ? par::ttv(a, dv, mode, f, nthreads) : seq::ttv(a, dv, mode, f));
  });
}

int ref_ttm_fib(void* x, void* u, uint32_t mode, void* fib, int variant, int nthreads,
                void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    const auto& du = *static_cast<DenseMatrix<float>*>(u);
    if (fib) {
      const auto& f = *static_cast<FiberIndex*>(fib);
      *out = new Coo(variant ? par::ttm(a, du, mode, f, nthreads) : seq::ttm(a, du, mode, f));
    } else {
      *out = new Coo(variant ? par::ttm(a, du, mode, nthreads) : seq::ttm(a, du, mode));
    }
  });
}

// factors: N matrix handles (factors[mode] may be NULL -> empty matrix).
// strategy: 0 privatize, 1 atomic (par only). Result: matrix handle.
int ref_mttkrp(void* x, void* const* factors, uint32_t mode, int variant, int nthreads,
               int strategy, void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    std::vector<DenseMatrix<float>> f(a.order());
    for (uint32_t d = 0; d < a.order(); ++d)
      if (factors[d]) f[d] = *static_cast<DenseMatrix<float>*>(factors[d]);
    *out = new DenseMatrix<float>(
        variant ? par::mttkrp(a, f, mode, nthreads, static_cast<MttkrpStrategy>(strategy))
                : seq::mttkrp(a, f, mode));
  });
}

// Timed variant that keeps the factor vector alive across calls.
void* ref_factors_new(void* x, void* const* factors) {
  const Coo& a = *static_cast<Coo*>(x);
  auto* f = new std::vector<DenseMatrix<float>>(a.order());
  for (uint32_t d = 0; d < a.order(); ++d)
    if (factors[d]) (*f)[d] = *static_cast<DenseMatrix<float>*>(factors[d]);
  return f;
}
void ref_factors_free(void* f) { delete static_cast<std::vector<DenseMatrix<float>>*>(f); }

int ref_mttkrp_fv(void* x, void* fv, uint32_t mode, int variant, int nthreads, int strategy,
                  void** out) {
  return guard([&] {
    const Coo& a = *static_cast<Coo*>(x);
    const auto& f = *static_cast<std::vector<DenseMatrix<float>>*>(fv);
    *out = new DenseMatrix<float>(
        variant ? par::mttkrp(a, f, mode, nthreads, static_cast<MttkrpStrategy>(strategy))
                : seq::mttkrp(a, f, mode));
  });
}

// ---- io (P/src/io.cpp) --------------------------------------------------------
// read_tns<float>(path, dims override when n_dims > 0) into a handle.
int ref_read_tns(const char* path, const uint32_t* dims, uint32_t n_dims, void** out) {
  return guard([&] {
    std::optional<std::vector<Index>> ov;
    if (dims) ov = std::vector<Index>(dims, dims + n_dims);
    *out = new Coo(read_tns<float>(path, ov));
  });
}

int ref_write_tns(void* x, const char* path) {
  return guard([&] { write_tns(*static_cast<Coo*>(x), path); });
}

int ref_max_threads() { return par::resolve_threads(0); }

}  // extern "C"
