// spten/gpu.hpp -- drop-in B200 entry points with the reference's signatures.
//
// A caller of the reference library (`spten`, /root/reference/proj = "P/")
// swaps `spten::seq::` / `spten::par::` for `spten::gpu::` and keeps its
// SparseTensorCOO<float> / DenseVector<float> / DenseMatrix<float> /
// FiberIndex values: this header includes the reference's own type headers
// (P/include/spten/tensor.hpp, ops.hpp), it does not redeclare them.
// Every function forwards to the C-ABI in include/spten_b200.h (H2D through
// pinned bounce buffers into device buffers kept per thread across calls,
// the sm_100a kernel chain on a per-thread stream, D2H likewise) and
//   * throws the reference's exception types: std::invalid_argument,
//     std::domain_error, std::overflow_error, std::bad_alloc,
//     std::runtime_error (CUDA failures);
//   * records the *sequential* reference's flop count through
//     spten::flops::record (P/src/kernels_seq.cpp:37,51,65,99,144,172), so
//     the reference's metering and reports keep working;
//   * reproduces the by-value outputs and metadata (dims, sort_order,
//     coalesced) and tew's in-place sort of its operands.
// Only float is provided (all BASELINE configurations are fp32); double
// stays with the reference implementation.
#pragma once

#include <optional>
#include <span>
#include <string>
#include <vector>

#include "spten/ops.hpp"
#include "spten/tensor.hpp"

namespace spten::gpu {

// P/include/spten/kernels_seq.hpp:18-20 (tew_eq): bit-identical to seq::tew_eq.
SparseTensorCOO<float> tew_eq(const SparseTensorCOO<float>& x, const SparseTensorCOO<float>& y,
                              ElemOp op);

// P/include/spten/kernels_seq.hpp:29-30 (tew): bit-identical to seq::tew,
// including the ascending in-place sort of both operands when their sort
// orders differ (P/src/kernel_detail.hpp:88-95).
SparseTensorCOO<float> tew(SparseTensorCOO<float>& x, SparseTensorCOO<float>& y, ElemOp op);

// P/include/spten/kernels_seq.hpp:33-34 (ts): bit-identical to seq::ts.
SparseTensorCOO<float> ts(const SparseTensorCOO<float>& x, float s, ScalarOp op);

// P/include/spten/kernels_seq.hpp:39-43 (ttv): indices bit-identical; values
// within 1e-5 of an fp64 recomputation (fp64 fiber accumulation).
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, const FiberIndex& fib);
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode);

// P/include/spten/kernels_seq.hpp:47-51 (ttm).
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, const FiberIndex& fib);
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode);

// P/include/spten/kernels_seq.hpp:59-61 (mttkrp): any storage order; an input
// sorted with `mode` leading goes to the deterministic segmented kernel,
// any other to a device-side plan (a mode-leading copy, R % 16 == 0) or sorted
// copy: fp64 accumulation, within 1e-5 of fp64 per entry. `strategy` mirrors
// par::mttkrp (P/include/spten/kernels_par.hpp:70-72): privatize -> those
// deterministic paths, atomic -> vector red.global.add (fp32, 1e-4 class).
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode);
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode,
                          MttkrpStrategy strategy);

// P/include/spten/tensor.hpp:151-165 (preprocessing), bit-identical.
void sort_lexicographic(SparseTensorCOO<float>& t, std::span<const unsigned> mode_order);
SparseTensorCOO<float> coalesce(const SparseTensorCOO<float>& t);
FiberIndex build_fiber_index(const SparseTensorCOO<float>& t, unsigned mode);

// P/include/spten/io.hpp:22-23 (read_tns<float>): the file is streamed through
// pinned buffers to the device, split and parsed there (include/spten_b200.h
// spt_tns_scan / spt_tns_parse); same entries (file order), dims, flags and
// error messages ("path:line: msg", std::runtime_error) as the reference.
// Orders above SPT_MAX_ORDER (8) throw std::overflow_error.
SparseTensorCOO<float> read_tns(const std::string& path,
                                std::optional<std::vector<Index>> dims = std::nullopt);

// The par:: twins (P/include/spten/kernels_par.hpp:35-72), so a caller of
// spten::par:: only swaps the namespace. The device is the parallelism:
// nthreads is accepted with any value (as par::resolve_threads accepts any,
// P/src/kernels_par.cpp:15-17) and has no effect.
namespace par {
SparseTensorCOO<float> tew_eq(const SparseTensorCOO<float>& x, const SparseTensorCOO<float>& y,
                              ElemOp op, int nthreads);
SparseTensorCOO<float> tew(SparseTensorCOO<float>& x, SparseTensorCOO<float>& y, ElemOp op,
                           int nthreads);
SparseTensorCOO<float> ts(const SparseTensorCOO<float>& x, float s, ScalarOp op, int nthreads);
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, const FiberIndex& fib, int nthreads);
SparseTensorCOO<float> ttv(const SparseTensorCOO<float>& x, const DenseVector<float>& v,
                           unsigned mode, int nthreads);
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, const FiberIndex& fib, int nthreads);
SparseTensorCOO<float> ttm(const SparseTensorCOO<float>& x, const DenseMatrix<float>& u,
                           unsigned mode, int nthreads);
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode,
                          int nthreads, MttkrpStrategy strategy);
}  // namespace par

}  // namespace spten::gpu
