// spten/gpu.hpp -- drop-in B200 entry points with the reference's signatures.
//
// A caller of the reference library (`spten`, /root/reference/proj = "P/")
// swaps `spten::seq::` / `spten::par::` for `spten::gpu::` and keeps its
// SparseTensorCOO<float> / DenseVector<float> / DenseMatrix<float> /
// FiberIndex values: this header includes the reference's own type headers
// (P/include/spten/tensor.hpp, ops.hpp), it does not redeclare them.
// Every function forwards to the C-ABI in include/spten_b200.h (H2D, one
// sm_100a kernel chain on a per-thread stream, D2H) and
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

#include <span>
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
// not sorted with `mode` leading is sorted on the device (a copy) and then
// reduced by the deterministic segmented kernel. `strategy` mirrors
// par::mttkrp (P/include/spten/kernels_par.hpp:70-72): privatize -> the
// segmented (one writer per row) kernel, atomic -> vector red.global.add.
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode);
DenseMatrix<float> mttkrp(const SparseTensorCOO<float>& x,
                          const std::vector<DenseMatrix<float>>& factors, unsigned mode,
                          MttkrpStrategy strategy);

// P/include/spten/tensor.hpp:151-165 (preprocessing), bit-identical.
void sort_lexicographic(SparseTensorCOO<float>& t, std::span<const unsigned> mode_order);
SparseTensorCOO<float> coalesce(const SparseTensorCOO<float>& t);
FiberIndex build_fiber_index(const SparseTensorCOO<float>& t, unsigned mode);

}  // namespace spten::gpu
