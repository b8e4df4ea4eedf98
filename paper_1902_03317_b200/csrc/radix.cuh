// Stable LSD radix sort of (packed tuple key, u32 payload) pairs -- the engine
// under sort_lexicographic (P/src/tensor.cpp:54-64). Hand-written for sm_100a
// (radix.cu): one histogram pass for every digit, then one single-sweep
// ("onesweep", decoupled look-back per digit) pass per digit. Key-width aware:
// only the significant bits of the packed tuple are sorted, split into equal
// digits of at most 8 bits; the first pass packs the key from the tensor's index
// arrays on the fly and the last pass unpacks it straight into them (or keeps
// only the permutation), so no separate pack / unpack / gather pass runs.
#pragma once

#include "internal.cuh"

namespace spt {
namespace radix {

// key = OR_j idx[j][entry] << shift[j]
struct PackSpec {
  const uint32_t* idx[SPT_MAX_ORDER];
  uint32_t shift[SPT_MAX_ORDER];
  int n;
};
// idx[j][pos] = (key >> shift[j]) & mask[j]
struct UnpackSpec {
  uint32_t* idx[SPT_MAX_ORDER];
  uint32_t shift[SPT_MAX_ORDER];
  uint32_t mask[SPT_MAX_ORDER];
  int n;
};

// The whole tuple fits one key of `nbits` (<= 64) bits: sorts the tensor's
// index arrays and its value words in place (pack -> passes -> unpack).
int sort_tuple_inplace(spt_ctx* ctx, const PackSpec& pack, const UnpackSpec& unpack,
                       uint32_t* vals, uint64_t n, uint32_t nbits, cudaStream_t st);

// One <=64-bit chunk of a wider tuple: stable sort of the entries listed by
// perm_in (nullptr: identity) on the chunk key; perm_out receives the new
// permutation (may alias perm_in).
int sort_chunk_perm(spt_ctx* ctx, const PackSpec& pack, const uint32_t* perm_in,
                    uint32_t* perm_out, uint64_t n, uint32_t nbits, cudaStream_t st);

}  // namespace radix
}  // namespace spt
