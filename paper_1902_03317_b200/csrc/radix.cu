// Hand-written stable LSD radix sort for sm_100a (see radix.cuh).
//
// Reference semantics: std::stable_sort of a permutation under compare_entries
// (P/src/tensor.cpp:54-64); a stable sort on the packed tuple key is exactly
// that order, duplicates included.
//
// Kernels:
//   hist_kernel      one read of the keys, shared-memory histograms of every
//                    digit at once, one global atomic per non-empty bin and CTA;
//   scan_kernel      exclusive scan of each digit's 256 bins (the bin bases);
//   onesweep_kernel  one pass: a CTA takes tile tickets in order, loads
//                    THREADS x ITEMS pairs warp-striped (coalesced), ranks them
//                    stably per warp with match.any on the digit (one private
//                    counter row per warp, no atomics), scans the rows over the
//                    warps and bins, publishes the tile's bin counts and finds
//                    its bins' global offsets by a decoupled look-back over
//                    epoch-tagged 64-bit words (count and flag in one word, so
//                    no fence), reorders the tile in shared memory and writes
//                    each bin's run with coalesced streaming stores.
// Fusions: the first pass reads the tensor's index arrays and packs the key in
// registers (no key array is materialised for it), the last pass either
// unpacks the key into the index arrays or writes only the permutation.
#include <algorithm>

#include "radix.cuh"

namespace spt {
namespace radix {
namespace {

constexpr int kBins = 256;
constexpr int kMaxPasses = 8;
constexpr int kThreads = 384;

enum Src { SRC_ARRAYS = 0, SRC_PACK_VAL = 1, SRC_PACK_IOTA = 2 };
enum Dst { DST_ARRAYS = 0, DST_UNPACK = 1, DST_PAY = 2 };

struct SrcDesc {
  const void* keys;     // SRC_ARRAYS: packed keys
  const uint32_t* pay;  // SRC_ARRAYS: payload; SRC_PACK_VAL: the value words
  PackSpec pack;        // SRC_PACK_*
};
struct DstDesc {
  void* keys;     // DST_ARRAYS
  uint32_t* pay;  // DST_ARRAYS / DST_PAY payload; DST_UNPACK: the value words
  UnpackSpec un;  // DST_UNPACK
};
struct Digits {
  int passes;
  uint32_t shift[kMaxPasses];
  uint32_t bits[kMaxPasses];
};

template <typename K>
__device__ __forceinline__ K pack_key(const PackSpec& p, uint64_t e) {
  K k = 0;
  // static indices: the spec stays in the constant bank (no local copy)
#pragma unroll
  for (int j = 0; j < SPT_MAX_ORDER; ++j)
    if (j < p.n) k |= static_cast<K>(__ldcs(p.idx[j] + e)) << p.shift[j];
  return k;
}

template <typename K, int SRC>
__device__ __forceinline__ K load_key(const SrcDesc& s, uint64_t i) {
  if (SRC == SRC_ARRAYS) return __ldcs(static_cast<const K*>(s.keys) + i);
  return pack_key<K>(s.pack, i);
}
template <int SRC>
__device__ __forceinline__ uint32_t load_pay(const SrcDesc& s, uint64_t i) {
  if (SRC == SRC_PACK_IOTA) return static_cast<uint32_t>(i);
  return __ldcs(s.pay + i);
}

// Histograms of every digit in one read of the keys.
template <typename K, int SRC>
__global__ void __launch_bounds__(256) hist_kernel(SrcDesc s, uint64_t n, Digits dg,
                                                   uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kMaxPasses * kBins];
  for (int j = threadIdx.x; j < dg.passes * kBins; j += blockDim.x) h[j] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x; b < n; b += stride) {
    const uint64_t i = b + threadIdx.x;
    const bool ok = i < n;
    const K key = ok ? load_key<K, SRC>(s, i) : K(0);
    const bool full = __all_sync(0xffffffffu, ok);
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p) {
      if (p >= dg.passes) continue;
      const uint32_t d = static_cast<uint32_t>(key >> dg.shift[p]) & ((1u << dg.bits[p]) - 1u);
      // a warp whose 32 keys share the digit (sorted or constant high bits)
      // adds once instead of serialising 32 same-address atomics
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
      if (full && __all_sync(0xffffffffu, d == d0)) {
        if (lane == 0) atomicAdd(&h[p * kBins + d0], 32u);
      } else if (ok) {
        atomicAdd(&h[p * kBins + d], 1u);
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < dg.passes * kBins; j += blockDim.x)
    if (h[j]) atomicAdd(&ghist[j], h[j]);
}

// base[p][b] = number of keys whose digit p is < b.
__global__ void __launch_bounds__(kBins) scan_kernel(const uint32_t* __restrict__ ghist,
                                                     uint32_t* __restrict__ base) {
  __shared__ uint32_t wsum[kBins / 32];
  const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t v = ghist[p * kBins + t];
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  uint32_t pre = 0;
  for (int k = 0; k < w; ++k) pre += wsum[k];
  base[p * kBins + t] = pre + inc - v;
}

__device__ __forceinline__ unsigned long long tag(uint32_t epoch, uint32_t flag, uint32_t count) {
  return (static_cast<unsigned long long>(epoch) << 34) |
         (static_cast<unsigned long long>(flag) << 32) | count;
}

template <typename K, int ITEMS>
constexpr size_t onesweep_smem() {
  return static_cast<size_t>(kThreads) * ITEMS * (sizeof(K) + 4) +
         (kThreads / 32) * kBins * 4 + 2 * kBins * 4;
}

template <typename K, int SRC, int DST, int ITEMS>
__global__ void __launch_bounds__(kThreads, 2)
    onesweep_kernel(SrcDesc s, DstDesc d, uint64_t n, uint32_t shift, uint32_t bits,
                    const uint32_t* __restrict__ base, unsigned long long* status, uint32_t epoch,
                    uint32_t* ticket) {
  constexpr int WARPS = kThreads / 32;
  constexpr int TILE = kThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char smem[];
  K* keys_s = reinterpret_cast<K*>(smem);
  uint32_t* pay_s = reinterpret_cast<uint32_t*>(keys_s + TILE);
  uint32_t* cnt = pay_s + TILE;             // [WARPS][kBins]
  uint32_t* bin_start = cnt + WARPS * kBins;  // tile-local start of each bin
  uint32_t* gbase = bin_start + kBins;        // global position of the bin's shared slot 0
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_tot[kBins / 32];

  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  for (int j = tid; j < WARPS * kBins; j += kThreads) cnt[j] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * TILE;
  const uint32_t valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), n - tile_base));
  const uint32_t mask = (1u << bits) - 1u;

  // Warp-striped load: item k of lane l is entry warp*32*ITEMS + k*32 + l of
  // the tile. Entries past the end get the all-ones key: they land at the end
  // of the last bin, i.e. at shared slots >= valid, and are never written.
  K key[ITEMS];
  uint32_t pay[ITEMS];
  const uint32_t wloc = warp * 32u * ITEMS + lane;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t loc = wloc + k * 32u;
    if (loc < valid) {
      key[k] = load_key<K, SRC>(s, tile_base + loc);
      pay[k] = load_pay<SRC>(s, tile_base + loc);
    } else {
      key[k] = ~K(0);
      pay[k] = 0;
    }
  }

  // Stable rank inside the warp: lanes holding the same digit form a group;
  // the group's first lane bumps the warp's private counter.
  uint32_t rank[ITEMS];
  uint32_t* wc = cnt + warp * kBins;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t dgt = static_cast<uint32_t>(key[k] >> shift) & mask;
    const uint32_t m = __match_any_sync(0xffffffffu, dgt);
    const int leader = __ffs(m) - 1;
    uint32_t old = 0;
    if (static_cast<int>(lane) == leader) {
      old = wc[dgt];
      wc[dgt] = old + __popc(m);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[k] = old + __popc(m & lt);
    __syncwarp();
  }
  __syncthreads();

  // Bin b = thread b: exclusive scan of its counts over the warps, then over
  // the bins; publish the tile's count of the bin.
  uint32_t total = 0;
  if (tid < kBins) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = cnt[w * kBins + tid];
      cnt[w * kBins + tid] = total;
      total += c;
    }
  }
  uint32_t inc = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (tid < kBins && lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  uint32_t vcount = 0;
  if (tid < kBins) {
    uint32_t pre = 0;
    for (unsigned w = 0; w < warp; ++w) pre += warp_tot[w];
    bin_start[tid] = pre + inc - total;
    vcount = total - (tid == mask ? static_cast<uint32_t>(TILE) - valid : 0u);
    if (tid <= mask)
      st_relaxed64(status + static_cast<size_t>(tile) * kBins + tid,
                   tag(epoch, tile == 0 ? 2u : 1u, vcount));
  }
  __syncthreads();

  // Reorder the tile by digit in shared memory.
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t dgt = static_cast<uint32_t>(key[k] >> shift) & mask;
    const uint32_t pos = bin_start[dgt] + wc[dgt] + rank[k];
    keys_s[pos] = key[k];
    pay_s[pos] = pay[k];
  }

  // Decoupled look-back per bin: counts of the bin in all earlier tiles.
  if (tid <= mask) {
    uint32_t before = 0;
    if (tile > 0) {
      int64_t t = static_cast<int64_t>(tile) - 1;
      while (true) {
        const unsigned long long w = ld_relaxed64(status + static_cast<size_t>(t) * kBins + tid);
        if ((w >> 34) != epoch) {
          __nanosleep(20);
          continue;
        }
        before += static_cast<uint32_t>(w);
        if (((w >> 32) & 3u) == 2u) break;
        --t;
      }
      st_relaxed64(status + static_cast<size_t>(tile) * kBins + tid,
                   tag(epoch, 2u, before + vcount));
    }
    gbase[tid] = base[tid] + before - bin_start[tid];
  }
  __syncthreads();

  // Each bin's run goes out contiguous: consecutive slots -> consecutive
  // global positions.
  for (uint32_t j = tid; j < valid; j += kThreads) {
    const K kk = keys_s[j];
    const uint32_t dgt = static_cast<uint32_t>(kk >> shift) & mask;
    const uint32_t pos = gbase[dgt] + j;
    if (DST == DST_ARRAYS) {
      __stcs(static_cast<K*>(d.keys) + pos, kk);
      __stcs(d.pay + pos, pay_s[j]);
    } else if (DST == DST_UNPACK) {
#pragma unroll
      for (int q = 0; q < SPT_MAX_ORDER; ++q)
        if (q < d.un.n)
          __stcs(d.un.idx[q] + pos, static_cast<uint32_t>(kk >> d.un.shift[q]) & d.un.mask[q]);
      __stcs(d.pay + pos, pay_s[j]);
    } else {
      __stcs(d.pay + pos, pay_s[j]);
    }
  }
}

// key[i] = packed chunk of entry perm[i] (the one gather a later chunk needs).
template <typename K>
__global__ void pack_perm_kernel(PackSpec spec, const uint32_t* __restrict__ perm,
                                 K* __restrict__ keys, uint64_t n) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (; i < n; i += stride) {
    const uint64_t e = perm[i];
    K k = 0;
#pragma unroll
    for (int j = 0; j < SPT_MAX_ORDER; ++j)
      if (j < spec.n) k |= static_cast<K>(spec.idx[j][e]) << spec.shift[j];
    keys[i] = k;
  }
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

Digits plan_digits(uint32_t nbits) {
  // equal digits of <= 8 bits; at least two passes, so that the first pass
  // (which reads the caller's arrays) never writes into them
  Digits dg{};
  if (nbits == 0) nbits = 1;
  int passes = static_cast<int>((nbits + 7) / 8);
  if (passes < 2) passes = 2;
  dg.passes = passes;
  uint32_t at = 0;
  for (int p = 0; p < passes; ++p) {
    const uint32_t w = nbits / passes + (static_cast<uint32_t>(p) < nbits % passes ? 1u : 0u);
    dg.shift[p] = at;
    dg.bits[p] = w;
    at += w;
  }
  return dg;
}

template <typename K>
constexpr int items_for() {
  return sizeof(K) == 8 ? 12 : 16;
}

template <typename K, int SRC, int DST>
int launch_pass(spt_ctx* ctx, const SrcDesc& s, const DstDesc& d, uint64_t n, uint32_t shift,
                uint32_t bits, const uint32_t* base, uint32_t* ticket, cudaStream_t st) {
  constexpr int ITEMS = items_for<K>();
  constexpr size_t smem = onesweep_smem<K, ITEMS>();
  auto kern = onesweep_kernel<K, SRC, DST, ITEMS>;
  SPT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));  // per device, cheap
  const uint64_t tile = static_cast<uint64_t>(kThreads) * ITEMS;
  const uint64_t tiles = (n + tile - 1) / tile;
  unsigned long long* status;
  SPT_TRY(ctx_status64(ctx, tiles * kBins, &status));
  uint32_t epoch;
  SPT_TRY(ctx_lookback(ctx, 0, 0, &epoch));
  kern<<<static_cast<unsigned>(tiles), kThreads, smem, st>>>(s, d, n, shift, bits, base, status,
                                                              epoch, ticket);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

struct Buffers {
  void* key[2];
  uint32_t* pay[2];
  uint32_t* hist;
  uint32_t* base;
  uint32_t* ticket;
};

template <typename K>
int carve(spt_ctx* ctx, uint64_t n, Buffers* b, cudaStream_t st) {
  const size_t kb = align_up(n * sizeof(K)), pb = align_up(n * 4);
  const size_t hb = align_up(kMaxPasses * kBins * 4);
  void* scratch;
  SPT_TRY(ctx_scratch(ctx, 2 * kb + 2 * pb + 2 * hb + 256, &scratch));
  char* p = static_cast<char*>(scratch);
  b->key[0] = p;
  b->key[1] = p + kb;
  b->pay[0] = reinterpret_cast<uint32_t*>(p + 2 * kb);
  b->pay[1] = reinterpret_cast<uint32_t*>(p + 2 * kb + pb);
  b->hist = reinterpret_cast<uint32_t*>(p + 2 * kb + 2 * pb);
  b->base = reinterpret_cast<uint32_t*>(p + 2 * kb + 2 * pb + hb);
  b->ticket = reinterpret_cast<uint32_t*>(p + 2 * kb + 2 * pb + 2 * hb);
  // hist and ticket are adjacent to base: one memset clears hist; tickets apart
  SPT_CUDA(cudaMemsetAsync(b->hist, 0, hb, st));
  SPT_CUDA(cudaMemsetAsync(b->ticket, 0, 256, st));
  return SPT_OK;
}

template <typename K, int SRC>
int histogram(spt_ctx* ctx, const SrcDesc& s, uint64_t n, const Digits& dg, const Buffers& b,
              cudaStream_t st) {
  const unsigned g = grid_for(n, 256, ctx->num_sms * 8);
  hist_kernel<K, SRC><<<g, 256, 0, st>>>(s, n, dg, b.hist);
  SPT_LAUNCHED(ctx);
  scan_kernel<<<dg.passes, kBins, 0, st>>>(b.hist, b.base);
  SPT_LAUNCHED(ctx);
  return SPT_OK;
}

template <typename K>
int tuple_inplace(spt_ctx* ctx, const PackSpec& pack, const UnpackSpec& unpack, uint32_t* vals,
                  uint64_t n, uint32_t nbits, cudaStream_t st) {
  const Digits dg = plan_digits(nbits);
  Buffers b;
  SPT_TRY(carve<K>(ctx, n, &b, st));
  SrcDesc s0{};
  s0.pack = pack;
  s0.pay = vals;
  SPT_TRY((histogram<K, SRC_PACK_VAL>(ctx, s0, n, dg, b, st)));
  int cur = 0;  // buffer the next pass writes
  for (int p = 0; p < dg.passes; ++p) {
    const bool first = p == 0, last = p == dg.passes - 1;
    SrcDesc s{};
    DstDesc d{};
    if (first) {
      s = s0;
    } else {
      s.keys = b.key[cur ^ 1];
      s.pay = b.pay[cur ^ 1];
    }
    if (last) {
      d.un = unpack;
      d.pay = vals;
    } else {
      d.keys = b.key[cur];
      d.pay = b.pay[cur];
    }
    const uint32_t* base = b.base + p * kBins;
    if (first)
      SPT_TRY((launch_pass<K, SRC_PACK_VAL, DST_ARRAYS>(ctx, s, d, n, dg.shift[p], dg.bits[p], base,
                                                        b.ticket + p, st)));
    else if (last)
      SPT_TRY((launch_pass<K, SRC_ARRAYS, DST_UNPACK>(ctx, s, d, n, dg.shift[p], dg.bits[p], base,
                                                      b.ticket + p, st)));
    else
      SPT_TRY((launch_pass<K, SRC_ARRAYS, DST_ARRAYS>(ctx, s, d, n, dg.shift[p], dg.bits[p], base,
                                                      b.ticket + p, st)));
    cur ^= 1;
  }
  return SPT_OK;
}

template <typename K>
int chunk_perm(spt_ctx* ctx, const PackSpec& pack, const uint32_t* perm_in, uint32_t* perm_out,
               uint64_t n, uint32_t nbits, cudaStream_t st) {
  const Digits dg = plan_digits(nbits);
  Buffers b;
  SPT_TRY(carve<K>(ctx, n, &b, st));
  SrcDesc s0{};
  int cur = 0;
  if (perm_in) {
    // later chunk: the keys of the entries in their current order (one
    // gather), then plain passes carrying the permutation
    pack_perm_kernel<K><<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, st>>>(
        pack, perm_in, static_cast<K*>(b.key[1]), n);
    SPT_LAUNCHED(ctx);
    s0.keys = b.key[1];
    s0.pay = perm_in;
    SPT_TRY((histogram<K, SRC_ARRAYS>(ctx, s0, n, dg, b, st)));
  } else {
    s0.pack = pack;
    SPT_TRY((histogram<K, SRC_PACK_IOTA>(ctx, s0, n, dg, b, st)));
  }
  for (int p = 0; p < dg.passes; ++p) {
    const bool first = p == 0, last = p == dg.passes - 1;
    SrcDesc s{};
    DstDesc d{};
    if (first) {
      s = s0;
    } else {
      s.keys = b.key[cur ^ 1];
      s.pay = b.pay[cur ^ 1];
    }
    if (last) {
      d.pay = perm_out;
    } else {
      d.keys = b.key[cur];
      d.pay = b.pay[cur];
    }
    const uint32_t* base = b.base + p * kBins;
    if (first && !perm_in)
      SPT_TRY((launch_pass<K, SRC_PACK_IOTA, DST_ARRAYS>(ctx, s, d, n, dg.shift[p], dg.bits[p],
                                                         base, b.ticket + p, st)));
    else if (last)
      SPT_TRY((launch_pass<K, SRC_ARRAYS, DST_PAY>(ctx, s, d, n, dg.shift[p], dg.bits[p], base,
                                                   b.ticket + p, st)));
    else
      SPT_TRY((launch_pass<K, SRC_ARRAYS, DST_ARRAYS>(ctx, s, d, n, dg.shift[p], dg.bits[p], base,
                                                      b.ticket + p, st)));
    cur ^= 1;
  }
  return SPT_OK;
}

}  // namespace

int sort_tuple_inplace(spt_ctx* ctx, const PackSpec& pack, const UnpackSpec& unpack,
                       uint32_t* vals, uint64_t n, uint32_t nbits, cudaStream_t st) {
  if (n < 2) return SPT_OK;
  if (nbits <= 32) return tuple_inplace<uint32_t>(ctx, pack, unpack, vals, n, nbits, st);
  return tuple_inplace<unsigned long long>(ctx, pack, unpack, vals, n, nbits, st);
}

int sort_chunk_perm(spt_ctx* ctx, const PackSpec& pack, const uint32_t* perm_in,
                    uint32_t* perm_out, uint64_t n, uint32_t nbits, cudaStream_t st) {
  if (nbits <= 32) return chunk_perm<uint32_t>(ctx, pack, perm_in, perm_out, n, nbits, st);
  return chunk_perm<unsigned long long>(ctx, pack, perm_in, perm_out, n, nbits, st);
}

}  // namespace radix
}  // namespace spt
