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
//                    stably per warp (peer masks from shared-memory atomicOr,
//                    one private counter row per warp), scans the rows over the
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
// Tile shape (tuning knobs): threads per CTA, resident CTAs per SM the
// register budget is set for, pairs per thread for 8- and 4-byte keys.
#ifndef SPT_RADIX_THREADS
#define SPT_RADIX_THREADS 384
#endif
#ifndef SPT_RADIX_MINB
#define SPT_RADIX_MINB 2
#endif
#ifndef SPT_RADIX_ITEMS64
#define SPT_RADIX_ITEMS64 12
#endif
#ifndef SPT_RADIX_ITEMS32
#define SPT_RADIX_ITEMS32 16
#endif
constexpr int kThreads = SPT_RADIX_THREADS;
static_assert(kThreads >= kBins && kThreads % 32 == 0, "one thread per bin");

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
#ifndef SPT_RADIX_HIST_U
#define SPT_RADIX_HIST_U 4
#endif
  constexpr int U = SPT_RADIX_HIST_U;  // keys per thread and step: U loads per array in flight
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * U;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x * U; b < n; b += stride) {
    K key[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = b + u * blockDim.x + threadIdx.x < n;
      key[u] = 0;
    }
    if (SRC == SRC_ARRAYS) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) key[u] = __ldcs(static_cast<const K*>(s.keys) + b + u * blockDim.x + threadIdx.x);
    } else {
#pragma unroll
      for (int j = 0; j < SPT_MAX_ORDER; ++j) {
        if (j < s.pack.n) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u])
              key[u] |= static_cast<K>(__ldcs(s.pack.idx[j] + b + u * blockDim.x + threadIdx.x))
                        << s.pack.shift[j];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool full = __all_sync(0xffffffffu, ok[u]);
#pragma unroll
      for (int p = 0; p < kMaxPasses; ++p) {
        if (p >= dg.passes) continue;
        const uint32_t d =
            static_cast<uint32_t>(key[u] >> dg.shift[p]) & ((1u << dg.bits[p]) - 1u);
        // a warp whose 32 keys share the digit (sorted or constant high bits)
        // adds once instead of serialising 32 same-address atomics
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
        if (dg.bits[p] <= 2) {
          // <= 4 bins: one ballot per bin, lane b adds bin b's count
          uint32_t mine = 0;
#pragma unroll
          for (uint32_t b4 = 0; b4 < 4; ++b4) {
            const uint32_t c = __popc(__ballot_sync(0xffffffffu, ok[u] && d == b4));
            if (lane == b4) mine = c;
          }
          if (lane < 4 && mine) atomicAdd(&h[p * kBins + lane], mine);
        } else if (full && __all_sync(0xffffffffu, d == d0)) {
          if (lane == 0) atomicAdd(&h[p * kBins + d0], 32u);
        } else if (ok[u]) {
          atomicAdd(&h[p * kBins + d], 1u);
        }
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
         (kThreads / 32) * kBins * 8 + 2 * kBins * 4;
}

// CB: the digit width when it is the full 8 bits (ballots fully unrolled),
// 0 = any width, read from `bits`.
template <typename K, int SRC, int DST, int ITEMS, int CB>
__global__ void __launch_bounds__(kThreads, SPT_RADIX_MINB)
    onesweep_kernel(SrcDesc s, DstDesc d, uint64_t n, uint32_t shift, uint32_t bits_rt,
                    const uint32_t* __restrict__ base, unsigned long long* status, uint32_t epoch,
                    uint32_t* ticket) {
  constexpr int WARPS = kThreads / 32;
  constexpr int TILE = kThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char smem[];
  K* keys_s = reinterpret_cast<K*>(smem);
  uint32_t* pay_s = reinterpret_cast<uint32_t*>(keys_s + TILE);
  uint2* pairs = reinterpret_cast<uint2*>(pay_s + TILE);  // [WARPS][kBins] {mask, count}
  uint32_t* bin_start = reinterpret_cast<uint32_t*>(pairs + WARPS * kBins);  // tile-local
  uint32_t* gbase = bin_start + kBins;        // global position of the bin's shared slot 0
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_tot[kBins / 32];

  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t bits = CB ? CB : bits_rt;
  // Passes are chained by programmatic dependent launch: once every CTA of
  // this pass has started, the next pass's CTAs may take the SMs this pass's
  // last wave leaves idle; they take their ticket and clear their counters,
  // then block in griddepcontrol.wait until this grid has completed and its
  // writes are visible.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  for (int j = tid; j < WARPS * kBins / 2; j += kThreads)
    reinterpret_cast<uint4*>(pairs)[j] = make_uint4(0, 0, 0, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
  if (SRC == SRC_ARRAYS) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t loc = wloc + k * 32u;
      key[k] = loc < valid ? __ldcs(static_cast<const K*>(s.keys) + tile_base + loc) : ~K(0);
    }
  } else {
    // one index array at a time: ITEMS independent loads in flight per array
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) key[k] = wloc + k * 32u < valid ? K(0) : ~K(0);
#pragma unroll
    for (int j = 0; j < SPT_MAX_ORDER; ++j) {
      if (j < s.pack.n) {
        const uint32_t* a = s.pack.idx[j] + tile_base;
        const uint32_t sh = s.pack.shift[j];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t loc = wloc + k * 32u;
          if (loc < valid) key[k] |= static_cast<K>(__ldcs(a + loc)) << sh;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t loc = wloc + k * 32u;
    pay[k] = loc < valid ? load_pay<SRC>(s, tile_base + loc) : 0u;
  }

  // Stable rank inside the warp. Each (warp, digit) owns a pair of words
  // {mask of the lanes holding the digit in this item, count in the earlier
  // items}: every lane ORs its bit into the mask and reads the pair back with
  // one 64-bit load -- its rank is count + lower peers -- and the group's first
  // lane stores {0, count + group size}. (8 ballots per item cost 3x the
  // instructions; match.any ~1000 cycles per warp-instruction under load.)
  uint32_t rank[ITEMS];
  uint2* wp = pairs + warp * kBins;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t dgt = static_cast<uint32_t>(key[k] >> shift) & mask;
    atomicOr(&wp[dgt].x, 1u << lane);
    __syncwarp();
    const uint2 mc = wp[dgt];
    __syncwarp();
    rank[k] = mc.y + __popc(mc.x & lt);
    if ((mc.x & lt) == 0) wp[dgt] = make_uint2(0u, mc.y + __popc(mc.x));
    __syncwarp();
  }
  __syncthreads();

  // Bin b = thread b: its count in the tile goes out at once (the successors'
  // look-back waits for it), then the exclusive scan over the bins and, per
  // bin, over the warps: pairs[w][b].y becomes the tile-local slot of warp w's
  // first item of bin b.
  uint32_t total = 0, vcount = 0;
  if (tid < kBins) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) total += pairs[w * kBins + tid].y;
    vcount = total - (tid == mask ? static_cast<uint32_t>(TILE) - valid : 0u);
    if (tid <= mask)
      st_relaxed64(status + static_cast<size_t>(tile) * kBins + tid,
                   tag(epoch, tile == 0 ? 2u : 1u, vcount));
  }
  uint32_t inc = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (tid < kBins && lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (tid < kBins) {
    uint32_t run = inc - total;
    for (unsigned w = 0; w < warp; ++w) run += warp_tot[w];
    bin_start[tid] = run;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = pairs[w * kBins + tid].y;
      pairs[w * kBins + tid].y = run;
      run += c;
    }
  }
  __syncthreads();

  // Reorder the tile by digit in shared memory.
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t dgt = static_cast<uint32_t>(key[k] >> shift) & mask;
    const uint32_t pos = wp[dgt].y + rank[k];
    keys_s[pos] = key[k];
    pay_s[pos] = pay[k];
  }

  // Decoupled look-back per bin: counts of the bin in all earlier tiles. A
  // whole wave of tiles publishes its aggregates at about the same time, so
  // the nearest inclusive prefix sits many tiles back; each thread therefore
  // reads kLook predecessors per round trip (independent loads, each a
  // coalesced 256-byte request per warp) instead of one.
  if (tid <= mask) {
    uint32_t before = 0;
    if (tile > 0) {
      constexpr int kLook = 8;
      int64_t t = static_cast<int64_t>(tile) - 1;  // next predecessor to consume
      bool done = false;
      while (!done) {
        unsigned long long w[kLook];
#pragma unroll
        for (int i = 0; i < kLook; ++i)
          w[i] = t - i >= 0 ? ld_relaxed64(status + static_cast<size_t>(t - i) * kBins + tid)
                            : tag(epoch, 2u, 0u);
        bool stall = false;
#pragma unroll
        for (int i = 0; i < kLook; ++i) {
          if (done || stall) continue;
          if ((w[i] >> 34) != epoch) {
            stall = true;  // not published yet: poll again from here
          } else {
            before += static_cast<uint32_t>(w[i]);
            done = ((w[i] >> 32) & 3u) == 2u;
          }
        }
        if (!done) {
          // consumed entries: every ready one before the first unpublished
          int used = 0;
#pragma unroll
          for (int i = kLook - 1; i >= 0; --i)
            if ((w[i] >> 34) != epoch) used = i;
          t -= stall ? used : kLook;
          if (stall) __nanosleep(20);
        }
      }
      st_relaxed64(status + static_cast<size_t>(tile) * kBins + tid,
                   tag(epoch, 2u, before + vcount));
    }
    gbase[tid] = base[tid] + before - bin_start[tid];
  }
  __syncthreads();

  // Each bin's run goes out contiguous: consecutive slots -> consecutive
  // global positions.
  {
    K kk[ITEMS];
    uint32_t pp[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t j = tid + k * kThreads;
      if (j < valid) {
        kk[k] = keys_s[j];
        pp[k] = pay_s[j];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t j = tid + k * kThreads;
      if (j >= valid) continue;
      const uint32_t dgt = static_cast<uint32_t>(kk[k] >> shift) & mask;
      const uint32_t pos = gbase[dgt] + j;
      if (DST == DST_ARRAYS) {
        __stcs(static_cast<K*>(d.keys) + pos, kk[k]);
        __stcs(d.pay + pos, pp[k]);
      } else if (DST == DST_UNPACK) {
#pragma unroll
        for (int q = 0; q < SPT_MAX_ORDER; ++q)
          if (q < d.un.n)
            __stcs(d.un.idx[q] + pos,
                   static_cast<uint32_t>(kk[k] >> d.un.shift[q]) & d.un.mask[q]);
        __stcs(d.pay + pos, pp[k]);
      } else {
        __stcs(d.pay + pos, pp[k]);
      }
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
  // digits of <= 8 bits; at least two passes, so that the first pass
  // (which reads the caller's arrays) never writes into them
  Digits dg{};
  if (nbits == 0) nbits = 1;
  int passes = static_cast<int>((nbits + 7) / 8);
  if (passes < 2) passes = 2;
  dg.passes = passes;
  // full 8-bit digits (their ballots unroll) and the remainder in the last
  uint32_t at = 0;
  for (int p = 0; p < passes; ++p) {
    const uint32_t w = std::min<uint32_t>(8u, nbits - at);
    dg.shift[p] = at;
    dg.bits[p] = w;
    at += w;
  }
  return dg;
}

template <typename K>
constexpr int items_for() {
  return sizeof(K) == 8 ? SPT_RADIX_ITEMS64 : SPT_RADIX_ITEMS32;
}

template <typename K, int SRC, int DST>
int launch_pass(spt_ctx* ctx, const SrcDesc& s, const DstDesc& d, uint64_t n, uint32_t shift,
                uint32_t bits, const uint32_t* base, uint32_t* ticket, cudaStream_t st) {
  constexpr int ITEMS = items_for<K>();
  constexpr size_t smem = onesweep_smem<K, ITEMS>();
  auto kern = bits == 8 ? onesweep_kernel<K, SRC, DST, ITEMS, 8>
                        : onesweep_kernel<K, SRC, DST, ITEMS, 0>;
  SPT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));  // per device, cheap
  const uint64_t tile = static_cast<uint64_t>(kThreads) * ITEMS;
  const uint64_t tiles = (n + tile - 1) / tile;
  unsigned long long* status;
  SPT_TRY(ctx_status64(ctx, tiles * kBins, &status));
  uint32_t epoch;
  SPT_TRY(ctx_lookback(ctx, 0, 0, &epoch));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(tiles));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  SPT_CUDA(cudaLaunchKernelEx(&cfg, kern, s, d, n, shift, bits, base,
                              static_cast<unsigned long long*>(status), epoch, ticket));
  ctx->launches++;
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
int carve(spt_ctx* ctx, uint64_t n, int npay, Buffers* b, cudaStream_t st) {
  const size_t kb = align_up(n * sizeof(K)), pb = align_up(n * 4);
  const size_t hb = align_up(kMaxPasses * kBins * 4);
  void* scratch;
  SPT_TRY(ctx_scratch(ctx, 2 * kb + npay * pb + 2 * hb + 256, &scratch));
  char* p = static_cast<char*>(scratch);
  b->key[0] = p;
  b->key[1] = p + kb;
  b->pay[0] = reinterpret_cast<uint32_t*>(p + 2 * kb);
  b->pay[1] = npay > 1 ? reinterpret_cast<uint32_t*>(p + 2 * kb + pb) : nullptr;
  b->hist = reinterpret_cast<uint32_t*>(p + 2 * kb + npay * pb);
  b->base = reinterpret_cast<uint32_t*>(p + 2 * kb + npay * pb + hb);
  b->ticket = reinterpret_cast<uint32_t*>(p + 2 * kb + npay * pb + 2 * hb);
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
  SPT_TRY(carve<K>(ctx, n, 2, &b, st));
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
  const int P = dg.passes;
  // Payload targets, chosen backwards from the last pass (-> perm_out): the
  // passes alternate between perm_out itself and one scratch array, so a
  // 1B-entry sort keeps one 4 GB payload buffer instead of two. Only a later
  // chunk (perm_in == perm_out is read by pass 0) with an odd pass count needs
  // a second one, for pass 0's output.
  const bool hazard = perm_in != nullptr && (P - 1) % 2 == 0;
  Buffers b;
  SPT_TRY(carve<K>(ctx, n, hazard ? 2 : 1, &b, st));
  auto pay_target = [&](int p) -> uint32_t* {
    if (p == 0 && hazard) return b.pay[1];
    return (P - 1 - p) % 2 == 0 ? perm_out : b.pay[0];
  };
  SrcDesc s0{};
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
  for (int p = 0; p < P; ++p) {
    const bool first = p == 0, last = p == P - 1;
    SrcDesc s{};
    DstDesc d{};
    if (first) {
      s = s0;
    } else {
      s.keys = b.key[(p - 1) & 1];
      s.pay = pay_target(p - 1);
    }
    d.keys = last ? nullptr : b.key[p & 1];
    d.pay = pay_target(p);
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
