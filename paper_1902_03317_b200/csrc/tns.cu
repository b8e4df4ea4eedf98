// Device-side ingest of the reference's text format (.tns): read_tns,
// P/src/io.cpp:42-120 (format: P/include/spten/io.hpp:14-20).
//
// The text is cut into 16 KB chunks; a line belongs to the chunk holding its
// first byte. Two passes, one CTA per chunk, each staging its chunk (plus the
// byte before it and, for the parse, a 2 KB tail) into shared memory with
// 16-byte loads, every thread owning the lines that start in its 64-byte
// segment (the staging is padded by 4 bytes per 64 so the 32 lanes' segments
// fall into distinct banks):
//   spt_tns_scan  -- count the entry lines of every chunk (first non-blank
//                    byte present and not '#'), the earliest entry line
//                    (atomicMin of its byte offset) for the order; one scan of
//                    the chunk counts gives every chunk's first output slot;
//   spt_tns_parse -- classify again, rank entries with a block scan, split
//                    tokens and parse the N 1-based indices and the value into
//                    slot order (= file order); per-mode maxima reduced in
//                    shared memory, one global atomic per CTA and mode.
// Acceptance is the reference's std::from_chars parsing: u64 digit strings
// for indices; for values the from_chars(float) grammar with correctly
// rounded decimal -> float conversion (Clinger's exact double path, else a
// double estimate accepted when it clears the neighbouring float midpoints
// by a margin, else settled exactly with big integers); out-of-range
// (overflow, or a nonzero value that rounds to zero) rejected like
// std::errc::result_out_of_range. Errors are the first failing line in file
// order (atomicMin of the line's byte offset), with the reference's
// messages; line numbers are counted only on that error path, and the host
// layer adds "path:line:".
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

struct spt_tns {
  spt_ctx* ctx = nullptr;
  const char* text = nullptr;
  uint64_t bytes = 0;
  uint64_t nchunks = 0;
  uint64_t* off = nullptr;  // [nchunks] first output slot of each chunk
  uint32_t order = 0;
  uint64_t nnz = 0;
  bool override_dims = false;
  uint32_t dims[SPT_MAX_ORDER] = {};
};

namespace {

enum TnsErr : uint32_t {
  kOk = 0,
  kTokenCount = 1,  // expected N+1 tokens, got K
  kBadIndex = 2,    // non-numeric index token
  kZeroIndex = 3,   // indices are 1-based; got 0
  kIndexRange = 4,  // index out of range (> 2^32-1)
  kOverDims = 5,    // index exceeds declared dimension
  kBadValue = 6,    // unparsable value
};


// ---- exact decimal -> float -------------------------------------------------

// Little-endian base-2^32 big integer. Sized for the slow path's worst case:
// <= kMaxDigits+1 significant digits (430 bits) times 10^|E| (|E| <= ~180
// there, 600 bits) or 2^151.
constexpr int kMaxDigits = 128;
struct Big {
  static constexpr int L = 48;
  uint32_t w[L];
  int n;
  __device__ void set(uint64_t v) {
    n = 0;
    while (v) w[n++] = static_cast<uint32_t>(v), v >>= 32;
  }
  __device__ void mul_add(uint32_t m, uint32_t a) {
    uint64_t carry = a;
    for (int i = 0; i < n; ++i) {
      const uint64_t t = (uint64_t)w[i] * m + carry;
      w[i] = static_cast<uint32_t>(t);
      carry = t >> 32;
    }
    if (carry && n < L) w[n++] = static_cast<uint32_t>(carry);
  }
  __device__ void pow10(int e) {
    for (; e >= 9; e -= 9) mul_add(1000000000u, 0);
    for (; e > 0; --e) mul_add(10u, 0);
  }
  __device__ void shl(int s) {
    const int words = s / 32, bits = s % 32;
    if (words && n) {
      const int nn = min(n + words, L);
      for (int i = nn - 1; i >= words; --i) w[i] = w[i - words];
      for (int i = 0; i < words; ++i) w[i] = 0;
      n = nn;
    }
    if (bits) {
      uint32_t carry = 0;
      for (int i = 0; i < n; ++i) {
        const uint32_t nc = w[i] >> (32 - bits);
        w[i] = (w[i] << bits) | carry;
        carry = nc;
      }
      if (carry && n < L) w[n++] = carry;
    }
  }
};

__device__ int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

// The significant decimal digits of a value token: chars [begin, end) minus
// the '.', the first nonzero, the first `nd` of them kept, then a trailing
// '1' when nonzero digits were dropped (`sticky`). Read straight from the
// text so the common path keeps no digit buffer.
template <class Src>
struct Digits {
  Src p;
  uint64_t base;
  int begin, end, nd;
  bool sticky;
  __device__ char operator[](int i) const { return p[base + i]; }
};

// sign(D * 10^E - m * 2^k), D the digit string.
template <class Src>
__device__ int cmp_decimal(const Digits<Src>& D, int E, uint64_t m, int k) {
  Big a, b;
  a.set(0);
  int taken = 0;
  for (int i = D.begin; i < D.end && taken < D.nd; ++i) {
    if (D[i] == '.') continue;
    a.mul_add(10u, static_cast<uint32_t>(D[i] - '0'));
    ++taken;
  }
  if (D.sticky) a.mul_add(10u, 1u);
  b.set(m);
  if (E >= 0) a.pow10(E);
  else b.pow10(-E);
  if (k >= 0) b.shl(k);
  else a.shl(-k);
  return big_cmp(a, b);
}

// f = fm * 2^fe for a finite non-negative float with these bits.
__device__ void float_parts(uint32_t bits, uint64_t* fm, int* fe) {
  if ((bits >> 23) == 0) {
    *fm = bits, *fe = -149;
  } else {
    *fm = (bits & 0x7FFFFFu) | 0x800000u;
    *fe = static_cast<int>(bits >> 23) - 150;
  }
}

// Correctly rounded float of D * 10^E (D: nd >= 1 digits, the first nonzero,
// m = its first min(nd, 19) digits, nt = their count): the exact path, else a
// double estimate moved to the right float by exact comparisons with the
// midpoints around it. false = out of range.
template <class Src>
__device__ bool decimal_to_float(const Digits<Src>& D, int E, uint64_t m, int nt, float* out) {
  const int nd = D.nd + D.sticky;
  const int mag = nd - 1 + E;  // value in [10^mag, 10^(mag+1))
  if (mag > 38) return false;   // >= 1e39 > FLT_MAX
  if (mag < -46) return false;  // < 1e-46, below denorm_min / 2 (7.0e-46)
  const int e10 = E + (nd - nt);
  if (nd <= 15 && e10 >= -22 && e10 <= 22) {
    // Clinger: m and 10^|e10| are exact doubles, so d is the correctly
    // rounded double; rounding it to float is then correct unless d sits
    // exactly on a float midpoint it did not start on (settled below).
    constexpr double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
    const double d = e10 >= 0 ? static_cast<double>(m) * p10[e10]
                              : static_cast<double>(m) / p10[-e10];
    const float f = __double2float_rn(d);
    if (isinf(f)) return false;
    const float g = d > static_cast<double>(f) ? nextafterf(f, INFINITY) : nextafterf(f, 0.f);
    const double mid = 0.5 * (static_cast<double>(f) + static_cast<double>(g));
    if (d != mid || d == static_cast<double>(f)) {
      if (f == 0.f) return false;
      *out = f;
      return true;
    }
  }
  // est is within a few double ulps of D * 10^E (19-digit m, exp10 <= 2 ulp,
  // one rounding): when est +- 2^-44 relative stays strictly between the
  // float midpoints around round(est), that float is the answer.
  const double est = static_cast<double>(m) * exp10(static_cast<double>(e10));
  constexpr double kEps = 0x1p-44;
  const double hi = est * (1 + kEps), lo = est * (1 - kEps);
  float f = __double2float_rn(est);
  if (isinf(f)) {
    if (lo > static_cast<double>(FLT_MAX) + 0x1p103) return false;  // past FLT_MAX's range
    f = FLT_MAX;
  } else if (f == 0.f) {
    if (hi < 0x1p-150) return false;  // below half of denorm_min
  } else {
    const double fd = f;
    const double up = 0.5 * (fd + (f == FLT_MAX ? 0x1p128 : static_cast<double>(
                                                                nextafterf(f, INFINITY))));
    const double dn = 0.5 * (fd + static_cast<double>(nextafterf(f, 0.f)));
    if (hi < up && lo > dn) {
      *out = f;
      return true;
    }
  }
  for (int iter = 0; iter < 8; ++iter) {
    const uint32_t bits = __float_as_uint(f);
    uint64_t fm;
    int fe;
    float_parts(bits, &fm, &fe);
    // upper midpoint (f + next(f)) / 2 = (2fm + 1) * 2^(fe-1); ties to even
    const int up = cmp_decimal(D, E, 2 * fm + 1, fe - 1);
    if (up > 0 || (up == 0 && (fm & 1))) {
      if (bits == 0x7F7FFFFFu) return false;  // rounds to infinity
      f = __uint_as_float(bits + 1);
      continue;
    }
    if (bits == 0) return false;  // a nonzero decimal rounding to zero
    // lower midpoint: (2fm - 1) * 2^(fe-1), or (4fm - 1) * 2^(fe-2) when f
    // opens a binade (its predecessor's spacing is half as wide)
    const bool boundary = (bits & 0x7FFFFFu) == 0 && (bits >> 23) > 1;
    const int lo = boundary ? cmp_decimal(D, E, 4 * fm - 1, fe - 2)
                            : cmp_decimal(D, E, 2 * fm - 1, fe - 1);
    if (lo < 0 || (lo == 0 && (fm & 1))) {
      f = __uint_as_float(bits - 1);
      continue;
    }
    break;
  }
  if (__float_as_uint(f) == 0) return false;
  *out = f;
  return true;
}

__device__ __forceinline__ char lower(char c) {
  return (c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : c;
}

// std::from_chars(float), chars_format::general, over the whole token
// S[s, s+n): [-](digits[.digits]|.digits)[(e|E)[+-]digits] | [-]inf |
// [-]infinity | [-]nan[(chars)], the words case-insensitive; no '+', no hex.
template <class Src>
__device__ bool parse_float(const Src& S, uint64_t s, int n, float* out) {
  auto at = [&](int k) { return S[s + k]; };
  int i = 0;
  bool neg = false;
  if (i < n && at(i) == '-') neg = true, ++i;
  if (i < n && (lower(at(i)) == 'i' || lower(at(i)) == 'n')) {
    auto word = [&](const char* w) {
      int k = 0;
      for (; w[k]; ++k)
        if (i + k >= n || lower(at(i + k)) != w[k]) return false;
      return true;
    };
    if ((word("infinity") && i + 8 == n) || (word("inf") && i + 3 == n)) {
      *out = neg ? -INFINITY : INFINITY;
      return true;
    }
    if (word("nan")) {
      int j = i + 3;
      bool ok = j == n;
      if (!ok && at(j) == '(') {
        ++j;
        while (j < n && (at(j) == '_' || (at(j) >= '0' && at(j) <= '9') ||
                         (lower(at(j)) >= 'a' && lower(at(j)) <= 'z')))
          ++j;
        ok = j + 1 == n && at(j) == ')';
      }
      if (ok) {
        const float q = __int_as_float(0x7FC00000);
        *out = neg ? -q : q;
        return true;
      }
    }
    return false;
  }
  Digits<Src> D{S, s, -1, 0, 0, false};
  uint64_t m = 0;  // the first 19 significant digits
  int nt = 0, E = 0, seen = 0;
  bool frac = false;
  for (; i < n; ++i) {
    const char c = at(i);
    if (c == '.' && !frac) {
      frac = true;
      continue;
    }
    if (c < '0' || c > '9') break;
    ++seen;
    if (D.nd == 0 && c == '0') {
      E -= frac;
      continue;
    }
    if (D.begin < 0) D.begin = i;
    if (D.nd < kMaxDigits) {
      ++D.nd;
      E -= frac;
      if (nt < 19) m = m * 10 + static_cast<uint64_t>(c - '0'), ++nt;
    } else {
      E += !frac;
      D.sticky |= c != '0';
    }
  }
  D.end = i;
  if (!seen) return false;
  if (i < n && (at(i) == 'e' || at(i) == 'E')) {
    int j = i + 1;
    bool eneg = false;
    if (j < n && (at(j) == '+' || at(j) == '-')) eneg = at(j) == '-', ++j;
    if (j < n && at(j) >= '0' && at(j) <= '9') {
      int ev = 0;
      for (; j < n && at(j) >= '0' && at(j) <= '9'; ++j)
        ev = ev < 10000000 ? ev * 10 + (at(j) - '0') : ev;
      E += eneg ? -ev : ev;
      i = j;
    }  // else the exponent is not part of the number and the token fails below
  }
  if (i != n) return false;
  float f = 0.f;
  if (D.nd) {
    // Dropped digits only matter against a midpoint (<= 112 significant
    // digits, fewer than the kept ones): D stands them in by a trailing 1.
    if (D.sticky) --E;
    if (!decimal_to_float(D, E, m, nt, &f)) return false;
  }
  *out = neg ? -f : f;
  return true;
}

// ---- chunked passes ---------------------------------------------------------

constexpr int kChunk = 16384;             // text bytes per CTA
constexpr int kThreads = 256;             // one 64-byte segment per thread
constexpr int kSeg = kChunk / kThreads;   // 64
constexpr int kPre = 16;                  // staged bytes before the chunk
constexpr int kTail = 2048;               // staged bytes after it (parse pass)
constexpr int kWinMax = kPre + kChunk + kTail;
constexpr int kPadded = kWinMax + (kWinMax / 64 + 1) * 4;

__device__ __forceinline__ uint32_t pad(uint32_t o) { return o + ((o >> 6) << 2); }

// Text bytes: the staged window from shared memory, the rest from global;
// before 0 and from `bytes` on, '\n' (so offset 0 starts a line and the end
// of the text ends one).
struct Src {
  const uint8_t* sm;
  int64_t ws;     // text offset of window byte 0 (may be negative)
  uint32_t wlen;  // staged bytes
  const char* g;
  uint64_t bytes;
  __device__ __forceinline__ char operator[](uint64_t pos) const {
    const uint64_t o = pos - static_cast<uint64_t>(ws);
    if (o < wlen) return static_cast<char>(sm[pad(static_cast<uint32_t>(o))]);
    return pos < bytes ? g[pos] : '\n';
  }
};

// Stage text [ws, ws + wlen) into sm (padded); out-of-text bytes become '\n'.
__device__ void stage(uint8_t* sm, const char* g, uint64_t bytes, int64_t ws, uint32_t wlen,
                      bool vec) {
  // ws is 16-aligned relative to the text; vec: g is 16-byte aligned too
  for (uint32_t o = threadIdx.x * 16; o < wlen; o += kThreads * 16) {
    const int64_t pos = ws + o;
    uint32_t w[4];
    if (vec && pos >= 0 && static_cast<uint64_t>(pos) + 16 <= bytes) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(g + pos));
      w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else {
      for (int k = 0; k < 4; ++k) {
        uint32_t x = 0;
        for (int b = 0; b < 4; ++b) {
          const int64_t q = pos + 4 * k + b;
          const uint32_t c = (q >= 0 && static_cast<uint64_t>(q) < bytes)
                                 ? static_cast<uint8_t>(g[q]) : static_cast<uint32_t>('\n');
          x |= c << (8 * b);
        }
        w[k] = x;
      }
    }
    uint32_t* d = reinterpret_cast<uint32_t*>(sm + pad(o));
    d[0] = w[0], d[1] = w[1], d[2] = w[2], d[3] = w[3];
  }
}

// Line starting at p: its end e (exclusive, without '\n' and one trailing
// '\r', P/src/io.cpp:65) and whether it is an entry line (a non-blank first
// byte that is not '#', io.cpp:66-67).
__device__ __forceinline__ bool line_at(const Src& S, uint64_t p, uint64_t* e) {
  uint64_t q = p;
  while (S[q] == ' ' || S[q] == '\t') ++q;
  uint64_t k = q;
  while (S[k] != '\n') ++k;
  if (k > p && S[k - 1] == '\r') --k;
  *e = k;
  return q < k && S[q] != '#';
}

struct Chunk {
  int64_t ws;
  uint32_t wlen;
  uint64_t c0, c1;  // the chunk's text range
};

__device__ __forceinline__ Chunk chunk_of(uint64_t c, uint64_t bytes, int tail) {
  Chunk k;
  k.c0 = c * kChunk;
  k.c1 = min(k.c0 + kChunk, bytes);
  k.ws = static_cast<int64_t>(k.c0) - kPre;
  k.wlen = static_cast<uint32_t>(kPre + (k.c1 - k.c0) + tail);
  return k;
}

// Bit i set: byte p = seg + i starts a line (p == 0 or byte p-1 is '\n'),
// for the thread's 64-byte segment [seg, seg + 64) of the staged window
// (window offset o = seg - ws, a multiple of 64 minus kPre's 16). Word-wide
// compares: no per-byte divergence.
__device__ __forceinline__ uint64_t line_starts(const uint8_t* sm, uint32_t o) {
  uint64_t nl = 0;
#pragma unroll
  for (int w = 0; w < 16; ++w) {
    const uint32_t x = *reinterpret_cast<const uint32_t*>(sm + pad(o + 4 * w));
    const uint32_t m = __vcmpeq4(x, 0x0A0A0A0Au) & 0x01010101u;
    nl |= static_cast<uint64_t>(((m * 0x00204081u) >> 21) & 0xFu) << (4 * w);
  }
  const uint64_t before = sm[pad(o - 1)] == '\n';
  return (nl << 1) | before;
}

// Entry line starting at p (P/src/io.cpp:65-67): its first byte that is not
// ' ' / '\t' exists, is not '#', and is not the '\r' stripped before a '\n'.
__device__ __forceinline__ bool is_entry(const Src& S, uint64_t p) {
  char c = S[p];
  while (c == ' ' || c == '\t') c = S[++p];
  return c != '\n' && c != '#' && !(c == '\r' && S[p + 1] == '\n');
}

// Entry lines among the starts in `m` (bits of segment base a, below limit).
__device__ __forceinline__ uint64_t entry_mask(const Src& S, uint64_t a, uint64_t m) {
  uint64_t e = 0;
  while (m) {
    const int i = __ffsll(static_cast<long long>(m)) - 1;
    m &= m - 1;
    if (is_entry(S, a + i)) e |= 1ull << i;
  }
  return e;
}

// Pass 1: entry lines per chunk; the earliest entry line's byte offset.
__global__ void __launch_bounds__(kThreads) tns_count_kernel(
    const char* g, uint64_t bytes, uint64_t nchunks, bool vec, uint64_t* counts,
    unsigned long long* first_entry) {
  __shared__ __align__(16) uint8_t sm[kPadded];
  __shared__ uint32_t s_cnt;
  __shared__ unsigned long long s_first;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const Chunk k = chunk_of(c, bytes, 0);
    if (threadIdx.x == 0) s_cnt = 0, s_first = ~0ull;
    stage(sm, g, bytes, k.ws, k.wlen, vec);
    __syncthreads();
    const Src S{sm, k.ws, k.wlen, g, bytes};
    const uint64_t a = k.c0 + threadIdx.x * kSeg;
    uint64_t m = 0;
    if (a < k.c1) {
      m = line_starts(sm, kPre + threadIdx.x * kSeg);
      if (k.c1 - a < 64) m &= (1ull << (k.c1 - a)) - 1;
      m = entry_mask(S, a, m);
    }
    uint32_t n = __popcll(m);
    unsigned long long first = m ? a + (__ffsll(static_cast<long long>(m)) - 1) : ~0ull;
    n = __reduce_add_sync(0xFFFFFFFFu, n);
#pragma unroll
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xFFFFFFFFu, first, o));
    if ((threadIdx.x & 31) == 0) {
      if (n) atomicAdd(&s_cnt, n);
      if (first != ~0ull) atomicMin(&s_first, first);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      counts[c] = s_cnt;
      if (s_first != ~0ull) atomicMin(first_entry, s_first);
    }
    __syncthreads();
  }
}

struct ParseArgs {
  uint32_t* idx[SPT_MAX_ORDER];
  float* val;
  uint32_t* maxidx;  // [N], atomicMax (no override)
  uint32_t dims[SPT_MAX_ORDER];
  uint32_t override_dims;
  uint32_t N;
  unsigned long long* err;  // byte offset of the first failing line (atomicMin)
};

// Parse the entry line [p, e) into slot `rank` (write) or just check it.
// Returns 0 or code | token << 8; span = the failing token, ntok = tokens.
__device__ uint32_t parse_line(const Src& S, uint64_t p, uint64_t e, const ParseArgs& P,
                               uint32_t rank, bool write, uint32_t* smax, uint64_t* span,
                               uint32_t* ntok) {
  uint32_t t = 0;  // the token count is checked first (P/src/io.cpp:69-78)
  {
    bool in = false;
    for (uint64_t k = p; k < e; ++k) {
      const char c = S[k];
      const bool w = c == ' ' || c == '\t';
      t += !w && !in;
      in = !w;
    }
  }
  *ntok = t;
  if (t != P.N + 1) return kTokenCount;
  uint64_t k = p;
  for (uint32_t d = 0; d <= P.N; ++d) {
    while (k < e && (S[k] == ' ' || S[k] == '\t')) ++k;
    const uint64_t s = k;
    while (k < e && S[k] != ' ' && S[k] != '\t') ++k;
    span[0] = s, span[1] = k;
    const int n = static_cast<int>(k - s);
    if (d < P.N) {
      uint64_t raw = 0;
      bool ok = true;
      for (int j = 0; j < n && ok; ++j) {
        const uint32_t c = static_cast<uint32_t>(static_cast<uint8_t>(S[s + j])) - '0';
        if (c > 9 || raw > (~0ull - c) / 10) ok = false;  // non-digit, or past u64
        else raw = raw * 10 + c;
      }
      if (!ok) return kBadIndex | d << 8;
      if (raw < 1) return kZeroIndex | d << 8;
      if (raw > 0xFFFFFFFFull) return kIndexRange | d << 8;
      const uint32_t id = static_cast<uint32_t>(raw - 1);
      if (P.override_dims && id >= P.dims[d]) return kOverDims | d << 8;
      if (write) {
        P.idx[d][rank] = id;
        if (!P.override_dims) atomicMax(smax + d, id);
      }
    } else {
      float v;
      if (!parse_float(S, s, n, &v)) return kBadValue | d << 8;
      if (write) P.val[rank] = v;
    }
  }
  return kOk;
}

// The hot-path twin of parse_line: one pass over the entry line at p,
// splitting tokens as it parses them (indices written as they are read,
// wherever the line later fails -- a failed parse returns no tensor). Same
// verdict as parse_line: the token count first, then the first failing token
// (P/src/io.cpp:69-109); the error path re-derives the code and token.
// Window-relative text access for the hot path: 32-bit offsets o from the
// window start ws; staged bytes from shared memory, the rest (lines running
// past the 2 KB tail) from global memory, '\n' past the end of the text.
struct Win {
  const uint8_t* sm;
  uint32_t wlen;
  int64_t ws;
  const char* g;
  uint64_t bytes;
  __device__ __forceinline__ char operator[](uint64_t pos) const {
    const uint32_t o = static_cast<uint32_t>(pos);
    if (o < wlen) return static_cast<char>(sm[pad(o)]);
    const uint64_t q = static_cast<uint64_t>(ws + static_cast<int64_t>(o));
    return q < bytes ? g[q] : '\n';
  }
};

// The shared copy of the output arrays / declared dims (indexed by token).
struct Outs {
  uint32_t* idx[SPT_MAX_ORDER];
  uint32_t dims[SPT_MAX_ORDER];
};

__device__ __forceinline__ bool token_end(const Win& S, char c, uint32_t k) {
  return c == ' ' || c == '\t' || c == '\n' || (c == '\r' && S[k + 1] == '\n');
}

__device__ uint32_t parse_entry(const Win& S, uint32_t o, const Outs& O, uint32_t N,
                                bool override_dims, float* val, uint32_t rank, uint32_t* smax) {
  uint32_t d = 0, err = kOk;
  uint32_t k = o;
  char c = S[k];
  for (;;) {
    while (c == ' ' || c == '\t') c = S[++k];
    if (c == '\n' || (c == '\r' && S[k + 1] == '\n')) break;
    const uint32_t s = k;
    if (d < N) {
      uint64_t raw = 0;
      uint32_t bad = 0;
      do {
        const uint32_t v = static_cast<uint32_t>(static_cast<uint8_t>(c)) - '0';
        bad |= v > 9;
        raw = raw * 10 + v;
        c = S[++k];
      } while (!token_end(S, c, k));
      if (k - s > 19 && !bad) {  // may pass 2^64 - 1: redo exactly (rare)
        uint64_t r = 0;
        for (uint32_t j = s; j < k; ++j) {
          const uint32_t v = static_cast<uint32_t>(static_cast<uint8_t>(S[j])) - '0';
          if (r > 1844674407370955161ull || (r == 1844674407370955161ull && v > 5)) bad = 1;
          r = r * 10 + v;
        }
      }
      if (err == kOk) {
        if (bad) err = kBadIndex;
        else if (raw < 1) err = kZeroIndex;
        else if (raw > 0xFFFFFFFFull) err = kIndexRange;
        else if (override_dims && raw - 1 >= O.dims[d]) err = kOverDims;
      }
      if (err == kOk) {
        const uint32_t id = static_cast<uint32_t>(raw - 1);
        O.idx[d][rank] = id;
        if (!override_dims) atomicMax(smax + d, id);
      }
    } else {
      do c = S[++k];
      while (!token_end(S, c, k));
      if (d == N && err == kOk) {
        float v;
        if (parse_float(S, s, static_cast<int>(k - s), &v)) val[rank] = v;
        else err = kBadValue;
      }
    }
    ++d;
  }
  return d != N + 1 ? kTokenCount : err;
}

// Pass 2: list the chunk's entry lines in file order (block scan of the
// per-thread entry counts from the chunk's first slot), then parse them
// round-robin, 32 lines per warp side by side.
__global__ void __launch_bounds__(kThreads) tns_parse_kernel(
    const char* g, uint64_t bytes, uint64_t nchunks, bool vec, const uint64_t* off,
    ParseArgs P) {
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  __shared__ __align__(16) uint8_t sm[kPadded];
  __shared__ uint16_t list[kChunk / 2];  // an entry line has >= 2 bytes
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t smax[SPT_MAX_ORDER];
  __shared__ Outs O;
  if (threadIdx.x < SPT_MAX_ORDER) {
    smax[threadIdx.x] = 0;
    O.idx[threadIdx.x] = P.idx[threadIdx.x];
    O.dims[threadIdx.x] = P.dims[threadIdx.x];
  }
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const Chunk k = chunk_of(c, bytes, kTail);
    stage(sm, g, bytes, k.ws, k.wlen, vec);
    __syncthreads();
    const Src S{sm, k.ws, k.wlen, g, bytes};
    const uint64_t a = k.c0 + threadIdx.x * kSeg;
    uint64_t m = 0;
    if (a < k.c1) {
      m = line_starts(sm, kPre + threadIdx.x * kSeg);
      if (k.c1 - a < 64) m &= (1ull << (k.c1 - a)) - 1;
      m = entry_mask(S, a, m);
    }
    uint32_t pos, total;
    Scan(scan_tmp).ExclusiveSum(static_cast<uint32_t>(__popcll(m)), pos, total);
    while (m) {
      const int i = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      list[pos++] = static_cast<uint16_t>(threadIdx.x * kSeg + i);
    }
    __syncthreads();
    const uint64_t base = off[c];
    const Win W{sm, k.wlen, k.ws, g, bytes};
    for (uint32_t i = threadIdx.x; i < total; i += kThreads) {
      const uint32_t o = kPre + list[i];  // window offset of the line
      if (parse_entry(W, o, O, P.N, P.override_dims, P.val, static_cast<uint32_t>(base + i),
                      smax) != kOk)
        atomicMin(P.err, static_cast<unsigned long long>(k.c0 + list[i]));
    }
    __syncthreads();  // sm, list and scan_tmp are reused by the next chunk
  }
  if (threadIdx.x < P.N && !P.override_dims && smax[threadIdx.x])
    atomicMax(P.maxidx + threadIdx.x, smax[threadIdx.x]);
}

// Tokens of the line starting at byte p (one thread).
__global__ void line_tokens_kernel(const char* g, uint64_t bytes, uint64_t p, uint32_t* out) {
  const Src S{nullptr, 0, 0, g, bytes};
  uint64_t e;
  line_at(S, p, &e);
  uint32_t t = 0;
  bool in = false;
  for (uint64_t k = p; k < e; ++k) {
    const bool w = S[k] == ' ' || S[k] == '\t';
    t += !w && !in;
    in = !w;
  }
  *out = t;
}

// '\n' bytes in [0, upto): the 1-based line number of byte `upto` minus one.
__global__ void count_newlines_kernel(const char* g, uint64_t upto, unsigned long long* count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < upto; i += stride)
    c += g[i] == '\n';
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

// The failing token of the line at byte p, and its token count (one thread).
__global__ void error_token_kernel(const char* g, uint64_t bytes, uint64_t p, ParseArgs P,
                                   uint64_t* span, uint32_t* ntok) {
  const Src S{nullptr, 0, 0, g, bytes};
  uint64_t e;
  line_at(S, p, &e);
  span[0] = span[1] = 0;
  ntok[1] = parse_line(S, p, e, P, 0, false, nullptr, span, ntok);
}

// Temporaries freed (stream-ordered) when the scope ends.
struct Scratch {
  spt_ctx* ctx;
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t get(T** p, size_t bytes) {
    const cudaError_t e = spt::tmp_alloc(ctx, p, bytes ? bytes : 1, st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

unsigned chunk_grid(spt_ctx* ctx, uint64_t nchunks) {
  return static_cast<unsigned>(std::min<uint64_t>(nchunks, static_cast<uint64_t>(ctx->num_sms) * 8));
}

// 1-based line number of the line starting at byte p.
int line_number(spt_ctx* ctx, const char* g, uint64_t p, cudaStream_t st, uint64_t* line) {
  Scratch tmp{ctx, st, {}};
  unsigned long long* d;
  SPT_CUDA(tmp.get(&d, 8));
  SPT_CUDA(cudaMemsetAsync(d, 0, 8, st));
  if (p) {
    count_newlines_kernel<<<spt::grid_for(p, 256, ctx->num_sms * 4), 256, 0, st>>>(g, p, d);
    SPT_LAUNCHED(ctx);
  }
  unsigned long long h = 0;
  SPT_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
  SPT_CUDA(cudaStreamSynchronize(st));
  *line = h + 1;
  return SPT_OK;
}

}  // namespace

extern "C" void spt_tns_destroy(spt_tns* s) {
  if (!s) return;
  cudaFree(s->off);
  delete s;
}

extern "C" int spt_tns_scan(spt_ctx* ctx, const char* d_text, uint64_t bytes,
                            const uint32_t* dims_override, uint32_t n_override, spt_tns** out,
                            uint32_t* order, uint64_t* nnz, uint64_t* err_line, void* stream) {
  if (!ctx || !out) return spt::set_error(SPT_EINVAL, "read_tns: null context or output");
  *out = nullptr;
  if (err_line) *err_line = 0;
  if (dims_override && n_override == 0)  // P/src/io.cpp:52
    return spt::set_error(SPT_EINVAL, "read_tns: dims override must not be empty");
  if (dims_override && n_override > SPT_MAX_ORDER)
    return spt::set_error(SPT_EOVERFLOW, "read_tns: order %u exceeds %d", n_override,
                          SPT_MAX_ORDER);
  if (bytes && !d_text) return spt::set_error(SPT_EINVAL, "read_tns: null text");
  if (bytes >> 47)
    return spt::set_error(SPT_EOVERFLOW, "read_tns: text of %llu bytes exceeds 2^47",
                          (unsigned long long)bytes);
  cudaStream_t st = spt::as_stream(stream);
  Scratch tmp{ctx, st, {}};
  spt_tns* s = new spt_tns;
  struct Owner {
    spt_tns*& s;
    ~Owner() { spt_tns_destroy(s); }
  } owner{s};
  s->ctx = ctx;
  s->text = d_text;
  s->bytes = bytes;
  s->nchunks = (bytes + kChunk - 1) / kChunk;
  unsigned long long first = ~0ull;
  if (s->nchunks) {
    uint64_t* counts;
    unsigned long long* dfirst;
    SPT_CUDA(cudaMalloc(&s->off, (s->nchunks + 1) * sizeof(uint64_t)));
    SPT_CUDA(tmp.get(&counts, (s->nchunks + 1) * sizeof(uint64_t)));
    SPT_CUDA(tmp.get(&dfirst, 8));
    SPT_CUDA(cudaMemsetAsync(dfirst, 0xFF, 8, st));
    SPT_CUDA(cudaMemsetAsync(counts + s->nchunks, 0, 8, st));
    const bool vec = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    tns_count_kernel<<<chunk_grid(ctx, s->nchunks), kThreads, 0, st>>>(
        d_text, bytes, s->nchunks, vec, counts, dfirst);
    SPT_LAUNCHED(ctx);
    size_t tb = 0;
    SPT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, s->off, s->nchunks + 1, st));
    char* scan_tmp;
    SPT_CUDA(tmp.get(&scan_tmp, tb));
    SPT_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, tb, counts, s->off, s->nchunks + 1, st));
    ctx->launches += 2;
    SPT_CUDA(cudaMemcpyAsync(&s->nnz, s->off + s->nchunks, 8, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaMemcpyAsync(&first, dfirst, 8, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
  }
  if (dims_override) {
    s->order = n_override;
    s->override_dims = true;
    std::memcpy(s->dims, dims_override, n_override * sizeof(uint32_t));
  } else if (s->nnz) {
    uint32_t* dt;
    SPT_CUDA(tmp.get(&dt, 4));
    line_tokens_kernel<<<1, 1, 0, st>>>(d_text, bytes, first, dt);
    SPT_LAUNCHED(ctx);
    uint32_t t = 0;
    SPT_CUDA(cudaMemcpyAsync(&t, dt, 4, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
    if (t < 2 || t - 1 > SPT_MAX_ORDER) {
      uint64_t line = 0;
      SPT_TRY(line_number(ctx, d_text, first, st, &line));
      if (err_line) *err_line = line;
      if (t < 2)  // P/src/io.cpp:71-72
        return spt::set_error(SPT_ERUNTIME, "need at least one index and a value per entry");
      return spt::set_error(SPT_EOVERFLOW, "order %u exceeds %d", t - 1, SPT_MAX_ORDER);
    }
    s->order = t - 1;
  } else {  // P/src/io.cpp:112-114
    return spt::set_error(SPT_ERUNTIME, "has no entries and no dims override; order is unknown");
  }
  if (order) *order = s->order;
  if (nnz) *nnz = s->nnz;
  *out = s;
  s = nullptr;  // handed to the caller
  return SPT_OK;
}

extern "C" int spt_tns_parse(spt_ctx* ctx, const spt_tns* s, spt_coo* z, uint64_t* err_line,
                             void* stream) {
  if (!ctx || !s || !z) return spt::set_error(SPT_EINVAL, "read_tns: null argument");
  if (err_line) *err_line = 0;
  if (s->nnz >= (1ull << 32))
    return spt::set_error(SPT_EOVERFLOW, "read_tns: %llu entries exceed the u32 offset range",
                          (unsigned long long)s->nnz);
  if (s->nnz) {
    for (uint32_t d = 0; d < s->order; ++d)
      if (!z->idx[d])
        return spt::set_error(SPT_EINVAL, "read_tns: null index array for mode %u", d);
    if (!z->val) return spt::set_error(SPT_EINVAL, "read_tns: null value array");
  }
  cudaStream_t st = spt::as_stream(stream);
  Scratch tmp{ctx, st, {}};
  unsigned long long* derr;
  uint32_t* maxidx;
  SPT_CUDA(tmp.get(&derr, 8));
  SPT_CUDA(tmp.get(&maxidx, SPT_MAX_ORDER * sizeof(uint32_t)));
  SPT_CUDA(cudaMemsetAsync(derr, 0xFF, 8, st));
  SPT_CUDA(cudaMemsetAsync(maxidx, 0, SPT_MAX_ORDER * sizeof(uint32_t), st));
  ParseArgs P{};
  for (uint32_t d = 0; d < s->order; ++d) P.idx[d] = z->idx[d], P.dims[d] = s->dims[d];
  P.val = z->val;
  P.maxidx = maxidx;
  P.override_dims = s->override_dims;
  P.N = s->order;
  P.err = derr;
  unsigned long long err = ~0ull;
  uint32_t mx[SPT_MAX_ORDER] = {};
  if (s->nchunks) {
    const bool vec = (reinterpret_cast<uintptr_t>(s->text) & 15) == 0;
    tns_parse_kernel<<<chunk_grid(ctx, s->nchunks), kThreads, 0, st>>>(
        s->text, s->bytes, s->nchunks, vec, s->off, P);
    SPT_LAUNCHED(ctx);
    SPT_CUDA(cudaMemcpyAsync(&err, derr, 8, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaMemcpyAsync(mx, maxidx, sizeof mx, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
  }
  if (err != ~0ull) {
    const uint64_t p = err;
    uint64_t line = 0;
    SPT_TRY(line_number(ctx, s->text, p, st, &line));
    if (err_line) *err_line = line;
    uint64_t* dspan;
    SPT_CUDA(tmp.get(&dspan, 3 * sizeof(uint64_t)));
    error_token_kernel<<<1, 1, 0, st>>>(s->text, s->bytes, p, P, dspan,
                                        reinterpret_cast<uint32_t*>(dspan + 2));
    SPT_LAUNCHED(ctx);
    uint64_t span[3] = {0, 0, 0};
    SPT_CUDA(cudaMemcpyAsync(span, dspan, sizeof span, cudaMemcpyDeviceToHost, st));
    SPT_CUDA(cudaStreamSynchronize(st));
    const uint32_t nt = static_cast<uint32_t>(span[2]);
    const uint32_t code = static_cast<uint32_t>(span[2] >> 32) & 0xFF;
    const uint32_t mode = static_cast<uint32_t>(span[2] >> 40) & 0xFF;
    std::string tok(static_cast<size_t>(std::min<uint64_t>(span[1] - span[0], 400)), '\0');
    if (!tok.empty())
      SPT_CUDA(cudaMemcpy(&tok[0], s->text + span[0], tok.size(), cudaMemcpyDeviceToHost));
    // the index as std::to_string prints it (codes 4, 5: a valid u64)
    unsigned long long raw = 0;
    for (char c : tok) raw = raw * 10 + static_cast<unsigned>(c - '0');
    switch (code) {  // messages of P/src/io.cpp:74-108
      case kTokenCount:
        return spt::set_error(SPT_ERUNTIME, "expected %u tokens, got %u", s->order + 1, nt);
      case kBadIndex:
        return spt::set_error(SPT_ERUNTIME, "non-numeric index token '%s'", tok.c_str());
      case kZeroIndex:
        return spt::set_error(SPT_ERUNTIME, "indices are 1-based; got 0");
      case kIndexRange:
        return spt::set_error(SPT_ERUNTIME, "index %llu out of range", raw);
      case kOverDims:
        return spt::set_error(SPT_ERUNTIME, "index %llu exceeds declared dimension %u of mode %u",
                              raw, s->dims[mode], mode);
      default:
        return spt::set_error(SPT_ERUNTIME, "unparsable value '%s'", tok.c_str());
    }
  }
  z->order = s->order;
  z->nnz = s->nnz;
  for (uint32_t d = 0; d < s->order; ++d)
    z->dims[d] = s->override_dims ? s->dims[d] : (s->nnz ? mx[d] + 1 : 0);
  z->has_sort_order = 0;
  z->coalesced = 0;
  return SPT_OK;
}
