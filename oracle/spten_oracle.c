/*
 * spten_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference library's CPU algorithms for the hot
 * path (spten, /root/reference/proj = "P/"), used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker.
 * The product (libspten_b200.so and the paper_1902_03317_b200 package) never
 * links, imports or calls this file.
 *
 * Every function follows the reference statement cited beside it, operation
 * for operation, in the reference's evaluation order and precision (fp32 for
 * the sequential kernels), so ts/tew_eq/tew/sort/coalesce/fiber-index results
 * are bit-identical to spten::seq. For the reductions (ttv/ttm/mttkrp) it
 * additionally returns an fp64 recomputation from the same fp32 inputs and
 * the fp64 sum of |terms|, which the tolerance tests use.
 *
 * Pinned against the real reference: tests/golden/*.npz are produced by the
 * reference itself (oracle/_ref, built from P/src by oracle/Makefile) through
 * tests/golden/make_golden.py, and tests/test_oracle.py checks this file
 * against them bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_ORDER 8

/* apply_elem, P/src/kernel_detail.hpp:19-27 */
static float elem(int op, float a, float b) {
  switch (op) {
    case 0: return a + b;
    case 1: return a - b;
    case 2: return a * b;
    default: return a / b;
  }
}

/* seq::ts, P/src/kernels_seq.cpp:55-67 (apply_scalar P/src/kernel_detail.hpp:29-32) */
void or_ts(uint64_t nnz, int order, const uint32_t* const* xi, const float* xv, float s, int op,
           uint32_t** zi, float* zv) {
  for (int d = 0; d < order; ++d) memcpy(zi[d], xi[d], nnz * sizeof(uint32_t));
  for (uint64_t m = 0; m < nnz; ++m) zv[m] = op == 0 ? xv[m] + s : xv[m] * s;
}

/* seq::tew_eq, P/src/kernels_seq.cpp:11-39. Returns 0 ok, 1 pattern mismatch
 * (invalid_argument), 2 division by a stored zero (domain_error); *err_entry
 * receives the failing entry (first failing entry, pattern checked first). */
int or_tew_eq(uint64_t nnz, int order, const uint32_t* const* xi, const float* xv,
              const uint32_t* const* yi, const float* yv, int op, uint32_t** zi, float* zv,
              uint64_t* err_entry) {
  for (int d = 0; d < order; ++d) memcpy(zi[d], xi[d], nnz * sizeof(uint32_t));
  for (uint64_t m = 0; m < nnz; ++m) {
    for (int d = 0; d < order; ++d)
      if (xi[d][m] != yi[d][m]) {
        *err_entry = m;
        return 1;
      }
    if (op == 3 && yv[m] == 0.0f) {
      *err_entry = m;
      return 2;
    }
    zv[m] = elem(op, xv[m], yv[m]);
  }
  return 0;
}

/* compare_entries, P/include/spten/tensor.hpp:94-104 */
static int cmp_entries(int order, const uint32_t* const* xi, uint64_t a, const uint32_t* const* yi,
                       uint64_t b, const uint32_t* mo) {
  for (int k = 0; k < order; ++k) {
    const uint32_t d = mo[k];
    const uint32_t ia = xi[d][a], ib = yi[d][b];
    if (ia != ib) return ia < ib ? -1 : 1;
  }
  return 0;
}

/* sort_lexicographic, P/src/tensor.cpp:54-64: the permutation that
 * std::stable_sort produces (bottom-up merge sort of 0..nnz-1; stable). */
void or_sort_perm(uint64_t nnz, int order, const uint32_t* const* xi, const uint32_t* mo,
                  uint64_t* perm) {
  uint64_t* tmp = (uint64_t*)malloc((nnz ? nnz : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < nnz; ++i) perm[i] = i;
  uint64_t* a = perm;
  uint64_t* b = tmp;
  for (uint64_t w = 1; w < nnz; w *= 2) {
    for (uint64_t lo = 0; lo < nnz; lo += 2 * w) {
      uint64_t mid = lo + w < nnz ? lo + w : nnz;
      uint64_t hi = lo + 2 * w < nnz ? lo + 2 * w : nnz;
      uint64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        /* take right only if strictly less: keeps equal entries in order */
        if (cmp_entries(order, xi, a[j], xi, a[i], mo) < 0) b[k++] = a[j++];
        else b[k++] = a[i++];
      }
      while (i < mid) b[k++] = a[i++];
      while (j < hi) b[k++] = a[j++];
    }
    uint64_t* t = a;
    a = b;
    b = t;
  }
  if (a != perm) memcpy(perm, a, nnz * sizeof(uint64_t));
  free(tmp);
}

/* gather_entries, P/src/tensor.cpp:39-50 (in place through a buffer). */
void or_apply_perm(uint64_t nnz, int order, uint32_t** xi, float* xv, const uint64_t* perm) {
  uint32_t* ib = (uint32_t*)malloc((nnz ? nnz : 1) * sizeof(uint32_t));
  for (int d = 0; d < order; ++d) {
    for (uint64_t m = 0; m < nnz; ++m) ib[m] = xi[d][perm[m]];
    memcpy(xi[d], ib, nnz * sizeof(uint32_t));
  }
  float* vb = (float*)ib;
  for (uint64_t m = 0; m < nnz; ++m) vb[m] = xv[perm[m]];
  memcpy(xv, vb, nnz * sizeof(float));
  free(ib);
}

/* coalesce on a sorted tensor, P/src/tensor.cpp:66-90: runs of equal tuples
 * (under the sort order) become one entry whose value is the fp32 sum in
 * storage order. Returns the output count. */
uint64_t or_coalesce_sorted(uint64_t nnz, int order, const uint32_t* const* xi, const float* xv,
                            const uint32_t* mo, uint32_t** zi, float* zv) {
  uint64_t out = 0;
  for (uint64_t m = 0; m < nnz;) {
    uint64_t e = m + 1;
    float acc = xv[m];
    while (e < nnz && cmp_entries(order, xi, m, xi, e, mo) == 0) {
      acc += xv[e];
      ++e;
    }
    for (int d = 0; d < order; ++d) zi[d][out] = xi[d][m];
    zv[out] = acc;
    ++out;
    m = e;
  }
  return out;
}

/* build_fiber_index, P/src/tensor.cpp:92-120. fptr needs nnz+1 slots;
 * returns nfibs. */
uint64_t or_fiber_index(uint64_t nnz, int order, const uint32_t* const* xi, int mode,
                        uint64_t* fptr) {
  uint64_t nf = 0;
  for (uint64_t m = 0; m < nnz; ++m) {
    int boundary = m == 0;
    for (int d = 0; d < order && !boundary; ++d) {
      if (d == mode) continue;
      if (xi[d][m] != xi[d][m - 1]) boundary = 1;
    }
    if (boundary) fptr[nf++] = m;
  }
  fptr[nf] = nnz;
  return nf;
}

/* merge_range, P/src/kernel_detail.hpp:47-84, over whole inputs sorted under
 * mo. op: 0 add, 1 sub, 2 mul. Returns the output count; *flops receives the
 * reference's flop count. */
uint64_t or_tew_merge(int order, uint64_t nx, const uint32_t* const* xi, const float* xv,
                      uint64_t ny, const uint32_t* const* yi, const float* yv, const uint32_t* mo,
                      int op, uint32_t** zi, float* zv, uint64_t* flops) {
  uint64_t m1 = 0, m2 = 0, out = 0, fl = 0;
#define EMIT(SRC, IDX, VAL)                                      \
  do {                                                           \
    for (int d = 0; d < order; ++d) zi[d][out] = SRC[d][IDX];   \
    zv[out++] = (VAL);                                           \
  } while (0)
  while (m1 < nx && m2 < ny) {
    const int c = cmp_entries(order, xi, m1, yi, m2, mo);
    if (c == 0) {
      EMIT(xi, m1, elem(op, xv[m1], yv[m2]));
      ++fl;
      ++m1;
      ++m2;
    } else if (c < 0) {
      if (op != 2) EMIT(xi, m1, xv[m1]);
      ++m1;
    } else {
      if (op == 0) EMIT(yi, m2, yv[m2]);
      else if (op == 1) {
        EMIT(yi, m2, -yv[m2]);
        ++fl;
      }
      ++m2;
    }
  }
  if (op != 2) {
    for (; m1 < nx; ++m1) EMIT(xi, m1, xv[m1]);
    for (; m2 < ny; ++m2) {
      EMIT(yi, m2, op == 1 ? -yv[m2] : yv[m2]);
      if (op == 1) ++fl;
    }
  }
#undef EMIT
  *flops = fl;
  return out;
}

/* seq::ttv, P/src/kernels_seq.cpp:69-101 (ttv_fiber_value
 * P/src/kernel_detail.hpp:121-128): fp32 fiber sums in storage order from 0,
 * output indices = fiber head's non-mode indices. z64/zabs (optional): fp64
 * recomputation and fp64 sum of |terms| from the same inputs. */
void or_ttv(int order, uint64_t nnz, const uint32_t* const* xi, const float* xv, const float* v,
            int mode, const uint64_t* fptr, uint64_t nfibs, uint32_t** zi, float* zv, double* z64,
            double* zabs) {
  (void)nnz;
  for (uint64_t f = 0; f < nfibs; ++f) {
    const uint64_t b = fptr[f], e = fptr[f + 1];
    int dz = 0;
    for (int d = 0; d < order; ++d)
      if (d != mode) zi[dz++][f] = xi[d][b];
    float acc = 0.0f;
    double a64 = 0.0, ab = 0.0;
    for (uint64_t m = b; m < e; ++m) {
      const float t = xv[m] * v[xi[mode][m]];
      acc += t;
      const double t64 = (double)xv[m] * (double)v[xi[mode][m]];
      a64 += t64;
      ab += fabs(t64);
    }
    zv[f] = acc;
    if (z64) z64[f] = a64;
    if (zabs) zabs[f] = ab;
  }
}

/* seq::ttm, P/src/kernels_seq.cpp:108-146 (ttm_fiber
 * P/src/kernel_detail.hpp:130-140). u is rows x R row-major. */
void or_ttm(int order, uint64_t nnz, const uint32_t* const* xi, const float* xv, const float* u,
            uint64_t R, int mode, const uint64_t* fptr, uint64_t nfibs, uint32_t** zi, float* zv,
            double* z64, double* zabs) {
  (void)nnz;
  for (uint64_t f = 0; f < nfibs; ++f) {
    const uint64_t b = fptr[f], e = fptr[f + 1];
    const uint64_t base = f * R;
    for (int d = 0; d < order; ++d) {
      for (uint64_t r = 0; r < R; ++r) zi[d][base + r] = d == mode ? (uint32_t)r : xi[d][b];
    }
    for (uint64_t r = 0; r < R; ++r) {
      zv[base + r] = 0.0f;
      if (z64) z64[base + r] = 0.0;
      if (zabs) zabs[base + r] = 0.0;
    }
    for (uint64_t m = b; m < e; ++m) {
      const float val = xv[m];
      const float* urow = u + (uint64_t)xi[mode][m] * R;
      for (uint64_t r = 0; r < R; ++r) {
        zv[base + r] += val * urow[r];
        const double t = (double)val * (double)urow[r];
        if (z64) z64[base + r] += t;
        if (zabs) zabs[base + r] += fabs(t);
      }
    }
  }
}

/* seq::mttkrp, P/src/kernels_seq.cpp:153-174 (mttkrp_row
 * P/src/kernel_detail.hpp:176-188): row[r] = val; row[r] *= F_d[i_d][r] for
 * d != mode ascending; out[i_mode][r] += row[r] (fp32, entry order).
 * out64 (optional): the fp64 recomputation; outabs: fp64 sum of |terms|. */
void or_mttkrp(int order, uint64_t nnz, const uint32_t* const* xi, const float* xv,
               const float* const* fac, uint64_t R, int mode, uint64_t rows, float* out,
               double* out64, double* outabs) {
  memset(out, 0, rows * R * sizeof(float));
  if (out64) memset(out64, 0, rows * R * sizeof(double));
  if (outabs) memset(outabs, 0, rows * R * sizeof(double));
  float* row = (float*)malloc((R ? R : 1) * sizeof(float));
  for (uint64_t m = 0; m < nnz; ++m) {
    for (uint64_t r = 0; r < R; ++r) row[r] = xv[m];
    for (int d = 0; d < order; ++d) {
      if (d == mode) continue;
      const float* f = fac[d] + (uint64_t)xi[d][m] * R;
      for (uint64_t r = 0; r < R; ++r) row[r] *= f[r];
    }
    float* o = out + (uint64_t)xi[mode][m] * R;
    for (uint64_t r = 0; r < R; ++r) o[r] += row[r];
    if (out64 || outabs) {
      for (uint64_t r = 0; r < R; ++r) {
        double t = (double)xv[m];
        for (int d = 0; d < order; ++d)
          if (d != mode) t *= (double)fac[d][(uint64_t)xi[d][m] * R + r];
        if (out64) out64[(uint64_t)xi[mode][m] * R + r] += t;
        if (outabs) outabs[(uint64_t)xi[mode][m] * R + r] += fabs(t);
      }
    }
  }
  free(row);
}
