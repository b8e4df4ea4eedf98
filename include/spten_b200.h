/*
 * spten_b200.h — C-ABI of the B200-native COO sparse-tensor kernels.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `spten` (PASTA, arXiv 1902.03317; reference at /root/reference/proj, "P/").
 * Every entry point below replaces one reference entry point, cited per
 * function. The C++ layer `include/spten/gpu.hpp` (namespace spten::gpu) puts
 * the reference's own signatures and types (SparseTensorCOO<float>,
 * DenseVector<float>, DenseMatrix<float>, FiberIndex) on top of this ABI; any
 * other FFI (ctypes, cffi, JNI, cgo) can bind these symbols directly.
 *
 * Conventions
 *  - Plain C: no CUDA or torch types. Streams are passed as `void*`
 *    (a cudaStream_t; NULL = legacy default stream).
 *  - Every function returns an spt_status; on failure spt_last_error()
 *    returns a thread-local message. Status codes map onto the reference's
 *    exception types (P/src/kernel_detail.hpp:38-44, P/src/kernels_seq.cpp:32-34).
 *  - Tensors are device-resident structure-of-arrays COO (spt_coo): one u32
 *    index array per mode + one f32 value array, all of length nnz, all device
 *    pointers. The layout is exactly the reference's SparseTensorCOO<float>
 *    (P/include/spten/tensor.hpp:22-57) with each std::vector replaced by a
 *    device pointer. 16-byte-aligned arrays take the vectorised paths.
 *  - Outputs are written into caller-provided device buffers. Sizes are known
 *    up front except for tew (merge) and coalesce/fiber_index, which take a
 *    capacity and return the produced count.
 *  - nnz must be < 2^32 (device offsets are u32); larger inputs get
 *    SPT_EOVERFLOW. Shard them (see paper_1902_03317_b200/parallel.py).
 *  - No CPU fallback exists anywhere behind this ABI.
 */
#ifndef SPTEN_B200_H
#define SPTEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SPT_API __attribute__((visibility("default")))
#else
#define SPT_API
#endif

#define SPT_MAX_ORDER 8
#define SPT_ABI_VERSION 1

/* Status codes. Reference exception each maps to (C++ layer rethrows it). */
typedef enum spt_status {
  SPT_OK = 0,
  SPT_EINVAL = 1,    /* std::invalid_argument (P/src/kernel_detail.hpp:38-44,110-118,158-172) */
  SPT_EDOMAIN = 2,   /* std::domain_error: tew_eq div by stored zero (P/src/kernels_seq.cpp:32-34) */
  SPT_EOVERFLOW = 3, /* std::overflow_error (index space / nnz beyond u32 offsets) */
  SPT_ENOMEM = 4,    /* std::bad_alloc (device allocation failed) */
  SPT_ERUNTIME = 5   /* std::runtime_error (CUDA error) */
} spt_status;

/* Same enumerator order as spten::ElemOp / ScalarOp / MttkrpStrategy
 * (P/include/spten/ops.hpp:5-7). */
typedef enum spt_elem_op { SPT_ADD = 0, SPT_SUB = 1, SPT_MUL = 2, SPT_DIV = 3 } spt_elem_op;
typedef enum spt_scalar_op { SPT_SCALAR_ADD = 0, SPT_SCALAR_MUL = 1 } spt_scalar_op;
typedef enum spt_mttkrp_strategy {
  SPT_MTTKRP_AUTO = -1,     /* segmented if sort_order[0]==mode, else a temporary plan
                               (R % 16 == 0) or a mode-leading sorted copy: always
                               deterministic, fp64 accumulation (the 1e-5 contract) */
  SPT_MTTKRP_SEGMENTED = 0, /* mode-sorted input; one writer per output row; deterministic;
                               launch shape (one wave / warp tiles / CTA tiles) picked by size */
  SPT_MTTKRP_ATOMIC = 1,    /* any order; vector red.global.add into a zeroed output
                               (fp32 sums in arrival order: the 1e-4 class, only on request) */
  SPT_MTTKRP_SEGMENTED_CTA = 2,  /* segmented, forced 2048-entry CTA tiles */
  SPT_MTTKRP_SEGMENTED_WARP = 3  /* segmented, forced 256-entry warp tiles */
} spt_mttkrp_strategy;

/* Device-resident COO tensor descriptor (mirror of SparseTensorCOO<float>,
 * P/include/spten/tensor.hpp:22-28). */
typedef struct spt_coo {
  uint32_t order;                    /* N, 1..SPT_MAX_ORDER */
  uint32_t _pad0;
  uint64_t nnz;                      /* entries */
  uint32_t dims[SPT_MAX_ORDER];      /* extents */
  uint32_t* idx[SPT_MAX_ORDER];      /* device: idx[d][m] = mode-d index of entry m */
  float* val;                        /* device: values[m] */
  int32_t sort_order[SPT_MAX_ORDER]; /* valid iff has_sort_order; sort_order[0] slowest key */
  int32_t has_sort_order;            /* std::optional<std::vector<unsigned>> engaged */
  int32_t coalesced;                 /* bool coalesced */
} spt_coo;

/* Opaque per-(device, stream-owner) context: scratch, error words,
 * look-back state. Not thread-safe: use one context per host thread/stream. */
typedef struct spt_ctx spt_ctx;

/* ---- library ------------------------------------------------------------- */
SPT_API int spt_abi_version(void);
SPT_API const char* spt_last_error(void);
/* Create a context on `device` (cudaSetDevice is called). */
SPT_API int spt_ctx_create(int device, spt_ctx** out);
SPT_API void spt_ctx_destroy(spt_ctx* ctx);
/* Hand back the context's cached device memory (sort scratch, look-back
 * state, the L2 flush buffer, its private pool of temporaries); they grow
 * again on demand. Synchronises the device. */
SPT_API int spt_ctx_trim(spt_ctx* ctx);
/* Number of kernels this context launched so far (evidence counter). */
SPT_API uint64_t spt_ctx_launches(const spt_ctx* ctx);
/* Deferred error check for calls made with SPT_FLAG_ASYNC: synchronises the
 * stream, decodes the sticky device error words, resets them. */
SPT_API int spt_ctx_check(spt_ctx* ctx, void* stream);

/* Flags accepted by the kernels' `flags` argument. */
#define SPT_FLAG_ASYNC 1u /* do not synchronise; data-dependent errors deferred to spt_ctx_check */

/* ---- TS: tensor-scalar ---------------------------------------------------
 * Replaces seq::ts / par::ts (P/include/spten/kernels_seq.hpp:33-34,
 * P/include/spten/kernels_par.hpp:50-51; body P/src/kernels_seq.cpp:55-67,
 * P/src/kernels_par.cpp:69-91). z gets x's indices (copied), values x+s or
 * x*s, x's dims/sort_order/coalesced. z->idx/z->val must hold x->nnz. */
SPT_API int spt_ts_f32(spt_ctx* ctx, const spt_coo* x, float s, int op, spt_coo* z, unsigned flags,
               void* stream);

/* ---- TEW-eq: elementwise op on identical patterns -------------------------
 * Replaces seq::tew_eq / par::tew_eq (P/include/spten/kernels_seq.hpp:18-20,
 * kernels_par.hpp:35-37; P/src/kernels_seq.cpp:11-39). Error precedence as
 * seq: the first failing entry decides; a pattern mismatch at entry m is
 * SPT_EINVAL, a stored zero divisor at entry m (pattern equal) SPT_EDOMAIN. */
SPT_API int spt_tew_eq_f32(spt_ctx* ctx, const spt_coo* x, const spt_coo* y, int op, spt_coo* z,
                   unsigned flags, void* stream);

/* ---- TEW: elementwise op via sorted merge ----------------------------------
 * Replaces the merge of seq::tew / par::tew (P/src/kernels_seq.cpp:41-53,
 * P/src/kernel_detail.hpp:50-84, P/src/kernels_par.cpp:144-177). x and y must
 * be coalesced and share a sort order (the host layer performs
 * unify_tew_sort, P/src/kernel_detail.hpp:88-95, with spt_sort_f32).
 * z buffers need capacity >= nnz_x+nnz_y (add/sub) or min(nnz) (mul);
 * the produced count is written to *h_nnz (host, synchronises) and/or
 * *d_nnz (device u64, stays async). z dims = per-mode max. */
SPT_API int spt_tew_f32(spt_ctx* ctx, const spt_coo* x, const spt_coo* y, int op, spt_coo* z,
                uint64_t z_capacity, uint64_t* h_nnz, uint64_t* d_nnz, unsigned flags,
                void* stream);

/* ---- preprocessing ---------------------------------------------------------
 * spt_sort_f32 replaces sort_lexicographic (P/include/spten/tensor.hpp:151-154,
 * P/src/tensor.cpp:54-64): in-place *stable* lexicographic sort of all entries
 * under mode_order (first = slowest key); sets x->sort_order. */
SPT_API int spt_sort_f32(spt_ctx* ctx, spt_coo* x, const uint32_t* mode_order, unsigned flags,
                 void* stream);
/* Replaces coalesce (P/src/tensor.cpp:66-90) for an already-sorted x: equal
 * tuples are summed in storage order (explicit zeros kept). z capacity >=
 * x->nnz; count to *h_nnz and/or *d_nnz. */
SPT_API int spt_coalesce_f32(spt_ctx* ctx, const spt_coo* x, spt_coo* z, uint64_t* h_nnz,
                     uint64_t* d_nnz, unsigned flags, void* stream);
/* Replaces build_fiber_index (P/src/tensor.cpp:92-120): d_fptr receives the
 * nfibs+1 u32 offsets (capacity >= nnz+1); nfibs to *h_nfibs and/or *d_nfibs. */
SPT_API int spt_fiber_index(spt_ctx* ctx, const spt_coo* x, uint32_t mode, uint32_t* d_fptr,
                    uint64_t* h_nfibs, uint64_t* d_nfibs, unsigned flags, void* stream);

/* ---- TTV ------------------------------------------------------------------
 * Replaces seq::ttv / par::ttv with a FiberIndex (P/include/spten/kernels_seq.hpp:39-41,
 * kernels_par.hpp:53-55;
 * P/src/kernels_seq.cpp:69-101, P/src/kernel_detail.hpp:106-128). z is order N-1
 * with nfibs entries (buffers sized by the caller); values are fp32 fiber sums
 * (tolerance class), indices bit-exact. */
SPT_API int spt_ttv_f32(spt_ctx* ctx, const spt_coo* x, const float* d_v, uint64_t v_len, uint32_t mode,
                const uint32_t* d_fptr, uint64_t nfibs, spt_coo* z, unsigned flags,
                void* stream);

/* ---- TTM ------------------------------------------------------------------
 * Replaces seq::ttm / par::ttm (P/include/spten/kernels_seq.hpp:47-49,
 * kernels_par.hpp:60-62;
 * P/src/kernels_seq.cpp:108-151, P/src/kernel_detail.hpp:132-140). u is
 * u_rows x R row-major (device); z has nfibs*R entries laid out f*R+r. */
SPT_API int spt_ttm_f32(spt_ctx* ctx, const spt_coo* x, const float* d_u, uint64_t u_rows,
                uint64_t u_cols, uint32_t mode, const uint32_t* d_fptr, uint64_t nfibs,
                spt_coo* z, unsigned flags, void* stream);

/* ---- MTTKRP ---------------------------------------------------------------
 * Replaces seq::mttkrp / par::mttkrp (P/include/spten/kernels_seq.hpp:59-61,
 * kernels_par.hpp:70-72; P/src/kernels_seq.cpp:153-174,
 * P/src/kernels_par.cpp:275-337, P/src/kernel_detail.hpp:153-188).
 * d_factors[d] (device, row-major rows[d] x cols[d]) for every mode d; entry
 * `mode` is ignored (may be NULL). d_out is dims[mode] x R row-major, fully
 * written (no pre-zeroing needed). Per-term products are formed in fp32 in
 * the reference's order (val * F_d0 * F_d1 ..., d ascending); accumulation is
 * fp64, rounded once per output element. */
SPT_API int spt_mttkrp_f32(spt_ctx* ctx, const spt_coo* x, const float* const* d_factors,
                   const uint64_t* rows, const uint64_t* cols, uint32_t mode, float* d_out,
                   int strategy, unsigned flags, void* stream);

/* ---- MTTKRP plans -----------------------------------------------------------
 * The preprocessing half of seq::mttkrp / par::mttkrp (same contract as
 * spt_mttkrp_f32, P/include/spten/kernels_seq.hpp:59-61): a copy of x sorted
 * with `mode` leading and the other modes by decreasing extent, whose most
 * gathered factor rows are served from shared memory. Built once (timed as
 * preprocessing, like the reference's sort_s, P/src/bench.cpp:363-368) and
 * executed any number of times with fresh factor values. Requires R % 16 == 0
 * and order 2..4 (otherwise SPT_EINVAL: use spt_mttkrp_f32). The plan holds its
 * own copy of x (indices and values): rebuild it if x changes. One stream at a
 * time per plan. */
typedef struct spt_mttkrp_plan spt_mttkrp_plan;
#define SPT_PLAN_NO_HOT 2u /* no shared-memory hot rows even when SPT_PLAN_HOT_MAX asks for them */
SPT_API int spt_mttkrp_plan_create(spt_ctx* ctx, const spt_coo* x, uint32_t mode, uint64_t R,
                                   unsigned flags, spt_mttkrp_plan** out, void* stream);
/* out = dims[mode] x R row-major (16-byte aligned), fully written. Factors as
 * for spt_mttkrp_f32 (16-byte aligned, cols == the plan's R). */
SPT_API int spt_mttkrp_plan_exec(spt_ctx* ctx, const spt_mttkrp_plan* plan,
                                 const float* const* d_factors, const uint64_t* rows,
                                 const uint64_t* cols, float* d_out, unsigned flags, void* stream);
/* Level order (tensor mode per level, outermost first; order-1 entries) and
 * rows per level served from shared memory. Any pointer may be NULL. */
SPT_API int spt_mttkrp_plan_info(const spt_mttkrp_plan* plan, uint32_t* level_modes,
                                 uint32_t* hot_per_level, uint32_t* nhot);
/* Waits for the stream that used the plan last (create or exec) and releases
 * its arrays to the context's stream-ordered pool on that stream -- no
 * device-wide synchronisation, so copies and kernels on other streams keep
 * running. A plan executed on several streams must be idle on all but the last
 * of them when it is destroyed; the context must outlive its plans. */
SPT_API void spt_mttkrp_plan_destroy(spt_mttkrp_plan* plan);

/* ---- multi-GPU MTTKRP (one process, one context per device) ---------------
 * SURVEY.md 8(e); the reference's analogue is the private-buffer reduction of
 * par::mttkrp (P/src/kernels_par.cpp:290-319). spt_row_aligned_cuts splits x
 * (sorted with `mode` leading) into `parts` entry ranges cut at row starts
 * (entry_cuts, parts+1 host u64) and the output row block each owns (row_lo,
 * parts+1 host u32: [row_lo[k], row_lo[k+1]), covering [0, dims[mode])). */
SPT_API int spt_row_aligned_cuts(spt_ctx* ctx, const spt_coo* x, uint32_t mode, uint32_t parts,
                                 uint64_t* entry_cuts, uint32_t* row_lo, void* stream);
/* Device k (ctxs[k], one per distinct device) holds shards[k] -- entries
 * [entry_cuts[k], entry_cuts[k+1]) of that sorted x -- and its factors
 * d_factors[k*order + d]; it computes its rows exactly into its own full
 * dims[mode] x R buffer d_out[k], then one NCCL group of in-place broadcasts
 * (root k: rows [row_lo[k], row_lo[k+1])) leaves the whole result in every
 * d_out[k]: (G-1)/G of the output per device, no cross-device sums. NCCL is
 * loaded on first use; ndev == 1 needs none. Synchronises every stream. */
SPT_API int spt_mttkrp_f32_multi(int ndev, spt_ctx* const* ctxs, const spt_coo* shards,
                                 const uint32_t* row_lo, const float* const* d_factors,
                                 const uint64_t* rows, const uint64_t* cols, uint32_t mode,
                                 float* const* d_out, void* const* streams);

/* ---- .tns text ingest on the device ----------------------------------------
 * Replaces spten::read_tns<float>(path, dims) (P/include/spten/io.hpp:22-23,
 * P/src/io.cpp:42-120) for text already in device memory (the caller reads
 * the file and copies its bytes up). spt_tns_scan splits lines, classifies
 * them and ranks the entry lines: it returns the order (from the first entry
 * line, or n_override when dims_override is given) and nnz so the caller can
 * size the output; spt_tns_parse fills z->idx[0..order) and z->val (device,
 * nnz each, in file order) and sets order, nnz, dims (per-mode max + 1, or the
 * override), has_sort_order = coalesced = 0. d_text must stay valid until
 * spt_tns_destroy. Parse errors return SPT_ERUNTIME with the reference's
 * message and *err_line = the failing 1-based line (the reference's
 * "path:line: msg"; prepend the path); an empty override is SPT_EINVAL.
 * Orders above SPT_MAX_ORDER and files of 2^32 lines or more are
 * SPT_EOVERFLOW. */
typedef struct spt_tns spt_tns;
SPT_API int spt_tns_scan(spt_ctx* ctx, const char* d_text, uint64_t bytes,
                         const uint32_t* dims_override, uint32_t n_override, spt_tns** out,
                         uint32_t* order, uint64_t* nnz, uint64_t* err_line, void* stream);
SPT_API int spt_tns_parse(spt_ctx* ctx, const spt_tns* scan, spt_coo* z, uint64_t* err_line,
                          void* stream);
SPT_API void spt_tns_destroy(spt_tns* scan);

/* ---- seeded synthetic generator (bench / test input, not a reference path) --
 * Draws `nnz` distinct tuples: per-mode index distribution `dist[d]`
 * (0 = uniform, s>0 = Zipf(s) over a seeded permutation of ids), duplicates
 * rejected in draw order (equivalent to sequential rejection sampling), then
 * values U[lo,hi). Result in draw order (unsorted) unless sort_order given. */
SPT_API int spt_gen_coo_f32(spt_ctx* ctx, spt_coo* x, uint64_t seed, const double* zipf_s, float lo,
                    float hi, const uint32_t* sort_order, void* stream);
/* Fill d_out[0..n) with U[lo,hi) floats from (seed, stream_id). */
SPT_API int spt_gen_uniform_f32(spt_ctx* ctx, float* d_out, uint64_t n, uint64_t seed,
                        uint64_t stream_id, float lo, float hi, void* stream);

/* Write >L2-sized garbage to flush the 126 MB L2 between timed repetitions. */
SPT_API int spt_l2_flush(spt_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPTEN_B200_H */
