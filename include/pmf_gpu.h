/*
 * pmf_gpu.h -- C-ABI of the B200-native CCD++ / ALS matrix-factorisation library
 *              (paper_1511_02433_b200/libpmf_gpu.so, sm_100a).
 *
 * Drop-in boundary for the parmf reference (/root/reference/proj/include/parmf, cited below as
 * `<header>:<line>`).  Plain pointers and sizes only; FP32 model (Real = float).  Every entry point
 * is synchronous and returns a pmf_status; pmf_last_error() gives the thread-local message.
 * There is no CPU fallback: without a CUDA device every compute entry point returns
 * PMF_RUNTIME_ERROR.
 *
 * Index/offset types follow types.hpp:14-21 (int32 indices, int64 offsets).  Factor matrices
 * crossing this boundary are row-major (W m x k, H n x k) exactly like FactorModel
 * (model.hpp:21-31).
 */
#ifndef PMF_GPU_H
#define PMF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMF_ABI_VERSION 1

/* Exception classes of the reference mapped to codes (types.hpp:35-44, ccd.hpp:43-49,
 * als.hpp:34-39, sparse.hpp:82-92, dense.hpp:82-84 and :110-111). */
typedef enum pmf_status {
    PMF_OK = 0,
    PMF_INVALID_ARGUMENT = 1,       /* std::invalid_argument                              */
    PMF_DATA_ERROR = 2,             /* parmf::data_error                                  */
    PMF_RUNTIME_ERROR = 3,          /* CUDA / NCCL / out of memory / no device            */
    PMF_NOT_POSITIVE_DEFINITE = 4,  /* parmf::not_positive_definite                       */
    PMF_OUT_OF_RANGE = 5,           /* std::out_of_range                                  */
    PMF_DOMAIN_ERROR = 6            /* std::domain_error (singular triangular factor)     */
} pmf_status;

/* parmf::Triplet<float> (sparse.hpp:20-25): 12 bytes, layout-identical, so a probe
 * std::span<const Triplet<float>> passes zero-copy. */
typedef struct pmf_triplet {
    int32_t user;
    int32_t item;
    float rating;
} pmf_triplet;

/* Borrowed view of RatingsMatrix<float> (sparse.hpp:151-161 accessors).  The cross-links are not
 * needed: the device keeps two residual copies updated by identical arithmetic. */
typedef struct pmf_matrix_view {
    int32_t m; /* users (rows)  */
    int32_t n; /* items (cols)  */
    int64_t nnz;
    const int64_t* row_start; /* m+1 */
    const int32_t* col_of;    /* nnz, strictly increasing within a row    */
    const float* val_row;     /* nnz */
    const int64_t* col_start; /* n+1 */
    const int32_t* row_of;    /* nnz, strictly increasing within a column */
    const float* val_col;     /* nnz */
} pmf_matrix_view;

/* CcdConfig (ccd.hpp:33-50); `workers` becomes num_gpus (1 = this process's device; N > 1 = a
 * device group of N ranks, see pmf_ctx_create_group; must be >= 1 like workers, ccd.hpp:43-49). */
typedef struct pmf_ccd_config {
    int32_t k;
    float lambda;
    int32_t outer_iters;
    int32_t inner_iters;
    uint64_t seed;
    int32_t num_gpus;
    int32_t flags; /* reserved, 0 */
} pmf_ccd_config;

/* AlsConfig (als.hpp:26-40).  flags bit 0 (PMF_ALS_WEIGHTED_LAMBDA) selects lambda*n_i*I instead
 * of the reference's plain lambda*I; off by default, never used for parity. */
#define PMF_ALS_WEIGHTED_LAMBDA 1
typedef struct pmf_als_config {
    int32_t k;
    float lambda;
    int32_t outer_iters;
    uint64_t seed;
    int32_t num_gpus;
    int32_t flags;
} pmf_als_config;

/* IterationRow (report.hpp:25-30) + train RMSE.  `seconds` is device time of the solver
 * phases only (metrics excluded, ccd.hpp:390-396, als.hpp:218-225). */
typedef struct pmf_iter_row {
    int32_t iteration;
    double seconds;
    double objective;  /* model.hpp:119-144, FP64 accumulation          */
    double rmse;       /* model.hpp:156-167, NaN without a probe        */
    double train_rmse; /* sqrt(sum_Omega (A - w.h)^2 / nnz), FP64       */
} pmf_iter_row;

/* TrainReport totals (report.hpp:36-70). */
typedef struct pmf_train_totals {
    double train_seconds;   /* sum of rows[].seconds                                        */
    double wall_seconds;    /* whole call, host clock (uploads, layout build, metrics)      */
    double final_objective;
    double final_rmse;
    double setup_seconds;   /* upload + device layout build                                 */
    int64_t h2d_bytes;
    int64_t d2h_bytes;
    int64_t kernel_launches; /* kernels launched by the solver phases                      */
} pmf_train_totals;

/* ---- whole-call entry points (drop-in for ccdpp_train / als_train / rmse / objective) -------- */

/* ccd.hpp:349-404 ccdpp_train<float>.  W_out m*k, H_out n*k row-major; rows_out[outer_iters];
 * totals_out may be NULL.  probe may be NULL when n_probe == 0. */
pmf_status pmf_ccdpp_train(const pmf_ccd_config* config, const pmf_matrix_view* a,
                           const pmf_triplet* probe, int64_t n_probe, float* W_out, float* H_out,
                           pmf_iter_row* rows_out, pmf_train_totals* totals_out);

/* als.hpp:188-233 als_train<float>. */
/* ccd.hpp:310-344 ccd_train (CcdVariant::kCcd): same inputs / outputs as pmf_ccdpp_train. */
pmf_status pmf_ccd_train(const pmf_ccd_config* config, const pmf_matrix_view* a,
                         const pmf_triplet* probe, int64_t n_probe, float* W_out, float* H_out,
                         pmf_iter_row* rows_out, pmf_train_totals* totals_out);
pmf_status pmf_als_train(const pmf_als_config* config, const pmf_matrix_view* a,
                         const pmf_triplet* probe, int64_t n_probe, float* W_out, float* H_out,
                         pmf_iter_row* rows_out, pmf_train_totals* totals_out);

/* model.hpp:156-167 rmse (predict model.hpp:103-114 in FP32, sequential t; FP64 error sum). */
pmf_status pmf_rmse(const float* W, const float* H, int32_t m, int32_t n, int32_t k,
                    const pmf_triplet* probe, int64_t n_probe, double* out);

/* model.hpp:119-144 objective (FP64 dot and accumulation) + lambda(|W|^2+|H|^2). */
pmf_status pmf_objective(const pmf_matrix_view* a, const float* W, const float* H, int32_t k,
                         double lambda, double* out);

/* ---- resident context: the matrix stays in HBM across calls --------------------------------- */

typedef struct pmf_ctx pmf_ctx;

/* Uploads CSR+CSC and builds the device layouts on `device` (-1 = current). */
pmf_status pmf_ctx_create(const pmf_matrix_view* a, int32_t device, pmf_ctx** out);
/* The same straight from triplets (RatingsMatrix::from_triplets + the context, sparse.hpp:73-149):
 * the CSR / CSC are built on the device and stay there; only the offsets and per-(panel, output)
 * segment lengths come to the host, which builds the layouts' structure; the residual / index streams
 * are filled on the device.  Same validation errors as pmf_matrix_from_triplets; layouts bitwise those
 * of pmf_ctx_create on the same matrix.  One device (world 1). */
pmf_status pmf_ctx_create_from_triplets(const pmf_triplet* triplets, int64_t nnz, int32_t m, int32_t n,
                                        int32_t device, pmf_ctx** out);
pmf_status pmf_ctx_destroy(pmf_ctx* ctx);

/* CCD++: W = 0, H = init_random_items(seed) (model.hpp:86-93), R = A. */
pmf_status pmf_ctx_ccdpp_begin(pmf_ctx* ctx, const pmf_ccd_config* config);
/* Runs n_outer outer iterations (each: for t in 0..k-1 the rank-one step, ccd.hpp:373-393).
 * iter_seconds (may be NULL) receives the device time of each iteration. */
pmf_status pmf_ctx_ccdpp_iterate(pmf_ctx* ctx, int32_t n_outer, double* iter_seconds);

/* ALS: W = 0, H = init_random_items(seed). */
/* Item/user-wise CCD (ccd.hpp:52-125, ccd_train :310-344; inner_iters validated and ignored);
 * one device only.  ccd_iterate runs whole epochs (W sweep, then H sweep). */
pmf_status pmf_ctx_ccd_begin(pmf_ctx* ctx, const pmf_ccd_config* config);
pmf_status pmf_ctx_ccd_iterate(pmf_ctx* ctx, int32_t n_outer, double* iter_seconds);
pmf_status pmf_ctx_als_begin(pmf_ctx* ctx, const pmf_als_config* config);
pmf_status pmf_ctx_als_iterate(pmf_ctx* ctx, int32_t n_outer, double* iter_seconds);

/* Uploads a probe set kept on the device for pmf_ctx_metrics (n_probe == 0 clears it). */
pmf_status pmf_ctx_set_probe(pmf_ctx* ctx, const pmf_triplet* probe, int64_t n_probe);
/* objective / probe RMSE (NaN without probe) / train RMSE of the current model. */
pmf_status pmf_ctx_metrics(pmf_ctx* ctx, double* objective, double* rmse, double* train_rmse);
/* Current model, row-major W m*k and H n*k. */
pmf_status pmf_ctx_get_model(pmf_ctx* ctx, float* W, float* H);
/* Sets the model (row-major) -- used to start the stage-level tests from a given state. */
pmf_status pmf_ctx_set_model(pmf_ctx* ctx, const float* W, const float* H, int32_t k);
/* CCD++ residual R = A - W H^T in both reference layouts (CSR order, CSC order); applies the
 * deferred writeback first (ccd.hpp:199-218). */
pmf_status pmf_ctx_get_residual(pmf_ctx* ctx, float* r_row, float* r_col);
/* Device time (ms) of the last iterate call's dominant sweep kernel launches, for roofline
 * reporting: sums over launches of {u-sweep, v-sweep} and their counts. */
pmf_status pmf_ctx_kernel_stats(pmf_ctx* ctx, double* usweep_ms, int64_t* usweep_launches,
                                double* vsweep_ms, int64_t* vsweep_launches);
/* Kernels launched by one outer iteration of the active solver (CCD++ graph or ALS phases). */
pmf_status pmf_ctx_launch_count(pmf_ctx* ctx, int64_t* per_iteration);
/* Diagnostic: runs one sweep (side 0 = u over CSR, 1 = v over CSC; promote or plain) on a copy of the
 * residual and returns per-CTA [start, end] globaltimer ns (2*ctas) and per-CTA layout stats
 * (24*ctas: long/medium/short units, entries, pieces, last panel, entries per class, then for unroll
 * 1/2/4/8 the per-class sums of ceil(len / (4 * lanes * unroll)) group-steps; rest 0). */
pmf_status pmf_ctx_debug_sweep_profile(pmf_ctx* ctx, int32_t side, int32_t promote, uint64_t* cta_ns,
                                      int64_t* cta_stats, int32_t* n_ctas);
/* Diagnostic: the device layout of one side (0 = CSR / u-sweep, 1 = CSC / v-sweep). */
typedef struct pmf_layout_info {
    int32_t n_panels, panel_size;   /* gather panels staged in shared memory, and their width */
    int32_t smem, idx16;            /* 1: panel-staged gathers / 16-bit panel-local indices */
    int32_t promote_fused;          /* 1: promote fused into one sweep; 0: residual pass + sweep */
    int32_t rmw_sub, sub_width;     /* residual pass sub-panels (split promote) and their width */
    int32_t n_units, n_slots, ctas;
    int64_t n_entries, n_real;      /* padded / real entries */
} pmf_layout_info;
pmf_status pmf_ctx_layout_info(pmf_ctx* ctx, int32_t side, pmf_layout_info* out);
/* Enables (1) / disables (0) per-sweep CUDA-event timing inside pmf_ctx_ccdpp_iterate. */
pmf_status pmf_ctx_set_profiling(pmf_ctx* ctx, int32_t on);

/* ---- stage-level entry points (ccd.hpp:233-271, als.hpp:72-108, dense.hpp:55-131) ----------
 * Host buffers in reference layout order; the same device kernels as training run on them. */

/* ccdpp_build_rhat (ccd.hpp:235-240): R += u v^T over rows with u_i != 0, both layouts. */
pmf_status pmf_ccdpp_build_rhat(const pmf_matrix_view* a, float* r_row, float* r_col,
                                const float* u, const float* v);
/* ccdpp_update_u (ccd.hpp:243-248) on residual values rhat_row (CSR order). */
pmf_status pmf_ccdpp_update_u(const pmf_matrix_view* a, const float* rhat_row, float* u,
                              const float* v, float lambda);
/* ccdpp_update_v (ccd.hpp:251-256) on residual values rhat_col (CSC order). */
pmf_status pmf_ccdpp_update_v(const pmf_matrix_view* a, const float* rhat_col, const float* u,
                              float* v, float lambda);
/* residual part of ccdpp_writeback (ccd.hpp:260-271): R -= u v^T, both layouts. */
pmf_status pmf_ccdpp_writeback(const pmf_matrix_view* a, float* r_row, float* r_col,
                               const float* u, const float* v);
/* solve_user_row (side 0) / solve_item_row (side 1) for every row of that side
 * (als.hpp:72-108): opposing is row-major (n*k or m*k), out is row-major. */
pmf_status pmf_als_solve_rows(const pmf_matrix_view* a, int32_t side, const float* opposing,
                              int32_t k, float lambda, float* out);
/* cholesky_factor_inplace + cholesky_solve_inplace (dense.hpp:74-124) on `batch` row-major
 * k*k SPD matrices: a is overwritten by L (strict upper zeroed), x by the solution. */
pmf_status pmf_cholesky_solve_batched(int32_t batch, int32_t k, float* a, float* x);

/* ---- predict path: top_n (model.hpp:172-209) ------------------------------------------------
 * For each users[u]: the `count` best items of row users[u] of W H^T (row-major m x k / n x k) that
 * are not in ex_items[ex_start[u] .. ex_start[u+1]) (strictly increasing), by score descending, ties
 * by ascending item; scores are predict()'s FP32 sums (model.hpp:103-114), bitwise.  out_items /
 * out_scores are n_users x count (item -1 past out_count[u] = min(count, n - excluded)).
 * Errors as the reference: count < 1 -> INVALID_ARGUMENT, user outside [0, m) -> OUT_OF_RANGE. */
pmf_status pmf_top_n(const float* W, const float* H, int32_t m, int32_t n, int32_t k,
                     const int32_t* users, int32_t n_users, int32_t count, const int64_t* ex_start,
                     const int32_t* ex_items, int32_t* out_items, float* out_scores, int32_t* out_count);

/* ---- model files (model.hpp:211-295 save_model / load_model, the PMFB v1 format, float) ------
 * load_model with W = H = NULL reads the header only; errors map to PMF_DATA_ERROR (data_error). */
pmf_status pmf_save_model(const char* path, const float* W, const float* H, int64_t m, int64_t n, int64_t k);
pmf_status pmf_load_model(const char* path, int64_t* m, int64_t* n, int64_t* k, float* W, float* H);

/* io.hpp:240-285 split_dataset: to_probe[e] = 1 for the entries the reference moves to the probe set
 * (users[] = the external user id of every rating, file order). */
pmf_status pmf_split_mask(const int64_t* users, int64_t n, double ratio, uint64_t seed, uint8_t* to_probe,
                          int64_t* n_probe);

/* ---- host helpers --------------------------------------------------------------------------- */

/* runtime.hpp:91-136 partition_balanced (bounds has p+1 entries). */
pmf_status pmf_partition_balanced(const int64_t* costs, int32_t count, int32_t p,
                                  int32_t* bounds);
/* sparse.hpp:73-149 RatingsMatrix::from_triplets into caller arrays (canonical order, the same
 * range / finiteness / duplicate errors); multithreaded counting sort. */
pmf_status pmf_matrix_from_triplets(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n,
                                    int64_t* row_start, int32_t* col_of, float* val_row,
                                    int64_t* col_start, int32_t* row_of, float* val_col);
/* The same on the GPU (ingest.cu): staged upload, validation pass, stable radix sorts by (user, item)
 * and (item, user) keys, offsets + first-duplicate pass, staged download.  Bitwise the same output
 * and the same errors as pmf_matrix_from_triplets / the reference (nnz < 2^31). */
pmf_status pmf_matrix_from_triplets_gpu(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n,
                                        int64_t* row_start, int32_t* col_of, float* val_row,
                                        int64_t* col_start, int32_t* row_of, float* val_col);
const char* pmf_last_error(void);
int32_t pmf_abi_version(void);
int32_t pmf_device_count(void);
/* Device blocks and page-locked host layout blocks of destroyed contexts stay cached for the next
 * context (no cudaFree / re-pinning in a caller's timed region); this returns the idle ones to the
 * driver (no reference counterpart).  Bytes released in *released (may be null). */
pmf_status pmf_release_cached_memory(int64_t* released);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink / NVSwitch) -------------------------- */

/* Host-only: the plan pmf_ctx_create_dist uses -- rank r owns CSR rows [row_bounds[r], row_bounds[r+1])
 * and CSC columns [col_bounds[r], col_bounds[r+1]) (partition_balanced over 4|Omega|,
 * runtime.hpp:73-136); replicated u/v/W/H live in a padded index space where block r occupies
 * [r*B, (r+1)*B) with B = block_rows (users) or block_cols (items), so every NCCL all-gather uses
 * equal counts.  row_bounds / col_bounds have world+1 entries. */
pmf_status pmf_dist_plan(const pmf_matrix_view* a, int32_t world, int32_t* row_bounds, int32_t* col_bounds,
                         int32_t* block_rows, int32_t* block_cols);
/* 128-byte ncclUniqueId produced on rank 0 and broadcast by the caller (e.g. torch.distributed). */
pmf_status pmf_nccl_unique_id(uint8_t* out128);
/* Like pmf_ctx_create, but this rank owns the CSR row block and CSC column block chosen by
 * partition_balanced over 4|Omega| costs (runtime.hpp:73-136); u/v (CCD++) and W/H blocks (ALS)
 * are all-gathered over NCCL after every sweep / half-step. */
pmf_status pmf_ctx_create_dist(const pmf_matrix_view* a, int32_t device, int32_t rank,
                               int32_t world, const uint8_t* nccl_id128, pmf_ctx** out);
/* One process driving a device group of num_gpus ranks with the same row / column block plan: rank
 * r on devices[r] (NULL: device r mod pmf_device_count(), so ranks may share a device).  The
 * all-gathers are device-to-device copies between the ranks' replicated vectors, ordered by
 * events; a group whose ranks share one device runs each outer iteration as one CUDA graph.  The
 * returned handle drives every rank through the pmf_ctx_* calls (model / metrics as one context).
 * The whole-call entry points use this for config num_gpus > 1 (the reference's `workers`,
 * ccd.hpp:39, als.hpp:30). */
pmf_status pmf_ctx_create_group(const pmf_matrix_view* a, int32_t num_gpus, const int32_t* devices,
                                pmf_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* PMF_GPU_H */
