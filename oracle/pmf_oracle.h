/*
 * pmf_oracle.h -- CPU restatement of the parmf reference algorithms (TEST INFRASTRUCTURE).
 *
 * This library is the parity CHECKER for the B200 path, never the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * Every function follows the reference file:line named in its comment
 * (paths relative to /root/reference/proj/include/parmf/ unless they start with tests/).
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit against
 *   (1) the golden vectors frozen in the reference's own tests
 *       (tests/oracle/gen_fixture_values.py, tests/ccd_test.cpp:253-280,
 *        tests/model_test.cpp:91-102, tests/dense_test.cpp:83-170, tests/als_test.cpp:14-135), and
 *   (2) the reference itself compiled here from its own headers (oracle/_ref/libparmf_ref.so,
 *       built by oracle/Makefile from /root/reference/proj/include) on seeded inputs.
 *
 * Every symbol exists twice: suffix _f32 (Real = float) and _f64 (Real = double), like the
 * reference's templates.  All arithmetic is compiled with -ffp-contract=off so products are
 * rounded before they are added, exactly as the reference's Release build (no -march, no FMA).
 */
#ifndef PMF_ORACLE_H
#define PMF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes mirror pmf_status in include/pmf_gpu.h */
enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_DATA_ERROR = 2, ORC_NOT_POSITIVE_DEFINITE = 4,
       ORC_OUT_OF_RANGE = 5, ORC_DOMAIN_ERROR = 6 };

typedef struct { int32_t user, item; float rating; } orc_triplet_f32;   /* sparse.hpp:20-25 */
typedef struct { int32_t user, item; double rating; } orc_triplet_f64;

typedef struct {
    int32_t iteration;
    double seconds;
    double objective;
    double rmse;        /* NaN without a probe */
    double train_rmse;  /* sqrt(sum_Omega (A - w.h)^2 / N), same accumulation as objective */
} orc_iter_row;

#define ORC_DECL(SUF, REAL)                                                                        \
    void orc_init_random_items##SUF(REAL* H, int64_t n, int k, uint64_t seed);                    \
    int orc_from_triplets##SUF(const orc_triplet##SUF* t, int64_t nnz, int32_t m, int32_t n,       \
                               int64_t* row_start, int32_t* col_of, REAL* val_row,                \
                               int64_t* col_start, int32_t* row_of, REAL* val_col,                \
                               int64_t* row_to_col);                                              \
    REAL orc_predict##SUF(const REAL* W, const REAL* H, int k, int32_t i, int32_t j);             \
    int orc_top_n##SUF(const REAL* W, const REAL* H, int32_t m, int32_t n, int k, int32_t i,      \
                       int32_t count, const int32_t* rated_sorted, int64_t n_rated,               \
                       int32_t* out_items, REAL* out_scores);                                     \
    double orc_objective##SUF(int32_t m, int32_t n, int k, const int64_t* row_start,              \
                              const int32_t* col_of, const REAL* val_row, const REAL* W,          \
                              const REAL* H, double lambda, double* loss_out);                    \
    int orc_rmse##SUF(const REAL* W, const REAL* H, int k, const orc_triplet##SUF* probe,         \
                      int64_t P, double* out);                                                    \
    void orc_ccdpp_build_rhat##SUF(int32_t m, const int64_t* row_start, const int32_t* col_of,    \
                                   const int64_t* row_to_col, REAL* r_row, REAL* r_col,           \
                                   const REAL* u, const REAL* v);                                 \
    void orc_ccdpp_update_u##SUF(int32_t m, const int64_t* row_start, const int32_t* col_of,      \
                                 const REAL* rhat_row, REAL* u, const REAL* v, REAL lambda);      \
    void orc_ccdpp_update_v##SUF(int32_t n, const int64_t* col_start, const int32_t* row_of,      \
                                 const REAL* rhat_col, const REAL* u, REAL* v, REAL lambda);      \
    void orc_ccdpp_writeback##SUF(int32_t m, int32_t n, int k, int t, const int64_t* row_start,   \
                                  const int32_t* col_of, const int64_t* row_to_col, REAL* r_row,  \
                                  REAL* r_col, REAL* W, REAL* H, const REAL* u, const REAL* v);   \
    int orc_ccd_train##SUF(int k, REAL lambda, int outer, uint64_t seed, int32_t m, int32_t n,     \
                           const int64_t* row_start, const int32_t* col_of, const REAL* val_row,  \
                           const int64_t* col_start, const int32_t* row_of, const REAL* val_col,  \
                           const int64_t* row_to_col, const orc_triplet##SUF* probe, int64_t P,   \
                           REAL* W, REAL* H, orc_iter_row* rows);                                 \
    int orc_ccdpp_train##SUF(int k, REAL lambda, int outer, int inner, uint64_t seed, int32_t m,  \
                             int32_t n, const int64_t* row_start, const int32_t* col_of,          \
                             const REAL* val_row, const int64_t* col_start,                       \
                             const int32_t* row_of, const REAL* val_col,                          \
                             const int64_t* row_to_col, const orc_triplet##SUF* probe, int64_t P, \
                             REAL* W, REAL* H, REAL* r_row, REAL* r_col, orc_iter_row* rows);     \
    void orc_gram_add_row_upper##SUF(REAL* gram, const REAL* h, int k);                           \
    void orc_gram_finish##SUF(REAL* gram, REAL lambda, int k);                                    \
    int orc_cholesky_factor##SUF(REAL* a, int k);                                                 \
    int orc_cholesky_solve##SUF(const REAL* l, REAL* x, int k);                                   \
    int orc_solve_row##SUF(const int64_t* start, const int32_t* idx, const REAL* vals,            \
                           int32_t row, const REAL* opposing, int k, REAL lambda, REAL* out,      \
                           REAL* gram);                                                           \
    int orc_als_half##SUF(int32_t count, const int64_t* start, const int32_t* idx,                \
                          const REAL* vals, const REAL* opposing, int k, REAL lambda, REAL* out); \
    int orc_als_train##SUF(int k, REAL lambda, int outer, uint64_t seed, int32_t m, int32_t n,    \
                           const int64_t* row_start, const int32_t* col_of, const REAL* val_row,  \
                           const int64_t* col_start, const int32_t* row_of, const REAL* val_col,  \
                           const orc_triplet##SUF* probe, int64_t P, REAL* W, REAL* H,            \
                           orc_iter_row* rows);

ORC_DECL(_f32, float)
ORC_DECL(_f64, double)
#undef ORC_DECL

/* tests/testutil.hpp generators (double ratings, as the reference fixtures use) */
int64_t orc_random_triplets(int32_t m, int32_t n, int32_t target, uint32_t seed, double lo,
                            double hi, orc_triplet_f64* out);
int64_t orc_planted_full(int32_t m, int32_t n, int k, double scale, uint32_t seed,
                         orc_triplet_f64* out);
int64_t orc_synth_ratings(int32_t m, int32_t n, int true_rank, int64_t target_nnz, uint32_t seed,
                          orc_triplet_f64* out);
void orc_carve_probe(orc_triplet_f64* train, int64_t count, int64_t probe_count, uint32_t seed);
int orc_partition_balanced(const int64_t* costs, int32_t count, int p, int32_t* bounds);
uint32_t orc_mt19937_first(uint32_t seed, int skip);

#ifdef __cplusplus
}
#endif
#endif
