// ref_driver.cpp -- C-ABI shim around the UNMODIFIED parmf reference headers (TEST INFRASTRUCTURE).
//
// Built by oracle/Makefile from the reference sources where they lie
// (/root/reference/proj/include, /root/reference/proj/tests/testutil.hpp) into
// oracle/_ref/libparmf_ref.so; nothing from /root/reference is copied into this repo.
// Used (a) to pin the C restatement in pmf_oracle.c bit-for-bit, (b) to generate the golden
// fixtures in tests/golden/, and (c) as the CPU reference arm of bench.py (`--impl reference`
// and the `cpu_baseline` leg).  It is never linked into the product library.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <stdexcept>
#include <vector>

#include "parmf/parmf.hpp"
#include "testutil.hpp"

using namespace parmf;

namespace {

thread_local char g_err[512];

int status_of(const std::exception& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    if (dynamic_cast<const not_positive_definite*>(&e)) return 4;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 5;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const data_error*>(&e)) return 2;
    if (dynamic_cast<const std::domain_error*>(&e)) return 6;
    return 3;
}

#define GUARD(...)                                    \
    try {                                             \
        __VA_ARGS__;                                  \
        return 0;                                     \
    } catch (const std::exception& e) {               \
        return status_of(e);                          \
    }

template <class Real>
struct RefTriplet {
    int32_t user, item;
    Real rating;
};

template <class Real>
std::vector<Triplet<Real>> to_trips(const RefTriplet<Real>* t, int64_t n) {
    std::vector<Triplet<Real>> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = {t[i].user, t[i].item, t[i].rating};
    return v;
}

struct IterRow {
    int32_t iteration;
    double seconds, objective, rmse, train_rmse;
};

template <class Real>
double train_loss(const FactorModel<Real>& model, const RatingsMatrix<Real>& a) {
    // data term of objective (model.hpp:125-139), same order
    return objective(model, a, 0.0);
}

template <class Real>
void copy_model(const FactorModel<Real>& m, Real* W, Real* H) {
    std::copy(m.w().begin(), m.w().end(), W);
    std::copy(m.h().begin(), m.h().end(), H);
}

template <class Real>
struct MatrixHandle {
    RatingsMatrix<Real> a;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

#define REF_DEFS(SUF, Real)                                                                         \
    void* ref_matrix_create##SUF(const RefTriplet<Real>* t, int64_t nnz, int32_t m, int32_t n,      \
                                 int* status) {                                                    \
        try {                                                                                       \
            auto* h = new MatrixHandle<Real>{RatingsMatrix<Real>::from_triplets(to_trips(t, nnz),   \
                                                                                m, n)};            \
            *status = 0;                                                                            \
            return h;                                                                               \
        } catch (const std::exception& e) {                                                         \
            *status = status_of(e);                                                                 \
            return nullptr;                                                                         \
        }                                                                                           \
    }                                                                                               \
    void ref_matrix_destroy##SUF(void* h) { delete static_cast<MatrixHandle<Real>*>(h); }           \
    int ref_matrix_export##SUF(void* h, int64_t* row_start, int32_t* col_of, Real* val_row,         \
                               int64_t* col_start, int32_t* row_of, Real* val_col,                  \
                               int64_t* xlink) {                                                    \
        const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                     \
        std::ranges::copy(a.row_start(), row_start);                                               \
        std::ranges::copy(a.col_of(), col_of);                                                     \
        std::ranges::copy(a.val_row(), val_row);                                                   \
        std::ranges::copy(a.col_start(), col_start);                                               \
        std::ranges::copy(a.row_of(), row_of);                                                     \
        std::ranges::copy(a.val_col(), val_col);                                                   \
        if (xlink) std::ranges::copy(a.xlink(), xlink);                                            \
        return 0;                                                                                   \
    }                                                                                               \
    void ref_init_random_items##SUF(Real* H, int32_t n, int k, uint64_t seed) {                     \
        FactorModel<Real> model(1, n, k);                                                           \
        init_random_items(model, seed);                                                             \
        std::ranges::copy(model.h(), H);                                                           \
    }                                                                                               \
    int ref_objective##SUF(void* h, const Real* W, const Real* H, int k, double lambda,             \
                           double* out) {                                                           \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            FactorModel<Real> model(a.rows(), a.cols(), k);                                         \
            std::copy(W, W + model.w().size(), model.w().begin());                                  \
            std::copy(H, H + model.h().size(), model.h().begin());                                  \
            *out = objective(model, a, lambda);                                                     \
        })                                                                                          \
    }                                                                                               \
    /* model.hpp:172-198 top_n through the reference's own function; returns the kept count */    \
    int ref_top_n##SUF(const Real* W, const Real* H, int32_t m, int32_t n, int k, int32_t i,        \
                       int32_t count, const int32_t* rated, int64_t n_rated, int32_t* out_items,    \
                       Real* out_scores, int32_t* kept) {                                           \
        GUARD({                                                                                     \
            FactorModel<Real> model(m, n, k);                                                       \
            std::copy(W, W + model.w().size(), model.w().begin());                                  \
            std::copy(H, H + model.h().size(), model.h().begin());                                  \
            std::vector<index_t> r(rated, rated + n_rated);                                         \
            const auto best = top_n(model, i, count, std::span<const index_t>(r));                  \
            for (size_t x = 0; x < best.size(); ++x) {                                              \
                out_items[x] = best[x].first;                                                       \
                out_scores[x] = best[x].second;                                                     \
            }                                                                                       \
            *kept = static_cast<int32_t>(best.size());                                              \
        })                                                                                          \
    }                                                                                               \
    int ref_rmse##SUF(const Real* W, const Real* H, int32_t m, int32_t n, int k,                    \
                      const RefTriplet<Real>* probe, int64_t P, double* out) {                      \
        GUARD({                                                                                     \
            FactorModel<Real> model(m, n, k);                                                       \
            std::copy(W, W + model.w().size(), model.w().begin());                                  \
            std::copy(H, H + model.h().size(), model.h().begin());                                  \
            const auto pr = to_trips(probe, P);                                                     \
            *out = rmse(model, std::span<const Triplet<Real>>(pr));                                 \
        })                                                                                          \
    }                                                                                               \
    /* ccd.hpp:349 ccdpp_train through the reference's own entry point */                          \
    int ref_ccdpp_train##SUF(void* h, int k, Real lambda, int outer, int inner, int workers,        \
                             uint64_t seed, const RefTriplet<Real>* probe, int64_t P, Real* W,      \
                             Real* H, IterRow* rows, double* train_seconds) {                       \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            CcdConfig<Real> c;                                                                      \
            c.k = k; c.lambda = lambda; c.outer_iters = outer; c.inner_iters = inner;              \
            c.workers = workers; c.seed = seed;                                                     \
            const auto pr = to_trips(probe, P);                                                     \
            auto [model, rep] = ccdpp_train(c, a, std::span<const Triplet<Real>>(pr));              \
            copy_model(model, W, H);                                                                \
            for (size_t i = 0; i < rep.rows.size(); ++i)                                            \
                rows[i] = {rep.rows[i].iteration, rep.rows[i].seconds, rep.rows[i].objective,       \
                           rep.rows[i].rmse, NAN};                                                  \
            *train_seconds = rep.train_seconds;                                                     \
        })                                                                                          \
    }                                                                                               \
    /* ccd.hpp:310-344 item/user-wise ccd_train through the reference's own entry point */         \
    int ref_ccd_train##SUF(void* h, int k, Real lambda, int outer, uint64_t seed,                   \
                           const RefTriplet<Real>* probe, int64_t P, Real* W, Real* H,              \
                           IterRow* rows) {                                                         \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            CcdConfig<Real> c;                                                                      \
            c.k = k; c.lambda = lambda; c.outer_iters = outer; c.variant = CcdVariant::kCcd;       \
            c.seed = seed;                                                                          \
            const auto pr = to_trips(probe, P);                                                     \
            auto [model, rep] = ccd_train(c, a, std::span<const Triplet<Real>>(pr));                \
            copy_model(model, W, H);                                                                \
            for (size_t i = 0; i < rep.rows.size(); ++i)                                            \
                rows[i] = {rep.rows[i].iteration, rep.rows[i].seconds, rep.rows[i].objective,       \
                           rep.rows[i].rmse, NAN};                                                  \
        })                                                                                          \
    }                                                                                               \
    /* stage-API loop (tests/acceptance_test.cpp:150-171 pattern): same schedule as ccdpp_train, */ \
    /* plus per-iteration train RMSE and the final residual in both layouts */                     \
    int ref_ccdpp_stage_loop##SUF(void* h, int k, Real lambda, int outer, int inner, int workers,   \
                                  uint64_t seed, const RefTriplet<Real>* probe, int64_t P,          \
                                  Real* W, Real* H, Real* r_row, Real* r_col, IterRow* rows,        \
                                  Real* W_hist, Real* H_hist) {                                     \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            FactorModel<Real> model(a.rows(), a.cols(), k);                                         \
            init_random_items(model, seed);                                                         \
            auto r = residual_from(a);                                                              \
            WorkerPool pool(workers);                                                               \
            const auto prow = partition_balanced(row_costs(a), workers);                           \
            const auto pcol = partition_balanced(col_costs(a), workers);                           \
            std::vector<Real> u(a.rows()), v(a.cols());                                             \
            const auto pr = to_trips(probe, P);                                                     \
            for (int iter = 1; iter <= outer; ++iter) {                                             \
                double secs = 0.0;                                                                  \
                for (int t = 0; t < k; ++t) {                                                       \
                    for (index_t i = 0; i < a.rows(); ++i) u[i] = model.w_at(i, t);                \
                    for (index_t j = 0; j < a.cols(); ++j) v[j] = model.h_at(j, t);                \
                    secs += ccdpp_build_rhat(r, u, v, prow, pool).seconds;                          \
                    for (int s = 0; s < inner; ++s) {                                               \
                        secs += ccdpp_update_u<Real>(r, u, v, lambda, prow, pool).seconds;          \
                        secs += ccdpp_update_v<Real>(r, u, v, lambda, pcol, pool).seconds;          \
                    }                                                                               \
                    for (const auto& st : ccdpp_writeback(r, model, t, u, v, prow, pcol, pool))     \
                        secs += st.seconds;                                                         \
                }                                                                                   \
                IterRow row{iter, secs, objective(model, a, static_cast<double>(lambda)), NAN,      \
                            0.0};                                                                   \
                if (P > 0) row.rmse = rmse(model, std::span<const Triplet<Real>>(pr));              \
                row.train_rmse = a.nnz() ? std::sqrt(train_loss(model, a) /                         \
                                                     static_cast<double>(a.nnz()))                  \
                                         : 0.0;                                                     \
                rows[iter - 1] = row;                                                               \
                if (W_hist)                                                                         \
                    copy_model(model, W_hist + static_cast<size_t>(iter - 1) * a.rows() * k,        \
                               H_hist + static_cast<size_t>(iter - 1) * a.cols() * k);              \
            }                                                                                       \
            copy_model(model, W, H);                                                                \
            std::ranges::copy(r.val_row(), r_row);                                                 \
            std::ranges::copy(r.val_col(), r_col);                                                 \
        })                                                                                          \
    }                                                                                               \
    /* als.hpp:188 als_train through the reference's own entry point, with train RMSE added */     \
    int ref_als_train##SUF(void* h, int k, Real lambda, int outer, int workers, uint64_t seed,      \
                           const RefTriplet<Real>* probe, int64_t P, Real* W, Real* H,              \
                           IterRow* rows, double* train_seconds) {                                  \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            AlsConfig<Real> c;                                                                      \
            c.k = k; c.lambda = lambda; c.outer_iters = outer; c.workers = workers; c.seed = seed; \
            const auto pr = to_trips(probe, P);                                                     \
            auto [model, rep] = als_train(c, a, std::span<const Triplet<Real>>(pr));                \
            copy_model(model, W, H);                                                                \
            for (size_t i = 0; i < rep.rows.size(); ++i)                                            \
                rows[i] = {rep.rows[i].iteration, rep.rows[i].seconds, rep.rows[i].objective,       \
                           rep.rows[i].rmse, NAN};                                                  \
            *train_seconds = rep.train_seconds;                                                     \
        })                                                                                          \
    }                                                                                               \
    /* als epochs via als_epoch (als.hpp:176) with per-epoch train RMSE */                          \
    int ref_als_epochs##SUF(void* h, int k, Real lambda, int outer, int workers, uint64_t seed,     \
                            const RefTriplet<Real>* probe, int64_t P, Real* W, Real* H,             \
                            IterRow* rows, Real* W_hist, Real* H_hist) {                            \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            FactorModel<Real> model(a.rows(), a.cols(), k);                                         \
            init_random_items(model, seed);                                                         \
            AlsRuntime<Real> rt(a, workers, k);                                                     \
            const auto pr = to_trips(probe, P);                                                     \
            for (int iter = 1; iter <= outer; ++iter) {                                             \
                double secs = 0.0;                                                                  \
                for (const auto& st : als_epoch(model, a, lambda, rt)) secs += st.seconds;          \
                IterRow row{iter, secs, objective(model, a, static_cast<double>(lambda)), NAN,      \
                            0.0};                                                                   \
                if (P > 0) row.rmse = rmse(model, std::span<const Triplet<Real>>(pr));              \
                row.train_rmse = a.nnz() ? std::sqrt(train_loss(model, a) /                         \
                                                     static_cast<double>(a.nnz()))                  \
                                         : 0.0;                                                     \
                rows[iter - 1] = row;                                                               \
                if (W_hist)                                                                         \
                    copy_model(model, W_hist + static_cast<size_t>(iter - 1) * a.rows() * k,        \
                               H_hist + static_cast<size_t>(iter - 1) * a.cols() * k);              \
            }                                                                                       \
            copy_model(model, W, H);                                                                \
        })                                                                                          \
    }                                                                                               \
    /* single stages on caller-supplied residuals (ccd.hpp:235-271), 1 worker */                    \
    int ref_ccdpp_update_u##SUF(void* h, const Real* rhat_row, Real* u, const Real* v,              \
                                Real lambda) {                                                      \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            auto r = residual_from(a);                                                              \
            std::copy(rhat_row, rhat_row + a.nnz(), r.val_row().begin());                           \
            WorkerPool pool(1);                                                                     \
            const auto rows = partition_uniform(a.rows(), 1);                                       \
            std::span<Real> us(u, a.rows());                                                        \
            std::span<const Real> vs(v, a.cols());                                                  \
            ccdpp_update_u<Real>(r, us, vs, lambda, rows, pool);                                    \
        })                                                                                          \
    }                                                                                               \
    int ref_ccdpp_update_v##SUF(void* h, const Real* rhat_col, const Real* u, Real* v,              \
                                Real lambda) {                                                      \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            auto r = residual_from(a);                                                              \
            std::copy(rhat_col, rhat_col + a.nnz(), r.val_col().begin());                           \
            WorkerPool pool(1);                                                                     \
            const auto cols = partition_uniform(a.cols(), 1);                                       \
            std::span<const Real> us(u, a.rows());                                                  \
            std::span<Real> vs(v, a.cols());                                                        \
            ccdpp_update_v<Real>(r, us, vs, lambda, cols, pool);                                    \
        })                                                                                          \
    }                                                                                               \
    int ref_solve_rows##SUF(void* h, int side, const Real* opposing, int k, Real lambda,            \
                            Real* out) {                                                            \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            std::vector<Real> gram(static_cast<size_t>(k) * k);                                     \
            const index_t cnt = side == 0 ? a.rows() : a.cols();                                    \
            const size_t opp = static_cast<size_t>(side == 0 ? a.cols() : a.rows()) * k;           \
            std::span<const Real> o(opposing, opp);                                                 \
            for (index_t r = 0; r < cnt; ++r) {                                                     \
                std::span<Real> dst(out + static_cast<size_t>(r) * k, static_cast<size_t>(k));      \
                if (side == 0) solve_user_row<Real>(a, r, o, k, lambda, dst, gram);                 \
                else solve_item_row<Real>(a, r, o, k, lambda, dst, gram);                           \
            }                                                                                       \
        })                                                                                          \
    }                                                                                               \
    int ref_cholesky_factor##SUF(Real* a, int k) {                                                  \
        GUARD({ cholesky_factor_inplace<Real>(std::span<Real>(a, static_cast<size_t>(k) * k), k); })\
    }                                                                                               \
    int ref_cholesky_solve##SUF(const Real* l, Real* x, int k) {                                    \
        GUARD({                                                                                     \
            cholesky_solve_inplace<Real>(std::span<const Real>(l, static_cast<size_t>(k) * k),      \
                                         std::span<Real>(x, static_cast<size_t>(k)), k);            \
        })                                                                                          \
    }                                                                                               \
    /* bench reference arm: time `steps` CCD++ rank-one steps (build, inner x (u,v), writeback) */ \
    /* on the full matrix with `workers` threads, from a steady-state-like model (W != 0). */       \
    int ref_ccdpp_sample##SUF(void* h, int k, Real lambda, int inner, int workers, int steps,       \
                              uint64_t seed, double* seconds_per_step) {                            \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            FactorModel<Real> model(a.rows(), a.cols(), k);                                         \
            init_random_items(model, seed);                                                         \
            std::mt19937 gen(static_cast<uint32_t>(seed) + 17u);                                    \
            for (auto& x : model.w())                                                               \
                x = static_cast<Real>(testutil::uniform(gen, 0.05, 0.25));                          \
            auto r = residual_from(a);                                                              \
            WorkerPool pool(workers);                                                               \
            const auto prow = partition_balanced(row_costs(a), workers);                           \
            const auto pcol = partition_balanced(col_costs(a), workers);                           \
            std::vector<Real> u(a.rows()), v(a.cols());                                             \
            double secs = 0.0;                                                                      \
            for (int s = 0; s < steps; ++s) {                                                       \
                const int t = s % k;                                                                \
                for (index_t i = 0; i < a.rows(); ++i) u[i] = model.w_at(i, t);                    \
                for (index_t j = 0; j < a.cols(); ++j) v[j] = model.h_at(j, t);                    \
                secs += ccdpp_build_rhat(r, u, v, prow, pool).seconds;                              \
                for (int q = 0; q < inner; ++q) {                                                   \
                    secs += ccdpp_update_u<Real>(r, u, v, lambda, prow, pool).seconds;              \
                    secs += ccdpp_update_v<Real>(r, u, v, lambda, pcol, pool).seconds;              \
                }                                                                                   \
                for (const auto& st : ccdpp_writeback(r, model, t, u, v, prow, pcol, pool))         \
                    secs += st.seconds;                                                             \
            }                                                                                       \
            *seconds_per_step = secs / steps;                                                       \
        })                                                                                          \
    }                                                                                               \
    /* bench reference arm for ALS: time `epochs` full als_epoch calls (als.hpp:176) */             \
    int ref_als_sample##SUF(void* h, int k, Real lambda, int workers, int epochs, uint64_t seed,     \
                            double* seconds_per_epoch) {                                            \
        GUARD({                                                                                     \
            const auto& a = static_cast<MatrixHandle<Real>*>(h)->a;                                 \
            FactorModel<Real> model(a.rows(), a.cols(), k);                                         \
            init_random_items(model, seed);                                                         \
            AlsRuntime<Real> rt(a, workers, k);                                                     \
            double secs = 0.0;                                                                      \
            for (int e = 0; e < epochs; ++e)                                                        \
                for (const auto& st : als_epoch(model, a, lambda, rt)) secs += st.seconds;          \
            *seconds_per_epoch = secs / epochs;                                                     \
        })                                                                                          \
    }

REF_DEFS(_f32, float)
REF_DEFS(_f64, double)

// tests/testutil.hpp generators through the reference's own code
int64_t ref_synth_ratings(int32_t m, int32_t n, int rank, int64_t target, uint32_t seed,
                          RefTriplet<double>* out) {
    const auto v = testutil::synth_ratings<double>(m, n, rank, target, seed);
    for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].user, v[i].item, v[i].rating};
    return static_cast<int64_t>(v.size());
}

int64_t ref_random_triplets(int32_t m, int32_t n, int target, uint32_t seed, double lo, double hi,
                            RefTriplet<double>* out) {
    const auto v = testutil::random_triplets<double>(m, n, target, seed, lo, hi);
    for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].user, v[i].item, v[i].rating};
    return static_cast<int64_t>(v.size());
}

int64_t ref_planted_full(int32_t m, int32_t n, int k, double scale, uint32_t seed,
                         RefTriplet<double>* out) {
    const auto v = testutil::planted_full<double>(m, n, k, scale, seed);
    for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].user, v[i].item, v[i].rating};
    return static_cast<int64_t>(v.size());
}

void ref_carve_probe(RefTriplet<double>* data, int64_t count, int64_t probe_count, uint32_t seed) {
    std::vector<Triplet<double>> train(static_cast<size_t>(count)), probe;
    for (int64_t i = 0; i < count; ++i) train[i] = {data[i].user, data[i].item, data[i].rating};
    testutil::carve_probe(train, probe, static_cast<size_t>(probe_count), seed);
    size_t o = 0;
    for (const auto& t : train) data[o++] = {t.user, t.item, t.rating};
    for (const auto& t : probe) data[o++] = {t.user, t.item, t.rating};
}

int ref_partition_balanced(const int64_t* costs, int32_t count, int p, int32_t* bounds) {
    GUARD({
        const auto part = partition_balanced(std::span<const std::int64_t>(costs, count), p);
        for (int r = 0; r < p; ++r) bounds[r] = part.range(r).first;
        bounds[p] = part.count();
    })
}

// model.hpp:233-295 through the reference (float): files written by one side read by the other
int ref_save_model_f32(const char* path, const float* W, const float* H, int32_t m, int32_t n, int k) {
    GUARD({
        FactorModel<float> model(m, n, k);
        std::copy(W, W + model.w().size(), model.w().begin());
        std::copy(H, H + model.h().size(), model.h().begin());
        save_model(path, model);
    })
}
int ref_load_model_f32(const char* path, int64_t* mnk, float* W, float* H) {
    GUARD({
        const auto model = load_model<float>(path);
        mnk[0] = model.users();
        mnk[1] = model.items();
        mnk[2] = model.rank();
        if (W) std::ranges::copy(model.w(), W);
        if (H) std::ranges::copy(model.h(), H);
    })
}

// io.hpp:240-285 split_dataset through the reference: the probe rows, in file order
int ref_split(const int64_t* users, const int64_t* items, const double* ratings, int64_t n, double ratio,
              uint64_t seed, int64_t* probe_users, int64_t* probe_items, double* probe_ratings, int64_t* n_probe) {
    GUARD({
        std::vector<RawTriplet> all(static_cast<size_t>(n));
        for (int64_t e = 0; e < n; ++e) all[static_cast<size_t>(e)] = {users[e], items[e], ratings[e]};
        const auto sp = split_dataset(all, ratio, seed);
        for (size_t x = 0; x < sp.probe.size(); ++x) {
            probe_users[x] = sp.probe[x].user;
            probe_items[x] = sp.probe[x].item;
            probe_ratings[x] = sp.probe[x].rating;
        }
        *n_probe = static_cast<int64_t>(sp.probe.size());
    })
}

}  // extern "C"
