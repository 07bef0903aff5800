// pmfgpu.hpp -- header-only C++ adapter from the parmf reference API to the B200 C-ABI (pmf_gpu.h).
//
// Include AFTER "parmf/parmf.hpp".  Signatures mirror the reference drivers so a parmf caller
// switches backends by changing the namespace:
//
//   parmf::ccdpp_train(config, a, probe)   (ccd.hpp:349)  ->  pmfgpu::ccdpp_train(config, a, probe)
//   parmf::als_train(config, a, probe)     (als.hpp:188)  ->  pmfgpu::als_train(config, a, probe)
//   parmf::run_training(spec, a, probe)    (bench.hpp:44) ->  pmfgpu::run_training(spec, a, probe)
//   parmf::rmse / parmf::objective         (model.hpp:156 / :119)
//
// Real = float only (the B200 path is FP32).  Status codes are rethrown as the reference's own
// exception types (types.hpp:35-44).  Link with paper_1511_02433_b200/libpmf_gpu.so.
#pragma once

#include <cmath>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pmf_gpu.h"

namespace pmfgpu {

inline void check(pmf_status s) {
    if (s == PMF_OK) return;
    const std::string msg = pmf_last_error();
    switch (s) {
        case PMF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PMF_DATA_ERROR: throw parmf::data_error(msg);
        case PMF_NOT_POSITIVE_DEFINITE: throw parmf::not_positive_definite(msg);
        case PMF_OUT_OF_RANGE: throw std::out_of_range(msg);
        case PMF_DOMAIN_ERROR: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline pmf_matrix_view view_of(const parmf::RatingsMatrix<float>& a) {
    pmf_matrix_view v;
    v.m = a.rows();
    v.n = a.cols();
    v.nnz = a.nnz();
    v.row_start = a.row_start().data();
    v.col_of = a.col_of().data();
    v.val_row = a.val_row().data();
    v.col_start = a.col_start().data();
    v.row_of = a.row_of().data();
    v.val_col = a.val_col().data();
    return v;
}

inline const pmf_triplet* probe_ptr(std::span<const parmf::Triplet<float>> probe) {
    static_assert(sizeof(parmf::Triplet<float>) == sizeof(pmf_triplet), "Triplet<float> layout");
    return reinterpret_cast<const pmf_triplet*>(probe.data());
}

namespace detail {
inline parmf::TrainReport report_of(const char* alg, int k, double lambda, int outer, int inner, int workers,
                                    std::uint64_t seed, const parmf::RatingsMatrix<float>& a,
                                    const std::vector<pmf_iter_row>& rows, const pmf_train_totals& tot) {
    parmf::TrainReport r;
    r.algorithm = alg;
    r.precision = "single";
    r.workers = workers;
    r.k = k;
    r.lambda = lambda;
    r.outer_iters = outer;
    r.inner_iters = inner;
    r.seed = seed;
    r.users = a.rows();
    r.items = a.cols();
    r.nnz = a.nnz();
    for (const auto& x : rows) r.rows.push_back({x.iteration, x.seconds, x.objective, x.rmse});
    r.stage_totals.push_back({std::string(alg) + "/gpu", tot.train_seconds,
                              static_cast<std::uint64_t>(tot.h2d_bytes), static_cast<std::uint64_t>(tot.d2h_bytes)});
    r.train_seconds = tot.train_seconds;
    r.wall_seconds = tot.wall_seconds;
    r.final_objective = tot.final_objective;
    r.final_rmse = tot.final_rmse;
    return r;
}
}  // namespace detail

// ccd.hpp:349-404
inline std::pair<parmf::FactorModel<float>, parmf::TrainReport> ccdpp_train(
    const parmf::CcdConfig<float>& config, const parmf::RatingsMatrix<float>& a,
    parmf::span_arg<const parmf::Triplet<float>> probe) {
    config.validate();
    // workers (ccd.hpp:39) -> GPUs: a device group of `workers` ranks (pmf_ctx_create_group)
    const pmf_ccd_config c{config.k, config.lambda, config.outer_iters, config.inner_iters, config.seed,
                           config.workers, 0};
    const pmf_matrix_view v = view_of(a);
    parmf::FactorModel<float> model(a.rows(), a.cols(), config.k);
    std::vector<pmf_iter_row> rows(static_cast<size_t>(config.outer_iters));
    pmf_train_totals tot{};
    check(pmf_ccdpp_train(&c, &v, probe_ptr(probe), static_cast<int64_t>(probe.size()), model.w().data(),
                          model.h().data(), rows.data(), &tot));
    if (probe.empty())
        for (auto& r : rows) r.rmse = std::numeric_limits<double>::quiet_NaN();
    return {std::move(model), detail::report_of("ccdpp", config.k, static_cast<double>(config.lambda),
                                                config.outer_iters, config.inner_iters, config.workers, config.seed,
                                                a, rows, tot)};
}

// ccd.hpp:310-344 (item/user-wise CCD; one device, inner_iters ignored like the reference)
inline std::pair<parmf::FactorModel<float>, parmf::TrainReport> ccd_train(
    const parmf::CcdConfig<float>& config, const parmf::RatingsMatrix<float>& a,
    parmf::span_arg<const parmf::Triplet<float>> probe) {
    config.validate();
    const pmf_ccd_config c{config.k, config.lambda, config.outer_iters, config.inner_iters, config.seed, 1, 0};
    const pmf_matrix_view v = view_of(a);
    parmf::FactorModel<float> model(a.rows(), a.cols(), config.k);
    std::vector<pmf_iter_row> rows(static_cast<size_t>(config.outer_iters));
    pmf_train_totals tot{};
    check(pmf_ccd_train(&c, &v, probe_ptr(probe), static_cast<int64_t>(probe.size()), model.w().data(),
                        model.h().data(), rows.data(), &tot));
    if (probe.empty())
        for (auto& r : rows) r.rmse = std::numeric_limits<double>::quiet_NaN();
    auto rep = detail::report_of("ccd", config.k, static_cast<double>(config.lambda), config.outer_iters, 1, 1,
                                 config.seed, a, rows, tot);
    return {std::move(model), std::move(rep)};
}

// als.hpp:188-233
inline std::pair<parmf::FactorModel<float>, parmf::TrainReport> als_train(
    const parmf::AlsConfig<float>& config, const parmf::RatingsMatrix<float>& a,
    parmf::span_arg<const parmf::Triplet<float>> probe) {
    config.validate();
    const pmf_als_config c{config.k, config.lambda, config.outer_iters, config.seed, config.workers, 0};  // als.hpp:30
    const pmf_matrix_view v = view_of(a);
    parmf::FactorModel<float> model(a.rows(), a.cols(), config.k);
    std::vector<pmf_iter_row> rows(static_cast<size_t>(config.outer_iters));
    pmf_train_totals tot{};
    check(pmf_als_train(&c, &v, probe_ptr(probe), static_cast<int64_t>(probe.size()), model.w().data(),
                        model.h().data(), rows.data(), &tot));
    return {std::move(model), detail::report_of("als", config.k, static_cast<double>(config.lambda),
                                                config.outer_iters, 1, config.workers, config.seed, a, rows, tot)};
}

// bench.hpp:44-74 (float only)
inline std::pair<parmf::FactorModel<float>, parmf::TrainReport> run_training(
    const parmf::RunSpec& spec, const parmf::RatingsMatrix<float>& a,
    parmf::span_arg<const parmf::Triplet<float>> probe) {
    if (spec.algorithm == parmf::Algorithm::kAls) {
        parmf::AlsConfig<float> c;
        c.k = spec.k;
        c.lambda = static_cast<float>(spec.lambda);
        c.outer_iters = spec.outer_iters;
        c.workers = spec.workers;
        c.seed = spec.seed;
        return als_train(c, a, probe);
    }
    parmf::CcdConfig<float> c;
    c.k = spec.k;
    c.lambda = static_cast<float>(spec.lambda);
    c.outer_iters = spec.outer_iters;
    c.inner_iters = spec.inner_iters;
    c.workers = spec.workers;
    c.seed = spec.seed;
    if (spec.algorithm == parmf::Algorithm::kCcd) {
        c.variant = parmf::CcdVariant::kCcd;
        return ccd_train(c, a, probe);
    }
    return ccdpp_train(c, a, probe);
}

// model.hpp:172-198 top_n(model, i, count, rated_sorted), scored on the B200
inline std::vector<std::pair<parmf::index_t, float>> top_n(const parmf::FactorModel<float>& model,
                                                           parmf::index_t i, parmf::index_t count,
                                                           std::span<const parmf::index_t> rated_sorted) {
    const int32_t user = i;
    const int64_t ex_start[2] = {0, static_cast<int64_t>(rated_sorted.size())};
    const int32_t none = 0;
    const size_t c = static_cast<size_t>(count > 0 ? count : 1);
    std::vector<int32_t> items(c);
    std::vector<float> scores(c);
    int32_t got = 0;
    check(pmf_top_n(model.w().data(), model.h().data(), model.users(), model.items(), model.rank(), &user, 1, count,
                    ex_start, rated_sorted.empty() ? &none : rated_sorted.data(), items.data(), scores.data(), &got));
    std::vector<std::pair<parmf::index_t, float>> out(static_cast<size_t>(got));
    for (int32_t x = 0; x < got; ++x) out[static_cast<size_t>(x)] = {items[static_cast<size_t>(x)], scores[static_cast<size_t>(x)]};
    return out;
}

// model.hpp:203-209 (rated items from the matrix row)
inline std::vector<std::pair<parmf::index_t, float>> top_n(const parmf::FactorModel<float>& model,
                                                           const parmf::RatingsMatrix<float>& a, parmf::index_t i,
                                                           parmf::index_t count) {
    std::vector<parmf::index_t> rated;
    rated.reserve(static_cast<size_t>(a.row_nnz(i)));
    for (const auto [item, pos] : a.row_slice(i)) rated.push_back(item);
    return top_n(model, i, count, rated);
}

// model.hpp:156-167
inline double rmse(const parmf::FactorModel<float>& model, parmf::span_arg<const parmf::Triplet<float>> probe) {
    double out = 0;
    check(pmf_rmse(model.w().data(), model.h().data(), model.users(), model.items(), model.rank(),
                   probe_ptr(probe), static_cast<int64_t>(probe.size()), &out));
    return out;
}

// model.hpp:119-144
inline double objective(const parmf::FactorModel<float>& model, const parmf::RatingsMatrix<float>& a,
                        double lambda) {
    const pmf_matrix_view v = view_of(a);
    double out = 0;
    check(pmf_objective(&v, model.w().data(), model.h().data(), model.rank(), lambda, &out));
    return out;
}

}  // namespace pmfgpu
