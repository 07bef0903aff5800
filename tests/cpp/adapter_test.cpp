// C++ drop-in check: a parmf caller switches ccdpp_train / als_train / rmse / objective from the
// reference (parmf::) to the B200 backend (pmfgpu::, include/pmfgpu.hpp) with the same types.
// Built by oracle/Makefile against the UNMODIFIED reference headers into oracle/_ref/adapter_test;
// run on the GPU box by tests/test_gpu_adapter.py.  Exit 0 = parity within 1e-4 relative.
#include <cmath>
#include <cstdio>

#include "parmf/parmf.hpp"
#include "pmfgpu.hpp"
#include "testutil.hpp"

static bool close(double a, double b, double tol) { return std::abs(a - b) <= tol * std::abs(b); }

int main() {
    auto d = testutil::synth_ratings<float>(943, 1682, 3, 100000, 777);
    std::vector<parmf::Triplet<float>> probe;
    testutil::carve_probe(d, probe, 10000, 5);
    const auto a = parmf::RatingsMatrix<float>::from_triplets(d, 943, 1682);
    parmf::CcdConfig<float> c;
    c.k = 10; c.lambda = 0.05f; c.outer_iters = 3; c.inner_iters = 15; c.seed = 1; c.workers = 4;
    const auto [m_ref, r_ref] = parmf::ccdpp_train(c, a, probe);
    const auto [m_gpu, r_gpu] = pmfgpu::ccdpp_train(c, a, probe);
    int bad = 0;
    for (size_t i = 0; i < r_ref.rows.size(); ++i) {
        std::printf("ccdpp iter %d objective ref %.10g gpu %.10g  rmse ref %.8f gpu %.8f\n", r_ref.rows[i].iteration,
                    r_ref.rows[i].objective, r_gpu.rows[i].objective, r_ref.rows[i].rmse, r_gpu.rows[i].rmse);
        bad += !close(r_gpu.rows[i].objective, r_ref.rows[i].objective, 1e-4) || !close(r_gpu.rows[i].rmse, r_ref.rows[i].rmse, 1e-4);
    }
    bad += !close(pmfgpu::rmse(m_gpu, probe), parmf::rmse(m_gpu, std::span<const parmf::Triplet<float>>(probe)), 1e-12);
    bad += !close(pmfgpu::objective(m_gpu, a, 0.05), parmf::objective(m_gpu, a, 0.05), 1e-12);
    parmf::AlsConfig<float> ac;
    ac.k = 10; ac.lambda = 0.05f; ac.outer_iters = 2; ac.seed = 1;
    const auto [ma, ra] = parmf::als_train(ac, a, probe);
    const auto [mg, rg] = pmfgpu::als_train(ac, a, probe);
    for (size_t i = 0; i < ra.rows.size(); ++i) {
        std::printf("als iter %d objective ref %.10g gpu %.10g\n", ra.rows[i].iteration, ra.rows[i].objective, rg.rows[i].objective);
        bad += !close(rg.rows[i].objective, ra.rows[i].objective, 1e-4);
    }
    // item/user-wise CCD through run_training's kCcd dispatch (ccd.hpp:310-344)
    parmf::RunSpec spec;
    spec.algorithm = parmf::Algorithm::kCcd;
    spec.k = 10; spec.lambda = 0.05; spec.outer_iters = 2; spec.seed = 1;
    const auto [mc_ref, rc_ref] = parmf::run_training(spec, a, std::span<const parmf::Triplet<float>>(probe));
    const auto [mc_gpu, rc_gpu] = pmfgpu::run_training(spec, a, probe);
    for (size_t i = 0; i < rc_ref.rows.size(); ++i) {
        std::printf("ccd iter %d objective ref %.10g gpu %.10g\n", rc_ref.rows[i].iteration, rc_ref.rows[i].objective,
                    rc_gpu.rows[i].objective);
        bad += !close(rc_gpu.rows[i].objective, rc_ref.rows[i].objective, 1e-4);
    }
    // top_n: identical rankings and scores on the same model (model.hpp:172-209)
    for (parmf::index_t i : {0, 17, 942}) {
        const auto r1 = parmf::top_n(m_gpu, a, i, 25);
        const auto r2 = pmfgpu::top_n(m_gpu, a, i, 25);
        bad += r1 != r2;
    }
    try {
        parmf::AlsConfig<float> badc;
        badc.lambda = 0.0f;
        pmfgpu::als_train(badc, a, probe);
        ++bad;
    } catch (const std::invalid_argument&) {
    }
    std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
    return bad ? 1 : 0;
}
