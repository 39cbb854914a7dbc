// adapter_check.cpp — the reference-side binding of INTEGRATION.md §2, compiled
// against the UNMODIFIED reference headers and sources (/root/reference/proj)
// and linked with libmicroadam_cuda.so (oracle/Makefile -> oracle/_ref/adapter_check).
//
// TEST INFRASTRUCTURE: it drives the reference's own training loop
// (run(Optimizer&, const Objective&, T, seed), optim.cpp:352-376) once with the
// reference's MicroAdamOptimizer and once with CudaMicroAdamOptimizer (the
// adapter a maintainer adds), and requires every iterate to be bit-identical
// and every StepReport to agree (update_nnz exactly, norms within 1e-12
// relative: the device sums in a fixed tree order). Blockwise and global
// (d > 8192) modes. Exit code 0 = drop-in confirmed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "microadam/optim.hpp"
#include "microadam/problems.hpp"
#include "microadam_cuda.h"

namespace microadam {

// ---- the adapter ----
class CudaMicroAdamOptimizer : public Optimizer {
public:
    CudaMicroAdamOptimizer(Vec theta0, const HyperParams& hp, bool blockwise = false)
        : theta_(std::move(theta0)), hp_(hp) {
        ma_config cfg;
        ma_config_default(&cfg);
        cfg.hp.beta1 = hp.beta1;
        cfg.hp.beta2 = hp.beta2;
        cfg.hp.eps = hp.eps;
        cfg.hp.lr = hp.lr;
        cfg.hp.weight_decay = hp.weight_decay;
        cfg.hp.window = hp.window;
        cfg.hp.density = hp.density;
        cfg.hp.k = hp.k ? *hp.k : 0;
        cfg.hp.bits = hp.bits;
        cfg.hp.block = hp.block;
        cfg.hp.bucket = hp.bucket;
        cfg.blockwise = blockwise ? 1 : 0;
        // fp64 on device + reject-before-mutate: bit-identical to MicroAdamOptimizer
        cfg.param_dtype = cfg.grad_dtype = cfg.value_dtype = MA_F64;
        cfg.finite_mode = MA_FINITE_STRICT;
        check(ma_create(&cfg, static_cast<int64_t>(theta_.size()), /*device=*/0, &h_));
        check(ma_set_params(h_, theta_.data()));
    }
    ~CudaMicroAdamOptimizer() override { ma_destroy(h_); }

    StepReport step(const Vec& grad) override {  // optim.cpp:164-190
        if (grad.size() != theta_.size()) throw std::invalid_argument("step: gradient dim mismatch");
        ma_step_report r{};
        check(ma_step_host(h_, theta_.data(), grad.data(), hp_.lr, &r));
        StepReport out;
        out.grad_norm = r.grad_norm;
        out.error_norm = r.error_norm;
        out.empirical_q = r.empirical_q;
        out.update_nnz = r.update_nnz;
        return out;
    }
    const Vec& params() const override { return theta_; }
    std::string_view name() const override { return "microadam"; }

private:
    static void check(ma_status st) {
        if (st == MA_OK) return;
        if (st == MA_ERR_INVALID_ARG || st == MA_ERR_DIM || st == MA_ERR_NONFINITE)
            throw std::invalid_argument(ma_last_error());
        if (st == MA_ERR_STATE) throw std::logic_error(ma_last_error());
        throw std::runtime_error(ma_last_error());
    }
    Vec theta_;
    HyperParams hp_;
    ma_handle* h_ = nullptr;
};

}  // namespace microadam

using namespace microadam;

static bool rel_ok(double a, double b) { return std::fabs(a - b) <= 1e-12 * std::fmax(std::fabs(b), 1e-300); }

static int compare(const char* what, const Objective& obj, const Vec& theta0, const HyperParams& hp,
                   bool blockwise, int64_t T) {
    MicroAdamOptimizer ref(theta0, hp, blockwise);
    CudaMicroAdamOptimizer dev(theta0, hp, blockwise);
    Trajectory a = run(ref, obj, T, /*seed=*/7);
    Trajectory b = run(dev, obj, T, /*seed=*/7);
    if (a.steps_completed != b.steps_completed) {
        std::printf("%s: steps %lld vs %lld\n", what, (long long)a.steps_completed, (long long)b.steps_completed);
        return 1;
    }
    for (int64_t t = 0; t < a.steps_completed; ++t) {
        const Vec& x = a.iterates[size_t(t)];
        const Vec& y = b.iterates[size_t(t)];
        if (std::memcmp(x.data(), y.data(), x.size() * sizeof(double)) != 0) {
            std::printf("%s: iterate %lld differs\n", what, (long long)t);
            return 1;
        }
        const StepReport& r = a.reports[size_t(t)];
        const StepReport& s = b.reports[size_t(t)];
        if (r.update_nnz != s.update_nnz || !rel_ok(s.grad_norm, r.grad_norm) ||
            !rel_ok(s.error_norm, r.error_norm) || !rel_ok(s.empirical_q, r.empirical_q) || r.loss != s.loss) {
            std::printf("%s: report %lld differs\n", what, (long long)t);
            return 1;
        }
    }
    std::printf("%s: %lld steps bit-identical (d = %zu, final loss %.17g)\n", what,
                (long long)a.steps_completed, theta0.size(), a.reports.back().loss);
    return 0;
}

int main() {
    int bad = 0;
    {
        const int64_t d = 9000;  // > 8192: the global mode runs ma_global.cu
        Objective obj = logistic_regression(/*n=*/d, d, /*separation=*/1.5, /*seed=*/3);
        HyperParams hp;
        hp.lr = 1e-2;
        hp.window = 4;
        Vec theta0(static_cast<size_t>(d), 0.0);
        bad |= compare("blockwise logistic", obj, theta0, hp, true, 12);
        bad |= compare("global logistic", obj, theta0, hp, false, 12);
    }
    {
        const int64_t d = 50000;
        Vec a(static_cast<size_t>(d)), bvec(static_cast<size_t>(d));
        for (int64_t i = 0; i < d; ++i) {
            a[size_t(i)] = 1.0 + double(i % 97) / 10.0;
            bvec[size_t(i)] = std::sin(double(i));
        }
        Objective obj = quadratic(a, bvec);
        HyperParams hp;
        hp.lr = 5e-3;
        hp.window = 6;
        hp.density = 0.02;
        Vec theta0(static_cast<size_t>(d));
        for (int64_t i = 0; i < d; ++i) theta0[size_t(i)] = std::cos(double(i) * 0.37);
        bad |= compare("blockwise quadratic", obj, theta0, hp, true, 15);
        bad |= compare("global quadratic", obj, theta0, hp, false, 8);
    }
    std::printf(bad ? "adapter FAILED\n" : "adapter ok\n");
    return bad;
}
