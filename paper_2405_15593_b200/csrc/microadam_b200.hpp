// microadam_b200.hpp — C++ host API over the C ABI (include/microadam_cuda.h).
//
// Mirrors the reference optimizer interface so code written against
// /root/reference/proj/include/microadam/optim.hpp can switch by namespace:
//
//   microadam::HyperParams        (optim.hpp:15-30)  -> microadam_b200::HyperParams
//   microadam::StepReport         (optim.hpp:32-38)  -> microadam_b200::StepReport
//   microadam::Optimizer          (optim.hpp:40-46)  -> microadam_b200::Optimizer
//   microadam::MicroAdamOptimizer (optim.hpp:98-128) -> microadam_b200::MicroAdamOptimizer
//                                                      (host Vec API, fp64 on device,
//                                                       bit-identical to the reference)
//
// plus the device-memory engine the north star names: construct from the
// parameter count and block/density/window/quant settings, then
// step(params, grads, lr) — microadam_b200::MicroAdam.
//
// Errors are thrown exactly where the reference throws: std::invalid_argument
// for invalid configs, dimension mismatch and non-finite gradients,
// std::logic_error for error_buffer() on a lossless engine; CUDA failures
// throw std::runtime_error.
#pragma once

#include <cstdint>
#include <optional>
#include <string_view>
#include <string>
#include <vector>

#include "../../include/microadam_cuda.h"

#pragma GCC visibility push(default)
namespace microadam_b200 {

using Vec = std::vector<double>;

struct HyperParams {
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
    double lr = 1e-3;
    double weight_decay = 0.0;
    int64_t window = 10;
    double density = 0.01;
    std::optional<int64_t> k;
    int bits = 4;
    int64_t block = 4096;
    int64_t bucket = 64;

    void validate() const;                 // optim.cpp:7-21
    int64_t resolve_k(int64_t dim) const;  // optim.cpp:23-30
    ma_hyperparams to_c() const;
};

struct StepReport {
    double grad_norm = 0.0;
    double error_norm = 0.0;
    double empirical_q = 0.0;
    int64_t update_nnz = 0;
    double loss = 0.0;
};

class Optimizer {
public:
    virtual ~Optimizer() = default;
    virtual StepReport step(const Vec& grad) = 0;
    virtual const Vec& params() const = 0;
    virtual std::string_view name() const = 0;
};

struct SparseSelection {  // compress.hpp:9-17
    int64_t dim = 0;
    std::vector<int64_t> indices;
    Vec values;
    int64_t size() const { return static_cast<int64_t>(indices.size()); }
};

struct GradientWindow {  // window.hpp:10-33 (read back from device)
    struct Row {
        int64_t stamp = 0;
        std::vector<int64_t> indices;
        Vec values;
    };
    int64_t dim = 0, capacity = 0, row_width = 0, head = 0, filled = 0, step = 0;
    std::vector<Row> rows;
};

struct QuantizedErrorBuffer {  // quantize.hpp:54-70 (read back from device)
    int64_t dim = 0;
    int bits = 4;
    int64_t bucket = 64;
    std::vector<uint8_t> codes;
    Vec lo, hi;
    int64_t num_buckets() const { return (dim + bucket - 1) / bucket; }
    Vec decode() const;  // quantize.cpp:164-178
};

struct DeviceOptions {
    ma_dtype param_dtype = MA_F32;
    ma_dtype grad_dtype = MA_F32;
    ma_dtype value_dtype = MA_BF16;
    ma_finite_mode finite_mode = MA_FINITE_FLAG;
    int device = 0;
    bool blockwise = true;
    int64_t block_begin = 0;  // shard: owned block range [begin, end); end < 0 = all
    int64_t block_end = -1;
};

// Device-memory engine: the caller owns θ and g on the device.
class MicroAdam {
public:
    MicroAdam(int64_t dim, const HyperParams& hp, const DeviceOptions& opt = {});
    ~MicroAdam();
    MicroAdam(const MicroAdam&) = delete;
    MicroAdam& operator=(const MicroAdam&) = delete;

    // θ -= lr · update, in place; asynchronous on `stream` unless want_report.
    StepReport step(void* d_params, const void* d_grads, double lr, void* stream = nullptr,
                    bool want_report = false);
    // Data-parallel step with the gradient reduce-scatter fused in
    // (ma_step_reduce): sources = every rank's gradient for this handle's range.
    StepReport step_reduce(void* d_params, void* d_grads, const std::vector<const void*>& sources,
                           float scale, double lr, void* stream = nullptr, bool want_report = false);
    void synchronize();  // throws std::invalid_argument on a flagged non-finite gradient

    ma_layout_info layout() const;
    int64_t step_count() const;
    GradientWindow window() const;
    QuantizedErrorBuffer error_buffer() const;
    ma_handle* handle() const { return h_; }
    // MADM v1 checkpoint of this engine + its device θ (checkpoint.cpp:50-140)
    void save_checkpoint(const std::string& path, const void* d_params) const;
    void load_checkpoint(const std::string& path, void* d_params /* nullable */);

private:
    ma_handle* h_ = nullptr;
    int64_t dim_ = 0;
    HyperParams hp_;
};

// Drop-in for microadam::MicroAdamOptimizer(theta0, hp, blockwise = false,
// lossless_error = false) (optim.hpp:103-104: the same defaults, so code written
// against the reference selects global Top-K here too):
// host vectors in and out, fp64 θ/g/window on the device, strict
// (reject-before-mutate) finiteness — bit-identical to the reference step.
class MicroAdamOptimizer : public Optimizer {
public:
    MicroAdamOptimizer(Vec theta0, HyperParams hp, bool blockwise = false,
                       bool lossless_error = false, int device = 0);
    ~MicroAdamOptimizer() override;
    StepReport step(const Vec& grad) override;
    const Vec& params() const override { return theta_; }
    std::string_view name() const override { return "microadam"; }

    GradientWindow window() const;
    QuantizedErrorBuffer error_buffer() const;
    bool lossless() const { return lossless_; }
    Vec error_vector() const;
    const SparseSelection& last_selection() const { return last_sel_; }
    int64_t step_count() const;
    const HyperParams& hyper() const { return hp_; }
    ma_handle* handle() const { return h_; }
    Vec& mutable_params() { return theta_; }

private:
    Vec theta_;
    HyperParams hp_;
    ma_handle* h_ = nullptr;
    SparseSelection last_sel_;
    bool lossless_ = false;
};

// save_checkpoint(path, opt) / resume (checkpoint.hpp:28-33): the reference's
// MADM v1 file; byte-identical to the reference's for the same state.
void save_checkpoint(const std::string& path, const MicroAdamOptimizer& opt);
void load_checkpoint(const std::string& path, MicroAdamOptimizer& opt);

}  // namespace microadam_b200
#pragma GCC visibility pop
