// microadam_b200.cpp — C++ host API (see microadam_b200.hpp) on the C ABI.
#include "microadam_b200.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

namespace microadam_b200 {

namespace {

[[noreturn]] void throw_status(ma_status st) {
    const std::string msg = ma_last_error();
    switch (st) {
        case MA_ERR_INVALID_ARG:
        case MA_ERR_DIM:
        case MA_ERR_NONFINITE:
            throw std::invalid_argument(msg);
        case MA_ERR_STATE:
            throw std::logic_error(msg);
        default:
            throw std::runtime_error(msg);
    }
}

void check(ma_status st) {
    if (st != MA_OK) throw_status(st);
}

GradientWindow read_window(ma_handle* h, int64_t dim, int64_t m) {
    ma_layout_info lay{};
    check(ma_get_layout(h, &lay));
    GradientWindow w;
    w.dim = dim;
    w.capacity = m;
    w.row_width = lay.row_width;
    std::vector<int64_t> stamps(static_cast<size_t>(m));
    check(ma_get_counters(h, &w.step, &w.head, &w.filled, stamps.data()));
    w.rows.resize(static_cast<size_t>(m));
    for (int64_t r = 0; r < m; ++r) {
        auto& row = w.rows[static_cast<size_t>(r)];
        row.stamp = stamps[static_cast<size_t>(r)];
        if (row.stamp == 0) continue;  // never written: empty, as in the reference
        row.indices.resize(static_cast<size_t>(lay.row_width));
        row.values.resize(static_cast<size_t>(lay.row_width));
        check(ma_read_window_row(h, r, row.indices.data(), row.values.data()));
    }
    return w;
}

QuantizedErrorBuffer read_error(ma_handle* h, int64_t dim, const HyperParams& hp) {
    ma_layout_info lay{};
    check(ma_get_layout(h, &lay));
    QuantizedErrorBuffer b;
    b.dim = lay.dim;
    (void)dim;
    b.bits = hp.bits;
    b.bucket = hp.bucket;
    b.codes.resize(static_cast<size_t>(lay.code_bytes));
    b.lo.resize(static_cast<size_t>(lay.num_buckets));
    b.hi.resize(static_cast<size_t>(lay.num_buckets));
    check(ma_read_error_buffer(h, b.codes.data(), b.lo.data(), b.hi.data()));
    return b;
}

}  // namespace

void HyperParams::validate() const {
    ma_config cfg;
    ma_config_default(&cfg);
    cfg.hp = to_c();
    // Validation of the hyperparameters alone: a 1-element vector never trips
    // the device-support checks that depend on d.
    const ma_status st = ma_validate(&cfg, k ? *k : 1);
    if (st == MA_ERR_INVALID_ARG) throw std::invalid_argument(ma_last_error());
}

int64_t HyperParams::resolve_k(int64_t dim) const {
    if (k) {
        if (*k > dim) throw std::invalid_argument("HyperParams: k exceeds dimension");
        return *k;
    }
    auto count = static_cast<int64_t>(std::ceil(density * static_cast<double>(dim)));
    return count < 1 ? 1 : (count > dim ? dim : count);
}

ma_hyperparams HyperParams::to_c() const {
    ma_hyperparams c{};
    c.beta1 = beta1;
    c.beta2 = beta2;
    c.eps = eps;
    c.lr = lr;
    c.weight_decay = weight_decay;
    c.window = window;
    c.density = density;
    c.k = k ? *k : 0;
    c.bits = bits;
    c.block = block;
    c.bucket = bucket;
    return c;
}

Vec QuantizedErrorBuffer::decode() const {
    Vec out(static_cast<size_t>(dim));
    const double mx = static_cast<double>((1u << bits) - 1u);
    for (int64_t i = 0; i < dim; ++i) {
        const int64_t b = i / bucket;
        const double lvl = lo[size_t(b)] == hi[size_t(b)] ? 0.0 : (hi[size_t(b)] - lo[size_t(b)]) / mx;
        // LSB-first bit stream of `bits`-wide codes (quantize.cpp:102-128)
        const int64_t pos = i * bits;
        uint32_t w = codes[size_t(pos >> 3)];
        for (int k = 1; 8 * k < int(pos & 7) + bits; ++k) w |= uint32_t(codes[size_t((pos >> 3) + k)]) << (8 * k);
        const uint32_t c = (w >> (pos & 7)) & ((1u << bits) - 1u);
        out[size_t(i)] = static_cast<double>(c) * lvl + lo[size_t(b)];
    }
    return out;
}

// ---------------------------------------------------------------------------
MicroAdam::MicroAdam(int64_t dim, const HyperParams& hp, const DeviceOptions& opt)
    : dim_(dim), hp_(hp) {
    ma_config cfg;
    ma_config_default(&cfg);
    cfg.hp = hp.to_c();
    cfg.blockwise = opt.blockwise ? 1 : 0;
    cfg.param_dtype = opt.param_dtype;
    cfg.grad_dtype = opt.grad_dtype;
    cfg.value_dtype = opt.value_dtype;
    cfg.finite_mode = opt.finite_mode;
    check(ma_create_shard(&cfg, dim, opt.block_begin, opt.block_end, opt.device, &h_));
}

MicroAdam::~MicroAdam() { ma_destroy(h_); }

StepReport MicroAdam::step(void* d_params, const void* d_grads, double lr, void* stream,
                           bool want_report) {
    ma_step_report r{};
    check(ma_step(h_, d_params, d_grads, lr, stream, want_report ? &r : nullptr));
    return StepReport{r.grad_norm, r.error_norm, r.empirical_q, r.update_nnz, r.loss};
}

StepReport MicroAdam::step_reduce(void* d_params, void* d_grads, const std::vector<const void*>& sources,
                                  float scale, double lr, void* stream, bool want_report) {
    ma_step_report r{};
    check(ma_step_reduce(h_, d_params, d_grads, sources.data(), static_cast<int32_t>(sources.size()), scale, lr,
                         stream, want_report ? &r : nullptr));
    return StepReport{r.grad_norm, r.error_norm, r.empirical_q, r.update_nnz, r.loss};
}

void MicroAdam::synchronize() { check(ma_sync(h_)); }

ma_layout_info MicroAdam::layout() const {
    ma_layout_info l{};
    check(ma_get_layout(h_, &l));
    return l;
}

int64_t MicroAdam::step_count() const {
    int64_t s = 0;
    check(ma_get_counters(h_, &s, nullptr, nullptr, nullptr));
    return s;
}

GradientWindow MicroAdam::window() const { return read_window(h_, dim_, hp_.window); }

QuantizedErrorBuffer MicroAdam::error_buffer() const { return read_error(h_, dim_, hp_); }

// ---------------------------------------------------------------------------
MicroAdamOptimizer::MicroAdamOptimizer(Vec theta0, HyperParams hp, bool blockwise,
                                       bool lossless_error, int device)
    : theta_(std::move(theta0)), hp_(hp) {
    ma_config cfg;
    ma_config_default(&cfg);
    cfg.hp = hp_.to_c();
    cfg.blockwise = blockwise ? 1 : 0;
    cfg.lossless_error = lossless_error ? 1 : 0;
    lossless_ = lossless_error;
    cfg.param_dtype = MA_F64;
    cfg.grad_dtype = MA_F64;
    cfg.value_dtype = MA_F64;
    cfg.finite_mode = MA_FINITE_STRICT;
    check(ma_create(&cfg, static_cast<int64_t>(theta_.size()), device, &h_));
    check(ma_set_params(h_, theta_.data()));
    last_sel_.dim = static_cast<int64_t>(theta_.size());
}

MicroAdamOptimizer::~MicroAdamOptimizer() { ma_destroy(h_); }

StepReport MicroAdamOptimizer::step(const Vec& grad) {
    if (grad.size() != theta_.size()) throw std::invalid_argument("step: gradient dim mismatch");
    ma_step_report r{};
    check(ma_step_host(h_, theta_.data(), grad.data(), hp_.lr, &r));
    // last_selection(): the row just written (slot head-1), values exact in fp64.
    int64_t head = 0;
    check(ma_get_counters(h_, nullptr, &head, nullptr, nullptr));
    ma_layout_info lay{};
    check(ma_get_layout(h_, &lay));
    const int64_t slot = (head + hp_.window - 1) % hp_.window;
    last_sel_.indices.resize(static_cast<size_t>(lay.row_width));
    last_sel_.values.resize(static_cast<size_t>(lay.row_width));
    check(ma_read_window_row(h_, slot, last_sel_.indices.data(), last_sel_.values.data()));
    return StepReport{r.grad_norm, r.error_norm, r.empirical_q, r.update_nnz, r.loss};
}

GradientWindow MicroAdamOptimizer::window() const {
    return read_window(h_, static_cast<int64_t>(theta_.size()), hp_.window);
}

QuantizedErrorBuffer MicroAdamOptimizer::error_buffer() const {
    return read_error(h_, static_cast<int64_t>(theta_.size()), hp_);
}

Vec MicroAdamOptimizer::error_vector() const {  // optim.cpp:160-162
    Vec out(theta_.size());
    check(ma_read_error_vector(h_, out.data()));
    return out;
}

int64_t MicroAdamOptimizer::step_count() const {
    int64_t s = 0;
    check(ma_get_counters(h_, &s, nullptr, nullptr, nullptr));
    return s;
}

void MicroAdam::save_checkpoint(const std::string& path, const void* d_params) const {
    check(ma_save_checkpoint(h_, d_params, 1, path.c_str()));
}

void MicroAdam::load_checkpoint(const std::string& path, void* d_params) {
    check(ma_load_checkpoint(h_, d_params, 1, path.c_str()));
}

void save_checkpoint(const std::string& path, const MicroAdamOptimizer& opt) {
    check(ma_save_checkpoint(opt.handle(), opt.params().data(), 0, path.c_str()));
}

void load_checkpoint(const std::string& path, MicroAdamOptimizer& opt) {
    check(ma_load_checkpoint(opt.handle(), opt.mutable_params().data(), 0, path.c_str()));
}

}  // namespace microadam_b200
