// ref_shim.cpp — extern "C" wrapper around the UNMODIFIED reference sources
// (/root/reference/proj/src/{compress,quantize,window,problems,optim,checkpoint}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libmicroadam_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (oracle/microadam_oracle.c) and to generate tests/golden/, and by bench.py's
// cpu_baseline / --impl reference leg to time the reference's own CPU step.
// Nothing in the product links or loads it.
//
// No reference source is copied here: this file only includes the reference
// headers and calls its public API (optim.hpp:98-128, compress.hpp,
// quantize.hpp, window.hpp).
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../include/ma_synth.h"
#include "microadam/checkpoint.hpp"
#include "microadam/compress.hpp"
#include "microadam/optim.hpp"
#include "microadam/quantize.hpp"
#include "microadam/window.hpp"

using namespace microadam;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 7;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

HyperParams make_hp(double beta1, double beta2, double eps, double lr, int64_t window,
                    double density, int64_t k, int bits, int64_t block, int64_t bucket) {
    HyperParams hp;
    hp.beta1 = beta1;
    hp.beta2 = beta2;
    hp.eps = eps;
    hp.lr = lr;
    hp.window = window;
    hp.density = density;
    if (k > 0) hp.k = k;
    hp.bits = bits;
    hp.block = block;
    hp.bucket = bucket;
    return hp;
}

// bf16 round-to-nearest-even of a double (identical rule to the oracle and
// the device); used only to produce bf16-valued synthetic gradients.
double bf16_round(double x) {
    if (!std::isfinite(x) || x == 0.0) return x;
    if (std::fabs(x) < 0x1p-126) return std::nearbyint(x * 0x1p133) * 0x1p-133;
    uint64_t u;
    std::memcpy(&u, &x, 8);
    uint64_t lsb = (u >> 45) & 1u;
    u += (uint64_t(1) << 44) - 1u + lsb;
    u &= ~((uint64_t(1) << 45) - 1u);
    double y;
    std::memcpy(&y, &u, 8);
    if (std::fabs(y) >= 0x1p128) return std::copysign(INFINITY, x);
    return y;
}

double round_dtype(double x, int dtype) {
    if (dtype == 1) return double(float(x));
    if (dtype == 2) return bf16_round(x);
    return x;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- MicroAdamOptimizer (optim.hpp:98-128) ----
void* ref_create(int64_t dim, const double* theta0, double beta1, double beta2, double eps,
                 double lr, int64_t window, double density, int64_t k, int bits, int64_t block,
                 int64_t bucket, int blockwise, int lossless, int* status) {
    MicroAdamOptimizer* out = nullptr;
    *status = guarded([&] {
        Vec th(theta0, theta0 + dim);
        out = new MicroAdamOptimizer(std::move(th),
                                     make_hp(beta1, beta2, eps, lr, window, density, k, bits,
                                             block, bucket),
                                     blockwise != 0, lossless != 0);
    });
    return out;
}

void ref_destroy(void* h) { delete static_cast<MicroAdamOptimizer*>(h); }

// ---- save_checkpoint / load_checkpoint (checkpoint.hpp:28-33) ----
int ref_save_checkpoint(void* h, const char* path) {
    return guarded([&] { save_checkpoint(path, *static_cast<MicroAdamOptimizer*>(h)); });
}

// Loads with the reference loader; out: dim, step, capacity, row_width, head, filled.
int ref_load_checkpoint(const char* path, int64_t* out6, double* theta /* dim, may be NULL */) {
    return guarded([&] {
        Checkpoint cp = load_checkpoint(path);
        out6[0] = cp.dim;
        out6[1] = cp.step;
        out6[2] = cp.capacity;
        out6[3] = cp.row_width;
        out6[4] = cp.head;
        out6[5] = cp.filled;
        if (theta) std::memcpy(theta, cp.theta.data(), cp.theta.size() * sizeof(double));
    });
}

int ref_step(void* h, const double* grad, int64_t n, double* report5) {
    auto* o = static_cast<MicroAdamOptimizer*>(h);
    return guarded([&] {
        StepReport r = o->step(Vec(grad, grad + n));
        if (report5) {
            report5[0] = r.grad_norm;
            report5[1] = r.error_norm;
            report5[2] = r.empirical_q;
            report5[3] = double(r.update_nnz);
            report5[4] = r.loss;
        }
    });
}

int64_t ref_dim(void* h) { return int64_t(static_cast<MicroAdamOptimizer*>(h)->params().size()); }

void ref_params(void* h, double* out) {
    const Vec& p = static_cast<MicroAdamOptimizer*>(h)->params();
    std::memcpy(out, p.data(), p.size() * sizeof(double));
}

int64_t ref_row_width(void* h) { return static_cast<MicroAdamOptimizer*>(h)->window().row_width; }

void ref_counters(void* h, int64_t* step, int64_t* head, int64_t* filled, int64_t* stamps) {
    const GradientWindow& w = static_cast<MicroAdamOptimizer*>(h)->window();
    *step = w.step;
    *head = w.head;
    *filled = w.filled;
    for (int64_t r = 0; r < w.capacity; ++r) stamps[r] = w.rows[size_t(r)].stamp;
}

// Copies window row `slot` (empty rows copy nothing). Returns its length.
int64_t ref_window_row(void* h, int64_t slot, int64_t* idx, double* val) {
    const GradientWindow& w = static_cast<MicroAdamOptimizer*>(h)->window();
    const auto& row = w.rows[size_t(slot)];
    for (size_t j = 0; j < row.indices.size(); ++j) {
        idx[j] = row.indices[j];
        val[j] = row.values[j];
    }
    return int64_t(row.indices.size());
}

int64_t ref_last_selection(void* h, int64_t* idx, double* val) {
    const SparseSelection& s = static_cast<MicroAdamOptimizer*>(h)->last_selection();
    for (size_t j = 0; j < s.indices.size(); ++j) {
        idx[j] = s.indices[j];
        val[j] = s.values[j];
    }
    return s.size();
}

int64_t ref_num_buckets(void* h) {
    return static_cast<MicroAdamOptimizer*>(h)->error_buffer().num_buckets();
}

int ref_error_buffer(void* h, uint8_t* codes, double* lo, double* hi) {
    auto* o = static_cast<MicroAdamOptimizer*>(h);
    return guarded([&] {
        const QuantizedErrorBuffer& b = o->error_buffer();
        std::memcpy(codes, b.codes.data(), b.codes.size());
        for (size_t i = 0; i < b.params.size(); ++i) {
            lo[i] = b.params[i].lo;
            hi[i] = b.params[i].hi;
        }
    });
}

void ref_error_vector(void* h, double* out) {
    Vec e = static_cast<MicroAdamOptimizer*>(h)->error_vector();
    std::memcpy(out, e.data(), e.size() * sizeof(double));
}

// ---- L1 primitives (compress.hpp, quantize.hpp, window.hpp) ----
int64_t ref_topk_blockwise(const double* x, int64_t d, int64_t block, int64_t per_block_k,
                           int64_t* idx, double* val) {
    int64_t n = -1;
    int st = guarded([&] {
        SparseSelection s = topk_blockwise(Vec(x, x + d), BlockLayout(d, block, per_block_k));
        for (size_t j = 0; j < s.indices.size(); ++j) {
            idx[j] = s.indices[j];
            val[j] = s.values[j];
        }
        n = s.size();
    });
    return st ? -1 : n;
}

int64_t ref_topk_global(const double* x, int64_t d, int64_t k, int64_t* idx, double* val) {
    int64_t n = -1;
    int st = guarded([&] {
        SparseSelection s = topk_global(Vec(x, x + d), k);
        for (size_t j = 0; j < s.indices.size(); ++j) {
            idx[j] = s.indices[j];
            val[j] = s.values[j];
        }
        n = s.size();
    });
    return st ? -1 : n;
}

int64_t ref_per_block_k(int64_t dim, int64_t block, double density) {
    int64_t k = -1;
    guarded([&] { k = BlockLayout::from_density(dim, block, density).per_block_k; });
    return k;
}

int ref_encode(const double* x, int64_t d, int bits, int64_t bucket, uint8_t* codes, double* lo,
               double* hi, double* level) {
    return guarded([&] {
        auto b = QuantizedErrorBuffer::encode(Vec(x, x + d), bits, bucket);
        std::memcpy(codes, b.codes.data(), b.codes.size());
        for (size_t i = 0; i < b.params.size(); ++i) {
            lo[i] = b.params[i].lo;
            hi[i] = b.params[i].hi;
            level[i] = b.params[i].level;
        }
    });
}

int ref_decode(const uint8_t* codes, const double* lo, const double* hi, int64_t d, int bits,
               int64_t bucket, double* out) {
    return guarded([&] {
        auto b = QuantizedErrorBuffer::zeros(d, bits, bucket);
        std::memcpy(b.codes.data(), codes, b.codes.size());
        for (size_t i = 0; i < b.params.size(); ++i) b.params[i] = QuantParams(lo[i], hi[i], bits);
        Vec e = b.decode();
        std::memcpy(out, e.data(), e.size() * sizeof(double));
    });
}

// GradientWindow fed explicit rows, then adam_stats (window.cpp:14-46).
int ref_adam_stats(int64_t dim, int64_t m, int64_t row_width, int64_t nrows, const int64_t* idx,
                   const double* val, double beta, int square, double* z) {
    return guarded([&] {
        GradientWindow w(dim, m, row_width);
        for (int64_t r = 0; r < nrows; ++r) {
            SparseSelection s;
            s.dim = dim;
            s.indices.assign(idx + r * row_width, idx + (r + 1) * row_width);
            s.values.assign(val + r * row_width, val + (r + 1) * row_width);
            w.push(s);
        }
        Vec out = w.adam_stats(beta, square != 0);
        std::memcpy(z, out.data(), out.size() * sizeof(double));
    });
}

// ---- CPU baseline timing: the unmodified reference step, one optimizer per
// thread over a block-aligned shard (bit-identical to the unsharded run,
// SURVEY.md §0 fact 1). Gradients are the ma_synth stream rounded to
// grad_dtype. Returns the max over threads of the mean seconds per step.
double ref_time_shards(int nthreads, int64_t shard_dim, int64_t steps, int64_t warmup,
                       int grad_dtype, int64_t block, int64_t bucket, double density,
                       int64_t window, double* per_thread_s) {
    std::vector<double> secs(size_t(nthreads), 0.0);
    std::atomic<int> failed{0};
    std::vector<std::thread> ts;
    for (int t = 0; t < nthreads; ++t) {
        ts.emplace_back([&, t] {
            try {
                int64_t off = int64_t(t) * shard_dim;
                Vec th(static_cast<size_t>(shard_dim));
                for (int64_t i = 0; i < shard_dim; ++i)
                    th[size_t(i)] = round_dtype(ma_synth_normal(1, 0, uint64_t(off + i)), grad_dtype);
                HyperParams hp;
                hp.window = window;
                hp.density = density;
                hp.block = block;
                hp.bucket = bucket;
                MicroAdamOptimizer opt(std::move(th), hp, true, false);
                Vec g(static_cast<size_t>(shard_dim));
                double total = 0.0;
                for (int64_t s = 0; s < warmup + steps; ++s) {
                    for (int64_t i = 0; i < shard_dim; ++i)
                        g[size_t(i)] = round_dtype(
                            ma_synth_normal(42, uint64_t(s + 1), uint64_t(off + i)), grad_dtype);
                    auto t0 = std::chrono::steady_clock::now();
                    opt.step(g);
                    auto t1 = std::chrono::steady_clock::now();
                    if (s >= warmup) total += std::chrono::duration<double>(t1 - t0).count();
                }
                secs[size_t(t)] = total / double(steps > 0 ? steps : 1);
            } catch (...) {
                failed = 1;
            }
        });
    }
    for (auto& th : ts) th.join();
    if (failed) return -1.0;
    double mx = 0.0;
    for (int t = 0; t < nthreads; ++t) {
        if (per_thread_s) per_thread_s[t] = secs[size_t(t)];
        mx = secs[size_t(t)] > mx ? secs[size_t(t)] : mx;
    }
    return mx;
}

}  // extern "C"
