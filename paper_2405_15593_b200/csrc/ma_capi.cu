// ma_capi.cu — host side of libmicroadam_cuda: the C ABI declared in
// include/microadam_cuda.h. Owns the per-handle device state (EF codes,
// bucket grids, window ring), the host counters of the reference's
// GradientWindow (step/head/filled/stamps, window.hpp:10-33), the glibc
// pow() weights (window.cpp:37,43 — computed here, on the host, exactly as the
// reference does) and kernel launches. No exception crosses the ABI.
#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/microadam_cuda.h"
#include "ma_internal.h"

namespace {

thread_local std::string g_last_error;

ma_status fail(ma_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

ma_status cuda_fail(cudaError_t e, const char* where) {
    return fail(MA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define MA_CUDA(call)                                      \
    do {                                                   \
        cudaError_t _e = (call);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

size_t dtype_size(int dt) { return dt == MA_F64 ? 8 : (dt == MA_F32 ? 4 : 2); }

// Resolved shape of a (possibly sharded) configuration.
struct Shape {
    int64_t dim_global = 0;
    int64_t block = 0;       // min(hp.block, dim) (optim.cpp:140)
    int64_t per_block_k = 0; // compress.cpp:28-33
    int64_t nblocks_global = 0;
    int64_t b0 = 0, b1 = 0;  // owned block range
    int64_t elem0 = 0, dim = 0;
    int64_t row_width = 0;   // Σ_b∈[b0,b1) min(per_block_k, len_b)
    int64_t bucket = 0, nbuckets = 0, bucket0 = 0;
    int64_t code_bytes = 0;
    int64_t kb_stride = 0;
    bool global = false;     // global Top-K over d > kMaxBlock (ma_global.cu)
    bool split = false;      // blockwise with B_q not dividing B_d: per-bucket re-quantization kernel
    bool big = false;        // blockwise B_d in (8192, 32767]: ma_bigblock.cu (+ split re-quantization)
};

// HyperParams::validate (optim.cpp:7-21) — same checks, same order.
ma_status validate_hp(const ma_hyperparams& hp) {
    if (!(hp.beta1 > 0.0 && hp.beta1 < 1.0))
        return fail(MA_ERR_INVALID_ARG, "HyperParams: beta1 must be in (0,1)");
    if (!(hp.beta2 > 0.0 && hp.beta2 < 1.0))
        return fail(MA_ERR_INVALID_ARG, "HyperParams: beta2 must be in (0,1)");
    if (!(hp.eps > 0.0)) return fail(MA_ERR_INVALID_ARG, "HyperParams: eps must be > 0");
    if (!(hp.lr > 0.0)) return fail(MA_ERR_INVALID_ARG, "HyperParams: lr must be > 0");
    if (!(hp.weight_decay >= 0.0))
        return fail(MA_ERR_INVALID_ARG, "HyperParams: weight_decay must be >= 0");
    if (hp.window < 1) return fail(MA_ERR_INVALID_ARG, "HyperParams: window must be >= 1");
    if (!(hp.density > 0.0) || hp.density > 1.0)
        return fail(MA_ERR_INVALID_ARG, "HyperParams: density must be in (0,1]");
    if (hp.bits < 1 || hp.bits > 24)
        return fail(MA_ERR_INVALID_ARG, "HyperParams: bits must be in [1,24]");
    if (hp.block < 1 || hp.block > 32767)
        return fail(MA_ERR_INVALID_ARG, "HyperParams: block must be in [1, 32767]");
    if (hp.bucket < 1) return fail(MA_ERR_INVALID_ARG, "HyperParams: bucket must be >= 1");
    return MA_OK;
}

ma_status resolve_shape(const ma_config* cfg, int64_t dim, int64_t b0, int64_t b1, Shape* out) {
    if (!cfg || !out) return fail(MA_ERR_INVALID_ARG, "null argument");
    ma_status st = validate_hp(cfg->hp);
    if (st != MA_OK) return st;
    const ma_hyperparams& hp = cfg->hp;
    if (dim < 1) return fail(MA_ERR_INVALID_ARG, "MicroAdamOptimizer: empty parameter vector");
    if (hp.k > dim) return fail(MA_ERR_INVALID_ARG, "HyperParams: k exceeds dimension");
    for (int dt : {cfg->param_dtype, cfg->grad_dtype, cfg->value_dtype})
        if (dt < MA_F64 || dt > MA_BF16) return fail(MA_ERR_INVALID_ARG, "unknown dtype");
    if (cfg->finite_mode < MA_FINITE_FLAG || cfg->finite_mode > MA_FINITE_OFF)
        return fail(MA_ERR_INVALID_ARG, "unknown finite_mode");
    if (hp.window > ma::kMaxWindow) return fail(MA_ERR_UNSUPPORTED, "window > 1024 not supported on device");

    Shape s;
    s.dim_global = dim;
    if (cfg->blockwise) {
        // optim.cpp:137-144: density = k/d when k is set; block = min(block, d).
        const double density = hp.k > 0 ? static_cast<double>(hp.k) / static_cast<double>(dim)
                                        : hp.density;
        if (!(density > 0.0) || density > 1.0)
            return fail(MA_ERR_INVALID_ARG, "BlockLayout: density must be in (0, 1]");
        s.block = hp.block < dim ? hp.block : dim;
        int64_t k = static_cast<int64_t>(std::ceil(density * static_cast<double>(s.block)));
        s.per_block_k = k < s.block ? k : s.block;
        if (s.per_block_k < 1)
            return fail(MA_ERR_INVALID_ARG, "BlockLayout: per_block_k must be in [1, block]");
    } else {
        // Global Top-K (compress.cpp:66-71) == one block spanning d.
        s.block = dim;
        int64_t k = hp.k > 0 ? hp.k
                             : static_cast<int64_t>(std::ceil(hp.density * static_cast<double>(dim)));
        s.per_block_k = k < 1 ? 1 : (k > dim ? dim : k);
    }
    if (!cfg->blockwise && s.block > ma::kMaxBlock) {
        // Global Top-K over the whole vector (compress.cpp:66-71): ma_global.cu
        if (4096 % hp.bucket != 0)
            return fail(MA_ERR_UNSUPPORTED, "global mode on device needs bucket | 4096");
        if (b0 != 0 || (b1 >= 0 && b1 != 1))
            return fail(MA_ERR_UNSUPPORTED, "global mode cannot be block-sharded");
        if (hp.bits != 4) return fail(MA_ERR_UNSUPPORTED, "global mode on device implements bits = 4");
        if (hp.window > ma::kMaxWindowGlobal) return fail(MA_ERR_UNSUPPORTED, "global mode on device: window <= 256");
        s.global = true;
    } else if (s.block > ma::kMaxBlock) {
        if (s.block > ma::kMaxBlockBig) return fail(MA_ERR_UNSUPPORTED, "block > 32767 not supported on device");
        if (hp.bits != 4 || cfg->lossless_error)
            return fail(MA_ERR_UNSUPPORTED, "block > 8192: 4-bit quantized EF only on device");
        s.big = true;  // the big-block kernel; EF re-quantized per bucket (split mode)
    }
    s.nblocks_global = (dim + s.block - 1) / s.block;
    if (!s.global && (s.big || (s.nblocks_global > 1 && (s.block % hp.bucket != 0 || s.block % 2 != 0)))) {
        // Buckets straddle Top-K blocks (quantize.cpp:142-162 buckets the whole
        // vector): the step selects per block, then re-quantizes per bucket.
        if (hp.bits != 4 || cfg->lossless_error)
            return fail(MA_ERR_UNSUPPORTED, "bucket not dividing block: 4-bit quantized EF only on device");
        if (b0 != 0 || (b1 >= 0 && b1 != s.nblocks_global))
            return fail(MA_ERR_UNSUPPORTED, "bucket not dividing block: whole-vector handles only");
        s.split = true;
    }
    if (b1 < 0) b1 = s.nblocks_global;
    if (b0 < 0 || b0 >= b1 || b1 > s.nblocks_global)
        return fail(MA_ERR_INVALID_ARG, "shard block range out of bounds");
    s.b0 = b0;
    s.b1 = b1;
    s.elem0 = b0 * s.block;
    const int64_t elem1 = b1 * s.block < dim ? b1 * s.block : dim;
    s.dim = elem1 - s.elem0;
    s.row_width = 0;
    for (int64_t b = b0; b < b1; ++b) {
        const int64_t len = (b + 1) * s.block <= dim ? s.block : dim - b * s.block;
        s.row_width += s.per_block_k < len ? s.per_block_k : len;
    }
    s.bucket = hp.bucket;
    s.bucket0 = s.elem0 / hp.bucket;
    s.nbuckets = (s.dim + hp.bucket - 1) / hp.bucket;
    s.code_bytes = (s.dim * hp.bits + 7) / 8;
    if (hp.bits != 4 && s.nblocks_global > 1 && (s.block * hp.bits) % 8 != 0)
        return fail(MA_ERR_UNSUPPORTED, "bits != 4 needs block * bits to be a multiple of 8");
    if (hp.bits != 4 && (s.elem0 * hp.bits) % 8 != 0)
        return fail(MA_ERR_UNSUPPORTED, "bits != 4 shards must start on a byte boundary");
    s.kb_stride = (s.per_block_k + 7) / 8 * 8;
    *out = s;
    return MA_OK;
}

void fill_layout(const Shape& s, const ma_config& cfg, ma_layout_info* o) {
    o->dim = s.dim;
    o->block = s.block;
    o->per_block_k = s.per_block_k;
    o->num_blocks = s.b1 - s.b0;
    o->row_width = s.row_width;
    o->num_buckets = s.nbuckets;
    o->code_bytes = s.code_bytes;
    o->kb_stride = s.kb_stride;
    const int64_t went = o->num_blocks * cfg.hp.window * s.kb_stride;
    o->state_bytes = s.code_bytes + s.nbuckets * 16 + went * ((s.global ? 8 : 2) + int64_t(dtype_size(cfg.value_dtype)));
}

}  // namespace

struct ma_handle {
    ma_config cfg{};
    Shape shape;
    ma::Variant variant{};
    ma::Variant tail_variant{};  // generic kernel for the partial tail block (fast path)
    bool fast = false;  // ma_fast.cu / ma_warp.cu kernel (else the generic ma_kernels.cu kernel)
    bool warp = false;  // fast path runs the warp-per-block kernel (ma_warp.cu)
    bool warp_exact = false;  // MA_WARP_EXACT=1: never the fp32-screened (lean) warp kernel
    bool tile = false;  // ma_tile.cu kernel where it applies (MA_TILE=0: the warp kernels)
    int persist_grid = 0;
    int device = 0;
    uint8_t* d_codes = nullptr;
    double2* d_meta = nullptr;
    int16_t* d_win_idx = nullptr;
    void* d_win_val = nullptr;
    unsigned int* d_flag = nullptr;
    double* d_partials = nullptr;
    double* d_report = nullptr;
    uint32_t* d_thresh = nullptr;
    unsigned int* d_dbg = nullptr;  // diagnostics counters (MA_DEBUG_COUNTERS=1)
    // global Top-K mode buffers (ma_global.cu)
    double* g_level = nullptr;
    uint16_t* g_selbits = nullptr;
    uint32_t* g_hist = nullptr;
    int2* g_cnt = nullptr;
    int2* g_selinfo = nullptr;
    unsigned long long* g_selstate = nullptr;
    uint64_t* g_cand = nullptr;
    int64_t* g_cand_idx = nullptr;
    uint64_t* g_seg_key = nullptr;
    int64_t* g_seg_idx = nullptr;
    unsigned* g_seg_n = nullptr;
    int32_t* g_tiles = nullptr;
    bool g_bounds_valid = false;  // per-row chunk bounds of the global window (emit keeps the new row's)
    int32_t* g_ovf = nullptr;
    unsigned cand_cap = 0;
    int32_t* g_bounds = nullptr;
    double* d_dense = nullptr;  // lossless error feedback (fp64 residual, dim elements)
    // bucket-split mode: second codes buffer (swapped every step) + selection bits
    uint8_t* d_codes2 = nullptr;
    uint32_t* d_split_sel = nullptr;
    // host counters (window.hpp:10-33)
    int64_t step = 0, head = 0, filled = 0;
    std::vector<int64_t> stamps;
    // host path (ma_step_host)
    void* d_theta = nullptr;
    void* d_gstage = nullptr;
    // ma_step_host sparse θ return: window-entry θ values gathered on device,
    // brought back with the ring indices (pinned), scattered by host threads
    void* d_gath = nullptr;
    int16_t* h_ring_idx = nullptr;
    void* h_gath = nullptr;
    bool theta_valid = false;
    // host buffer known to equal the device θ (the last ma_step_host output);
    // the sparse θ return is only valid into that buffer
    const void* host_synced = nullptr;
    cudaStream_t host_stream = nullptr;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // ma_step_host copy streams
    cudaStream_t last_stream = nullptr;
    int64_t launches = 0;
    // sparse propagation: the step's kernel arguments between ma_step_front and ma_step_stats
    ma::StepArgs* pending = nullptr;
    // completion of the handle's last enqueued work (ma_sync and the readers
    // wait on it: stream-scoped, never a device-wide synchronize)
    cudaEvent_t done_ev = nullptr;
    // ma_step_host chunk events, created once and reused across calls
    std::vector<cudaEvent_t> host_ev;
    // ma_step_allgather with a report: the report sums are all-reduced over it
    const ma_comm* report_comm = nullptr;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void free_handle(ma_handle* h) {
    if (!h) return;
    DeviceGuard g(h->device);
    cudaFree(h->d_codes);
    cudaFree(h->d_meta);
    cudaFree(h->d_win_idx);
    cudaFree(h->d_win_val);
    cudaFree(h->d_flag);
    cudaFree(h->d_partials);
    cudaFree(h->d_report);
    cudaFree(h->d_thresh);
    cudaFree(h->d_dbg);
    cudaFree(h->d_theta);
    cudaFree(h->d_gstage);
    cudaFree(h->d_gath);
    if (h->h_ring_idx) cudaFreeHost(h->h_ring_idx);
    if (h->h_gath) cudaFreeHost(h->h_gath);
    cudaFree(h->g_level);
    cudaFree(h->g_selbits);
    cudaFree(h->g_hist);
    cudaFree(h->g_cnt);
    cudaFree(h->g_selinfo);
    cudaFree(h->g_selstate);
    cudaFree(h->g_cand);
    cudaFree(h->g_cand_idx);
    cudaFree(h->g_seg_key);
    cudaFree(h->g_seg_idx);
    cudaFree(h->g_seg_n);
    cudaFree(h->g_tiles);
    cudaFree(h->g_ovf);
    cudaFree(h->g_bounds);
    cudaFree(h->d_dense);
    cudaFree(h->d_codes2);
    cudaFree(h->d_split_sel);
    if (h->done_ev) cudaEventDestroy(h->done_ev);
    for (cudaEvent_t e : h->host_ev) cudaEventDestroy(e);
    if (h->host_stream) cudaStreamDestroy(h->host_stream);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h->pending;
    delete h;
}

constexpr unsigned kGlobalCandCap = 1u << 20;  // global radix select: keys kept after three digits

// Record the completion of everything the handle enqueued on `st`.
ma_status mark_done(ma_handle* h, cudaStream_t st) {
    if (!h->done_ev) MA_CUDA(cudaEventCreateWithFlags(&h->done_ev, cudaEventDisableTiming));
    MA_CUDA(cudaEventRecord(h->done_ev, st));
    h->last_stream = st;
    return MA_OK;
}
// Wait for the handle's last step (event-scoped: other streams and handles on
// the device keep running).
ma_status wait_done(ma_handle* h) {
    if (h->done_ev) MA_CUDA(cudaEventSynchronize(h->done_ev));
    return MA_OK;
}

// The host counters before a step: a step whose launch fails leaves the
// handle as it was (the reference throws before any mutation, optim.cpp:34-37).
struct CounterSnap {
    int64_t step, head, filled, stamp;
};
CounterSnap snap_counters(const ma_handle* h) {
    return CounterSnap{h->step, h->head, h->filled, h->stamps[size_t(h->head)]};
}
void restore_counters(ma_handle* h, const CounterSnap& c) {
    h->step = c.step;
    h->head = c.head;
    h->filled = c.filled;
    h->stamps[size_t(c.head)] = c.stamp;
}
#define MA_CUDA_ROLLBACK(h, snap, call)                     \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) {                            \
            restore_counters((h), (snap));                  \
            return cuda_fail(_e, #call);                    \
        }                                                   \
    } while (0)

// Advance the host counters exactly like GradientWindow::push (window.cpp:14-26)
// and build the kernel weights like adam_stats (window.cpp:28-46).
int64_t push_and_weights(ma_handle* h, ma::StepArgs* a) {
    const ma_hyperparams& hp = h->cfg.hp;
    const int64_t slot = h->head;
    ++h->step;
    h->stamps[size_t(slot)] = h->step;
    h->head = (h->head + 1) % hp.window;
    h->filled = h->step < hp.window ? h->step : hp.window;
    for (int64_t r = 0; r < h->filled; ++r) {
        // Rows with stamp 0 are skipped by the reference (window.cpp:33); with
        // rows written in slot order every r < filled has a stamp.
        a->w1[r] = std::pow(hp.beta1, static_cast<double>(h->step - h->stamps[size_t(r)]));
        a->w2[r] = std::pow(hp.beta2, static_cast<double>(h->step - h->stamps[size_t(r)]));
    }
    a->scale1 = (1.0 - hp.beta1) / (1.0 - std::pow(hp.beta1, static_cast<double>(h->step)));
    a->scale2 = (1.0 - hp.beta2) / (1.0 - std::pow(hp.beta2, static_cast<double>(h->step)));
    for (int64_t r = 0; r < h->filled; ++r) {
        a->c1[r] = static_cast<float>(a->w1[r] * a->scale1);
        a->c2[r] = static_cast<float>(std::sqrt(a->w2[r] * a->scale2));
    }
    a->eps32 = static_cast<float>(hp.eps);
    a->filled = static_cast<int32_t>(h->filled);
    a->slot = static_cast<int32_t>(slot);
    return slot;
}

void base_args(ma_handle* h, ma::StepArgs* a) {
    std::memset(a, 0, sizeof(*a));
    const Shape& s = h->shape;
    a->codes = h->d_codes;
    a->meta = h->d_meta;
    a->win_idx = h->d_win_idx;
    a->win_val = h->d_win_val;
    a->flag = h->d_flag;
    a->thresh = h->d_thresh;
    a->dbg = h->d_dbg;
    a->dim = s.dim;
    a->num_blocks = s.b1 - s.b0;
    a->block = static_cast<int32_t>(s.block);
    a->per_block_k = static_cast<int32_t>(s.per_block_k);
    a->kb_stride = static_cast<int32_t>(s.kb_stride);
    a->bucket = static_cast<int32_t>(s.bucket);
    a->m = static_cast<int32_t>(h->cfg.hp.window);
    a->check_finite = h->cfg.finite_mode == MA_FINITE_FLAG ? 1 : 0;
    a->g_dtype = h->cfg.grad_dtype;
    a->p_dtype = h->cfg.param_dtype;
    a->v_dtype = h->cfg.value_dtype;
    a->eps = h->cfg.hp.eps;
    a->force_exact = h->warp_exact ? 1 : 0;
    a->dense = h->d_dense;
    a->split_sel = h->shape.split ? h->d_split_sel : nullptr;
    a->bits = static_cast<int32_t>(h->cfg.hp.bits);
}

// Fast path: the persistent kernel takes the range's full blocks and the
// generic kernel the shard's partial tail block (if it is in the range).
cudaError_t launch(ma_handle* h, ma::StepArgs& a, int64_t nblocks, cudaStream_t st) {
    if (h->shape.big) return ma::launch_step_big(a, nblocks, st);
    if (!h->fast) return ma::launch_step(a, h->variant, nblocks, st);
    const Shape& s = h->shape;
    const int64_t nb_shard = s.b1 - s.b0;
    const bool tail_partial = (s.dim % s.block) != 0 && a.block_offset + nblocks == nb_shard;
    const int64_t nfull = nblocks - (tail_partial ? 1 : 0);
    if (nfull > 0) {
        a.block_count = nfull;
        const int64_t grid = std::min<int64_t>(nfull, h->persist_grid);
        cudaError_t e = (h->tile && ma::tile_ok(a))               ? ma::launch_step_tile(a, st)
                        : (h->warp && ma::warp_can_run(a)) ? ma::launch_step_warp(a, st)
                                                           : ma::launch_step_fast(a, h->variant, int(grid), st);
        if (e != cudaSuccess) return e;
    }
    if (tail_partial) {
        ma::StepArgs t = a;
        t.block_offset = a.block_offset + nfull;
        t.block_count = 1;
        ++h->launches;
        return ma::launch_step(t, h->tail_variant, 1, st);
    }
    return cudaSuccess;
}

ma_status allreduce_report(ma_handle* h, cudaStream_t st);  // after struct ma_comm (below)

ma_status finish_report(ma_handle* h, cudaStream_t st, ma_step_report* report) {
    MA_CUDA(ma::launch_report_reduce(h->d_partials, h->shape.b1 - h->shape.b0, h->d_report, st));
    ++h->launches;
    if (h->report_comm) {  // ma_step_allgather: the five sums over all ranks' shards
        ma_status rs = allreduce_report(h, st);
        if (rs != MA_OK) return rs;
    }
    double r[ma::kReportFields];
    MA_CUDA(cudaMemcpyAsync(r, h->d_report, sizeof(r), cudaMemcpyDeviceToHost, st));
    MA_CUDA(cudaStreamSynchronize(st));
    const double na = std::sqrt(r[1]);
    report->grad_norm = std::sqrt(r[0]);
    report->empirical_q = na > 0.0 ? std::sqrt(r[2]) / na : 0.0;
    report->error_norm = std::sqrt(r[3]);
    report->update_nnz = static_cast<int64_t>(r[4]);
    report->loss = 0.0;
    return MA_OK;
}

ma_status strict_prescan(ma_handle* h, const void* d_grads, cudaStream_t st) {
    MA_CUDA(cudaMemsetAsync(h->d_flag, 0, sizeof(unsigned), st));
    MA_CUDA(ma::launch_finite_scan(d_grads, h->cfg.grad_dtype, h->shape.dim, h->d_flag, st));
    ++h->launches;
    if (h->cfg.grad_dtype == MA_F64 && h->step > 0) {
        // a = g + e can overflow only for f64 gradients (bf16/f32 g plus an EF
        // bounded by earlier finite a stays finite in fp64)
        MA_CUDA(ma::launch_finite_scan_a(static_cast<const double*>(d_grads), h->d_codes, h->d_meta, h->d_dense,
                                         h->shape.dim, h->shape.bucket, int(h->cfg.hp.bits), h->d_flag, st));
        ++h->launches;
    }
    unsigned flag = 0;
    MA_CUDA(cudaMemcpyAsync(&flag, h->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, st));
    MA_CUDA(cudaStreamSynchronize(st));
    if (flag) {
        const unsigned zero = 0;
        MA_CUDA(cudaMemcpy(h->d_flag, &zero, sizeof(zero), cudaMemcpyHostToDevice));
        return fail(MA_ERR_NONFINITE, "step gradient: non-finite entry");
    }
    return MA_OK;
}

// Global Top-K step (ma_global.cu): host-driven radix select of the k-th
// largest |a| key, then emit / re-quantize / ADAM_STATS / update kernels.
ma_status run_step_global(ma_handle* h, void* d_params, const void* d_grads, double lr, cudaStream_t st,
                          ma_step_report* report) {
    const Shape& s = h->shape;
    ma::StepArgs a;
    base_args(h, &a);
    const CounterSnap snap = snap_counters(h);
    push_and_weights(h, &a);
    ma::GlobalArgs g{};
    g.grads = d_grads;
    g.params = d_params;
    g.codes = h->d_codes;
    g.meta = h->d_meta;
    g.level = h->g_level;
    g.win_idx = reinterpret_cast<int64_t*>(h->d_win_idx);
    g.win_val = h->d_win_val;
    g.selbits = h->g_selbits;
    g.hist = h->g_hist;
    g.cnt = h->g_cnt;
    g.sel_info = h->g_selinfo;
    g.sel_state = h->g_selstate;
    g.cand = h->g_cand;
    g.cand_idx = h->g_cand_idx;
    g.seg_key = h->g_seg_key;
    g.seg_idx = h->g_seg_idx;
    g.seg_n = h->g_seg_n;
    g.tiles = h->g_tiles;
    g.cand_n = reinterpret_cast<unsigned int*>(h->g_selstate + 3);
    g.cand_cap = h->cand_cap;
    g.ovf_list = h->g_ovf;
    g.ovf_n = reinterpret_cast<unsigned int*>(h->g_selstate + 4);
    g.bounds = h->g_bounds;
    g.partials = report ? h->d_partials : nullptr;
    g.flag = h->d_flag;
    g.dense = h->d_dense;
    g.dim = s.dim;
    g.nbuckets = s.nbuckets;
    g.bucket = s.bucket;
    g.bucket_shift = 0;
    while ((int64_t(1) << g.bucket_shift) < s.bucket) ++g.bucket_shift;
    g.k = s.per_block_k;
    g.row_stride = s.kb_stride;
    g.slot = a.slot;
    g.g_dtype = h->cfg.grad_dtype;
    g.p_dtype = h->cfg.param_dtype;
    g.v_dtype = h->cfg.value_dtype;
    g.check_finite = a.check_finite;
    g.eps = a.eps;
    g.lr = lr;
    g.scale1 = a.scale1;
    g.scale2 = a.scale2;
    MA_CUDA_ROLLBACK(h, snap, ma::g_launch_levels(g, st));
    // G1-G2 entirely on the device: the six radix digits are picked by a
    // one-warp kernel after each histogram, row offsets / ties per chunk by a
    // one-CTA scan — the step never waits for the host.
    MA_CUDA(ma::g_launch_select(g, st));
    MA_CUDA(ma::g_launch_count(g, st));
    h->launches += 31;  // levels, select (init, bracket 2 x 3 + compact, 6 x (hist, hist_cand, pick), next), count x3
    MA_CUDA(ma::g_launch_emit(g, st));
    MA_CUDA(ma::g_launch_requant(g, st));
    ma::GWeights w;
    for (int64_t r = 0; r < h->filled; ++r) {
        w.w1[r] = a.w1[r];
        w.w2[r] = a.w2[r];
    }
    MA_CUDA(ma::g_launch_stats_update(g, w, int(h->filled), !h->g_bounds_valid, st));
    h->launches += (ma::global_fused_emit(g) ? 3 : 4) + (h->g_bounds_valid ? 0 : 1);
    h->g_bounds_valid = true;
    ma_status ms = mark_done(h, st);
    if (ms != MA_OK) return ms;
    if (report) {
        MA_CUDA(ma::launch_report_reduce(h->d_partials, ma::global_chunks(s.dim), h->d_report, st));
        ++h->launches;
        double r[ma::kReportFields];
        MA_CUDA(cudaMemcpyAsync(r, h->d_report, sizeof(r), cudaMemcpyDeviceToHost, st));
        MA_CUDA(cudaStreamSynchronize(st));
        const double na = std::sqrt(r[1]);
        report->grad_norm = std::sqrt(r[0]);
        report->empirical_q = na > 0.0 ? std::sqrt(r[2]) / na : 0.0;
        report->error_norm = std::sqrt(r[3]);
        report->update_nnz = static_cast<int64_t>(r[4]);
        report->loss = 0.0;
    }
    return MA_OK;
}

ma_status run_step(ma_handle* h, void* d_params, const void* d_grads, double lr, cudaStream_t st,
                   ma_step_report* report) {
    if (!(lr > 0.0)) return fail(MA_ERR_INVALID_ARG, "step: lr must be > 0");
    if (!d_params || !d_grads) return fail(MA_ERR_INVALID_ARG, "step: null buffer");
    if (h->cfg.finite_mode == MA_FINITE_STRICT) {
        ma_status s = strict_prescan(h, d_grads, st);
        if (s != MA_OK) return s;
    }
    if (h->shape.global) return run_step_global(h, d_params, d_grads, lr, st, report);
    ma::StepArgs a;
    base_args(h, &a);
    a.grads = d_grads;
    a.params = d_params;
    a.lr = lr;
    a.lr32 = static_cast<float>(lr);
    a.partials = report ? h->d_partials : nullptr;
    const CounterSnap snap = snap_counters(h);
    const Shape& s = h->shape;
    if (s.split) {
        MA_CUDA(cudaMemsetAsync(h->d_split_sel, 0, size_t((s.dim + 31) / 32) * 4, st));
        MA_CUDA(cudaMemsetAsync(h->d_codes2, 0, size_t(s.code_bytes + 3) / 4 * 4, st));
    }
    push_and_weights(h, &a);
    MA_CUDA_ROLLBACK(h, snap, launch(h, a, s.b1 - s.b0, st));
    ++h->launches;
    if (s.split) {  // per-bucket re-quantization from the old codes into the second buffer
        MA_CUDA_ROLLBACK(h, snap, ma::launch_requant_buckets(d_grads, h->cfg.grad_dtype, h->d_codes, h->d_codes2,
                                                             h->d_meta, h->d_split_sel, s.dim, s.bucket,
                                                             report ? h->d_partials + 3 : nullptr, st));
        ++h->launches;
        std::swap(h->d_codes, h->d_codes2);
    }
    ma_status ms = mark_done(h, st);
    if (ms != MA_OK) return ms;
    if (report) return finish_report(h, st, report);
    return MA_OK;
}

}  // namespace

extern "C" {

void ma_config_default(ma_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->hp.beta1 = 0.9;
    cfg->hp.beta2 = 0.999;
    cfg->hp.eps = 1e-8;
    cfg->hp.lr = 1e-3;
    cfg->hp.weight_decay = 0.0;
    cfg->hp.window = 10;
    cfg->hp.density = 0.01;
    cfg->hp.k = 0;
    cfg->hp.bits = 4;
    cfg->hp.block = 4096;
    cfg->hp.bucket = 64;
    cfg->blockwise = 1;
    cfg->lossless_error = 0;
    cfg->param_dtype = MA_F32;
    cfg->grad_dtype = MA_F32;
    cfg->value_dtype = MA_BF16;
    cfg->finite_mode = MA_FINITE_FLAG;
}

ma_status ma_validate(const ma_config* cfg, int64_t dim) {
    Shape s;
    return resolve_shape(cfg, dim, 0, -1, &s);
}

ma_status ma_layout(const ma_config* cfg, int64_t dim, int64_t block_begin, int64_t block_end,
                    ma_layout_info* out) {
    Shape s;
    ma_status st = resolve_shape(cfg, dim, block_begin, block_end, &s);
    if (st != MA_OK) return st;
    if (!out) return fail(MA_ERR_INVALID_ARG, "null out");
    fill_layout(s, *cfg, out);
    return MA_OK;
}

ma_status ma_create_shard(const ma_config* cfg, int64_t dim, int64_t block_begin,
                          int64_t block_end, int device, ma_handle** out) {
    if (!out) return fail(MA_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    Shape s;
    ma_status st = resolve_shape(cfg, dim, block_begin, block_end, &s);
    if (st != MA_OK) return st;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MA_ERR_CUDA, "no CUDA device visible (the device path has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(MA_ERR_INVALID_ARG, "device out of range");
    DeviceGuard g(device);
    ma_handle* h = new (std::nothrow) ma_handle();
    if (!h) return fail(MA_ERR_INVALID_ARG, "out of host memory");
    h->cfg = *cfg;
    h->shape = s;
    h->device = device;
    h->stamps.assign(size_t(cfg->hp.window), 0);
    const int64_t nb = s.b1 - s.b0;
    const size_t went = size_t(nb) * size_t(cfg->hp.window) * size_t(s.kb_stride);
    int smem_max = 0;
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const char* force_generic = std::getenv("MA_FORCE_GENERIC");
    // global Top-K handles (block = d, possibly >= 2^31) never use these kernels
    const int blk_i = s.global ? 4096 : int(s.block);
    const ma::Variant fv = ma::pick_fast_variant(blk_i, int(s.bucket), int(cfg->hp.window),
                                                 int(s.kb_stride), cfg->grad_dtype,
                                                 cfg->param_dtype, cfg->value_dtype);
    h->tail_variant = ma::pick_variant(blk_i);
    // the generic kernel's shared memory (needed for a partial tail block or when
    // no other kernel runs this shape)
    const size_t generic_smem = ma::step_smem_bytes(h->tail_variant.nt, h->tail_variant.ept, blk_i, int(s.bucket),
                                                    int(cfg->hp.window), int(s.kb_stride), int(cfg->hp.bits));
    size_t smem = 0;
    const bool no_generic_env = !(force_generic && force_generic[0] == '1');
    if (fv.nt && no_generic_env) {
        const size_t fs = ma::fast_smem_bytes(fv, blk_i, int(s.bucket), int(cfg->hp.window),
                                              int(s.kb_stride), cfg->grad_dtype, cfg->param_dtype,
                                              cfg->value_dtype);
        const int per_sm = fs <= size_t(smem_max) ? ma::fast_blocks_per_sm(fv, int(s.bucket), fs) : 0;
        if (per_sm > 0) {
            int nsm = 0;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
            h->variant = fv;
            h->fast = true;
            h->persist_grid = per_sm * nsm;
            smem = std::max(smem, fs);
        }
    }
    const char* force_cta = std::getenv("MA_FAST_CTA");  // A/B: the CTA-per-block fast kernel
    const bool warp_ok = !(force_cta && force_cta[0] == '1') &&
                         ma::warp_path_ok(blk_i, int(s.bucket), int(s.per_block_k), int(cfg->hp.window),
                                          int(s.kb_stride), cfg->grad_dtype, cfg->param_dtype, cfg->value_dtype) &&
                         ma::warp_smem_bytes(int(s.bucket)) <= size_t(smem_max);
    if (h->fast && warp_ok) h->warp = true;
    // long windows (m * k_b beyond the CTA kernel's staging): the warp kernels alone
    // (the exact one reads the rows from global memory; k_b <= 64)
    if (!h->fast && no_generic_env && warp_ok && s.per_block_k <= 64) {
        h->fast = h->warp = true;
        h->variant = h->tail_variant;
    }
    const char* warp_exact = std::getenv("MA_WARP_EXACT");
    h->warp_exact = warp_exact && warp_exact[0] == '1';
    // MA_TILE=1: the TMA-fed CTA-per-block kernel (ma_tile.cu) where it applies;
    // the lean warp kernel stays the default (faster on B200)
    const char* tile_env = std::getenv("MA_TILE");
    h->tile = h->warp && !h->warp_exact && tile_env && tile_env[0] == '1';
    if (!h->fast) h->variant = h->tail_variant;
    if (s.global) {
        h->fast = h->warp = h->tile = false;
        smem = ma::global_requant_smem(s.bucket);
    }
    if (cfg->lossless_error || cfg->hp.bits != 4 || s.split) {  // dense EF / other widths / split: generic kernel
        h->fast = h->warp = h->tile = false;
        h->variant = h->tail_variant;
    }
    const bool tail_block = !s.global && (s.dim % s.block) != 0 && s.b1 == s.nblocks_global;
    if (s.big) {
        h->fast = h->warp = h->tile = false;
        smem = ma::big_block_smem_bytes(int(s.block), int(cfg->hp.window), int(s.kb_stride));
    } else if (!s.global && (!h->fast || tail_block)) {
        smem = std::max(smem, generic_smem);
    }
    if (smem > size_t(smem_max)) {
        delete h;
        return fail(MA_ERR_UNSUPPORTED, "block/window shape needs more shared memory than one SM has");
    }
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void** p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(p, bytes ? bytes : 16);
        if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes ? bytes : 16);
    };
    alloc(reinterpret_cast<void**>(&h->d_codes), size_t(s.code_bytes + 3) / 4 * 4);
    if (s.split) {
        alloc(reinterpret_cast<void**>(&h->d_codes2), size_t(s.code_bytes + 3) / 4 * 4);
        alloc(reinterpret_cast<void**>(&h->d_split_sel), size_t((s.dim + 31) / 32) * 4);
    }
    alloc(reinterpret_cast<void**>(&h->d_meta), size_t(s.nbuckets) * sizeof(double2));
    alloc(reinterpret_cast<void**>(&h->d_win_idx), went * (s.global ? sizeof(int64_t) : sizeof(int16_t)));
    if (s.global) {
        const int64_t nch = ma::global_chunks(s.dim);
        alloc(reinterpret_cast<void**>(&h->g_level), size_t(s.nbuckets) * sizeof(double));
        alloc(reinterpret_cast<void**>(&h->g_selbits), size_t(nch) * 256 * sizeof(uint16_t));
        alloc(reinterpret_cast<void**>(&h->g_hist), 2048 * sizeof(uint32_t));
        alloc(reinterpret_cast<void**>(&h->g_cnt), size_t(nch) * sizeof(int2));
        alloc(reinterpret_cast<void**>(&h->g_selinfo), size_t(nch) * sizeof(int2));
        alloc(reinterpret_cast<void**>(&h->g_selstate), 16 * sizeof(unsigned long long));
        alloc(reinterpret_cast<void**>(&h->g_ovf), size_t(nch) * sizeof(int32_t));
        // MA_GLOBAL_CAND_CAP (tests): a small capacity forces the overflow path
        const char* cc = std::getenv("MA_GLOBAL_CAND_CAP");
        // default: d / 128 keys (the carried bracket's collection), 1M..64M
        const int64_t cap_d = std::min<int64_t>(int64_t(64) << 20, std::max<int64_t>(kGlobalCandCap, s.dim / 128));
        h->cand_cap = cc ? static_cast<unsigned>(std::strtoul(cc, nullptr, 10)) : static_cast<unsigned>(cap_d);
        alloc(reinterpret_cast<void**>(&h->g_cand), size_t(h->cand_cap) * sizeof(uint64_t));
        alloc(reinterpret_cast<void**>(&h->g_cand_idx), size_t(h->cand_cap) * sizeof(int64_t));
        alloc(reinterpret_cast<void**>(&h->g_seg_key), size_t(h->cand_cap) * sizeof(uint64_t));
        alloc(reinterpret_cast<void**>(&h->g_seg_idx), size_t(h->cand_cap) * sizeof(int64_t));
        alloc(reinterpret_cast<void**>(&h->g_seg_n), size_t(ma::kBracketCtas) * sizeof(unsigned));
        alloc(reinterpret_cast<void**>(&h->g_tiles), size_t(nch / 1024 + 1) * 4 * sizeof(int32_t));
        alloc(reinterpret_cast<void**>(&h->g_bounds), size_t(cfg->hp.window) * size_t(nch + 1) * sizeof(int32_t));
    }
    alloc(&h->d_win_val, went * dtype_size(cfg->value_dtype));
    alloc(reinterpret_cast<void**>(&h->d_flag), sizeof(unsigned));
    if (cfg->lossless_error) alloc(reinterpret_cast<void**>(&h->d_dense), size_t(s.dim) * sizeof(double));
    alloc(reinterpret_cast<void**>(&h->d_partials),
          size_t(s.global ? ma::global_chunks(s.dim) : nb) * ma::kReportFields * sizeof(double));
    alloc(reinterpret_cast<void**>(&h->d_report), ma::kReportFields * sizeof(double));
    alloc(reinterpret_cast<void**>(&h->d_thresh), size_t(nb) * sizeof(uint32_t));
    const char* dbg = std::getenv("MA_DEBUG_COUNTERS");
    if (dbg && dbg[0] == '1') alloc(reinterpret_cast<void**>(&h->d_dbg), 32 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        free_handle(h);
        return cuda_fail(e, "ma_create");
    }
    *out = h;
    return MA_OK;
}

ma_status ma_create(const ma_config* cfg, int64_t dim, int device, ma_handle** out) {
    return ma_create_shard(cfg, dim, 0, -1, device, out);
}

ma_status ma_destroy(ma_handle* h) {
    free_handle(h);
    return MA_OK;
}

ma_status ma_step(ma_handle* h, void* d_params, const void* d_grads, double lr, void* stream,
                  ma_step_report* report) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    DeviceGuard g(h->device);
    return run_step(h, d_params, d_grads, lr, static_cast<cudaStream_t>(stream), report);
}

ma_status ma_step_reduce(ma_handle* h, void* d_params, void* d_grads, const void* const* d_srcs, int32_t nsrc,
                         float scale, double lr, void* stream, ma_step_report* report) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (!d_srcs || nsrc < 1 || nsrc > ma::kMaxRanks)
        return fail(MA_ERR_INVALID_ARG, "step_reduce: nsrc must be in [1, 8]");
    for (int r = 0; r < nsrc; ++r)
        if (!d_srcs[r]) return fail(MA_ERR_INVALID_ARG, "step_reduce: null gradient source");
    if (!(lr > 0.0)) return fail(MA_ERR_INVALID_ARG, "step: lr must be > 0");
    if (!d_params || !d_grads) return fail(MA_ERR_INVALID_ARG, "step: null buffer");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Shape& s = h->shape;
    ma::StepArgs a;
    base_args(h, &a);
    a.rs_n = nsrc;
    a.rs_scale = scale;
    for (int r = 0; r < nsrc; ++r) a.rs_src[r] = d_srcs[r];
    const char* env = std::getenv("MA_RS_UNFUSED");
    const bool fused = h->fast && h->warp && !s.global && h->cfg.finite_mode != MA_FINITE_STRICT && !report &&
                       !(env && env[0] == '1') && ma::lean_rs_ok(a);
    if (!fused) {  // reduce into d_grads, then the ordinary step
        MA_CUDA(ma::launch_reduce_grads(d_srcs, nsrc, scale, h->cfg.grad_dtype, d_grads, 0, s.dim, st));
        ++h->launches;
        return run_step(h, d_params, d_grads, lr, st, report);
    }
    // The lean kernel reduces its full blocks itself; the partial tail block
    // (generic kernel, launched after it) is reduced up front.
    if (s.dim % s.block) {
        MA_CUDA(ma::launch_reduce_grads(d_srcs, nsrc, scale, h->cfg.grad_dtype, d_grads, (s.dim / s.block) * s.block,
                                        s.dim, st));
        ++h->launches;
    }
    a.grads = d_grads;
    a.params = d_params;
    a.lr = lr;
    a.lr32 = static_cast<float>(lr);
    const CounterSnap snap = snap_counters(h);
    push_and_weights(h, &a);
    MA_CUDA_ROLLBACK(h, snap, launch(h, a, s.b1 - s.b0, st));
    ++h->launches;
    return mark_done(h, st);
}

ma_status ma_set_params(ma_handle* h, const void* h_params) {
    if (!h || !h_params) return fail(MA_ERR_INVALID_ARG, "null argument");
    DeviceGuard g(h->device);
    const size_t pbytes = size_t(h->shape.dim) * dtype_size(h->cfg.param_dtype);
    if (!h->d_theta) MA_CUDA(cudaMalloc(&h->d_theta, pbytes));
    MA_CUDA(cudaMemcpy(h->d_theta, h_params, pbytes, cudaMemcpyHostToDevice));
    h->theta_valid = true;
    h->host_synced = h_params;
    return MA_OK;
}

ma_status ma_step_host(ma_handle* h, void* h_params, const void* h_grads, double lr,
                       ma_step_report* report) {
    if (!h || !h_params || !h_grads) return fail(MA_ERR_INVALID_ARG, "null argument");
    DeviceGuard g(h->device);
    const Shape& s = h->shape;
    const size_t gsz = dtype_size(h->cfg.grad_dtype), psz = dtype_size(h->cfg.param_dtype);
    if (!h->host_stream) MA_CUDA(cudaStreamCreateWithFlags(&h->host_stream, cudaStreamNonBlocking));
    if (!h->d_gstage) MA_CUDA(cudaMalloc(&h->d_gstage, size_t(s.dim) * gsz));
    if (!h->theta_valid) {
        ma_status st = ma_set_params(h, h_params);
        if (st != MA_OK) return st;
    }
    cudaStream_t st = h->host_stream;
    if (h->cfg.finite_mode == MA_FINITE_STRICT || report || s.global || s.split) {
        // Whole-vector path: strict pre-scan / report need the full gradient;
        // global Top-K (ma_global.cu) selects over the whole vector at once.
        MA_CUDA(cudaMemcpyAsync(h->d_gstage, h_grads, size_t(s.dim) * gsz, cudaMemcpyHostToDevice, st));
        ma_status r = run_step(h, h->d_theta, h->d_gstage, lr, st, report);
        if (r != MA_OK) return r;
        MA_CUDA(cudaMemcpyAsync(h_params, h->d_theta, size_t(s.dim) * psz, cudaMemcpyDeviceToHost, st));
        MA_CUDA(cudaStreamSynchronize(st));
        h->host_synced = h_params;
        return ma_sync(h);
    }
    // Chunked pipeline: H2D grads of chunk c+1 overlaps the step of chunk c
    // and the return of θ for chunk c-1 (two copy engines + SMs busy at once).
    // θ changes only at window coordinates (optim.cpp:183-187: u = 0 off the
    // window), so with MA_HOST_SPARSE=1 the return is sparse: the window ring
    // indices and the θ values gathered at them (4 bytes per window entry
    // against 2 per parameter for bf16 θ), scattered into h_params by host
    // threads as each chunk lands. Off by default: the scatter still touches
    // nearly every cache line of host θ and on a 16-core host costs more than
    // the dense D2H it replaces (7B: 314 vs 291 ms per call).
    ma::StepArgs a;
    base_args(h, &a);
    a.grads = h->d_gstage;
    a.params = h->d_theta;
    a.lr = lr;
    a.lr32 = static_cast<float>(lr);
    const CounterSnap snap = snap_counters(h);
    push_and_weights(h, &a);
    const int64_t nb = s.b1 - s.b0;
    const int64_t m = h->cfg.hp.window, kbs = s.kb_stride;
    const char* sparse_env = std::getenv("MA_HOST_SPARSE");
    const bool sparse_ret =
        !s.global && h->host_synced == h_params && sparse_env && sparse_env[0] == '1';
    const size_t ring_n = size_t(nb) * size_t(m) * size_t(kbs);
    if (sparse_ret && !h->d_gath) {
        MA_CUDA(cudaMalloc(&h->d_gath, ring_n * psz));
        MA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->h_ring_idx), ring_n * sizeof(int16_t)));
        MA_CUDA(cudaMallocHost(&h->h_gath, ring_n * psz));
    }
    const int64_t chunk_blocks = std::max<int64_t>(1, (int64_t(64) << 20) / (s.block * int64_t(gsz)));
    const int64_t nchunks = (nb + chunk_blocks - 1) / chunk_blocks;
    // chunk events: created on the first call, reused afterwards
    while (h->host_ev.size() < size_t(3 * nchunks)) {
        cudaEvent_t e = nullptr;
        MA_CUDA_ROLLBACK(h, snap, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->host_ev.push_back(e);
    }
    cudaEvent_t* up = h->host_ev.data();
    cudaEvent_t* done = up + nchunks;
    cudaEvent_t* back = done + nchunks;
    if (!h->s_h2d) MA_CUDA_ROLLBACK(h, snap, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    if (!h->s_d2h) MA_CUDA_ROLLBACK(h, snap, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    cudaStream_t s_h2d = h->s_h2d, s_d2h = h->s_d2h;
    const int filled = static_cast<int>(h->filled);
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t cb0 = c * chunk_blocks, cb1 = std::min(nb, cb0 + chunk_blocks);
        const int64_t e0 = cb0 * s.block, e1 = std::min(s.dim, cb1 * s.block);
        MA_CUDA(cudaMemcpyAsync(static_cast<char*>(h->d_gstage) + e0 * gsz,
                                static_cast<const char*>(h_grads) + e0 * gsz, size_t(e1 - e0) * gsz,
                                cudaMemcpyHostToDevice, s_h2d));
        MA_CUDA(cudaEventRecord(up[size_t(c)], s_h2d));
        MA_CUDA(cudaStreamWaitEvent(st, up[size_t(c)], 0));
        a.block_offset = cb0;
        if (c == 0) MA_CUDA_ROLLBACK(h, snap, launch(h, a, cb1 - cb0, st));  // nothing mutated yet
        else MA_CUDA(launch(h, a, cb1 - cb0, st));
        ++h->launches;
        if (sparse_ret) {
            MA_CUDA(ma::launch_gather_window_theta(h->d_win_idx, h->d_theta, h->cfg.param_dtype, h->d_gath, cb0, cb1,
                                                   int(m), int(kbs), int(s.per_block_k), filled, s.block, s.dim, st));
            ++h->launches;
        }
        MA_CUDA(cudaEventRecord(done[size_t(c)], st));
        MA_CUDA(cudaStreamWaitEvent(s_d2h, done[size_t(c)], 0));
        if (sparse_ret) {
            const size_t q0 = size_t(cb0) * size_t(m * kbs), qn = size_t(cb1 - cb0) * size_t(m * kbs);
            MA_CUDA(cudaMemcpyAsync(h->h_ring_idx + q0, h->d_win_idx + q0, qn * sizeof(int16_t),
                                    cudaMemcpyDeviceToHost, s_d2h));
            MA_CUDA(cudaMemcpyAsync(static_cast<char*>(h->h_gath) + q0 * psz,
                                    static_cast<const char*>(h->d_gath) + q0 * psz, qn * psz,
                                    cudaMemcpyDeviceToHost, s_d2h));
        } else {
            MA_CUDA(cudaMemcpyAsync(static_cast<char*>(h_params) + e0 * psz,
                                    static_cast<const char*>(h->d_theta) + e0 * psz,
                                    size_t(e1 - e0) * psz, cudaMemcpyDeviceToHost, s_d2h));
        }
        MA_CUDA(cudaEventRecord(back[size_t(c)], s_d2h));
    }
    if (sparse_ret) {
        // host scatter: h_params[block base + idx] = θ for every live window entry
        std::atomic<int64_t> next{0};
        std::atomic<int> err{0};
        const int nthreads = static_cast<int>(std::max<unsigned>(1, std::min<unsigned>(32, std::thread::hardware_concurrency())));
        auto worker = [&]() {
            for (;;) {
                const int64_t c = next.fetch_add(1);
                if (c >= nchunks) return;
                if (cudaEventSynchronize(back[size_t(c)]) != cudaSuccess) {
                    err = 1;
                    return;
                }
                const int64_t cb0 = c * chunk_blocks, cb1 = std::min(nb, cb0 + chunk_blocks);
                for (int64_t b = cb0; b < cb1; ++b) {
                    const int64_t base = b * s.block;
                    const int64_t len = std::min(s.block, s.dim - base);
                    const int64_t kb = std::min(s.per_block_k, len);
                    for (int r = 0; r < filled; ++r) {
                        const size_t q = size_t((b * m + r) * kbs);
                        const int16_t* ix = h->h_ring_idx + q;
                        const unsigned char* vv = static_cast<const unsigned char*>(h->h_gath) + q * psz;
                        unsigned char* hp = static_cast<unsigned char*>(h_params) + size_t(base) * psz;
                        if (psz == 2) {
                            for (int64_t j = 0; j < kb; ++j)
                                reinterpret_cast<uint16_t*>(hp)[ix[j]] = reinterpret_cast<const uint16_t*>(vv)[j];
                        } else if (psz == 4) {
                            for (int64_t j = 0; j < kb; ++j)
                                reinterpret_cast<uint32_t*>(hp)[ix[j]] = reinterpret_cast<const uint32_t*>(vv)[j];
                        } else {
                            for (int64_t j = 0; j < kb; ++j)
                                reinterpret_cast<uint64_t*>(hp)[ix[j]] = reinterpret_cast<const uint64_t*>(vv)[j];
                        }
                    }
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        if (err) return fail(MA_ERR_CUDA, "ma_step_host: sparse θ return failed");
    }
    MA_CUDA(cudaStreamSynchronize(s_d2h));
    { ma_status ms = mark_done(h, st); if (ms != MA_OK) return ms; }
    h->host_synced = h_params;
    return ma_sync(h);
}

ma_status ma_sync(ma_handle* h) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    DeviceGuard g(h->device);
    ma_status ws = wait_done(h);
    if (ws != MA_OK) return ws;
    unsigned flag = 0;
    MA_CUDA(cudaMemcpy(&flag, h->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag) {
        const unsigned zero = 0;
        MA_CUDA(cudaMemcpy(h->d_flag, &zero, sizeof(zero), cudaMemcpyHostToDevice));
        return fail(MA_ERR_NONFINITE, "step gradient: non-finite entry (state of that step is undefined)");
    }
    return MA_OK;
}

ma_status ma_get_counters(const ma_handle* h, int64_t* step, int64_t* head, int64_t* filled,
                          int64_t* stamps) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (step) *step = h->step;
    if (head) *head = h->head;
    if (filled) *filled = h->filled;
    if (stamps) std::memcpy(stamps, h->stamps.data(), h->stamps.size() * sizeof(int64_t));
    return MA_OK;
}

ma_status ma_read_error_buffer(ma_handle* h, uint8_t* codes, double* lo, double* hi) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (h->d_dense) return fail(MA_ERR_STATE, "error_buffer: engine uses dense error storage");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    if (codes) MA_CUDA(cudaMemcpy(codes, h->d_codes, size_t(h->shape.code_bytes), cudaMemcpyDeviceToHost));
    if (lo || hi) {
        std::vector<double2> meta(size_t(h->shape.nbuckets));
        MA_CUDA(cudaMemcpy(meta.data(), h->d_meta, meta.size() * sizeof(double2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < meta.size(); ++i) {
            if (lo) lo[i] = meta[i].x;
            if (hi) hi[i] = meta[i].y;
        }
    }
    return MA_OK;
}

ma_status ma_read_error_buffer_blocks(ma_handle* h, int64_t block_begin, int64_t block_end, uint8_t* codes,
                                      double* lo, double* hi) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (h->d_dense) return fail(MA_ERR_STATE, "error_buffer: engine uses dense error storage");
    const Shape& s = h->shape;
    // global Top-K handles: "blocks" are 4096-element chunks of the vector
    const int64_t unit = s.global ? 4096 : s.block;
    const int64_t nunits = s.global ? (s.dim + unit - 1) / unit : s.b1 - s.b0;
    if (block_begin < 0 || block_end > nunits || block_begin >= block_end)
        return fail(MA_ERR_INVALID_ARG, "block range outside the handle");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    const int64_t e0 = block_begin * unit, e1 = std::min(s.dim, block_end * unit);
    const int64_t bits = h->cfg.hp.bits;
    if (codes) {
        const int64_t c0 = (e0 * bits) / 8, c1 = (e1 * bits + 7) / 8;
        MA_CUDA(cudaMemcpy(codes, h->d_codes + c0, size_t(c1 - c0), cudaMemcpyDeviceToHost));
    }
    if (lo || hi) {
        const int64_t q0 = e0 / s.bucket, q1 = (e1 + s.bucket - 1) / s.bucket;
        std::vector<double2> meta(size_t(q1 - q0));
        MA_CUDA(cudaMemcpy(meta.data(), h->d_meta + q0, meta.size() * sizeof(double2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < meta.size(); ++i) {
            if (lo) lo[i] = meta[i].x;
            if (hi) hi[i] = meta[i].y;
        }
    }
    return MA_OK;
}

namespace {
double widen(const void* p, int dt, size_t i) {
    if (dt == MA_F64) return static_cast<const double*>(p)[i];
    if (dt == MA_F32) return double(static_cast<const float*>(p)[i]);
    uint32_t u = uint32_t(static_cast<const uint16_t*>(p)[i]) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return double(f);
}
}  // namespace

ma_status ma_read_error_vector(ma_handle* h, double* out) {
    if (!h || !out) return fail(MA_ERR_INVALID_ARG, "null argument");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    const Shape& s = h->shape;
    if (h->d_dense) {
        MA_CUDA(cudaMemcpy(out, h->d_dense, size_t(s.dim) * sizeof(double), cudaMemcpyDeviceToHost));
        return MA_OK;
    }
    // QuantizedErrorBuffer::decode (quantize.cpp:164-178): c * level + lo
    std::vector<uint8_t> codes(static_cast<size_t>(s.code_bytes));
    std::vector<double2> meta(static_cast<size_t>(s.nbuckets));
    MA_CUDA(cudaMemcpy(codes.data(), h->d_codes, codes.size(), cudaMemcpyDeviceToHost));
    MA_CUDA(cudaMemcpy(meta.data(), h->d_meta, meta.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    const int bits = int(h->cfg.hp.bits);
    const double max_code = double((1u << bits) - 1u);
    for (int64_t i = 0; i < s.dim; ++i) {
        const double2 m = meta[size_t(i / s.bucket)];
        const double level = m.x == m.y ? 0.0 : (m.y - m.x) / max_code;
        const int64_t pos = i * bits;  // LSB-first bit stream (quantize.cpp:116-128)
        uint32_t w = codes[size_t(pos >> 3)];
        for (int k = 1; 8 * k < int(pos & 7) + bits; ++k) w |= uint32_t(codes[size_t((pos >> 3) + k)]) << (8 * k);
        const double c = double((w >> (pos & 7)) & ((1u << bits) - 1u));
        out[i] = c * level + m.x;
    }
    return MA_OK;
}

ma_status ma_read_window_blocks(ma_handle* h, int64_t slot, int64_t block_begin, int64_t block_end,
                                int64_t* indices, double* values) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (slot < 0 || slot >= h->cfg.hp.window) return fail(MA_ERR_INVALID_ARG, "slot out of range");
    const Shape& s = h->shape;
    if (s.global) return fail(MA_ERR_UNSUPPORTED, "window_blocks: blockwise handles only");
    if (block_begin < 0 || block_end > s.b1 - s.b0 || block_begin >= block_end)
        return fail(MA_ERR_INVALID_ARG, "block range outside the handle");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    const int64_t nb = block_end - block_begin, m = h->cfg.hp.window, kbs = s.kb_stride;
    const size_t vsz = dtype_size(h->cfg.value_dtype);
    std::vector<int16_t> idx(size_t(nb * kbs));
    std::vector<unsigned char> val(size_t(nb * kbs) * vsz);
    const int64_t q = (block_begin * m + slot) * kbs;
    MA_CUDA(cudaMemcpy2D(idx.data(), size_t(kbs) * 2, h->d_win_idx + q, size_t(m * kbs) * 2, size_t(kbs) * 2,
                         size_t(nb), cudaMemcpyDeviceToHost));
    MA_CUDA(cudaMemcpy2D(val.data(), size_t(kbs) * vsz, static_cast<char*>(h->d_win_val) + size_t(q) * vsz,
                         size_t(m * kbs) * vsz, size_t(kbs) * vsz, size_t(nb), cudaMemcpyDeviceToHost));
    int64_t n = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t start = (block_begin + b) * s.block;
        const int64_t len = std::min(s.block, s.dim - start);
        const int64_t kb = std::min(s.per_block_k, len);
        for (int64_t j = 0; j < kb; ++j, ++n) {
            if (indices) indices[n] = s.elem0 + start + idx[size_t(b * kbs + j)];
            if (values) values[n] = widen(val.data(), h->cfg.value_dtype, size_t(b * kbs + j));
        }
    }
    return MA_OK;
}

ma_status ma_read_window_row(ma_handle* h, int64_t slot, int64_t* indices, double* values) {
    if (!h) return fail(MA_ERR_INVALID_ARG, "null handle");
    if (slot < 0 || slot >= h->cfg.hp.window) return fail(MA_ERR_INVALID_ARG, "slot out of range");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    const Shape& s = h->shape;
    const int64_t nb = s.b1 - s.b0, m = h->cfg.hp.window, kbs = s.kb_stride;
    const size_t vsz = dtype_size(h->cfg.value_dtype);
    if (s.global) {  // [m][kb_stride] int64 global indices
        std::vector<int64_t> gi(static_cast<size_t>(s.row_width));
        std::vector<unsigned char> gv(size_t(s.row_width) * vsz);
        MA_CUDA(cudaMemcpy(gi.data(), reinterpret_cast<const int64_t*>(h->d_win_idx) + slot * kbs,
                           gi.size() * 8, cudaMemcpyDeviceToHost));
        MA_CUDA(cudaMemcpy(gv.data(), static_cast<const char*>(h->d_win_val) + size_t(slot * kbs) * vsz, gv.size(),
                           cudaMemcpyDeviceToHost));
        for (int64_t j = 0; j < s.row_width; ++j) {
            if (indices) indices[j] = gi[size_t(j)];
            if (values) values[j] = widen(gv.data(), h->cfg.value_dtype, size_t(j));
        }
        return MA_OK;
    }
    // Strided 2-D copy of just this slot: one row of kb_stride per block.
    std::vector<int16_t> idx(size_t(nb * kbs));
    std::vector<unsigned char> val(size_t(nb * kbs) * vsz);
    MA_CUDA(cudaMemcpy2D(idx.data(), size_t(kbs) * 2, h->d_win_idx + slot * kbs, size_t(m * kbs) * 2,
                         size_t(kbs) * 2, size_t(nb), cudaMemcpyDeviceToHost));
    MA_CUDA(cudaMemcpy2D(val.data(), size_t(kbs) * vsz,
                         static_cast<char*>(h->d_win_val) + size_t(slot * kbs) * vsz,
                         size_t(m * kbs) * vsz, size_t(kbs) * vsz, size_t(nb), cudaMemcpyDeviceToHost));
    int64_t n = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t start = b * s.block;
        const int64_t len = std::min(s.block, s.dim - start);
        const int64_t kb = std::min(s.per_block_k, len);
        for (int64_t j = 0; j < kb; ++j, ++n) {
            if (indices) indices[n] = s.elem0 + start + idx[size_t(b * kbs + j)];
            if (values) values[n] = widen(val.data(), h->cfg.value_dtype, size_t(b * kbs + j));
        }
    }
    return MA_OK;
}

namespace {
// Window rows as SparseSelection::validate (compress.cpp:8-17) and the ring
// layout require: for every written row (stamp != 0), indices inside the
// handle's range, strictly increasing, and (blockwise) each block's entries
// inside that block.
ma_status check_window_rows(const ma_handle* h, int64_t step, int64_t head, const int64_t* stamps,
                            const int64_t* win_indices) {
    const Shape& s = h->shape;
    const int64_t m = h->cfg.hp.window;
    if (step < 0 || head < 0 || head >= m) return fail(MA_ERR_INVALID_ARG, "bad counters");
    for (int64_t r = 0; r < m; ++r) {
        if (stamps[r] == 0) continue;
        const int64_t* row = win_indices + r * s.row_width;
        for (int64_t j = 0; j < s.row_width; ++j) {
            if (row[j] < s.elem0 || row[j] >= s.elem0 + s.dim)
                return fail(MA_ERR_INVALID_ARG, "window index outside the vector");
            if (j > 0 && row[j] <= row[j - 1])
                return fail(MA_ERR_INVALID_ARG, "window row indices are not strictly increasing");
        }
        if (s.global) continue;
        int64_t n = 0;
        for (int64_t b = 0; b < s.b1 - s.b0; ++b) {
            const int64_t start = s.elem0 + b * s.block;
            const int64_t len = std::min(s.block, s.elem0 + s.dim - start);
            const int64_t kb = std::min(s.per_block_k, len);
            for (int64_t j = 0; j < kb; ++j, ++n)
                if (row[n] < start || row[n] >= start + len)
                    return fail(MA_ERR_INVALID_ARG, "window index outside its block");
        }
    }
    return MA_OK;
}
}  // namespace

ma_status ma_write_state(ma_handle* h, const uint8_t* codes, const double* lo, const double* hi,
                         int64_t step, int64_t head, const int64_t* stamps,
                         const int64_t* win_indices, const double* win_values) {
    if (!h || !codes || !lo || !hi || !stamps || !win_indices || !win_values)
        return fail(MA_ERR_INVALID_ARG, "null argument");
    const Shape& s = h->shape;
    const int64_t m = h->cfg.hp.window;
    { ma_status cs = check_window_rows(h, step, head, stamps, win_indices); if (cs != MA_OK) return cs; }
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    // Everything is validated and staged on the host first; the device state
    // changes only when the whole input is valid (SparseSelection::validate,
    // compress.cpp:8-17: strictly increasing indices inside the vector).
    std::vector<double2> meta(size_t(s.nbuckets));
    for (size_t i = 0; i < meta.size(); ++i) meta[i] = make_double2(lo[i], hi[i]);
    auto commit_ef = [&]() -> ma_status {
        MA_CUDA(cudaMemcpy(h->d_codes, codes, size_t(s.code_bytes), cudaMemcpyHostToDevice));
        MA_CUDA(cudaMemcpy(h->d_meta, meta.data(), meta.size() * sizeof(double2), cudaMemcpyHostToDevice));
        return MA_OK;
    };
    const int64_t nb = s.b1 - s.b0, kbs = s.kb_stride;
    const int vdt = h->cfg.value_dtype;
    const size_t vsz = dtype_size(vdt);
    auto put_val = [&](unsigned char* dst, double v) {
        if (vdt == MA_F64) {
            std::memcpy(dst, &v, 8);
        } else if (vdt == MA_F32) {
            const float f = float(v);
            std::memcpy(dst, &f, 4);
        } else {
            const float f = float(v);  // caller passes bf16-representable values
            uint32_t u;
            std::memcpy(&u, &f, 4);
            const uint16_t hb = uint16_t(u >> 16);
            std::memcpy(dst, &hb, 2);
        }
    };
    if (s.global) {
        std::vector<int64_t> gi(static_cast<size_t>(m * kbs), 0);
        std::vector<unsigned char> gv(size_t(m * kbs) * vsz, 0);
        for (int64_t r = 0; r < m; ++r)
            for (int64_t j = 0; j < s.row_width; ++j) {
                const int64_t idx = win_indices[r * s.row_width + j];
                if (stamps[r] != 0 && (idx < 0 || idx >= s.dim))
                    return fail(MA_ERR_INVALID_ARG, "window index outside the vector");
                if (stamps[r] != 0 && j > 0 && idx <= win_indices[r * s.row_width + j - 1])
                    return fail(MA_ERR_INVALID_ARG, "window row indices are not strictly increasing");
                gi[size_t(r * kbs + j)] = idx < 0 ? 0 : idx;
                put_val(&gv[size_t(r * kbs + j) * vsz], win_values[r * s.row_width + j]);
            }
        { ma_status cs = commit_ef(); if (cs != MA_OK) return cs; }
        MA_CUDA(cudaMemcpy(h->d_win_idx, gi.data(), gi.size() * 8, cudaMemcpyHostToDevice));
        h->g_bounds_valid = false;  // every row changed: the next step recomputes all chunk bounds
        MA_CUDA(cudaMemcpy(h->d_win_val, gv.data(), gv.size(), cudaMemcpyHostToDevice));
        h->step = step;
        h->head = head;
        h->filled = step < m ? step : m;
        std::memcpy(h->stamps.data(), stamps, size_t(m) * sizeof(int64_t));
        return MA_OK;
    }
    std::vector<int16_t> idx(size_t(nb * m * kbs), 0);
    std::vector<unsigned char> val(size_t(nb * m * kbs) * vsz, 0);
    for (int64_t r = 0; r < m; ++r) {
        int64_t n = r * s.row_width;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t start = b * s.block;
            const int64_t len = std::min(s.block, s.dim - start);
            const int64_t kb = std::min(s.per_block_k, len);
            for (int64_t j = 0; j < kb; ++j, ++n) {
                const int64_t rel = win_indices[n] - s.elem0 - start;
                if (stamps[r] != 0 && (rel < 0 || rel >= len))
                    return fail(MA_ERR_INVALID_ARG, "window index outside its block");
                if (stamps[r] != 0 && j > 0 && win_indices[n] <= win_indices[n - 1])
                    return fail(MA_ERR_INVALID_ARG, "window row indices are not strictly increasing");
                const size_t q = size_t((b * m + r) * kbs + j);
                idx[q] = int16_t(rel < 0 ? 0 : rel);
                const double v = win_values[n];
                if (vdt == MA_F64) {
                    std::memcpy(&val[q * 8], &v, 8);
                } else if (vdt == MA_F32) {
                    const float f = float(v);
                    std::memcpy(&val[q * 4], &f, 4);
                } else {
                    const float f = float(v);  // caller passes bf16-representable values
                    uint32_t u;
                    std::memcpy(&u, &f, 4);
                    const uint16_t hb = uint16_t(u >> 16);
                    std::memcpy(&val[q * 2], &hb, 2);
                }
            }
        }
    }
    { ma_status cs = commit_ef(); if (cs != MA_OK) return cs; }
    MA_CUDA(cudaMemcpy(h->d_win_idx, idx.data(), idx.size() * 2, cudaMemcpyHostToDevice));
    MA_CUDA(cudaMemset(h->d_thresh, 0, size_t(nb) * sizeof(uint32_t)));
    MA_CUDA(cudaMemcpy(h->d_win_val, val.data(), val.size(), cudaMemcpyHostToDevice));
    h->step = step;
    h->head = head;
    h->filled = step < m ? step : m;
    std::memcpy(h->stamps.data(), stamps, size_t(m) * sizeof(int64_t));
    return MA_OK;
}

// ---------------------------------------------------------------------------
// MADM v1 checkpoints (checkpoint.cpp:50-140): the reference's on-disk format,
// written from / restored into device state. Little-endian fields: "MADM",
// version 1, lossless flag, dim, step, θ as f64, window header (capacity,
// row_width, head, filled), rows 0..filled-1 (stamp, int64 indices, f64
// values), then bits, bucket, num_buckets, (lo, hi) per bucket, code bytes.
// ---------------------------------------------------------------------------
namespace {

struct CkptFile {
    std::FILE* f = nullptr;
    ~CkptFile() {
        if (f) std::fclose(f);
    }
};

bool put_bytes(std::FILE* f, const void* p, size_t n) { return std::fwrite(p, 1, n, f) == n; }
bool put_i64(std::FILE* f, int64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(static_cast<uint64_t>(v) >> (8 * i));
    return put_bytes(f, b, 8);
}
bool get_bytes(std::FILE* f, void* p, size_t n) { return std::fread(p, 1, n, f) == n; }
bool get_i64(std::FILE* f, int64_t* v) {
    unsigned char b[8];
    if (!get_bytes(f, b, 8)) return false;
    uint64_t u = 0;
    for (int i = 0; i < 8; ++i) u |= static_cast<uint64_t>(b[i]) << (8 * i);
    *v = static_cast<int64_t>(u);
    return true;
}
// f64 arrays: the host is little-endian (x86-64 / aarch64), as the format.
bool put_f64s(std::FILE* f, const double* v, size_t n) { return put_bytes(f, v, n * 8); }
bool get_f64s(std::FILE* f, double* v, size_t n) { return get_bytes(f, v, n * 8); }

constexpr size_t kCkptChunk = size_t(1) << 22;  // elements per θ staging chunk

}  // namespace

ma_status ma_save_checkpoint(ma_handle* h, const void* params, int32_t params_on_device, const char* path) {
    if (!h || !params || !path) return fail(MA_ERR_INVALID_ARG, "null argument");
    const Shape& s = h->shape;
    if (s.dim != s.dim_global) return fail(MA_ERR_UNSUPPORTED, "checkpoint: sharded handles are not supported");
    DeviceGuard g(h->device);
    { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
    CkptFile cf;
    cf.f = std::fopen(path, "wb");
    if (!cf.f) return fail(MA_ERR_INVALID_ARG, std::string("checkpoint: cannot open ") + path + " for writing");
    std::FILE* f = cf.f;
    const int64_t m = h->cfg.hp.window;
    const unsigned char head8[6] = {'M', 'A', 'D', 'M', 1, static_cast<unsigned char>(h->d_dense ? 1 : 0)};  // magic, version, lossless
    bool ok = put_bytes(f, head8, 6) && put_i64(f, s.dim) && put_i64(f, h->step);
    // θ (optim.hpp params()) widened to f64
    const int pdt = h->cfg.param_dtype;
    const size_t psz = dtype_size(pdt);
    std::vector<unsigned char> raw;
    std::vector<double> wide;
    for (int64_t i0 = 0; ok && i0 < s.dim; i0 += int64_t(kCkptChunk)) {
        const size_t n = size_t(std::min<int64_t>(int64_t(kCkptChunk), s.dim - i0));
        raw.resize(n * psz);
        const unsigned char* src = static_cast<const unsigned char*>(params) + size_t(i0) * psz;
        if (params_on_device) MA_CUDA(cudaMemcpy(raw.data(), src, n * psz, cudaMemcpyDeviceToHost));
        else std::memcpy(raw.data(), src, n * psz);
        wide.resize(n);
        for (size_t i = 0; i < n; ++i) wide[i] = widen(raw.data(), pdt, i);
        ok = put_f64s(f, wide.data(), n);
    }
    ok = ok && put_i64(f, m) && put_i64(f, s.row_width) && put_i64(f, h->head) && put_i64(f, h->filled);
    std::vector<int64_t> idx(static_cast<size_t>(s.row_width));
    std::vector<double> val(static_cast<size_t>(s.row_width));
    for (int64_t r = 0; ok && r < h->filled; ++r) {
        ma_status st = ma_read_window_row(h, r, idx.data(), val.data());
        if (st != MA_OK) return st;
        ok = put_i64(f, h->stamps[size_t(r)]) && put_bytes(f, idx.data(), idx.size() * 8) &&
             put_f64s(f, val.data(), val.size());
    }
    if (h->d_dense) {  // lossless: the dense error vector (checkpoint.cpp:72-73)
        std::vector<double> ev(static_cast<size_t>(s.dim));
        ma_status st = ma_read_error_vector(h, ev.data());
        if (st != MA_OK) return st;
        ok = ok && put_f64s(f, ev.data(), ev.size());
        if (!ok || std::fflush(f) != 0)
            return fail(MA_ERR_INVALID_ARG, std::string("checkpoint: write failed for ") + path);
        return MA_OK;
    }
    std::vector<uint8_t> codes(static_cast<size_t>(s.code_bytes));
    std::vector<double> lo(static_cast<size_t>(s.nbuckets)), hi(static_cast<size_t>(s.nbuckets));
    ma_status st = ma_read_error_buffer(h, codes.data(), lo.data(), hi.data());
    if (st != MA_OK) return st;
    const unsigned char bits = static_cast<unsigned char>(h->cfg.hp.bits);
    ok = ok && put_bytes(f, &bits, 1) && put_i64(f, s.bucket) && put_i64(f, s.nbuckets);
    for (int64_t q = 0; ok && q < s.nbuckets; ++q)
        ok = put_f64s(f, &lo[size_t(q)], 1) && put_f64s(f, &hi[size_t(q)], 1);
    ok = ok && put_i64(f, s.code_bytes) && put_bytes(f, codes.data(), codes.size());
    if (!ok || std::fflush(f) != 0) return fail(MA_ERR_INVALID_ARG, std::string("checkpoint: write failed for ") + path);
    return MA_OK;
}

ma_status ma_load_checkpoint(ma_handle* h, void* params, int32_t params_on_device, const char* path) {
    if (!h || !path) return fail(MA_ERR_INVALID_ARG, "null argument");
    const Shape& s = h->shape;
    if (s.dim != s.dim_global) return fail(MA_ERR_UNSUPPORTED, "checkpoint: sharded handles are not supported");
    DeviceGuard g(h->device);
    CkptFile cf;
    cf.f = std::fopen(path, "rb");
    if (!cf.f) return fail(MA_ERR_INVALID_ARG, std::string("checkpoint: cannot open ") + path);
    std::FILE* f = cf.f;
    if (std::fseek(f, 0, SEEK_END) != 0) return fail(MA_ERR_INVALID_ARG, "checkpoint: cannot seek");
    const long long fsize = std::ftell(f);
    std::rewind(f);
    unsigned char head8[6];
    if (!get_bytes(f, head8, 6)) return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    if (std::memcmp(head8, "MADM", 4) != 0) return fail(MA_ERR_INVALID_ARG, "checkpoint: bad magic");
    if (head8[4] != 1) return fail(MA_ERR_INVALID_ARG, "checkpoint: unsupported version");
    if ((head8[5] != 0) != (h->d_dense != nullptr))
        return fail(MA_ERR_INVALID_ARG, "checkpoint: lossless flag does not match the optimizer");
    int64_t dim = 0, step = 0, cap = 0, rw = 0, head = 0, filled = 0;
    if (!get_i64(f, &dim) || !get_i64(f, &step)) return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    if (dim != s.dim) return fail(MA_ERR_DIM, "checkpoint: dimension differs from the optimizer's");
    // θ is read last (streamed): first parse and validate everything after it,
    // so a malformed file leaves θ and the optimizer state untouched.
    const long long theta_off = std::ftell(f);
    if (theta_off < 0 || fsize - theta_off < static_cast<long long>(dim) * 8)
        return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    if (std::fseek(f, static_cast<long>(theta_off + static_cast<long long>(dim) * 8), SEEK_SET) != 0)
        return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    if (!get_i64(f, &cap) || !get_i64(f, &rw) || !get_i64(f, &head) || !get_i64(f, &filled))
        return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    const int64_t m = h->cfg.hp.window;
    if (cap != m || rw != s.row_width || filled < 0 || filled > cap || head < 0 || head >= cap)
        return fail(MA_ERR_INVALID_ARG, "checkpoint: window header does not match the optimizer");
    std::vector<int64_t> stamps(static_cast<size_t>(m), 0), idx(static_cast<size_t>(m * rw), 0);
    std::vector<double> val(static_cast<size_t>(m * rw), 0.0);
    for (int64_t r = 0; r < filled; ++r) {
        if (!get_i64(f, &stamps[size_t(r)]) || !get_bytes(f, &idx[size_t(r * rw)], size_t(rw) * 8) ||
            !get_f64s(f, &val[size_t(r * rw)], size_t(rw)))
            return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    }
    { ma_status cs = check_window_rows(h, step, head, stamps.data(), idx.data()); if (cs != MA_OK) return cs; }
    std::vector<double> ev;
    unsigned char bits = 0;
    int64_t bucket = 0, nbk = 0, nbytes = 0;
    std::vector<double> lo, hi;
    std::vector<uint8_t> codes;
    if (h->d_dense) {  // lossless: dense error vector after the window state
        ev.resize(static_cast<size_t>(dim));
        if (!get_f64s(f, ev.data(), ev.size())) return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    } else {
        if (!get_bytes(f, &bits, 1) || !get_i64(f, &bucket) || !get_i64(f, &nbk))
            return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
        if (bits != h->cfg.hp.bits || bucket != s.bucket || nbk != s.nbuckets)
            return fail(MA_ERR_INVALID_ARG, "checkpoint: bucket count mismatch");
        lo.resize(static_cast<size_t>(nbk));
        hi.resize(static_cast<size_t>(nbk));
        for (int64_t q = 0; q < nbk; ++q)
            if (!get_f64s(f, &lo[size_t(q)], 1) || !get_f64s(f, &hi[size_t(q)], 1))
                return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
        if (!get_i64(f, &nbytes) || nbytes != s.code_bytes)
            return fail(MA_ERR_INVALID_ARG, "checkpoint: code length mismatch");
        codes.resize(static_cast<size_t>(nbytes));
        if (!get_bytes(f, codes.data(), codes.size())) return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
    }
    // The whole file is valid: θ, then the optimizer state.
    if (params) {
        if (std::fseek(f, static_cast<long>(theta_off), SEEK_SET) != 0)
            return fail(MA_ERR_INVALID_ARG, "checkpoint: cannot seek");
        const int pdt = h->cfg.param_dtype;
        const size_t psz = dtype_size(pdt);
        std::vector<double> wide;
        std::vector<unsigned char> raw;
        for (int64_t i0 = 0; i0 < dim; i0 += int64_t(kCkptChunk)) {
            const size_t n = size_t(std::min<int64_t>(int64_t(kCkptChunk), dim - i0));
            wide.resize(n);
            if (!get_f64s(f, wide.data(), n)) return fail(MA_ERR_INVALID_ARG, "checkpoint: truncated file");
            raw.resize(n * psz);
            for (size_t i = 0; i < n; ++i) {
                if (pdt == MA_F64) {
                    std::memcpy(&raw[i * 8], &wide[i], 8);
                } else if (pdt == MA_F32) {
                    const float x = float(wide[i]);
                    std::memcpy(&raw[i * 4], &x, 4);
                } else {  // bf16: values written from a bf16 θ are exact; others round to nearest even
                    const float x = float(wide[i]);
                    uint32_t u;
                    std::memcpy(&u, &x, 4);
                    const uint16_t b = uint16_t((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
                    std::memcpy(&raw[i * 2], &b, 2);
                }
            }
            unsigned char* dst = static_cast<unsigned char*>(params) + size_t(i0) * psz;
            if (params_on_device) MA_CUDA(cudaMemcpy(dst, raw.data(), raw.size(), cudaMemcpyHostToDevice));
            else std::memcpy(dst, raw.data(), raw.size());
        }
    }
    ma_status st;
    if (h->d_dense) {
        { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
        MA_CUDA(cudaMemcpy(h->d_dense, ev.data(), ev.size() * sizeof(double), cudaMemcpyHostToDevice));
        std::vector<uint8_t> zc(static_cast<size_t>(s.code_bytes), 0);
        std::vector<double> z0(static_cast<size_t>(s.nbuckets), 0.0);
        st = ma_write_state(h, zc.data(), z0.data(), z0.data(), step, head, stamps.data(), idx.data(), val.data());
    } else {
        // rows >= filled are unwritten (stamp 0): ma_write_state zero-fills them
        st = ma_write_state(h, codes.data(), lo.data(), hi.data(), step, head, stamps.data(), idx.data(),
                            val.data());
    }
    if (st != MA_OK) return st;
    if (params && !params_on_device) h->theta_valid = false;  // ma_step_host re-uploads θ
    h->host_synced = nullptr;
    return MA_OK;
}

// ---------------------------------------------------------------------------
// Sparse parameter propagation: ma_step split into a
// sharded front (EF decode, Top-K, window row, EF re-quantization over a block
// range), a row exchange, and ADAM_STATS + update replicated over all blocks,
// so ranks exchange only the new window rows (4·k_b/B_d ≈ 0.04 B/param)
// instead of θ. front(all) + stats(all) is bit-identical to ma_step.
// ---------------------------------------------------------------------------
ma_status ma_step_front(ma_handle* h, const void* d_grads, int64_t block_begin, int64_t block_end,
                        void* d_stage_idx, void* d_stage_val, void* stream) {
    if (!h || !d_grads || !d_stage_idx || !d_stage_val) return fail(MA_ERR_INVALID_ARG, "null argument");
    const Shape& s = h->shape;
    const int64_t nb = s.b1 - s.b0;
    if (block_begin < 0 || block_end > nb || block_begin >= block_end)
        return fail(MA_ERR_INVALID_ARG, "step_front: block range outside the handle");
    if (s.dim % s.block != 0 || !h->warp)
        return fail(MA_ERR_UNSUPPORTED, "step_front: needs whole 4096-blocks and the warp kernel");
    if (h->cfg.finite_mode == MA_FINITE_STRICT)
        return fail(MA_ERR_UNSUPPORTED, "step_front: strict finiteness needs the fused step");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ma::StepArgs a;
    base_args(h, &a);
    if (!ma::lean_phase_ok(a)) return fail(MA_ERR_UNSUPPORTED, "step_front: dtype/bucket not on the lean kernel");
    const size_t gsz = dtype_size(h->cfg.grad_dtype);
    // the kernel addresses g by handle element index; the caller's buffer starts at block_begin
    a.grads = static_cast<const unsigned char*>(d_grads) - size_t(block_begin * s.block) * gsz;
    a.params = nullptr;
    a.lr = h->cfg.hp.lr;
    a.lr32 = static_cast<float>(a.lr);
    const CounterSnap snap = snap_counters(h);
    push_and_weights(h, &a);
    a.block_offset = block_begin;
    a.block_count = block_end - block_begin;
    a.stage_idx = static_cast<int16_t*>(d_stage_idx);
    a.stage_val = d_stage_val;
    a.stage_b0 = block_begin;
    if (!h->pending) h->pending = new (std::nothrow) ma::StepArgs;
    if (!h->pending) {
        restore_counters(h, snap);
        return fail(MA_ERR_INVALID_ARG, "out of host memory");
    }
    MA_CUDA_ROLLBACK(h, snap, ma::launch_step_lean_phase(a, 1, st));
    ++h->launches;
    *h->pending = a;
    return mark_done(h, st);
}

ma_status ma_scatter_rows(ma_handle* h, const void* d_rows_idx, const void* d_rows_val, int64_t block_begin,
                          int64_t block_end, void* stream) {
    if (!h || !d_rows_idx || !d_rows_val) return fail(MA_ERR_INVALID_ARG, "null argument");
    if (!h->pending) return fail(MA_ERR_STATE, "scatter_rows: no ma_step_front in flight");
    const Shape& s = h->shape;
    const int64_t nb = s.b1 - s.b0, m = h->cfg.hp.window, kbs = s.kb_stride;
    if (block_begin < 0 || block_end > nb || block_begin >= block_end)
        return fail(MA_ERR_INVALID_ARG, "scatter_rows: block range outside the handle");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t slot = h->pending->slot;
    const size_t vsz = dtype_size(h->cfg.value_dtype);
    const size_t rows = size_t(block_end - block_begin);
    MA_CUDA(cudaMemcpy2DAsync(h->d_win_idx + (block_begin * m + slot) * kbs, size_t(m * kbs) * 2, d_rows_idx,
                              size_t(kbs) * 2, size_t(kbs) * 2, rows, cudaMemcpyDeviceToDevice, st));
    MA_CUDA(cudaMemcpy2DAsync(static_cast<unsigned char*>(h->d_win_val) + size_t((block_begin * m + slot) * kbs) * vsz,
                              size_t(m * kbs) * vsz, d_rows_val, size_t(kbs) * vsz, size_t(kbs) * vsz, rows,
                              cudaMemcpyDeviceToDevice, st));
    return MA_OK;
}

ma_status ma_step_stats(ma_handle* h, void* d_params, double lr, void* stream) {
    if (!h || !d_params) return fail(MA_ERR_INVALID_ARG, "null argument");
    if (!h->pending) return fail(MA_ERR_STATE, "step_stats: no ma_step_front in flight");
    if (!(lr > 0.0)) return fail(MA_ERR_INVALID_ARG, "step: lr must be > 0");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ma::StepArgs a = *h->pending;
    a.params = d_params;
    a.lr = lr;
    a.lr32 = static_cast<float>(lr);
    a.block_offset = 0;
    a.block_count = h->shape.b1 - h->shape.b0;
    MA_CUDA(ma::launch_step_lean_phase(a, 2, st));
    ++h->launches;
    delete h->pending;
    h->pending = nullptr;
    return mark_done(h, st);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Data-parallel collectives over NCCL (north star: "each GPU
// owns its slice ... only the updated bf16 parameters are all-gathered with
// NCCL over NVLink"). A shard handle (ma_create_shard) owns the block range
// sharding.py assigns to its rank: ranks take per = ceil(num_blocks / nranks)
// whole blocks each (the last rank the remainder), so rank r's elements start
// at r * per * block. The step itself needs no exchange (block sharding is
// bit-exact: compress.cpp:73-85 partitions the Top-K by block; the host
// counters, hence the bias correction of window.cpp:43, are replicated).
// ---------------------------------------------------------------------------
struct ma_comm {
    ma::nccl::Comm comm = nullptr;
    int nranks = 1, rank = 0;
    bool owned = false;
    int device = 0;
};

namespace {

const ma::nccl::Api* nccl_api() {
    std::string err;
    const ma::nccl::Api* a = ma::nccl::api(&err);
    if (!a) fail(MA_ERR_NCCL, err);
    return a;
}

#define MA_NCCL(api, call)                                                         \
    do {                                                                           \
        const int _r = (call);                                                     \
        if (_r != 0) return fail(MA_ERR_NCCL, ma::nccl::describe((api), _r) + " in " #call); \
    } while (0)

// The rank's partition (sharding.py:partition_blocks) must be the handle's range.
ma_status check_partition(const ma_handle* h, const ma_comm* c, int64_t* per_out) {
    const Shape& s = h->shape;
    if (s.global) return fail(MA_ERR_UNSUPPORTED, "collectives: global Top-K mode is not block-sharded");
    const int64_t nbg = s.nblocks_global;
    const int64_t per = (nbg + c->nranks - 1) / c->nranks;
    const int64_t b0 = int64_t(c->rank) * per, b1 = std::min(b0 + per, nbg);
    if (per * (c->nranks - 1) >= nbg)
        return fail(MA_ERR_INVALID_ARG, "collectives: some rank would own no block");
    if (s.b0 != b0 || s.b1 != b1)
        return fail(MA_ERR_INVALID_ARG, "collectives: the handle's block range is not this rank's partition "
                                        "(ranks own ceil(num_blocks / nranks) blocks each)");
    *per_out = per;
    return MA_OK;
}

}  // namespace


namespace {
ma_status allreduce_report(ma_handle* h, cudaStream_t st) {
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    MA_NCCL(a, a->AllReduce(h->d_report, h->d_report, ma::kReportFields, ma::nccl::kFloat64, ma::nccl::kSum,
                            h->report_comm->comm, st));
    return MA_OK;
}
}  // namespace

extern "C" {

ma_status ma_comm_unique_id(uint8_t* id) {
    if (!id) return fail(MA_ERR_INVALID_ARG, "null argument");
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    ma::nccl::IdBytes u;
    MA_NCCL(a, a->GetUniqueId(&u));
    std::memcpy(id, u.internal, sizeof(u.internal));
    return MA_OK;
}

ma_status ma_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int device, ma_comm** out) {
    if (!id || !out) return fail(MA_ERR_INVALID_ARG, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(MA_ERR_INVALID_ARG, "comm: bad rank / nranks");
    *out = nullptr;
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    DeviceGuard g(device);
    ma::nccl::IdBytes u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    ma::nccl::Comm cm = nullptr;
    MA_NCCL(a, a->CommInitRank(&cm, nranks, u, rank));
    ma_comm* c = new (std::nothrow) ma_comm;
    if (!c) {
        a->CommDestroy(cm);
        return fail(MA_ERR_INVALID_ARG, "out of host memory");
    }
    c->comm = cm;
    c->nranks = nranks;
    c->rank = rank;
    c->owned = true;
    c->device = device;
    *out = c;
    return MA_OK;
}

ma_status ma_comm_wrap(void* nccl_comm, ma_comm** out) {
    if (!nccl_comm || !out) return fail(MA_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    ma_comm* c = new (std::nothrow) ma_comm;
    if (!c) return fail(MA_ERR_INVALID_ARG, "out of host memory");
    c->comm = static_cast<ma::nccl::Comm>(nccl_comm);
    int n = 0, r = 0;
    const int e1 = a->CommCount(c->comm, &n), e2 = a->CommUserRank(c->comm, &r);
    if (e1 || e2) {
        delete c;
        return fail(MA_ERR_NCCL, ma::nccl::describe(a, e1 ? e1 : e2) + " in ma_comm_wrap");
    }
    c->nranks = n;
    c->rank = r;
    cudaGetDevice(&c->device);
    *out = c;
    return MA_OK;
}

ma_status ma_comm_destroy(ma_comm* c) {
    if (!c) return MA_OK;
    ma_status st = MA_OK;
    if (c->owned && c->comm) {
        const ma::nccl::Api* a = nccl_api();
        if (a) {
            DeviceGuard g(c->device);
            const int r = a->CommDestroy(c->comm);
            if (r) st = fail(MA_ERR_NCCL, ma::nccl::describe(a, r) + " in ncclCommDestroy");
        }
    }
    delete c;
    return st;
}

ma_status ma_comm_info(const ma_comm* c, int32_t* nranks, int32_t* rank) {
    if (!c) return fail(MA_ERR_INVALID_ARG, "null comm");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return MA_OK;
}

ma_status ma_allgather_params(ma_handle* h, void* d_params_full, int64_t full_elems, ma_comm* c, void* stream) {
    if (!h || !d_params_full || !c) return fail(MA_ERR_INVALID_ARG, "null argument");
    int64_t per = 0;
    { ma_status st = check_partition(h, c, &per); if (st != MA_OK) return st; }
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Shape& s = h->shape;
    const size_t psz = dtype_size(h->cfg.param_dtype);
    const int64_t stride = per * s.block;  // elements per (padded) shard
    unsigned char* full = static_cast<unsigned char*>(d_params_full);
    if (c->nranks == 1) return MA_OK;
    if (full_elems >= stride * c->nranks) {
        // equal chunks of the padded layout: one in-place all-gather
        MA_NCCL(a, a->AllGather(full + size_t(c->rank) * size_t(stride) * psz, full, size_t(stride) * psz,
                                ma::nccl::kUint8, c->comm, st));
    } else if (full_elems == s.dim_global) {
        // exact-length θ: every rank broadcasts its (possibly shorter, last) shard in place
        MA_NCCL(a, a->GroupStart());
        for (int r = 0; r < c->nranks; ++r) {
            const int64_t e0 = int64_t(r) * stride, e1 = std::min(e0 + stride, s.dim_global);
            const int rc = a->Broadcast(full + size_t(e0) * psz, full + size_t(e0) * psz, size_t(e1 - e0) * psz,
                                        ma::nccl::kUint8, r, c->comm, st);
            if (rc) {
                a->GroupEnd();
                return fail(MA_ERR_NCCL, ma::nccl::describe(a, rc) + " in ncclBroadcast");
            }
        }
        MA_NCCL(a, a->GroupEnd());
    } else {
        return fail(MA_ERR_INVALID_ARG, "allgather_params: full_elems must be dim or >= nranks * shard stride");
    }
    return mark_done(h, st);
}

ma_status ma_step_allgather(ma_handle* h, void* d_params_full, int64_t full_elems, const void* d_grads, double lr,
                            ma_comm* c, void* stream, ma_step_report* report) {
    if (!h || !d_params_full || !d_grads || !c) return fail(MA_ERR_INVALID_ARG, "null argument");
    int64_t per = 0;
    { ma_status st = check_partition(h, c, &per); if (st != MA_OK) return st; }
    if (full_elems < h->shape.dim_global) return fail(MA_ERR_INVALID_ARG, "step_allgather: full θ too short");
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    void* shard = static_cast<unsigned char*>(d_params_full) + size_t(h->shape.elem0) * dtype_size(h->cfg.param_dtype);
    h->report_comm = c->nranks > 1 ? c : nullptr;
    const ma_status rs = run_step(h, shard, d_grads, lr, st, report);
    h->report_comm = nullptr;
    if (rs != MA_OK) return rs;
    return ma_allgather_params(h, d_params_full, full_elems, c, stream);
}

ma_status ma_exchange_rows(ma_handle* h, const void* d_stage_idx, const void* d_stage_val, int64_t stage_blocks,
                           void* d_rows_idx, void* d_rows_val, ma_comm* c, void* stream) {
    if (!h || !d_stage_idx || !d_stage_val || !d_rows_idx || !d_rows_val || !c)
        return fail(MA_ERR_INVALID_ARG, "null argument");
    if (!h->pending) return fail(MA_ERR_STATE, "exchange_rows: no ma_step_front in flight");
    const Shape& s = h->shape;
    const int64_t nb = s.b1 - s.b0;
    const int64_t per = (nb + c->nranks - 1) / c->nranks;
    if (stage_blocks != per)
        return fail(MA_ERR_INVALID_ARG, "exchange_rows: stage_blocks must be ceil(num_blocks / nranks)");
    const ma::nccl::Api* a = nccl_api();
    if (!a) return MA_ERR_NCCL;
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t vsz = dtype_size(h->cfg.value_dtype);
    const size_t ent = size_t(per) * size_t(s.kb_stride);
    if (c->nranks == 1) return ma_scatter_rows(h, d_stage_idx, d_stage_val, 0, nb, stream);
    MA_NCCL(a, a->GroupStart());
    int rc = a->AllGather(d_stage_idx, d_rows_idx, ent * 2, ma::nccl::kUint8, c->comm, st);
    if (!rc) rc = a->AllGather(d_stage_val, d_rows_val, ent * vsz, ma::nccl::kUint8, c->comm, st);
    const int rc2 = a->GroupEnd();
    if (rc || rc2) return fail(MA_ERR_NCCL, ma::nccl::describe(a, rc ? rc : rc2) + " in exchange_rows");
    return ma_scatter_rows(h, d_rows_idx, d_rows_val, 0, nb, stream);
}

}  // extern "C"

extern "C" {

ma_status ma_get_layout(const ma_handle* h, ma_layout_info* out) {
    if (!h || !out) return fail(MA_ERR_INVALID_ARG, "null argument");
    fill_layout(h->shape, h->cfg, out);
    return MA_OK;
}

int64_t ma_kernel_launches(const ma_handle* h) { return h ? h->launches : 0; }

ma_status ma_debug_counters(ma_handle* h, int64_t* out, int n) {
    if (!h || !out || n < 0) return fail(MA_ERR_INVALID_ARG, "bad argument");
    DeviceGuard g(h->device);
    unsigned v[32] = {};
    if (h->d_dbg) {
        { ma_status ws = wait_done(h); if (ws != MA_OK) return ws; }
        MA_CUDA(cudaMemcpy(v, h->d_dbg, sizeof(v), cudaMemcpyDeviceToHost));
    }
    // [0, 8): event counters; [8, 20): per-phase warp cycles (MA_LEAN_PROF builds)
    for (int i = 0; i < n && i < 20; ++i) {
        if (i < 8) {
            out[i] = v[i];
        } else {
            unsigned long long c;
            std::memcpy(&c, reinterpret_cast<const unsigned char*>(v) + 32 + 8 * (i - 8), sizeof(c));
            out[i] = static_cast<int64_t>(c);
        }
    }
    return MA_OK;
}

const char* ma_last_error(void) { return g_last_error.c_str(); }

const char* ma_version(void) { return "microadam_cuda 0.1 (sm_100a, ABI 1)"; }

ma_status ma_fill_synthetic(void* d_out, int32_t dtype, int64_t n, uint64_t seed, uint64_t step,
                            int64_t offset, int32_t levels, void* stream) {
    if (!d_out || dtype < MA_F64 || dtype > MA_BF16) return fail(MA_ERR_INVALID_ARG, "bad argument");
    MA_CUDA(ma::launch_fill_synthetic(d_out, dtype, n, seed, step, offset, levels,
                                      static_cast<cudaStream_t>(stream)));
    return MA_OK;
}

}  // extern "C"
