// ma_kernels.cu — sm_100a kernels of the MicroAdam optimizer step.
//
// One fused kernel runs the whole reference step (optim.cpp:164-190) for one
// Top-K block per CTA, reading every input once from HBM and writing every
// output once:
//
//   P1  EF decode + accumulate   a = g + (code·level + lo)       quantize.cpp:164-178, optim.cpp:166-168
//   P2  block Top-K select        (|a| desc, idx asc), radix      compress.cpp:39-53, 73-85
//   P3  window write + residual   slot `head` ← (rel idx, V(a))   window.cpp:14-26, compress.cpp:95-102
//   P4  4-bit re-quantization     per-bucket min/max, nearest     quantize.cpp:7-24, 42-55, 142-162
//   P5  nibble pack               low nibble first                quantize.cpp:102-114
//   P6  ADAM_STATS + update       window rows in slot order       window.cpp:28-46, optim.cpp:183-187
//
// Arithmetic on the EF/Top-K/stats path is fp64 with explicit round-to-nearest
// intrinsics (__dmul_rn/__dadd_rn/__ddiv_rn/__dsqrt_rn) and the library is
// built with -fmad=false: the reference build has no FMA and a
// contracted decode changes ~37% of accumulator bits.
#include <cuda_bf16.h>

#include "../../include/ma_synth.h"
#include "ma_device.cuh"
#include "ma_internal.h"

#include <math_constants.h>

namespace ma {
namespace {

using namespace dev;

// ---------------------------------------------------------------------------
// Shared-memory carve-up (identical on host and device).
// ---------------------------------------------------------------------------
struct SmemLayout {
    size_t lo, lvl, a, z1, z2, eval, ckey, red, owner, hist, cidx, scan, misc, eidx, code, selm;
    size_t total;

    __host__ __device__ static size_t take(size_t& off, size_t bytes) {
        off = (off + 15) & ~size_t(15);
        const size_t r = off;
        off += bytes;
        return r;
    }
    // code_w: bytes per staged code (1 for bits <= 8, 4 up to 24)
    __host__ __device__ SmemLayout(int nt, int ept, int block, int bucket, int m, int kbs, int code_w = 1) {
        const size_t nbk = size_t((block + bucket - 1) / bucket) + 1;  // +1: buckets may straddle blocks
        const size_t ent = size_t(m) * size_t(kbs);
        size_t off = 0;
        lo = take(off, nbk * 8);
        lvl = take(off, nbk * 8);
        a = take(off, size_t(block) * 8);
        z1 = take(off, ent * 8);
        z2 = take(off, ent * 8);
        eval = take(off, ent * 8);
        ckey = take(off, size_t(kCandCap) * 8);
        red = take(off, size_t(nt / 32) * kReportFields * 8);
        owner = take(off, size_t(block) * 4);
        hist = take(off, 256 * 4);
        cidx = take(off, size_t(kCandCap) * 4);
        scan = take(off, (size_t(ept / 2) * size_t(nt / 32) + 1) * 4);
        misc = take(off, 32 * 4);
        eidx = take(off, ent * 2);
        code = take(off, size_t(block) * size_t(code_w));
        selm = take(off, size_t(block));
        total = (off + 15) & ~size_t(15);
    }
};

// Exclusive rank, in element order, of the flagged elements of the block.
// Thread `tid` holds elements e = 2*(j*NT + tid) + p at register slot 2j+p, so
// element order is (j, warp, lane, p). Returns the flagged total.
// Code of element i in the LSB-first bit stream of width `bits` (quantize.cpp:116-128).
__device__ __forceinline__ uint32_t read_code(const uint8_t* codes, int64_t i, int bits) {
    const int64_t pos = i * bits;
    const int64_t byte0 = pos >> 3;
    const int sh = static_cast<int>(pos & 7);
    uint32_t w = codes[byte0];
    for (int k = 1; 8 * k < sh + bits; ++k) w |= static_cast<uint32_t>(codes[byte0 + k]) << (8 * k);
    return (w >> sh) & ((1u << bits) - 1u);
}

template <int NT, int EPT>
__device__ __forceinline__ int block_rank(uint32_t flags, int (&rank)[EPT], int* scan) {
    constexpr int NW = NT / 32;
    constexpr int NP = EPT / 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    __syncthreads();  // previous users of scan[] are done
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        const uint32_t f0 = (flags >> (2 * j)) & 1u, f1 = (flags >> (2 * j + 1)) & 1u;
        const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, f0), b1 = __ballot_sync(0xFFFFFFFFu, f1);
        const int pre = __popc(b0 & lt) + __popc(b1 & lt);
        rank[2 * j] = pre;
        rank[2 * j + 1] = pre + static_cast<int>(f0);
        if (lane == 0) scan[j * NW + warp] = __popc(b0) + __popc(b1);
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int n = NP * NW;
        int carry = 0;
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const int v = i < n ? scan[i] : 0;
            int incl = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += t;
            }
            if (i < n) scan[i] = carry + incl - v;
            carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        if (lane == 0) scan[n] = carry;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        const int off = scan[j * NW + warp];
        rank[2 * j] += off;
        rank[2 * j + 1] += off;
    }
    return scan[NP * NW];
}

template <int NT>
__device__ __forceinline__ void block_sum5(double (&v)[kReportFields], double* red, double* out) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int f = 0; f < kReportFields; ++f) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[f] += __shfl_xor_sync(0xFFFFFFFFu, v[f], off);
        if (lane == 0) red[warp * kReportFields + f] = v[f];
    }
    __syncthreads();
    if (threadIdx.x < kReportFields) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[w * kReportFields + threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// The fused step kernel: one CTA per Top-K block.
// ---------------------------------------------------------------------------
template <int NT, int EPT>
__global__ void __launch_bounds__(NT) microadam_step_kernel(const __grid_constant__ StepArgs p) {
    constexpr int NP = EPT / 2;
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout L(NT, EPT, p.block, p.bucket, p.m, p.kb_stride, p.bits > 8 ? 4 : 1);
    double* s_lo = reinterpret_cast<double*>(smem + L.lo);
    double* s_lvl = reinterpret_cast<double*>(smem + L.lvl);
    double* s_a = reinterpret_cast<double*>(smem + L.a);
    double* s_z1 = reinterpret_cast<double*>(smem + L.z1);
    double* s_z2 = reinterpret_cast<double*>(smem + L.z2);
    double* s_eval = reinterpret_cast<double*>(smem + L.eval);
    uint64_t* s_ckey = reinterpret_cast<uint64_t*>(smem + L.ckey);
    double* s_red = reinterpret_cast<double*>(smem + L.red);
    int* s_owner = reinterpret_cast<int*>(smem + L.owner);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    int* s_cidx = reinterpret_cast<int*>(smem + L.cidx);
    int* s_scan = reinterpret_cast<int*>(smem + L.scan);
    int* s_misc = reinterpret_cast<int*>(smem + L.misc);
    int16_t* s_eidx = reinterpret_cast<int16_t*>(smem + L.eidx);
    uint8_t* s_code = reinterpret_cast<uint8_t*>(smem + L.code);
    uint32_t* s_code32 = reinterpret_cast<uint32_t*>(smem + L.code);  // bits > 8
    uint8_t* s_selm = reinterpret_cast<uint8_t*>(smem + L.selm);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int block = p.block, bucket = p.bucket, kbs = p.kb_stride;
    const int64_t b = p.block_offset + blockIdx.x;
    const int64_t base = b * static_cast<int64_t>(block);
    const int len = static_cast<int>(min(static_cast<int64_t>(block), p.dim - base));
    const int kb = min(p.per_block_k, len);
    const int64_t bk0 = base / bucket;  // bucket of the block's first element (buckets may straddle blocks)
    const int nbk = static_cast<int>((base + len - 1) / bucket - bk0 + 1);
    const bool want_report = p.partials != nullptr;
    const int bits = p.bits;
    const double max_code = static_cast<double>((1u << bits) - 1u);  // QuantParams::max_code
    auto elem = [&](int i) { return 2 * ((i >> 1) * NT + tid) + (i & 1); };

    // ---- P0: old bucket grids (QuantParams ctor, quantize.cpp:7-13) ----
    for (int i = tid; i < nbk; i += NT) {
        const double2 mt = p.meta[bk0 + i];
        s_lo[i] = mt.x;
        s_lvl[i] = (mt.x == mt.y) ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), max_code);
    }
    for (int i = tid; i < len; i += NT) s_selm[i] = 0;
    __syncthreads();

    // ---- P1: decode + accumulate (quantize.cpp:164-178, optim.cpp:166-168) ----
    double a[EPT];
    uint32_t valid = 0;
    bool bad = false;
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        const int e = 2 * (j * NT + tid);
        a[2 * j] = 0.0;
        a[2 * j + 1] = 0.0;
        if (e < len) {
            double g0, g1 = 0.0;
            const bool two = e + 1 < len;
            const bool odd = (base & 1) != 0;  // odd B_d (bucket-split mode): pairs straddle words / code bytes
            if (two && !odd) {
                ld_pair(p.grads, p.g_dtype, base + e, g0, g1);
            } else {
                g0 = ld_val(p.grads, p.g_dtype, base + e);
                if (two) g1 = ld_val(p.grads, p.g_dtype, base + e + 1);
            }
            const uint32_t byte = (p.dense || bits != 4) ? 0u
                                  : (odd ? (uint32_t(p.codes[(base + e) >> 1]) >> 4) |
                                               (two ? uint32_t(p.codes[(base + e + 1) >> 1] & 15u) << 4 : 0u)
                                         : p.codes[(base + e) >> 1]);
            const uint32_t c0 = bits == 4 ? (byte & 15u) : (p.dense ? 0u : read_code(p.codes, base + e, bits));
            const int bA = static_cast<int>((base + e) / bucket - bk0);
            const double e0 = p.dense ? p.dense[base + e]
                                      : __dadd_rn(__dmul_rn(static_cast<double>(c0), s_lvl[bA]), s_lo[bA]);
            a[2 * j] = __dadd_rn(g0, e0);
            valid |= 1u << (2 * j);
            bad |= !isfinite(g0) || !isfinite(a[2 * j]);
            if (want_report) {
                rep[0] += g0 * g0;
                rep[1] += a[2 * j] * a[2 * j];
            }
            if (two) {
                const int bB = static_cast<int>((base + e + 1) / bucket - bk0);
                const uint32_t c1 = bits == 4 ? (byte >> 4) : (p.dense ? 0u : read_code(p.codes, base + e + 1, bits));
                const double e1 = p.dense ? p.dense[base + e + 1]
                                          : __dadd_rn(__dmul_rn(static_cast<double>(c1), s_lvl[bB]), s_lo[bB]);
                a[2 * j + 1] = __dadd_rn(g1, e1);
                valid |= 1u << (2 * j + 1);
                bad |= !isfinite(g1) || !isfinite(a[2 * j + 1]);
                if (want_report) {
                    rep[0] += g1 * g1;
                    rep[1] += a[2 * j + 1] * a[2 * j + 1];
                }
            }
        }
    }
    if (p.check_finite && bad) atomicOr(p.flag, 1u);

    // ---- P2: block Top-K (compress.cpp:73-85) ----
    uint32_t sel = valid;
    if (kb < len)
        sel = block_topk<NT, EPT>(
            a, valid, kb, s_hist, s_misc, s_ckey, s_cidx, s_selm, elem,
            [&](uint32_t m, int (&r)[EPT]) { block_rank<NT, EPT>(m, r, s_scan); });

    // ---- P3: window row `slot` (window.cpp:14-26) + residual (compress.cpp:95-102) ----
    int rank[EPT];
    block_rank<NT, EPT>(sel, rank, s_scan);
    const int slot = p.slot;
    const int64_t wrow = (b * p.m + slot) * static_cast<int64_t>(kbs);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        if (!((valid >> i) & 1u)) continue;
        const int e = elem(i);
        if ((sel >> i) & 1u) {
            const int pos = rank[i];
            if (p.split_sel) atomicOr(p.split_sel + ((base + e) >> 5), 1u << ((base + e) & 31));
            p.win_idx[wrow + pos] = static_cast<int16_t>(e);
            st_val(p.win_val, p.v_dtype, wrow + pos, a[i]);
            s_eidx[slot * kbs + pos] = static_cast<int16_t>(e);
            s_eval[slot * kbs + pos] = round_to(a[i], p.v_dtype);
            s_a[e] = 0.0;
        } else {
            s_a[e] = a[i];
            if (want_report) rep[2] += a[i] * a[i];
        }
    }
    // Older rows of this block's window (any order; consumed in slot order in P6).
    const int filled = p.filled;
    for (int t = tid; t < filled * kb; t += NT) {
        const int r = t / kb;
        if (r == slot) continue;
        const int j = t - r * kb;
        const int64_t g = (b * p.m + r) * static_cast<int64_t>(kbs) + j;
        s_eidx[r * kbs + j] = p.win_idx[g];
        s_eval[r * kbs + j] = ld_val(p.win_val, p.v_dtype, g);
    }
    __syncthreads();

    // ---- lossless EF: the residual itself is the new error (optim.cpp:172-173) ----
    if (p.dense) {
        for (int i = tid; i < len; i += NT) {
            p.dense[base + i] = s_a[i];
            if (want_report) rep[3] += s_a[i] * s_a[i];
        }
    }
    // ---- P4: re-quantize the residual (quantize.cpp:15-24, 42-55, 142-162) ----
    // (bucket-split mode: launch_requant_buckets does it over the whole vector)
    for (int bk = (p.dense || p.split_sel) ? nbk : warp; bk < nbk; bk += NW) {
        const int s = bk * bucket;
        const int n = min(bucket, len - s);
        double lo = s_a[s], hi = s_a[s];
        for (int i = lane; i < n; i += 32) {
            const double x = s_a[s + i];
            lo = fmin(lo, x);
            hi = fmax(hi, x);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
            hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
        }
        const double level = (lo == hi) ? 0.0 : __ddiv_rn(__dsub_rn(hi, lo), max_code);
        if (lane == 0) p.meta[bk0 + bk] = make_double2(lo, hi);
        // Guarded reciprocal: floor((x-lo)*(1/level)+0.5) equals the exact
        // quotient's unless t lands within 7e-15 of an integer; such t take
        // the IEEE division.
        const bool fast = level >= 0x1p-1000;
        // |d·rn(1/level) − d/level| ≤ q·1.5·2^-52 with q ≤ max_code: a margin of
        // max_code·2^-44 (≥ 1e-12) around the integers is conservative.
        const double guard = fmax(1e-12, max_code * 0x1p-44);
        const double rinv = fast ? __drcp_rn(level) : 0.0;
        for (int i = lane; i < n; i += 32) {
            const double x = s_a[s + i];
            uint32_t c = 0;
            if (level != 0.0) {
                const double d = __dsub_rn(x, lo);
                double t = __dadd_rn(__dmul_rn(d, rinv), 0.5);
                double f = floor(t);
                const double fr = __dsub_rn(t, f);
                if (!fast || fr < guard || fr > 1.0 - guard) f = floor(__dadd_rn(__ddiv_rn(d, level), 0.5));
                f = f < 0.0 ? 0.0 : (f > max_code ? max_code : f);
                c = static_cast<uint32_t>(f);
            }
            if (bits > 8) s_code32[s + i] = c;
            else s_code[s + i] = static_cast<uint8_t>(c);
            if (want_report) {
                const double en = __dadd_rn(__dmul_rn(static_cast<double>(c), level), lo);
                rep[3] += en * en;
            }
        }
    }
    __syncthreads();

    // ---- P5: pack (quantize.cpp:102-114): LSB-first bit stream; the block
    // starts on a byte boundary (block * bits % 8 == 0, checked at create) ----
    if (!p.dense && !p.split_sel && bits != 4) {
        const int nbytes = (len * bits + 7) / 8;
        for (int jb = tid; jb < nbytes; jb += NT) {
            uint32_t byte = 0;
            const int b0 = jb * 8;
            for (int i = b0 / bits; i < len && i * bits < b0 + 8; ++i) {
                const int sh = i * bits - b0;  // bit position of code i relative to this byte
                const uint32_t c = bits > 8 ? s_code32[i] : s_code[i];
                byte |= sh >= 0 ? (c << sh) : (c >> -sh);
            }
            p.codes[(base * bits) / 8 + jb] = static_cast<uint8_t>(byte & 0xFFu);
        }
    }
    for (int i = (p.dense || p.split_sel || bits != 4) ? (len + 1) / 2 : tid; i < (len + 1) / 2; i += NT) {
        const uint32_t lo4 = s_code[2 * i];
        const uint32_t hi4 = (2 * i + 1 < len) ? s_code[2 * i + 1] : 0u;
        p.codes[(base >> 1) + i] = static_cast<uint8_t>(lo4 | (hi4 << 4));
    }

    // ---- P6: ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    // Each coordinate gets one owner entry; the owner accumulates every row's
    // contribution in physical slot order (rows hold unique indices, so a row
    // pass is race-free), matching the reference's summation order exactly.
    const int nent = filled * kb;
    for (int t = tid; t < nent; t += NT) {
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        atomicExch(&s_owner[s_eidx[e]], e);  // any entry of the coordinate may own it
    }
    __syncthreads();
    for (int t = tid; t < nent; t += NT) {
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        if (s_owner[s_eidx[e]] == e) {
            s_z1[e] = 0.0;
            s_z2[e] = 0.0;
        }
    }
    __syncthreads();
    for (int r = 0; r < filled; ++r) {
        const double w1 = p.w1[r], w2 = p.w2[r];
        for (int j = tid; j < kb; j += NT) {
            const int e = r * kbs + j;
            const int o = s_owner[s_eidx[e]];
            const double v = s_eval[e];
            s_z1[o] = __dadd_rn(s_z1[o], __dmul_rn(w1, v));
            s_z2[o] = __dadd_rn(s_z2[o], __dmul_rn(w2, __dmul_rn(v, v)));
        }
        __syncthreads();
    }
    for (int t = tid; t < nent; t += NT) {
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        const int idx = s_eidx[e];
        if (s_owner[idx] != e) continue;
        const double mhat = __dmul_rn(s_z1[e], p.scale1);
        const double vhat = __dmul_rn(s_z2[e], p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        const double th = ld_val(p.params, p.p_dtype, base + idx);
        st_val(p.params, p.p_dtype, base + idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        if (want_report && u != 0.0) rep[4] += 1.0;
    }
    if (want_report) block_sum5<NT>(rep, s_red, p.partials + b * kReportFields);
}

__global__ void finite_scan_kernel(const void* g, int dt, int64_t n, unsigned int* flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        bad |= !isfinite(ld_val(g, dt, i));
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// check_finite on a = g + e (compress.cpp:76 via topk_blockwise) for f64
// gradients, the only dtype whose sum with a finite EF can overflow: e is the
// decoded quantized buffer (quantize.cpp:164-178, LSB-first codes) or the
// dense residual of a lossless engine.
__global__ void finite_scan_a_kernel(const double* g, const uint8_t* codes, const double2* meta,
                                     const double* dense, int64_t n, int64_t bucket, int bits,
                                     unsigned int* flag) {
    bool bad = false;
    const uint32_t cmask = (1u << bits) - 1u;
    const double max_code = static_cast<double>(cmask);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        double e;
        if (dense) {
            e = dense[i];
        } else {
            const double2 mt = meta[i / bucket];
            const double level = mt.x == mt.y ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), max_code);
            const int64_t pos = i * bits;
            uint32_t w = codes[pos >> 3];
            for (int k = 1; 8 * k < int(pos & 7) + bits; ++k) w |= uint32_t(codes[(pos >> 3) + k]) << (8 * k);
            e = __dadd_rn(__dmul_rn(static_cast<double>((w >> (pos & 7)) & cmask), level), mt.x);
        }
        bad |= !isfinite(__dadd_rn(g[i], e));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void report_reduce_kernel(const double* partials, int64_t nblocks, double* out) {
    __shared__ double red[1024 / 32][kReportFields];
    double v[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x)
        for (int f = 0; f < kReportFields; ++f) v[f] += partials[b * kReportFields + f];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int f = 0; f < kReportFields; ++f) {
        for (int off = 16; off > 0; off >>= 1) v[f] += __shfl_xor_sync(0xFFFFFFFFu, v[f], off);
        if (lane == 0) red[warp][f] = v[f];
    }
    __syncthreads();
    if (threadIdx.x < kReportFields) {
        double s = 0.0;
        for (int w = 0; w < int(blockDim.x / 32); ++w) s += red[w][threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// θ at every live window entry of blocks [b0, b1), same [block][m][kb_stride]
// layout as the ring (ma_step_host's sparse D2H: θ changes only there).
__global__ void gather_window_theta_kernel(const int16_t* win_idx, const void* theta, int pdt, void* out,
                                           int64_t b0, int64_t b1, int m, int kbs, int kb, int filled,
                                           int64_t block, int64_t dim) {
    const int64_t per = int64_t(filled) * kbs;
    const int64_t n = (b1 - b0) * per;
    const int psz = pdt == F64 ? 8 : (pdt == F32 ? 4 : 2);
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = b0 + t / per;
        const int64_t rj = t % per;
        const int j = static_cast<int>(rj % kbs);
        const int64_t len = (b + 1) * block <= dim ? block : dim - b * block;
        if (j >= (kb < len ? kb : len)) continue;
        const int64_t q = (b * m) * kbs + rj;  // ring position (rows r < filled are contiguous)
        const int64_t e = b * block + win_idx[q];
        const unsigned char* src = static_cast<const unsigned char*>(theta) + e * psz;
        unsigned char* dst = static_cast<unsigned char*>(out) + q * psz;
        if (psz == 2) *reinterpret_cast<uint16_t*>(dst) = *reinterpret_cast<const uint16_t*>(src);
        else if (psz == 4) *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
        else *reinterpret_cast<uint64_t*>(dst) = *reinterpret_cast<const uint64_t*>(src);
    }
}

// Bucket-split re-quantization (quantize.cpp:15-24, 42-55, 102-114, 142-162
// over the whole vector): one warp per bucket, two passes over its elements —
// exact fp64 (lo, hi) of the residual, then the codes by the guarded
// reciprocal / IEEE quotient of the generic kernel's P4. Nibbles go to the
// zeroed codes_new with atomicOr (an odd bucket shares a byte with the next).
__global__ void requant_buckets_kernel(const void* grads, int gdt, const uint8_t* codes_old, uint8_t* codes_new,
                                       double2* meta, const uint32_t* sel, int64_t dim, int64_t bucket,
                                       double* err2) {
    const int lane = threadIdx.x & 31;
    const int64_t nq = (dim + bucket - 1) / bucket;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    double e2 = 0.0;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += warps) {
        const int64_t s0 = q * bucket, s1 = s0 + bucket < dim ? s0 + bucket : dim;
        const double2 old = meta[q];
        const double lvl0 = old.x == old.y ? 0.0 : __ddiv_rn(__dsub_rn(old.y, old.x), 15.0);
        auto resid = [&](int64_t i) {
            if ((sel[i >> 5] >> (i & 31)) & 1u) return 0.0;
            const uint32_t c = (codes_old[i >> 1] >> ((i & 1) * 4)) & 15u;
            return __dadd_rn(ld_val(grads, gdt, i), __dadd_rn(__dmul_rn(static_cast<double>(c), lvl0), old.x));
        };
        double lo = CUDART_INF, hi = -CUDART_INF;
        for (int64_t i = s0 + lane; i < s1; i += 32) {
            const double r = resid(i);
            lo = r < lo ? r : lo;
            hi = r > hi ? r : hi;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off), oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
            lo = ol < lo ? ol : lo;
            hi = oh > hi ? oh : hi;
        }
        const double level = lo == hi ? 0.0 : __ddiv_rn(__dsub_rn(hi, lo), 15.0);
        const bool fast = level >= 0x1p-1000;
        const double rinv = fast ? __drcp_rn(level) : 0.0;
        const double guard = fmax(1e-12, 15.0 * 0x1p-44);
        for (int64_t i = s0 + lane; i < s1; i += 32) {
            uint32_t c = 0;
            if (level != 0.0) {
                const double d = __dsub_rn(resid(i), lo);
                const double t = __dadd_rn(__dmul_rn(d, rinv), 0.5);
                double f = floor(t);
                const double fr = __dsub_rn(t, f);
                if (!fast || fr < guard || fr > 1.0 - guard) f = floor(__dadd_rn(__ddiv_rn(d, level), 0.5));
                f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                c = static_cast<uint32_t>(f);
            }
            if (c) atomicOr(reinterpret_cast<unsigned int*>(codes_new) + (i >> 3), c << (4 * (i & 7)));
            if (err2) {
                const double en = __dadd_rn(__dmul_rn(static_cast<double>(c), level), lo);
                e2 += en * en;
            }
        }
        if (lane == 0) meta[q] = make_double2(lo, hi);
    }
    if (err2) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) e2 += __shfl_xor_sync(0xFFFFFFFFu, e2, off);
        if (lane == 0 && e2 != 0.0) atomicAdd(err2, e2);
    }
}

__global__ void fill_synthetic_kernel(void* out, int dt, int64_t n, uint64_t seed, uint64_t step,
                                      int64_t offset, int levels) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t gi = static_cast<uint64_t>(offset + i);
        const double v = ma_synth_value(levels, seed, step, gi);
        st_val(out, dt, i, v);
    }
}

template <int NT, int EPT>
cudaError_t launch_variant(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    const size_t smem = SmemLayout(NT, EPT, a.block, a.bucket, a.m, a.kb_stride, a.bits > 8 ? 4 : 1).total;
    auto k = microadam_step_kernel<NT, EPT>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k<<<static_cast<unsigned>(nblocks), NT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

size_t step_smem_bytes(int nt, int ept, int block, int bucket, int m, int kb_stride, int bits) {
    return SmemLayout(nt, ept, block, bucket, m, kb_stride, bits > 8 ? 4 : 1).total;
}

Variant pick_variant(int block) {
    if (block <= 128) return {64, 2};
    if (block <= 1024) return {128, 8};
    if (block <= 4096) return {256, 16};
    if (block <= 8192) return {512, 16};
    return {0, 0};
}

cudaError_t launch_step(const StepArgs& a, Variant v, int64_t nblocks, cudaStream_t s) {
    if (nblocks <= 0) return cudaSuccess;
    if (nblocks > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    switch (v.nt) {
        case 64: return launch_variant<64, 2>(a, nblocks, s);
        case 128: return launch_variant<128, 8>(a, nblocks, s);
        case 256: return launch_variant<256, 16>(a, nblocks, s);
        case 512: return launch_variant<512, 16>(a, nblocks, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

cudaError_t launch_requant_buckets(const void* grads, int gdt, const uint8_t* codes_old, uint8_t* codes_new,
                                   double2* meta, const uint32_t* sel, int64_t dim, int64_t bucket, double* err2,
                                   cudaStream_t s) {
    const int64_t nq = (dim + bucket - 1) / bucket;
    const int64_t want = (nq + 7) / 8;
    const unsigned grid = static_cast<unsigned>(want < 148 * 32 ? want : 148 * 32);
    requant_buckets_kernel<<<grid, 256, 0, s>>>(grads, gdt, codes_old, codes_new, meta, sel, dim, bucket, err2);
    return cudaGetLastError();
}

cudaError_t launch_finite_scan(const void* g, int dtype, int64_t n, unsigned int* flag,
                               cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    finite_scan_kernel<<<grid, 256, 0, s>>>(g, dtype, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_finite_scan_a(const double* g, const uint8_t* codes, const double2* meta, const double* dense,
                                 int64_t n, int64_t bucket, int bits, unsigned int* flag, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    finite_scan_a_kernel<<<grid, 256, 0, s>>>(g, codes, meta, dense, n, bucket, bits, flag);
    return cudaGetLastError();
}

cudaError_t launch_report_reduce(const double* partials, int64_t nblocks, double* out5,
                                 cudaStream_t s) {
    report_reduce_kernel<<<1, 1024, 0, s>>>(partials, nblocks, out5);
    return cudaGetLastError();
}

cudaError_t launch_gather_window_theta(const int16_t* win_idx, const void* theta, int pdt, void* out, int64_t b0,
                                      int64_t b1, int m, int kbs, int kb, int filled, int64_t block, int64_t dim,
                                      cudaStream_t s) {
    const int64_t n = (b1 - b0) * int64_t(filled) * kbs;
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    gather_window_theta_kernel<<<grid, 256, 0, s>>>(win_idx, theta, pdt, out, b0, b1, m, kbs, kb, filled, block, dim);
    return cudaGetLastError();
}

struct RsSrc {
    const void* p[kMaxRanks];
};

// Unfused reduce-scatter of ma_step_reduce: fixed rank order, fp32 sums for
// bf16/f32 gradients (fp64 for f64), one multiply by the scale, one rounding.
__global__ void reduce_grads_kernel(RsSrc src, int n, float scale, int gdt, void* dst, int64_t e0, int64_t e1) {
    for (int64_t e = e0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < e1;
         e += int64_t(gridDim.x) * blockDim.x) {
        if (gdt == F64) {
            double acc = static_cast<const double*>(src.p[0])[e];
            for (int r = 1; r < n; ++r) acc = __dadd_rn(acc, static_cast<const double*>(src.p[r])[e]);
            static_cast<double*>(dst)[e] = __dmul_rn(acc, static_cast<double>(scale));
        } else if (gdt == F32) {
            float acc = static_cast<const float*>(src.p[0])[e];
            for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, static_cast<const float*>(src.p[r])[e]);
            static_cast<float*>(dst)[e] = __fmul_rn(acc, scale);
        } else {
            auto ld = [&](int r) {
                return __uint_as_float(uint32_t(static_cast<const uint16_t*>(src.p[r])[e]) << 16);
            };
            float acc = ld(0);
            for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, ld(r));
            static_cast<uint16_t*>(dst)[e] = static_cast<uint16_t>(bf16x2_bits(__fmul_rn(acc, scale), 0.0f));
        }
    }
}

cudaError_t launch_reduce_grads(const void* const* srcs, int nsrc, float scale, int gdt, void* dst, int64_t e0,
                                int64_t e1, cudaStream_t s) {
    if (e1 <= e0) return cudaSuccess;
    if (nsrc < 1 || nsrc > kMaxRanks) return cudaErrorInvalidValue;
    RsSrc src{};
    for (int r = 0; r < nsrc; ++r) src.p[r] = srcs[r];
    const int64_t want = (e1 - e0 + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    reduce_grads_kernel<<<grid, 256, 0, s>>>(src, nsrc, scale, gdt, dst, e0, e1);
    return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(void* out, int dtype, int64_t n, uint64_t seed, uint64_t step,
                                  int64_t offset, int levels, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148 * 32 ? want : 148 * 32);
    fill_synthetic_kernel<<<grid, 256, 0, s>>>(out, dtype, n, seed, step, offset, levels);
    return cudaGetLastError();
}

}  // namespace ma
