// ma_fast.cu — the fast sm_100a MicroAdam step kernel (default layouts).
//
// Same contract and bit-exact results as the generic kernel (ma_kernels.cu),
// restructured for the HBM roofline:
//
//  * Lane-contiguous groups: a thread owns runs of 8 consecutive elements, so
//    g / EF codes / bucket grids arrive as 16 B / 4 B / 16 B vector loads, a
//    4-bit code word is one 32-bit store, and a B_q-bucket is LPB = B_q/8
//    adjacent lanes: the bucket min/max is 7 register DMNMX + log2(LPB)
//    shuffle levels (quantize.cpp:15-24).
//  * θ is staged HBM→smem→HBM with 1-D bulk async copies (cp.async.bulk +
//    mbarrier, SASS UBLKCP), issued at CTA start and overlapped with P1-P4.
//  * Block Top-K fast path: each block carries a 32-bit threshold on the
//    high word of |a| from the previous step (≈ the 64th-largest key). The
//    candidates above it (typically ~64) are ranked exactly by
//    (|a| desc, index asc) — high word first, full 64-bit key and index only
//    on ties — so the selection is always exact; the threshold only decides
//    the work. Outside [k_b, kCandCap] candidates the generic radix select
//    runs. The selection lands in a per-element bitmap whose word prefix
//    gives every selected element its ascending window position.
//  * ADAM_STATS without a per-row barrier: each window coordinate gets one
//    owner entry (last-writer-wins + a duplicate mark). Coordinates present in
//    one row take z = 0 + w·v directly; duplicated ones are re-summed by the
//    owner over the rows in physical slot order (binary search in the sorted
//    rows), reproducing window.cpp:32-39's summation order exactly.
//  * Quantization uses q = (x-lo)·RN(1/level) in fp64 and a 2^-20 fixed-point
//    fp32 guard: floor(q+1/2) is exact unless q+1/2 lies within 32·2^-20 of an
//    integer (error bound ≈ 3·2^-20), in which case the IEEE quotient decides.
#include <cstdlib>

#include "../../include/ma_synth.h"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kTarget = 64;  // candidate rank that seeds the next step's threshold

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t hi_key(double x) {
    return static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(x)) >> 32) & 0x7FFFFFFFu;
}
__device__ __forceinline__ bool not_finite(double x) {
    return (hi_key(x) & 0x7FF00000u) == 0x7FF00000u;
}

__host__ __device__ inline int dtype_bytes(int dt) { return dt == F64 ? 8 : (dt == F32 ? 4 : 2); }

struct FastLayout {
    size_t theta, eval, ckey, red, eidx, owner, hist, ckhi, cidx, sel, tmpb, wpref, misc, dup, selm,
        bar, total;
    __host__ __device__ static size_t take(size_t& off, size_t bytes, size_t align = 16) {
        off = (off + align - 1) & ~(align - 1);
        const size_t r = off;
        off += bytes;
        return r;
    }
    __host__ __device__ FastLayout(int nt, int block, int m, int kbs, int pdt) {
        const size_t ent = size_t(m) * size_t(kbs);
        const size_t nwords = size_t((block + 31) / 32);
        size_t off = 0;
        theta = take(off, size_t(block) * size_t(dtype_bytes(pdt)), 128);
        eval = take(off, ent * 8);
        ckey = take(off, size_t(kCandCap + 4) * 8);
        red = take(off, size_t(nt / 32) * kReportFields * 8);
        bar = take(off, 8, 8);
        eidx = take(off, ent * 2);
        owner = take(off, size_t(block) * 2);
        hist = take(off, 256 * 4);
        ckhi = take(off, size_t(kCandCap + 4) * 4);
        cidx = take(off, size_t(kCandCap + 4) * 4);
        sel = take(off, nwords * 4);
        tmpb = take(off, nwords * 4);
        wpref = take(off, (nwords + 1) * 4);
        misc = take(off, 96 * 4);
        dup = take(off, size_t(block));
        selm = take(off, size_t(block));
        total = (off + 127) & ~size_t(127);
    }
};

// Load 8 consecutive elements starting at element i (8-aligned) as doubles.
__device__ __forceinline__ void ld8(const void* p, int dt, int64_t i, double (&x)[8]) {
    if (dt == BF16) {
        const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p) + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
            x[2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
        }
    } else if (dt == F32) {
        const float4 v0 = *reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
        const float4 v1 = *reinterpret_cast<const float4*>(static_cast<const float*>(p) + i + 4);
        x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
        x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
    } else {
        const double2* q = reinterpret_cast<const double2*>(static_cast<const double*>(p) + i);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 v = q[k];
            x[2 * k] = v.x;
            x[2 * k + 1] = v.y;
        }
    }
}

// Exclusive prefix (in word order) of popcounts of bits[0..nwords) into pref;
// one warp. pref[nwords] = total.
__device__ __forceinline__ void word_prefix(const uint32_t* bits, int nwords, int* pref) {
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int base = 0; base < nwords; base += 32) {
        const int w = base + lane;
        const int v = w < nwords ? __popc(bits[w]) : 0;
        int incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += t;
        }
        if (w < nwords) pref[w] = carry + incl - v;
        carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    if (lane == 0) pref[nwords] = carry;
}

template <int NT, int G, int LPB>
__global__ void __launch_bounds__(NT, (G == 2 ? (NT >= 512 ? 1 : 3) : (NT >= 512 ? 2 : 4))) microadam_step_fast(const __grid_constant__ StepArgs p) {
    constexpr int NW = NT / 32;
    constexpr int EPT = 8 * G;
    constexpr int BUCKET = 8 * LPB;
    static_assert(EPT <= 32, "selection masks are 32-bit");
    extern __shared__ __align__(128) unsigned char smem[];
    const int m = p.m, kbs = p.kb_stride, block = p.block;
    const FastLayout L(NT, block, m, kbs, p.p_dtype);
    unsigned char* s_theta = smem + L.theta;
    double* s_eval = reinterpret_cast<double*>(smem + L.eval);
    uint64_t* s_ckey = reinterpret_cast<uint64_t*>(smem + L.ckey);
    double* s_red = reinterpret_cast<double*>(smem + L.red);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    int16_t* s_eidx = reinterpret_cast<int16_t*>(smem + L.eidx);
    uint16_t* s_owner = reinterpret_cast<uint16_t*>(smem + L.owner);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    uint32_t* s_ckhi = reinterpret_cast<uint32_t*>(smem + L.ckhi);
    int* s_cidx = reinterpret_cast<int*>(smem + L.cidx);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + L.sel);
    uint32_t* s_tmpb = reinterpret_cast<uint32_t*>(smem + L.tmpb);
    int* s_wpref = reinterpret_cast<int*>(smem + L.wpref);
    int* s_misc = reinterpret_cast<int*>(smem + L.misc);
    uint8_t* s_dup = reinterpret_cast<uint8_t*>(smem + L.dup);
    uint8_t* s_selm = reinterpret_cast<uint8_t*>(smem + L.selm);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = p.block_offset + blockIdx.x;
    const int64_t base = b * static_cast<int64_t>(block);
    const int len = static_cast<int>(min(static_cast<int64_t>(block), p.dim - base));
    const int kb = min(p.per_block_k, len);
    const int nwords = (len + 31) / 32;
    const int psz = dtype_bytes(p.p_dtype);
    const bool bulk = ((len * psz) & 15) == 0;
    const bool want_report = p.partials != nullptr;
    const int filled = p.filled, slot = p.slot;
    auto elem = [&](int s) { return ((s >> 3) * NT + tid) * 8 + (s & 7); };

    // ---- prologue: θ tile HBM→smem (bulk async), bitmaps, window rows ----
    if (tid == 0 && bulk) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        mbar_expect_tx(s_bar, static_cast<uint32_t>(len * psz));
        bulk_g2s(s_theta, static_cast<const unsigned char*>(p.params) + base * psz,
                 static_cast<uint32_t>(len * psz), s_bar);
    }
    for (int w = tid; w < nwords; w += NT) {
        s_sel[w] = 0;
        s_tmpb[w] = 0;
    }
    if (tid == 0) s_misc[NW + 1] = -1;  // 0xFFFFFFFF: atomicMin seed (fallback path)

    // P1 loads: g (vector), 4-bit code word, bucket grid.
    double a[EPT];
    uint32_t cw[G];
    double2 mt[G];
    uint32_t valid = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int e0 = (g * NT + tid) * 8;
        cw[g] = 0;
        mt[g] = make_double2(0.0, 0.0);
        if (e0 < len) {
            const int n8 = min(8, len - e0);
            double x[8];
            if (n8 == 8) {
                ld8(p.grads, p.g_dtype, base + e0, x);
                cw[g] = *reinterpret_cast<const uint32_t*>(p.codes + ((base + e0) >> 1));
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = i < n8 ? ld_val(p.grads, p.g_dtype, base + e0 + i) : 0.0;
                for (int i = 0; i < (n8 + 1) / 2; ++i)
                    cw[g] |= static_cast<uint32_t>(p.codes[((base + e0) >> 1) + i]) << (8 * i);
            }
            mt[g] = p.meta[(base + e0) / BUCKET];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[g * 8 + i] = x[i];
            valid |= ((n8 == 8) ? 0xFFu : ((1u << n8) - 1u)) << (8 * g);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[g * 8 + i] = 0.0;
        }
    }
    // Older window rows of this block into smem; owner/dup marks (pass A).
    for (int t = tid; t < filled * kb; t += NT) {
        const int r = t / kb;
        if (r == slot) continue;
        const int j = t - r * kb;
        const int64_t gi = (b * m + r) * static_cast<int64_t>(kbs) + j;
        const int e = r * kbs + j;
        const int idx = p.win_idx[gi];
        s_eidx[e] = static_cast<int16_t>(idx);
        s_eval[e] = ld_val(p.win_val, p.v_dtype, gi);
        s_owner[idx] = static_cast<uint16_t>(e);
        s_dup[idx] = 0;
    }
    if (!bulk)
        for (int i = tid; i < len; i += NT)
            st_val(s_theta, p.p_dtype, i, ld_val(p.params, p.p_dtype, base + i));

    // ---- P1: decode + accumulate (quantize.cpp:164-178, optim.cpp:166-168) ----
    bool bad = false;
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double lo = mt[g].x, hi = mt[g].y;
        const double level = (lo == hi) ? 0.0 : __ddiv_rn(__dsub_rn(hi, lo), 15.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int s = g * 8 + i;
            if (!((valid >> s) & 1u)) continue;
            const double gv = a[s];
            const double e = __dadd_rn(__dmul_rn(static_cast<double>((cw[g] >> (4 * i)) & 15u), level), lo);
            a[s] = __dadd_rn(gv, e);
            bad |= not_finite(gv) | not_finite(a[s]);
            if (want_report) {
                rep[0] += gv * gv;
                rep[1] += a[s] * a[s];
            }
        }
    }
    if (p.check_finite && bad) atomicOr(p.flag, 1u);

    // ---- P2: block Top-K (compress.cpp:39-53, 73-85) ----
    const uint32_t T = max(p.thresh[b], 1u);
    uint32_t cmask = 0;
#pragma unroll
    for (int s = 0; s < EPT; ++s)
        if (((valid >> s) & 1u) && hi_key(a[s]) >= T) cmask |= 1u << s;
    const int cnt = __popc(cmask);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) s_misc[warp] = incl;
    __syncthreads();  // [1] counts, bitmaps zeroed, window rows + pass-A marks

    int c = 0, wbase = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int v = s_misc[w];
        wbase += (w < warp) ? v : 0;
        c += v;
    }
    uint32_t tnext = 0;
    if (c >= kb && c <= kCandCap) {
        // Fast path: exact rank among the candidates.
        int slot_c = wbase + incl - cnt;
#pragma unroll
        for (int s = 0; s < EPT; ++s) {
            if ((cmask >> s) & 1u) {
                s_ckey[slot_c] = key_of(a[s]);
                s_ckhi[slot_c] = hi_key(a[s]);
                s_cidx[slot_c] = elem(s);
                ++slot_c;
            }
        }
        if (tid < 4) s_ckhi[c + tid] = 0;  // pad for 16-byte scans (T >= 1, so pads never tie)
        __syncthreads();  // [2]
        const int target = (c > kTarget ? kTarget : c) - 1;
        for (int t = tid; t < c; t += NT) {
            const uint32_t kh = s_ckhi[t];
            int above = 0, eq = 0;
            for (int q = 0; q < c; q += 4) {
                const uint4 v = *reinterpret_cast<const uint4*>(s_ckhi + q);
                above += (v.x > kh) + (v.y > kh) + (v.z > kh) + (v.w > kh);
                eq += (v.x == kh) + (v.y == kh) + (v.z == kh) + (v.w == kh);
            }
            int rank = above;
            if (eq > 1) {
                const uint64_t kt = s_ckey[t];
                const int it = s_cidx[t];
                for (int q = 0; q < c; ++q) {
                    if (q == t || s_ckhi[q] != kh) continue;
                    const uint64_t kq = s_ckey[q];
                    rank += (kq > kt) || (kq == kt && s_cidx[q] < it);
                }
            }
            const int idx = s_cidx[t];
            if (rank < kb) atomicOr(&s_sel[idx >> 5], 1u << (idx & 31));
            if (rank == target) s_misc[NW] = static_cast<int>(c > kTarget ? kh : (kh > (1u << 16) ? kh - (1u << 16) : 1u));
        }
    } else {
        // Generic exact radix select (rare: first step, distribution shifts, ties).
        auto tie_rank = [&](uint32_t mask, int (&r)[EPT]) {
            __syncthreads();
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const uint32_t bits = (mask >> (8 * g)) & 0xFFu;
                const int e0 = (g * NT + tid) * 8;
                if (bits) atomicOr(&s_tmpb[e0 >> 5], bits << (e0 & 31));
            }
            __syncthreads();
            if (warp == 0) word_prefix(s_tmpb, nwords, s_wpref);
            __syncthreads();
#pragma unroll
            for (int s = 0; s < EPT; ++s) {
                if ((mask >> s) & 1u) {
                    const int e = elem(s);
                    r[s] = s_wpref[e >> 5] + __popc(s_tmpb[e >> 5] & ((1u << (e & 31)) - 1u));
                }
            }
        };
        for (int i = tid; i < len; i += NT) s_selm[i] = 0;
        __syncthreads();
        const uint32_t sel = block_topk<NT, EPT>(a, valid, kb, s_hist, s_misc + 32, s_ckey, s_cidx,
                                                 s_selm, elem, tie_rank);
        uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint32_t bits = (sel >> (8 * g)) & 0xFFu;
            const int e0 = (g * NT + tid) * 8;
            if (bits) atomicOr(&s_sel[e0 >> 5], bits << (e0 & 31));
        }
#pragma unroll
        for (int s = 0; s < EPT; ++s)
            if ((sel >> s) & 1u) kmin = min(kmin, hi_key(a[s]));
        kmin = __reduce_min_sync(0xFFFFFFFFu, kmin);
        if (lane == 0) atomicMin(reinterpret_cast<unsigned int*>(&s_misc[NW + 1]), kmin);
        (void)tnext;
    }
    __syncthreads();  // [3] selection bitmap complete
    if (warp == 0) word_prefix(s_sel, nwords, s_wpref);
    if (tid == 0) {
        uint32_t tn;
        if (c >= kb && c <= kCandCap) {
            tn = static_cast<uint32_t>(s_misc[NW]);
        } else {
            const uint32_t kmin = static_cast<uint32_t>(s_misc[NW + 1]);
            tn = kmin > (1u << 17) ? kmin - (1u << 17) : 1u;  // ~1/8 binade below the k-th key
        }
        p.thresh[b] = tn;
    }
    __syncthreads();  // [4] word prefix

    // ---- P3: window row `slot` (window.cpp:14-26) + residual (compress.cpp:95-102)
    // ---- P4: 4-bit re-quantization (quantize.cpp:7-24, 42-55, 102-114, 142-162)
    const int64_t wrow = (b * m + slot) * static_cast<int64_t>(kbs);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int e0 = (g * NT + tid) * 8;
        const uint32_t vmask = (valid >> (8 * g)) & 0xFFu;
        uint32_t sel8 = 0;
        int pos = 0;
        if (vmask) {
            const uint32_t word = s_sel[e0 >> 5];
            sel8 = (word >> (e0 & 31)) & 0xFFu;
            pos = s_wpref[e0 >> 5] + __popc(word & ((1u << (e0 & 31)) - 1u));
        }
        double lo = __longlong_as_double(0x7FF0000000000000ll);  // +inf
        double hi = -lo;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int s = g * 8 + i;
            if (!((vmask >> i) & 1u)) continue;
            if ((sel8 >> i) & 1u) {
                const int e = e0 + i;
                p.win_idx[wrow + pos] = static_cast<int16_t>(e);
                st_val(p.win_val, p.v_dtype, wrow + pos, a[s]);
                s_eidx[slot * kbs + pos] = static_cast<int16_t>(e);
                s_eval[slot * kbs + pos] = round_to(a[s], p.v_dtype);
                s_owner[e] = static_cast<uint16_t>(slot * kbs + pos);
                s_dup[e] = 0;
                ++pos;
                a[s] = 0.0;
            } else if (want_report) {
                rep[2] += a[s] * a[s];
            }
            lo = fmin(lo, a[s]);
            hi = fmax(hi, a[s]);
        }
#pragma unroll
        for (int off = 1; off < LPB; off <<= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
            hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
        }
        if (!vmask) continue;
        const double level = (lo == hi) ? 0.0 : __ddiv_rn(__dsub_rn(hi, lo), 15.0);
        const bool fastq = level >= 0x1p-1000;
        const double rinv = fastq ? __drcp_rn(level) : 0.0;
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int s = g * 8 + i;
            if (!((vmask >> i) & 1u) || level == 0.0) continue;
            const double d = __dsub_rn(a[s], lo);
            uint32_t code;
            bool exact = !fastq;
            if (fastq) {
                const float qf = __double2float_rn(__dmul_rn(d, rinv));
                const uint32_t x = __float2uint_rz(__fmaf_rn(qf, 1048576.0f, 524288.0f));
                const uint32_t frac = x & 0xFFFFFu;
                code = x >> 20;
                exact = frac < 32u || frac > 0xFFFFFu - 32u;
            }
            if (exact) {
                double f = floor(__dadd_rn(__ddiv_rn(d, level), 0.5));
                f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                code = static_cast<uint32_t>(f);
            }
            word |= code << (4 * i);
        }
        if (want_report) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (!((vmask >> i) & 1u)) continue;
                const double en =
                    __dadd_rn(__dmul_rn(static_cast<double>((word >> (4 * i)) & 15u), level), lo);
                rep[3] += en * en;
            }
        }
        if (vmask == 0xFFu) {
            *reinterpret_cast<uint32_t*>(p.codes + ((base + e0) >> 1)) = word;
        } else {
            const int n8 = __popc(vmask);
            for (int i = 0; i < (n8 + 1) / 2; ++i)
                p.codes[((base + e0) >> 1) + i] = static_cast<uint8_t>(word >> (8 * i));
        }
        if ((lane & (LPB - 1)) == 0) p.meta[(base + e0) / BUCKET] = make_double2(lo, hi);
    }
    __syncthreads();  // [5] new row + its marks

    // ---- P6: ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    const int nent = filled * kb;
    for (int t = tid; t < nent; t += NT) {  // pass B: duplicate marks
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        const int idx = s_eidx[e];
        if (s_owner[idx] != e) s_dup[idx] = 1;
    }
    __syncthreads();  // [6]
    if (bulk)
        while (!mbar_try_wait(s_bar, 0)) {
        }
    for (int t = tid; t < nent; t += NT) {  // pass C: owners accumulate + update θ
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        const int idx = s_eidx[e];
        if (s_owner[idx] != e) continue;
        double z1, z2;
        if (!s_dup[idx]) {
            const double v = s_eval[e];
            z1 = __dadd_rn(0.0, __dmul_rn(p.w1[r], v));
            z2 = __dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(v, v)));
        } else {
            z1 = 0.0;
            z2 = 0.0;
            for (int rr = 0; rr < filled; ++rr) {
                const int16_t* row = s_eidx + rr * kbs;
                int lo_i = 0, hi_i = kb;  // lower_bound in the ascending row
                while (lo_i < hi_i) {
                    const int mid = (lo_i + hi_i) >> 1;
                    if (row[mid] < idx) lo_i = mid + 1; else hi_i = mid;
                }
                if (lo_i < kb && row[lo_i] == idx) {
                    const double v = s_eval[rr * kbs + lo_i];
                    z1 = __dadd_rn(z1, __dmul_rn(p.w1[rr], v));
                    z2 = __dadd_rn(z2, __dmul_rn(p.w2[rr], __dmul_rn(v, v)));
                }
            }
        }
        const double mhat = __dmul_rn(z1, p.scale1);
        const double vhat = __dmul_rn(z2, p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        const double th = ld_val(s_theta, p.p_dtype, idx);
        st_val(s_theta, p.p_dtype, idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        if (want_report && u != 0.0) rep[4] += 1.0;
    }
    fence_proxy_async_smem();
    __syncthreads();  // [7] θ tile final
    if (bulk) {
        if (tid == 0) {
            bulk_s2g(static_cast<unsigned char*>(p.params) + base * psz, s_theta,
                     static_cast<uint32_t>(len * psz));
            bulk_wait_read();
        }
    } else {
        for (int i = tid; i < len; i += NT)
            st_val(p.params, p.p_dtype, base + i, ld_val(s_theta, p.p_dtype, i));
    }
    if (want_report) {
        // deterministic block reduction (same tree as the generic kernel)
#pragma unroll
        for (int f = 0; f < kReportFields; ++f) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) s_red[warp * kReportFields + f] = rep[f];
        }
        __syncthreads();
        if (tid < kReportFields) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += s_red[w * kReportFields + tid];
            p.partials[b * kReportFields + tid] = s;
        }
    }
}

template <int NT, int G, int LPB>
cudaError_t launch_fast_variant(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    const size_t smem = FastLayout(NT, a.block, a.m, a.kb_stride, a.p_dtype).total;
    auto k = microadam_step_fast<NT, G, LPB>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k<<<static_cast<unsigned>(nblocks), NT, smem, s>>>(a);
    return cudaGetLastError();
}

template <int LPB>
cudaError_t launch_fast_lpb(const StepArgs& a, Variant v, int64_t nblocks, cudaStream_t s) {
    if (v.nt == 128 && v.ept == 8) return launch_fast_variant<128, 1, LPB>(a, nblocks, s);
    if (v.nt == 256 && v.ept == 8) return launch_fast_variant<256, 1, LPB>(a, nblocks, s);
    if (v.nt == 256 && v.ept == 16) return launch_fast_variant<256, 2, LPB>(a, nblocks, s);
    if (v.nt == 512 && v.ept == 8) return launch_fast_variant<512, 1, LPB>(a, nblocks, s);
    if (v.nt == 512 && v.ept == 16) return launch_fast_variant<512, 2, LPB>(a, nblocks, s);
    return cudaErrorInvalidConfiguration;
}

}  // namespace

Variant pick_fast_variant(int block, int bucket, int m, int kb_stride) {
    if (block % 8 != 0 || block % bucket != 0) return {0, 0};
    if (bucket != 16 && bucket != 32 && bucket != 64) return {0, 0};
    if (m * kb_stride > 65535) return {0, 0};
    if (block <= 1024) return {128, 8};
    if (block <= 2048) return {256, 8};
    if (block <= 4096) {
        const char* g2 = std::getenv("MA_FAST_G2");  // A/B switch: 256 threads x 16 elements
        return (g2 && g2[0] == '1') ? Variant{256, 16} : Variant{512, 8};
    }
    if (block <= 8192) return {512, 16};
    return {0, 0};
}

size_t fast_smem_bytes(Variant v, int block, int m, int kb_stride, int p_dtype) {
    return FastLayout(v.nt, block, m, kb_stride, p_dtype).total;
}

cudaError_t launch_step_fast(const StepArgs& a, Variant v, int64_t nblocks, cudaStream_t s) {
    if (nblocks <= 0) return cudaSuccess;
    if (nblocks > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    switch (a.bucket) {
        case 16: return launch_fast_lpb<2>(a, v, nblocks, s);
        case 32: return launch_fast_lpb<4>(a, v, nblocks, s);
        case 64: return launch_fast_lpb<8>(a, v, nblocks, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace ma
