// ma_tile.cu — the default sm_100a MicroAdam step kernel ("tile" kernel).
//
// One 128-thread CTA owns one B_d = 4096 Top-K block at a time
// (optim.cpp:164-190); CTAs are persistent and double-buffered: while a block
// is processed, the next block's inputs stream HBM -> shared memory by TMA
//   * g through a 2-D tensor map with the 128-byte swizzle (UTMALDG), so every
//     thread reads its 32 consecutive gradients bank-conflict free,
//   * the packed EF codes, the bucket (lo, hi), θ and the block's m window
//     rows (indices + values) by 1-D bulk copies (UBLKCP),
// all completing on one mbarrier per stage. Thread t owns elements
// [32t, 32t + 32): half of one B_q = 64 bucket, so bucket min/max is a
// register reduction plus one shuffle.
//
// The streaming work is fp32 (packed FFMA2/FADD2, 3-input FMNMX) with proven
// error bounds; every decision fp32 cannot settle is re-taken in the
// reference's fp64 arithmetic, so results are bit-identical to the exact
// kernels:
//  * pass 1 (optim.cpp:166-168, quantize.cpp:164-178): a32 = g + (c·level + lo)
//    kept in 32 registers; |a32| screened against the Top-K threshold carried
//    from the previous step. Hits are re-evaluated exactly (fp64) into the
//    candidate list.
//  * Top-K (compress.cpp:39-53, 73-85): warp 0 bisects the k_b-th largest key
//    over the candidates (ties: full key, then lower index) while warps 1-3
//    mark the old window rows for ADAM_STATS; overfull screens are refined
//    from the hit masks; a missed threshold falls back to an exact radix
//    descent over the block in shared memory.
//  * pass 2 (compress.cpp:95-102, quantize.cpp:15-24, 42-55, 102-114): the
//    residual from the registers; bucket min/max by FMNMX3; one FFMA2 per two
//    elements yields y = 257 + 2t + G (t = the code's quotient estimate) whose
//    mantissa holds the 4-bit code at bits 16..19 (packed by byte permutes)
//    and a 15-bit fraction. Elements with y within G of an integer are the
//    only ones whose status is undecided: the bucket's min and max candidates
//    (y ~ 257, 287) — re-evaluated exactly to give the exact (lo, hi) — and
//    quotients near a rounding boundary — recoded by the IEEE quotient
//    (quantize.cpp:51-53). Buckets outside the bounds run exactly in fp64.
//  * ADAM_STATS + update (window.cpp:28-46, optim.cpp:183-187) from the rows
//    and θ in shared memory: seen/dup bitmaps; coordinates in one row take the
//    bf16-θ fp32 screen (exact fp64 otherwise); duplicated coordinates are
//    summed in physical slot order by warp 0 (match.any over the ordered list).
//
// Error bounds (per bucket q, previous (lo, hi), M = max(|lo|, |hi|)):
//   |a32 - a| <= E_q + |a32| 2^-23,  E_q = M 2^-21 + 2^-120   (ma_warp.cu)
//   pass 2: eps = E_q + max|r32| 2^-22 bounds |r32 - r|; with R = M32 - m32,
//   |t - q| <= 60 eps / R + 2^-20 (ratio and product roundings), and the
//   constant of the FFMA adds <= |c| 2^-24. The guard G (in y units) is
//   2 (90 eps / R + |c| 2^-23 + 2^-14); buckets with G > 1/8 go exact.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <math_constants.h>

#include <mutex>

#include "ma_async.cuh"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kT = 128;           // threads per CTA (one 4096-element Top-K block)
constexpr int kBlk = 4096;
constexpr int kNbk = 64;          // B_q = 64 buckets per block
constexpr int kRefineMax = 1024;  // hits refined from the masks (else the radix path)
constexpr int kTarget = 64;       // carried-threshold target hit count

#ifndef MA_TILE_MINB
#define MA_TILE_MINB 5  // resident CTAs per SM the tile kernel is compiled for
#endif

// Per-CTA shared memory (bytes from a 1024-aligned base; host and device agree).
struct TLay {
    uint32_t g, codes, meta, theta, widx, wval, stage, st0, st1;
    uint32_t sel, seen, dup, wpref, cval, cidx, hist, dupl, misc, bars, total;
    __host__ __device__ TLay(int gsz, int psz, int vsz, int m, int kbs, int cap, int nent) {
        size_t o = 0;
        g = 0;                 o = size_t(kBlk) * gsz;  // swizzle-128B TMA destination
        codes = uint32_t(o);   o += kBlk / 2;
        meta = uint32_t(o);    o += kNbk * 16;
        widx = uint32_t(o);    o = align_up(o + size_t(m) * kbs * 2, 16);
        wval = uint32_t(o);    o = align_up(o + size_t(m) * kbs * vsz, 16);
        stage = uint32_t(align_up(o, 1024));
        st0 = 0;
        st1 = stage;
        o = 2 * size_t(stage);
        theta = uint32_t(o);   o = align_up(o + size_t(kBlk) * psz, 16);  // single-buffered
        sel = uint32_t(o);     o += 512;
        seen = uint32_t(o);    o += 512;
        dup = uint32_t(o);     o += 512;
        wpref = uint32_t(o);   o = align_up(o + (cap * 2 > 512 ? size_t(cap) * 2 : 512), 16);  // word prefix; tie members
        cval = uint32_t(o);    o = align_up(o + size_t(cap) * 8, 16);
        cidx = uint32_t(o);    o = align_up(o + size_t(cap) * 2, 16);
        hist = uint32_t(o);    o += 512;
        dupl = uint32_t(o);    o = align_up(o + size_t(nent + 4 * 32 + 4) * 4, 16);
        misc = uint32_t(o);    o += 64 * 4;
        bars = uint32_t(o);    o += 24;
        total = uint32_t(align_up(o, 128)) + 1024;  // + base alignment slack
    }
};

// misc[] slots
enum : int {
    kCnt = 0,       // candidate counter (2 slots: iteration parity)
    kNeedSlow = 16, // warp 0 found the candidates short of k_b (2 slots: parity)
    kNcand = 2,     // slow path: candidate count (-1: selection written to the bitmap)
    kPfx = 3,       // slow path: key prefix high word
    kDigit = 4,     // radix digit / refine results (3 ints)
    kWarpTot = 8,   // per-warp scan totals (4)
    kDupN = 12,     // per-warp duplicate-entry counts (4)
};

template <int GDT_, int PDT_, int VDT_, int CAPL_>
struct TK {
    static constexpr int GDT = GDT_, PDT = PDT_, VDT = VDT_, CAPL = CAPL_, CAP = 32 * CAPL_;
    static constexpr int gsz = GDT == F32 ? 4 : 2;
    static constexpr int psz = PDT == F32 ? 4 : 2;
    static constexpr int vsz = VDT == F32 ? 4 : 2;
};

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}

template <int DT>
__device__ __forceinline__ float ldf(const unsigned char* p, int i) {
    if constexpr (DT == F32) return reinterpret_cast<const float*>(p)[i];
    else return __uint_as_float(uint32_t(reinterpret_cast<const uint16_t*>(p)[i]) << 16);
}
template <int DT>
__device__ __forceinline__ double ldd(const unsigned char* p, int i) {
    return static_cast<double>(ldf<DT>(p, i));
}

// Byte offset of block element e in the swizzled g tile (128-byte rows, the
// 16-byte chunk index XORed with row % 8 — CU_TENSOR_MAP_SWIZZLE_128B).
template <int GDT>
__device__ __forceinline__ uint32_t g_off(int e_) {
    constexpr uint32_t esz = GDT == F32 ? 4u : 2u;
    constexpr uint32_t per_row = 128u / esz, per_chunk = 16u / esz;
    const uint32_t e = static_cast<uint32_t>(e_);
    const uint32_t row = e / per_row, chunk = (e % per_row) / per_chunk;
    return row * 128u + ((chunk ^ (row & 7u)) << 4) + (e % per_chunk) * esz;
}

// Exact a of block element e (optim.cpp:166-168, quantize.cpp:164-178): the
// same fp64 operations as the reference, from the staged g and codes.
template <int GDT>
__device__ __forceinline__ double exact_a(const unsigned char* st_g, const unsigned char* st_codes, int e, double lo,
                                          double level) {
    const double g = static_cast<double>(
        GDT == F32 ? *reinterpret_cast<const float*>(st_g + g_off<GDT>(e))
                   : __uint_as_float(uint32_t(*reinterpret_cast<const uint16_t*>(st_g + g_off<GDT>(e))) << 16));
    const uint32_t ue = static_cast<uint32_t>(e);
    const uint32_t c = (st_codes[ue >> 1] >> ((ue & 1u) * 4u)) & 15u;
    return __dadd_rn(g, __dadd_rn(__dmul_rn(static_cast<double>(c), level), lo));
}

// quantize_nearest's IEEE path (quantize.cpp:51-53). Out of line: rare.
__device__ __noinline__ uint32_t ieee_code(double x, double lo, double level) {
    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(x, lo), level), 0.5));
    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
    return static_cast<uint32_t>(f);
}

// level = rn((hi - lo) / 15) (QuantParams, quantize.cpp:7-13) without a
// division: q0 = rn(x c) with c = rn(1/15); the remainder r = x - 15 q0 is
// exact (one FMA), and rn(q0 + r c) is the correctly rounded quotient: x/15 is
// never a rounding midpoint (x - 15 m is an odd multiple of ulp/2 for every
// midpoint m, so its distance to one is >= ulp 2^-5) while q0 + r c differs
// from x/15 by <= ulp 2^-53. Quotients near the subnormal range (and x = 0,
// inf, NaN) take the IEEE division.
__device__ __forceinline__ double div15(double x) {
    if (!(x >= 0x1p-960 && x <= 0x1p1000)) return __ddiv_rn(x, 15.0);
    const double c = 0x1.1111111111111p-4;  // rn(1/15)
    const double q0 = __dmul_rn(x, c);
    const double r = __fma_rn(-q0, 15.0, x);
    return __fma_rn(r, c, q0);
}

// t / kb for 0 <= t < 2^20 via a float reciprocal and one fix-up each way.
__device__ __forceinline__ int div_kb(int t, int kb, float inv_kb) {
    int r = __float2int_rz(static_cast<float>(t) * inv_kb);
    r -= (r * kb > t);
    r += ((r + 1) * kb <= t);
    return r;
}

// The whole bucket in fp64 (pass 2 fallback for buckets outside the fp32
// bounds): exact residuals, min/max with the partner thread, IEEE codes.
// Both threads of the bucket call it (pair_mask = their lanes). Out of line: rare.
struct ExactOut {
    uint4 w;
    double lo, hi;
};
template <int GDT>
__device__ __noinline__ ExactOut exact_bucket(const unsigned char* st_g, const unsigned char* st_codes, int tid,
                                              uint32_t selw, double lo_old, double lv_old, uint32_t pair_mask) {
    double mn = CUDART_INF, mx = -CUDART_INF;
    for (int i = 0; i < 32; ++i) {
        const double r = ((selw >> i) & 1u) ? 0.0 : exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo_old, lv_old);
        mn = i == 0 ? r : (r < mn ? r : mn);
        mx = i == 0 ? r : (r > mx ? r : mx);
    }
    const double omn = __shfl_xor_sync(pair_mask, mn, 1), omx = __shfl_xor_sync(pair_mask, mx, 1);
    // std::min / std::max keep the earlier element on ties (quantize.cpp:18-21)
    const bool first = (tid & 1) == 0;
    ExactOut o;
    o.lo = first ? (omn < mn ? omn : mn) : (mn < omn ? mn : omn);
    o.hi = first ? (omx > mx ? omx : mx) : (mx > omx ? mx : omx);
    o.w = make_uint4(0u, 0u, 0u, 0u);
    const double level = o.lo == o.hi ? 0.0 : div15(__dsub_rn(o.hi, o.lo));
    if (level == 0.0) return o;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const double r = ((selw >> i) & 1u) ? 0.0 : exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo_old, lv_old);
        w[i >> 3] |= ieee_code(r, o.lo, level) << (4 * (i & 7));
    }
    o.w = make_uint4(w[0], w[1], w[2], w[3]);
    return o;
}

// a32 of block element e recomputed from the stage with the very operations of
// pass 1 (fp32, round-to-nearest: identical bits).
template <int GDT>
__device__ __forceinline__ float a32_at(const unsigned char* st_g, const unsigned char* st_codes, int e, float lo32,
                                        float lv32) {
    const float g = GDT == F32 ? *reinterpret_cast<const float*>(st_g + g_off<GDT>(e))
                               : __uint_as_float(uint32_t(*reinterpret_cast<const uint16_t*>(st_g + g_off<GDT>(e))) << 16);
    const uint32_t ue = static_cast<uint32_t>(e);
    const uint32_t c = (st_codes[ue >> 1] >> ((ue & 1u) * 4u)) & 15u;
    const float cf = __fadd_rn(__uint_as_float(0x4B000000u | c), -8388608.0f);
    return __fadd_rn(g, __fmaf_rn(cf, lv32, lo32));
}

// bf16 θ update screen (optim.cpp:183-187 rounded to bf16): the fp32 estimate
// x32 = θ - lr32·u32 is within |lr u| 2^-20.6 + |x| 2^-24 of the fp64 result
// (9 fp32 roundings of at most 2^-24 and a 2-ulp division, against < 2^-49 for
// the fp64 chain), i.e. within m = |lr u| 2^(132 - ex) + 4 ulps of x32's
// binade (ex = its biased exponent; x2 across a binade edge, x2 slack). When
// the 16 bits below the bf16 mantissa are more than m from the rounding
// midpoint 0x8000, x and x32 round to the same bf16: store it, return true.
__device__ __forceinline__ bool bf16_screen_store(const StepArgs& p, int64_t gidx, float th, float u, float den) {
    const float x = __fmaf_rn(-p.lr32, u, th);
    const uint32_t xb = __float_as_uint(x);
    const uint32_t ex = (xb >> 23) & 0xFFu;
    const int mid = static_cast<int>(xb & 0xFFFFu) - 0x8000;
    const float lu = fabsf(p.lr32 * u);
    const bool range = ex >= 27u && ex <= 227u && den < 0x1p120f && lu <= __uint_as_float((ex + 4u) << 23);
    const int marg = __float2int_ru(lu * __uint_as_float((259u - ex) << 23)) + 4;
    if (!(range && (mid > marg || mid < -marg))) return false;
    static_cast<uint16_t*>(p.params)[gidx] = static_cast<uint16_t>((xb + 0x7FFFu + ((xb >> 16) & 1u)) >> 16);
    return true;
}

// ADAM_STATS + update of one coordinate with a single window entry
// (window.cpp:28-46 with one term, optim.cpp:183-187), fp64, reference order.
template <int PDT>
__device__ __noinline__ void exact_single(const StepArgs* pp, int64_t gidx, double th, double v, int r) {
    const StepArgs& p = *pp;
    const double mhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w1[r], v)), p.scale1);
    const double vhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(v, v))), p.scale2);
    const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
    st_t<PDT>(p.params, gidx, __dsub_rn(th, __dmul_rn(p.lr, u)));
}

// Radix descent over the block in shared memory (all threads): the carried
// threshold missed (first step, drift) or keys tie heavily. 7-bit digits of
// the 63-bit |a| key from bit 62, until the keys at or above the prefix fit
// the candidate list (gathered; returns their count and sets misc[kPfx] to the
// prefix's high word), or all 63 bits are fixed with more ties than that: then
// the selection (every key above K* plus the lowest-index ties,
// compress.cpp:43-48) goes straight to the bitmap and -1 is returned.
template <class K>
__device__ __noinline__ int slow_select(const StepArgs* pp, unsigned char* smem, const unsigned char* st, double lo,
                                        double level, int kc) {
    const StepArgs& p = *pp;
    const TLay L(K::gsz, K::psz, K::vsz, p.m, p.kb_stride, K::CAP, p.m * p.per_block_k);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + L.sel);
    int* misc = reinterpret_cast<int*>(smem + L.misc);
    double* s_cval = reinterpret_cast<double*>(smem + L.cval);
    int16_t* s_cidx = reinterpret_cast<int16_t*>(smem + L.cidx);
    const unsigned char* st_g = st + L.g;
    const unsigned char* st_codes = st + L.codes;
    const int kb = p.per_block_k;
    auto key = [&](int i) { return key_of(exact_a<K::GDT>(st_g, st_codes, tid * 32 + i, lo, level)); };
    uint64_t prefix = 0, pmask = 0;
    int need = kb, above_total = 0, binc = 0;
    for (int sh = 56;; sh -= 7) {
        hist[tid] = 0;
        __syncthreads();
        uint64_t kmx = 0;
        for (int i = 0; i < 32; ++i) {
            const uint64_t k = key(i);
            kmx = k > kmx ? k : kmx;
            if ((k & pmask) == prefix) atomicAdd(&hist[(k >> sh) & 127u], 1u);
        }
        if (sh == 56 && p.check_finite && (kmx >> 48) >= 0x7FF0u) atomicOr(p.flag, 1u);  // inf/NaN in g or a
        __syncthreads();
        if (warp == 0) {
            const uint32_t h0 = hist[lane * 4], h1 = hist[lane * 4 + 1], h2 = hist[lane * 4 + 2],
                           h3 = hist[lane * 4 + 3];
            const int local = int(h0 + h1 + h2 + h3);
            int incl = local;  // inclusive suffix over lanes >= lane
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_down_sync(0xFFFFFFFFu, incl, off);
                if (lane + off < 32) incl += t;
            }
            const int s3 = incl - local + int(h3), s2 = s3 + int(h2), s1 = s2 + int(h1), s0 = s1 + int(h0);
            int dl = -1;
            if (s0 >= need) dl = lane * 4;
            if (s1 >= need) dl = lane * 4 + 1;
            if (s2 >= need) dl = lane * 4 + 2;
            if (s3 >= need) dl = lane * 4 + 3;
            const int d = __reduce_max_sync(0xFFFFFFFFu, dl);
            const int owner = d >> 2, sd = d & 3;
            const int sfx = sd == 0 ? s0 : (sd == 1 ? s1 : (sd == 2 ? s2 : s3));
            const int hd = int(sd == 0 ? h0 : (sd == 1 ? h1 : (sd == 2 ? h2 : h3)));
            const int above = __shfl_sync(0xFFFFFFFFu, sfx - hd, owner);
            const int bc = __shfl_sync(0xFFFFFFFFu, hd, owner);
            if (lane == 0) {
                misc[kDigit] = d;
                misc[kDigit + 1] = above;
                misc[kDigit + 2] = bc;
            }
        }
        __syncthreads();
        const int d = misc[kDigit], above = misc[kDigit + 1];
        binc = misc[kDigit + 2];
        above_total += above;
        need -= above;
        prefix |= static_cast<uint64_t>(d) << sh;
        pmask |= uint64_t(127) << sh;
        if (above_total + binc <= K::CAP || sh == 0) break;
    }
    __syncthreads();  // everyone has read misc[kDigit..]
    if (above_total + binc <= K::CAP) {
        if (tid == 0) misc[kc] = 0;
        __syncthreads();
        for (int i = 0; i < 32; ++i) {
            const double a = exact_a<K::GDT>(st_g, st_codes, tid * 32 + i, lo, level);
            if (key_of(a) >= prefix) {
                const int q = atomicAdd(&misc[kc], 1);
                s_cval[q] = a;
                s_cidx[q] = static_cast<int16_t>(tid * 32 + i);
            }
        }
        if (tid == 0) misc[kPfx] = static_cast<int>(prefix >> 32);
        __syncthreads();
        return above_total + binc;
    }
    // All 63 bits fixed: K* = prefix; the first `need` keys equal to K* in index
    // order are selected (thread t owns elements 32t.. in order: a block scan).
    uint32_t gt = 0, eq = 0;
    for (int i = 0; i < 32; ++i) {
        const uint64_t k = key(i);
        gt |= static_cast<uint32_t>(k > prefix) << i;
        eq |= static_cast<uint32_t>(k == prefix) << i;
    }
    const int ne = __popc(eq);
    int incl = ne;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) misc[kWarpTot + warp] = incl;
    __syncthreads();
    int before = incl - ne;
    for (int w = 0; w < warp; ++w) before += misc[kWarpTot + w];
    uint32_t selm = gt;
    for (int i = 0; i < 32; ++i)
        if ((eq >> i) & 1u) {
            if (before < need) selm |= 1u << i;
            ++before;
        }
    s_sel[tid] = selm;
    if (tid == 0) misc[kPfx] = static_cast<int>(prefix >> 32);
    if (p.dbg && tid == 0) atomicAdd(p.dbg + 0, 1u);
    __syncthreads();
    return -1;
}

// Duplicated window coordinates (window.cpp:32-39: terms summed in physical
// slot order), warp 0. The per-warp ordered lists concatenate to the entry
// order (slot, position); taken 32 entries at a time, match.any groups a
// coordinate's entries, the coordinate's running sums live in shared memory
// (indexed by its rank among the duplicated coordinates), and one lane per
// coordinate applies the update at the end. Out of line.
template <class K>
__device__ __noinline__ void dup_updates(const StepArgs* pp, unsigned char* smem, unsigned char* st, int64_t base) {
    const StepArgs& p = *pp;
    const TLay L(K::gsz, K::psz, K::vsz, p.m, p.kb_stride, K::CAP, p.m * p.per_block_k);
    const int lane = threadIdx.x & 31;
    const int kbs = p.kb_stride;
    const int* misc = reinterpret_cast<const int*>(smem + L.misc);
    const uint32_t* s_dup = reinterpret_cast<const uint32_t*>(smem + L.dup);
    const int* dupl = reinterpret_cast<const int*>(smem + L.dupl);
    const unsigned char* swv = st + L.wval;
    const unsigned char* sth = smem + L.theta;
    const int seg = (p.m * p.per_block_k + 3) / 4 + 32;  // per-warp list segment
    int nseg[4];
    int ndup = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        nseg[w] = misc[kDupN + w];
        ndup += nseg[w];
    }
    if (ndup == 0) return;
    if (p.dbg && lane == 0) atomicAdd(p.dbg + 5, static_cast<unsigned>(ndup));
    auto entry = [&](int q) {  // q-th entry of the concatenated list
        int w = 0;
        while (w < 3 && q >= nseg[w]) q -= nseg[w++];
        return dupl[w * seg + q];
    };
    // θ -= lr·u from the exact fp64 moments (optim.cpp:183-187): the bf16 screen
    // of the division, the fp64 chain otherwise
    auto finish = [&](int idx, double z1, double z2) {
        const double mhat = __dmul_rn(z1, p.scale1);
        const double vhat = __dmul_rn(z2, p.scale2);
        const float th32 = ldf<K::PDT>(sth, idx);
        if constexpr (K::PDT == BF16) {
            const float den = __fadd_rn(p.eps32, __fsqrt_rn(__double2float_rn(vhat)));
            const float u = __fdividef(__double2float_rn(mhat), den);
            if (bf16_screen_store(p, base + idx, th32, u, den)) return;
        }
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        st_t<K::PDT>(p.params, base + idx, __dsub_rn(static_cast<double>(th32), __dmul_rn(p.lr, u)));
    };
    if (ndup <= 32) {
        // one list entry per lane (list order = physical slot order): the
        // coordinate's peers by match.any, its lowest lane sums their terms in
        // lane order (window.cpp:32-39) and applies the update
        const bool has = lane < ndup;
        const int x = has ? entry(lane) : 0;
        const int idx = x >> 16, r = (x >> 8) & 0xFF, pos = x & 0xFF;
        double t1 = 0.0, t2 = 0.0;
        if (has) {
            const double v = ldd<K::VDT>(swv, r * kbs + pos);
            t1 = __dmul_rn(p.w1[r], v);
            t2 = __dmul_rn(p.w2[r], __dmul_rn(v, v));
        }
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, has ? idx : -1 - lane);
        const int cnt = has ? __popc(peers) : 0;
        const int maxc = __reduce_max_sync(0xFFFFFFFFu, cnt);
        uint32_t rem = peers;
        double z1 = 0.0, z2 = 0.0;
        for (int k = 0; k < maxc; ++k) {
            const int src = rem ? __ffs(rem) - 1 : lane;
            rem &= rem - 1;
            const double a1 = __shfl_sync(0xFFFFFFFFu, t1, src);
            const double a2 = __shfl_sync(0xFFFFFFFFu, t2, src);
            if (k < cnt) {
                z1 = __dadd_rn(z1, a1);
                z2 = __dadd_rn(z2, a2);
            }
        }
        if (has && (__ffs(peers) - 1) == lane) finish(idx, z1, z2);
        return;
    }
    // rank of a duplicated coordinate among all of them (word prefix of s_dup)
    int* s_dpref = reinterpret_cast<int*>(smem + L.wpref);
    uint32_t dv[4];
    int loc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        dv[k] = s_dup[lane * 4 + k];
        loc += __popc(dv[k]);
    }
    int incl = loc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    const int ndupc = __shfl_sync(0xFFFFFFFFu, incl, 31);
    int run = incl - loc;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_dpref[lane * 4 + k] = run;
        run += __popc(dv[k]);
    }
    // running sums in the stage's g tile (dead after pass 2)
    double2* zz = reinterpret_cast<double2*>(st + L.g);
    int16_t* zc = reinterpret_cast<int16_t*>(st + L.g + kBlk * K::gsz - 2 * 512);
    const int zcap = (kBlk * K::gsz - 2 * 512) / 16 < 512 ? (kBlk * K::gsz - 2 * 512) / 16 : 512;
    __syncwarp();
    for (int id0 = 0; id0 < ndupc; id0 += zcap) {
        const int nz = min(zcap, ndupc - id0);
        for (int i = lane; i < nz; i += 32) zz[i] = make_double2(0.0, 0.0);
        __syncwarp();
        for (int c0 = 0; c0 < ndup; c0 += 32) {
            bool has = c0 + lane < ndup;
            const int x = has ? entry(c0 + lane) : 0;
            const int idx = x >> 16, r = (x >> 8) & 0xFF, pos = x & 0xFF;
            int id = 0;
            if (has) {
                id = s_dpref[idx >> 5] + __popc(s_dup[idx >> 5] & ((1u << (idx & 31)) - 1u)) - id0;
                has = id >= 0 && id < nz;
            }
            double t1 = 0.0, t2 = 0.0;
            if (has) {
                const double v = ldd<K::VDT>(swv, r * kbs + pos);
                t1 = __dmul_rn(p.w1[r], v);
                t2 = __dmul_rn(p.w2[r], __dmul_rn(v, v));
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, has ? idx : -1 - lane);
            const int cnt = has ? __popc(peers) : 0;
            const int maxc = __reduce_max_sync(0xFFFFFFFFu, cnt);
            const bool leader = has && (__ffs(peers) - 1) == lane;
            double z1 = 0.0, z2 = 0.0;
            if (leader) {
                const double2 z0 = zz[id];
                z1 = z0.x;
                z2 = z0.y;
            }
            uint32_t rem = peers;
            for (int k = 0; k < maxc; ++k) {  // lane order = list order = slot order
                const int src = rem ? __ffs(rem) - 1 : lane;
                rem &= rem - 1;
                const double a1 = __shfl_sync(0xFFFFFFFFu, t1, src);
                const double a2 = __shfl_sync(0xFFFFFFFFu, t2, src);
                if (k < cnt) {
                    z1 = __dadd_rn(z1, a1);
                    z2 = __dadd_rn(z2, a2);
                }
            }
            if (leader) {
                zz[id] = make_double2(z1, z2);
                zc[id] = static_cast<int16_t>(idx);
            }
            __syncwarp();
        }
        for (int i = lane; i < nz; i += 32) {
            const double2 z = zz[i];
            finish(zc[i], z.x, z.y);
        }
        __syncwarp();
    }
}

template <class K>
__global__ void __launch_bounds__(kT, MA_TILE_MINB)
    microadam_step_tile(const __grid_constant__ StepArgs p, const __grid_constant__ CUtensorMap gmap) {
    constexpr int GDT = K::GDT, PDT = K::PDT, VDT = K::VDT, CAPL = K::CAPL, CAP = K::CAP;
    constexpr int gsz = K::gsz, psz = K::psz, vsz = K::vsz;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kb = p.per_block_k, kbs = p.kb_stride, m = p.m, slot = p.slot, filled = p.filled;
    const TLay L(gsz, psz, vsz, m, kbs, CAP, m * kb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + L.sel);
    uint32_t* s_seen = reinterpret_cast<uint32_t*>(smem + L.seen);
    uint32_t* s_dup = reinterpret_cast<uint32_t*>(smem + L.dup);
    int* s_wpref = reinterpret_cast<int*>(smem + L.wpref);
    int16_t* s_memb = reinterpret_cast<int16_t*>(smem + L.wpref);
    double* s_cval = reinterpret_cast<double*>(smem + L.cval);
    int16_t* s_cidx = reinterpret_cast<int16_t*>(smem + L.cidx);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    int* s_dupl = reinterpret_cast<int*>(smem + L.dupl);
    int* misc = reinterpret_cast<int*>(smem + L.misc);
    const int wib = m * kbs * 2, wvb = m * kbs * vsz;
    const uint32_t tx_bytes = uint32_t(kBlk * gsz + kBlk / 2 + kNbk * 16 + wib + wvb);
    const int64_t nb = p.block_count;
    const int seg = (m * kb + 3) / 4 + 32;  // per-warp duplicate-list segment
    const float inv_kb = __frcp_rn(static_cast<float>(kb));

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);  // θ (single buffer)
        fence_mbar_init();
    }
    s_sel[tid] = 0;
    s_seen[tid] = 0;
    s_dup[tid] = 0;
    s_hist[tid] = 0;
    if (tid < 64) misc[tid] = 0;
    __syncthreads();

    auto issue = [&](int64_t bl, int s) {  // thread 0: block bl's inputs into stage s
        const int64_t b = p.block_offset + bl;
        unsigned char* st = smem + (s ? L.st1 : L.st0);
        mbar_expect_tx(&bars[s], tx_bytes);
        tma_2d(st + L.g, &gmap, 0, static_cast<int>(b * (kBlk * gsz / 128)), &bars[s]);
        bulk_g2s(st + L.codes, p.codes + b * (kBlk / 2), kBlk / 2, &bars[s]);
        bulk_g2s(st + L.meta, p.meta + b * kNbk, kNbk * 16, &bars[s]);
        bulk_g2s(st + L.widx, p.win_idx + b * m * kbs, wib, &bars[s]);
        bulk_g2s(st + L.wval, static_cast<const unsigned char*>(p.win_val) + b * m * kbs * vsz, wvb, &bars[s]);
    };
    int64_t bl = blockIdx.x;
    if (tid == 0 && bl < nb) issue(bl, 0);

    for (int it = 0; bl < nb; ++it, bl += gridDim.x) {
        const int s = it & 1;
        const int kc = kCnt + (it & 1);
        const int64_t b = p.block_offset + bl;
        if (tid == 0) {
            fence_proxy_async_smem();
            // θ of this block (read by ADAM_STATS, after pass 1 and the select)
            mbar_expect_tx(&bars[2], uint32_t(kBlk * psz));
            bulk_g2s(smem + L.theta, static_cast<const unsigned char*>(p.params) + b * kBlk * psz, kBlk * psz,
                     &bars[2]);
            if (bl + gridDim.x < nb) issue(bl + gridDim.x, s ^ 1);
        }
        const int64_t base = b * kBlk;
        unsigned char* st = smem + (s ? L.st1 : L.st0);
        const unsigned char* st_g = st + L.g;
        const unsigned char* st_codes = st + L.codes;
        int16_t* swi = reinterpret_cast<int16_t*>(st + L.widx);
        unsigned char* swv = st + L.wval;
        const unsigned char* sth = smem + L.theta;
        const uint32_t tstate = __ldg(p.thresh + b);
        const uint32_t T = tstate & 0xFFFFu;
        mbar_wait(&bars[s], (it >> 1) & 1);

        // ---- bucket grid (quantize.cpp:7-13) and the fp32 screen constants ----
        const double2 mt = reinterpret_cast<const double2*>(st + L.meta)[tid >> 1];
        const double lo = mt.x;
        const double level = (mt.x == mt.y) ? 0.0 : div15(__dsub_rn(mt.y, mt.x));
        const double Mq = fmax(fabs(mt.x), fabs(mt.y));
        float E = __double2float_ru(Mq * 0x1p-21 + 0x1p-120);
        if (!(Mq < 0x1p100)) E = CUDART_INF_F;
        float Tf = CUDART_INF_F;  // T == 0: no carried threshold, no screen hits
        if (T != 0) {
            const double VT = __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(T) << 48));
            Tf = __double2float_rd((VT - static_cast<double>(E)) * (1.0 - 0x1p-22));
        }
        if (!(Tf > 0.0f)) Tf = 0.0f;
        const float lo32 = __double2float_rn(lo), lv32 = __double2float_rn(level);

        // ---- pass 1: a32 = g + (c·level32 + lo32), 32 consecutive elements ----
        float a[32];
        {
            const uint4 cv = reinterpret_cast<const uint4*>(st_codes)[tid];
            const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
            const float2 lv2 = make_float2(lv32, lv32), lo2 = make_float2(lo32, lo32);
            const float2 m23 = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
            for (int w = 0; w < 4; ++w) {  // 8 elements: one 16-byte chunk of bf16 g
                uint32_t gw[8];
                if constexpr (GDT == F32) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int chunk = (2 * w + h) ^ (tid & 7);
                        const uint4 v = *reinterpret_cast<const uint4*>(st_g + tid * 128 + chunk * 16);
                        gw[4 * h + 0] = v.x;
                        gw[4 * h + 1] = v.y;
                        gw[4 * h + 2] = v.z;
                        gw[4 * h + 3] = v.w;
                    }
                } else {
                    const int row = tid >> 1;
                    const int chunk = ((tid & 1) * 4 + w) ^ (row & 7);
                    const uint4 v = *reinterpret_cast<const uint4*>(st_g + row * 128 + chunk * 16);
                    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        gw[2 * k] = vw[k] << 16;
                        gw[2 * k + 1] = vw[k] & 0xFFFF0000u;
                    }
                }
                const uint32_t ce = cw[w] & 0x0F0F0F0Fu, co = (cw[w] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float2 c = make_float2(__uint_as_float(__byte_perm(ce, 0x4B000000u, 0x7540u | k)),
                                           __uint_as_float(__byte_perm(co, 0x4B000000u, 0x7540u | k)));
                    c = __fadd2_rn(c, m23);                           // exact: the code as a float
                    const float2 e = __ffma2_rn(c, lv2, lo2);         // c·level32 + lo32
                    const float2 r = __fadd2_rn(make_float2(__uint_as_float(gw[2 * k]), __uint_as_float(gw[2 * k + 1])), e);
                    a[8 * w + 2 * k] = r.x;
                    a[8 * w + 2 * k + 1] = r.y;
                }
            }
        }
        // hit <=> a^2 - T2 >= 0 with T2 = rd(Tf^2): a superset of |a| >= Tf (a
        // NaN gives the canonical positive NaN: a hit); the sign bits of one
        // FFMA2 per pair are gathered by funnel shifts (bit i = element i).
        uint32_t hits;
        {
            const float T2 = __fmul_rd(Tf, Tf);
            const float2 nt2 = make_float2(-T2, -T2);
            uint32_t neg = 0;
#pragma unroll
            for (int i = 30; i >= 0; i -= 2) {
                const float2 d = __ffma2_rn(make_float2(a[i], a[i + 1]), make_float2(a[i], a[i + 1]), nt2);
                neg = __funnelshift_l(__float_as_uint(d.y), neg, 1);
                neg = __funnelshift_l(__float_as_uint(d.x), neg, 1);
            }
            hits = ~neg;
        }

        // ---- candidates: the hits' exact a (fp64) at atomic list positions ----
        {
            // list positions: a warp scan, one shared atomic per warp (a per-thread
            // atomic on one word serializes the whole CTA)
            const int nh = __popc(hits);
            int incl = nh;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += t;
            }
            int wbase = 0;
            if (lane == 31 && incl) wbase = atomicAdd(&misc[kc], incl);
            int pos = __shfl_sync(0xFFFFFFFFu, wbase, 31) + incl - nh;
            uint32_t hb = hits;
            while (hb) {
                const int i = __ffs(hb) - 1;
                hb &= hb - 1;
                if (pos < CAP) {
                    s_cval[pos] = exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo, level);
                    s_cidx[pos] = static_cast<int16_t>(tid * 32 + i);
                }
                ++pos;
            }
        }
        __syncthreads();  // B1
        const int cnt = misc[kc];
        // the other parity's counters were last used in the previous block: reset
        // them for the next one (no end-of-block barrier: see B3)
        if (tid == 0) {
            misc[kCnt + ((it + 1) & 1)] = 0;
            misc[kNeedSlow + ((it + 1) & 1)] = 0;
        }
        int ncand = -1;
        uint32_t base16 = T, floor16 = T;
        bool slow = !(T != 0 && cnt >= kb && cnt <= kRefineMax);
        if (!slow && cnt > CAP) {
            // Overfull screen: a key16 histogram of the exact hits at or above T
            // (from the masks, no block re-read) gives T1 = T + d with >= k_b
            // hits; those at or above T1 become the candidates.
            {
                uint32_t hb = hits;
                while (hb) {
                    const int i = __ffs(hb) - 1;
                    hb &= hb - 1;
                    const uint32_t k16 = hi_key(exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo, level)) >> 16;
                    if (k16 >= T) atomicAdd(&s_hist[min(k16 - T, 31u)], 1u);
                }
            }
            __syncthreads();
            if (warp == 0) {
                int sfx = static_cast<int>(s_hist[lane]);
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int t = __shfl_down_sync(0xFFFFFFFFu, sfx, off);
                    if (lane + off < 32) sfx += t;
                }
                const uint32_t ok = __ballot_sync(0xFFFFFFFFu, sfx >= kb);
                const int d = ok ? 31 - __clz(ok) : -1;
                const int n = ok ? __shfl_sync(0xFFFFFFFFu, sfx, d) : 0;
                if (lane == 0) {
                    misc[kDigit] = d;
                    misc[kDigit + 1] = n;
                    misc[kc] = 0;
                }
            }
            __syncthreads();
            const int d = misc[kDigit], n = misc[kDigit + 1];
            s_hist[tid] = 0;
            if (d >= 0 && n <= CAP) {
                const uint32_t T1 = T + static_cast<uint32_t>(d);
                uint32_t hb = hits;
                while (hb) {
                    const int i = __ffs(hb) - 1;
                    hb &= hb - 1;
                    const double av = exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo, level);
                    if ((hi_key(av) >> 16) >= T1) {
                        const int q = atomicAdd(&misc[kc], 1);
                        s_cval[q] = av;
                        s_cidx[q] = static_cast<int16_t>(tid * 32 + i);
                    }
                }
                ncand = n;
                base16 = floor16 = T1;
            } else {
                slow = true;
            }
            if (p.dbg && tid == 0) atomicAdd(p.dbg + 6, 1u);
            __syncthreads();
        } else if (!slow) {
            ncand = cnt;
        }

        // Old window rows (r != slot) marked into seen / dup (any order).
        // entry t = row r * k_b + position: (r, pos) advanced incrementally
        auto mark_rows = [&](int t0, int stride, bool old_only) {
            const int nent = filled * kb;
            const int sq = div_kb(stride, kb, inv_kb), sr = stride - sq * kb;
            int r = div_kb(t0, kb, inv_kb), pos = t0 - r * kb;
            for (int t = t0; t < nent; t += stride) {
                if (!(old_only && r == slot)) {
                    const int idx = swi[r * kbs + pos];
                    const uint32_t bit = 1u << (idx & 31);
                    if (atomicOr(&s_seen[idx >> 5], bit) & bit) atomicOr(&s_dup[idx >> 5], bit);
                }
                r += sq;
                pos += sr;
                if (pos >= kb) {
                    pos -= kb;
                    ++r;
                }
            }
        };
        // Warp 0: exact selection among the candidates, window row, new-row marks,
        // next threshold. Returns false if the candidates hold fewer than k_b
        // keys at or above base16 (then the radix path runs).
        auto select_emit = [&](int nc, uint32_t b16, uint32_t f16, bool from_bitmap) -> bool {
            const int64_t row0 = static_cast<int64_t>(slot) * kbs;
            int16_t* gwi = p.win_idx + b * m * static_cast<int64_t>(kbs);
            unsigned char* gwv = static_cast<unsigned char*>(p.win_val) + b * m * static_cast<int64_t>(kbs) * vsz;
            uint32_t selc = 0;
            uint32_t next_t;
            if (!from_bitmap) {
                uint32_t kh[CAPL];
#pragma unroll
                for (int c = 0; c < CAPL; ++c) {
                    const int q = lane + 32 * c;
                    kh[c] = q < nc ? hi_key(s_cval[q]) : 0u;
                }
                auto count_ge = [&](uint32_t v) {
                    int c = 0;
#pragma unroll
                    for (int s2 = 0; s2 < CAPL; ++s2) c += kh[s2] >= v;
                    return __reduce_add_sync(0xFFFFFFFFu, c);
                };
                int clo = count_ge(b16 << 16);
                if (clo < kb) return false;
                uint32_t kml = 0;
#pragma unroll
                for (int c = 0; c < CAPL; ++c) kml = max(kml, kh[c]);
                const uint32_t kmax = __reduce_max_sync(0xFFFFFFFFu, kml);
                if (p.check_finite && kmax >= 0x7FF00000u && lane == 0) atomicOr(p.flag, 1u);  // inf/NaN
                // bisection for lo with count(lo) >= kb > count(hi), early exit at == kb
                uint32_t lo_k = b16 << 16, hi_k = kmax + 1;
                while (clo != kb && hi_k - lo_k > 1) {
                    const uint32_t mid = lo_k + (hi_k - lo_k) / 2;
                    const int c = count_ge(mid);
                    if (c >= kb) {
                        lo_k = mid;
                        clo = c;
                    } else {
                        hi_k = mid;
                    }
                }
#pragma unroll
                for (int c = 0; c < CAPL; ++c)
                    if (kh[c] > lo_k || (clo == kb && kh[c] == lo_k)) selc |= 1u << c;
                if (clo != kb) {
                    // ties on the k_b-th high word: full key, then the lower index
                    const int need = kb - count_ge(lo_k + 1);
                    int nm = 0;
#pragma unroll
                    for (int c = 0; c < CAPL; ++c) {
                        const bool mem = kh[c] == lo_k && lane + 32 * c < nc;
                        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mem);
                        if (mem) s_memb[nm + __popc(bal & lanemask_lt())] = static_cast<int16_t>(lane + 32 * c);
                        nm += __popc(bal);
                    }
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < CAPL; ++c) {
                        const int q = lane + 32 * c;
                        if (kh[c] == lo_k && q < nc) {
                            const uint64_t kq = key_of(s_cval[q]);
                            const int iq = s_cidx[q];
                            int rank = 0;
                            for (int t = 0; t < nm; ++t) {
                                const int o = s_memb[t];
                                const uint64_t ko = key_of(s_cval[o]);
                                rank += (ko > kq) || (ko == kq && s_cidx[o] < iq);
                            }
                            if (rank < need) selc |= 1u << c;
                        }
                    }
                    __syncwarp();
                    if (p.dbg && lane == 0) atomicAdd(p.dbg + 7, 1u);
                }
#pragma unroll
                for (int c = 0; c < CAPL; ++c)
                    if ((selc >> c) & 1u) {
                        const int e = s_cidx[lane + 32 * c];
                        atomicOr(&s_sel[e >> 5], 1u << (e & 31));
                    }
                // next threshold: the largest key16 t in [floor16, lo16] whose
                // candidate count reaches `want` (drift-corrected target)
                const int planned = T ? static_cast<int>(tstate >> 16) : 0;
                const int target = max(kTarget, kb + (kb >> 1));
                int want = planned ? (target * planned) / max(cnt, 1) : target;
                want = min(max(want, kb + (kb >> 2)), CAP - (CAP >> 2));
                const uint32_t lo16 = lo_k >> 16;
                const uint32_t fl = min(f16, lo16);
                uint32_t t;
                int c = count_ge(fl << 16);
                if (c < want) {
                    t = fl;
                    if (t > 1) {
                        --t;
                        c += c >> 2;
                    }
                } else {
                    uint32_t l2 = fl, h2 = lo16 + 1;
                    while (h2 - l2 > 1) {
                        const uint32_t mid = l2 + (h2 - l2) / 2;
                        const int cm = count_ge(mid << 16);
                        if (cm >= want) {
                            l2 = mid;
                            c = cm;
                        } else {
                            h2 = mid;
                        }
                    }
                    t = l2;
                }
                next_t = t | (static_cast<uint32_t>(min(c, 0xFFFF)) << 16);
            } else {
                const uint32_t h = static_cast<uint32_t>(misc[kPfx]) >> 16;
                next_t = h > 2 ? h - 2 : 1u;
            }
            if (lane == 0) p.thresh[b] = (next_t & 0xFFFFu) ? next_t : (next_t | 1u);
            __syncwarp();
            // window row `slot` (window.cpp:14-26) at ascending positions
            {
                uint32_t wv[4];
                int loc = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    wv[k] = s_sel[lane * 4 + k];
                    loc += __popc(wv[k]);
                }
                int incl = loc;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                    if (lane >= off) incl += t;
                }
                int run = incl - loc;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    s_wpref[lane * 4 + k] = run;
                    run += __popc(wv[k]);
                }
            }
            __syncwarp();
            auto put = [&](int pos, int e, double av) {
                gwi[row0 + pos] = static_cast<int16_t>(e);
                st_t<VDT>(gwv, row0 + pos, av);
                swi[row0 + pos] = static_cast<int16_t>(e);
                st_t<VDT>(swv, row0 + pos, av);
                if constexpr (true) {
                    const uint32_t bit = 1u << (e & 31);  // new-row mark
                    if (atomicOr(&s_seen[e >> 5], bit) & bit) atomicOr(&s_dup[e >> 5], bit);
                }
            };
            if (!from_bitmap) {
#pragma unroll
                for (int c = 0; c < CAPL; ++c)
                    if ((selc >> c) & 1u) {
                        const int q = lane + 32 * c;
                        const int e = s_cidx[q];
                        put(s_wpref[e >> 5] + __popc(s_sel[e >> 5] & ((1u << (e & 31)) - 1u)), e, s_cval[q]);
                    }
            } else {
                for (int w = lane; w < kBlk / 32; w += 32) {
                    uint32_t bits = s_sel[w];
                    int pos = s_wpref[w];
                    // lo / level of element e's bucket: the meta of the stage
                    while (bits) {
                        const int e = w * 32 + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const double2 me = reinterpret_cast<const double2*>(st + L.meta)[e >> 6];
                        const double lv = (me.x == me.y) ? 0.0 : div15(__dsub_rn(me.y, me.x));
                        put(pos++, e, exact_a<GDT>(st_g, st_codes, e, me.x, lv));
                    }
                }
            }
            return true;
        };

        bool marked_old = false;
        if (!slow) {
            if (warp == 0) {
                if (!select_emit(ncand, base16, floor16, false) && lane == 0) misc[kNeedSlow + (it & 1)] = 1;
            } else {
                mark_rows(tid - 32, kT - 32, true);
            }
            marked_old = true;
            __syncthreads();  // B2
            if (misc[kNeedSlow + (it & 1)]) slow = true;
        }
        if (slow) {
            if (!marked_old) mark_rows(tid, kT, true);
            const int nc = slow_select<K>(&p, smem, st, lo, level, kc);  // barriers inside
            if (warp == 0) {
                if (nc >= 0) {
                    const uint32_t ph = static_cast<uint32_t>(misc[kPfx]);
                    select_emit(nc, ph >> 16, (ph + 0xFFFFu) >> 16, false);
                } else {
                    select_emit(0, 0, 0, true);
                }
                if (p.dbg && lane == 0) atomicAdd(p.dbg + 2, 1u);
            }
            __syncthreads();  // B2'
        }

        // ---- pass 2: residual + bucket (lo, hi) + 4-bit codes ----
        const uint32_t selw = s_sel[tid];
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if ((selw >> i) & 1u) a[i] = 0.0f;
        float mn = a[0], mx = a[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) {
            mn = fminf(mn, a[i]);
            mx = fmaxf(mx, a[i]);
        }
        mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 1));
        const float R = mx - mn;
        const float eps = E + fmaxf(fabsf(mn), fabsf(mx)) * 0x1p-22f;
        // y = 257 + 2t + G with t ≈ (r - lo) / level (see the file header)
        const float k2 = __fdividef(30.0f, R);
        const float cmag = 258.0f + fabsf(mn * k2);
        const float G = 2.0f * (90.0f * eps / R + cmag * 0x1p-23f + 0x1p-14f);
        bool fast = R >= 0x1p-100f && R <= 0x1p100f && G <= 0.125f && eps < CUDART_INF_F;
        {
            const bool pf = __shfl_xor_sync(0xFFFFFFFFu, fast, 1);  // (every lane shuffles)
            fast = fast && pf;                                        // uniform per bucket (thread pair)
        }
        const uint32_t pm = 3u << (lane & 30);                  // the pair's lanes
        uint32_t word[4] = {0u, 0u, 0u, 0u};
        double lo_new, hi_new;
        if (fast) {
            const float c2 = __fmaf_rn(-mn, k2, 257.0f + G);
            const uint32_t Gu = static_cast<uint32_t>(2.0f * G * 32768.0f) + 2u;  // 2G in y ulps (2^-15)
            const float2 k22 = make_float2(k2, k2), c22 = make_float2(c2, c2);
            uint32_t yb[32];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float2 y = __ffma2_rn(make_float2(a[i], a[i + 1]), k22, c22);
                yb[i] = __float_as_uint(y.x);
                yb[i + 1] = __float_as_uint(y.y);
            }
            uint32_t fm = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) fm |= static_cast<uint32_t>((yb[i] & 0x7FFFu) < Gu) << i;
            // codes: byte 2 of each y word, packed by byte permutes
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t* y = yb + 8 * w;
                const uint32_t ev = __byte_perm(__byte_perm(y[0], y[2], 0x0062), __byte_perm(y[4], y[6], 0x0062), 0x5410);
                const uint32_t od = __byte_perm(__byte_perm(y[1], y[3], 0x0062), __byte_perm(y[5], y[7], 0x0062), 0x5410);
                // byte 2 of y = exponent LSB (1) << 7 | code: keep the code nibbles
                word[w] = (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
            }
            // flagged elements: min / max candidates and boundary quotients
            // (y recomputed from the stage: no dynamic register indexing)
            double lmin = CUDART_INF, lmax = -CUDART_INF;
            uint32_t bnd = 0;
            bool bad = false;
            uint32_t f = fm;
            while (f) {
                const int i = __ffs(f) - 1;
                f &= f - 1;
                const bool is_sel = (selw >> i) & 1u;
                const float r32 = is_sel ? 0.0f : a32_at<GDT>(st_g, st_codes, tid * 32 + i, lo32, lv32);
                const uint32_t N = (__float_as_uint(__fmaf_rn(r32, k2, c2)) >> 15) & 31u;  // floor(y - 256)
                if (N == 1u || N == 31u) {
                    const double r = is_sel ? 0.0 : exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo, level);
                    if (N == 1u) {
                        if (r < lmin) lmin = r;  // strict: the earlier element wins ties (std::min)
                    } else if (r > lmax) {
                        lmax = r;
                    }
                } else if ((N & 1u) == 0u) {
                    bnd |= 1u << i;
                } else if (N == 0u || N > 31u) {
                    bad = true;
                }
            }
            // combine with the partner (element order: even thread first)
            const double omin = __shfl_xor_sync(pm, lmin, 1), omax = __shfl_xor_sync(pm, lmax, 1);
            const bool first = (tid & 1) == 0;
            lo_new = first ? (omin < lmin ? omin : lmin) : (lmin < omin ? lmin : omin);
            hi_new = first ? (omax > lmax ? omax : lmax) : (lmax > omax ? lmax : omax);
            bad |= !(lo_new < CUDART_INF) || !(hi_new > -CUDART_INF);
            {
                const bool pb = __shfl_xor_sync(pm, bad, 1);  // both lanes shuffle, then combine
                bad = bad || pb;
            }
            if (bad) {
                const ExactOut o = exact_bucket<GDT>(st_g, st_codes, tid, selw, lo, level, pm);
                word[0] = o.w.x; word[1] = o.w.y; word[2] = o.w.z; word[3] = o.w.w;
                lo_new = o.lo;
                hi_new = o.hi;
                if (p.dbg) atomicAdd(p.dbg + 1, 32u);
            } else if (bnd) {
                const double lvn = lo_new == hi_new ? 0.0 : div15(__dsub_rn(hi_new, lo_new));
                while (bnd) {
                    const int i = __ffs(bnd) - 1;
                    bnd &= bnd - 1;
                    const double r = ((selw >> i) & 1u) ? 0.0 : exact_a<GDT>(st_g, st_codes, tid * 32 + i, lo, level);
                    const uint32_t c = ieee_code(r, lo_new, lvn) << (4 * (i & 7));
                    const uint32_t msk = ~(15u << (4 * (i & 7)));
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        if (w == (i >> 3)) word[w] = (word[w] & msk) | c;
                }
                if (p.dbg) atomicAdd(p.dbg + 1, 1u);
            }
        } else {
            const ExactOut o = exact_bucket<GDT>(st_g, st_codes, tid, selw, lo, level, pm);
            word[0] = o.w.x; word[1] = o.w.y; word[2] = o.w.z; word[3] = o.w.w;
            lo_new = o.lo;
            hi_new = o.hi;
        }
        reinterpret_cast<uint4*>(p.codes + base / 2)[tid] = make_uint4(word[0], word[1], word[2], word[3]);
        if ((tid & 1) == 0) p.meta[base / 64 + (tid >> 1)] = make_double2(lo_new, hi_new);

        // ---- ADAM_STATS + update: coordinates held by one entry ----
        mbar_wait(&bars[2], it & 1);
        {
            const int nent = filled * kb;
            const int per = (nent + 3) / 4;  // warp w: entries [w per, (w+1) per), in order
            const int t0 = warp * per, t1 = min(nent, t0 + per);
            int nd = 0;
            int* dl = s_dupl + warp * seg;
            const int sq = div_kb(32, kb, inv_kb), sr = 32 - sq * kb;
            int r = div_kb(t0 + lane, kb, inv_kb), pos = (t0 + lane) - r * kb;
            for (int tb = t0; tb < t1; tb += 32) {
                const int t = tb + lane;
                const bool act = t < t1;
                int idx = 0;
                bool dup = false;
                if (act) {
                    idx = swi[r * kbs + pos];
                    dup = (s_dup[idx >> 5] >> (idx & 31)) & 1u;
                }
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, dup);
                if (dup) dl[nd + __popc(bal & lanemask_lt())] = (idx << 16) | (r << 8) | pos;
                nd += __popc(bal);
                if (act && !dup) {
                    const int e = r * kbs + pos;
                    if constexpr (PDT == BF16) {
                        // bf16 θ: fp32 estimate x32 = θ - lr32·c1 v / (eps32 + |v| c2),
                        // within |lr u| 2^-20.6 + |x| 2^-24 of the fp64 result: final
                        // when more than 512 ulps from the bf16 rounding midpoint.
                        const float th = ldf<PDT>(sth, idx);
                        const float v = ldf<VDT>(swv, e);
                        const float den = __fmaf_rn(fabsf(v), p.c2[r], p.eps32);
                        const float u = __fdividef(p.c1[r] * v, den);
                        if (!bf16_screen_store(p, base + idx, th, u, den))
                            exact_single<PDT>(&p, base + idx, static_cast<double>(th), static_cast<double>(v), r);
                    } else {
                        exact_single<PDT>(&p, base + idx, ldd<PDT>(sth, idx), ldd<VDT>(swv, e), r);
                    }
                }
                r += sq;
                pos += sr;
                if (pos >= kb) {
                    pos -= kb;
                    ++r;
                }
            }
            if (lane == 0) misc[kDupN + warp] = nd;
        }
        __syncthreads();  // B3
        // No end-of-block barrier: warp 0 applies the duplicated coordinates
        // while warps 1-3 go on to the next block's pass 1. Everything warp 0
        // still reads here (dup lists, θ buffer, this stage) is rewritten only
        // after it reaches the next block's B1 (thread 0 issues the next TMA
        // fills itself), and every scratch word reused before B1 is reset on
        // the side that finishes with it.
        if (warp == 0) {
            dup_updates<K>(&p, smem, st, base);
            __syncwarp();
            s_seen[lane * 4 + 0] = 0;
            s_seen[lane * 4 + 1] = 0;
            s_seen[lane * 4 + 2] = 0;
            s_seen[lane * 4 + 3] = 0;
            s_dup[lane * 4 + 0] = 0;
            s_dup[lane * 4 + 1] = 0;
            s_dup[lane * 4 + 2] = 0;
            s_dup[lane * 4 + 3] = 0;
            fence_proxy_async_smem();  // generic writes to this stage before its next TMA fill
            __syncwarp();
        } else {
            for (int i = tid - 32; i < 128; i += kT - 32) {
                s_sel[i] = 0;
                s_hist[i] = 0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

template <class K>
cudaError_t launch_kt(const StepArgs& a, const CUtensorMap& map, cudaStream_t s) {
    const TLay L(K::gsz, K::psz, K::vsz, a.m, a.kb_stride, K::CAP, a.m * a.per_block_k);
    auto k = microadam_step_tile<K>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
    if (err != cudaSuccess) return err;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kT, L.total);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t grid = std::min<int64_t>(a.block_count, int64_t(per_sm) * nsm);
    k<<<static_cast<unsigned>(grid), kT, L.total, s>>>(a, map);
    return cudaGetLastError();
}

constexpr int dtype_key_t(int g, int p, int v) { return g * 9 + p * 3 + v; }

#define MA_TILE_DTYPES(X) \
    X(BF16, BF16, BF16)   \
    X(F32, F32, BF16)     \
    X(F32, F32, F32)      \
    X(BF16, F32, BF16)    \
    X(BF16, BF16, F32)

}  // namespace

bool tile_ok(const StepArgs& a) {
    if (a.partials || a.force_exact || a.block != kBlk || a.bucket != 64 || a.bits != 4 || a.dense) return false;
    if (a.per_block_k < 1 || a.per_block_k > 256 || a.m < 1 || a.m > 255) return false;
    if (a.rs_n > 0 || a.stage_idx) return false;
    switch (dtype_key_t(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_) case dtype_key_t(G_, P_, V_):
        MA_TILE_DTYPES(MA_CASE)
#undef MA_CASE
        break;
        default: return false;
    }
    const int cap = a.per_block_k > 64 ? 512 : 128;
    const int gsz = a.g_dtype == F32 ? 4 : 2, psz = a.p_dtype == F32 ? 4 : 2, vsz = a.v_dtype == F32 ? 4 : 2;
    const TLay L(gsz, psz, vsz, a.m, a.kb_stride, cap, a.m * a.per_block_k);
    return L.total <= 227u * 1024u;
}

cudaError_t launch_step_tile(const StepArgs& a, cudaStream_t s) {
    if (a.block_count <= 0) return cudaSuccess;
    if (!tile_ok(a)) return cudaErrorInvalidConfiguration;
    auto enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    // g tensor: the full blocks [block_offset, block_offset + block_count) as
    // 128-byte rows; one box = one 4096-element block, 128-byte swizzle
    const int esz = a.g_dtype == F32 ? 4 : 2;
    const cuuint64_t per_row = 128 / esz;
    const cuuint64_t rows = static_cast<cuuint64_t>(a.block_offset + a.block_count) * (kBlk / per_row);
    CUtensorMap map;
    const cuuint64_t gdim[2] = {per_row, rows};
    const cuuint64_t gstride[1] = {128};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(per_row), static_cast<cuuint32_t>(kBlk / per_row)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     const_cast<void*>(a.grads), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    switch (dtype_key_t(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_)                                                                       \
    case dtype_key_t(G_, P_, V_):                                                                 \
        return a.per_block_k > 64 ? launch_kt<TK<G_, P_, V_, 16>>(a, map, s)                      \
                                  : launch_kt<TK<G_, P_, V_, 4>>(a, map, s);
        MA_TILE_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace ma
