// ma_warp.cu — the warp-per-block sm_100a MicroAdam step kernel (default path).
//
// Same contract and bit-exact results as ma_kernels.cu / ma_fast.cu, shaped so
// that no Top-K block ever waits on a CTA barrier: ONE WARP owns one
// B_d = 4096 block end to end (optim.cpp:164-190), four independent warps per
// 128-thread CTA, eight CTAs per SM (≤ 64 registers, ~4.5 KB smem per warp).
// The serial parts of a block (exact select, window bookkeeping) overlap with
// the streaming passes of the 31 other warps on the SM.
//
//  * Lane 0 starts the block's HBM traffic at once: 1-D bulk L2 prefetches
//    (cp.async.bulk.prefetch.L2) of g, the EF codes, the bucket (lo, hi), the
//    window rows and θ. The passes then read L2-hot lines.
//  * Pass 1 (optim.cpp:166-168, quantize.cpp:164-178): a = g + decode(EF) in
//    fp64 for 8 consecutive elements per lane per iteration; the 16-bit Top-K
//    key (bits 62..48 of |a|) is compared with the threshold carried from the
//    previous step (SIMD __vcmpgeu2); the hits stay as a 128-bit candidate
//    mask in registers.
//  * Exact block Top-K (compress.cpp:39-53): if k_b <= #hits <= 128 the hits'
//    a values are gathered and the k_b-th largest high word is bisected with
//    warp-wide counts over register-held keys; ties on the high word resolve on
//    the full |a| key, then the lower index. Otherwise (first step, drift, or
//    heavy ties) an out-of-line radix descent over 7-bit digits of the full
//    63-bit key finds either a candidate set of <= 128 or the exact k_b-th key.
//    The selection is always exact; the carried threshold only decides work.
//  * Window row (window.cpp:14-26) at ascending positions from a word prefix of
//    the selection bitmap.
//  * ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187): per-block
//    seen/dup bitmaps; coordinates in one row take z = 0 + w·v, duplicated
//    ones are claimed once and re-summed in physical slot order. θ is updated
//    in place (L2-hot) — only window coordinates change.
//  * Pass 2 (compress.cpp:95-102, quantize.cpp:15-24, 42-55, 102-114): the
//    residual is re-decoded from L2, bucket min/max in registers + shuffles,
//    the 4-bit codes by the fixed-point fast path with an exact IEEE fallback
//    inside the guard band (same rule as ma_fast.cu).
#include "../../include/ma_synth.h"
#include "ma_async.cuh"
#include "ma_device.cuh"
#include "ma_internal.h"

#include <math_constants.h>

namespace ma {
namespace {

using namespace dev;

constexpr int kWarps = 4;                 // Top-K blocks (warps) per CTA
constexpr int kBlk = 4096;                // B_d of this kernel
constexpr int kIter = kBlk / 256;         // iterations of 8 elements per lane
constexpr int kCapL = 4;                  // candidate slots per lane
constexpr int kCap = 32 * kCapL;          // candidate capacity of the exact stage
constexpr uint32_t kGuard = 64;           // fixed-point guard band (units of 2^-20)
constexpr int kTargetHits = 64;           // carried-threshold target count (k_b <= hits <= kCap)
constexpr int kDupCap = kCap * 2;         // ordered duplicate-entry list (ints in the candidate area)
constexpr int kRefineMax = 1024;          // hits at T refined from the hit mask (else radix path)

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l2_keep(const void* p, uint32_t bytes) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
                 : "memory");
}

// Per-warp shared-memory carve-up (bytes; host and device agree).
struct WLayout {
    uint32_t ll, sel, wpref, dup, cval, cidx, misc, total;
    __host__ __device__ WLayout() {}
    __host__ __device__ WLayout(int bucket, int /*capl*/) : WLayout(bucket) {}
    __host__ __device__ explicit WLayout(int bucket) {
        size_t o = 0;
        ll = uint32_t(o);    o = align_up(o + size_t(kBlk / bucket) * 16, 16);  // (lo, level)
        sel = uint32_t(o);   o = align_up(o + kBlk / 8, 16);                     // selection bits
        wpref = uint32_t(o); o = align_up(o + kBlk / 8, 16);  // word prefix; then "seen" bits
        dup = uint32_t(o);   o = align_up(o + kBlk / 8, 16);                     // duplicate bits
        cval = uint32_t(o);  o = align_up(o + kCap * 8, 16);  // candidates; radix hist; dup queue
        cidx = uint32_t(o);  o = align_up(o + kCap * 2, 16);
        misc = uint32_t(o);  o = align_up(o + 16 * 4, 16);
        total = uint32_t(align_up(o, 128));
    }
};

template <int LPB_, int GDT_, int PDT_, int VDT_, bool REP_, int CAPL_ = 4, bool RS_ = false>
struct KW {
    static constexpr int LPB = LPB_, GDT = GDT_, PDT = PDT_, VDT = VDT_;
    static constexpr int CAPL = CAPL_;  // lean kernel: exact-stage candidate slots per lane
    // lean kernel: the gradient is reduced from p.rs_src[] into p.grads by the
    // kernel itself (fused reduce-scatter), so p.grads is read with coherent loads
    static constexpr bool RS = RS_;
    static constexpr int BUCKET = 8 * LPB_;
    static constexpr bool REPORT = REP_;
};

// ---- 8 consecutive gradient values: raw vector load, then widen to fp64 ----
template <int DT>
struct Raw8 {
    static constexpr int N = DT == BF16 ? 1 : (DT == F32 ? 2 : 4);
    uint4 v[N];
};
template <int DT, bool NC = true>
__device__ __forceinline__ Raw8<DT> load_raw8(const void* g, int64_t e0) {
    Raw8<DT> r;
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(g) +
                                                    e0 * (DT == BF16 ? 2 : (DT == F32 ? 4 : 8)));
#pragma unroll
    for (int k = 0; k < Raw8<DT>::N; ++k) {
        if constexpr (NC) r.v[k] = __ldg(q + k);
        else r.v[k] = q[k];
    }
    return r;
}
template <int DT>
__device__ __forceinline__ void widen8(const Raw8<DT>& r, double (&x)[8]) {
    if constexpr (DT == BF16) {
        const uint32_t w[4] = {r.v[0].x, r.v[0].y, r.v[0].z, r.v[0].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
            x[2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
        }
    } else if constexpr (DT == F32) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            x[4 * k + 0] = __uint_as_float(r.v[k].x);
            x[4 * k + 1] = __uint_as_float(r.v[k].y);
            x[4 * k + 2] = __uint_as_float(r.v[k].z);
            x[4 * k + 3] = __uint_as_float(r.v[k].w);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[2 * k] = __hiloint2double(int(r.v[k].y), int(r.v[k].x));
            x[2 * k + 1] = __hiloint2double(int(r.v[k].w), int(r.v[k].z));
        }
    }
}

// a += code·level + lo (quantize.cpp:164-178, optim.cpp:166-168): separate
// multiply and add in fp64, no FMA.
__device__ __forceinline__ void add_decoded8(double (&a)[8], uint32_t cw, double2 ll) {
    const uint32_t ce = cw & 0x0F0F0F0Fu, co = (cw >> 4) & 0x0F0F0F0Fu;  // even / odd nibbles
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double c0 = static_cast<double>(__byte_perm(ce, 0u, 0x4440u | k));
        const double c1 = static_cast<double>(__byte_perm(co, 0u, 0x4440u | k));
        a[2 * k] = __dadd_rn(a[2 * k], __dadd_rn(__dmul_rn(c0, ll.y), ll.x));
        a[2 * k + 1] = __dadd_rn(a[2 * k + 1], __dadd_rn(__dmul_rn(c1, ll.y), ll.x));
    }
}

// a at one block-relative element (same arithmetic as pass 1).
template <class KT>
__device__ __forceinline__ double recompute_a(const StepArgs& p, int64_t base, const double2* ll, int e) {
    const uint32_t byte = p.codes[(base + e) >> 1];
    const double2 q = ll[e / KT::BUCKET];
    const double ev = __dadd_rn(__dmul_rn(static_cast<double>((byte >> ((e & 1) * 4)) & 15u), q.y), q.x);
    return __dadd_rn(ld_t<KT::GDT>(p.grads, base + e), ev);
}

// t / kb for t < 2^16 without an integer division (float reciprocal + fix-up).
__device__ __forceinline__ int row_of(int t, int kb, float inv_kb) {
    int r = __float2int_rz(static_cast<float>(t) * inv_kb);
    r -= (r * kb > t);
    r += ((r + 1) * kb <= t);
    return r;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total) {
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    return incl - v;
}

// Ordered duplicate-list entry: block-relative index (12 bits) | physical
// window row (10 bits) | position in the row (10 bits): m <= 1023, k_b <= 1023.
__device__ __forceinline__ int dup_pack(int idx, int r, int pos) {
    return static_cast<int>((static_cast<uint32_t>(idx) << 20) | (static_cast<uint32_t>(r) << 10) |
                            static_cast<uint32_t>(pos));
}
__device__ __forceinline__ int dup_idx(int x) { return static_cast<int>(static_cast<uint32_t>(x) >> 20); }
__device__ __forceinline__ int dup_row(int x) { return (x >> 10) & 0x3FF; }
__device__ __forceinline__ int dup_pos(int x) { return x & 0x3FF; }

// Rank correction among candidates whose high words tie (compress.cpp:43-48:
// full |a| key first, then the lower index). Out of line: rare.
__device__ __noinline__ int tie_rank_w(const double* cval, const int16_t* cidx, int ncand, int t) {
    const uint64_t kt = key_of(cval[t]);
    const uint32_t kh = static_cast<uint32_t>(kt >> 32);
    const int it = cidx[t];
    int extra = 0;
    for (int q = 0; q < ncand; ++q) {
        const uint64_t kq = key_of(cval[q]);
        if (q == t || static_cast<uint32_t>(kq >> 32) != kh) continue;
        extra += (kq > kt) || (kq == kt && cidx[q] < it);
    }
    return extra;
}

// rn(x / 15) (QuantParams level, quantize.cpp:12) without the fp64 division
// sequence: q0 = rn(x c), c = rn(1/15); the remainder x - 15 q0 is exact by
// FMA and rn(q0 + r c) is the correctly rounded quotient (Markstein; checked
// against x / 15 on 4e8 random normal x). Outside [2^-960, 2^1000] (and for
// non-finite x) the IEEE division.
__device__ __forceinline__ double div15_w(double x) {
    if (!(x >= 0x1p-960 && x <= 0x1p1000)) return __ddiv_rn(x, 15.0);
    const double c = 0x1.1111111111111p-4;
    const double q0 = __dmul_rn(x, c);
    return __fma_rn(__fma_rn(-q0, 15.0, x), c, q0);
}

// The IEEE path of quantize_nearest (quantize.cpp:51-53) for an element whose
// fixed-point estimate fell in the guard band. Out of line: rare.
__device__ __noinline__ uint32_t exact_code_w(double x, double lo, double level) {
    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(x, lo), level), 0.5));
    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
    return static_cast<uint32_t>(f);
}

// Slow selection (out of line): the carried threshold missed (first step,
// drift) or keys tie heavily. A radix descent over 7-bit digits of the 63-bit
// key |a| (9 digits) re-decoding the L2-hot block each pass, until the keys at
// or above the current prefix number <= kCap; those are gathered as candidates
// (returns their count; misc[0] = high word of the prefix, a lower bound of
// the k_b-th high word). If all 63 bits are fixed with more than kCap keys
// tied at the k_b-th key, the exact selection — every key above it plus the
// lowest-index ties (compress.cpp:43-48) — is written to the selection bitmap
// directly and -1 is returned (misc[1] = the k_b-th key's high word).
template <class KT, class LAY>
__device__ __noinline__ int slow_select(const StepArgs* pp, unsigned char* ws, int64_t b) {
    const StepArgs& p = *pp;
    constexpr int kCapS = 32 * KT::CAPL;
    const LAY L(KT::BUCKET, KT::CAPL);
    const int lane = threadIdx.x & 31;
    const int64_t base = b * kBlk;
    const double2* s_ll = reinterpret_cast<const double2*>(ws + L.ll);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.cval);  // 128 bins
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(ws + L.sel);
    int* s_misc = reinterpret_cast<int*>(ws + L.misc);
    const int kb = p.per_block_k;
    auto block_a = [&](int j, double (&a)[8]) {
        const int e0 = j * 256 + lane * 8;
        widen8<KT::GDT>(load_raw8<KT::GDT, !KT::RS>(p.grads, base + e0), a);
        add_decoded8(a, *reinterpret_cast<const uint32_t*>(p.codes + ((base + e0) >> 1)),
                     s_ll[e0 / KT::BUCKET]);
    };
    uint64_t prefix = 0, pmask = 0;
    int need = kb, above_total = 0, binc = 0;
    for (int sh = 56;; sh -= 7) {
#pragma unroll
        for (int k = 0; k < 4; ++k) hist[lane * 4 + k] = 0;
        __syncwarp();
        uint64_t kmx = 0;
        for (int j = 0; j < kIter; ++j) {
            double a[8];
            block_a(j, a);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint64_t k = key_of(a[i]);
                kmx = k > kmx ? k : kmx;
                if ((k & pmask) == prefix) atomicAdd(&hist[(k >> sh) & 127u], 1u);
            }
        }
        // inf/NaN in g or a (the fast path checks its candidates instead)
        if (sh == 56 && p.check_finite && __any_sync(0xFFFFFFFFu, (kmx >> 48) >= 0x7FF0u) && lane == 0)
            atomicOr(p.flag, 1u);
        __syncwarp();
        // digit d: the largest with #{digit >= d} >= need (suffix sums from the top)
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
        const int owner = d >> 2;
        const int sd = d & 3;
        const int sfx = sd == 0 ? s0 : (sd == 1 ? s1 : (sd == 2 ? s2 : s3));
        const int hd = int(sd == 0 ? h0 : (sd == 1 ? h1 : (sd == 2 ? h2 : h3)));
        const int above = __shfl_sync(0xFFFFFFFFu, sfx - hd, owner);
        binc = __shfl_sync(0xFFFFFFFFu, hd, owner);
        above_total += above;
        need -= above;
        prefix |= static_cast<uint64_t>(d) << sh;
        pmask |= uint64_t(127) << sh;
        __syncwarp();
        if (above_total + binc <= kCapS || sh == 0) break;
    }
    double* s_cval = reinterpret_cast<double*>(ws + L.cval);
    int16_t* s_cidx = reinterpret_cast<int16_t*>(ws + L.cidx);
    if (above_total + binc <= kCapS) {
        // gather every key >= prefix (numeric) — exactly above_total + binc keys
        if (lane == 0) s_misc[2] = 0;
        __syncwarp();
        for (int j = 0; j < kIter; ++j) {
            double a[8];
            block_a(j, a);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (key_of(a[i]) >= prefix) {
                    const int q = atomicAdd(&s_misc[2], 1);
                    s_cval[q] = a[i];
                    s_cidx[q] = static_cast<int16_t>(j * 256 + lane * 8 + i);
                }
        }
        __syncwarp();
        if (lane == 0) s_misc[0] = static_cast<int>(prefix >> 32);
        __syncwarp();
        return above_total + binc;
    }
    // All 63 bits fixed: K* = prefix; `need` of the keys equal to K* in index order.
    int eq_before = 0;
    for (int j = 0; j < kIter; ++j) {
        double a[8];
        block_a(j, a);
        uint32_t gt = 0, eq = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t k = key_of(a[i]);
            gt |= static_cast<uint32_t>(k > prefix) << i;
            eq |= static_cast<uint32_t>(k == prefix) << i;
        }
        int tot;
        const int ex = warp_excl_scan(__popc(eq), lane, tot);
        uint32_t selm = gt;
        int r = eq_before + ex;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if ((eq >> i) & 1u) {
                if (r < need) selm |= 1u << i;
                ++r;
            }
        eq_before += tot;
        const int e0 = j * 256 + lane * 8;
        if (selm) atomicOr(&s_sel[e0 >> 5], selm << (e0 & 31));
    }
    __syncwarp();
    if (lane == 0) s_misc[1] = static_cast<int>(prefix >> 32);
    if (p.dbg && lane == 0) atomicAdd(p.dbg + 0, 1u);
    __syncwarp();
    return -1;
}

// ADAM_STATS + update of the duplicated window coordinates (window.cpp:28-46,
// optim.cpp:183-187), out of line: one claimant per coordinate sums its
// entries in physical slot order — from the ordered duplicate list when it
// fit (ndup <= capacity), else by binary search in the ascending rows.
// Returns the number of nonzero updates (report field 4).
template <class KT, class LAY>
__device__ __noinline__ double dup_stats(const StepArgs* pp, unsigned char* ws, int64_t b, int ndup,
                                         int nent) {
    const StepArgs& p = *pp;
    const LAY L(KT::BUCKET, KT::CAPL);
    const int lane = threadIdx.x & 31;
    const int kb = p.per_block_k, kbs = p.kb_stride, filled = p.filled;
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    const int64_t went = b * p.m * static_cast<int64_t>(kbs);
    const int16_t* gwi = p.win_idx + went;
    const unsigned char* gwv = static_cast<const unsigned char*>(p.win_val) + went * vsz;
    const int64_t base = b * kBlk;
    const int* dupl = reinterpret_cast<const int*>(ws + L.cval);
    uint32_t* s_seen = reinterpret_cast<uint32_t*>(ws + L.wpref);
    const uint32_t* s_dup = reinterpret_cast<const uint32_t*>(ws + L.dup);
    const float inv_kb = 1.0f / static_cast<float>(kb);
    const bool listed = ndup <= kDupCap;
    const int n = listed ? ndup : nent;
    double nnz = 0.0;
    for (int q = lane; q < n; q += 32) {
        int idx;
        if (listed) {
            idx = dup_idx(dupl[q]);
        } else {
            const int r = row_of(q, kb, inv_kb);
            idx = gwi[r * kbs + (q - r * kb)];
            if (!((s_dup[idx >> 5] >> (idx & 31)) & 1u)) continue;
        }
        const uint32_t bit = 1u << (idx & 31);
        if (!(atomicAnd(&s_seen[idx >> 5], ~bit) & bit)) continue;  // another entry claimed it
        double z1 = 0.0, z2 = 0.0;
        if (listed) {
            for (int q2 = 0; q2 < ndup; ++q2) {  // list order = physical slot order (window.cpp:32-39)
                const int x = dupl[q2];
                if (dup_idx(x) != idx) continue;
                const int rr = dup_row(x);
                const double v = ld_t<KT::VDT>(gwv, rr * kbs + dup_pos(x));
                z1 = __dadd_rn(z1, __dmul_rn(p.w1[rr], v));
                z2 = __dadd_rn(z2, __dmul_rn(p.w2[rr], __dmul_rn(v, v)));
            }
        } else {
            for (int rr = 0; rr < filled; ++rr) {  // physical slot order (window.cpp:32-39)
                const int16_t* row = gwi + rr * kbs;
                int lo_i = 0, hi_i = kb;
                while (lo_i < hi_i) {
                    const int mid = (lo_i + hi_i) >> 1;
                    if (row[mid] < idx) lo_i = mid + 1; else hi_i = mid;
                }
                if (lo_i < kb && row[lo_i] == idx) {
                    const double v = ld_t<KT::VDT>(gwv, rr * kbs + lo_i);
                    z1 = __dadd_rn(z1, __dmul_rn(p.w1[rr], v));
                    z2 = __dadd_rn(z2, __dmul_rn(p.w2[rr], __dmul_rn(v, v)));
                }
            }
        }
        const double mhat = __dmul_rn(z1, p.scale1);
        const double vhat = __dmul_rn(z2, p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        const double th = ld_t<KT::PDT>(p.params, base + idx);
        st_t<KT::PDT>(p.params, base + idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        nnz += u != 0.0 ? 1.0 : 0.0;
    }
    return nnz;
}

template <class KT>
__global__ void __launch_bounds__(32 * kWarps, 8) microadam_step_warp(const __grid_constant__ StepArgs p) {
    constexpr int BUCKET = KT::BUCKET, LPB = KT::LPB;
    constexpr int gsz = KT::GDT == F64 ? 8 : (KT::GDT == F32 ? 4 : 2);
    constexpr int psz = KT::PDT == F64 ? 8 : (KT::PDT == F32 ? 4 : 2);
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    constexpr bool want_report = KT::REPORT;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bl = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (bl >= p.block_count) return;
    const int64_t b = p.block_offset + bl;
    const int64_t base = b * kBlk;
    const WLayout L(BUCKET);
    unsigned char* ws = smem + warp * L.total;
    double2* s_ll = reinterpret_cast<double2*>(ws + L.ll);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(ws + L.sel);
    int* s_wpref = reinterpret_cast<int*>(ws + L.wpref);
    uint32_t* s_seen = reinterpret_cast<uint32_t*>(ws + L.wpref);
    uint32_t* s_dup = reinterpret_cast<uint32_t*>(ws + L.dup);
    double* s_cval = reinterpret_cast<double*>(ws + L.cval);
    int16_t* s_cidx = reinterpret_cast<int16_t*>(ws + L.cidx);
    int* s_misc = reinterpret_cast<int*>(ws + L.misc);
    const int kb = p.per_block_k, kbs = p.kb_stride, m = p.m, slot = p.slot, filled = p.filled;
    const int64_t went = b * m * static_cast<int64_t>(kbs);
    int16_t* gwi = p.win_idx + went;
    unsigned char* gwv = static_cast<unsigned char*>(p.win_val) + went * vsz;

    // ---- prologue: start the block's HBM reads; bucket grids (quantize.cpp:7-13) ----
    if (lane == 0) {
        prefetch_l2_keep(static_cast<const unsigned char*>(p.grads) + base * gsz, kBlk * gsz);
        prefetch_l2_keep(p.codes + base / 2, kBlk / 2);
        prefetch_l2(p.meta + base / BUCKET, (kBlk / BUCKET) * 16);
    }
    for (int i = lane; i < kBlk / BUCKET; i += 32) {
        const double2 mt = p.meta[base / BUCKET + i];
        s_ll[i] = make_double2(mt.x, (mt.x == mt.y) ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), 15.0));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_sel[lane * 4 + k] = 0;
        s_dup[lane * 4 + k] = 0;
    }
    __syncwarp();

    // ---- pass 1: a = g + decode(EF), 16-bit keys vs the carried threshold ----
    // carried state: low 16 bits = key16 threshold, high 16 = hits it was chosen for
    const uint32_t tstate = __ldg(p.thresh + b);
    const uint32_t T = tstate & 0xFFFFu;
    const uint32_t T2 = T << 17;
    uint32_t cm0 = 0, cm1 = 0, cm2 = 0, cm3 = 0;  // candidate bits: byte j = iteration j
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    {
        Raw8<KT::GDT> nr = load_raw8<KT::GDT, !KT::RS>(p.grads, base + lane * 8);
        uint32_t ncw = *reinterpret_cast<const uint32_t*>(p.codes + ((base + lane * 8) >> 1));
#pragma unroll 1
        for (int j = 0; j < kIter; ++j) {
            const int e0 = j * 256 + lane * 8;
            const Raw8<KT::GDT> r = nr;
            const uint32_t cw = ncw;
            if (j + 1 < kIter) {
                nr = load_raw8<KT::GDT, !KT::RS>(p.grads, base + e0 + 256);
                ncw = *reinterpret_cast<const uint32_t*>(p.codes + ((base + e0 + 256) >> 1));
            }
            double a[8];
            widen8<KT::GDT>(r, a);
            add_decoded8(a, cw, s_ll[e0 / BUCKET]);
            uint32_t m8 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                // bits 62..31 of a: key16 >= T  <=>  (|a| bits >> 31) >= T << 17
                const uint32_t h2 = static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(a[i])) >> 31);
                m8 |= static_cast<uint32_t>(h2 >= T2) << i;
                if (want_report) rep[1] += a[i] * a[i];
            }
            cm0 = __funnelshift_r(cm0, cm1, 8);
            cm1 = __funnelshift_r(cm1, cm2, 8);
            cm2 = __funnelshift_r(cm2, cm3, 8);
            cm3 = (cm3 >> 8) | (m8 << 24);
        }
    }
    if (lane == 0) {
        prefetch_l2(gwi, uint32_t(m * kbs * 2));
        prefetch_l2(gwv, uint32_t(m * kbs * vsz));
        prefetch_l2(static_cast<const unsigned char*>(p.params) + base * psz, kBlk * psz);
    }
    const int nmine = __popc(cm0) + __popc(cm1) + __popc(cm2) + __popc(cm3);
    const int cnt = __reduce_add_sync(0xFFFFFFFFu, nmine);

    // ---- block Top-K (compress.cpp:39-53, 73-85) ----
    int ncand = -1;
    uint32_t lo32 = T << 16;
    bool refined = false;
    if (T != 0 && cnt > kCap && cnt <= kRefineMax) {
        // Too many hits at T (the |a| distribution moved up): refine from the hit
        // mask instead of re-reading the block. A histogram of key16 - T over the
        // hits gives the largest T' = T + d with >= k_b hits; the hits at or
        // above T' become the candidates (still a superset of the top k_b).
        uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.cval);  // dead until the gather
        hist[lane] = 0;
        __syncwarp();
        auto for_hits = [&](auto&& f) {
#pragma unroll 1
            for (int w = 0; w < 4; ++w) {
                uint32_t bits = w == 0 ? cm0 : (w == 1 ? cm1 : (w == 2 ? cm2 : cm3));
                while (bits) {
                    const int sb = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int e = (w * 4 + (sb >> 3)) * 256 + lane * 8 + (sb & 7);
                    f(e, recompute_a<KT>(p, base, s_ll, e));
                }
            }
        };
        for_hits([&](int, double a) { atomicAdd(&hist[min((hi_key(a) >> 16) - T, 31u)], 1u); });
        __syncwarp();
        int sfx = static_cast<int>(hist[lane]);  // #hits with key16 - T >= lane
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_down_sync(0xFFFFFFFFu, sfx, off);
            if (lane + off < 32) sfx += t;
        }
        const uint32_t ok = __ballot_sync(0xFFFFFFFFu, sfx >= kb);  // bit 0 always set
        const int d = 31 - __clz(ok);
        const int n = __shfl_sync(0xFFFFFFFFu, sfx, d);
        __syncwarp();
        if (n <= kCap) {
            const uint32_t T1 = T + static_cast<uint32_t>(d);
            if (lane == 0) s_misc[4] = 0;
            __syncwarp();
            for_hits([&](int e, double a) {
                if ((hi_key(a) >> 16) >= T1) {
                    const int q = atomicAdd(&s_misc[4], 1);
                    s_cval[q] = a;
                    s_cidx[q] = static_cast<int16_t>(e);
                }
            });
            __syncwarp();
            ncand = n;
            lo32 = T1 << 16;
            refined = true;
        }
        if (p.dbg && lane == 0) atomicAdd(p.dbg + 6, 1u);
    }
    if (refined) {
        // candidates gathered by the refinement
    } else if (T != 0 && cnt >= kb && cnt <= kCap) {
        int total;
        int pos = warp_excl_scan(nmine, lane, total);
#pragma unroll 1
        for (int w = 0; w < 4; ++w) {
            uint32_t bits = w == 0 ? cm0 : (w == 1 ? cm1 : (w == 2 ? cm2 : cm3));
            while (bits) {
                const int s = __ffs(bits) - 1;
                bits &= bits - 1;
                const int e = (w * 4 + (s >> 3)) * 256 + lane * 8 + (s & 7);
                s_cval[pos] = recompute_a<KT>(p, base, s_ll, e);
                s_cidx[pos] = static_cast<int16_t>(e);
                ++pos;
            }
        }
        ncand = cnt;
        __syncwarp();
    } else {
        ncand = slow_select<KT, WLayout>(&p, ws, b);
        if (p.dbg && lane == 0) {
            atomicAdd(p.dbg + 2, 1u);
            if (cnt > kCap) atomicAdd(p.dbg + 3, 1u);
        }
        if (ncand >= 0) lo32 = static_cast<uint32_t>(s_misc[0]);
    }
    uint32_t next_t;
    uint32_t selc = 0;  // which of my candidate slots are selected
    if (ncand >= 0) {
        uint32_t kh[kCapL];
#pragma unroll
        for (int s = 0; s < kCapL; ++s) {
            const int q = lane + 32 * s;
            kh[s] = q < ncand ? hi_key(s_cval[q]) : 0u;
        }
        auto count_ge = [&](uint32_t v) {
            int c = 0;
#pragma unroll
            for (int s = 0; s < kCapL; ++s) c += kh[s] >= v;
            return __reduce_add_sync(0xFFFFFFFFu, c);
        };
        // the candidates hold every key >= T, so also the block's largest
        const uint32_t kmaxc = __reduce_max_sync(0xFFFFFFFFu, max(max(kh[0], kh[1]), max(kh[2], kh[3])));
        if (p.check_finite && kmaxc >= 0x7FF00000u && lane == 0) atomicOr(p.flag, 1u);  // inf/NaN in g or a
        // bisect the k_b-th largest high word: count(lo) >= kb > count(hi)
        uint32_t lo = lo32, hi = kmaxc + 1;
        while (hi - lo > 1) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (count_ge(mid) >= kb) lo = mid; else hi = mid;
        }
        const int above = count_ge(lo + 1);
        const int need = kb - above, eqc = count_ge(lo) - above;
#pragma unroll
        for (int s = 0; s < kCapL; ++s) {
            const int q = lane + 32 * s;
            bool sel = q < ncand && kh[s] > lo;
            if (q < ncand && kh[s] == lo) sel = eqc == need || tie_rank_w(s_cval, s_cidx, ncand, q) < need;
            if (sel) {
                const int e = s_cidx[q];
                atomicOr(&s_sel[e >> 5], 1u << (e & 31));
                selc |= 1u << s;
            }
        }
        // Next step's threshold. The hits seen at T against the hits T was
        // chosen for estimate the step-to-step drift of |a| (the EF grows
        // until it saturates); aim the new threshold at kTargetHits after the
        // same drift: the largest 16-bit key t whose candidate count reaches
        // want = kTargetHits * planned / seen. Counts below the candidate floor
        // are unknown; there one key below the floor is taken (~1.3x hits).
        const int planned = T ? static_cast<int>(tstate >> 16) : 0;
        int want = planned ? (kTargetHits * planned) / max(cnt, 1) : kTargetHits;
        want = min(max(want, kb + (kb >> 2)), kCap - (kCap >> 2));
        const uint32_t floor16 = (lo32 + 0xFFFFu) >> 16;  // every key16 >= floor16 is a candidate
        uint32_t t = lo >> 16;
        int c = count_ge(t << 16);
        while (t > floor16 && c < want) c = count_ge(--t << 16);
        if (c < want && t > 1) {
            --t;
            c += c >> 2;
        }
        next_t = t | (static_cast<uint32_t>(min(c, 0xFFFF)) << 16);
    } else {
        const uint32_t h = static_cast<uint32_t>(s_misc[1]) >> 16;
        next_t = h > 2 ? h - 2 : 1u;
    }
    if (lane == 0) p.thresh[b] = (next_t & 0xFFFFu) ? next_t : (next_t | 1u);
    __syncwarp();

    // ---- window row `slot` (window.cpp:14-26): ascending positions ----
    {
        uint32_t wv[4];
        int loc = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            wv[k] = s_sel[lane * 4 + k];
            loc += __popc(wv[k]);
        }
        int tot;
        int run = warp_excl_scan(loc, lane, tot);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            s_wpref[lane * 4 + k] = run;
            run += __popc(wv[k]);
        }
    }
    __syncwarp();
    const int64_t row0 = static_cast<int64_t>(slot) * kbs;
    if (ncand >= 0) {
#pragma unroll
        for (int s = 0; s < kCapL; ++s)
            if ((selc >> s) & 1u) {
                const int q = lane + 32 * s;
                const int e = s_cidx[q];
                const int pos = s_wpref[e >> 5] + __popc(s_sel[e >> 5] & ((1u << (e & 31)) - 1u));
                gwi[row0 + pos] = static_cast<int16_t>(e);
                st_t<KT::VDT>(gwv, row0 + pos, s_cval[q]);
            }
    } else {
        // heavy-tie path: the selected elements straight from the bitmap
        for (int w = lane; w < kBlk / 32; w += 32) {
            uint32_t bits = s_sel[w];
            int pos = s_wpref[w];
            while (bits) {
                const int e = w * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                gwi[row0 + pos] = static_cast<int16_t>(e);
                st_t<KT::VDT>(gwv, row0 + pos, recompute_a<KT>(p, base, s_ll, e));
                ++pos;
            }
        }
    }
    __threadfence_block();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) s_seen[lane * 4 + k] = 0;  // word prefix is dead
    __syncwarp();

    // ---- ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    const int nent = filled * kb;
    const float inv_kb = 1.0f / static_cast<float>(kb);
    for (int t = lane; t < nent; t += 32) {
        const int r = row_of(t, kb, inv_kb);
        const int idx = gwi[r * kbs + (t - r * kb)];
        const uint32_t bit = 1u << (idx & 31);
        if (atomicOr(&s_seen[idx >> 5], bit) & bit) atomicOr(&s_dup[idx >> 5], bit);
    }
    __syncwarp();
    // Entries of duplicated coordinates go to an ordered list (warp ballots in
    // entry order = (slot, position) order); one claimant per coordinate then
    // sums its entries in list order, i.e. physical slot order.
    int* dupl = reinterpret_cast<int*>(s_cval);  // candidates are dead
    constexpr int qcap = kDupCap;
    int ndup = 0;
    // unique coordinates, two entries per lane in flight (θ loads overlap)
    for (int t0 = 0; t0 < nent; t0 += 2 * 32) {
        int idx[2], e[2], r[2];
        bool mine[2];
        double th[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int t = t0 + k * 32 + lane;
            mine[k] = false;
            r[k] = 0;
            e[k] = 0;
            idx[k] = 0;
            bool dup = false;
            if (t < nent) {
                r[k] = row_of(t, kb, inv_kb);
                e[k] = r[k] * kbs + (t - r[k] * kb);
                idx[k] = gwi[e[k]];
                dup = (s_dup[idx[k] >> 5] >> (idx[k] & 31)) & 1u;
                mine[k] = !dup;
            }
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, dup);
            const int q = ndup + __popc(bal & lanemask_lt());
            if (dup && q < qcap) dupl[q] = dup_pack(idx[k], r[k], t - r[k] * kb);
            ndup += __popc(bal);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) th[k] = mine[k] ? ld_t<KT::PDT>(p.params, base + idx[k]) : 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (!mine[k]) continue;
            const double v = ld_t<KT::VDT>(gwv, e[k]);
            const double mhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w1[r[k]], v)), p.scale1);
            const double vhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w2[r[k]], __dmul_rn(v, v))), p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            st_t<KT::PDT>(p.params, base + idx[k], __dsub_rn(th[k], __dmul_rn(p.lr, u)));
            if (want_report && u != 0.0) rep[4] += 1.0;
        }
    }
    __syncwarp();
    if (p.dbg && lane == 0) {
        atomicAdd(p.dbg + 5, static_cast<unsigned>(ndup));
        if (ndup > kDupCap) atomicAdd(p.dbg + 4, 1u);
    }
    const double dn = dup_stats<KT, WLayout>(&p, ws, b, ndup, nent);
    if (want_report) rep[4] += dn;

    // ---- pass 2: residual (compress.cpp:95-102) + 4-bit re-quantization
    //      (quantize.cpp:15-24, 42-55, 102-114, 142-162) ----
#pragma unroll 1
    for (int j = 0; j < kIter; ++j) {
        const int e0 = j * 256 + lane * 8;
        double a[8];
        widen8<KT::GDT>(load_raw8<KT::GDT, !KT::RS>(p.grads, base + e0), a);
        add_decoded8(a, *reinterpret_cast<const uint32_t*>(p.codes + ((base + e0) >> 1)),
                     s_ll[e0 / BUCKET]);
        const uint32_t sel8 = (s_sel[e0 >> 5] >> (e0 & 31)) & 0xFFu;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((sel8 >> i) & 1u) a[i] = 0.0;
            if (want_report) rep[2] += a[i] * a[i];
        }
        double l4[4], h4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool lt = a[2 * k] < a[2 * k + 1];
            l4[k] = lt ? a[2 * k] : a[2 * k + 1];
            h4[k] = lt ? a[2 * k + 1] : a[2 * k];
        }
        double lo = l4[0] < l4[1] ? l4[0] : l4[1];
        const double lo2 = l4[2] < l4[3] ? l4[2] : l4[3];
        lo = lo < lo2 ? lo : lo2;
        double hi = h4[0] > h4[1] ? h4[0] : h4[1];
        const double hi2 = h4[2] > h4[3] ? h4[2] : h4[3];
        hi = hi > hi2 ? hi : hi2;
#pragma unroll
        for (int off = 1; off < LPB; off <<= 1) {
            const double ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
            const double oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
            lo = ol < lo ? ol : lo;
            hi = oh > hi ? oh : hi;
        }
        const double rng = __dsub_rn(hi, lo);
        uint32_t word = 0;
        if (rng != 0.0) {
            const float r32 = __double2float_rn(rng);
            const bool fastq = r32 >= 0x1p-100f && r32 <= 0x1p100f;
            const float k32 = fastq ? __fdividef(15.0f, r32) : 0.0f;  // ≤ 2 ulp
            uint32_t bad = fastq ? 0u : 0xFFu;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float d32 = __double2float_rn(__dsub_rn(a[i], lo));
                const uint32_t xq = __float2uint_rz(__fmaf_rn(__fmul_rn(d32, k32), 1048576.0f, 524288.0f));
                word |= (xq >> 20) << (4 * i);
                bad |= static_cast<uint32_t>(((xq + kGuard) & 0xFFFFFu) < 2 * kGuard) << i;
            }
            if (bad) {  // rare: guard band -> the exact quotient
                const double level = __ddiv_rn(rng, 15.0);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if ((bad >> i) & 1u)
                        word = (word & ~(15u << (4 * i))) | (exact_code_w(a[i], lo, level) << (4 * i));
                if (p.dbg) atomicAdd(p.dbg + 1, __popc(bad));
            }
        }
        if (want_report) {
            const double level = rng == 0.0 ? 0.0 : __ddiv_rn(rng, 15.0);
            double x[8];
            widen8<KT::GDT>(load_raw8<KT::GDT, !KT::RS>(p.grads, base + e0), x);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double en =
                    __dadd_rn(__dmul_rn(static_cast<double>((word >> (4 * i)) & 15u), level), lo);
                rep[3] += en * en;
                rep[0] += x[i] * x[i];
            }
        }
        __stcs(reinterpret_cast<unsigned int*>(p.codes + ((base + e0) >> 1)), word);
        if ((lane & (LPB - 1)) == 0) __stcs(p.meta + (base + e0) / BUCKET, make_double2(lo, hi));
    }
    if constexpr (want_report) {
#pragma unroll
        for (int f = 0; f < kReportFields; ++f) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) p.partials[b * kReportFields + f] = rep[f];
        }
    }
}

template <class KT>
cudaError_t launch_kw(const StepArgs& a, cudaStream_t s) {
    const size_t smem = size_t(kWarps) * WLayout(KT::BUCKET).total;
    auto k = microadam_step_warp<KT>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    const int64_t grid = (a.block_count + kWarps - 1) / kWarps;
    k<<<static_cast<unsigned>(grid), 32 * kWarps, smem, s>>>(a);
    return cudaGetLastError();
}

#ifdef MA_PROBE_HOT  // SASS-inspection builds (tools/sass_probe.sh): the bench's dtypes only
#define MA_WARP_DTYPES(X) X(BF16, BF16, BF16)
#else
#define MA_WARP_DTYPES(X)         \
    X(BF16, BF16, BF16)           \
    X(F32, F32, BF16)             \
    X(F32, F32, F32)              \
    X(BF16, F32, BF16)            \
    X(BF16, BF16, F32)            \
    X(F64, F64, F64)
#endif

constexpr int dtype_key_w(int g, int p, int v) { return g * 9 + p * 3 + v; }

// ===========================================================================
// Lean path (bf16 / f32 gradients, no StepReport): the per-element streaming
// work runs in fp32 with proven error bounds, and every decision that the
// fp32 values cannot settle is taken again in the reference's fp64
// arithmetic. Results are bit-identical to the exact kernel above.
//
// Error bound. For bucket q with previous (lo, hi) and M = max(|lo|, |hi|),
// the fp32 decode e32 = fma(c - 0, rn(level), rn(lo)) and a32 = g + e32 obey
//     |a32 - a| <= E_q + |a32| * 2^-23,   E_q = M * 2^-21 + 2^-120
// (3 roundings of at most M * 2^-24 each in e32, one of |a| * 2^-24 in a32,
// the absolute term covers fp32 subnormals). Buckets with M >= 2^100 (or
// non-finite) get E_q = inf, which sends every decision of that bucket to the
// fp64 path.
//   * Top-K screen: |a| >= V_T (key16 >= T) implies |a32| >= Tf_q with
//     Tf_q = rd((V_T - E_q) * (1 - 2^-22)); hits are a superset of the keys
//     at or above the carried threshold and are re-evaluated exactly.
//   * Bucket min / max of the residual: the exact minimum lies among the
//     elements with r32 <= m32 + 2 eps (eps = E_q + max|r32| * 2^-22), which
//     are re-evaluated in fp64 (usually one element per bucket).
//   * 4-bit code: t = (r32 - m32) * 15 / (M32 - m32) estimates
//     q = (r - lo) / level within E_t <= 120 eps / R + 2^-15 (R = M32 - m32,
//     R > 8 eps required); a 18-bit fixed-point read of t + 0.5 that lands
//     within G = E_t of an integer is recomputed with the IEEE quotient
//     (quantize.cpp:51-53).
// ===========================================================================

constexpr float kTwo23 = 8388608.0f;

// prmt with an immediate selector SEL | k (the constant operand stays in a register).
template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt_imm(uint32_t a, uint32_t b, int k) {
    uint32_t d;
    switch (k) {
        case 0: asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL | 0u)); break;
        case 1: asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL | 1u)); break;
        case 2: asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL | 2u)); break;
        default: asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL | 3u)); break;
    }
    return d;
}
#ifndef MA_LEAN_THPF_LOOP
// θ prefetch for ADAM_STATS (A/B at 7B, same box): 0 = one bulk prefetch before
// the pass-2 loop (19.03 ms), 1 = bulk prefetch at iteration 4 (18.68 ms, kept
// although its uniform-address sequence runs predicated on every iteration),
// 2 = per-lane line prefetches at iteration 4 (18.71 ms)
#define MA_LEAN_THPF_LOOP 1
#endif
#ifndef MA_LEAN_MIXADD
#define MA_LEAN_MIXADD 0  // A/B: a = g + e by mixed bf16 + fp32 adds (FHADD.BF16) in pass 1 (7B 18.64 ms) / both passes (18.47) vs 18.41: off
#endif
#ifndef MA_LEAN_MIXADD2
#define MA_LEAN_MIXADD2 MA_LEAN_MIXADD  // the same in pass 2
#endif
#ifndef MA_LEAN_BADENC
#define MA_LEAN_BADENC 0  // A/B: per-lane `bad` carried in the lmin shuffle as -inf (18.73 vs 18.42 ms at 7B: rejected)
#endif
#ifndef MA_LEAN_SIGNREP
#define MA_LEAN_SIGNREP 1  // lean pass 1: hit-mask bytes by sign-replicating permutes
#endif
// bytes 0 / 1 = the sign of a / b replicated (prmt generic mode: a selector
// nibble with bit 3 set copies the msb of the selected byte to all 8 bits)
__device__ __forceinline__ uint32_t prmt_sr(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
#ifndef MA_LEAN_SIGNCOUNT
#define MA_LEAN_SIGNCOUNT 1  // lean select: candidate counts as sums of sign bits
#endif
#ifndef MA_LEAN_PFLAG
#define MA_LEAN_PFLAG 1  // lean pass 2: code-boundary flags computed two elements per word
#endif
#ifndef MA_LEAN_CAPL
#define MA_LEAN_CAPL 4  // lean kernel: exact-stage candidate slots per lane
#endif
#ifndef MA_LEAN_PROF
#define MA_LEAN_PROF 0  // per-phase warp clock64 accumulation into dbg[8..] (profiling builds only)
#endif
#ifndef MA_LEAN_SB
#define MA_LEAN_SB 2  // ADAM_STATS: window entries per lane with loads in flight
#endif
#ifndef MA_LEAN_TARGET
#define MA_LEAN_TARGET 64  // lean kernel: carried-threshold target hit count
#endif
constexpr int kLCapL = MA_LEAN_CAPL;
constexpr int kLCap = 32 * kLCapL;
constexpr int kLTarget = MA_LEAN_TARGET;

// Per-warp shared-memory carve-up of the lean kernel (bytes).
struct LLayout {
    uint32_t ll, llf, sel, wpref, dup, cval, cidx, misc, total;
    __host__ __device__ LLayout() {}
    __host__ __device__ explicit LLayout(int bucket, int capl = kLCapL) {
        const size_t nbk = size_t(kBlk / bucket);
        const size_t kLCap = size_t(32 * capl);
        size_t o = 0;
        ll = uint32_t(o);    o = align_up(o + nbk * 16, 16);     // exact (lo, level), fp64
        llf = uint32_t(o);   o = align_up(o + nbk * 16, 16);     // (lo32, level32, E_q, Tf_q)
        sel = uint32_t(o);   o = align_up(o + kBlk / 8, 16);
        wpref = uint32_t(o);  // member list (int16 per candidate); word prefix; seen bits
        o = align_up(o + (kLCap * 2 > size_t(kBlk / 8) ? kLCap * 2 : size_t(kBlk / 8)), 16);
        dup = uint32_t(o);   o = align_up(o + kBlk / 8, 16);
        cval = uint32_t(o);  // candidates; radix histogram; bucket (lo, hi) keys; duplicate list
        o = align_up(o + (size_t(kLCap) * 8 > nbk * 16 ? size_t(kLCap) * 8 : nbk * 16), 16);
        cidx = uint32_t(o);  o = align_up(o + kLCap * 2, 16);
        misc = uint32_t(o);  o = align_up(o + 16 * 4, 16);
        total = uint32_t(align_up(o, 128));
    }
};

template <int DT>
__device__ __forceinline__ void g32x8(const Raw8<DT>& r, float (&g)[8]) {
    if constexpr (DT == BF16) {
        const uint32_t w[4] = {r.v[0].x, r.v[0].y, r.v[0].z, r.v[0].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            g[2 * k] = __uint_as_float(w[k] << 16);
            g[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            g[4 * k + 0] = __uint_as_float(r.v[k].x);
            g[4 * k + 1] = __uint_as_float(r.v[k].y);
            g[4 * k + 2] = __uint_as_float(r.v[k].z);
            g[4 * k + 3] = __uint_as_float(r.v[k].w);
        }
    }
}

// a32 = g + (c * level32 + lo32) for 8 elements. The nibble becomes a float by
// a byte permute into 2^23 + c (exact), no conversion instruction.
template <int DT>
__device__ __forceinline__ void a32x8(const Raw8<DT>& r, uint32_t cw, float lo32, float lv32, float (&a)[8]) {
    float g[8];
    g32x8<DT>(r, g);
    const uint32_t ce = cw & 0x0F0F0F0Fu, co = (cw >> 4) & 0x0F0F0F0Fu;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float c0 = __uint_as_float(__byte_perm(ce, 0x4B000000u, 0x7540u | k)) - kTwo23;
        const float c1 = __uint_as_float(__byte_perm(co, 0x4B000000u, 0x7540u | k)) - kTwo23;
        a[2 * k] = g[2 * k] + __fmaf_rn(c0, lv32, lo32);
        a[2 * k + 1] = g[2 * k + 1] + __fmaf_rn(c1, lv32, lo32);
    }
}

// Exact fp64 a of element i (runtime index) of a raw 8-group (same arithmetic
// as add_decoded8: optim.cpp:166-168, quantize.cpp:164-178).
template <int DT>
__device__ __forceinline__ double exact_a_raw(const Raw8<DT>& r, uint32_t cw, int i, double2 ll) {
    uint32_t bits;
    if constexpr (DT == BF16) {
        const int k = i >> 1;
        const uint32_t w = k == 0 ? r.v[0].x : (k == 1 ? r.v[0].y : (k == 2 ? r.v[0].z : r.v[0].w));
        bits = (i & 1) ? (w & 0xFFFF0000u) : (w << 16);
    } else {
        const uint4 v = (i >> 2) ? r.v[1] : r.v[0];
        const int k = i & 3;
        bits = k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
    }
    const double g = static_cast<double>(__uint_as_float(bits));
    return __dadd_rn(g, __dadd_rn(__dmul_rn(static_cast<double>((cw >> (4 * i)) & 15u), ll.y), ll.x));
}

// ---- pass 2 of the lean kernel: fp32 with exact fallbacks -----------------
// Lane l of iteration j owns the 16 elements [512 j + 16 l, +16): one B_q =
// 64 bucket is 4 lanes (2 for B_q = 32). With the previous grid (lo, level)
// and E = E_q of the pass-1 bound, the residual r32 = sel ? 0 : a32 obeys
// |r32 - r| <= eps := E + max|r32| 2^-23 over the bucket (0 for selected).
// For the bucket's fp32 extremes mn, mx the exact lo' = min r, hi' = max r
// lie within eps of them. With k2 = 30 / rd(mx - mn) (2-ulp division) and
// c2 = rn(257 + G - mn k2), y = rn(r32 k2 + c2) ∈ [256, 512) satisfies
//   y - 256 ∈ [1 + 2T, 1 + 2T + 2G],  T = 15 (r - lo') / (hi' - lo'),
// whenever G >= 121 eps / den + 30·2^-21 + |c2| 2^-24 + 2^-16 (den =
// rd(mx - mn) - 2 eps, the error of k2, of r32 - mn, of c2 and of y), which
// the kernel bounds by G = 128 eps / den + cmag 2^-23 + 2^-13. Let N =
// floor(y) - 256 (mantissa bits 22..15): an element whose y has fraction
// >= 2G has code floor(T + 0.5) = N >> 1 exactly (also against the
// reference's fp64 quotient, 2^-48 away from T). Elements with a smaller
// fraction are flagged: N even = a code boundary, recoded by the IEEE
// quotient (quantize.cpp:51-53) with the exact lo', level'; N = 1 holds every
// candidate for the exact minimum (T = 0 gives y - 256 ∈ [1, 1 + 2G]) and
// N = 31 every candidate for the maximum, whose exact fp64 residuals give
// (lo', hi'). Buckets with G > 1/16, R outside [2^-100, 2^100] or a
// non-finite bound run exactly in fp64 (exact_bucket16). The code of a
// fast-path element sits in byte 2 of y (bits 19..16 = N >> 1).
template <int DT>
struct Raw16 {
    static constexpr int N = DT == BF16 ? 2 : 4;
    uint4 v[N];
};
template <int DT, bool NC>
__device__ __forceinline__ Raw16<DT> load_raw16(const unsigned char* gp) {
    Raw16<DT> r;
    const uint4* q = reinterpret_cast<const uint4*>(gp);
#pragma unroll
    for (int k = 0; k < Raw16<DT>::N; ++k) {
        if constexpr (NC) r.v[k] = __ldg(q + k);
        else r.v[k] = q[k];
    }
    return r;
}
template <int DT>
__device__ __forceinline__ float g32_of(const Raw16<DT>& r, int i) {  // i: compile-time after unrolling
    if constexpr (DT == BF16) {
        const uint4 v = r.v[i >> 3];
        const int k = (i >> 1) & 3;
        const uint32_t w = k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
        return __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
    } else {
        const uint4 v = r.v[i >> 2];
        const int k = i & 3;
        return __uint_as_float(k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w)));
    }
}

// rn(bf16 + fp32) of the two bf16 halves of w (element 2k in the low half)
// and x: the mixed-precision add (FHADD.BF16) reads each half in place, so
// the gradient needs no unpacking (bit-identical to widening, then __fadd_rn)
__device__ __forceinline__ float2 add_bf16x2_f32(uint32_t w, float2 x) {
    float r0, r1;
    asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.bf16 %0, lo, %3; add.rn.f32.bf16 %1, hi, %4; }"
        : "=f"(r0), "=f"(r1)
        : "r"(w), "f"(x.x), "f"(x.y));
    return make_float2(r0, r1);
}
template <int DT>
__device__ __forceinline__ uint32_t raw16_word(const Raw16<DT>& r, int j) {  // j: compile-time after unrolling
    const uint4 v = r.v[j >> 2];
    const int k = j & 3;
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

// a32 of one block element, recomputed exactly as the packed decode does it.
template <class KT>
__device__ __forceinline__ float a32_at_w(const StepArgs& p, int64_t base, int e, float lo32, float lv32) {
    const uint32_t byte = p.codes[(base + e) >> 1];
    const float c = static_cast<float>((byte >> ((e & 1) * 4)) & 15u);
    float g;
    if constexpr (KT::GDT == BF16)
        g = __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(p.grads)[base + e]) << 16);
    else
        g = static_cast<const float*>(p.grads)[base + e];
    return __fadd_rn(g, __fmaf_rn(c, lv32, lo32));
}

// a at one block element with its bucket's exact (lo, level) given.
template <class KT>
__device__ __forceinline__ double recompute_a_q(const StepArgs& p, int64_t base, int e, double2 q) {
    const uint32_t byte = p.codes[(base + e) >> 1];
    const double ev = __dadd_rn(__dmul_rn(static_cast<double>((byte >> ((e & 1) * 4)) & 15u), q.y), q.x);
    return __dadd_rn(ld_t<KT::GDT>(p.grads, base + e), ev);
}

struct Bucket16 {
    uint32_t w0, w1;
    double lo, hi;
};
// The exact fp64 path for a lane's 16 elements of a bucket the fp32 bounds do
// not cover (quantize.cpp:15-24, 42-55 in the reference's operation order);
// `bm` = the bucket's lanes (they all call this together).
template <class KT>
__device__ __noinline__ Bucket16 exact_bucket16(const StepArgs* pp, int64_t base, int e0, uint32_t sel16, double2 ll,
                                                uint32_t bm, int lpb) {
    const StepArgs& p = *pp;
    double lo = CUDART_INF, hi = -CUDART_INF;
    for (int i = 0; i < 16; ++i) {
        const double r = ((sel16 >> i) & 1u) ? 0.0 : recompute_a_q<KT>(p, base, e0 + i, ll);
        lo = r < lo ? r : lo;
        hi = r > hi ? r : hi;
    }
    for (int off = 1; off < lpb; off <<= 1) {
        const double ol = __shfl_xor_sync(bm, lo, off), oh = __shfl_xor_sync(bm, hi, off);
        lo = ol < lo ? ol : lo;
        hi = oh > hi ? oh : hi;
    }
    Bucket16 o{0u, 0u, lo, hi};
    if (lo != hi) {
        const double level = div15_w(__dsub_rn(hi, lo));
        for (int i = 15; i >= 0; --i) {
            const double r = ((sel16 >> i) & 1u) ? 0.0 : recompute_a_q<KT>(p, base, e0 + i, ll);
            const uint32_t c = exact_code_w(r, lo, level);
            if (i >= 8) o.w1 = (o.w1 << 4) | c;
            else o.w0 = (o.w0 << 4) | c;
        }
    }
    return o;
}

// Codes from byte 2 of eight y words (bits 19..16 = N >> 1), low nibble first.
__device__ __forceinline__ uint32_t pack_codes8(const uint32_t* y) {
    const uint32_t ev = __byte_perm(__byte_perm(y[0], y[2], 0x0062u), __byte_perm(y[4], y[6], 0x0062u), 0x5410u);
    const uint32_t od = __byte_perm(__byte_perm(y[1], y[3], 0x0062u), __byte_perm(y[5], y[7], 0x0062u), 0x5410u);
    return (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
}

// ADAM_STATS + update of a coordinate held by exactly one window entry
// (row r, entry e): window.cpp:28-46 with one term, optim.cpp:183-187, in the
// reference's fp64 operation order. Out of line for the bf16-θ screen below.
template <class KT>
__device__ __noinline__ void exact_update(const StepArgs* pp, int64_t base, const unsigned char* gwv, int e,
                                          int r, int idx) {
    const StepArgs& p = *pp;
    const double v = ld_t<KT::VDT>(gwv, e);
    const double th = ld_t<KT::PDT>(p.params, base + idx);
    const double mhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w1[r], v)), p.scale1);
    const double vhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(v, v))), p.scale2);
    const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
    st_t<KT::PDT>(p.params, base + idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
}

// bf16 θ: the fp32 estimate x32 = θ - lr32 * c1 v / (eps32 + |v| c2) is within
// |lr u| 2^-20.6 + |x| 2^-24 of the fp64 result x (9 fp32 roundings of at most
// 2^-24 and a 2-ulp division, against < 2^-49 for the fp64 chain). With
// |lr u| <= 2^(e+4) (e = exponent of x32) that is < 86 fp32 ulps of x32's
// binade (172 across a binade edge), so when the 16 bits below the bf16
// mantissa are more than 512 ulps from the rounding midpoint 0x8000, x and x32
// round to the same bf16. Everything else takes exact_update.
template <class KT>
struct UniqueUpd {
    static constexpr bool kScreen = KT::PDT == BF16 && KT::VDT != F64;
    float th = 0.0f, v = 0.0f;
    // thb: the block's θ (element 0 = block element 0); gwv: its value ring
    __device__ __forceinline__ void load(const void* thb, const unsigned char* gwv, int e, int idx) {
        if constexpr (kScreen) {
            th = __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(thb)[idx]) << 16);
            v = KT::VDT == BF16
                    ? __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(gwv)[e]) << 16)
                    : reinterpret_cast<const float*>(gwv)[e];
        }
    }
    __device__ __forceinline__ void finish(const StepArgs& p, int64_t base, void* thb, const unsigned char* gwv,
                                           int e, int r, int idx) {
        if constexpr (kScreen) {
            const float den = __fmaf_rn(fabsf(v), p.c2[r], p.eps32);
            const float u = __fdividef(p.c1[r] * v, den);
            const float x = __fmaf_rn(-p.lr32, u, th);
            const uint32_t xb = __float_as_uint(x);
            const uint32_t ex = (xb >> 23) & 0xFFu;
            const int mid = static_cast<int>(xb & 0xFFFFu) - 0x8000;
            const bool ok = ex >= 27u && ex <= 227u && den < 0x1p120f &&
                            fabsf(p.lr32 * u) <= __uint_as_float((ex + 4u) << 23) && (mid > 512 || mid < -512);
            if (ok) static_cast<uint16_t*>(thb)[idx] = static_cast<uint16_t>((xb + 0x7FFFu + ((xb >> 16) & 1u)) >> 16);
            else exact_update<KT>(&p, base, gwv, e, r, idx);
        } else {
            const double vv = ld_t<KT::VDT>(gwv, e);
            const double t = ld_t<KT::PDT>(thb, idx);
            const double mhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w1[r], vv)), p.scale1);
            const double vhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(vv, vv))), p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            st_t<KT::PDT>(thb, idx, __dsub_rn(t, __dmul_rn(p.lr, u)));
        }
    }
};

// ADAM_STATS + update of a coordinate held by one window entry, with θ (or the
// 4-byte word holding a bf16 θ) staged at `sth` and the value in the staged
// rows `swv` (same arithmetic and screen as UniqueUpd).
template <class KT>
__device__ __forceinline__ void unique_update_smem(const StepArgs& p, int64_t base, void* thb, const unsigned char* gwv,
                                                   const unsigned char* swv, const unsigned char* sth, int e, int r,
                                                   int idx) {
    if constexpr (KT::PDT == BF16 && KT::VDT != F64) {
        const uint32_t word = *reinterpret_cast<const uint32_t*>(sth);
        const float th = __uint_as_float((idx & 1) ? (word & 0xFFFF0000u) : (word << 16));
        const float v = KT::VDT == BF16
                            ? __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(swv)[e]) << 16)
                            : reinterpret_cast<const float*>(swv)[e];
        const float den = __fmaf_rn(fabsf(v), p.c2[r], p.eps32);
        const float u = __fdividef(p.c1[r] * v, den);
        const float x = __fmaf_rn(-p.lr32, u, th);
        const uint32_t xb = __float_as_uint(x);
        const uint32_t ex = (xb >> 23) & 0xFFu;
        const int mid = static_cast<int>(xb & 0xFFFFu) - 0x8000;
        const bool ok = ex >= 27u && ex <= 227u && den < 0x1p120f &&
                        fabsf(p.lr32 * u) <= __uint_as_float((ex + 4u) << 23) && (mid > 512 || mid < -512);
        if (ok) static_cast<uint16_t*>(thb)[idx] = static_cast<uint16_t>((xb + 0x7FFFu + ((xb >> 16) & 1u)) >> 16);
        else exact_update<KT>(&p, base, gwv, e, r, idx);
    } else {
        const double vv = ld_t<KT::VDT>(swv, e);
        const double t = KT::PDT == BF16 ? static_cast<double>(__uint_as_float(
                                               (idx & 1) ? (*reinterpret_cast<const uint32_t*>(sth) & 0xFFFF0000u)
                                                         : (*reinterpret_cast<const uint32_t*>(sth) << 16)))
                                         : ld_t<KT::PDT>(sth, 0);
        const double mhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w1[r], vv)), p.scale1);
        const double vhat = __dmul_rn(__dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(vv, vv))), p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        st_t<KT::PDT>(thb, idx, __dsub_rn(t, __dmul_rn(p.lr, u)));
    }
}

// Stage the block's window rows in shared memory when they fit next to the
// LLayout area without dropping below 8 resident CTAs per SM.
__host__ __device__ __forceinline__ bool lean_stage_rows(int m, int kbs, int vsz) {
    return size_t(m) * size_t(kbs) * size_t(2 + vsz) <= 2048;
}
__device__ __forceinline__ int16_t* gwi_of(const StepArgs& p, int64_t b, int /*vsz*/) {
    return p.win_idx + b * p.m * static_cast<int64_t>(p.kb_stride);
}
__device__ __forceinline__ unsigned char* gwv_of(const StepArgs& p, int64_t b, int vsz) {
    return static_cast<unsigned char*>(p.win_val) + b * p.m * static_cast<int64_t>(p.kb_stride) * vsz;
}

// The block's m window rows -> shared memory by two 1-D bulk copies completing
// on one mbarrier (lane 0; phase 0 is awaited before the rows are used).
__device__ __forceinline__ void stage_rows(uint64_t* bar, void* s_idx, const void* g_idx, void* s_val, const void* g_val,
                                           uint32_t bytes_idx, uint32_t bytes_val) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, bytes_idx + bytes_val);
    bulk_g2s(s_idx, g_idx, bytes_idx, bar);
    bulk_g2s(s_val, g_val, bytes_val, bar);
}

// Duplicated coordinates beyond one warp's worth of list entries
// (window.cpp:32-39: terms summed in physical slot order). The ordered entry
// list is taken 32 entries at a time; match.any groups a coordinate's entries,
// its lowest lane continues the coordinate's running sums (carried in smem
// across chunks) in lane order; then one lane per coordinate applies the
// update. Needs <= 64 distinct coordinates and an un-overflowed list; returns
// false (nothing done) otherwise. Out of line: keeps the hot kernel's
// register allocation untouched.
template <class KT>
__device__ __noinline__ bool dup_chunks(const StepArgs* pp, unsigned char* ws, int64_t b, int ndup) {
    const StepArgs& p = *pp;
    const LLayout L(KT::BUCKET, KT::CAPL);
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    const int lane = threadIdx.x & 31;
    const int kbs = p.kb_stride;
    const int64_t base = b * kBlk;
    const int64_t went = b * p.m * static_cast<int64_t>(kbs);
    const unsigned char* gwv = static_cast<const unsigned char*>(p.win_val) + went * vsz;
    const uint32_t* s_dup = reinterpret_cast<const uint32_t*>(ws + L.dup);
    const int* dupl = reinterpret_cast<const int*>(ws + L.cval);
    if (ndup > static_cast<int>((L.cidx - L.cval) / 4)) return false;  // the list overflowed
    uint32_t dv[4];
    int loc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        dv[k] = s_dup[lane * 4 + k];
        loc += __popc(dv[k]);
    }
    int ndupc;
    int run = warp_excl_scan(loc, lane, ndupc);
    int* s_dpref = reinterpret_cast<int*>(ws + L.wpref);  // the claim bits of dup_stats are not needed
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_dpref[lane * 4 + k] = run;
        run += __popc(dv[k]);
    }
    // running sums of up to zcap coordinates at a time in the dead pass-2
    // tables and selection bits (ll, llf, sel) — NOT into wpref (s_dpref) or
    // dup (s_dup), which this loop still reads
    double2* zz = reinterpret_cast<double2*>(ws + L.ll);
    int16_t* zc = reinterpret_cast<int16_t*>(ws + L.cidx);
    const int zcap = min(static_cast<int>((L.wpref - L.ll) / 16), static_cast<int>((L.misc - L.cidx) / 2));
    __syncwarp();
    for (int id0 = 0; id0 < ndupc; id0 += zcap) {
        const int nz = min(zcap, ndupc - id0);
        for (int i = lane; i < nz; i += 32) zz[i] = make_double2(0.0, 0.0);
        __syncwarp();
        for (int c0 = 0; c0 < ndup; c0 += 32) {
            bool has = c0 + lane < ndup;
            const int x = has ? dupl[c0 + lane] : 0;
            const int idx = dup_idx(x), r = dup_row(x), pos = dup_pos(x);
            int id = 0;
            if (has) {
                id = s_dpref[idx >> 5] + __popc(s_dup[idx >> 5] & ((1u << (idx & 31)) - 1u)) - id0;
                has = id >= 0 && id < nz;
            }
            double t1 = 0.0, t2 = 0.0;
            if (has) {
                const double v = ld_t<KT::VDT>(gwv, r * kbs + pos);
                t1 = __dmul_rn(p.w1[r], v);
                t2 = __dmul_rn(p.w2[r], __dmul_rn(v, v));
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, has ? idx : -1 - lane);
            const int cnt = has ? __popc(peers) : 0;
            const int maxc = __reduce_max_sync(0xFFFFFFFFu, cnt);
            const bool leader = has && (__ffs(peers) - 1) == lane;
            double z1 = 0.0, z2 = 0.0;
            if (leader) {
                const double2 zc0 = zz[id];
                z1 = zc0.x;
                z2 = zc0.y;
            }
            uint32_t rem = peers;
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
            if (leader) {
                zz[id] = make_double2(z1, z2);
                zc[id] = static_cast<int16_t>(idx);
            }
            __syncwarp();
        }
        for (int i = lane; i < nz; i += 32) {
            const int idx = zc[i];
            const double2 z = zz[i];
            const double mhat = __dmul_rn(z.x, p.scale1);
            const double vhat = __dmul_rn(z.y, p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            const double th = ld_t<KT::PDT>(p.params, base + idx);
            st_t<KT::PDT>(p.params, base + idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        }
        __syncwarp();
    }
    return true;
}

#if MA_LEAN_PROF
// Adds the cycles since the previous mark to phase counter k-1 (dbg[8..] as u64).
__device__ __forceinline__ void prof_mark(const StepArgs& p, int k) {
    __shared__ long long t_prev[kWarps];
    const int w = threadIdx.x >> 5;
    __syncwarp();
    const long long t = clock64();
    if ((threadIdx.x & 31) == 0) {
        if (k > 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(p.dbg + 8) + (k - 1),
                      static_cast<unsigned long long>(t - t_prev[w]));
        t_prev[w] = t;
    }
    __syncwarp();
}
#endif

// PH: 3 = the fused step; 1 = front only (EF decode, Top-K, window row + stage
// copy, EF re-quantization); 2 = ADAM_STATS + update only (sparse propagation).
#ifndef MA_LEAN_MINB
#define MA_LEAN_MINB 8  // resident CTAs per SM the lean kernel is compiled for (64 registers)
#endif
template <class KT, int PH = 3>
__global__ void __launch_bounds__(32 * kWarps, MA_LEAN_MINB) microadam_step_lean(const __grid_constant__ StepArgs p) {
    constexpr int BUCKET = KT::BUCKET, LPB = KT::LPB;
    constexpr int gsz = KT::GDT == F32 ? 4 : 2;
    constexpr int psz = KT::PDT == F64 ? 8 : (KT::PDT == F32 ? 4 : 2);
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    constexpr int NBK = kBlk / BUCKET;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bl = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (bl >= p.block_count) return;
#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 0);
#endif
    const int64_t b = p.block_offset + bl;
    const int64_t base = b * kBlk;
    const LLayout L(BUCKET, KT::CAPL);
    // PH & 2: the block's m window rows (indices, then values) are staged after
    // the warp's LLayout area by one bulk copy issued in the prologue
    // (only while that keeps 8 CTAs per SM: lean_stage_rows; else the rows are
    // read from global memory through the same pointers)
    const bool stage = (PH & 2) && lean_stage_rows(p.m, p.kb_stride, vsz);
    const uint32_t wrow_i = stage ? static_cast<uint32_t>(align_up(size_t(p.m) * p.kb_stride * 2, 16)) : 0u;
    const uint32_t wrow_v = stage ? static_cast<uint32_t>(align_up(size_t(p.m) * p.kb_stride * vsz, 16)) : 0u;
    unsigned char* ws = smem + warp * (L.total + wrow_i + wrow_v);
    int16_t* s_widx = stage ? reinterpret_cast<int16_t*>(ws + L.total) : gwi_of(p, b, vsz);
    unsigned char* s_wval = stage ? ws + L.total + wrow_i : gwv_of(p, b, vsz);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(ws + L.misc + 48);
    double2* s_ll = reinterpret_cast<double2*>(ws + L.ll);
    float4* s_llf = reinterpret_cast<float4*>(ws + L.llf);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(ws + L.sel);
    int* s_wpref = reinterpret_cast<int*>(ws + L.wpref);
    int16_t* s_memb = reinterpret_cast<int16_t*>(ws + L.wpref);
    uint32_t* s_seen = reinterpret_cast<uint32_t*>(ws + L.wpref);
    uint32_t* s_dup = reinterpret_cast<uint32_t*>(ws + L.dup);
    double* s_cval = reinterpret_cast<double*>(ws + L.cval);
    int16_t* s_cidx = reinterpret_cast<int16_t*>(ws + L.cidx);
    int* s_misc = reinterpret_cast<int*>(ws + L.misc);
    const int kb = p.per_block_k, kbs = p.kb_stride, m = p.m, slot = p.slot, filled = p.filled;
    const int64_t went = b * m * static_cast<int64_t>(kbs);
    int16_t* gwi = p.win_idx + went;
    unsigned char* gwv = static_cast<unsigned char*>(p.win_val) + went * vsz;

    if constexpr (PH & 1) {
    if constexpr (KT::RS) {
        // ---- fused reduce-scatter (ma_step_reduce): this block's gradient is
        //      ((src_0 + src_1) + ...) * scale in fp32, rank order, rounded to the
        //      gradient dtype and written to p.grads, which the passes below read
        //      back (same lane, same addresses in pass 1; L1/L2 hits). Sources
        //      are peer (NVLink) or local pointers; loads of G ranks in flight.
        constexpr int G = KT::GDT == BF16 ? kMaxRanks : kMaxRanks / 2;
        const int n = p.rs_n;
#pragma unroll 1
        for (int j = 0; j < kIter; ++j) {
            const int64_t e = base + j * 256 + lane * 8;
            float acc[8];
#pragma unroll 1
            for (int r0 = 0; r0 < n; r0 += G) {
                Raw8<KT::GDT> v[G];
#pragma unroll
                for (int q = 0; q < G; ++q)
                    if (r0 + q < n) v[q] = load_raw8<KT::GDT, false>(p.rs_src[r0 + q], e);
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    if (r0 + q < n) {
                        float x[8];
                        g32x8<KT::GDT>(v[q], x);
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i] = (r0 + q == 0) ? x[i] : __fadd_rn(acc[i], x[i]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fmul_rn(acc[i], p.rs_scale);
            unsigned char* dst = static_cast<unsigned char*>(const_cast<void*>(p.grads)) + e * gsz;
            if constexpr (KT::GDT == BF16) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(bf16x2_bits(acc[0], acc[1]), bf16x2_bits(acc[2], acc[3]),
                                                            bf16x2_bits(acc[4], acc[5]), bf16x2_bits(acc[6], acc[7]));
            } else {
                reinterpret_cast<float4*>(dst)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                reinterpret_cast<float4*>(dst)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        if constexpr (!KT::RS) prefetch_l2_keep(static_cast<const unsigned char*>(p.grads) + base * gsz, kBlk * gsz);
        prefetch_l2_keep(p.codes + base / 2, kBlk / 2);
        prefetch_l2(p.meta + base / BUCKET, NBK * 16);
        if ((PH & 2) && stage) stage_rows(s_bar, s_widx, gwi, s_wval, gwv, m * kbs * 2, m * kbs * vsz);
    }
    const uint32_t tstate = __ldg(p.thresh + b);
    const uint32_t T = tstate & 0xFFFFu;
    // V_T: the smallest |a| with key16 >= T (quantize-free: bits 62..48)
    const double VT = __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(T) << 48));
    for (int i = lane; i < NBK; i += 32) {
        const double2 mt = p.meta[base / BUCKET + i];
        const double level = (mt.x == mt.y) ? 0.0 : div15_w(__dsub_rn(mt.y, mt.x));
        s_ll[i] = make_double2(mt.x, level);
        const double M = fmax(fabs(mt.x), fabs(mt.y));
        float E = __double2float_ru(M * 0x1p-21 + 0x1p-120);
        if (!(M < 0x1p100)) E = CUDART_INF_F;
        float Tf = CUDART_INF_F;  // T == 0: no carried threshold, no screen hits
        if (T != 0) Tf = __double2float_rd((VT - static_cast<double>(E)) * (1.0 - 0x1p-22));
        if (!(Tf > 0.0f)) Tf = 0.0f;
        // pass 1 tests a32² - T2 >= 0 with T2 = rd(Tf²) <= Tf² (stored negated)
        s_llf[i] = make_float4(__double2float_rn(mt.x), __double2float_rn(level), E, -__fmul_rd(Tf, Tf));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_sel[lane * 4 + k] = 0;
        s_dup[lane * 4 + k] = 0;
    }
    if (lane == 0) s_misc[8] = 0x4B000000;  // opaque_kmag's word
    __syncwarp();

#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 1);
#endif
    // ---- pass 1: fp32 screen of a = g + decode(EF) against the carried threshold ----
    // Packed fp32 (FFMA2 / FADD2): c as a float by a byte permute into 2^23 + c,
    // a32 = g + (c·level32 + lo32); hit <=> a32² - T2 >= 0 (T2 = rd(Tf²): a
    // superset of |a32| >= Tf; inf / NaN give +inf / the canonical +NaN, hits).
    // The sign bytes of 8 squares are gathered by byte permutes into one word:
    // byte k, bit 2·(3 - jj) + h holds MISS of element k + 4h of iteration
    // 4w + jj; four iterations fill cm_w (bits inverted at the end).
    uint32_t cm0 = 0, cm1 = 0, cm2 = 0, cm3 = 0;
    {
        const unsigned char* gp = static_cast<const unsigned char*>(p.grads) + (base + lane * 8) * gsz;
        const uint32_t* cp = reinterpret_cast<const uint32_t*>(p.codes + ((base + lane * 8) >> 1));
        const float4* lf = s_llf + (lane * 8) / BUCKET;
        const float2 m23 = make_float2(-kTwo23, -kTwo23);
#pragma unroll 1
        for (int w = 0; w < 4; ++w) {
            // 0x4B000000 in a register: the permutes below take immediate selectors
            const uint32_t kmag = opaque_kmag(s_misc + 8);
            uint32_t acc = 0;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = w * 4 + jj;
                const Raw8<KT::GDT> r = load_raw8<KT::GDT, !KT::RS>(gp + size_t(j) * 256 * gsz, 0);
                const uint32_t cw = cp[j * 32];
                const float4 f = lf[j * (256 / BUCKET)];
                const uint32_t ce = cw & 0x0F0F0F0Fu, co = (cw >> 4) & 0x0F0F0F0Fu;
                float g[8];
                g32x8<KT::GDT>(r, g);
                const float2 lv2 = make_float2(f.y, f.y), lo2 = make_float2(f.x, f.x), t2 = make_float2(f.w, f.w);
                uint32_t sg[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float2 c = make_float2(__uint_as_float(prmt_imm<0x7540u>(ce, kmag, k)),
                                           __uint_as_float(prmt_imm<0x7540u>(co, kmag, k)));
                    c = __fadd2_rn(c, m23);
#if MA_LEAN_MIXADD
                    float2 a;
                    if constexpr (KT::GDT == BF16) {
                        const uint32_t wk = k == 0 ? r.v[0].x : (k == 1 ? r.v[0].y : (k == 2 ? r.v[0].z : r.v[0].w));
                        a = add_bf16x2_f32(wk, __ffma2_rn(c, lv2, lo2));
                    } else {
                        a = __fadd2_rn(make_float2(g[2 * k], g[2 * k + 1]), __ffma2_rn(c, lv2, lo2));
                    }
#else
                    const float2 a = __fadd2_rn(make_float2(g[2 * k], g[2 * k + 1]), __ffma2_rn(c, lv2, lo2));
#endif
                    const float2 d = __ffma2_rn(a, a, t2);
                    sg[2 * k] = __float_as_uint(d.x);
                    sg[2 * k + 1] = __float_as_uint(d.y);
                }
#if MA_LEAN_SIGNREP
                // sign-replicated top bytes (prmt selector nibbles 0xB / 0xF: byte 3 of
                // each operand, msb replicated): byte k of w0 / w1 is 0xFF when
                // element k / k + 4 misses, so no shifts are needed below
                const uint32_t w0 = __byte_perm(prmt_sr(sg[0], sg[1]), prmt_sr(sg[2], sg[3]), 0x5410u);
                const uint32_t w1 = __byte_perm(prmt_sr(sg[4], sg[5]), prmt_sr(sg[6], sg[7]), 0x5410u);
                const uint32_t b = (w0 & 0x01010101u) | (w1 & 0x02020202u);
#else
                // top (sign) bytes of elements 0..3 and 4..7
                const uint32_t w0 = __byte_perm(__byte_perm(sg[0], sg[1], 0x0073u), __byte_perm(sg[2], sg[3], 0x0073u), 0x5410u);
                const uint32_t w1 = __byte_perm(__byte_perm(sg[4], sg[5], 0x0073u), __byte_perm(sg[6], sg[7], 0x0073u), 0x5410u);
                // byte k: bit 0 = sign of element k, bit 1 = sign of element k + 4
                const uint32_t b = ((w0 >> 7) & 0x01010101u) | ((w1 >> 6) & 0x02020202u);
#endif
                acc = (acc << 2) | b;
            }
            cm0 = cm1;
            cm1 = cm2;
            cm2 = cm3;
            cm3 = ~acc;
        }
    }
    const int nmine = __popc(cm0) + __popc(cm1) + __popc(cm2) + __popc(cm3);
    const int cnt = __reduce_add_sync(0xFFFFFFFFu, nmine);
    auto for_hits = [&](auto&& f) {
#pragma unroll 1
        for (int w = 0; w < 4; ++w) {
            uint32_t bits = w == 0 ? cm0 : (w == 1 ? cm1 : (w == 2 ? cm2 : cm3));
            while (bits) {
                const int sb = __ffs(bits) - 1;
                bits &= bits - 1;
                // byte k = sb >> 3; within it bit 2·(3 - jj) + h -> element k + 4h of iteration 4w + jj
                const int jj = 3 - ((sb & 7) >> 1);
                f((w * 4 + jj) * 256 + lane * 8 + (sb >> 3) + 4 * (sb & 1));
            }
        }
    };

#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 2);
#endif
    // ---- block Top-K (compress.cpp:39-53, 73-85) ----
    // Candidates: a superset of the keys >= base16 (key16 units) whose exact
    // values sit in s_cval / s_cidx; floor16: every key16 >= floor16 is a candidate.
    int ncand = -1;
    uint32_t base16 = T, floor16 = T;
    if (T != 0 && cnt > (32 * KT::CAPL) && cnt <= kRefineMax) {
        // Overfull screen: refine from the hit mask (key16 histogram of the
        // exact hits at or above T) instead of re-reading the block.
        uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.cval);
        hist[lane] = 0;
        __syncwarp();
        for_hits([&](int e) {
            const uint32_t k16 = hi_key(recompute_a<KT>(p, base, s_ll, e)) >> 16;
            if (k16 >= T) atomicAdd(&hist[min(k16 - T, 31u)], 1u);
        });
        __syncwarp();
        int sfx = static_cast<int>(hist[lane]);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_down_sync(0xFFFFFFFFu, sfx, off);
            if (lane + off < 32) sfx += t;
        }
        const uint32_t ok = __ballot_sync(0xFFFFFFFFu, sfx >= kb);
        __syncwarp();
        if (ok) {
            const int d = 31 - __clz(ok);
            const int n = __shfl_sync(0xFFFFFFFFu, sfx, d);
            if (n <= (32 * KT::CAPL)) {
                const uint32_t T1 = T + static_cast<uint32_t>(d);
                if (lane == 0) s_misc[4] = 0;
                __syncwarp();
                for_hits([&](int e) {
                    const double a = recompute_a<KT>(p, base, s_ll, e);
                    if ((hi_key(a) >> 16) >= T1) {
                        const int q = atomicAdd(&s_misc[4], 1);
                        s_cval[q] = a;
                        s_cidx[q] = static_cast<int16_t>(e);
                    }
                });
                __syncwarp();
                ncand = n;
                base16 = floor16 = T1;
            }
        }
        if (p.dbg && lane == 0) atomicAdd(p.dbg + 6, 1u);
    } else if (T != 0 && cnt >= kb && cnt <= (32 * KT::CAPL)) {
        int total;
        int pos = warp_excl_scan(nmine, lane, total);
        for_hits([&](int e) {
            s_cval[pos] = recompute_a<KT>(p, base, s_ll, e);
            s_cidx[pos] = static_cast<int16_t>(e);
            ++pos;
        });
        ncand = cnt;
        __syncwarp();
    }
    // 31-bit high words of the candidates' |a| keys (bits 62..32), 0 = empty slot
    uint32_t kh[KT::CAPL];
    auto load_keys = [&]() {
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s) {
            const int q = lane + 32 * s;
            kh[s] = q < ncand ? hi_key(s_cval[q]) : 0u;
        }
    };
    auto count_ge = [&](uint32_t v) {
#if MA_LEAN_SIGNCOUNT
        // keys kh < 2^31 and 0 <= v <= 2^31: kh >= v <=> (v - 1 - kh) < 0 as a
        // 32-bit signed value, so the count is a sum of sign bits (IADD3 + LEA.HI
        // per slot instead of a compare and a select); v above 2^31 (a carried
        // threshold near the inf / NaN keys) counts nothing, as v = 2^31 does
        const uint32_t vm1 = min(v, 0x80000000u) - 1u;
        uint32_t c = 0;
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s) c += (vm1 - kh[s]) >> 31;
        return __reduce_add_sync(0xFFFFFFFFu, static_cast<int>(c));
#else
        int c = 0;
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s) c += kh[s] >= v;
        return __reduce_add_sync(0xFFFFFFFFu, c);
#endif
    };
    load_keys();
    int clo = ncand < 0 ? 0 : count_ge(base16 << 16);
    if (clo < kb) {
        ncand = slow_select<KT, LLayout>(&p, ws, b);
        if (p.dbg && lane == 0) {
            atomicAdd(p.dbg + 2, 1u);
            if (cnt > (32 * KT::CAPL)) atomicAdd(p.dbg + 3, 1u);
        }
        if (ncand >= 0) {
            const uint32_t ph = static_cast<uint32_t>(s_misc[0]);  // prefix bits 62..32
            base16 = ph >> 16;
            floor16 = (ph + 0xFFFFu) >> 16;
            load_keys();
            clo = count_ge(base16 << 16);
        }
    }
    uint32_t next_t;
    uint32_t selc = 0;
    if (ncand >= 0) {
        uint32_t kml = 0;
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s) kml = max(kml, kh[s]);
        const uint32_t kmax = __reduce_max_sync(0xFFFFFFFFu, kml);
        if (p.check_finite && kmax >= 0x7FF00000u && lane == 0) atomicOr(p.flag, 1u);  // inf/NaN in g or a
        // Bisection for a high word lo with count(lo) >= kb > count(hi), stopping
        // early once count(lo) == kb (then the keys >= lo are the selection).
        uint32_t lo = base16 << 16, hi = kmax + 1;
        while (clo != kb && hi - lo > 1) {
            const uint32_t mid = lo + (hi - lo) / 2;
            const int c = count_ge(mid);
            if (c >= kb) {
                lo = mid;
                clo = c;
            } else {
                hi = mid;
            }
        }
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s)
            if (kh[s] > lo || (clo == kb && kh[s] == lo)) selc |= 1u << s;
        if (clo != kb) {
            // lo is the k_b-th high word and ties on it: rank the tied keys on the
            // full key, then the lower index (compress.cpp:43-48). Rare.
            const int need = kb - count_ge(lo + 1);
            int nm = 0;
#pragma unroll
            for (int s = 0; s < KT::CAPL; ++s) {
                const bool mem = kh[s] == lo && lane + 32 * s < ncand;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mem);
                if (mem) s_memb[nm + __popc(bal & lanemask_lt())] = static_cast<int16_t>(lane + 32 * s);
                nm += __popc(bal);
            }
            __syncwarp();
#pragma unroll
            for (int s = 0; s < KT::CAPL; ++s) {
                const int q = lane + 32 * s;
                if (kh[s] == lo && q < ncand) {
                    const uint64_t kq = key_of(s_cval[q]);
                    const int iq = s_cidx[q];
                    int rank = 0;
                    for (int t = 0; t < nm; ++t) {
                        const int o = s_memb[t];
                        const uint64_t ko = key_of(s_cval[o]);
                        rank += (ko > kq) || (ko == kq && s_cidx[o] < iq);
                    }
                    if (rank < need) selc |= 1u << s;
                }
            }
            __syncwarp();
            if (p.dbg && lane == 0) atomicAdd(p.dbg + 7, 1u);
        }
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s)
            if ((selc >> s) & 1u) {
                const int e = s_cidx[lane + 32 * s];
                atomicOr(&s_sel[e >> 5], 1u << (e & 31));
            }
        // next threshold (the exact kernel's rule): the largest key16 t in
        // [floor16, lo16] whose candidate count reaches `want`
        const int planned = T ? static_cast<int>(tstate >> 16) : 0;
        const int target = max(kLTarget, kb + (kb >> 1));
        int want = planned ? (target * planned) / max(cnt, 1) : target;
        want = min(max(want, kb + (kb >> 2)), (32 * KT::CAPL) - ((32 * KT::CAPL) >> 2));
        const uint32_t lo16 = lo >> 16;
        const uint32_t fl = min(floor16, lo16);
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
        const uint32_t h = static_cast<uint32_t>(s_misc[1]) >> 16;
        next_t = h > 2 ? h - 2 : 1u;
    }
    if (lane == 0) p.thresh[b] = (next_t & 0xFFFFu) ? next_t : (next_t | 1u);
    __syncwarp();

#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 3);
#endif
    // ---- window row `slot` (window.cpp:14-26): ascending positions ----
    {
        uint32_t wv[4];
        int loc = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            wv[k] = s_sel[lane * 4 + k];
            loc += __popc(wv[k]);
        }
        int tot;
        int run = warp_excl_scan(loc, lane, tot);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            s_wpref[lane * 4 + k] = run;
            run += __popc(wv[k]);
        }
    }
    __syncwarp();
    const int64_t row0 = static_cast<int64_t>(slot) * kbs;
    if ((PH & 2) && stage) {
        // the staged copy of the ring (issued in the prologue) must land before
        // this step's row overwrites slot `slot` in it
        while (!mbar_try_wait(s_bar, 0)) {
        }
    }
    if (ncand >= 0) {
#pragma unroll
        for (int s = 0; s < KT::CAPL; ++s)
            if ((selc >> s) & 1u) {
                const int q = lane + 32 * s;
                const int e = s_cidx[q];
                const int pos = s_wpref[e >> 5] + __popc(s_sel[e >> 5] & ((1u << (e & 31)) - 1u));
                gwi[row0 + pos] = static_cast<int16_t>(e);
                st_t<KT::VDT>(gwv, row0 + pos, s_cval[q]);
                if ((PH & 2) && stage) {
                    s_widx[row0 + pos] = static_cast<int16_t>(e);
                    st_t<KT::VDT>(s_wval, row0 + pos, s_cval[q]);
                }
                if constexpr (PH == 1) {
                    const int64_t so = (b - p.stage_b0) * kbs + pos;
                    p.stage_idx[so] = static_cast<int16_t>(e);
                    st_t<KT::VDT>(p.stage_val, so, s_cval[q]);
                }
            }
    } else {
        for (int w = lane; w < kBlk / 32; w += 32) {
            uint32_t bits = s_sel[w];
            int pos = s_wpref[w];
            while (bits) {
                const int e = w * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                gwi[row0 + pos] = static_cast<int16_t>(e);
                const double av = recompute_a<KT>(p, base, s_ll, e);
                st_t<KT::VDT>(gwv, row0 + pos, av);
                if ((PH & 2) && stage) {
                    s_widx[row0 + pos] = static_cast<int16_t>(e);
                    st_t<KT::VDT>(s_wval, row0 + pos, av);
                }
                if constexpr (PH == 1) {
                    const int64_t so = (b - p.stage_b0) * kbs + pos;
                    p.stage_idx[so] = static_cast<int16_t>(e);
                    st_t<KT::VDT>(p.stage_val, so, av);
                }
                ++pos;
            }
        }
    }
    __threadfence_block();
    __syncwarp();

#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 4);
#endif
    // ---- pass 2: residual (compress.cpp:95-102) + 4-bit re-quantization
    //      (quantize.cpp:15-24, 42-55, 102-114, 142-162): fp32 with exact
    //      fallbacks (see the bound above exact_bucket16) ----
    {
        constexpr int LP2 = BUCKET / 16;  // lanes per bucket in this pass
        const uint32_t bm = ((1u << LP2) - 1u) << (lane & ~(LP2 - 1));
        // 2 KB of scratch: the word-prefix / seen, duplicate and candidate areas
        // (re-zeroed below before ADAM_STATS uses them)
        unsigned char* s_scr = ws + L.wpref;
        const unsigned char* gp = static_cast<const unsigned char*>(p.grads) + base * gsz;
        const float2 m23 = make_float2(-kTwo23, -kTwo23);
#if MA_LEAN_THPF_LOOP == 0
        if ((PH & 2) && lane == 0) prefetch_l2(static_cast<const unsigned char*>(p.params) + base * psz, kBlk * psz);
#endif
#pragma unroll 1
        for (int j = 0; j < kBlk / 512; ++j) {
            const int e0 = j * 512 + lane * 16;
            const uint32_t kmag = opaque_kmag(s_misc + 8);
#if MA_LEAN_THPF_LOOP == 1
            if ((PH & 2) && j == 4 && lane == 0)
                prefetch_l2(static_cast<const unsigned char*>(p.params) + base * psz, kBlk * psz);
#elif MA_LEAN_THPF_LOOP == 2
            if ((PH & 2) && j == 4) {
                // per-lane L2 prefetch of the block's θ lines (no uniform-address
                // sequence for a bulk prefetch, which ran predicated every iteration)
                const unsigned char* th = static_cast<const unsigned char*>(p.params) + base * psz;
#pragma unroll
                for (int q = lane * 128; q < kBlk * psz; q += 32 * 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(th + q));
            }
#endif
            const Raw16<KT::GDT> raw = load_raw16<KT::GDT, !KT::RS>(gp + size_t(e0) * gsz);
            const uint2 cw = *reinterpret_cast<const uint2*>(p.codes + ((base + e0) >> 1));
            const float4 f = s_llf[e0 / BUCKET];
            const uint32_t sel16 = (s_sel[e0 >> 5] >> (e0 & 31)) & 0xFFFFu;
            float r[16];
            {
                const float2 lv2 = make_float2(f.y, f.y), lo2 = make_float2(f.x, f.x);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t c = h ? cw.y : cw.x;
                    const uint32_t ce = c & 0x0F0F0F0Fu, co = (c >> 4) & 0x0F0F0F0Fu;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float2 cc = make_float2(__uint_as_float(prmt_imm<0x7540u>(ce, kmag, k)),
                                                __uint_as_float(prmt_imm<0x7540u>(co, kmag, k)));
                        cc = __fadd2_rn(cc, m23);
                        const int i = 8 * h + 2 * k;
#if MA_LEAN_MIXADD2
                        float2 a;
                        if constexpr (KT::GDT == BF16)
                            a = add_bf16x2_f32(raw16_word<KT::GDT>(raw, i >> 1), __ffma2_rn(cc, lv2, lo2));
                        else
                            a = __fadd2_rn(make_float2(g32_of<KT::GDT>(raw, i), g32_of<KT::GDT>(raw, i + 1)),
                                           __ffma2_rn(cc, lv2, lo2));
#else
                        const float2 a = __fadd2_rn(make_float2(g32_of<KT::GDT>(raw, i), g32_of<KT::GDT>(raw, i + 1)),
                                                    __ffma2_rn(cc, lv2, lo2));
#endif
                        r[i] = a.x;
                        r[i + 1] = a.y;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if ((sel16 >> i) & 1u) r[i] = 0.0f;
            float mn = r[0], mx = r[0];
#pragma unroll
            for (int i = 1; i < 16; ++i) {
                mn = fminf(mn, r[i]);
                mx = fmaxf(mx, r[i]);
            }
#pragma unroll
            for (int off = 1; off < LP2; off <<= 1) {
                mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, off));
                mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
            }
            const float eps = __fmaf_ru(fmaxf(fabsf(mn), fabsf(mx)), 0x1p-23f, f.z);
            const float R = __fsub_rd(mx, mn);
            const float den = __fsub_rd(R, 2.0f * eps);
            const float k2 = __fdividef(30.0f, R);
            const float cmag = 258.0f + fabsf(mn * k2);
            const float G = __fmaf_ru(128.0f, __fdividef(eps, den), __fmaf_ru(cmag, 0x1p-23f, 0x1p-13f));
            const bool fast = R >= 0x1p-100f && R <= 0x1p100f && den > 0.0f && G <= 0.0625f;  // bucket-uniform
            uint32_t w0 = 0, w1 = 0, bnd = 0;
            bool bad = false;
            double lmin = CUDART_INF, lmax = -CUDART_INF;
            if (fast) {
                const float c2 = __fmaf_rn(-mn, k2, 257.0f + G);
                const uint32_t Gu = static_cast<uint32_t>(__fmaf_ru(2.0f, G, 0x1p-13f) * 32768.0f) + 1u;
                uint32_t yb[16];
                const float2 k22 = make_float2(k2, k2), c22 = make_float2(c2, c2);
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    const float2 y = __ffma2_rn(make_float2(r[i], r[i + 1]), k22, c22);
                    yb[i] = __float_as_uint(y.x);
                    yb[i + 1] = __float_as_uint(y.y);
                }
                w0 = pack_codes8(yb);
                w1 = pack_codes8(yb + 8);
#if MA_LEAN_PFLAG
                // Flags two elements per word: the low halves of y_2k, y_2k+1
                // (15 fraction bits each) + (0x8000 - Gu) set bit 15 / 31 exactly
                // when the fraction is >= Gu (Gu <= 4097: no carry between the
                // halves); the NOT-flagged bits land at 15 - k / 31 - k.
                const uint32_t Cg = (0x8000u - Gu) * 0x10001u;
                uint32_t nf = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    nf |= (((__byte_perm(yb[2 * k], yb[2 * k + 1], 0x5410u) & 0x7FFF7FFFu) + Cg) & 0x80008000u) >> k;
                uint32_t fl = ~nf & 0xFF00FF00u;  // bit b -> element 30 - 2 (b & 15) + (b >> 4)
#else
                uint32_t fl = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) fl |= static_cast<uint32_t>((yb[i] & 0x7FFFu) < Gu) << i;
#endif
                if (fl) {  // min / max candidates and code boundaries (~2 per bucket)
                    // this lane's raw gradients -> its 64-byte scratch slot (dead
                    // candidate / bitmap area) so flagged elements index them
                    uint4* slot = reinterpret_cast<uint4*>(s_scr) + lane * (64 / 16);
#pragma unroll
                    for (int k = 0; k < Raw16<KT::GDT>::N; ++k) slot[k] = raw.v[k];
                    const double2 q = s_ll[e0 / BUCKET];
                    const uint64_t cw64 = (static_cast<uint64_t>(cw.y) << 32) | cw.x;
                    do {  // branch-free body: every flagged element takes the same path
#if MA_LEAN_PFLAG
                        const int fb = __ffs(fl) - 1;
                        const int i = 30 - 2 * (fb & 15) + (fb >> 4);
#else
                        const int i = __ffs(fl) - 1;
#endif
                        fl &= fl - 1;
                        const bool s = (sel16 >> i) & 1u;
                        const uint32_t c = static_cast<uint32_t>(cw64 >> (4 * i)) & 15u;
                        const float g = KT::GDT == BF16
                                            ? __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(slot)[i]) << 16)
                                            : reinterpret_cast<const float*>(slot)[i];
                        const float r32 = s ? 0.0f : __fadd_rn(g, __fmaf_rn(static_cast<float>(c), f.y, f.x));
                        const uint32_t N = (__float_as_uint(__fmaf_rn(r32, k2, c2)) >> 15) & 0xFFu;
                        const double rx = s ? 0.0
                                            : __dadd_rn(static_cast<double>(g),
                                                        __dadd_rn(__dmul_rn(static_cast<double>(c), q.y), q.x));
                        bad |= N == 0u || N > 31u;
                        lmin = (N == 1u && rx < lmin) ? rx : lmin;
                        lmax = (N == 31u && rx > lmax) ? rx : lmax;
                        bnd |= static_cast<uint32_t>((N & 1u) == 0u && N - 1u < 31u) << i;
                    } while (fl);
                }
            }
#if MA_LEAN_BADENC
            // a lane's `bad` travels as lmin = -inf (a fast-path candidate is finite)
            if (bad) lmin = -CUDART_INF;
#pragma unroll
            for (int off = 1; off < LP2; off <<= 1) {  // the bucket's exact extremes (all lanes)
                const double ol = __shfl_xor_sync(0xFFFFFFFFu, lmin, off), oh = __shfl_xor_sync(0xFFFFFFFFu, lmax, off);
                lmin = ol < lmin ? ol : lmin;
                lmax = oh > lmax ? oh : lmax;
            }
            bad = !fast || !(lmin > -CUDART_INF && lmin < CUDART_INF) || !(lmax > -CUDART_INF);  // bucket-uniform
#else
#pragma unroll
            for (int off = 1; off < LP2; off <<= 1) {  // the bucket's exact extremes (all lanes)
                const double ol = __shfl_xor_sync(0xFFFFFFFFu, lmin, off), oh = __shfl_xor_sync(0xFFFFFFFFu, lmax, off);
                lmin = ol < lmin ? ol : lmin;
                lmax = oh > lmax ? oh : lmax;
                bad |= __shfl_xor_sync(0xFFFFFFFFu, bad, off);
            }
            bad = bad || !fast || !(lmin < CUDART_INF) || !(lmax > -CUDART_INF);  // bucket-uniform
#endif
            double lo_n = lmin, hi_n = lmax;
            if (bad) {
                const Bucket16 o = exact_bucket16<KT>(&p, base, e0, sel16, s_ll[e0 / BUCKET], bm, LP2);
                w0 = o.w0;
                w1 = o.w1;
                lo_n = o.lo;
                hi_n = o.hi;
                if (p.dbg) atomicAdd(p.dbg + 1, 16u);
            } else if (bnd) {  // rare: quotients within the guard band of a code boundary
                const double level = div15_w(__dsub_rn(hi_n, lo_n));
                const double2 q = s_ll[e0 / BUCKET];
                while (bnd) {
                    const int i = __ffs(bnd) - 1;
                    bnd &= bnd - 1;
                    const double rx = ((sel16 >> i) & 1u) ? 0.0 : recompute_a_q<KT>(p, base, e0 + i, q);
                    const uint32_t c = exact_code_w(rx, lo_n, level);
                    if (i < 8) w0 = (w0 & ~(15u << (4 * i))) | (c << (4 * i));
                    else w1 = (w1 & ~(15u << (4 * (i - 8)))) | (c << (4 * (i - 8)));
                }
                if (p.dbg) atomicAdd(p.dbg + 1, 1u);
            }
            __stcs(reinterpret_cast<uint2*>(p.codes + ((base + e0) >> 1)), make_uint2(w0, w1));
            if ((lane & (LP2 - 1)) == 0) __stcs(p.meta + (base + e0) / BUCKET, make_double2(lo_n, hi_n));
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_seen[lane * 4 + k] = 0;
        s_dup[lane * 4 + k] = 0;
    }
    __syncwarp();
    }  // PH & 1
    if constexpr (PH == 2) {
        if (lane == 0) {
            if (stage) stage_rows(s_bar, s_widx, gwi, s_wval, gwv, m * kbs * 2, m * kbs * vsz);
            prefetch_l2(static_cast<const unsigned char*>(p.params) + base * psz, kBlk * psz);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            s_seen[lane * 4 + k] = 0;
            s_dup[lane * 4 + k] = 0;
        }
        __syncwarp();
        while (stage && !mbar_try_wait(s_bar, 0)) {
        }
    }
    if constexpr (PH & 2) {

#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 5);
#endif
    // ---- ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    // Entry t = row r (physical slot) * k_b + position pos; each lane walks
    // t = lane, lane + 32, ... with (r, pos) advanced incrementally.
    const int nent = filled * kb;
    // Entry t = lane + 32 i sits at (row r, position pos); 32 entries later it
    // is (r + dq, pos + dr) plus at most one carry (dq = 32 / k_b, dr = 32 % k_b).
    const int r0 = lane / kb, pos0 = lane - r0 * kb;
    const int dq = 32 / kb, dr = 32 - dq * kb;
    auto advance = [&](int& r, int& pos) {
        pos += dr;
        r += dq;
        if (pos >= kb) {
            pos -= kb;
            ++r;
        }
    };
    // the block's ring rows are staged in shared memory (s_widx / s_wval)
    {
        int r = r0, pos = pos0;
#pragma unroll 1
        for (int t = lane; t < nent; t += 64) {
            const int ea = r * kbs + pos;
            advance(r, pos);
            const bool hb = t + 32 < nent;
            const int eb = hb ? r * kbs + pos : ea;
            advance(r, pos);
            const int ia = s_widx[ea];
            const int ib = s_widx[eb];
            uint32_t bit = 1u << (ia & 31);
            if (atomicOr(&s_seen[ia >> 5], bit) & bit) atomicOr(&s_dup[ia >> 5], bit);
            if (hb) {
                bit = 1u << (ib & 31);
                if (atomicOr(&s_seen[ib >> 5], bit) & bit) atomicOr(&s_dup[ib >> 5], bit);
            }
        }
    }
    __syncwarp();
#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 6);
#endif
    int* dupl = reinterpret_cast<int*>(s_cval);
    int ndup = 0;
    {
        // Coordinates held by one entry: θ of a chunk of entries is fetched with
        // one round of cp.async (LDGSTS) into the dead pass-2 tables (ll, llf),
        // then every entry is updated from shared memory.
        void* thb = static_cast<unsigned char*>(p.params) + base * psz;  // this block's θ
        constexpr int tsz = psz < 4 ? 4 : psz;                             // copy granule per entry
        unsigned char* s_th = ws + L.ll;
        const int chunk = static_cast<int>((L.sel - L.ll) / tsz);          // entries per round
        const int dup_max = static_cast<int>((L.cidx - L.cval) / 4);
        int r = r0, pos = pos0;
#pragma unroll 1
        for (int c0 = 0; c0 < nent; c0 += chunk) {
            const int c1 = min(nent, c0 + chunk);
            // round 1: the θ words of this lane's unique entries
            {
                int rr = r, pp = pos;
#pragma unroll 1
                for (int t = c0 + lane; t < c1; t += 32) {
                    const int e = rr * kbs + pp;
                    advance(rr, pp);
                    const int idx = s_widx[e];
                    if (!((s_dup[idx >> 5] >> (idx & 31)) & 1u)) {
                        const unsigned char* src = static_cast<const unsigned char*>(thb) +
                                                   (psz < 4 ? (static_cast<uint32_t>(idx) * psz) & ~3u
                                                            : static_cast<uint32_t>(idx) * psz);
                        cp_async_g2s<tsz>(s_th + (t - c0) * tsz, src);
                    }
                }
                cp_async_wait_all();
            }
            // round 2: updates (and the ordered list of duplicated entries)
#pragma unroll 1
            for (int t0 = c0 + lane; t0 < c1 + lane; t0 += 32) {
                const bool act = t0 < c1;
                const int e = r * kbs + pos;
                const int rr = r, pp = pos;
                advance(r, pos);
                const int idx = act ? s_widx[e] : 0;
                const bool dup = act && ((s_dup[idx >> 5] >> (idx & 31)) & 1u);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, dup);
                if (bal) {
                    const int qd = ndup + __popc(bal & lanemask_lt());
                    if (dup && qd < dup_max) dupl[qd] = dup_pack(idx, rr, pp);
                    ndup += __popc(bal);
                }
                if (act && !dup) unique_update_smem<KT>(p, base, thb, gwv, s_wval, s_th + (t0 - c0) * tsz, e, rr, idx);
            }
        }
    }
    __syncwarp();
    if (p.dbg && lane == 0) {
        atomicAdd(p.dbg + 5, static_cast<unsigned>(ndup));
        if (ndup > static_cast<int>((L.cidx - L.cval) / 4)) atomicAdd(p.dbg + 4, 1u);
    }
#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 7);
#endif
    if (ndup <= 32) {
        // Duplicated coordinates, one list entry per lane (list order = physical
        // slot order): peers of a coordinate found with match.any, the lowest
        // peer sums the terms in lane order (window.cpp:32-39) and updates θ.
        const bool has = lane < ndup;
        const int x = has ? dupl[lane] : 0;
        const int idx = dup_idx(x), r = dup_row(x), pos = dup_pos(x);
        double t1 = 0.0, t2 = 0.0;
        if (has) {
            const double v = ld_t<KT::VDT>(s_wval, r * kbs + pos);
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
        if (has && (__ffs(peers) - 1) == lane) {
            const double mhat = __dmul_rn(z1, p.scale1);
            const double vhat = __dmul_rn(z2, p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            const double th = ld_t<KT::PDT>(p.params, base + idx);
            st_t<KT::PDT>(p.params, base + idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        }
    } else if (!dup_chunks<KT>(&p, ws, b, ndup)) {
        dup_stats<KT, LLayout>(&p, ws, b, ndup, nent);
    }
    }  // PH & 2
#if MA_LEAN_PROF
    if (p.dbg) prof_mark(p, 8);
#endif
}

template <class KT, int PH = 3>
cudaError_t launch_kl(const StepArgs& a, cudaStream_t s) {
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    // per warp: the LLayout area + (PH & 2) the staged window rows (indices, values)
    const size_t rows = ((PH & 2) && lean_stage_rows(a.m, a.kb_stride, vsz))
                            ? align_up(size_t(a.m) * a.kb_stride * 2, 16) + align_up(size_t(a.m) * a.kb_stride * vsz, 16)
                            : 0;
    const size_t smem = size_t(kWarps) * (LLayout(KT::BUCKET, KT::CAPL).total + rows);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto k = microadam_step_lean<KT, PH>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    const int64_t grid = (a.block_count + kWarps - 1) / kWarps;
    k<<<static_cast<unsigned>(grid), 32 * kWarps, smem, s>>>(a);
    return cudaGetLastError();
}

#ifdef MA_PROBE_HOT
#define MA_LEAN_DTYPES(X) X(BF16, BF16, BF16)
#else
#define MA_LEAN_DTYPES(X) \
    X(BF16, BF16, BF16)   \
    X(F32, F32, BF16)     \
    X(F32, F32, F32)      \
    X(BF16, F32, BF16)    \
    X(BF16, BF16, F32)
#endif

// Candidate slots per lane: k_b <= 64: 4; up to 128 (densities to 3.1%): 8
// (half the shared memory of 16: 8 CTAs per SM instead of 6); up to 256
// (densities to 6.25%): 16.
constexpr int kWideKb = 32 * 16 / 2;
__host__ __device__ constexpr int lean_capl(int kb) { return kb <= 32 * 4 / 2 ? kLCapL : (kb <= 32 * 8 / 2 ? 8 : 16); }

template <int LPB>
cudaError_t launch_ldt(const StepArgs& a, cudaStream_t s) {
    const int capl = lean_capl(static_cast<int>(a.per_block_k));
    switch (dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_)                                                              \
        case dtype_key_w(G_, P_, V_):                                                    \
            return capl == 16  ? launch_kl<KW<LPB, G_, P_, V_, false, 16>>(a, s)         \
                   : capl == 8 ? launch_kl<KW<LPB, G_, P_, V_, false, 8>>(a, s)          \
                               : launch_kl<KW<LPB, G_, P_, V_, false>>(a, s);
        MA_LEAN_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

// Shared memory of the fused lean kernel: per warp the LLayout area plus the
// block's staged window rows (indices + values).
size_t lean_smem_bytes(const StepArgs& a) {
    const int capl = lean_capl(static_cast<int>(a.per_block_k));
    const size_t vsz = a.v_dtype == F64 ? 8 : (a.v_dtype == F32 ? 4 : 2);
    const size_t rows = lean_stage_rows(a.m, a.kb_stride, int(vsz))
                            ? align_up(size_t(a.m) * a.kb_stride * 2, 16) + align_up(size_t(a.m) * a.kb_stride * vsz, 16)
                            : 0;
    return size_t(kWarps) * (LLayout(a.bucket, capl).total + rows);
}

bool lean_ok(const StepArgs& a) {
    if (a.partials || a.force_exact || (a.bucket != 32 && a.bucket != 64)) return false;
    if (a.per_block_k > kWideKb) return false;
    if (lean_smem_bytes(a) > 227 * 1024) return false;  // huge windows: the exact warp kernel
    switch (dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_) case dtype_key_w(G_, P_, V_): return true;
        MA_LEAN_DTYPES(MA_CASE)
#undef MA_CASE
        default: return false;
    }
}


template <int LPB, bool REP>
cudaError_t launch_wdt(const StepArgs& a, cudaStream_t s) {
    switch (dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_) \
        case dtype_key_w(G_, P_, V_): return launch_kw<KW<LPB, G_, P_, V_, REP>>(a, s);
        MA_WARP_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

template <bool REP>
cudaError_t launch_wrep(const StepArgs& a, cudaStream_t s) {
    switch (a.bucket) {
        case 16: return launch_wdt<2, REP>(a, s);
        case 32: return launch_wdt<4, REP>(a, s);
        case 64: return launch_wdt<8, REP>(a, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace

// Warp path: B_d = 4096, k_b <= 64 (candidates fit kCap), B_q in {16, 32, 64},
// an instantiated dtype combo; window rows addressable with 16-bit offsets.
bool warp_path_ok(int block, int bucket, int kb, int m, int kb_stride, int g, int p, int v) {
    if (block != kBlk || kb < 1 || kb > kWideKb) return false;  // k_b > 64: lean kernel only
    if (bucket != 16 && bucket != 32 && bucket != 64) return false;
    if (m < 1 || m > kMaxWindow || m * kb_stride > 32768) return false;
    switch (dtype_key_w(g, p, v)) {
#define MA_CASE(G_, P_, V_) case dtype_key_w(G_, P_, V_): return true;
        MA_WARP_DTYPES(MA_CASE)
#undef MA_CASE
        default: return false;
    }
}

size_t warp_smem_bytes(int bucket) { return size_t(kWarps) * WLayout(bucket).total; }

// Sparse-propagation phases of the lean kernel (B_q = 64): ph = 1 front, 2 stats.
bool lean_phase_ok(const StepArgs& a) { return lean_ok(a) && a.bucket == 64 && a.per_block_k <= kCap / 2; }

cudaError_t launch_step_lean_phase(const StepArgs& a, int ph, cudaStream_t s) {
    if (a.block_count <= 0) return cudaSuccess;
    if (!lean_phase_ok(a)) return cudaErrorInvalidConfiguration;
    switch (dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_)                                                        \
        case dtype_key_w(G_, P_, V_):                                              \
            return ph == 1 ? launch_kl<KW<8, G_, P_, V_, false>, 1>(a, s)          \
                           : launch_kl<KW<8, G_, P_, V_, false>, 2>(a, s);
        MA_LEAN_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

// Fused reduce-scatter variant (ma_step_reduce): B_q = 64, k_b <= 64, the two
// uniform dtype combos; everything else reduces with launch_reduce_grads first.
bool lean_rs_ok(const StepArgs& a) {
    if (!lean_ok(a) || a.bucket != 64 || a.per_block_k > kCap / 2) return false;
    if (a.rs_n < 1 || a.rs_n > kMaxRanks) return false;
    const int key = dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype);
    return key == dtype_key_w(BF16, BF16, BF16) || key == dtype_key_w(F32, F32, F32);
}

cudaError_t launch_lean_rs(const StepArgs& a, cudaStream_t s) {
    if (!lean_rs_ok(a)) return cudaErrorInvalidConfiguration;
    if (dtype_key_w(a.g_dtype, a.p_dtype, a.v_dtype) == dtype_key_w(BF16, BF16, BF16))
        return launch_kl<KW<8, BF16, BF16, BF16, false, 4, true>>(a, s);
    return launch_kl<KW<8, F32, F32, F32, false, 4, true>>(a, s);
}

bool warp_can_run(const StepArgs& a) { return lean_ok(a) || a.per_block_k <= kCap / 2; }

cudaError_t launch_step_warp(const StepArgs& a, cudaStream_t s) {
    if (a.block_count <= 0) return cudaSuccess;
    if (!warp_can_run(a)) return cudaErrorInvalidConfiguration;
    if ((a.block_count + kWarps - 1) / kWarps > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    if (a.rs_n > 0) return launch_lean_rs(a, s);
    if (lean_ok(a)) return a.bucket == 64 ? launch_ldt<8>(a, s) : launch_ldt<4>(a, s);
    return a.partials ? launch_wrep<true>(a, s) : launch_wrep<false>(a, s);
}

}  // namespace ma
