// ma_fast.cu — the fast sm_100a MicroAdam step kernel (default layouts).
//
// Same contract and bit-exact results as the generic kernel (ma_kernels.cu),
// shaped for the HBM roofline: one 128-thread CTA per FULL 4096-element Top-K
// block, 4 CTAs resident per SM (128 registers/thread, ~54 KB smem each). The
// one partial tail block of a shard, if any, goes to the generic kernel.
//
//  * A thread owns 32 CONTIGUOUS elements (half a 64-bucket): g arrives as
//    16 B vector loads, the 32 EF codes as one 16 B load and leave as one 16 B
//    store, and the accumulator a (fp64) stays in 32 register pairs from the
//    decode (P1) to the re-quantization (P3) — a is computed once. A copy in
//    smem (interleaved, conflict-free) serves the dynamic-index consumers
//    (candidate gather, the exact fallback, the guard-band path).
//  * θ and the block's m window rows are staged HBM→smem at CTA start with 1-D
//    bulk async copies on an mbarrier (SASS UBLKCP); θ returns with one bulk
//    store.
//  * Block Top-K: a threshold t on 16-bit keys (bits 62..48 of |a|) with
//    k_b <= #{key16 >= t} <= cap is carried per block from the previous step
//    (or found by bisection on block-wide counts). The candidates above t are
//    selected exactly by (|a| desc, index asc): warp bisection on the 32-bit
//    high word, full key then lower index on ties (compress.cpp:39-53). Only
//    when more than `cap` keys tie at 16-bit resolution does an out-of-line
//    exact radix select run. Window positions come from a word prefix of the
//    selection bitmap (one bitmap word == one thread's 32 elements).
//  * Bucket min/max (quantize.cpp:15-24): in-register compare-exchange tree
//    over the thread's elements, one partner shuffle for B_q = 64.
//  * Quantization: q ≈ (x−lo)·15/(hi−lo) in fp32 from the exact fp64
//    difference, in 2^-20 fixed point; floor(q+1/2) is taken from it unless
//    q+1/2 lies within 64·2^-20 of an integer (error bound ≈ 4·2^-20), in which
//    case the IEEE quotient (x−lo)/level of quantize.cpp:51 decides.
//  * ADAM_STATS with no per-row barrier: every window coordinate gets one
//    owner row (last-writer-wins byte + duplicate bit); unique coordinates take
//    z = 0 + w·v, duplicated ones are re-summed by the owner in physical slot
//    order (binary search in the ascending rows) — window.cpp:32-39's order.
#include <cstdlib>

#include "../../include/ma_synth.h"
#include "ma_async.cuh"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kNT = 128;             // threads per CTA
constexpr int kEPT = 32;             // contiguous elements per thread
constexpr int kBlock = kNT * kEPT;   // 4096
constexpr uint32_t kGuard = 64;      // fixed-point guard band (units of 2^-20)
constexpr int kMaxRowsFast = 127;    // owner byte: row (7 bits) + duplicate bit

// Candidate capacity of the exact-select stage: 2 k_b, at least 128, at most 512.
__host__ __device__ inline int cand_cap(int kb) {
    const int c = ((2 * kb + 3) / 4) * 4;
    return c < 128 ? 128 : (c > 512 ? 512 : c);
}

// Shared-memory carve-up (host and device agree).
struct Layout5 {
    uint32_t theta, widx, wval, a, cval, ckey, red, bar, owner, ckhi, cidx, sel, tmpb, wpref, hist,
        misc, total;
    __host__ __device__ Layout5() {}
    __host__ __device__ Layout5(int m, int kbs, int pdt, int vdt, int cap) {
        const size_t ent = size_t(m) * size_t(kbs);
        size_t o = 0;
        theta = uint32_t(o); o = align_up(o + size_t(kBlock) * dtype_bytes(pdt), 128);
        widx = uint32_t(o);  o = align_up(o + ent * 2, 128);
        wval = uint32_t(o);  o = align_up(o + ent * dtype_bytes(vdt), 128);
        a = uint32_t(o);     o = align_up(o + size_t(kBlock) * 8, 16);
        cval = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 8, 16);
        ckey = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 8, 16);
        red = uint32_t(o);   o = align_up(o + size_t(kNT / 32) * kReportFields * 8, 16);
        bar = uint32_t(o);   o = align_up(o + 16, 16);
        owner = uint32_t(o); o = align_up(o + size_t(kBlock), 16);
        ckhi = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 4, 16);
        cidx = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 4, 16);
        sel = uint32_t(o);   o = align_up(o + size_t(kBlock / 32) * 4, 16);
        tmpb = uint32_t(o);  o = align_up(o + size_t(kBlock / 32) * 4, 16);
        wpref = uint32_t(o); o = align_up(o + size_t(kBlock / 32 + 1) * 4, 16);
        hist = uint32_t(o);  o = align_up(o + 256 * 4, 16);
        misc = uint32_t(o);  o = align_up(o + 96 * 4, 16);
        total = uint32_t(align_up(o, 128));
    }
};

// Compile-time shape of one fast-kernel instantiation.
template <int BQ_, int GDT_, int PDT_, int VDT_, bool REP_>
struct K {
    static constexpr int BQ = BQ_, GDT = GDT_, PDT = PDT_, VDT = VDT_;
    static constexpr bool REPORT = REP_;
    static constexpr int NBK = kEPT / BQ_ > 0 ? kEPT / BQ_ : 1;  // buckets per thread (1 or 2)
};

struct Ctx {
    const StepArgs* p;
    unsigned char* smem;
    Layout5 L;
    int64_t b, base;
    int kb, m, kbs, slot;
};

template <class KT>
__device__ __forceinline__ Ctx make_ctx(const StepArgs& p) {
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    Ctx c;
    c.p = &p;
    c.smem = smem_dyn;
    c.m = p.m;
    c.kbs = p.kb_stride;
    c.kb = p.per_block_k;
    c.slot = p.slot;
    c.L = Layout5(p.m, p.kb_stride, KT::PDT, KT::VDT, cand_cap(p.per_block_k));
    c.b = p.block_offset + blockIdx.x;
    c.base = c.b * kBlock;
    return c;
}

// a of element e from the interleaved smem copy: thread t = e/32, slot i = e%32
// lives at double index ((i/2)*kNT + t)*2 + (i&1) (16 B per thread per pair:
// the P1 stores are bank-conflict free).
__device__ __forceinline__ double smem_a(const unsigned char* smem, const Layout5& L, int e) {
    const int t = e >> 5, i = e & 31;
    return reinterpret_cast<const double*>(smem + L.a)[((i >> 1) * kNT + t) * 2 + (i & 1)];
}

// 32 consecutive g values starting at element e0 (32-aligned) as doubles.
template <int DT>
__device__ __forceinline__ void load_g32(const void* g, int64_t e0, double (&x)[kEPT]) {
    if constexpr (DT == BF16) {
        const uint4* q = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + e0);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint4 u = __ldg(q + v);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                x[8 * v + 2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
                x[8 * v + 2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
            }
        }
    } else if constexpr (DT == F32) {
        const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(g) + e0);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const float4 u = __ldg(q + v);
            x[4 * v] = u.x; x[4 * v + 1] = u.y; x[4 * v + 2] = u.z; x[4 * v + 3] = u.w;
        }
    } else {
        const double2* q = reinterpret_cast<const double2*>(static_cast<const double*>(g) + e0);
#pragma unroll
        for (int v = 0; v < 16; ++v) {
            const double2 u = __ldg(q + v);
            x[2 * v] = u.x;
            x[2 * v + 1] = u.y;
        }
    }
}

__device__ __forceinline__ uint32_t key16(double x) { return hi_key(x) >> 16; }

// Rank correction among candidates whose high words tie (compress.cpp:43-48:
// full |a| key first, then the lower index). Out of line: rare.
__device__ __noinline__ int tie_rank_hi(const double* cval, const uint32_t* ckhi, const int* cidx,
                                        int ncand, int t) {
    const uint32_t kh = ckhi[t];
    const uint64_t kt = key_of(cval[t]);
    const int it = cidx[t];
    int extra = 0;
    for (int q = 0; q < ncand; ++q) {
        if (q == t || ckhi[q] != kh) continue;
        const uint64_t kq = key_of(cval[q]);
        extra += (kq > kt) || (kq == kt && cidx[q] < it);
    }
    return extra;
}

// The IEEE path of quantize_nearest (quantize.cpp:51-53) for one element.
__device__ __noinline__ uint32_t exact_code(double x, double lo, double level) {
    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(x, lo), level), 0.5));
    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
    return static_cast<uint32_t>(f);
}

// t / kb for t < 2^16 without an integer division (float reciprocal + fix-up).
__device__ __forceinline__ int row_of(int t, int kb, float inv_kb) {
    int r = __float2int_rz(static_cast<float>(t) * inv_kb);
    r -= (r * kb > t);
    r += ((r + 1) * kb <= t);
    return r;
}

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

__device__ __forceinline__ void wait_stage(uint64_t* bar) {
    while (!mbar_try_wait(bar, 0)) {
    }
}

// Selected element e (value a) -> window row `slot` at its ascending position
// (window.cpp:14-26): global ring, the staged rows, and its owner mark.
template <class KT>
__device__ __forceinline__ void emit_selected(const Ctx& c, int e, double a) {
    const StepArgs& p = *c.p;
    const uint32_t* s_sel = reinterpret_cast<const uint32_t*>(c.smem + c.L.sel);
    const int* s_wpref = reinterpret_cast<const int*>(c.smem + c.L.wpref);
    const int pos = s_wpref[e >> 5] + __popc(s_sel[e >> 5] & ((1u << (e & 31)) - 1u));
    const int64_t g = (c.b * c.m + c.slot) * static_cast<int64_t>(c.kbs) + pos;
    p.win_idx[g] = static_cast<int16_t>(e);
    st_t<KT::VDT>(p.win_val, g, a);
    const int ent = c.slot * c.kbs + pos;
    reinterpret_cast<int16_t*>(c.smem + c.L.widx)[ent] = static_cast<int16_t>(e);
    st_t<KT::VDT>(c.smem + c.L.wval, ent, a);
    (c.smem + c.L.owner)[e] = static_cast<uint8_t>(c.slot);
}

// Exact fallback selection (compress.cpp:39-53) for blocks where more than
// `cap` keys tie at 16-bit resolution: the generic radix select (ma_device.cuh)
// over the smem copy of a. Sets the selection bitmap + prefix, emits the new
// row and misc[1] = next threshold.
template <class KT>
__device__ __noinline__ void fallback_select(const StepArgs* pp) {
    const Ctx c = make_ctx<KT>(*pp);
    unsigned char* sm = c.smem;
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(sm + c.L.sel);
    uint32_t* s_tmpb = reinterpret_cast<uint32_t*>(sm + c.L.tmpb);
    int* s_wpref = reinterpret_cast<int*>(sm + c.L.wpref);
    int* s_misc = reinterpret_cast<int*>(sm + c.L.misc);
    uint8_t* selm = sm + c.L.owner;  // scratch; owner marks are written afterwards
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nwords = kBlock / 32;
    for (int i = tid; i < kBlock; i += kNT) selm[i] = 0;
    for (int w = tid; w < nwords; w += kNT) s_tmpb[w] = 0;
    auto elem = [&](int s) { return s * kNT + tid; };
    double a[kEPT];
#pragma unroll
    for (int s = 0; s < kEPT; ++s) a[s] = smem_a(sm, c.L, elem(s));
    __syncthreads();
    auto tie_rank = [&](uint32_t mask, int (&r)[kEPT]) {
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kEPT; ++s)
            if ((mask >> s) & 1u) atomicOr(&s_tmpb[elem(s) >> 5], 1u << (elem(s) & 31));
        __syncthreads();
        if (warp == 0) word_prefix(s_tmpb, nwords, s_wpref);
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kEPT; ++s)
            if ((mask >> s) & 1u) {
                const int e = elem(s);
                r[s] = s_wpref[e >> 5] + __popc(s_tmpb[e >> 5] & ((1u << (e & 31)) - 1u));
            }
    };
    const uint32_t sel = block_topk<kNT, kEPT>(
        a, 0xFFFFFFFFu, c.kb, reinterpret_cast<uint32_t*>(sm + c.L.hist), s_misc + 32,
        reinterpret_cast<uint64_t*>(sm + c.L.ckey), reinterpret_cast<int*>(sm + c.L.cidx), selm,
        elem, tie_rank);
    uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
    for (int s = 0; s < kEPT; ++s)
        if ((sel >> s) & 1u) {
            atomicOr(&s_sel[elem(s) >> 5], 1u << (elem(s) & 31));
            kmin = min(kmin, hi_key(a[s]));
        }
    kmin = __reduce_min_sync(0xFFFFFFFFu, kmin);
    if (lane == 0) atomicMin(reinterpret_cast<unsigned int*>(&s_misc[2]), kmin);
    __syncthreads();
    if (warp == 0) word_prefix(s_sel, nwords, s_wpref);
    __syncthreads();
    wait_stage(reinterpret_cast<uint64_t*>(sm + c.L.bar));
#pragma unroll
    for (int s = 0; s < kEPT; ++s)
        if ((sel >> s) & 1u) emit_selected<KT>(c, elem(s), a[s]);
    if (tid == 0) {
        const uint32_t km = static_cast<uint32_t>(s_misc[2]) >> 16;
        s_misc[1] = static_cast<int>(km > 1 ? km - 1 : 1u);
    }
}

// min and max of n consecutive register values a[o..o+n) (n a power of two):
// one compare-exchange per pair, then two trees. No NaN / -0.0 can occur.
template <int N>
__device__ __forceinline__ void minmax_tree(const double (&a)[kEPT], int o, double& lo, double& hi) {
    double l[N / 2], h[N / 2];
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
        const bool lt = a[o + 2 * k] < a[o + 2 * k + 1];
        l[k] = lt ? a[o + 2 * k] : a[o + 2 * k + 1];
        h[k] = lt ? a[o + 2 * k + 1] : a[o + 2 * k];
    }
#pragma unroll
    for (int w = N / 4; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) {
            l[k] = l[k + w] < l[k] ? l[k + w] : l[k];
            h[k] = h[k + w] > h[k] ? h[k + w] : h[k];
        }
    lo = l[0];
    hi = h[0];
}

template <class KT>
__global__ void __launch_bounds__(kNT, 4) microadam_step_fast(const __grid_constant__ StepArgs p) {
    constexpr int NW = kNT / 32;
    constexpr int BQ = KT::BQ, NBK = KT::NBK, EPB = kEPT / NBK;  // elements per (thread, bucket)
    constexpr bool want_report = KT::REPORT;
    constexpr int psz = KT::PDT == F64 ? 8 : (KT::PDT == F32 ? 4 : 2);
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    extern __shared__ __align__(128) unsigned char smem[];
    const Ctx c = make_ctx<KT>(p);
    const Layout5& L = c.L;
    unsigned char* sth = smem + L.theta;
    int16_t* swi = reinterpret_cast<int16_t*>(smem + L.widx);
    unsigned char* swv = smem + L.wval;
    double2* s_a2 = reinterpret_cast<double2*>(smem + L.a);
    double* s_cval = reinterpret_cast<double*>(smem + L.cval);
    double* s_red = reinterpret_cast<double*>(smem + L.red);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    uint8_t* s_owner = smem + L.owner;
    uint32_t* s_ckhi = reinterpret_cast<uint32_t*>(smem + L.ckhi);
    int* s_cidx = reinterpret_cast<int*>(smem + L.cidx);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + L.sel);
    int* s_wpref = reinterpret_cast<int*>(smem + L.wpref);
    int* s_misc = reinterpret_cast<int*>(smem + L.misc);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kb = c.kb, kbs = c.kbs, slot = c.slot, filled = p.filled, m = c.m;
    const int nent = filled * kb;
    const int cap = cand_cap(kb);
    const float inv_kb = 1.0f / static_cast<float>(kb);
    const int64_t b = c.b, base = c.base;
    const int e0 = tid * kEPT;  // my 32 contiguous elements

    // ---- prologue: θ + window rows HBM→smem (bulk async) ----
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        const uint32_t bt = uint32_t(kBlock * psz), bi = uint32_t(m * kbs * 2),
                       bv = uint32_t(m * kbs * vsz);
        mbar_expect_tx(s_bar, bt + bi + bv);
        const int64_t went = b * m * static_cast<int64_t>(kbs);
        bulk_g2s(sth, static_cast<const unsigned char*>(p.params) + base * psz, bt, s_bar);
        bulk_g2s(swi, p.win_idx + went, bi, s_bar);
        bulk_g2s(swv, static_cast<const unsigned char*>(p.win_val) + went * vsz, bv, s_bar);
        s_misc[NW] = 0;  // candidate counter
        s_misc[2] = -1;  // fallback kmin seed
    }
    s_sel[tid] = 0;  // one bitmap word per thread (kBlock / 32 == kNT)
    const uint32_t carried = __ldg(p.thresh + b);

    // ---- P1: a = g + decode(EF) (quantize.cpp:164-178, optim.cpp:166-168) ----
    double a[kEPT];
    load_g32<KT::GDT>(p.grads, base + e0, a);
    const uint4 cw4 = __ldg(reinterpret_cast<const uint4*>(p.codes + ((base + e0) >> 1)));
    const uint32_t cw[4] = {cw4.x, cw4.y, cw4.z, cw4.w};
    double blo[NBK], blvl[NBK];
#pragma unroll
    for (int k = 0; k < NBK; ++k) {  // QuantParams ctor (quantize.cpp:7-13)
        const double2 mt = __ldg(p.meta + (base + e0 + k * EPB) / BQ);
        blo[k] = mt.x;
        blvl[k] = (mt.x == mt.y) ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), 15.0);
    }
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    uint32_t kmax = 0, cm = 0;
#pragma unroll
    for (int i = 0; i < kEPT; ++i) {
        const int k = i / EPB;
        const double ev = __dadd_rn(
            __dmul_rn(static_cast<double>((cw[i >> 3] >> (4 * (i & 7))) & 15u), blvl[k]), blo[k]);
        if (want_report) rep[0] += a[i] * a[i];
        a[i] = __dadd_rn(a[i], ev);
        if (want_report) rep[1] += a[i] * a[i];
        const uint32_t kh = key16(a[i]);
        kmax = max(kmax, kh);
        cm |= static_cast<uint32_t>(kh >= carried) << i;
    }
#pragma unroll
    for (int j = 0; j < kEPT / 2; ++j) s_a2[j * kNT + tid] = make_double2(a[2 * j], a[2 * j + 1]);
    if (p.check_finite && kmax >= 0x7FF0u) atomicOr(p.flag, 1u);  // inf/NaN in g or a

    // ---- P2: block Top-K (compress.cpp:39-53, 73-85) ----
    int* s_cnt = s_misc + 64;  // [2][NW] per-warp counts, double-buffered
    auto publish = [&](int n, int par) -> int {
        n = __reduce_add_sync(0xFFFFFFFFu, n);
        if (lane == 0) s_cnt[par * NW + warp] = n;
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) tot += s_cnt[par * NW + w];
        return tot;
    };
    auto mask_ge = [&](uint32_t t) {
        uint32_t mk = 0;
#pragma unroll
        for (int i = 0; i < kEPT; ++i) mk |= static_cast<uint32_t>(key16(a[i]) >= t) << i;
        return mk;
    };
    const uint32_t wmax = __reduce_max_sync(0xFFFFFFFFu, kmax);
    if (lane == 0) s_misc[48 + warp] = static_cast<int>(wmax);
    int par = 0;
    const int cnt0 = publish(__popc(cm), par);  // [A0]: counts, warp maxima, smem a
    uint32_t bmax = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) bmax = max(bmax, static_cast<uint32_t>(s_misc[48 + w]));
    uint32_t t16 = carried;
    bool found = carried != 0 && cnt0 >= kb && cnt0 <= cap;
    if (!found) {
        uint32_t lo = 0, hi = bmax + 1, mid;  // invariant: count(lo) >= kb > count(hi)
        if (carried == 0) {
            mid = bmax >= 8 ? bmax - 8 : bmax / 2;  // ~half a binade below the block max
        } else if (cnt0 > cap) {
            lo = carried;
            mid = (lo + hi) / 2;
        } else {
            hi = carried;
            mid = carried > 8 ? carried - 8 : carried / 2;
        }
        while (hi - lo > 1) {
            if (mid <= lo || mid >= hi) mid = (lo + hi) / 2;
            par ^= 1;
            const int n = publish(__popc(mask_ge(mid)), par);
            if (p.dbg && tid == 0) atomicAdd(p.dbg + 2, 1u);
            if (n > cap) {
                lo = mid;
            } else if (n < kb) {
                hi = mid;
            } else {
                found = true;
                t16 = mid;
                break;
            }
            mid = (lo + hi) / 2;
        }
        if (found) cm = mask_ge(t16);
    }
    if (found) {
        // Gather the candidates (warp-aggregated slots, values from the smem copy).
        const int n = __popc(cm);
        int incl = n;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += t;
        }
        int slot0 = 0;
        if (lane == 31 && incl) slot0 = atomicAdd(&s_misc[NW], incl);
        int sidx = __shfl_sync(0xFFFFFFFFu, slot0, 31) + incl - n;
        uint32_t mk = cm;
        while (mk) {
            const int i = __ffs(mk) - 1;
            mk &= mk - 1;
            const double av = reinterpret_cast<const double*>(s_a2)[((i >> 1) * kNT + tid) * 2 + (i & 1)];
            s_cval[sidx] = av;
            s_ckhi[sidx] = hi_key(av);
            s_cidx[sidx] = e0 + i;
            ++sidx;
        }
        __syncthreads();  // [A] candidates
        const int ncand = s_misc[NW];
        if (warp == 0) {
            // Exact Top-k_b among the candidates: bisect the k_b-th largest high
            // word with warp-wide counts; ties resolve on the full |a| key, then
            // the lower index.
            auto count_ge = [&](uint32_t v) {
                int cnt = 0;
                for (int q = lane; q < ncand; q += 32) cnt += s_ckhi[q] >= v;
                return __reduce_add_sync(0xFFFFFFFFu, cnt);
            };
            uint32_t lo = t16 << 16, hi = (bmax + 1) << 16;  // count(lo) >= kb > count(hi)
            while (hi - lo > 1) {
                const uint32_t mid = lo + (hi - lo) / 2;
                if (count_ge(mid) >= kb) lo = mid; else hi = mid;
            }
            const int above = count_ge(lo + 1);
            const int need = kb - above, eqc = count_ge(lo) - above;
            for (int q = lane; q < ncand; q += 32) {
                const uint32_t kh = s_ckhi[q];
                bool sel = kh > lo;
                if (kh == lo) sel = eqc == need || tie_rank_hi(s_cval, s_ckhi, s_cidx, ncand, q) < need;
                if (sel) atomicOr(&s_sel[s_cidx[q] >> 5], 1u << (s_cidx[q] & 31));
            }
            if (lane == 0) {
                const uint32_t h = lo >> 16;  // next step: one 16-bit bucket below the k_b-th key
                s_misc[1] = static_cast<int>(h > 1 ? h - 1 : 1u);
            }
        }
        __syncthreads();  // [B] selection bitmap
        if (warp == 0) word_prefix(s_sel, kBlock / 32, s_wpref);
        __syncthreads();  // [C] positions
        wait_stage(s_bar);
        for (int t = tid; t < ncand; t += kNT) {
            const int e = s_cidx[t];
            if ((s_sel[e >> 5] >> (e & 31)) & 1u) emit_selected<KT>(c, e, s_cval[t]);
        }
    } else {
        fallback_select<KT>(&p);  // more than `cap` keys tie at 16-bit resolution
        if (p.dbg && tid == 0) atomicAdd(p.dbg + 0, 1u);
    }
    if (tid == 0) p.thresh[b] = static_cast<uint32_t>(s_misc[1]);

    // ---- pass A (older rows): owner row per coordinate ----
    wait_stage(s_bar);
    for (int t = tid; t < nent; t += kNT) {
        const int r = row_of(t, kb, inv_kb);
        if (r == slot) continue;
        s_owner[swi[r * kbs + (t - r * kb)]] = static_cast<uint8_t>(r);
    }

    // ---- P3/P4: residual (compress.cpp:95-102) + 4-bit re-quantization
    //      (quantize.cpp:15-24, 42-55, 102-114, 142-162) ----
    {
        const uint32_t sel32 = s_sel[tid];  // my 32 elements
#pragma unroll
        for (int i = 0; i < kEPT; ++i)
            if ((sel32 >> i) & 1u) a[i] = 0.0;
        if (want_report) {
#pragma unroll
            for (int i = 0; i < kEPT; ++i) rep[2] += a[i] * a[i];
        }
        uint32_t word[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < NBK; ++k) {
            double lo, hi;
            minmax_tree<EPB>(a, k * EPB, lo, hi);
            if constexpr (BQ > kEPT) {  // B_q = 64: the partner lane holds the other half
                const double ol = __shfl_xor_sync(0xFFFFFFFFu, lo, 1);
                const double oh = __shfl_xor_sync(0xFFFFFFFFu, hi, 1);
                lo = ol < lo ? ol : lo;
                hi = oh > hi ? oh : hi;
            }
            const double rng = __dsub_rn(hi, lo);
            if (rng != 0.0) {
                const float r32 = __double2float_rn(rng);
                const bool fastq = r32 >= 0x1p-100f && r32 <= 0x1p100f;
                const float kk = fastq ? __fdiv_rn(15.0f * 1048576.0f, r32) : 0.0f;  // 15/rng in 2^-20
                uint32_t gmin = fastq ? 0xFFFFFu : 0u;
#pragma unroll
                for (int j = 0; j < EPB; ++j) {
                    const int i = k * EPB + j;
                    const float d32 = __double2float_rn(__dsub_rn(a[i], lo));
                    const uint32_t xq = __float2uint_rz(__fmaf_rn(d32, kk, 524288.0f));  // (q+1/2)*2^20
                    word[i >> 3] |= (xq >> 20) << (4 * (i & 7));
                    gmin = min(gmin, (xq + kGuard) & 0xFFFFFu);
                }
                if (gmin < 2 * kGuard) {  // rare: some element in the guard band -> IEEE quotient
                    const double level = __ddiv_rn(rng, 15.0);
#pragma unroll
                    for (int w = k * EPB / 8; w < (k + 1) * EPB / 8; ++w) {
#pragma unroll 1
                        for (int j = 0; j < 8; ++j) {
                            const int i = 8 * w + j;
                            const double x = ((sel32 >> i) & 1u)
                                                 ? 0.0
                                                 : reinterpret_cast<const double*>(s_a2)[((i >> 1) * kNT + tid) * 2 + (i & 1)];
                            const float d32 = __double2float_rn(__dsub_rn(x, lo));
                            const uint32_t xq = __float2uint_rz(__fmaf_rn(d32, kk, 524288.0f));
                            if (fastq && ((xq + kGuard) & 0xFFFFFu) >= 2 * kGuard) continue;
                            const uint32_t code = exact_code(x, lo, level);
                            word[w] = (word[w] & ~(15u << (4 * j))) | (code << (4 * j));
                            if (p.dbg) atomicAdd(p.dbg + 1, 1u);
                        }
                    }
                }
            }
            if (want_report) {
                const double level = rng == 0.0 ? 0.0 : __ddiv_rn(rng, 15.0);
#pragma unroll
                for (int j = 0; j < EPB; ++j) {
                    const int i = k * EPB + j;
                    const double en = __dadd_rn(
                        __dmul_rn(static_cast<double>((word[i >> 3] >> (4 * (i & 7))) & 15u), level), lo);
                    rep[3] += en * en;
                }
            }
            if (BQ <= kEPT || (lane & 1) == 0)
                p.meta[(base + e0 + k * EPB) / BQ] = make_double2(lo, hi);
        }
        *reinterpret_cast<uint4*>(p.codes + ((base + e0) >> 1)) = make_uint4(word[0], word[1], word[2], word[3]);
    }
    __syncthreads();  // [D] all owner rows written (older rows + new row)

    // ---- P6 pass B: duplicate bit (coordinate present in more than one row) ----
    for (int t = tid; t < nent; t += kNT) {
        const int r = row_of(t, kb, inv_kb);
        const int idx = swi[r * kbs + (t - r * kb)];
        if ((s_owner[idx] & 0x7F) != r) s_owner[idx] |= 0x80;
    }
    __syncthreads();  // [E]

    // ---- P6 pass C: ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    for (int t = tid; t < nent; t += kNT) {
        const int r = row_of(t, kb, inv_kb);
        const int e = r * kbs + (t - r * kb);
        const int idx = swi[e];
        const uint32_t own = s_owner[idx];
        if ((own & 0x7F) != static_cast<uint32_t>(r)) continue;
        double z1, z2;
        if (!(own & 0x80)) {
            const double v = ld_t<KT::VDT>(swv, e);
            z1 = __dadd_rn(0.0, __dmul_rn(p.w1[r], v));
            z2 = __dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(v, v)));
        } else {
            z1 = 0.0;
            z2 = 0.0;
            for (int rr = 0; rr < filled; ++rr) {
                const int16_t* row = swi + rr * kbs;
                int lo_i = 0, hi_i = kb;
                while (lo_i < hi_i) {
                    const int mid = (lo_i + hi_i) >> 1;
                    if (row[mid] < idx) lo_i = mid + 1; else hi_i = mid;
                }
                if (lo_i < kb && row[lo_i] == idx) {
                    const double v = ld_t<KT::VDT>(swv, rr * kbs + lo_i);
                    z1 = __dadd_rn(z1, __dmul_rn(p.w1[rr], v));
                    z2 = __dadd_rn(z2, __dmul_rn(p.w2[rr], __dmul_rn(v, v)));
                }
            }
        }
        const double mhat = __dmul_rn(z1, p.scale1);
        const double vhat = __dmul_rn(z2, p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        const double th = ld_t<KT::PDT>(sth, idx);
        st_t<KT::PDT>(sth, idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        if (want_report && u != 0.0) rep[4] += 1.0;
    }
    fence_proxy_async_smem();
    __syncthreads();  // [F] θ tile final
    if (tid == 0) {
        bulk_s2g(static_cast<unsigned char*>(p.params) + base * psz, sth,
                 static_cast<uint32_t>(kBlock * psz));
        bulk_wait_read();
    }
    if constexpr (want_report) {
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

template <class KT>
cudaError_t launch_k(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    const size_t smem = Layout5(a.m, a.kb_stride, KT::PDT, KT::VDT, cand_cap(a.per_block_k)).total;
    auto k = microadam_step_fast<KT>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k<<<static_cast<unsigned>(nblocks), kNT, smem, s>>>(a);
    return cudaGetLastError();
}

// Instantiated dtype combos (g, θ, window value); others use the generic kernel.
#define MA_FAST_DTYPES(X) \
    X(BF16, BF16, BF16)   \
    X(F32, F32, BF16)     \
    X(F32, F32, F32)      \
    X(BF16, F32, BF16)    \
    X(F64, F64, F64)

constexpr int dtype_key(int g, int p, int v) { return g * 9 + p * 3 + v; }

template <int BQ, bool REP>
cudaError_t launch_dt(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    switch (dtype_key(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_) \
        case dtype_key(G_, P_, V_): return launch_k<K<BQ, G_, P_, V_, REP>>(a, nblocks, s);
        MA_FAST_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

template <bool REP>
cudaError_t launch_rep(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    switch (a.bucket) {
        case 16: return launch_dt<16, REP>(a, nblocks, s);
        case 32: return launch_dt<32, REP>(a, nblocks, s);
        case 64: return launch_dt<64, REP>(a, nblocks, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

bool fast_dtypes(int g, int p, int v) {
    switch (dtype_key(g, p, v)) {
#define MA_CASE(G_, P_, V_) case dtype_key(G_, P_, V_): return true;
        MA_FAST_DTYPES(MA_CASE)
#undef MA_CASE
        default: return false;
    }
}

}  // namespace

// Fast path: B_d = 4096, B_q in {16, 32, 64}, m <= 127, and an instantiated
// dtype combo (MA_FAST_DTYPES).
Variant pick_fast_variant(int block, int bucket, int m, int kb_stride, int g_dtype, int p_dtype,
                          int v_dtype) {
    if (bucket != 16 && bucket != 32 && bucket != 64) return {0, 0};
    if (block != kBlock || !fast_dtypes(g_dtype, p_dtype, v_dtype)) return {0, 0};
    if (m > kMaxRowsFast || m * kb_stride > 32768) return {0, 0};
    return {kNT, kEPT};
}

size_t fast_smem_bytes(Variant v, int block, int bucket, int m, int kb_stride, int g_dtype,
                       int p_dtype, int v_dtype) {
    (void)v;
    (void)block;
    (void)bucket;
    (void)g_dtype;
    return Layout5(m, kb_stride, p_dtype, v_dtype, cand_cap(kb_stride)).total;
}

int fast_blocks_per_sm(Variant v, int bucket, size_t smem) {
    (void)v;
    (void)bucket;
    (void)smem;
    return 4;
}

cudaError_t launch_step_fast(const StepArgs& a, Variant v, int grid, cudaStream_t s) {
    (void)grid;
    (void)v;
    if (a.block_count <= 0) return cudaSuccess;
    if (a.block_count > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    return a.partials ? launch_rep<true>(a, a.block_count, s) : launch_rep<false>(a, a.block_count, s);
}

}  // namespace ma
