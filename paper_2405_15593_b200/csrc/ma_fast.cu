// ma_fast.cu — the fast sm_100a MicroAdam step kernel (default layouts).
//
// Same contract and bit-exact results as the generic kernel (ma_kernels.cu),
// shaped for the HBM roofline: one small CTA (128 threads, 4 warps, ~25 KB
// smem, ≤ 64 registers) per FULL Top-K block, 8 CTAs resident per SM, so
// eight blocks' load / compute / barrier phases overlap on every SM. The one
// partial tail block of a shard, if any, goes to the generic kernel.
//
//  * θ and the block's m window rows are staged HBM→smem at CTA start with
//    1-D bulk async copies on an mbarrier (SASS UBLKCP); θ returns with one
//    bulk store. g, the 4-bit EF codes and (lo, hi) stream through registers.
//  * Lane-contiguous groups: a thread owns runs of 8 consecutive elements, so
//    a B_q bucket is LPB = B_q/8 adjacent lanes: its min/max is 7 register
//    DMNMX + log2(LPB) shuffle levels (quantize.cpp:15-24) and its 4-bit code
//    word one 32-bit store. The levels of the stored EF (quantize.cpp:7-13)
//    are computed once per block into smem.
//  * P1 decodes a = g + e only for the Top-K keys; P3 recomputes a (an
//    L2-hot re-read of g and the codes) instead of holding 32 doubles/thread.
//  * Block Top-K: P1 keeps a 16-bit key (bits 62..48 of |a|) per element in
//    registers. A threshold t with k_b <= #{key16 >= t} <= cap is taken from
//    the previous step (one 16-bit bucket below its k_b-th key, carried per block) or
//    found by bisection on block-wide counts (SIMD __vcmpgeu2 + popc, one
//    barrier per probe). The candidates above t are ranked exactly by
//    (|a| desc, index asc) — high word first, full key and index only on ties
//    — so the selection is always exact; t only decides the work. Only when
//    more than `cap` keys tie at 16-bit resolution does an out-of-line exact
//    radix select run. Selected elements get their ascending window position
//    from a word prefix of a selection bitmap.
//  * ADAM_STATS with no per-row barrier: every window coordinate gets one
//    owner row (last-writer-wins byte + duplicate bit). Coordinates present in
//    one row take z = 0 + w·v; duplicated ones are re-summed by the owner in
//    physical slot order (binary search in the ascending rows), i.e. exactly
//    window.cpp:32-39's summation order.
//  * Quantization: q ≈ (x−lo)·15/(hi−lo) in fp32 from the exact fp64
//    difference, in 2^-20 fixed point; floor(q+1/2) is taken from it unless
//    q+1/2 lies within 64·2^-20 of an integer (error bound ≈ 4·2^-20), in
//    which case the IEEE quotient (x−lo)/level of quantize.cpp:51 decides.
#include <cstdlib>

#include "../../include/ma_synth.h"
#include "ma_async.cuh"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kNT = 128;          // threads per CTA
constexpr int kEPT = 32;          // elements per thread at B_d = 4096 (fallback view)
constexpr uint32_t kGuard = 64;   // fixed-point guard band (units of 2^-20)
constexpr int kMaxRowsFast = 127; // owner byte holds the row (7 bits) + a duplicate bit

// Candidate capacity of the exact-rank stage: 2 k_b, at least 128, at most 512.
__host__ __device__ inline int cand_cap(int kb) {
    const int c = ((2 * kb + 3) / 4) * 4;
    return c < 128 ? 128 : (c > 512 ? 512 : c);
}

// Shared-memory carve-up (host and device agree).
struct Layout4 {
    uint32_t theta, widx, wval, lo, lvl, cval, red, bar, owner, selm, ckhi, cidx, sel, tmpb, wpref,
        hist, misc, ckey, k16, total;
    __host__ __device__ Layout4() {}
    __host__ __device__ Layout4(int block, int bucket, int m, int kbs, int pdt, int vdt, int cap) {
        const size_t ent = size_t(m) * size_t(kbs);
        const size_t nbk = size_t(block / bucket);
        const size_t nwords = size_t(block / 32);
        size_t o = 0;
        theta = uint32_t(o); o = align_up(o + size_t(block) * dtype_bytes(pdt), 128);
        widx = uint32_t(o);  o = align_up(o + ent * 2, 128);
        wval = uint32_t(o);  o = align_up(o + ent * dtype_bytes(vdt), 128);
        lo = uint32_t(o);    o = align_up(o + nbk * 8, 16);
        lvl = uint32_t(o);   o = align_up(o + nbk * 8, 16);
        cval = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 8, 16);
        ckey = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 8, 16);
        red = uint32_t(o);   o = align_up(o + size_t(kNT / 32) * kReportFields * 8, 16);
        bar = uint32_t(o);   o = align_up(o + 16, 16);
        k16 = uint32_t(o);   o = align_up(o + size_t(block) * 2, 16);
        owner = uint32_t(o); o = align_up(o + size_t(block), 16);
        selm = owner;  // fallback scratch; owner marks are written after the selection
        ckhi = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 4, 16);
        cidx = uint32_t(o);  o = align_up(o + size_t(cap + 4) * 4, 16);
        sel = uint32_t(o);   o = align_up(o + nwords * 4, 16);
        tmpb = uint32_t(o);  o = align_up(o + nwords * 4, 16);
        wpref = uint32_t(o); o = align_up(o + (nwords + 1) * 4, 16);
        hist = uint32_t(o);  o = align_up(o + 256 * 4, 16);
        misc = uint32_t(o);  o = align_up(o + 96 * 4, 16);
        total = uint32_t(align_up(o, 128));
    }
};

// Compile-time shape of one fast-kernel instantiation.
template <int G_, int LPB_, int GDT_, int PDT_, int VDT_, bool REP_>
struct K {
    static constexpr int G = G_, LPB = LPB_, GDT = GDT_, PDT = PDT_, VDT = VDT_;
    static constexpr bool REPORT = REP_;
    static constexpr int BUCKET = 8 * LPB_, BLOCK = 8 * kNT * G_;
};

struct Ctx {
    const StepArgs* p;
    unsigned char* smem;
    Layout4 L;
    int64_t b, base;
    int block, bucket, nwords, kb, m, kbs, slot;
};

template <class KT>
__device__ __forceinline__ Ctx make_ctx(const StepArgs& p) {
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    Ctx c;
    c.p = &p;
    c.smem = smem_dyn;
    c.block = KT::BLOCK;
    c.bucket = KT::BUCKET;
    c.nwords = KT::BLOCK / 32;
    c.m = p.m;
    c.kbs = p.kb_stride;
    c.kb = p.per_block_k;
    c.slot = p.slot;
    c.L = Layout4(KT::BLOCK, KT::BUCKET, p.m, p.kb_stride, KT::PDT, KT::VDT, cand_cap(p.per_block_k));
    c.b = p.block_offset + blockIdx.x;
    c.base = c.b * KT::BLOCK;
    return c;
}

// 8 consecutive g values (element e0, 8-aligned) as doubles.
template <int DT>
__device__ __forceinline__ void load_g8(const void* g, int64_t e0, double (&x)[8]) {
    if constexpr (DT == BF16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + e0));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
            x[2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
        }
    } else if constexpr (DT == F32) {
        const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(g) + e0);
        const float4 v0 = __ldg(q), v1 = __ldg(q + 1);
        x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
        x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
    } else {
        const double2* q = reinterpret_cast<const double2*>(static_cast<const double*>(g) + e0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 v = __ldg(q + k);
            x[2 * k] = v.x;
            x[2 * k + 1] = v.y;
        }
    }
}

// a = g + (code·level + lo) for the 8 elements at e0 (quantize.cpp:164-178,
// optim.cpp:166-168): separate multiply and add, fp64, no FMA.
template <class KT>
__device__ __forceinline__ void decode8(const Ctx& c, int e0, double (&a)[8]) {
    const StepArgs& p = *c.p;
    load_g8<KT::GDT>(p.grads, c.base + e0, a);
    const uint32_t cw = __ldg(reinterpret_cast<const uint32_t*>(p.codes + ((c.base + e0) >> 1)));
    const int bk = e0 / KT::BUCKET;
    const double lo = reinterpret_cast<const double*>(c.smem + c.L.lo)[bk];
    const double level = reinterpret_cast<const double*>(c.smem + c.L.lvl)[bk];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        a[i] = __dadd_rn(a[i], __dadd_rn(__dmul_rn(static_cast<double>((cw >> (4 * i)) & 15u), level), lo));
}

template <class KT>
__device__ __forceinline__ double recompute_a(const Ctx& c, int e) {
    const StepArgs& p = *c.p;
    const uint32_t byte = p.codes[(c.base + e) >> 1];
    const int bk = e / KT::BUCKET;
    const double lo = reinterpret_cast<const double*>(c.smem + c.L.lo)[bk];
    const double level = reinterpret_cast<const double*>(c.smem + c.L.lvl)[bk];
    const double ev = __dadd_rn(__dmul_rn(static_cast<double>((byte >> ((e & 1) * 4)) & 15u), level), lo);
    return __dadd_rn(ld_t<KT::GDT>(p.grads, c.base + e), ev);
}

// t / kb for t < 2^16 without an integer division (float reciprocal + fix-up).
__device__ __forceinline__ int row_of(int t, int kb, float inv_kb) {
    int r = __float2int_rz(static_cast<float>(t) * inv_kb);
    r -= (r * kb > t);
    r += ((r + 1) * kb <= t);
    return r;
}

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

// The IEEE path of quantize_nearest (quantize.cpp:51-53): the code of x in a
// bucket with grid (lo, level), for elements whose fast fixed-point estimate
// fell in the guard band. Out of line: rare, and scalar arguments only.
__device__ __noinline__ uint32_t exact_code(double x, double lo, double level) {
    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(x, lo), level), 0.5));
    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
    return static_cast<uint32_t>(f);
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
// `cap` keys tie at 16-bit resolution: the generic radix select on a recomputed from
// the (L2-hot) inputs. Sets the selection bitmap + prefix, emits the new row
// and misc[1] = next threshold.
template <class KT>
__device__ __noinline__ void fallback_select(const StepArgs* pp) {
    const Ctx c = make_ctx<KT>(*pp);
    unsigned char* sm = c.smem;
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(sm + c.L.sel);
    uint32_t* s_tmpb = reinterpret_cast<uint32_t*>(sm + c.L.tmpb);
    int* s_wpref = reinterpret_cast<int*>(sm + c.L.wpref);
    int* s_misc = reinterpret_cast<int*>(sm + c.L.misc);
    uint8_t* selm = sm + c.L.selm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < c.block; i += kNT) selm[i] = 0;
    for (int w = tid; w < c.nwords; w += kNT) s_tmpb[w] = 0;
    auto elem = [&](int s) { return s * kNT + tid; };
    double a[kEPT];
    uint32_t valid = 0;
#pragma unroll
    for (int s = 0; s < kEPT; ++s) {
        a[s] = 0.0;
        if (elem(s) < c.block) {
            a[s] = recompute_a<KT>(c, elem(s));
            valid |= 1u << s;
        }
    }
    __syncthreads();
    auto tie_rank = [&](uint32_t mask, int (&r)[kEPT]) {
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kEPT; ++s)
            if ((mask >> s) & 1u) atomicOr(&s_tmpb[elem(s) >> 5], 1u << (elem(s) & 31));
        __syncthreads();
        if (warp == 0) word_prefix(s_tmpb, c.nwords, s_wpref);
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kEPT; ++s)
            if ((mask >> s) & 1u) {
                const int e = elem(s);
                r[s] = s_wpref[e >> 5] + __popc(s_tmpb[e >> 5] & ((1u << (e & 31)) - 1u));
            }
    };
    const uint32_t sel = block_topk<kNT, kEPT>(
        a, valid, c.kb, reinterpret_cast<uint32_t*>(sm + c.L.hist), s_misc + 32,
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
    if (warp == 0) word_prefix(s_sel, c.nwords, s_wpref);
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

template <class KT>
__global__ void __launch_bounds__(kNT, 8) microadam_step_fast(const __grid_constant__ StepArgs p) {
    constexpr int NW = kNT / 32;
    constexpr int G = KT::G, LPB = KT::LPB, BUCKET = KT::BUCKET, BLOCK = KT::BLOCK;
    static_assert(8 * G <= kEPT, "candidate masks are 32-bit");
    extern __shared__ __align__(128) unsigned char smem[];
    const Ctx c = make_ctx<KT>(p);
    const Layout4& L = c.L;
    unsigned char* sth = smem + L.theta;
    int16_t* swi = reinterpret_cast<int16_t*>(smem + L.widx);
    unsigned char* swv = smem + L.wval;
    double* s_lo = reinterpret_cast<double*>(smem + L.lo);
    double* s_lvl = reinterpret_cast<double*>(smem + L.lvl);
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
    constexpr int psz = KT::PDT == F64 ? 8 : (KT::PDT == F32 ? 4 : 2);
    constexpr int vsz = KT::VDT == F64 ? 8 : (KT::VDT == F32 ? 4 : 2);
    const int kb = c.kb, kbs = c.kbs, slot = c.slot, filled = p.filled, m = c.m;
    const int nent = filled * kb;
    const int cap = cand_cap(kb);
    const float inv_kb = 1.0f / static_cast<float>(kb);
    const int64_t b = c.b, base = c.base;
    constexpr bool want_report = KT::REPORT;

    // ---- prologue: θ + window rows HBM→smem (bulk async), bucket grids ----
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        const uint32_t bt = uint32_t(BLOCK * psz), bi = uint32_t(m * kbs * 2),
                       bv = uint32_t(m * kbs * vsz);
        mbar_expect_tx(s_bar, bt + bi + bv);
        const int64_t went = b * m * static_cast<int64_t>(kbs);
        bulk_g2s(sth, static_cast<const unsigned char*>(p.params) + base * psz, bt, s_bar);
        bulk_g2s(swi, p.win_idx + went, bi, s_bar);
        bulk_g2s(swv, static_cast<const unsigned char*>(p.win_val) + went * vsz, bv, s_bar);
    }
    const uint32_t T = max(__ldg(p.thresh + b), 1u);
    for (int i = tid; i < BLOCK / BUCKET; i += kNT) {  // QuantParams ctor, quantize.cpp:7-13
        const double2 mt = __ldg(p.meta + base / BUCKET + i);
        s_lo[i] = mt.x;
        s_lvl[i] = (mt.x == mt.y) ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), 15.0);
    }
    for (int w = tid; w < BLOCK / 32; w += kNT) s_sel[w] = 0;
    if (tid == 0) {
        s_misc[NW] = 0;  // candidate counter
        s_misc[2] = -1;  // fallback kmin seed
    }
    __syncthreads();  // [L]

    // ---- P1: a = g + decode(EF) -> 16-bit Top-K keys (bits 62..48 of |a|:
    //      exponent + 4 mantissa bits) in smem, counted against the carried
    //      threshold on the fly ----
    uint16_t* s_k16 = reinterpret_cast<uint16_t*>(smem + L.k16);
    const uint32_t carried = __ldg(p.thresh + b);
    uint32_t kmax = 0;
    int cnt0 = 0;
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    {
        const uint32_t tt = carried | (carried << 16);
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
            const int e0 = (g * kNT + tid) * 8;
            double a[8];
            decode8<KT>(c, e0, a);
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t h0 = hi_key(a[2 * k]) >> 16, h1 = hi_key(a[2 * k + 1]) >> 16;
                w[k] = h0 | (h1 << 16);
                kmax = max(kmax, max(h0, h1));
                cnt0 += __popc(__vcmpgeu2(w[k], tt));
                if (want_report) rep[1] += a[2 * k] * a[2 * k] + a[2 * k + 1] * a[2 * k + 1];
            }
            *reinterpret_cast<uint4*>(s_k16 + e0) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    if (p.check_finite && kmax >= 0x7FF0u) atomicOr(p.flag, 1u);  // inf/NaN in g or a

    // ---- P2: block Top-K (compress.cpp:39-53, 73-85). Find a 16-bit threshold t
    //      with k_b <= #{key16 >= t} <= cap (carried from the previous step, else
    //      bisection on block-wide counts), then rank those candidates exactly. ----
    int* s_cnt = s_misc + 64;  // [2][NW] per-warp counts, double-buffered
    auto publish = [&](int n, int par) -> int {
        n = __reduce_add_sync(0xFFFFFFFFu, n >> 4);
        if (lane == 0) s_cnt[par * NW + warp] = n;
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) tot += s_cnt[par * NW + w];
        return tot;
    };
    auto block_count = [&](uint32_t t, int par) -> int {
        const uint32_t tt = t | (t << 16);
        int n = 0;
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
            const uint4 v = *reinterpret_cast<const uint4*>(s_k16 + (g * kNT + tid) * 8);
            n += __popc(__vcmpgeu2(v.x, tt)) + __popc(__vcmpgeu2(v.y, tt)) +
                 __popc(__vcmpgeu2(v.z, tt)) + __popc(__vcmpgeu2(v.w, tt));
        }
        return publish(n, par);
    };
    const uint32_t wmax = __reduce_max_sync(0xFFFFFFFFu, kmax);
    if (lane == 0) s_misc[48 + warp] = static_cast<int>(wmax);
    int par = 0;
    cnt0 = publish(cnt0, par);  // [A0] also publishes the warp maxima and the keys
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
            const int n = block_count(mid, par);
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
    }
    if (tid == 0) s_misc[NW] = 0;
    __syncthreads();  // candidate counter reset visible
    if (found) {
        // Collect the candidates: each thread scans its 32 keys and recomputes a
        // only for its candidates (warp-aggregated slot allocation).
        const uint32_t tt = t16 | (t16 << 16);
        uint32_t cm = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint4 v = *reinterpret_cast<const uint4*>(s_k16 + (g * kNT + tid) * 8);
            const uint32_t r[4] = {__vcmpgeu2(v.x, tt), __vcmpgeu2(v.y, tt), __vcmpgeu2(v.z, tt),
                                   __vcmpgeu2(v.w, tt)};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                cm |= ((r[k] & 1u) | ((r[k] >> 15) & 2u)) << (g * 8 + 2 * k);
        }
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
        while (cm) {
            const int sb = __ffs(cm) - 1;
            cm &= cm - 1;
            const int e = ((sb >> 3) * kNT + tid) * 8 + (sb & 7);
            const double av = recompute_a<KT>(c, e);
            s_cval[sidx] = av;
            s_ckhi[sidx] = hi_key(av);
            s_cidx[sidx] = e;
            ++sidx;
        }
        __syncthreads();  // [A] candidates
        const int ncand = s_misc[NW];
        if (warp == 0) {
            // Exact Top-k_b among the candidates (compress.cpp:39-53): bisect the
            // k_b-th largest high word with warp-wide counts; ties on the high
            // word resolve on the full |a| key, then the lower index.
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
        if (warp == 0) word_prefix(s_sel, BLOCK / 32, s_wpref);
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
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        const int e0 = (g * kNT + tid) * 8;
        double a[8];
        decode8<KT>(c, e0, a);
        const uint32_t sel8 = (s_sel[e0 >> 5] >> (e0 & 31)) & 0xFFu;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((sel8 >> i) & 1u) a[i] = 0.0;
            if (want_report) rep[2] += a[i] * a[i];
        }
        // min / max of the 8 residuals (quantize.cpp:15-24; no NaN, no -0.0 here):
        // a compare-exchange per pair, then two 4-way trees.
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
            const float k32 = fastq ? __fdiv_rn(15.0f, r32) : 0.0f;
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
                        word = (word & ~(15u << (4 * i))) | (exact_code(a[i], lo, level) << (4 * i));
                if (p.dbg) atomicAdd(p.dbg + 1, __popc(bad));
            }
        }
        if (want_report) {
            const double level = rng == 0.0 ? 0.0 : __ddiv_rn(rng, 15.0);
            double x[8];
            load_g8<KT::GDT>(p.grads, base + e0, x);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double en =
                    __dadd_rn(__dmul_rn(static_cast<double>((word >> (4 * i)) & 15u), level), lo);
                rep[3] += en * en;
                rep[0] += x[i] * x[i];
            }
        }
        *reinterpret_cast<uint32_t*>(p.codes + ((base + e0) >> 1)) = word;
        if ((lane & (LPB - 1)) == 0) p.meta[(base + e0) / BUCKET] = make_double2(lo, hi);
    }
    __syncthreads();  // [D] all owner rows written (older rows + new row)

    // ---- P6 pass B: duplicate bit (coordinate present in more than one row) ----
    for (int t = tid; t < nent; t += kNT) {
        const int r = row_of(t, kb, inv_kb);
        const int idx = swi[r * kbs + (t - r * kb)];
        if ((s_owner[idx] & 0x7F) != r) s_owner[idx] |= 0x80;
    }
    __syncthreads();  // [E]

    // ---- P6 pass C: ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187).
    //      Coordinates held by one row are finished inline; owners of duplicated
    //      coordinates are queued and re-summed in slot order afterwards, so a
    //      warp never carries the m-row search for a single lane. ----
    int* s_dupq = s_misc + 80;  // [0] count; the queue reuses the dead candidate-value area
    int* dupq = reinterpret_cast<int*>(s_cval);
    const int qcap = (L.ckey - L.cval) / 2;  // ints in cval+ckey, >= 4 * (cap + 4)
    if (tid == 0) s_dupq[0] = 0;
    __syncthreads();
    auto update = [&](int idx, double z1, double z2) {
        const double mhat = __dmul_rn(z1, p.scale1);
        const double vhat = __dmul_rn(z2, p.scale2);
        const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
        const double th = ld_t<KT::PDT>(sth, idx);
        st_t<KT::PDT>(sth, idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
        if (want_report && u != 0.0) rep[4] += 1.0;
    };
    auto dup_sum = [&](int idx) {
        double z1 = 0.0, z2 = 0.0;
        for (int rr = 0; rr < filled; ++rr) {  // physical slot order (window.cpp:32-39)
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
        update(idx, z1, z2);
    };
    for (int t = tid; t < nent; t += kNT) {
        const int r = row_of(t, kb, inv_kb);
        const int e = r * kbs + (t - r * kb);
        const int idx = swi[e];
        const uint32_t own = s_owner[idx];
        if ((own & 0x7F) != static_cast<uint32_t>(r)) continue;
        if (own & 0x80) {
            const int q = atomicAdd(&s_dupq[0], 1);
            if (q < qcap) dupq[q] = idx; else dup_sum(idx);  // queue overflow: inline
            continue;
        }
        const double v = ld_t<KT::VDT>(swv, e);
        update(idx, __dadd_rn(0.0, __dmul_rn(p.w1[r], v)),
               __dadd_rn(0.0, __dmul_rn(p.w2[r], __dmul_rn(v, v))));
    }
    __syncthreads();
    const int ndup = min(s_dupq[0], qcap);
    for (int q = tid; q < ndup; q += kNT) dup_sum(dupq[q]);
    fence_proxy_async_smem();
    __syncthreads();  // [F] θ tile final
    if (tid == 0) {
        bulk_s2g(static_cast<unsigned char*>(p.params) + base * psz, sth,
                 static_cast<uint32_t>(BLOCK * psz));
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
    const size_t smem =
        Layout4(KT::BLOCK, KT::BUCKET, a.m, a.kb_stride, KT::PDT, KT::VDT, cand_cap(a.per_block_k)).total;
    auto k = microadam_step_fast<KT>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k<<<static_cast<unsigned>(nblocks), kNT, smem, s>>>(a);
    return cudaGetLastError();
}

// Instantiated dtype combos (g, θ, window value); others use the generic kernel.
#define MA_FAST_DTYPES(X)         \
    X(BF16, BF16, BF16)           \
    X(F32, F32, BF16)             \
    X(F32, F32, F32)              \
    X(BF16, F32, BF16)            \
    X(F64, F64, F64)

constexpr int dtype_key(int g, int p, int v) { return g * 9 + p * 3 + v; }

template <int LPB, bool REP>
cudaError_t launch_dt(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    switch (dtype_key(a.g_dtype, a.p_dtype, a.v_dtype)) {
#define MA_CASE(G_, P_, V_) \
        case dtype_key(G_, P_, V_): return launch_k<K<4, LPB, G_, P_, V_, REP>>(a, nblocks, s);
        MA_FAST_DTYPES(MA_CASE)
#undef MA_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}

template <bool REP>
cudaError_t launch_rep(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    switch (a.bucket) {
        case 16: return launch_dt<2, REP>(a, nblocks, s);
        case 32: return launch_dt<4, REP>(a, nblocks, s);
        case 64: return launch_dt<8, REP>(a, nblocks, s);
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
    if (block != 4096 || !fast_dtypes(g_dtype, p_dtype, v_dtype)) return {0, 0};
    if (m > kMaxRowsFast || m * kb_stride > 32768) return {0, 0};
    return {kNT, block / kNT};
}

size_t fast_smem_bytes(Variant v, int block, int bucket, int m, int kb_stride, int g_dtype,
                       int p_dtype, int v_dtype) {
    (void)v;
    (void)g_dtype;
    const int kb = kb_stride;  // upper bound of per_block_k (kb_stride = round_up(k_b, 8))
    return Layout4(block, bucket, m, kb_stride, p_dtype, v_dtype, cand_cap(kb)).total;
}

int fast_blocks_per_sm(Variant v, int bucket, size_t smem) {
    (void)v;
    (void)bucket;
    (void)smem;
    return 8;
}

cudaError_t launch_step_fast(const StepArgs& a, Variant v, int grid, cudaStream_t s) {
    (void)grid;
    (void)v;
    if (a.block_count <= 0) return cudaSuccess;
    if (a.block_count > 0x7FFFFFFFll) return cudaErrorInvalidConfiguration;
    return a.partials ? launch_rep<true>(a, a.block_count, s) : launch_rep<false>(a, a.block_count, s);
}

}  // namespace ma
