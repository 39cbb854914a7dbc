// ma_fast.cu — the fast sm_100a MicroAdam step kernel (default layouts).
//
// Same contract and bit-exact results as the generic kernel (ma_kernels.cu),
// built for the HBM roofline. Persistent CTAs walk the shard's FULL Top-K
// blocks (the one partial tail block, if any, goes to the generic kernel):
//
//  * Double-buffered bulk-async staging: while block i is processed, one
//    thread streams block i+gridDim's inputs — g, the 4-bit EF codes, the
//    (lo, hi) bucket grids, θ and the block's m window rows — HBM→smem with
//    1-D cp.async.bulk copies completing on a per-stage mbarrier (SASS
//    UBLKCP). θ is updated in smem and written back with one bulk store.
//  * Lane-contiguous groups: a thread owns runs of 8 consecutive elements, so
//    a B_q bucket is LPB = B_q/8 adjacent lanes and its min/max is 7 register
//    DMNMX + log2(LPB) shuffle levels (quantize.cpp:15-24); a code word is
//    one 32-bit store.
//  * Block Top-K fast path: each block carries a 32-bit threshold on the high
//    word of |a| (≈ the kTarget-th largest key of the previous step). The
//    candidates above it are ranked exactly by (|a| desc, index asc) — high
//    word first, full key and index only on ties — so the selection is always
//    exact; the threshold only decides the work. Outside [k_b, kCandCap]
//    candidates an out-of-line exact radix select runs, recomputing a from
//    the staged inputs.
//  * ADAM_STATS with no per-row barrier: every window coordinate gets one
//    owner entry (last-writer-wins + duplicate marks). Coordinates present in
//    one row take z = 0 + w·v; duplicated ones are re-summed by the owner in
//    physical slot order (binary search in the ascending rows), i.e. exactly
//    window.cpp:32-39's summation order.
//  * Quantization: q ≈ (x−lo)·15/(hi−lo) in fp32 from the exact fp64
//    difference, in 2^-20 fixed point; floor(q+1/2) is taken from it unless
//    q+1/2 lies within 64·2^-20 of an integer (error bound ≈ 10·2^-20), in
//    which case the IEEE quotient (x−lo)/level of quantize.cpp:51 decides.
#include <cstdlib>

#include "../../include/ma_synth.h"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kTarget = 56;      // candidate rank that seeds the next step's threshold
constexpr uint32_t kGuard = 64;  // fixed-point guard band (units of 2^-20)

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
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t hi_key(double x) {
    return static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(x)) >> 32) & 0x7FFFFFFFu;
}

__host__ __device__ inline int dtype_bytes(int dt) { return dt == F64 ? 8 : (dt == F32 ? 4 : 2); }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }

// Shared-memory carve-up (host and device agree).
struct PLayout {
    // per-stage offsets (relative to the stage base) and stage size
    uint32_t g, codes, meta, theta, widx, wval, stage;
    // persistent regions
    uint32_t stage0, lvl, owner, dup, sel, tmpb, wpref, ckey, cval, ckhi, cidx, crank, misc, red, hist,
        bar, total;
    __host__ __device__ PLayout() {}
    __host__ __device__ PLayout(int nt, int block, int bucket, int m, int kbs, int gdt, int pdt,
                                int vdt) {
        const size_t ent = size_t(m) * size_t(kbs);
        const size_t nbk = size_t(block / bucket);
        const size_t nwords = size_t(block / 32);
        size_t o = 0;
        theta = uint32_t(o); o = align_up(o + size_t(block) * dtype_bytes(pdt), 128);
        g = uint32_t(o);     o = align_up(o + size_t(block) * dtype_bytes(gdt), 128);
        codes = uint32_t(o); o = align_up(o + size_t(block) / 2, 128);
        meta = uint32_t(o);  o = align_up(o + nbk * 16, 128);
        widx = uint32_t(o);  o = align_up(o + ent * 2, 128);
        wval = uint32_t(o);  o = align_up(o + ent * dtype_bytes(vdt), 128);
        stage = uint32_t(o);
        size_t q = 0;
        stage0 = uint32_t(q); q = align_up(q + 2 * size_t(stage), 128);
        lvl = uint32_t(q);    q = align_up(q + nbk * 8, 16);
        ckey = uint32_t(q);   q = align_up(q + size_t(kCandCap + 4) * 8, 16);
        cval = uint32_t(q);   q = align_up(q + size_t(kCandCap + 4) * 8, 16);
        red = uint32_t(q);    q = align_up(q + size_t(nt / 32) * kReportFields * 8, 16);
        bar = uint32_t(q);    q = align_up(q + 16, 16);
        owner = uint32_t(q);  q = align_up(q + size_t(block) * 2, 16);
        ckhi = uint32_t(q);   q = align_up(q + size_t(kCandCap + 4) * 4, 16);
        cidx = uint32_t(q);   q = align_up(q + size_t(kCandCap + 4) * 4, 16);
        crank = uint32_t(q);  q = align_up(q + size_t(kCandCap + 4) * 4, 16);
        sel = uint32_t(q);    q = align_up(q + nwords * 4, 16);
        tmpb = uint32_t(q);   q = align_up(q + nwords * 4, 16);
        wpref = uint32_t(q);  q = align_up(q + (nwords + 1) * 4, 16);
        hist = uint32_t(q);   q = align_up(q + 256 * 4, 16);
        misc = uint32_t(q);   q = align_up(q + 96 * 4, 16);
        dup = uint32_t(q);    q = align_up(q + size_t(block), 16);
        total = uint32_t(align_up(q, 128));
    }
};

// Everything the per-block phases need, precomputed once per CTA.
struct Ctx {
    const StepArgs* p;
    unsigned char* smem;
    PLayout L;
    int block, bucket, nbk, nwords, kb, m, kbs, filled, slot;
};

// a(e) recomputed from the staged inputs (used by the out-of-line fallback).
__device__ __forceinline__ double recompute_a(const Ctx& c, const unsigned char* st, int e) {
    const double2* smt = reinterpret_cast<const double2*>(st + c.L.meta);
    const double* s_lvl = reinterpret_cast<const double*>(c.smem + c.L.lvl);
    const uint8_t* codes = st + c.L.codes;
    const int bk = e / c.bucket;
    const uint32_t code = (codes[e >> 1] >> ((e & 1) * 4)) & 15u;
    const double ev = __dadd_rn(__dmul_rn(static_cast<double>(code), s_lvl[bk]), smt[bk].x);
    return __dadd_rn(ld_val(st + c.L.g, c.p->g_dtype, e), ev);
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

// Record selected element e (value a) at window position pos of row `slot`:
// global ring, the staged rows (for P6), and the owner/dup marks.
__device__ __forceinline__ void emit_selected(const Ctx& c, unsigned char* st, int64_t b, int e,
                                              double a, int pos) {
    const StepArgs& p = *c.p;
    const int64_t g = (b * c.m + c.slot) * static_cast<int64_t>(c.kbs) + pos;
    p.win_idx[g] = static_cast<int16_t>(e);
    st_val(p.win_val, p.v_dtype, g, a);
    const int ent = c.slot * c.kbs + pos;
    reinterpret_cast<int16_t*>(st + c.L.widx)[ent] = static_cast<int16_t>(e);
    st_val(st + c.L.wval, p.v_dtype, ent, a);
    reinterpret_cast<uint16_t*>(c.smem + c.L.owner)[e] = static_cast<uint16_t>(ent);
    reinterpret_cast<uint8_t*>(c.smem + c.L.dup)[e] = 0;
}

// Exact fallback selection (compress.cpp:39-53) for blocks whose candidate
// count left [k_b, kCandCap]: generic radix select on a recomputed from smem.
// Leaves the selection bitmap, the new window row and misc[1] = next
// threshold; ends with a barrier.
template <int NT>
__device__ __noinline__ void fallback_select(const Ctx& c, unsigned char* st, int64_t b) {
    constexpr int EPT = 16;  // covers blocks up to NT*16 elements
    unsigned char* sm = c.smem;
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(sm + c.L.sel);
    uint32_t* s_tmpb = reinterpret_cast<uint32_t*>(sm + c.L.tmpb);
    int* s_wpref = reinterpret_cast<int*>(sm + c.L.wpref);
    int* s_misc = reinterpret_cast<int*>(sm + c.L.misc);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto elem = [&](int s) { return s * NT + tid; };
    double a[EPT];
    uint32_t valid = 0;
#pragma unroll
    for (int s = 0; s < EPT; ++s) {
        const int e = elem(s);
        a[s] = 0.0;
        if (e < c.block) {
            a[s] = recompute_a(c, st, e);
            valid |= 1u << s;
        }
    }
    __syncthreads();  // the staged g buffer becomes scratch (selm) below
    uint8_t* selm = st + c.L.g;
    for (int i = tid; i < c.block; i += NT) selm[i] = 0;
    for (int w = tid; w < c.nwords; w += NT) s_tmpb[w] = 0;
    __syncthreads();
    auto tie_rank = [&](uint32_t mask, int (&r)[EPT]) {
        __syncthreads();
#pragma unroll
        for (int s = 0; s < EPT; ++s)
            if ((mask >> s) & 1u) {
                const int e = elem(s);
                atomicOr(&s_tmpb[e >> 5], 1u << (e & 31));
            }
        __syncthreads();
        if (warp == 0) word_prefix(s_tmpb, c.nwords, s_wpref);
        __syncthreads();
#pragma unroll
        for (int s = 0; s < EPT; ++s)
            if ((mask >> s) & 1u) {
                const int e = elem(s);
                r[s] = s_wpref[e >> 5] + __popc(s_tmpb[e >> 5] & ((1u << (e & 31)) - 1u));
            }
    };
    const uint32_t sel = block_topk<NT, EPT>(
        a, valid, c.kb, reinterpret_cast<uint32_t*>(sm + c.L.hist), s_misc + 32,
        reinterpret_cast<uint64_t*>(sm + c.L.ckey), reinterpret_cast<int*>(sm + c.L.cidx), selm,
        elem, tie_rank);
    uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
    for (int s = 0; s < EPT; ++s)
        if ((sel >> s) & 1u) {
            const int e = elem(s);
            atomicOr(&s_sel[e >> 5], 1u << (e & 31));
            kmin = min(kmin, hi_key(a[s]));
        }
    kmin = __reduce_min_sync(0xFFFFFFFFu, kmin);
    if (lane == 0) atomicMin(reinterpret_cast<unsigned int*>(&s_misc[2]), kmin);
    __syncthreads();
    if (warp == 0) word_prefix(s_sel, c.nwords, s_wpref);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < EPT; ++s)
        if ((sel >> s) & 1u) {
            const int e = elem(s);
            const int pos = s_wpref[e >> 5] + __popc(s_sel[e >> 5] & ((1u << (e & 31)) - 1u));
            emit_selected(c, st, b, e, a[s], pos);
        }
    if (tid == 0) {
        const uint32_t km = static_cast<uint32_t>(s_misc[2]);
        s_misc[1] = static_cast<int>(km > (1u << 15) ? km - (1u << 15) : 1u);
    }
    __syncthreads();
}

// Bulk-copy block b's inputs into stage `st` (one thread).
__device__ __forceinline__ void issue_stage(const Ctx& c, unsigned char* st, uint64_t* bar, int64_t b) {
    const StepArgs& p = *c.p;
    const int gsz = dtype_bytes(p.g_dtype), psz = dtype_bytes(p.p_dtype), vsz = dtype_bytes(p.v_dtype);
    const int64_t base = b * c.block;
    const uint32_t bg = uint32_t(c.block * gsz), bc = uint32_t(c.block / 2),
                   bm = uint32_t(c.nbk * 16), bt = uint32_t(c.block * psz),
                   bi = uint32_t(c.m * c.kbs * 2), bv = uint32_t(c.m * c.kbs * vsz);
    mbar_expect_tx(bar, bg + bc + bm + bt + bi + bv);
    const int64_t went = b * c.m * static_cast<int64_t>(c.kbs);
    bulk_g2s(st + c.L.g, static_cast<const unsigned char*>(p.grads) + base * gsz, bg, bar);
    bulk_g2s(st + c.L.codes, p.codes + (base >> 1), bc, bar);
    bulk_g2s(st + c.L.meta, p.meta + base / c.bucket, bm, bar);
    bulk_g2s(st + c.L.theta, static_cast<const unsigned char*>(p.params) + base * psz, bt, bar);
    bulk_g2s(st + c.L.widx, p.win_idx + went, bi, bar);
    bulk_g2s(st + c.L.wval, static_cast<const unsigned char*>(p.win_val) + went * vsz, bv, bar);
}

template <int NT, int G, int LPB>
__global__ void __launch_bounds__(NT, (NT * G >= 512 ? 2 : 3))
microadam_step_persistent(const __grid_constant__ StepArgs p) {
    constexpr int NW = NT / 32;
    constexpr int BUCKET = 8 * LPB;
    extern __shared__ __align__(128) unsigned char smem[];
    Ctx c;
    c.p = &p;
    c.smem = smem;
    c.block = p.block;
    c.bucket = BUCKET;
    c.nbk = p.block / BUCKET;
    c.nwords = p.block / 32;
    c.m = p.m;
    c.kbs = p.kb_stride;
    c.kb = p.per_block_k;  // full blocks: min(per_block_k, block) == per_block_k
    c.filled = p.filled;
    c.slot = p.slot;
    c.L = PLayout(NT, p.block, BUCKET, p.m, p.kb_stride, p.g_dtype, p.p_dtype, p.v_dtype);
    const PLayout& L = c.L;
    double* s_lvl = reinterpret_cast<double*>(smem + L.lvl);
    uint64_t* s_ckey = reinterpret_cast<uint64_t*>(smem + L.ckey);
    double* s_cval = reinterpret_cast<double*>(smem + L.cval);
    double* s_red = reinterpret_cast<double*>(smem + L.red);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    uint16_t* s_owner = reinterpret_cast<uint16_t*>(smem + L.owner);
    uint32_t* s_ckhi = reinterpret_cast<uint32_t*>(smem + L.ckhi);
    int* s_cidx = reinterpret_cast<int*>(smem + L.cidx);
    int* s_crank = reinterpret_cast<int*>(smem + L.crank);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + L.sel);
    int* s_misc = reinterpret_cast<int*>(smem + L.misc);
    uint8_t* s_dup = reinterpret_cast<uint8_t*>(smem + L.dup);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int psz = dtype_bytes(p.p_dtype);
    const int kb = c.kb, kbs = c.kbs, filled = c.filled, slot = c.slot;
    const int nent = filled * kb;
    const bool want_report = p.partials != nullptr;
    const int64_t b_first = p.block_offset + blockIdx.x;
    const int64_t b_end = p.block_offset + p.block_count;

    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        if (b_first < b_end) issue_stage(c, smem + L.stage0, &s_bar[0], b_first);
    }
    __syncthreads();

    int it = 0;
    for (int64_t b = b_first; b < b_end; b += gridDim.x, ++it) {
        const int sidx = it & 1;
        unsigned char* st = smem + L.stage0 + sidx * L.stage;
        if (tid == 0) {
            const int64_t bn = b + gridDim.x;
            if (bn < b_end) {
                bulk_wait_read();  // the other stage's θ store (previous block) has been read
                issue_stage(c, smem + L.stage0 + (sidx ^ 1) * L.stage, &s_bar[sidx ^ 1], bn);
            }
        }
        const uint32_t T = max(p.thresh[b], 1u);
        while (!mbar_try_wait(&s_bar[sidx], (it >> 1) & 1)) {
        }
        const double2* smt = reinterpret_cast<const double2*>(st + L.meta);
        int16_t* swi = reinterpret_cast<int16_t*>(st + L.widx);
        unsigned char* swv = st + L.wval;
        unsigned char* sth = st + L.theta;
        const int64_t base = b * static_cast<int64_t>(c.block);

        // ---- pre: bucket levels of the stored EF (quantize.cpp:7-13), pass-A marks of
        //      the older rows, selection bitmap reset ----
        for (int i = tid; i < c.nbk; i += NT) {
            const double2 mt = smt[i];
            s_lvl[i] = (mt.x == mt.y) ? 0.0 : __ddiv_rn(__dsub_rn(mt.y, mt.x), 15.0);
        }
        for (int t = tid; t < nent; t += NT) {
            const int r = t / kb;
            if (r == slot) continue;
            const int e = r * kbs + (t - r * kb);
            const int idx = swi[e];
            s_owner[idx] = static_cast<uint16_t>(e);
            s_dup[idx] = 0;
        }
        for (int w = tid; w < c.nwords; w += NT) s_sel[w] = 0;
        if (tid == 0) {
            s_misc[NW] = 0;  // candidate counter
            s_misc[2] = -1;  // fallback kmin seed
        }
        __syncthreads();  // [1]

        // ---- P1: a = g + decode(EF) (quantize.cpp:164-178, optim.cpp:166-168) ----
        double a[8 * G];
        uint32_t kmax = 0, cmask = 0;
        double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int e0 = (g * NT + tid) * 8;
            const int bk = e0 / BUCKET;
            double x[8];
            if (p.g_dtype == BF16) {
                const uint4 v = *reinterpret_cast<const uint4*>(st + L.g + e0 * 2);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    x[2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
                    x[2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
                }
            } else if (p.g_dtype == F32) {
                const float4 v0 = *reinterpret_cast<const float4*>(st + L.g + e0 * 4);
                const float4 v1 = *reinterpret_cast<const float4*>(st + L.g + e0 * 4 + 16);
                x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
                x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = reinterpret_cast<const double*>(st + L.g)[e0 + k];
            }
            const uint32_t cw = reinterpret_cast<const uint32_t*>(st + L.codes)[e0 >> 3];
            const double lo = smt[bk].x, level = s_lvl[bk];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double ev = __dadd_rn(__dmul_rn(static_cast<double>((cw >> (4 * i)) & 15u), level), lo);
                const double av = __dadd_rn(x[i], ev);
                a[g * 8 + i] = av;
                const uint32_t kh = hi_key(av);
                kmax = max(kmax, kh);
                cmask |= static_cast<uint32_t>(kh >= T) << (g * 8 + i);
                if (want_report) {
                    rep[0] += x[i] * x[i];
                    rep[1] += av * av;
                }
            }
        }
        if (p.check_finite && kmax >= 0x7FF00000u) atomicOr(p.flag, 1u);  // inf/NaN in g or a

        // ---- P2: block Top-K (compress.cpp:39-53, 73-85) ----
        const int cnt = __popc(cmask);
        int incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += t;
        }
        int wslot = 0;
        if (lane == 31 && incl) wslot = atomicAdd(&s_misc[NW], incl);
        wslot = __shfl_sync(0xFFFFFFFFu, wslot, 31) + incl - cnt;
        if (wslot + cnt <= kCandCap) {
#pragma unroll
            for (int s = 0; s < 8 * G; ++s) {
                if ((cmask >> s) & 1u) {
                    s_ckey[wslot] = key_of(a[s]);
                    s_ckhi[wslot] = hi_key(a[s]);
                    s_cval[wslot] = a[s];
                    s_cidx[wslot] = ((s >> 3) * NT + tid) * 8 + (s & 7);
                    ++wslot;
                }
            }
        }
        __syncthreads();  // [A] candidates
        const int ncand = s_misc[NW];
        if (ncand >= kb && ncand <= kCandCap) {
            if (tid < 4) s_ckhi[ncand + tid] = 0;  // pads never tie (T >= 1)
            const int target = (ncand > kTarget ? kTarget : ncand) - 1;
            __syncthreads();
            for (int t = tid; t < ncand; t += NT) {
                const uint32_t kh = s_ckhi[t];
                int above = 0, eq = 0;
                for (int q = 0; q < ncand; q += 4) {
                    const uint4 v = *reinterpret_cast<const uint4*>(s_ckhi + q);
                    above += (v.x > kh) + (v.y > kh) + (v.z > kh) + (v.w > kh);
                    eq += (v.x == kh) + (v.y == kh) + (v.z == kh) + (v.w == kh);
                }
                int rank = above;
                if (eq > 1) {
                    const uint64_t kt = s_ckey[t];
                    const int it_ = s_cidx[t];
                    for (int q = 0; q < ncand; ++q) {
                        if (q == t || s_ckhi[q] != kh) continue;
                        const uint64_t kq = s_ckey[q];
                        rank += (kq > kt) || (kq == kt && s_cidx[q] < it_);
                    }
                }
                s_crank[t] = rank;
                if (rank == target)
                    s_misc[1] = static_cast<int>(ncand > kTarget ? kh : (kh > (1u << 15) ? kh - (1u << 15) : 1u));
            }
            __syncthreads();  // [B] ranks
            for (int t = tid; t < ncand; t += NT) {
                if (s_crank[t] >= kb) continue;
                const int idx = s_cidx[t];
                int pos = 0;
                for (int q = 0; q < ncand; ++q) pos += (s_crank[q] < kb) & (s_cidx[q] < idx);
                atomicOr(&s_sel[idx >> 5], 1u << (idx & 31));
                emit_selected(c, st, b, idx, s_cval[t], pos);
            }
            __syncthreads();  // [C] selection, new row, its marks
        } else {
            fallback_select<NT>(c, st, b);
        }
        if (tid == 0) p.thresh[b] = static_cast<uint32_t>(s_misc[1]);

        // ---- P6 pass B: duplicate marks ----
        for (int t = tid; t < nent; t += NT) {
            const int r = t / kb;
            const int e = r * kbs + (t - r * kb);
            const int idx = swi[e];
            if (s_owner[idx] != e) s_dup[idx] = 1;
        }

        // ---- P3/P4: residual (compress.cpp:95-102) + 4-bit re-quantization
        //      (quantize.cpp:15-24, 42-55, 102-114, 142-162) ----
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int e0 = (g * NT + tid) * 8;
            const uint32_t sel8 = (s_sel[e0 >> 5] >> (e0 & 31)) & 0xFFu;
            double lo = __longlong_as_double(0x7FF0000000000000ll), hi = -lo;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int s = g * 8 + i;
                if ((sel8 >> i) & 1u) a[s] = 0.0;
                else if (want_report) rep[2] += a[s] * a[s];
                lo = fmin(lo, a[s]);
                hi = fmax(hi, a[s]);
            }
#pragma unroll
            for (int off = 1; off < LPB; off <<= 1) {
                lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
                hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
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
                    const float d32 = __double2float_rn(__dsub_rn(a[g * 8 + i], lo));
                    const uint32_t xq =
                        __float2uint_rz(__fmaf_rn(__fmul_rn(d32, k32), 1048576.0f, 524288.0f));
                    word |= (xq >> 20) << (4 * i);
                    bad |= static_cast<uint32_t>(((xq + kGuard) & 0xFFFFFu) < 2 * kGuard) << i;
                }
                if (bad) {  // rare: exact IEEE quotient for the elements in the guard band
                    const double level = __ddiv_rn(rng, 15.0);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (!((bad >> i) & 1u)) continue;
                        double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(a[g * 8 + i], lo), level), 0.5));
                        f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                        word = (word & ~(15u << (4 * i))) | (static_cast<uint32_t>(f) << (4 * i));
                    }
                }
            }
            if (want_report) {
                const double level = rng == 0.0 ? 0.0 : __ddiv_rn(rng, 15.0);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const double en =
                        __dadd_rn(__dmul_rn(static_cast<double>((word >> (4 * i)) & 15u), level), lo);
                    rep[3] += en * en;
                }
            }
            reinterpret_cast<uint32_t*>(p.codes + ((base + e0) >> 1))[0] = word;
            if ((lane & (LPB - 1)) == 0) p.meta[(base + e0) / BUCKET] = make_double2(lo, hi);
        }
        __syncthreads();  // [D] dup marks complete

        // ---- P6 pass C: ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
        for (int t = tid; t < nent; t += NT) {
            const int r = t / kb;
            const int e = r * kbs + (t - r * kb);
            const int idx = swi[e];
            if (s_owner[idx] != e) continue;
            double z1, z2;
            if (!s_dup[idx]) {
                const double v = ld_val(swv, p.v_dtype, e);
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
                        const double v = ld_val(swv, p.v_dtype, rr * kbs + lo_i);
                        z1 = __dadd_rn(z1, __dmul_rn(p.w1[rr], v));
                        z2 = __dadd_rn(z2, __dmul_rn(p.w2[rr], __dmul_rn(v, v)));
                    }
                }
            }
            const double mhat = __dmul_rn(z1, p.scale1);
            const double vhat = __dmul_rn(z2, p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            const double th = ld_val(sth, p.p_dtype, idx);
            st_val(sth, p.p_dtype, idx, __dsub_rn(th, __dmul_rn(p.lr, u)));
            if (want_report && u != 0.0) rep[4] += 1.0;
        }
        fence_proxy_async_smem();
        __syncthreads();  // [E] θ tile final
        if (tid == 0)
            bulk_s2g(static_cast<unsigned char*>(p.params) + base * psz, sth,
                     static_cast<uint32_t>(c.block * psz));
        if (want_report) {
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
    if (tid == 0) bulk_wait_all();
}

template <int NT, int G, int LPB>
cudaError_t launch_persistent(const StepArgs& a, int grid, cudaStream_t s) {
    const size_t smem = PLayout(NT, a.block, 8 * LPB, a.m, a.kb_stride, a.g_dtype, a.p_dtype,
                                a.v_dtype).total;
    auto k = microadam_step_persistent<NT, G, LPB>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k<<<grid, NT, smem, s>>>(a);
    return cudaGetLastError();
}

template <int NT, int G, int LPB>
int occupancy_of(size_t smem) {
    auto k = microadam_step_persistent<NT, G, LPB>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, NT, smem) != cudaSuccess) return 0;
    return n;
}

template <int LPB>
cudaError_t launch_lpb(const StepArgs& a, Variant v, int grid, cudaStream_t s) {
    const int key = v.nt * 100 + v.ept;
    switch (key) {
        case 12808: return launch_persistent<128, 1, LPB>(a, grid, s);
        case 25608: return launch_persistent<256, 1, LPB>(a, grid, s);
        case 51208: return launch_persistent<512, 1, LPB>(a, grid, s);
        case 12816: return launch_persistent<128, 2, LPB>(a, grid, s);
        case 25616: return launch_persistent<256, 2, LPB>(a, grid, s);
        case 51216: return launch_persistent<512, 2, LPB>(a, grid, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

template <int LPB>
int occupancy_lpb(Variant v, size_t smem) {
    const int key = v.nt * 100 + v.ept;
    switch (key) {
        case 12808: return occupancy_of<128, 1, LPB>(smem);
        case 25608: return occupancy_of<256, 1, LPB>(smem);
        case 51208: return occupancy_of<512, 1, LPB>(smem);
        case 12816: return occupancy_of<128, 2, LPB>(smem);
        case 25616: return occupancy_of<256, 2, LPB>(smem);
        case 51216: return occupancy_of<512, 2, LPB>(smem);
        default: return 0;
    }
}

}  // namespace

// Fast path: B_q in {16, 32, 64}; B_d = 8*NT or 16*NT for NT in {128, 256, 512}
// (one or two 8-element groups per thread); m*kb_stride <= 65535.
Variant pick_fast_variant(int block, int bucket, int m, int kb_stride) {
    if (bucket != 16 && bucket != 32 && bucket != 64) return {0, 0};
    if (block % bucket != 0 || m * kb_stride > 65535 || block % 1024 != 0) return {0, 0};
    const char* g2 = std::getenv("MA_FAST_G2");  // A/B switch: two groups per thread
    const bool two = g2 && g2[0] == '1';
    for (int nt : {128, 256, 512}) {
        if (!two && block == 8 * nt) return {nt, 8};
        if (two && block == 16 * nt) return {nt, 16};
    }
    if (block == 16 * 512) return {512, 16};  // B_d = 8192
    if (block == 1024) return {128, 8};
    return {0, 0};
}

size_t fast_smem_bytes(Variant v, int block, int bucket, int m, int kb_stride, int g_dtype,
                       int p_dtype, int v_dtype) {
    return PLayout(v.nt, block, bucket, m, kb_stride, g_dtype, p_dtype, v_dtype).total;
}

int fast_blocks_per_sm(Variant v, int bucket, size_t smem) {
    switch (bucket) {
        case 16: return occupancy_lpb<2>(v, smem);
        case 32: return occupancy_lpb<4>(v, smem);
        case 64: return occupancy_lpb<8>(v, smem);
        default: return 0;
    }
}

cudaError_t launch_step_fast(const StepArgs& a, Variant v, int grid, cudaStream_t s) {
    if (a.block_count <= 0) return cudaSuccess;
    switch (a.bucket) {
        case 16: return launch_lpb<2>(a, v, grid, s);
        case 32: return launch_lpb<4>(a, v, grid, s);
        case 64: return launch_lpb<8>(a, v, grid, s);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace ma
