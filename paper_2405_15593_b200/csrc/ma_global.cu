// ma_global.cu — global Top-K mode (MicroAdamOptimizer with blockwise = false,
// the reference's default: topk_global, compress.cpp:66-71) for d > 8192.
//
// Correctness-first pipeline over the whole vector, every decision in the
// reference's fp64 arithmetic (a = g + (c·level + lo), optim.cpp:166-168,
// quantize.cpp:164-178):
//   G0  per-bucket level = (hi - lo) / 15 of the current EF (quantize.cpp:7-13)
//   G1  radix histograms of the 63-bit |a| keys, six digit passes (11-bit
//       digits, then 8), each digit picked on the device by one warp: the
//       exact k-th key K* and how many ties at K* the selection takes
//       (compress.cpp:39-53: |a| desc, idx asc)
//   G2  per 4096-chunk counts of keys > K* and == K*, then one CTA scans them
//       into row offsets and ties per chunk (lowest indices first)
//   G3  emit: the selected entries in ascending index order at their global
//       row positions, the selection bitmap
// No host synchronisation inside the step.
//   G4  residual (compress.cpp:95-102) + bucket min/max + 4-bit codes by the
//       IEEE quotient (quantize.cpp:15-24, 42-55, 102-114), StepReport sums
//   G5  ADAM_STATS as window.cpp:28-46 does it, per 4096-chunk in shared
//       memory: each row's entries of the chunk (bounds found once per step)
//       accumulated row by row in physical slot order, then
//   G6  the update θ -= lr · mhat / (eps + sqrt(vhat)) (optim.cpp:183-187) for
//       every coordinate with a nonzero accumulator (u = 0 elsewhere).
// Passes over d read the gradient and codes 8 elements per thread (g_a8).
// Window rows: int64 global indices [m][row stride] + values (any d).
#include <math_constants.h>

#include <cstdlib>

#include "ma_async.cuh"
#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kChunk = 4096;     // elements per CTA in G2/G3/G4
#ifndef MA_RQ8_UNROLL
#define MA_RQ8_UNROLL 1  // A/B: 2 = both 2048-element halves of a chunk in flight
#endif
constexpr int kRq8Unroll = MA_RQ8_UNROLL;
constexpr int kThreads = 256;
constexpr int kPer = kChunk / kThreads;  // 16 elements per thread (strided by 256)

__device__ __forceinline__ int64_t global_chunks_d(int64_t dim) { return (dim + kChunk - 1) / kChunk; }
constexpr int kStage = 1024;  // window entries per chunk staged in shared memory by g_stats_update

__device__ __forceinline__ double g_a(const GlobalArgs& p, int64_t i) {
    if (p.dense) return __dadd_rn(ld_val(p.grads, p.g_dtype, i), p.dense[i]);  // lossless (optim.cpp:166-168)
    const int64_t q = i >> p.bucket_shift;  // bucket | 4096: a power of two
    const double lo = p.meta[q].x;
    const uint32_t byte = p.codes[i >> 1];
    const double c = static_cast<double>((byte >> ((i & 1) * 4)) & 15u);
    const double e = __dadd_rn(__dmul_rn(c, p.level[q]), lo);
    return __dadd_rn(ld_val(p.grads, p.g_dtype, i), e);
}

// a at the 8 consecutive elements [i0, i0 + 8) (i0 % 8 == 0), same arithmetic
// as g_a; entries at or past dim are 0 and `nv` says how many are valid. One
// 16-byte gradient load (bf16), one 4-byte code word and one bucket grid when
// the bucket holds the whole group.
__device__ __forceinline__ int g_a8(const GlobalArgs& p, int64_t i0, double (&a)[8]) {
    const int nv = p.dim - i0 >= 8 ? 8 : static_cast<int>(p.dim - i0);
    const bool vec = nv == 8 && p.bucket_shift >= 3 && !p.dense &&
                     (reinterpret_cast<uintptr_t>(p.grads) & 15u) == 0;
    if (!vec) {
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = e < nv ? g_a(p, i0 + e) : 0.0;
        return nv;
    }
    const int64_t q = i0 >> p.bucket_shift;
    const double lo = p.meta[q].x, lv = p.level[q];
    const uint32_t cw = *reinterpret_cast<const uint32_t*>(p.codes + (i0 >> 1));
    double g[8];
    if (p.g_dtype == BF16) {
        const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p.grads) + i0);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            g[2 * k] = static_cast<double>(__uint_as_float(w[k] << 16));
            g[2 * k + 1] = static_cast<double>(__uint_as_float(w[k] & 0xFFFF0000u));
        }
    } else if (p.g_dtype == F32) {
        const float4* f = reinterpret_cast<const float4*>(static_cast<const float*>(p.grads) + i0);
        const float4 x = f[0], y = f[1];
        g[0] = x.x; g[1] = x.y; g[2] = x.z; g[3] = x.w;
        g[4] = y.x; g[5] = y.y; g[6] = y.z; g[7] = y.w;
    } else {
        const double2* d2 = reinterpret_cast<const double2*>(static_cast<const double*>(p.grads) + i0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 t = d2[k];
            g[2 * k] = t.x;
            g[2 * k + 1] = t.y;
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const double c = static_cast<double>((cw >> (4 * e)) & 15u);
        a[e] = __dadd_rn(g[e], __dadd_rn(__dmul_rn(c, lv), lo));
    }
    return 8;
}

__global__ void g_levels(GlobalArgs p) {
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < p.nbuckets;
         q += int64_t(gridDim.x) * blockDim.x) {
        const double2 m = p.meta[q];
        p.level[q] = m.x == m.y ? 0.0 : __ddiv_rn(__dsub_rn(m.y, m.x), 15.0);
    }
}

// One radix digit: histogram of (key >> shift) & (nbins - 1) over keys whose
// bits above the digit equal `prefix` (under `pmask`).
// collect: also append the keys that share the prefix (the candidates of the
// remaining digits) to p.cand; from_cand: passes after the collecting one read
// p.cand instead of re-decoding the vector, unless it overflowed.
template <bool PRIV>
__global__ void g_hist(GlobalArgs p, int shift, int nbins, int collect, int from_cand) {
    // PRIV (first digits, keys crowd a few bins): one histogram per warp and
    // plain shared atomics; otherwise one per CTA with match.any aggregation
    extern __shared__ uint32_t s_hw[];
    __shared__ uint32_t s_h1[PRIV ? 1 : 2048];
    uint32_t* h = PRIV ? s_hw + (threadIdx.x >> 5) * 2048 : s_h1;
    const uint64_t prefix = p.sel_state[0], pmask = p.sel_state[1];
    if (from_cand && *p.cand_n <= p.cand_cap) return;  // g_hist_cand covers this digit
    if (p.sel_state[8]) return;                          // the bracket holds K*: g_hist_cand
    for (int i = threadIdx.x; i < (PRIV ? 2048 * (kThreads / 32) : nbins); i += blockDim.x) (PRIV ? s_hw : s_h1)[i] = 0;
    __syncthreads();
    bool bad = false;
    const int64_t ngroups = (p.dim + 7) / 8;
    for (int64_t gi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; gi < ngroups;
         gi += int64_t(gridDim.x) * blockDim.x) {
        double a[8];
        const int nv = g_a8(p, gi * 8, a);
        const unsigned act = __activemask();
        uint32_t inm = 0;
        int bins[8];
        int above = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint64_t k = key_of(a[e]);
            bad |= e < nv && (k >> 52) >= 0x7FFu;  // inf / NaN (check_finite in topk_global)
            const bool in = e < nv && (k & pmask) == prefix;
            above += e < nv && (k & pmask) > prefix;
            bins[e] = in ? static_cast<int>((k >> shift) & uint64_t(nbins - 1)) : -1;
            inm |= static_cast<uint32_t>(in) << e;
        }
        if (collect) {
            // keys above the collected prefix are above K*: count them per
            // chunk (a warp's 32 groups lie in one 4096-chunk)
            const int wsum = __reduce_add_sync(act, above);
            if (wsum && (threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(&p.cnt[(gi * 8) / kChunk].x, wsum);
        }
        if (!__any_sync(act, inm != 0)) continue;  // later digits: few keys share the prefix
        if constexpr (PRIV) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (bins[e] >= 0) atomicAdd(&h[bins[e]], 1u);
        } else {
            // one atomic per distinct bin per warp (keys crowd a few exponent bins)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned peers = __match_any_sync(act, bins[e]);
                if (bins[e] >= 0 && (__ffs(peers) - 1) == (threadIdx.x & 31)) atomicAdd(&h[bins[e]], __popc(peers));
            }
        }
        if (collect) {
            const int n = __popc(inm);
            int incl = n;  // warp-aggregated slot reservation
            const int lane = threadIdx.x & 31;
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(act, incl, off);
                if (lane >= off && ((act >> (lane - off)) & 1u)) incl += t;
            }
            const int last = 31 - __clz(act);
            const int tot = __shfl_sync(act, incl, last);
            unsigned base = 0;
            if (lane == last) base = atomicAdd(p.cand_n, static_cast<unsigned>(tot));
            base = __shfl_sync(act, base, last) + static_cast<unsigned>(incl - n);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if ((inm >> e) & 1u) {
                    if (base < p.cand_cap) {
                        p.cand[base] = key_of(a[e]);
                        p.cand_idx[base] = gi * 8 + e;
                    }
                    ++base;
                }
        }
    }
    if (bad && p.check_finite) atomicOr(p.flag, 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) {
        uint32_t v = 0;
        if constexpr (PRIV) {
            for (int w = 0; w < kThreads / 32; ++w) v += s_hw[w * 2048 + i];
        } else {
            v = s_h1[i];
        }
        if (v) atomicAdd(&p.hist[i], v);
    }
}

template <int NT = kThreads>
__device__ __forceinline__ int cta_excl_scan(int v, int* s_tmp, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) s_tmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        int x = lane < NT / 32 ? s_tmp[lane] : 0;
        int xi = x;
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, xi, off);
            if (lane >= off) xi += t;
        }
        if (lane < NT / 32) s_tmp[lane] = xi - x;
        if (lane == NT / 32 - 1) s_tmp[32] = xi;
    }
    __syncthreads();
    total = s_tmp[32];
    const int r = s_tmp[w] + incl - v;
    __syncthreads();
    return r;
}

// Counts of keys > K* and == K* per chunk.
__global__ void g_count(GlobalArgs p, int64_t nch) {
    __shared__ int s_tmp[33];
    if (*p.cand_n <= p.cand_cap) return;  // g_count_cand: the collect pass counted
    const uint64_t kstar = p.sel_state[0];
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {  // persistent: cheap when skipped
        const int64_t e0 = c * kChunk + int64_t(threadIdx.x) * kPer;
        int gt = 0, eq = 0;
        for (int h = 0; h < kPer / 8; ++h) {
            if (e0 + 8 * h >= p.dim) break;
            double a[8];
            const int nv = g_a8(p, e0 + 8 * h, a);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint64_t k = key_of(a[e]);
                gt += e < nv && k > kstar;
                eq += e < nv && k == kstar;
            }
        }
        int tg, te;
        cta_excl_scan(gt, s_tmp, tg);
        cta_excl_scan(eq, s_tmp, te);
        if (threadIdx.x == 0) p.cnt[c] = make_int2(tg, te);
    }
}

// Selected entries of a chunk at their global row positions, ascending index.
// Thread t owns the 16 consecutive elements [c0 + 16 t, c0 + 16 t + 16).
__global__ void g_emit(GlobalArgs p) {
    __shared__ int s_tmp[33];
    const int64_t c0 = int64_t(blockIdx.x) * kChunk;
    const int64_t e0 = c0 + int64_t(threadIdx.x) * kPer;
    const int2 cs = p.sel_info[blockIdx.x];  // (row offset, ties to take in this chunk)
    if (threadIdx.x == 0) {  // the new row's chunk bounds (what g_bounds would find)
        const int64_t nch = global_chunks_d(p.dim);
        int32_t* bd = p.bounds + int64_t(p.slot) * (nch + 1);
        bd[blockIdx.x] = cs.x;
        if (blockIdx.x == nch - 1) bd[nch] = static_cast<int32_t>(p.k);
    }
    uint32_t gtm = 0, eqm = 0;
    const uint64_t kstar = p.sel_state[0];
    double av[kPer];
#pragma unroll
    for (int h = 0; h < kPer / 8; ++h) {
        double a8[8];
        const int nv = e0 + 8 * h < p.dim ? g_a8(p, e0 + 8 * h, a8) : 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int j = 8 * h + e;
            av[j] = e < nv ? a8[e] : 0.0;
            const uint64_t k = key_of(av[j]);
            gtm |= static_cast<uint32_t>(e < nv && k > kstar) << j;
            eqm |= static_cast<uint32_t>(e < nv && k == kstar) << j;
        }
    }
    int te;
    int tie_before = cta_excl_scan(__popc(eqm), s_tmp, te);
    uint32_t selm = gtm;
    for (int j = 0; j < kPer; ++j)
        if ((eqm >> j) & 1u) {
            if (tie_before < cs.y) selm |= 1u << j;
            ++tie_before;
        }
    int tot;
    int pos = cs.x + cta_excl_scan(__popc(selm), s_tmp, tot);
    int64_t* ri = p.win_idx + int64_t(p.slot) * p.row_stride;
    for (int j = 0; j < kPer; ++j)
        if ((selm >> j) & 1u) {
            ri[pos] = e0 + j;
            st_val(p.win_val, p.v_dtype, int64_t(p.slot) * p.row_stride + pos, av[j]);
            ++pos;
        }
    if (e0 < p.dim) p.selbits[e0 / kPer] = static_cast<uint16_t>(selm);
}

// Re-quantization for 8 <= B_q <= 256 with the elements in registers: thread
// t of a chunk holds the 8-groups t and t + 256, a bucket spans B_q / 8
// consecutive threads (shuffle min/max), codes packed 8 to a word. Same
// arithmetic and IEEE-quotient guard as g_requant.
//
// EMIT: G3 fused in (one pass over d fewer): the selection of the chunk is
// decided here from the keys (> K*, or == K* among the first ties of the
// chunk's quota, index order: the 8-groups of h = 0 then h = 1, thread order
// within) and written to the window row at the chunk's row offset, exactly as
// g_emit writes it.
template <int LPB, bool EMIT>
__global__ void __launch_bounds__(kThreads, 4) g_requant8(GlobalArgs p, int64_t chunk0) {
    __shared__ double s_red[kThreads / 32][4];
    __shared__ int s_tmp[33];
    const int64_t cb = chunk0 + blockIdx.x;  // this CTA's chunk
    const int64_t c0 = cb * kChunk;
    double rep[4] = {0.0, 0.0, 0.0, 0.0};
    int2 cs = make_int2(0, 0);
    uint64_t kstar = 0;
    if constexpr (EMIT) {
        cs = p.sel_info[cb];  // (row offset, ties to take in this chunk)
        kstar = p.sel_state[0];
    }
    int64_t* ri = p.win_idx + int64_t(p.slot) * p.row_stride;
    if (EMIT && threadIdx.x == 0) {  // the new row's chunk bounds (what g_bounds would find)
        const int64_t nch = global_chunks_d(p.dim);
        int32_t* bd = p.bounds + int64_t(p.slot) * (nch + 1);
        bd[cb] = cs.x;
        if (cb == nch - 1) bd[nch] = static_cast<int32_t>(p.k);
    }
#pragma unroll kRq8Unroll
    for (int h = 0; h < kChunk / (8 * kThreads); ++h) {
        const int64_t i0 = c0 + 8 * (int64_t(threadIdx.x) + int64_t(h) * kThreads);
        double a[8];
        const int nv = i0 < p.dim ? g_a8(p, i0, a) : 0;
        uint32_t sw;
        if constexpr (EMIT) {
            // high words first: keys whose high word is below K*'s are below it
            const uint32_t ks_hi = static_cast<uint32_t>(kstar >> 32);
            uint32_t maybe = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                maybe |= static_cast<uint32_t>((static_cast<uint32_t>(__double2hiint(a[e])) & 0x7FFFFFFFu) >= ks_hi) << e;
            if (nv < 8) maybe &= (1u << nv) - 1u;
            uint32_t gtm = 0, eqm = 0;
            if (maybe) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint64_t k = key_of(a[e]);
                    gtm |= static_cast<uint32_t>(k > kstar) << e;
                    eqm |= static_cast<uint32_t>(k == kstar) << e;
                }
                gtm &= maybe;
                eqm &= maybe;
            }
            // one scan of (above, ties) packed in 16-bit halves (<= 2048 each);
            // a second only in the chunk holding ties at K*
            int both;
            const int pre = cta_excl_scan(__popc(gtm) | (__popc(eqm) << 16), s_tmp, both);
            const int te = both >> 16;
            sw = gtm;
            int tot = both & 0xFFFF;
            int pos = cs.x + (pre & 0xFFFF);
            if (te) {
                int tie_before = pre >> 16;
                for (uint32_t m = eqm; m; m &= m - 1) {
                    if (tie_before < cs.y) sw |= m & (0u - m);
                    ++tie_before;
                }
                pos = cs.x + cta_excl_scan(__popc(sw), s_tmp, tot);
            }
            for (uint32_t m = sw; m; m &= m - 1) {
                const int e = __ffs(m) - 1;
                ri[pos] = i0 + e;
                st_val(p.win_val, p.v_dtype, int64_t(p.slot) * p.row_stride + pos, a[e]);
                ++pos;
            }
            cs.x += tot;
            cs.y -= te;
        } else {
            sw = nv ? (p.selbits[i0 / kPer] >> (i0 % kPer)) & 0xFFu : 0u;
        }
        double lo = CUDART_INF, hi = -CUDART_INF;
        if (p.partials) {
            for (int e = 0; e < nv; ++e) {
                const double r = ((sw >> e) & 1u) ? 0.0 : a[e];
                const double g = ld_val(p.grads, p.g_dtype, i0 + e);
                rep[0] += g * g;
                rep[1] += a[e] * a[e];
                rep[2] += r * r;
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = ((sw >> e) & 1u) ? 0.0 : a[e];
        if (nv == 8) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                lo = a[e] < lo ? a[e] : lo;
                hi = a[e] > hi ? a[e] : hi;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (e < nv) {
                    lo = a[e] < lo ? a[e] : lo;
                    hi = a[e] > hi ? a[e] : hi;
                }
        }
#pragma unroll
        for (int off = 1; off < LPB; off <<= 1) {
            const double ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
            const double oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
            lo = ol < lo ? ol : lo;
            hi = oh > hi ? oh : hi;
        }
        if (nv == 0) continue;
        // code = clamp(floor((r - lo) / level + 0.5)) (quantize.cpp:42-55): one
        // DFMA forms 2^24 + t + 0.5 + 2^-15 with t = (r - lo) * 15 / (hi - lo)
        // to fp32 accuracy; its low word holds the code in bits 28..31. A
        // fraction within 2^-14 of an integer sends the group to the IEEE
        // quotient (same bound as the blockwise lean kernel, ma_warp.cu pass 2).
        const double rng = __dsub_rn(hi, lo);
        uint32_t word = 0;
        if (rng != 0.0) {
            const float r32 = __double2float_rn(rng);
            bool bad = true;
            if (r32 >= 0x1p-100f && r32 <= 0x1p100f) {
                const double k64 = static_cast<double>(__fdividef(15.0f, r32));
                const double add = 0x1p24 + 0.5 + 0x1p-15;
                bad = false;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    const uint32_t y = static_cast<uint32_t>(__double_as_longlong(__fma_rn(__dsub_rn(a[e], lo), k64, add)));
                    word = __funnelshift_l(y, word, 4);
                    bad |= e < nv && (y << 4) < (2u << 17);
                }
            }
            if (bad) {
                const double level = __ddiv_rn(rng, 15.0);
                word = 0;
                for (int e = 7; e >= 0; --e) {
                    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(a[e], lo), level), 0.5));
                    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                    word = (word << 4) | static_cast<uint32_t>(f);
                }
            }
        }
        if (nv < 8) word &= (1u << (4 * nv)) - 1u;  // padding nibbles stay 0
        if (p.partials) {
            const double level = rng == 0.0 ? 0.0 : __ddiv_rn(rng, 15.0);
            for (int e = 0; e < nv; ++e) {
                const double en = __dadd_rn(__dmul_rn(static_cast<double>((word >> (4 * e)) & 15u), level), lo);
                rep[3] += en * en;
            }
        }
        if (nv == 8) {
            *reinterpret_cast<uint32_t*>(p.codes + (i0 >> 1)) = word;
        } else {
            for (int b = 0; 2 * b < nv; ++b) p.codes[(i0 >> 1) + b] = static_cast<uint8_t>(word >> (8 * b));
        }
        if ((threadIdx.x & (LPB - 1)) == 0) p.meta[i0 >> p.bucket_shift] = make_double2(lo, hi);
    }
    if (p.partials) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int f = 0; f < 4; ++f) {
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) s_red[w][f] = rep[f];
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            double sum = 0.0;
            for (int w2 = 0; w2 < kThreads / 32; ++w2) sum += s_red[w2][threadIdx.x];
            p.partials[cb * kReportFields + threadIdx.x] = sum;
        }
    }
}

// g_requant8<L, true> in fp32 with exact fallbacks, for whole chunks of bf16
// gradients (no StepReport): the blockwise lean kernel's pass-2 argument
// (ma_warp.cu, above exact_bucket16) on this kernel's layout (thread t owns
// the 8-groups t and t + 256, a bucket spans LPB threads).
//   a32 = rn(g + fma(c, rn(level), rn(lo))) is within E_q + |a32| 2^-23 of
//   the fp64 a (E_q = M 2^-21 + 2^-120, M = max(|lo|, |hi|) of the bucket's
//   previous grid; M >= 2^100: E_q = inf, the bucket goes exact).
//   * Selection: |a| >= K* implies |a32| >= Tf = rd((K* - E_q)(1 - 2^-22));
//     only those elements are decoded in fp64 and compared with K* exactly.
//   * Residual min / max, 4-bit codes: y = rn(r32 k2 + c2) = 257 + 2T + [0, 2G]
//     (T = 15 (r - lo') / (hi' - lo')); byte 2 of y is the code unless y's
//     fraction is below 2G: N = 1 / 31 mark the candidates of the exact
//     minimum / maximum, even N a code boundary (IEEE quotient, quantize.cpp:
//     51-53). Buckets the bound cannot settle take the fp64 path of
//     g_requant8 (same operation order, so the same ties and codes).
// one element's a in the reference's arithmetic, out of line (rare calls)
__device__ __noinline__ double g_a1(const GlobalArgs* p, int64_t i) { return g_a(*p, i); }

template <int LPB>
__global__ void __launch_bounds__(kThreads, 4) g_requant8f(GlobalArgs p) {
    __shared__ int s_tmp[33];
    __shared__ int s_kmag[kThreads / 32];
    s_kmag[threadIdx.x >> 5] = 0x4B000000;  // opaque_kmag's word, one per warp (each lane reads its own store)
    const int64_t cb = blockIdx.x, c0 = cb * kChunk;
    int2 cs = p.sel_info[cb];  // (row offset, ties to take in this chunk)
    const uint64_t kstar = p.sel_state[0];
    const double kd = __longlong_as_double(static_cast<long long>(kstar));
    int64_t* ri = p.win_idx + int64_t(p.slot) * p.row_stride;
    if (threadIdx.x == 0) {  // the new row's chunk bounds (what g_bounds would find)
        const int64_t nch = global_chunks_d(p.dim);
        int32_t* bd = p.bounds + int64_t(p.slot) * (nch + 1);
        bd[cb] = cs.x;
        if (cb == nch - 1) bd[nch] = static_cast<int32_t>(p.k);
    }
    const unsigned lane = threadIdx.x & 31u;
    const unsigned bm = LPB >= 32 ? 0xFFFFFFFFu : (((1u << LPB) - 1u) << (lane & ~(LPB - 1u)));  // the bucket's lanes
#pragma unroll 1
    for (int h = 0; h < kChunk / (8 * kThreads); ++h) {
        const int64_t i0 = c0 + 8 * (int64_t(threadIdx.x) + int64_t(h) * kThreads);
        const int64_t q = i0 >> p.bucket_shift;
        const double2 mt = p.meta[q];
        const double lv = p.level[q];
        const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p.grads) + i0);
        const uint32_t cw = *reinterpret_cast<const uint32_t*>(p.codes + (i0 >> 1));
        // one element's exact a from the registers (g_a: optim.cpp:166-168, quantize.cpp:164-178)
        auto exact_a = [&](int e) -> double {
            const int wi = e >> 1;
            const uint32_t wv = wi == 0 ? v.x : (wi == 1 ? v.y : (wi == 2 ? v.z : v.w));
            const float g = __uint_as_float((e & 1) ? (wv & 0xFFFF0000u) : (wv << 16));
            const double c = static_cast<double>((cw >> (4 * e)) & 15u);
            return __dadd_rn(static_cast<double>(g), __dadd_rn(__dmul_rn(c, lv), mt.x));
        };
        const double M = fmax(fabs(mt.x), fabs(mt.y));
        float E = __double2float_ru(__dadd_ru(__dmul_ru(M, 0x1p-21), 0x1p-120));
        if (!(M < 0x1p100)) E = CUDART_INF_F;
        // a32 of the 8 elements
        float a32[8];
        {
            const float2 lv2 = make_float2(__double2float_rn(lv), __double2float_rn(lv));
            const float2 lo2 = make_float2(__double2float_rn(mt.x), __double2float_rn(mt.x));
            const float2 m23 = make_float2(-8388608.0f, -8388608.0f);
            const uint32_t ce = cw & 0x0F0F0F0Fu, co = (cw >> 4) & 0x0F0F0F0Fu;
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            const uint32_t kmag = opaque_kmag(&s_kmag[threadIdx.x >> 5]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2 c2 = make_float2(__uint_as_float(__byte_perm(ce, kmag, 0x7540u | k)),
                                        __uint_as_float(__byte_perm(co, kmag, 0x7540u | k)));
                c2 = __fadd2_rn(c2, m23);
                const float2 a2 = __fadd2_rn(make_float2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xFFFF0000u)),
                                             __ffma2_rn(c2, lv2, lo2));
                a32[2 * k] = a2.x;
                a32[2 * k + 1] = a2.y;
            }
        }
        // ---- selection (compress.cpp:39-53 over the whole vector) + emit ----
        float tf = __double2float_rd(__dmul_rd(__dsub_rd(kd, static_cast<double>(E)), 1.0 - 0x1p-22));
        if (!(tf > 0.0f)) tf = 0.0f;
        uint32_t maybe = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) maybe |= static_cast<uint32_t>(!(fabsf(a32[e]) < tf)) << e;
        uint32_t gtm = 0, eqm = 0;
        for (uint32_t m = maybe; m; m &= m - 1) {
            const int e = __ffs(m) - 1;
            const uint64_t k = key_of(exact_a(e));
            gtm |= static_cast<uint32_t>(k > kstar) << e;
            eqm |= static_cast<uint32_t>(k == kstar) << e;
        }
        int both;
        const int pre = cta_excl_scan(__popc(gtm) | (__popc(eqm) << 16), s_tmp, both);
        const int te = both >> 16;
        uint32_t sw = gtm;
        int tot = both & 0xFFFF;
        int pos = cs.x + (pre & 0xFFFF);
        if (te) {
            int tie_before = pre >> 16;
            for (uint32_t m = eqm; m; m &= m - 1) {
                if (tie_before < cs.y) sw |= m & (0u - m);
                ++tie_before;
            }
            pos = cs.x + cta_excl_scan(__popc(sw), s_tmp, tot);
        }
        for (uint32_t m = sw; m; m &= m - 1) {
            const int e = __ffs(m) - 1;
            ri[pos] = i0 + e;
            st_val(p.win_val, p.v_dtype, int64_t(p.slot) * p.row_stride + pos, exact_a(e));
            ++pos;
        }
        cs.x += tot;
        cs.y -= te;
        // ---- residual (compress.cpp:95-102) + re-quantization (quantize.cpp:15-24, 42-55) ----
        float r32[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) r32[e] = ((sw >> e) & 1u) ? 0.0f : a32[e];
        float mn = fminf(fminf(fminf(r32[0], r32[1]), fminf(r32[2], r32[3])), fminf(fminf(r32[4], r32[5]), fminf(r32[6], r32[7])));
        float mx = fmaxf(fmaxf(fmaxf(r32[0], r32[1]), fmaxf(r32[2], r32[3])), fmaxf(fmaxf(r32[4], r32[5]), fmaxf(r32[6], r32[7])));
#pragma unroll
        for (int off = 1; off < LPB; off <<= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, off));
            mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
        }
        const float eps = __fmaf_ru(fmaxf(fabsf(mn), fabsf(mx)), 0x1p-23f, E);
        const float R = __fsub_rd(mx, mn);
        const float den = __fsub_rd(R, 2.0f * eps);
        const float k2 = __fdividef(30.0f, R);
        const float cmag = 258.0f + fabsf(mn * k2);
        const float G = __fmaf_ru(128.0f, __fdividef(eps, den), __fmaf_ru(cmag, 0x1p-23f, 0x1p-13f));
        const bool fast = R >= 0x1p-100f && R <= 0x1p100f && den > 0.0f && G <= 0.0625f;  // bucket-uniform
        uint32_t word = 0, bnd = 0;
        bool bad = false;
        double lmin = CUDART_INF, lmax = -CUDART_INF;
        if (fast) {
            const float c2 = __fmaf_rn(-mn, k2, 257.0f + G);
            const uint32_t Gu = static_cast<uint32_t>(__fmaf_ru(2.0f, G, 0x1p-13f) * 32768.0f) + 1u;
            uint32_t yb[8];
            const float2 k22 = make_float2(k2, k2), c22 = make_float2(c2, c2);
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const float2 y = __ffma2_rn(make_float2(r32[e], r32[e + 1]), k22, c22);
                yb[e] = __float_as_uint(y.x);
                yb[e + 1] = __float_as_uint(y.y);
            }
            {
                const uint32_t ev = __byte_perm(__byte_perm(yb[0], yb[2], 0x0062u), __byte_perm(yb[4], yb[6], 0x0062u), 0x5410u);
                const uint32_t od = __byte_perm(__byte_perm(yb[1], yb[3], 0x0062u), __byte_perm(yb[5], yb[7], 0x0062u), 0x5410u);
                word = (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
            }
            uint32_t fl = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) fl |= static_cast<uint32_t>((yb[e] & 0x7FFFu) < Gu) << e;
            for (uint32_t m = fl; m; m &= m - 1) {  // min / max candidates and code boundaries (~2 per bucket)
                const int e = __ffs(m) - 1;
                uint32_t ye = yb[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) ye = k == e ? yb[k] : ye;
                const uint32_t N = (ye >> 15) & 0xFFu;
                const double rx = ((sw >> e) & 1u) ? 0.0 : exact_a(e);
                bad |= N == 0u || N > 31u;
                lmin = (N == 1u && rx < lmin) ? rx : lmin;
                lmax = (N == 31u && rx > lmax) ? rx : lmax;
                bnd |= static_cast<uint32_t>((N & 1u) == 0u && N - 1u < 31u) << e;
            }
        }
#pragma unroll
        for (int off = 1; off < LPB; off <<= 1) {  // the bucket's exact extremes
            const double ol = __shfl_xor_sync(0xFFFFFFFFu, lmin, off), oh = __shfl_xor_sync(0xFFFFFFFFu, lmax, off);
            lmin = ol < lmin ? ol : lmin;
            lmax = oh > lmax ? oh : lmax;
            bad |= __shfl_xor_sync(0xFFFFFFFFu, static_cast<int>(bad), off) != 0;
        }
        bad = bad || !fast || !(lmin < CUDART_INF) || !(lmax > -CUDART_INF);  // bucket-uniform
        double lo = lmin, hi = lmax;
        if (bad) {  // the fp64 path of g_requant8 for this bucket (its lanes: bm)
            double a[8];
            g_a8(p, i0, a);
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = ((sw >> e) & 1u) ? 0.0 : a[e];
            lo = CUDART_INF;
            hi = -CUDART_INF;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                lo = a[e] < lo ? a[e] : lo;
                hi = a[e] > hi ? a[e] : hi;
            }
#pragma unroll
            for (int off = 1; off < LPB; off <<= 1) {
                const double ol = __shfl_xor_sync(bm, lo, off);
                const double oh = __shfl_xor_sync(bm, hi, off);
                lo = ol < lo ? ol : lo;
                hi = oh > hi ? oh : hi;
            }
            const double rng = __dsub_rn(hi, lo);
            word = 0;
            if (rng != 0.0) {
                const double level = __ddiv_rn(rng, 15.0);
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(a[e], lo), level), 0.5));
                    f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                    word = (word << 4) | static_cast<uint32_t>(f);
                }
            }
        } else if (bnd) {  // rare: quotients within the guard band of a code boundary
            const double level = __ddiv_rn(__dsub_rn(hi, lo), 15.0);
            for (uint32_t m = bnd; m; m &= m - 1) {
                const int e = __ffs(m) - 1;
                const double rx = ((sw >> e) & 1u) ? 0.0 : exact_a(e);
                double f = floor(__dadd_rn(__ddiv_rn(__dsub_rn(rx, lo), level), 0.5));
                f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                word = (word & ~(15u << (4 * e))) | (static_cast<uint32_t>(f) << (4 * e));
            }
        }
        // every lane of the bucket is done reading the previous grid (g_a) before
        // its first lane overwrites it
        __syncwarp();
        *reinterpret_cast<uint32_t*>(p.codes + (i0 >> 1)) = word;
        if ((threadIdx.x & (LPB - 1)) == 0) p.meta[q] = make_double2(lo, hi);
    }
}

// Lossless error feedback (optim.cpp:172-173): the residual of the selection
// is the new error, kept dense in fp64 (read before it is overwritten: each
// thread owns its elements); report sums.
__global__ void g_residual_dense(GlobalArgs p) {
    __shared__ double s_red[kThreads / 32][4];
    const int64_t c0 = int64_t(blockIdx.x) * kChunk;
    double rep[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = threadIdx.x; j < kChunk; j += kThreads) {
        const int64_t i = c0 + j;
        if (i >= p.dim) break;
        const double g = ld_val(p.grads, p.g_dtype, i);
        const double a = __dadd_rn(g, p.dense[i]);
        const bool s = (p.selbits[i / kPer] >> (i % kPer)) & 1u;
        const double r = s ? 0.0 : a;
        p.dense[i] = r;
        rep[0] += g * g;
        rep[1] += a * a;
        rep[2] += r * r;
        rep[3] += r * r;
    }
    if (p.partials) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int f = 0; f < 4; ++f) {
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) s_red[w][f] = rep[f];
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            double sum = 0.0;
            for (int w2 = 0; w2 < kThreads / 32; ++w2) sum += s_red[w2][threadIdx.x];
            p.partials[int64_t(blockIdx.x) * kReportFields + threadIdx.x] = sum;
        }
    }
}

// Residual, bucket (lo, hi), 4-bit codes by the IEEE quotient; report sums.
__global__ void g_requant(GlobalArgs p) {
    extern __shared__ double s_a[];  // kChunk residuals
    __shared__ double s_red[kThreads / 32][4];
    const int64_t c0 = int64_t(blockIdx.x) * kChunk;
    const int n = static_cast<int>(p.dim - c0 < kChunk ? p.dim - c0 : kChunk);
    double rep[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j0 = 8 * threadIdx.x; j0 < n; j0 += 8 * kThreads) {
        double a8[8];
        const int64_t i0 = c0 + j0;
        const int nv = g_a8(p, i0, a8);
        const uint32_t sw = (p.selbits[i0 / kPer] >> (i0 % kPer)) & 0xFFu;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (e >= nv) break;
            const double a = a8[e];
            const double r = ((sw >> e) & 1u) ? 0.0 : a;
            s_a[j0 + e] = r;
            if (p.partials) {
                const double g = ld_val(p.grads, p.g_dtype, i0 + e);
                rep[0] += g * g;
                rep[1] += a * a;
                rep[2] += r * r;
            }
        }
    }
    __syncthreads();
    // buckets inside this chunk (kChunk % bucket == 0): 8 threads per bucket
    // reduce (lo, hi) (quant_params, quantize.cpp:15-24), one writes the grid
    const int B = static_cast<int>(p.bucket);
    const int nqmax = kChunk >> p.bucket_shift;  // buckets per chunk (bucket | 4096)
    double* s_lo = reinterpret_cast<double*>(s_a + kChunk);
    double* s_lv = s_lo + nqmax;
    double* s_ri = s_lv + nqmax;  // rn(1 / level) (0 when the division decides)
    const int nq = (n + B - 1) / B;
    for (int q0 = threadIdx.x / 8; q0 < ((nq + 31) / 32) * 32; q0 += kThreads / 8) {
        const int q = q0, sub = threadIdx.x & 7;
        double lo = 0.0, hi = 0.0;
        bool any = false;
        if (q < nq) {
            const int j0 = q * B, j1 = j0 + B < n ? j0 + B : n;
            for (int j = j0 + sub; j < j1; j += 8) {
                const double x = s_a[j];
                if (!any) {
                    lo = hi = x;
                    any = true;
                } else {
                    lo = x < lo ? x : lo;
                    hi = x > hi ? x : hi;
                }
            }
        }
        for (int off = 1; off < 8; off <<= 1) {  // lanes of a bucket are 8 consecutive threads
            const double ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
            const double oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
            const bool oa = __shfl_xor_sync(0xFFFFFFFFu, any, off);
            if (oa && (!any || ol < lo)) lo = ol;
            if (oa && (!any || oh > hi)) hi = oh;
            any = any || oa;
        }
        if (q < nq && sub == 0) {
            p.meta[(c0 >> p.bucket_shift) + q] = make_double2(lo, hi);
            s_lo[q] = lo;
            const double lv = lo == hi ? 0.0 : __ddiv_rn(__dsub_rn(hi, lo), 15.0);
            s_lv[q] = lv;
            s_ri[q] = lv >= 0x1p-1000 ? __drcp_rn(lv) : 0.0;
        }
    }
    __syncthreads();
    // codes: thread t packs bytes (2 elements each); floor((x - lo) * (1/level) + 0.5)
    // equals the IEEE quotient's unless it lands within 1e-12 of an integer,
    // where the division decides (quantize.cpp:51-53)
    for (int jb = threadIdx.x; jb * 2 < n; jb += kThreads) {
        uint32_t byte = 0;
        for (int h = 0; h < 2; ++h) {
            const int j = jb * 2 + h;
            if (j >= n) break;
            const int q = j >> p.bucket_shift;
            const double level = s_lv[q];
            uint32_t c = 0;
            if (level != 0.0) {
                const double d = __dsub_rn(s_a[j], s_lo[q]);
                const double ri = s_ri[q];
                double f = 0.0;
                if (ri != 0.0) {
                    const double t = __dadd_rn(__dmul_rn(d, ri), 0.5);
                    f = floor(t);
                    const double fr = __dsub_rn(t, f);
                    if (fr < 1e-12 || fr > 1.0 - 1e-12) f = floor(__dadd_rn(__ddiv_rn(d, level), 0.5));
                } else {
                    f = floor(__dadd_rn(__ddiv_rn(d, level), 0.5));
                }
                f = f < 0.0 ? 0.0 : (f > 15.0 ? 15.0 : f);
                c = static_cast<uint32_t>(f);
            }
            byte |= c << (4 * h);
            if (p.partials) {
                const double en = __dadd_rn(__dmul_rn(static_cast<double>(c), level), s_lo[q]);
                rep[3] += en * en;
            }
        }
        p.codes[(c0 >> 1) + jb] = static_cast<uint8_t>(byte);
    }
    if (p.partials) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int f = 0; f < 4; ++f) {
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) s_red[w][f] = rep[f];
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            double s = 0.0;
            for (int w2 = 0; w2 < kThreads / 32; ++w2) s += s_red[w2][threadIdx.x];
            p.partials[int64_t(blockIdx.x) * kReportFields + threadIdx.x] = s;
        }
    }
}

// Window entries of each chunk: rows are ascending (the emit order, and
// SparseSelection::validate for loaded checkpoints), so bounds[r][c] = first
// entry j of row r with idx >= c·kChunk, for c in [0, nch]; each entry writes
// the bounds of the chunks between its predecessor's and its own.
__global__ void g_bounds(GlobalArgs p, int filled) {
    const int64_t nch = global_chunks_d(p.dim);
    const int64_t n = int64_t(filled) * p.k;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = t / p.k, j = t - r * p.k;
        const int64_t* ri = p.win_idx + r * p.row_stride;
        int32_t* bd = p.bounds + r * (nch + 1);
        const int64_t c = ri[j] / kChunk;
        const int64_t cp = j > 0 ? ri[j - 1] / kChunk : -1;
        for (int64_t cc = cp + 1; cc <= c; ++cc) bd[cc] = static_cast<int32_t>(j);
        if (j == p.k - 1)
            for (int64_t cc = c + 1; cc <= nch; ++cc) bd[cc] = static_cast<int32_t>(p.k);
    }
}

// Every row's entry range of chunk c (one memory latency): s_j0[r] = first
// entry, s_off = exclusive prefix of the per-row counts. Returns the total.
__device__ __forceinline__ int chunk_rows(const GlobalArgs& p, int64_t c, int filled, int* s_j0, int* s_off) {
    const int64_t nch = global_chunks_d(p.dim);
    for (int r = threadIdx.x; r < filled; r += blockDim.x) {
        const int32_t* bd = p.bounds + int64_t(r) * (nch + 1);
        s_j0[r] = bd[c];
        s_off[r + 1] = bd[c + 1] - bd[c];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_off[0] = 0;
        for (int r = 0; r < filled; ++r) s_off[r + 1] += s_off[r];
    }
    __syncthreads();
    return s_off[filled];
}

// θ -= lr · (z1 s1) / (eps + sqrt(z2 s2)) at element i (optim.cpp:183-187).
__device__ __forceinline__ void g_apply(const GlobalArgs& p, int64_t i, double z1, double z2, double& nnz) {
    const double mhat = __dmul_rn(z1, p.scale1);
    const double vhat = __dmul_rn(z2, p.scale2);
    const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
    if (u != 0.0) nnz += 1.0;
    const double th = ld_val(p.params, p.p_dtype, i);
    st_val(p.params, p.p_dtype, i, __dsub_rn(th, __dmul_rn(p.lr, u)));
}

__device__ __forceinline__ void g_nnz_partial(const GlobalArgs& p, int64_t c, double nnz, double* s_red) {
    if (!p.partials) return;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    for (int off = 16; off > 0; off >>= 1) nnz += __shfl_xor_sync(0xFFFFFFFFu, nnz, off);
    if (lane == 0) s_red[wi] = nnz;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int w2 = 0; w2 < static_cast<int>(blockDim.x / 32); ++w2) sum += s_red[w2];
        p.partials[c * kReportFields + 4] = sum;
    }
    __syncthreads();
}

// ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) for one 4096-
// element chunk without dense accumulators: the chunk's window entries (a few
// hundred: rows ascending, bounds found once per step) are staged in shared
// memory; each coordinate's owner is its entry in the earliest row (atomicMin
// over entry indices), the rows are summed into per-owner accumulators in
// physical slot order — z += w·v, z += w·v², the reference's fp64 operation
// order — and owners apply the update to the chunk's θ staged in shared
// memory. Chunks with more than kStage entries go to an overflow list for
// g_stats_update_dense.
__global__ void g_stats_update(GlobalArgs p, const __grid_constant__ GWeights w, int filled) {
    extern __shared__ uint4 s_th4[];  // the chunk's θ, staged with 16-byte loads
    __shared__ double s_red[kThreads / 32];
    __shared__ int s_j0[kMaxWindowGlobal], s_off[kMaxWindowGlobal + 1];
    __shared__ int16_t s_ei[kStage];
    __shared__ double s_ev[kStage];
    __shared__ double s_z1[kStage], s_z2[kStage];  // per owner entry
    __shared__ int s_first[kChunk];                // owner entry per coordinate (touched ones)
    const int64_t c = blockIdx.x, c0 = c * kChunk;
    const int psz = p.p_dtype == F64 ? 8 : (p.p_dtype == F32 ? 4 : 2);
    const int n = static_cast<int>(p.dim - c0 < kChunk ? p.dim - c0 : kChunk);
    // θ of the chunk, coalesced: ~10% of it is updated, but at that density
    // nearly every 32-byte sector is touched, so a scattered update moves the
    // same bytes with a dependent load per element
    const bool vec = n == kChunk && (reinterpret_cast<uintptr_t>(p.params) & 15u) == 0;
    const int nv16 = kChunk * psz / 16;
    if (vec) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(p.params) + c0 * psz);
        for (int t = threadIdx.x; t < nv16; t += kThreads) s_th4[t] = src[t];
    }
    const int total = chunk_rows(p, c, filled, s_j0, s_off);
    if (total > kStage) {
        if (threadIdx.x == 0) p.ovf_list[atomicAdd(p.ovf_n, 1u)] = static_cast<int>(c);
        return;
    }
    for (int e = threadIdx.x; e < total; e += kThreads) {
        int r = 0;
        while (s_off[r + 1] <= e) ++r;
        const int64_t q = int64_t(r) * p.row_stride + s_j0[r] + (e - s_off[r]);
        s_ei[e] = static_cast<int16_t>(p.win_idx[q] - c0);
        s_ev[e] = ld_val(p.win_val, p.v_dtype, q);
    }
    __syncthreads();
    // owner of a coordinate = its entry in the earliest row (entries are
    // concatenated in slot order, so the smallest entry index)
    for (int e = threadIdx.x; e < total; e += kThreads) s_first[s_ei[e]] = 0x7FFF;
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += kThreads) atomicMin(&s_first[s_ei[e]], e);
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += kThreads)
        if (s_first[s_ei[e]] == e) {
            s_z1[e] = 0.0;
            s_z2[e] = 0.0;
        }
    __syncthreads();
    for (int r = 0; r < filled; ++r) {  // slot order: z += w·v, z += w·v² (window.cpp:37-41)
        for (int e = s_off[r] + threadIdx.x; e < s_off[r + 1]; e += kThreads) {
            const int o = s_first[s_ei[e]];
            const double v = s_ev[e];
            s_z1[o] = __dadd_rn(s_z1[o], __dmul_rn(w.w1[r], v));
            s_z2[o] = __dadd_rn(s_z2[o], __dmul_rn(w.w2[r], __dmul_rn(v, v)));
        }
        __syncthreads();
    }
    double nnz = 0.0;
    for (int e = threadIdx.x; e < total; e += kThreads) {
        const int i = s_ei[e];
        if (s_first[i] != e) continue;
        const double z1 = s_z1[e], z2 = s_z2[e];
        if (z1 == 0.0 && z2 == 0.0) continue;
        if (vec) {
            const double mhat = __dmul_rn(z1, p.scale1);
            const double vhat = __dmul_rn(z2, p.scale2);
            const double u = __ddiv_rn(mhat, __dadd_rn(p.eps, __dsqrt_rn(vhat)));
            if (u != 0.0) nnz += 1.0;
            void* th = s_th4;
            st_val(th, p.p_dtype, i, __dsub_rn(ld_val(th, p.p_dtype, i), __dmul_rn(p.lr, u)));
        } else {
            g_apply(p, c0 + i, z1, z2, nnz);
        }
    }
    if (vec) {
        __syncthreads();
        uint4* dst = reinterpret_cast<uint4*>(static_cast<unsigned char*>(p.params) + c0 * psz);
        for (int t = threadIdx.x; t < nv16; t += kThreads) dst[t] = s_th4[t];
    }
    g_nnz_partial(p, c, nnz, s_red);
}

// ADAM_STATS + update for one 4096-chunk, sparse form: coordinates held by one
// window entry (most of them) are updated from that entry alone — z = 0 + w·v,
// z = 0 + w·v² (window.cpp:37-41 with one term) — and the few held by several
// entries are summed in physical slot order by their owner (the entry in the
// earliest row) over the chunk's duplicate list sorted into entry order.
// Chunks with more than kDupList duplicate entries (dense windows) or more
// than kStage entries go to the overflow list (g_stats_update_dense) before
// anything is written.
constexpr int kDupList = 64;
#ifndef MA_STATS_NT
#define MA_STATS_NT 256
#endif
constexpr int kStatsThreads = MA_STATS_NT;  // threads per chunk of g_stats_sparse
template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 7 : 12) g_stats_sparse(GlobalArgs p, const __grid_constant__ GWeights w,
                                                           int filled) {
    extern __shared__ uint4 s_th4[];  // the chunk's θ, staged with 16-byte loads
    __shared__ double s_red[NT / 32];
    __shared__ int s_j0[kMaxWindowGlobal], s_off[kMaxWindowGlobal + 1];
    __shared__ int16_t s_ei[kStage];
    __shared__ uint8_t s_er[kStage];
    __shared__ double s_ev[kStage];
    __shared__ uint32_t s_seen[kChunk / 32], s_dup[kChunk / 32];
    __shared__ int16_t s_dl[kDupList], s_ds[kDupList];
    __shared__ int s_nd;
    const int64_t c = blockIdx.x, c0 = c * kChunk;
    const int psz = p.p_dtype == F64 ? 8 : (p.p_dtype == F32 ? 4 : 2);
    const int n = static_cast<int>(p.dim - c0 < kChunk ? p.dim - c0 : kChunk);
    const bool vec = n == kChunk && (reinterpret_cast<uintptr_t>(p.params) & 15u) == 0;
    // θ of the chunk: one bulk copy (TMA) in flight while the window entries load
    __shared__ __align__(8) uint64_t s_bar;
    if (vec && threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&s_bar, kChunk * psz);
        bulk_g2s(s_th4, static_cast<const unsigned char*>(p.params) + c0 * psz, kChunk * psz, &s_bar);
    }
    auto theta_landed = [&] {
        if (vec)
            while (!mbar_try_wait(&s_bar, 0)) {
            }
    };
    for (int t = threadIdx.x; t < kChunk / 32; t += NT) {
        s_seen[t] = 0;
        s_dup[t] = 0;
    }
    if (threadIdx.x == 0) s_nd = 0;
    const int total = chunk_rows(p, c, filled, s_j0, s_off);  // (synchronises)
    if (total > kStage) {
        if (threadIdx.x == 0) p.ovf_list[atomicAdd(p.ovf_n, 1u)] = static_cast<int>(c);
        theta_landed();  // no bulk copy may still target this CTA's shared memory
        return;
    }
    for (int e = threadIdx.x; e < total; e += NT) {
        int r = 0;
        while (s_off[r + 1] <= e) ++r;
        const int64_t q = int64_t(r) * p.row_stride + s_j0[r] + (e - s_off[r]);
        const int i = static_cast<int>(p.win_idx[q] - c0);
        s_ei[e] = static_cast<int16_t>(i);
        s_er[e] = static_cast<uint8_t>(r);
        s_ev[e] = ld_val(p.win_val, p.v_dtype, q);
        const uint32_t bit = 1u << (i & 31);
        if (atomicOr(&s_seen[i >> 5], bit) & bit) atomicOr(&s_dup[i >> 5], bit);
    }
    __syncthreads();
    int nd_t = 0;
    for (int e = threadIdx.x; e < total; e += NT) nd_t += (s_dup[s_ei[e] >> 5] >> (s_ei[e] & 31)) & 1u;
    nd_t = __reduce_add_sync(0xFFFFFFFFu, nd_t);
    if ((threadIdx.x & 31) == 0 && nd_t) atomicAdd(&s_nd, nd_t);
    __syncthreads();
    const int nd = s_nd;
    if (nd > kDupList) {
        if (threadIdx.x == 0) p.ovf_list[atomicAdd(p.ovf_n, 1u)] = static_cast<int>(c);
        theta_landed();
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_nd = 0;
    theta_landed();
    __syncthreads();
    double nnz = 0.0;
    void* th = s_th4;
    for (int e = threadIdx.x; e < total; e += NT) {
        const int i = s_ei[e];
        if ((s_dup[i >> 5] >> (i & 31)) & 1u) {
            s_dl[atomicAdd(&s_nd, 1)] = static_cast<int16_t>(e);
            continue;
        }
        const int r = s_er[e];
        const double v = s_ev[e];
        const double z1 = __dadd_rn(0.0, __dmul_rn(w.w1[r], v));
        const double z2 = __dadd_rn(0.0, __dmul_rn(w.w2[r], __dmul_rn(v, v)));
        if (z1 == 0.0 && z2 == 0.0) continue;
        if (vec) {
            const double u = __ddiv_rn(__dmul_rn(z1, p.scale1), __dadd_rn(p.eps, __dsqrt_rn(__dmul_rn(z2, p.scale2))));
            if (u != 0.0) nnz += 1.0;
            st_val(th, p.p_dtype, i, __dsub_rn(ld_val(th, p.p_dtype, i), __dmul_rn(p.lr, u)));
        } else {
            g_apply(p, c0 + i, z1, z2, nnz);
        }
    }
    __syncthreads();
    if (threadIdx.x < nd) {  // duplicate list into entry (= slot) order
        const int e = s_dl[threadIdx.x];
        int rank = 0;
        for (int j = 0; j < nd; ++j) rank += s_dl[j] < e;
        s_ds[rank] = static_cast<int16_t>(e);
    }
    __syncthreads();
    if (threadIdx.x < nd) {
        const int e = s_ds[threadIdx.x], i = s_ei[e];
        bool owner = true;
        for (int j = 0; j < static_cast<int>(threadIdx.x); ++j) owner &= s_ei[s_ds[j]] != i;
        if (owner) {
            double z1 = 0.0, z2 = 0.0;
            for (int j = threadIdx.x; j < nd; ++j) {
                const int ej = s_ds[j];
                if (s_ei[ej] != i) continue;
                const int r = s_er[ej];
                const double v = s_ev[ej];
                z1 = __dadd_rn(z1, __dmul_rn(w.w1[r], v));
                z2 = __dadd_rn(z2, __dmul_rn(w.w2[r], __dmul_rn(v, v)));
            }
            if (z1 != 0.0 || z2 != 0.0) {
                if (vec) {
                    const double u =
                        __ddiv_rn(__dmul_rn(z1, p.scale1), __dadd_rn(p.eps, __dsqrt_rn(__dmul_rn(z2, p.scale2))));
                    if (u != 0.0) nnz += 1.0;
                    st_val(th, p.p_dtype, i, __dsub_rn(ld_val(th, p.p_dtype, i), __dmul_rn(p.lr, u)));
                } else {
                    g_apply(p, c0 + i, z1, z2, nnz);
                }
            }
        }
    }
    if (vec) {  // θ back by one bulk copy once every update landed in shared memory
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_s2g(static_cast<unsigned char*>(p.params) + c0 * psz, s_th4, kChunk * psz);
        }
    }
    g_nnz_partial(p, c, nnz, s_red);
    if (vec && threadIdx.x == 0) bulk_wait_read();
}

// Chunks with more window entries than kStage: dense accumulators in shared
// memory, rows in slot order (persistent CTAs over the overflow list).
__global__ void g_stats_update_dense(GlobalArgs p, const __grid_constant__ GWeights w, int filled) {
    extern __shared__ double s_z[];  // [kChunk] z1, [kChunk] z2
    __shared__ double s_red[kThreads / 32];
    __shared__ int s_j0[kMaxWindowGlobal], s_off[kMaxWindowGlobal + 1];
    double* s_z1 = s_z;
    double* s_z2 = s_z + kChunk;
    const unsigned novf = *p.ovf_n;
    for (unsigned o = blockIdx.x; o < novf; o += gridDim.x) {
        const int64_t c = p.ovf_list[o], c0 = c * kChunk;
        chunk_rows(p, c, filled, s_j0, s_off);
        for (int j = threadIdx.x; j < kChunk; j += kThreads) {
            s_z1[j] = 0.0;
            s_z2[j] = 0.0;
        }
        __syncthreads();
        for (int r = 0; r < filled; ++r) {
            const int64_t rb = int64_t(r) * p.row_stride + s_j0[r];
            for (int e = threadIdx.x; e < s_off[r + 1] - s_off[r]; e += kThreads) {
                const int i = static_cast<int>(p.win_idx[rb + e] - c0);
                const double v = ld_val(p.win_val, p.v_dtype, rb + e);
                s_z1[i] = __dadd_rn(s_z1[i], __dmul_rn(w.w1[r], v));
                s_z2[i] = __dadd_rn(s_z2[i], __dmul_rn(w.w2[r], __dmul_rn(v, v)));
            }
            __syncthreads();
        }
        double nnz = 0.0;
        for (int j = threadIdx.x; j < kChunk; j += kThreads) {
            if (c0 + j >= p.dim) break;
            const double z1 = s_z1[j], z2 = s_z2[j];
            if (z1 == 0.0 && z2 == 0.0) continue;
            g_apply(p, c0 + j, z1, z2, nnz);
        }
        g_nnz_partial(p, c, nnz, s_red);
    }
}

// One digit's histogram over the collected candidate keys.
__global__ void g_hist_cand(GlobalArgs p, int shift, int nbins, int early) {
    __shared__ uint32_t h[2048];
    const unsigned n = *p.cand_n;
    if (n > p.cand_cap) return;           // overflowed: the full pass runs instead
    if (early && !p.sel_state[8]) return;  // leading digits: only over a bracket's keys
    const uint64_t prefix = p.sel_state[0], pmask = p.sel_state[1];
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const unsigned n32 = (n + 31u) & ~31u;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += gridDim.x * blockDim.x) {
        const uint64_t k = i < n ? p.cand[i] : 0;
        const int bin = i < n && (k & pmask) == prefix ? static_cast<int>((k >> shift) & uint64_t(nbins - 1)) : -1;
        // one atomic per distinct bin per warp (a bracket's keys crowd a few bins)
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        if (bin >= 0 && (__ffs(peers) - 1) == (threadIdx.x & 31)) atomicAdd(&h[bin], __popc(peers));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
        if (h[i]) atomicAdd(&p.hist[i], h[i]);
}

// Per-chunk (> K*, == K*) counts from the collected keys, on top of the
// above-prefix counts the collecting pass made (unless the buffer overflowed:
// then g_count recounts every chunk).
__global__ void g_count_cand(GlobalArgs p) {
    const unsigned n = *p.cand_n;
    if (n > p.cand_cap) return;
    const uint64_t kstar = p.sel_state[0];
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t k = p.cand[i];
        const int64_t c = p.cand_idx[i] / kChunk;
        if (k > kstar) atomicAdd(&p.cnt[c].x, 1);
        else if (k == kstar) atomicAdd(&p.cnt[c].y, 1);
    }
}

// Carried bracket (one pass over d instead of three): K* moves little from
// step to step, so the keys in [Kc - W, Kc + W] around the previous step's K*
// are collected with their indices and the keys above the bracket only
// counted (per chunk, and in total). When above < k <= above + collected and
// the buffer held them all, the k-th largest key lies in the bracket and the
// six digit picks run over the collected keys alone (g_hist_cand): the same
// exact K* and tie count as the full passes. Otherwise the step falls back to
// the full digit passes (g_bracket_check resets the state). The bracket only
// decides which kernels do the work, never the result.
// sel_state: [5] Kc, [6] W (0: no bracket yet), [7] keys above, [8] bracket ok
__global__ void __launch_bounds__(256, 6) g_bracket(GlobalArgs p, int pass) {
    __shared__ unsigned long long s_above;
    __shared__ unsigned s_cn;  // keys collected into this CTA's segment
    __shared__ int s_kmag[8];
    s_kmag[threadIdx.x >> 5] = 0x4B000000;  // opaque_kmag's word, one per warp (each lane reads its own store)
    if (pass == 0 ? p.sel_state[6] == 0 : p.sel_state[11] == 0) return;  // no bracket yet / no retry
    // [lo, hi] widened to whole 2^32 steps of the key: the tests below read
    // only the high word of |a| (keys >= lo32 << 32 and <= hi32 << 32 | ~0u)
    const uint32_t lo32 = static_cast<uint32_t>(p.sel_state[12] >> 32);
    const uint32_t hi32 = static_cast<uint32_t>(p.sel_state[13] >> 32), span = hi32 - lo32;
    // keys go to this CTA's segment of seg_key / seg_idx, slots taken with a
    // shared-memory counter (a global one serialises every warp in L2)
    const unsigned seg_cap = p.cand_cap / gridDim.x;
    uint64_t* sk = p.seg_key + size_t(blockIdx.x) * seg_cap;
    int64_t* si = p.seg_idx + size_t(blockIdx.x) * seg_cap;
    if (threadIdx.x == 0) {
        s_above = 0;
        s_cn = 0;
    }
    __syncthreads();
    uint32_t mx = 0;  // largest high word: inf / NaN (check_finite in topk_global)
    unsigned above_t = 0;
    const int lane = threadIdx.x & 31;
    const int64_t ngroups = (p.dim + 7) / 8;
    // fp32 screen (bf16 gradients, a bucket holds each 8-group): groups whose
    // 8 keys are certainly below the bracket skip the fp64 decode. a32 =
    // rn(g + rn(c lv32 + lo32)) is within 2^-23 (15|lv| + |lo|) + |a32| 2^-24
    // (x 1.01) of the fp64 a (quantize.cpp:164-178 + optim.cpp:166-168:
    // lv32, lo32, the FFMA and the FADD each round once); a group passes when
    // some |a32| (1 + 2^-22) + 2 (15|lv32| + |lo32|) 2^-22 + 2^-126 >= the
    // bracket's lower end rounded down to fp32, or is NaN.
    const bool scr = p.g_dtype == BF16 && !p.dense && p.bucket_shift >= 3 &&
                     (reinterpret_cast<uintptr_t>(p.grads) & 15u) == 0 && lo32 > 0;
    const float t32 = __double2float_rd(__longlong_as_double(static_cast<long long>(uint64_t(lo32) << 32)));
    for (int64_t gi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; gi < ngroups;
         gi += int64_t(gridDim.x) * blockDim.x) {
        const unsigned act = __activemask();
        uint32_t hit = 0xFFu;  // elements the fp64 decode must see
        if (scr && gi * 8 + 8 <= p.dim) {
            const int64_t i0 = gi * 8, q = i0 >> p.bucket_shift;
            const float lo32f = __double2float_rn(p.meta[q].x), lv32 = __double2float_rn(p.level[q]);
            const float eb = __fmaf_ru(__fmaf_ru(15.0f, fabsf(lv32), fabsf(lo32f)), 0x1p-21f, 0x1p-126f);
            const float thr = __fsub_rd(t32, eb);
            const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p.grads) + i0);
            const uint32_t cw = *reinterpret_cast<const uint32_t*>(p.codes + (i0 >> 1));
            const uint32_t ce = cw & 0x0F0F0F0Fu, co = (cw >> 4) & 0x0F0F0F0Fu;
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            const float2 lv2 = make_float2(lv32, lv32), lo2 = make_float2(lo32f, lo32f);
            const float2 m23 = make_float2(-8388608.0f, -8388608.0f);
            const uint32_t kmag = opaque_kmag(&s_kmag[threadIdx.x >> 5]);
            hit = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2 c2 = make_float2(__uint_as_float(__byte_perm(ce, kmag, 0x7540u | k)),
                                        __uint_as_float(__byte_perm(co, kmag, 0x7540u | k)));
                c2 = __fadd2_rn(c2, m23);
                const float2 a2 = __fadd2_rn(make_float2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xFFFF0000u)),
                                             __ffma2_rn(c2, lv2, lo2));
                hit |= static_cast<uint32_t>(!(__fmul_ru(fabsf(a2.x), 1.0f + 0x1p-22f) < thr)) << (2 * k);
                hit |= static_cast<uint32_t>(!(__fmul_ru(fabsf(a2.y), 1.0f + 0x1p-22f) < thr)) << (2 * k + 1);
            }
        }
        double a[8];
        uint32_t inm = 0;
        int above = 0;
        if (hit == 0xFFu) {  // not screened (or every element hit): the 8-group decode
            const int nv = g_a8(p, gi * 8, a);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t h = static_cast<uint32_t>(__double2hiint(a[e])) & 0x7FFFFFFFu;
                if (e < nv) {
                    mx = max(mx, h);
                    above += h > hi32;
                    inm |= static_cast<uint32_t>(h - lo32 <= span) << e;
                }
            }
        } else {
            for (uint32_t m = hit; m; m &= m - 1) {  // the few screen hits, one at a time
                const int e = __ffs(m) - 1;
                a[e] = g_a(p, gi * 8 + e);
                const uint32_t h = static_cast<uint32_t>(__double2hiint(a[e])) & 0x7FFFFFFFu;
                mx = max(mx, h);
                above += h > hi32;
                inm |= static_cast<uint32_t>(h - lo32 <= span) << e;
            }
        }
        // keys above the bracket are above K*: count them per chunk (a warp's
        // 32 groups lie in one 4096-chunk)
        const int wsum = __reduce_add_sync(act, above);
        if (wsum && lane == __ffs(act) - 1) atomicAdd(&p.cnt[(gi * 8) / kChunk].x, wsum);
        above_t += above;
        if (!__any_sync(act, inm != 0)) continue;
        const int n = __popc(inm);
        int incl = n;  // warp-aggregated slot reservation
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(act, incl, off);
            if (lane >= off && ((act >> (lane - off)) & 1u)) incl += t;
        }
        const int last = 31 - __clz(act);
        const int tot = __shfl_sync(act, incl, last);
        unsigned base = 0;
        if (lane == last) base = atomicAdd(&s_cn, static_cast<unsigned>(tot));
        base = __shfl_sync(act, base, last) + static_cast<unsigned>(incl - n);
        while (inm) {
            const int e = __ffs(inm) - 1;
            inm &= inm - 1;
            if (base < seg_cap) {
                sk[base] = key_of(a[e]);
                si[base] = gi * 8 + e;
            }
            ++base;
        }
    }
    if (mx >= 0x7FF00000u && p.check_finite) atomicOr(p.flag, 1u);
    above_t = __reduce_add_sync(0xFFFFFFFFu, above_t);
    if (lane == 0 && above_t) atomicAdd(&s_above, static_cast<unsigned long long>(above_t));
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_above) atomicAdd(&p.sel_state[7], s_above);
        p.seg_n[blockIdx.x] = s_cn;
        if (blockIdx.x == 0) p.sel_state[14] = 1;  // the per-chunk counts now hold this pass's
    }
}

// Does the bracket hold the k-th largest key? Yes: the digit picks start over
// the collected keys with k - above entries to place (g_bracket_compact packs
// the segments into cand first). No, on the first pass without overflow: one
// retry with a bracket 4x as wide on the side K* lies (the counts say which).
// Otherwise: full digit passes from a clean state (g_cnt_reset clears the
// per-chunk counts a bracket pass made).
// sel_state: [8] ok, [10] width exponent, [11] retry pending, [12]/[13] the
// bracket [lo, hi], [14] per-chunk counts dirty, [15] reset them
__global__ void g_bracket_check(GlobalArgs p, int pass) {
    __shared__ unsigned long long s_n;
    __shared__ int s_ovf;
    if (pass == 1 && p.sel_state[11] == 0) return;  // no retry pending: state stands
    if (threadIdx.x == 0) {
        s_n = 0;
        s_ovf = 0;
    }
    __syncthreads();
    const unsigned long long attempted = pass == 0 ? p.sel_state[6] : 1ull, above = p.sel_state[7];
    const unsigned seg_cap = p.cand_cap / kBracketCtas;
    unsigned long long n_t = 0;
    int ovf_t = 0;
    if (attempted)
        for (int b = threadIdx.x; b < kBracketCtas; b += blockDim.x) {
            const unsigned c = p.seg_n[b];
            n_t += c;
            ovf_t |= c > seg_cap;
        }
    atomicAdd(&s_n, n_t);
    if (ovf_t) s_ovf = 1;
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned long long n = s_n, k = static_cast<unsigned long long>(p.k);
    const bool ok = attempted && !s_ovf && above < k && above + n >= k;
    p.sel_state[8] = ok;
    p.sel_state[11] = 0;
    p.sel_state[15] = !ok && p.sel_state[14];
    p.sel_state[14] = 0;
    if (ok) {
        p.sel_state[2] = k - above;
        *p.cand_n = static_cast<unsigned>(n);
        return;
    }
    *p.cand_n = 0;
    p.sel_state[2] = k;
    p.sel_state[7] = 0;
    if (!attempted) return;
    long long e = static_cast<long long>(p.sel_state[10]) + (s_ovf ? -1 : 1);  // for the next step
    p.sel_state[10] = static_cast<unsigned long long>(e < 0 ? 0 : (e > 12 ? 12 : e));
    if (pass == 0 && !s_ovf) {
        const unsigned long long lo = (p.sel_state[12] >> 32) << 32, hi = p.sel_state[13] | 0xFFFFFFFFull;
        const unsigned long long wide = 4 * (hi - lo + 1);
        if (above >= k) {  // K* above the bracket
            p.sel_state[12] = hi + 1;
            p.sel_state[13] = hi + wide > hi ? hi + wide : ~0ull;
        } else {  // K* below it
            p.sel_state[13] = lo > 0 ? lo - 1 : 0;
            p.sel_state[12] = lo > wide ? lo - wide : 0;
        }
        p.sel_state[11] = lo > 0 || above >= k;  // nothing below a bracket starting at 0
    }
}

__global__ void g_cnt_reset(GlobalArgs p, int64_t nch) {
    if (!p.sel_state[15]) return;
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < nch; c += int64_t(gridDim.x) * blockDim.x)
        p.cnt[c] = make_int2(0, 0);
}

// Segments -> cand[0, n) (order is irrelevant to the digit picks and counts).
__global__ void g_bracket_compact(GlobalArgs p) {
    __shared__ unsigned s_off;
    if (!p.sel_state[8]) return;
    const unsigned b = blockIdx.x, seg_cap = p.cand_cap / kBracketCtas;
    unsigned off_t = 0;
    for (unsigned j = threadIdx.x; j < b; j += blockDim.x) off_t += p.seg_n[j];
    off_t = __reduce_add_sync(0xFFFFFFFFu, off_t);
    if (threadIdx.x == 0) s_off = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_off, off_t);
    __syncthreads();
    const unsigned n = p.seg_n[b], off = s_off;
    for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
        p.cand[off + i] = p.seg_key[size_t(b) * seg_cap + i];
        p.cand_idx[off + i] = p.seg_idx[size_t(b) * seg_cap + i];
    }
}

// The next step's bracket. K* drifts while the error feedback builds up (the
// keys grow as unselected coordinates accumulate) and jitters with the
// gradients, so the bracket spans both "no change" and "the same change
// again": centre K* + delta / 2, half-width |delta| (at least 2^40, ~2^-12 of
// a binade) times 2^(e-1), e adapted: +1 after a miss, -1 after an overflow or
// a crowded buffer. sel_state[9]: this step's K* for the next delta.
__global__ void g_bracket_next(GlobalArgs p) {
    const unsigned long long kstar = p.sel_state[0], prev = p.sel_state[9];
    const bool first = p.sel_state[6] == 0;
    long long e = first ? 2 : static_cast<long long>(p.sel_state[10]);
    if (!first && p.sel_state[8] && *p.cand_n > p.cand_cap / 8 && e > 0) --e;
    const long long delta = first ? 0 : static_cast<long long>(kstar) - static_cast<long long>(prev);
    const unsigned long long ad = static_cast<unsigned long long>(delta < 0 ? -delta : delta);
    const unsigned long long base = ad > (1ull << 40) ? ad : (1ull << 40);
    unsigned long long w = e >= 1 ? base << (e - 1) : base >> 1;
    if (w > (1ull << 58)) w = 1ull << 58;
    const long long c = static_cast<long long>(kstar) + delta / 2;
    const unsigned long long cc = static_cast<unsigned long long>(c < 0 ? 0 : c);
    p.sel_state[6] = w;
    p.sel_state[12] = cc > w ? cc - w : 0;
    p.sel_state[13] = cc + w;
    p.sel_state[9] = kstar;
    p.sel_state[10] = static_cast<unsigned long long>(e);
}

// Radix select state: no key prefix yet, k entries still to place.
__global__ void g_sel_init(GlobalArgs p, int64_t nch) {
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) p.hist[i] = 0;
    for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) p.cnt[c] = make_int2(0, 0);
    if (threadIdx.x == 0) {
        p.sel_state[0] = 0;
        p.sel_state[1] = 0;
        p.sel_state[2] = static_cast<unsigned long long>(p.k);
        *p.cand_n = 0;
        p.sel_state[7] = 0;
        p.sel_state[8] = 0;
        p.sel_state[11] = 0;
        p.sel_state[14] = 0;
        p.sel_state[15] = 0;
    }
}

// After one digit's histogram: the digit of the k-th largest key is the
// highest bin d with (keys in bins > d) < need <= (keys in bins >= d) (bin 0
// takes the rest); need drops by the keys above it. One warp walks the bins
// from the top 32 at a time; the histogram is cleared for the next digit.
__global__ void g_pick(GlobalArgs p, int shift, int nbins) {
    const int lane = threadIdx.x;
    const unsigned long long need = p.sel_state[2];
    unsigned long long above = 0;
    int d = 0;
    for (int top = nbins - 1; top > 0; top -= 32) {
        const int bin = top - lane;
        const unsigned long long c = bin > 0 ? p.hist[bin] : 0ull;
        unsigned long long incl = c;  // inclusive sum over lanes 0..lane (bins top..bin)
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += t;
        }
        const unsigned hit = __ballot_sync(0xFFFFFFFFu, bin > 0 && above + incl >= need);
        if (hit) {
            const int l = __ffs(hit) - 1;
            d = top - l;
            above += __shfl_sync(0xFFFFFFFFu, incl - c, l);
            break;
        }
        above += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    __syncwarp();
    if (lane == 0) {
        p.sel_state[0] |= static_cast<unsigned long long>(d) << shift;
        p.sel_state[1] |= static_cast<unsigned long long>(nbins - 1) << shift;
        p.sel_state[2] = need - above;
    }
    for (int i = lane; i < nbins; i += 32) p.hist[i] = 0;
}

// Row offsets and ties per chunk from the (> K*, == K*) counts: ties go to the
// lowest indices (compress.cpp:43-48), entries in ascending index order. One
// CTA scans the chunks 1024 at a time.
constexpr int kAllocThreads = 1024;
__global__ void g_alloc(GlobalArgs p, int64_t nch) {
    __shared__ int s_tmp[33];
    __shared__ long long s_carry[2];
    if (threadIdx.x == 0) {
        s_carry[0] = 0;  // row offset
        s_carry[1] = 0;  // ties at K* in earlier chunks
    }
    __syncthreads();
    const long long ties = static_cast<long long>(p.sel_state[2]);
    for (int64_t c0 = 0; c0 < nch; c0 += kAllocThreads) {
        const int64_t c = c0 + threadIdx.x;
        const int2 cnt = c < nch ? p.cnt[c] : make_int2(0, 0);
        int tot_eq;
        const long long eq_before = s_carry[1] + cta_excl_scan<kAllocThreads>(cnt.y, s_tmp, tot_eq);
        long long take = ties - eq_before;
        take = take < 0 ? 0 : (take > cnt.y ? cnt.y : take);
        int tot_n;
        const long long off = s_carry[0] + cta_excl_scan<kAllocThreads>(cnt.x + static_cast<int>(take), s_tmp, tot_n);
        if (c < nch) p.sel_info[c] = make_int2(static_cast<int>(off), static_cast<int>(take));
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry[0] += tot_n;
            s_carry[1] += tot_eq;
        }
        __syncthreads();
    }
}

// G3 fused into the register re-quantization (8 <= B_q <= 256, 4-bit EF)
bool g_fused_emit(const GlobalArgs& a) {
    static const bool on = [] {  // A/B: MA_GLOBAL_FUSED_EMIT=0 keeps g_emit separate
        const char* e = std::getenv("MA_GLOBAL_FUSED_EMIT");
        return !(e && e[0] == '0');
    }();
    return on && !a.dense && a.bucket >= 8 && a.bucket <= 256 && (a.bucket & (a.bucket - 1)) == 0;
}

bool g_use_bracket() {
    static const bool on = [] {  // A/B and tests: MA_GLOBAL_BRACKET=0 runs the full digit passes
        const char* e = std::getenv("MA_GLOBAL_BRACKET");
        return !(e && e[0] == '0');
    }();
    return on;
}

// g_alloc in three launches for many chunks: per-tile sums of the (> K*, == K*)
// counts, one CTA scans the tiles (the ties a tile takes follow from the ties
// before it: clamp(T - eq_before, 0, tile_eq)), then every tile scans its
// chunks from its carries — the same offsets / ties as the one-CTA scan.
__global__ void g_alloc_tiles(GlobalArgs p, int64_t nch) {
    __shared__ int s_tmp[33];
    const int64_t c = int64_t(blockIdx.x) * kAllocThreads + threadIdx.x;
    const int2 cnt = c < nch ? p.cnt[c] : make_int2(0, 0);
    int tg, te;
    cta_excl_scan<kAllocThreads>(cnt.x, s_tmp, tg);
    cta_excl_scan<kAllocThreads>(cnt.y, s_tmp, te);
    if (threadIdx.x == 0) {
        p.tiles[4 * blockIdx.x + 0] = tg;
        p.tiles[4 * blockIdx.x + 1] = te;
    }
}

__global__ void g_alloc_scan(GlobalArgs p, int64_t ntiles) {
    __shared__ int s_tmp[33];
    __shared__ long long s_carry[2];
    if (threadIdx.x == 0) {
        s_carry[0] = 0;
        s_carry[1] = 0;
    }
    __syncthreads();
    const long long ties = static_cast<long long>(p.sel_state[2]);
    for (int64_t t0 = 0; t0 < ntiles; t0 += kAllocThreads) {
        const int64_t t = t0 + threadIdx.x;
        const int tg = t < ntiles ? p.tiles[4 * t + 0] : 0, te = t < ntiles ? p.tiles[4 * t + 1] : 0;
        int tot_eq;
        const long long eq_before = s_carry[1] + cta_excl_scan<kAllocThreads>(te, s_tmp, tot_eq);
        long long take = ties - eq_before;
        take = take < 0 ? 0 : (take > te ? te : take);
        int tot_n;
        const long long off = s_carry[0] + cta_excl_scan<kAllocThreads>(tg + static_cast<int>(take), s_tmp, tot_n);
        if (t < ntiles) {
            p.tiles[4 * t + 2] = static_cast<int>(off);
            p.tiles[4 * t + 3] = static_cast<int>(eq_before);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry[0] += tot_n;
            s_carry[1] += tot_eq;
        }
        __syncthreads();
    }
}

__global__ void g_alloc_final(GlobalArgs p, int64_t nch) {
    __shared__ int s_tmp[33];
    const long long ties = static_cast<long long>(p.sel_state[2]);
    const int64_t c = int64_t(blockIdx.x) * kAllocThreads + threadIdx.x;
    const int2 cnt = c < nch ? p.cnt[c] : make_int2(0, 0);
    const long long off0 = p.tiles[4 * blockIdx.x + 2], eqb0 = p.tiles[4 * blockIdx.x + 3];
    int tot_eq;
    const long long eq_before = eqb0 + cta_excl_scan<kAllocThreads>(cnt.y, s_tmp, tot_eq);
    long long take = ties - eq_before;
    take = take < 0 ? 0 : (take > cnt.y ? cnt.y : take);
    int tot_n;
    const long long off = off0 + cta_excl_scan<kAllocThreads>(cnt.x + static_cast<int>(take), s_tmp, tot_n);
    if (c < nch) p.sel_info[c] = make_int2(static_cast<int>(off), static_cast<int>(take));
}

unsigned grid_for(int64_t n, int per) {
    const int64_t want = (n + per - 1) / per;
    return static_cast<unsigned>(want < 148 * 16 ? (want > 0 ? want : 1) : 148 * 16);
}

}  // namespace

int64_t global_chunks(int64_t dim) { return (dim + kChunk - 1) / kChunk; }
bool global_fused_emit(const GlobalArgs& a) { return g_fused_emit(a); }

size_t global_requant_smem(int64_t bucket) {
    // residuals + per-bucket lo, level, 1/level
    return size_t(kChunk) * 8 + 3 * size_t(kChunk / (bucket < kChunk ? bucket : kChunk)) * 8;
}

cudaError_t g_launch_levels(const GlobalArgs& a, cudaStream_t s) {
    g_levels<<<grid_for(a.nbuckets, 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

// G1 (compress.cpp:39-53 over the whole vector): the exact k-th largest |a|
// key K* and how many of its ties to take, 11-bit digits from bit 62 down,
// then 8 bits, each digit picked on the device (no host round trip).
cudaError_t g_launch_select(const GlobalArgs& a, cudaStream_t s) {
    static const int kShift[6] = {52, 41, 30, 19, 8, 0};
    constexpr size_t kPrivSmem = size_t(2048) * 4 * (kThreads / 32);
    static const int g_priv_passes = [] {  // A/B knob: leading digits with per-warp histograms
        const char* e = std::getenv("MA_GLOBAL_PRIV_PASSES");
        const int n = e ? std::atoi(e) : 2;
        return n < 0 ? 0 : (n > 2 ? 2 : n);  // digit 3 collects: never the per-warp variant
    }();
    static const bool g_hist_match = [] {
        const char* e = std::getenv("MA_GLOBAL_HIST_MATCH");  // A/B: match.any on every digit
        return e && e[0] == '1';
    }();
    // the smem opt-in is per device / context: set it on every launch (cheap)
    const bool g_hist_priv =
        !g_hist_match &&
        cudaFuncSetAttribute(g_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPrivSmem)) == cudaSuccess;
    const int64_t nch = global_chunks(a.dim);
    g_sel_init<<<1, 1024, 0, s>>>(a, nch);
    if (g_use_bracket()) {
        const unsigned rg = static_cast<unsigned>(nch < 148 * 64 ? (nch + 255) / 256 + 1 : 148 * 4);
        for (int pass = 0; pass < 2; ++pass) {  // the bracket, then one retry beside it on a miss
            g_bracket<<<kBracketCtas, 256, 0, s>>>(a, pass);
            g_bracket_check<<<1, 256, 0, s>>>(a, pass);
            g_cnt_reset<<<rg, 256, 0, s>>>(a, nch);
        }
        g_bracket_compact<<<kBracketCtas, 256, 0, s>>>(a);
    }
    // digit 3 collects the keys sharing the 22-bit prefix; digits 4-6 read
    // them (a few thousand keys) instead of re-decoding d elements. With a
    // bracket holding K*, every digit reads the bracket's keys (the full
    // passes return at once).
    for (int pass = 0; pass < 6; ++pass) {
        const int nbins = pass == 5 ? 256 : 2048;
        if (pass < g_priv_passes && g_hist_priv) {
            g_hist<true><<<grid_for(a.dim, 256 * 16), 256, kPrivSmem, s>>>(a, kShift[pass], nbins, 0, 0);
        } else {
            g_hist<false><<<grid_for(a.dim, 256 * 16), 256, 0, s>>>(a, kShift[pass], nbins, pass == 2, pass > 2);
        }
        g_hist_cand<<<148 * 2, 256, 0, s>>>(a, kShift[pass], nbins, pass <= 2);
        g_pick<<<1, 32, 0, s>>>(a, kShift[pass], nbins);
    }
    if (g_use_bracket()) g_bracket_next<<<1, 1, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t g_launch_count(const GlobalArgs& a, cudaStream_t s) {
    const int64_t nch = global_chunks(a.dim);
    g_count<<<static_cast<unsigned>(nch < 148 * 8 ? nch : 148 * 8), kThreads, 0, s>>>(a, nch);
    g_count_cand<<<256, 256, 0, s>>>(a);
    const int64_t ntiles = (nch + kAllocThreads - 1) / kAllocThreads;
    const char* tiled_env = std::getenv("MA_GLOBAL_ALLOC_TILED");  // tests: 1 = always the tiled scan
    if (ntiles <= 4 && !(tiled_env && tiled_env[0] == '1')) {
        g_alloc<<<1, kAllocThreads, 0, s>>>(a, nch);
    } else {
        g_alloc_tiles<<<static_cast<unsigned>(ntiles), kAllocThreads, 0, s>>>(a, nch);
        g_alloc_scan<<<1, kAllocThreads, 0, s>>>(a, ntiles);
        g_alloc_final<<<static_cast<unsigned>(ntiles), kAllocThreads, 0, s>>>(a, nch);
    }
    return cudaGetLastError();
}

cudaError_t g_launch_emit(const GlobalArgs& a, cudaStream_t s) {
    if (g_fused_emit(a)) return cudaSuccess;  // g_requant8<L, true> emits
    g_emit<<<static_cast<unsigned>(global_chunks(a.dim)), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t g_launch_requant(const GlobalArgs& a, cudaStream_t s) {
    const unsigned nch = static_cast<unsigned>(global_chunks(a.dim));
    if (a.dense) {
        g_residual_dense<<<nch, kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    const bool emit = g_fused_emit(a);  // g_launch_emit left G3 to this kernel
    // the fp32 form (g_requant8f) for whole chunks of bf16 gradients without a
    // StepReport; the partial last chunk (and everything else) in fp64
    const unsigned nfull = static_cast<unsigned>(a.dim / kChunk);
    const char* f32_env = std::getenv("MA_GLOBAL_RQ_FP32");  // A/B: 0 = the fp64 kernel everywhere
    const bool fp32 = !(f32_env && f32_env[0] == '0') && a.g_dtype == BF16 && !a.partials &&
                      (reinterpret_cast<uintptr_t>(a.grads) & 15u) == 0;
#define MA_RQ8(L)                                                                   \
    if (emit && fp32) {                                                             \
        if (nfull) g_requant8f<L><<<nfull, kThreads, 0, s>>>(a);                    \
        if (nfull < nch) g_requant8<L, true><<<nch - nfull, kThreads, 0, s>>>(a, nfull); \
    } else if (emit) {                                                              \
        g_requant8<L, true><<<nch, kThreads, 0, s>>>(a, 0);                          \
    } else {                                                                        \
        g_requant8<L, false><<<nch, kThreads, 0, s>>>(a, 0);                         \
    }                                                                               \
    return cudaGetLastError();
    switch (a.bucket) {  // the register path for 8 <= B_q <= 256
        case 8: MA_RQ8(1)
        case 16: MA_RQ8(2)
        case 32: MA_RQ8(4)
        case 64: MA_RQ8(8)
        case 128: MA_RQ8(16)
        case 256: MA_RQ8(32)
        default: break;
    }
#undef MA_RQ8
    const size_t smem = global_requant_smem(a.bucket);
    cudaError_t e = cudaFuncSetAttribute(g_requant, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    g_requant<<<static_cast<unsigned>(global_chunks(a.dim)), kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t g_launch_stats_update(const GlobalArgs& a, const GWeights& w, int filled, bool all_bounds,
                                  cudaStream_t s) {
    // the emitters write the new row's chunk bounds; every row's only after a
    // state load (or before the first step)
    if (all_bounds) g_bounds<<<grid_for(int64_t(filled) * a.k, 256 * 4), 256, 0, s>>>(a, filled);
    cudaError_t e = cudaMemsetAsync(a.ovf_n, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    const size_t th_smem = size_t(kChunk) * (a.p_dtype == F64 ? 8 : (a.p_dtype == F32 ? 4 : 2));
    static const bool sparse = [] {  // A/B: MA_GLOBAL_STATS_SPARSE=0 runs the owner / row-loop kernel
        const char* v = std::getenv("MA_GLOBAL_STATS_SPARSE");
        return !(v && v[0] == '0');
    }();
    if (sparse) {
        e = cudaFuncSetAttribute(g_stats_sparse<kStatsThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(th_smem));
        if (e != cudaSuccess) return e;
        g_stats_sparse<kStatsThreads><<<static_cast<unsigned>(global_chunks(a.dim)), kStatsThreads, th_smem, s>>>(a, w, filled);
    } else {
        e = cudaFuncSetAttribute(g_stats_update, cudaFuncAttributeMaxDynamicSharedMemorySize, int(th_smem));
        if (e != cudaSuccess) return e;
        g_stats_update<<<static_cast<unsigned>(global_chunks(a.dim)), kThreads, th_smem, s>>>(a, w, filled);
    }
    const size_t smem = size_t(kChunk) * 2 * sizeof(double);
    e = cudaFuncSetAttribute(g_stats_update_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    g_stats_update_dense<<<148 * 2, kThreads, smem, s>>>(a, w, filled);
    return cudaGetLastError();
}

}  // namespace ma
