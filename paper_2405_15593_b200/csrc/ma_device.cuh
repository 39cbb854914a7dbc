// ma_device.cuh — device helpers shared by the step kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "ma_internal.h"

namespace ma {
namespace dev {

constexpr uint64_t kAbsMask = 0x7FFFFFFFFFFFFFFFull;

__device__ __forceinline__ uint64_t key_of(double x) {
    return static_cast<uint64_t>(__double_as_longlong(x)) & kAbsMask;
}

// Round-to-nearest-even of a double to bfloat16 (one rounding, subnormals and
// overflow to inf included: the sm_100 F2F.BF16.F64 conversion), returned as the
// exactly representable double. Same rule as oracle/microadam_oracle.c:mo_bf16_round.
__device__ __forceinline__ uint16_t bf16_bits(double x) {
    uint16_t r;
    asm("{ .reg .b16 t; cvt.rn.bf16.f64 t, %1; mov.b16 %0, t; }" : "=h"(r) : "d"(x));
    return r;
}
// Two fp32 values to packed bf16 (RNE; lo in the low half), one instruction.
__device__ __forceinline__ uint32_t bf16x2_bits(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ double bf16_round(double x) {
    return static_cast<double>(__uint_as_float(static_cast<uint32_t>(bf16_bits(x)) << 16));
}

__device__ __forceinline__ double round_to(double x, int dt) {
    if (dt == F64) return x;
    if (dt == F32) return static_cast<double>(__double2float_rn(x));
    return bf16_round(x);
}

__device__ __forceinline__ double ld_val(const void* p, int dt, int64_t i) {
    if (dt == F64) return static_cast<const double*>(p)[i];
    if (dt == F32) return static_cast<double>(static_cast<const float*>(p)[i]);
    const uint32_t u = static_cast<const uint16_t*>(p)[i];
    return static_cast<double>(__uint_as_float(u << 16));
}

// Two consecutive elements starting at an even index (aligned vector load).
__device__ __forceinline__ void ld_pair(const void* p, int dt, int64_t i, double& x0, double& x1) {
    if (dt == F64) {
        const double2 v = static_cast<const double2*>(p)[i >> 1];
        x0 = v.x;
        x1 = v.y;
    } else if (dt == F32) {
        const float2 v = static_cast<const float2*>(p)[i >> 1];
        x0 = v.x;
        x1 = v.y;
    } else {
        const uint32_t v = static_cast<const uint32_t*>(p)[i >> 1];
        x0 = static_cast<double>(__uint_as_float(v << 16));
        x1 = static_cast<double>(__uint_as_float(v & 0xFFFF0000u));
    }
}

__device__ __forceinline__ void st_val(void* p, int dt, int64_t i, double x) {
    if (dt == F64) {
        static_cast<double*>(p)[i] = x;
    } else if (dt == F32) {
        static_cast<float*>(p)[i] = __double2float_rn(x);
    } else {
        static_cast<uint16_t*>(p)[i] = bf16_bits(x);
    }
}

// Compile-time-dtype variants (the fast kernel instantiates per dtype combo).
template <int DT>
__device__ __forceinline__ double ld_t(const void* p, int64_t i) {
    if constexpr (DT == F64) return static_cast<const double*>(p)[i];
    else if constexpr (DT == F32) return static_cast<double>(static_cast<const float*>(p)[i]);
    else return static_cast<double>(__uint_as_float(uint32_t(static_cast<const uint16_t*>(p)[i]) << 16));
}
template <int DT>
__device__ __forceinline__ void st_t(void* p, int64_t i, double x) {
    if constexpr (DT == F64) static_cast<double*>(p)[i] = x;
    else if constexpr (DT == F32) static_cast<float*>(p)[i] = __double2float_rn(x);
    else static_cast<uint16_t*>(p)[i] = bf16_bits(x);
}
template <int DT>
__device__ __forceinline__ double round_t(double x) {
    if constexpr (DT == F64) return x;
    else if constexpr (DT == F32) return static_cast<double>(__double2float_rn(x));
    else return bf16_round(x);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}


// Warp 0: locate the bin holding the need-th largest element of a 256-bin
// histogram. out = {bin, count above bin, count in bin}; bin = -1 if the
// histogram holds fewer than `need` elements.
__device__ __forceinline__ void find_bin(const uint32_t* hist, uint32_t need, int* out) {
    const int lane = threadIdx.x & 31;
    uint32_t h[8];
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        h[q] = hist[lane * 8 + q];
        s += h[q];
    }
    uint32_t incl = s;  // Σ over lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_down_sync(0xFFFFFFFFu, incl, off);
        if (lane + off < 32) incl += v;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 0);
    if (total < need) {
        if (lane == 0) {
            out[0] = -1;
            out[1] = 0;
            out[2] = static_cast<int>(total);
        }
        return;
    }
    uint32_t cum = incl - s;
#pragma unroll
    for (int q = 7; q >= 0; --q) {
        if (cum < need && cum + h[q] >= need) {
            out[0] = lane * 8 + q;
            out[1] = static_cast<int>(cum);
            out[2] = static_cast<int>(h[q]);
        }
        cum += h[q];
    }
}

template <int NT>
__device__ __forceinline__ void block_zero_hist(uint32_t* hist) {
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
}

// Block Top-K (compress.cpp:39-53 semantics): select exactly `kb` of the
// valid elements, the first under (|a| desc, index asc). Returns the
// selection bitmask over the thread's register slots.
//
// Keys are the fp64 bit patterns with the sign cleared (monotone in |a|,
// -0.0 == +0.0). Pass 1 is a 256-bin histogram of key>>45 (1/128 binade per
// bin) over the top 256 bins below the block maximum, which usually leaves a
// handful of candidates; a general 8-bit-digit radix select from bit 62
// covers the rest. Once the candidates fit kCandCap they are ranked exactly
// by (key desc, index asc); if all 63 bits tie, the lowest indices win.
//
// `elem(i)` maps register slot i to its block-relative element index;
// `tie_rank(mask, rank)` returns, for the flagged slots, their exclusive rank
// in element-index order across the block (all threads must call it).
template <int NT, int EPT, class Elem, class TieRank>
__device__ uint32_t block_topk(const double (&a)[EPT], uint32_t valid, int kb, uint32_t* hist,
                               int* misc, uint64_t* ckey, int* cidx, uint8_t* selm, Elem elem,
                               TieRank tie_rank) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    uint32_t sel = 0;
    uint32_t tmax = 0;
#pragma unroll
    for (int i = 0; i < EPT; ++i)
        if ((valid >> i) & 1u) tmax = max(tmax, static_cast<uint32_t>(key_of(a[i]) >> 45));
    tmax = __reduce_max_sync(0xFFFFFFFFu, tmax);
    if (lane == 0) misc[warp] = static_cast<int>(tmax);
    block_zero_hist<NT>(hist);
    __syncthreads();
    uint32_t top = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) top = max(top, static_cast<uint32_t>(misc[w]));
    const uint32_t tbase = top >= 255u ? top - 255u : 0u;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        if ((valid >> i) & 1u) {
            const uint32_t t = static_cast<uint32_t>(key_of(a[i]) >> 45);
            if (t >= tbase) atomicAdd(&hist[t - tbase], 1u);
        }
    }
    __syncthreads();
    if (warp == 0) find_bin(hist, static_cast<uint32_t>(kb), misc + 16);
    __syncthreads();

    int need = kb;
    int fs;
    uint64_t prefix;
    int cnt;
    if (misc[16] >= 0) {
        prefix = tbase + static_cast<uint32_t>(misc[16]);
        need -= misc[17];
        cnt = misc[18];
        fs = 45;
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (((valid >> i) & 1u) && (key_of(a[i]) >> 45) > prefix) sel |= 1u << i;
    } else {
        fs = 63;
        prefix = 0;
        cnt = 0x7FFFFFFF;  // unknown; forces a radix pass
    }

    for (;;) {
        // Candidates: valid, unselected, key >> fs == prefix.
        uint32_t cand = 0;
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (((valid >> i) & 1u) && !((sel >> i) & 1u) && (key_of(a[i]) >> fs) == prefix)
                cand |= 1u << i;
        if (cnt == need) {
            sel |= cand;
            break;
        }
        if (cnt <= kCandCap) {
            __syncthreads();  // misc[20] / ckey reuse
            if (tid == 0) misc[20] = 0;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                if ((cand >> i) & 1u) {
                    const int s = atomicAdd(&misc[20], 1);
                    ckey[s] = key_of(a[i]);
                    cidx[s] = elem(i);
                }
            }
            __syncthreads();
            const int n = misc[20];
            for (int c = tid; c < n; c += NT) {
                const uint64_t kc = ckey[c];
                const int ic = cidx[c];
                int r = 0;
                for (int q = 0; q < n; ++q) {
                    const uint64_t kq = ckey[q];
                    r += (kq > kc) || (kq == kc && cidx[q] < ic);
                }
                if (r < need) selm[ic] = 1;
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < EPT; ++i)
                if (((cand >> i) & 1u) && selm[elem(i)]) sel |= 1u << i;
            break;
        }
        if (fs == 0) {
            // Exact 63-bit ties beyond the cap: lowest indices win.
            int rank[EPT];
            tie_rank(cand, rank);
#pragma unroll
            for (int i = 0; i < EPT; ++i)
                if (((cand >> i) & 1u) && rank[i] < need) sel |= 1u << i;
            break;
        }
        const int ns = fs > 8 ? fs - 8 : 0;
        const int width = fs - ns;
        const uint32_t mask = (1u << width) - 1u;
        __syncthreads();  // hist / misc reuse
        block_zero_hist<NT>(hist);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if ((cand >> i) & 1u)
                atomicAdd(&hist[static_cast<uint32_t>(key_of(a[i]) >> ns) & mask], 1u);
        __syncthreads();
        if (warp == 0) find_bin(hist, static_cast<uint32_t>(need), misc + 16);
        __syncthreads();
        const uint32_t bin = static_cast<uint32_t>(misc[16]);
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (((cand >> i) & 1u) && (static_cast<uint32_t>(key_of(a[i]) >> ns) & mask) > bin)
                sel |= 1u << i;
        need -= misc[17];
        cnt = misc[18];
        prefix = (prefix << width) | bin;
        fs = ns;
    }
    return sel;
}

// 0x4B000000 (2^23 as fp32 bits, the nibble -> float decode constant) read back
// from shared memory by a volatile load ptxas cannot fold: with a literal, ptxas
// under register pressure encodes the constant as PRMT's immediate and moves
// every selector from a uniform register instead (one extra IMAD.U32 per
// decoded element). The word is written by the reading thread itself (or by
// the warp before a __syncwarp).
__device__ __forceinline__ uint32_t opaque_kmag(const int* s_word) {
    uint32_t v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];"
                 : "=r"(v)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_word))));
    return v;
}

}  // namespace dev
}  // namespace ma
