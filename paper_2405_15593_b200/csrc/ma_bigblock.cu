// ma_bigblock.cu — the blockwise step for Top-K blocks larger than the
// register-resident kernels hold: B_d in (8192, 32767] (the reference's
// BlockLayout limit, compress.hpp:23 kMaxBlock; optim.cpp:17-18).
//
// One 512-thread CTA per Top-K block; the block's a = g + decode(EF) is
// recomputed from global memory (L2-resident: <= 80 KB of g and codes per
// block) in the reference's fp64 operation order (optim.cpp:166-168,
// quantize.cpp:164-178) whenever a pass needs it:
//   select  (compress.cpp:39-53, 73-85): radix select over the 63-bit |a| keys,
//           8-bit digits from bit 56 with a 256-bin shared histogram; once the
//           keys sharing the prefix fit kCand they are collected and the
//           remaining digits resolve in shared memory. Ties at the k_b-th key
//           go to the lowest indices.
//   emit    the selected entries in ascending index order (CTA scans) into the
//           window ring at this step's slot (window.cpp:14-26), the selection
//           into the bucket-split bitmap; EF re-quantization then runs per
//           bucket over the whole vector (requant_buckets_kernel, ma_kernels.cu).
//   stats   ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) as in
//           the generic kernel: one owner entry per coordinate, rows summed in
//           physical slot order, the owner updates θ.
#include <math_constants.h>

#include "ma_device.cuh"
#include "ma_internal.h"

namespace ma {
namespace {

using namespace dev;

constexpr int kBT = 512;       // threads per CTA
constexpr int kCand = 2048;    // keys resolved in shared memory

__device__ __forceinline__ double div15_b(double x) {  // rn(x / 15), as div15_w (ma_warp.cu)
    if (!(x >= 0x1p-960 && x <= 0x1p1000)) return __ddiv_rn(x, 15.0);
    const double c = 0x1.1111111111111p-4;
    const double q0 = __dmul_rn(x, c);
    return __fma_rn(__fma_rn(-q0, 15.0, x), c, q0);
}

// a at global element gi (4-bit EF, bucket-split layout: any bucket).
__device__ __forceinline__ double big_a(const StepArgs& p, int64_t gi, double& g) {
    const double2 mt = p.meta[gi / p.bucket];
    const double level = mt.x == mt.y ? 0.0 : div15_b(__dsub_rn(mt.y, mt.x));
    const uint32_t c = (p.codes[gi >> 1] >> ((gi & 1) * 4)) & 15u;
    g = ld_val(p.grads, p.g_dtype, gi);
    return __dadd_rn(g, __dadd_rn(__dmul_rn(static_cast<double>(c), level), mt.x));
}

template <int NT>
__device__ __forceinline__ int cta_scan(int v, int* s_tmp, int& total) {  // exclusive, thread order
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) s_tmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int x = lane < NT / 32 ? s_tmp[lane] : 0;
        int xi = x;
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, xi, off);
            if (lane >= off) xi += t;
        }
        if (lane < NT / 32) s_tmp[lane] = xi - x;
        if (lane == 31) s_tmp[32] = xi;
    }
    __syncthreads();
    total = s_tmp[32];
    const int r = s_tmp[w] + incl - v;
    __syncthreads();
    return r;
}

// Shared-memory carve-up (host and device agree).
struct BigLayout {
    size_t hist, misc, tmp, ckey, cidx, owner, eidx, eval, z1, z2, total;
    __host__ __device__ BigLayout(int block, int m, int kbs) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            o = (o + 15) & ~size_t(15);
            const size_t r = o;
            o += bytes;
            return r;
        };
        hist = take(256 * 4);
        misc = take(16 * 8);
        tmp = take(33 * 4);
        // select: candidate keys / indices; later (stats) the per-coordinate owners
        const size_t ent = size_t(m) * size_t(kbs);
        const size_t sel_bytes = size_t(kCand) * 12;
        const size_t own_bytes = size_t(block) * 4;
        ckey = take(sel_bytes > own_bytes ? sel_bytes : own_bytes);
        cidx = ckey + size_t(kCand) * 8;
        owner = ckey;
        eidx = take(ent * 2);
        eval = take(ent * 8);
        z1 = take(ent * 8);
        z2 = take(ent * 8);
        total = (o + 15) & ~size_t(15);
    }
};

__global__ void __launch_bounds__(kBT) big_block_kernel(const __grid_constant__ StepArgs p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const BigLayout L(p.block, p.m, p.kb_stride);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    unsigned long long* misc = reinterpret_cast<unsigned long long*>(smem + L.misc);
    int* s_tmp = reinterpret_cast<int*>(smem + L.tmp);
    uint64_t* ckey = reinterpret_cast<uint64_t*>(smem + L.ckey);
    int* cidx = reinterpret_cast<int*>(smem + L.cidx);
    int* s_owner = reinterpret_cast<int*>(smem + L.owner);
    int16_t* s_eidx = reinterpret_cast<int16_t*>(smem + L.eidx);
    double* s_eval = reinterpret_cast<double*>(smem + L.eval);
    double* s_z1 = reinterpret_cast<double*>(smem + L.z1);
    double* s_z2 = reinterpret_cast<double*>(smem + L.z2);
    int* s_find = reinterpret_cast<int*>(misc + 4);  // find_bin output (3 ints)

    const int tid = threadIdx.x;
    const int64_t b = p.block_offset + blockIdx.x;
    const int64_t base = b * static_cast<int64_t>(p.block);
    const int len = static_cast<int>(min(static_cast<int64_t>(p.block), p.dim - base));
    const int kb = min(p.per_block_k, len);
    const int kbs = p.kb_stride;
    const int per = (len + kBT - 1) / kBT;  // contiguous elements per thread (index order = thread order)
    const int i0 = min(len, tid * per), i1 = min(len, i0 + per);
    const bool want_report = p.partials != nullptr;

    // ---- select: k_b-th largest key K* and the ties it takes ----
    uint64_t prefix = 0, pmask = 0;
    int need = kb;
    bool decided = kb >= len;  // every element selected
    bool exact_k = false;      // all 63 bits fixed: K* = prefix, `need` ties at K*
    int ncand = -1;            // >= 0: the keys sharing the prefix are in ckey / cidx
    bool bad = false;
    for (int shift = 56; !decided && shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kBT) hist[i] = 0;
        __syncthreads();
        if (ncand < 0) {
            for (int i = i0; i < i1; ++i) {
                double g;
                const uint64_t k = key_of(big_a(p, base + i, g));
                if (shift == 56) bad |= (k >> 52) >= 0x7FFu;
                if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
            }
        } else {
            for (int c = tid; c < ncand; c += kBT)
                if ((ckey[c] & pmask) == prefix) atomicAdd(&hist[(ckey[c] >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) find_bin(hist, static_cast<uint32_t>(need), s_find);
        __syncthreads();
        const int bin = s_find[0], above = s_find[1], inbin = s_find[2];
        prefix |= static_cast<uint64_t>(bin) << shift;
        pmask |= uint64_t(255) << shift;
        need -= above;
        if (inbin == need) {
            decided = true;  // every key sharing the prefix is selected
        } else if (shift == 0) {
            exact_k = true;
        } else if (ncand < 0 && inbin <= kCand) {
            // collect the keys sharing the prefix (one more pass), resolve in smem
            if (tid == 0) misc[0] = 0;
            __syncthreads();
            for (int i = i0; i < i1; ++i) {
                double g;
                const uint64_t k = key_of(big_a(p, base + i, g));
                if ((k & pmask) == prefix) {
                    const int q = static_cast<int>(atomicAdd(&misc[0], 1ull));
                    ckey[q] = k;
                    cidx[q] = i;
                }
            }
            __syncthreads();
            ncand = static_cast<int>(misc[0]);
            __syncthreads();
        }
        __syncthreads();
    }
    if (p.check_finite && __syncthreads_or(bad) && tid == 0) atomicOr(p.flag, 1u);
    // selected(k, i): k above the decided prefix, or k == K* among the lowest-index `need` ties
    auto above_k = [&](uint64_t k) { return kb >= len || (k & pmask) > prefix || (decided && (k & pmask) == prefix); };
    auto tie_k = [&](uint64_t k) { return exact_k && k == prefix; };

    // ---- emit: window row at ascending positions + the bucket-split bitmap ----
    int ntie = 0, nsel = 0;
    for (int i = i0; i < i1; ++i) {
        double g;
        const uint64_t k = key_of(big_a(p, base + i, g));
        ntie += tie_k(k);
    }
    int tot;
    int tie_before = cta_scan<kBT>(ntie, s_tmp, tot);
    for (int i = i0; i < i1; ++i) {
        double g;
        const uint64_t k = key_of(big_a(p, base + i, g));
        const bool t = tie_k(k);
        nsel += above_k(k) || (t && tie_before < need);
        tie_before += t;
    }
    int pos = cta_scan<kBT>(nsel, s_tmp, tot);
    tie_before = cta_scan<kBT>(ntie, s_tmp, tot);
    const int slot = p.slot;
    const int64_t wrow = (b * p.m + slot) * static_cast<int64_t>(kbs);
    double rep[kReportFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = i0; i < i1; ++i) {
        double g;
        const double a = big_a(p, base + i, g);
        const uint64_t k = key_of(a);
        const bool t = tie_k(k);
        const bool s = above_k(k) || (t && tie_before < need);
        tie_before += t;
        if (want_report) {
            rep[0] += g * g;
            rep[1] += a * a;
            if (!s) rep[2] += a * a;
        }
        if (s) {
            p.win_idx[wrow + pos] = static_cast<int16_t>(i);
            st_val(p.win_val, p.v_dtype, wrow + pos, a);
            s_eidx[slot * kbs + pos] = static_cast<int16_t>(i);
            s_eval[slot * kbs + pos] = round_to(a, p.v_dtype);
            atomicOr(p.split_sel + ((base + i) >> 5), 1u << ((base + i) & 31));
            ++pos;
        }
    }
    // older rows of the block's window (consumed in slot order below)
    const int filled = p.filled;
    for (int t = tid; t < filled * kb; t += kBT) {
        const int r = t / kb;
        if (r == slot) continue;
        const int j = t - r * kb;
        const int64_t g = (b * p.m + r) * static_cast<int64_t>(kbs) + j;
        s_eidx[r * kbs + j] = p.win_idx[g];
        s_eval[r * kbs + j] = ld_val(p.win_val, p.v_dtype, g);
    }
    __syncthreads();

    // ---- ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187) ----
    const int nent = filled * kb;
    for (int t = tid; t < nent; t += kBT) {
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        atomicExch(&s_owner[s_eidx[e]], e);  // any entry of the coordinate may own it
    }
    __syncthreads();
    for (int t = tid; t < nent; t += kBT) {
        const int r = t / kb;
        const int e = r * kbs + (t - r * kb);
        if (s_owner[s_eidx[e]] == e) {
            s_z1[e] = 0.0;
            s_z2[e] = 0.0;
        }
    }
    __syncthreads();
    for (int r = 0; r < filled; ++r) {  // rows hold unique indices: a row pass is race-free
        const double w1 = p.w1[r], w2 = p.w2[r];
        for (int j = tid; j < kb; j += kBT) {
            const int e = r * kbs + j;
            const int o = s_owner[s_eidx[e]];
            const double v = s_eval[e];
            s_z1[o] = __dadd_rn(s_z1[o], __dmul_rn(w1, v));
            s_z2[o] = __dadd_rn(s_z2[o], __dmul_rn(w2, __dmul_rn(v, v)));
        }
        __syncthreads();
    }
    for (int t = tid; t < nent; t += kBT) {
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
    if (want_report) {  // Σ e_new² (rep[3]) comes from the per-bucket re-quantization
        __shared__ double red[kBT / 32][kReportFields];
        const int lane = tid & 31, w = tid >> 5;
        for (int f = 0; f < kReportFields; ++f) {
            for (int off = 16; off > 0; off >>= 1) rep[f] += __shfl_xor_sync(0xFFFFFFFFu, rep[f], off);
            if (lane == 0) red[w][f] = rep[f];
        }
        __syncthreads();
        if (tid < kReportFields) {
            double s = 0.0;
            for (int w2 = 0; w2 < kBT / 32; ++w2) s += red[w2][tid];
            p.partials[b * kReportFields + tid] = s;
        }
    }
}

}  // namespace

size_t big_block_smem_bytes(int block, int m, int kb_stride) { return BigLayout(block, m, kb_stride).total; }

cudaError_t launch_step_big(const StepArgs& a, int64_t nblocks, cudaStream_t s) {
    if (nblocks <= 0) return cudaSuccess;
    const size_t smem = BigLayout(a.block, a.m, a.kb_stride).total;
    cudaError_t e = cudaFuncSetAttribute(big_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    big_block_kernel<<<static_cast<unsigned>(nblocks), kBT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ma
