/*
 * ma_synth.h — counter-based synthetic inputs shared by the device bench path
 * and the CPU checkers, so both sides see bit-identical gradients and θ₀
 * without host↔device transfers (SURVEY.md §8(d) "Synthetic inputs").
 *
 * value(seed, step, i) = (s - 131070) * 2^-15, with s the sum of the four
 * 16-bit lanes of a splitmix64 hash of (seed, step, i): an Irwin–Hall(4)
 * approximation of N(0, 1.155²) whose every value is an exact multiple of
 * 2^-15 below 2^3 in magnitude, so it is exactly representable in fp32 and
 * fp64 and rounds deterministically to bf16. No libm call is involved, so the
 * host (gcc) and device (nvcc) produce identical bits.
 *
 * Plain C99; usable from C, C++ and CUDA (__host__ __device__ when nvcc).
 */
#ifndef MA_SYNTH_H
#define MA_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define MA_HD __host__ __device__ __forceinline__
#else
#define MA_HD static inline
#endif

MA_HD uint64_t ma_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

MA_HD uint64_t ma_synth_hash(uint64_t seed, uint64_t step, uint64_t index) {
    return ma_splitmix64(ma_splitmix64(ma_splitmix64(seed) ^ step) ^ index);
}

/* Gaussian-like value, exact multiple of 2^-15 in (-4, 4). */
MA_HD double ma_synth_normal(uint64_t seed, uint64_t step, uint64_t index) {
    uint64_t h = ma_synth_hash(seed, step, index);
    int64_t s = (int64_t)(h & 0xFFFFu) + (int64_t)((h >> 16) & 0xFFFFu) +
                (int64_t)((h >> 32) & 0xFFFFu) + (int64_t)(h >> 48);
    return (double)(s - 131070) * (1.0 / 32768.0);
}

/* Tie-heavy variant: 16 levels {-7.5, ..., 7.5} (many exact |x| ties). */
MA_HD double ma_synth_levels(uint64_t seed, uint64_t step, uint64_t index) {
    uint64_t h = ma_synth_hash(seed, step, index);
    return (double)(int64_t)(h & 15u) - 7.5;
}

/* Heavy-tailed, scale-varying variant (test and bench stress input): the
 * Gaussian-like value times 2^(e_block + e_tail), where e_block in [-16, 16]
 * is drawn per 4096-element block and changes every 4 steps (gradient scale
 * differing by 2^32 across blocks and drifting over time), and e_tail in
 * [0, 12] is nonzero for 1 element in 64 (outliers up to 2^12 times the
 * block's scale). Every value is an exact fp32 (|x| < 2^15, multiples of
 * 2^-31), so host and device round it to bf16 identically. */
MA_HD double ma_synth_heavy(uint64_t seed, uint64_t step, uint64_t index) {
    uint64_t hb = ma_synth_hash(seed ^ 0xB10CB10CB10CB10Cull, step >> 2, index >> 12);
    int eb = (int)(hb % 33u) - 16;
    uint64_t ht = ma_synth_hash(seed ^ 0x7A117A117A117A11ull, step, index);
    int et = (ht & 63u) == 0 ? (int)((ht >> 6) % 13u) : 0;
    int e = eb + et;
    double scale = 1.0;
    for (int k = 0; k < (e < 0 ? -e : e); ++k) scale = e < 0 ? scale * 0.5 : scale * 2.0;
    return ma_synth_normal(seed, step, index) * scale;
}

/* mode 0: ma_synth_normal, 1: ma_synth_levels, 2: ma_synth_heavy */
MA_HD double ma_synth_value(int mode, uint64_t seed, uint64_t step, uint64_t index) {
    return mode == 1 ? ma_synth_levels(seed, step, index)
                     : (mode == 2 ? ma_synth_heavy(seed, step, index) : ma_synth_normal(seed, step, index));
}

#endif /* MA_SYNTH_H */
