/*
 * microadam_oracle.c — CPU restatement of the reference MicroAdam blockwise
 * optimizer step. TEST INFRASTRUCTURE ONLY: this file is the checker that
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the
 * CUDA path against. Nothing in paper_2405_15593_b200/ links, loads or calls
 * it, and it is never the thing measured or shipped.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement bit-for-bit
 * against (1) the reference's own known-answer tests (transcribed from
 * /root/reference/proj/tests/*.cpp) and (2) tests/golden/*.npz, produced by
 * running the unmodified reference sources (oracle/ref_shim.cpp, built by
 * oracle/Makefile into oracle/_ref/) through oracle/make_golden.py.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Arithmetic is IEEE fp64 with no contraction (build
 * with -ffp-contract=off and no -march, exactly like the reference's CMake
 * Release build).
 *
 * One deliberate extension over the reference: the stored window values and
 * θ can be rounded to a narrower dtype (fp32 / bf16) after each step, which is
 * what the device path stores. With both dtypes = F64 the restatement is the
 * reference; with narrower dtypes it is the "composed oracle" of SURVEY.md
 * §8(c) (reference algorithm, values rounded where the device stores them).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/ma_synth.h"

enum { MO_F64 = 0, MO_F32 = 1, MO_BF16 = 2 };
enum { MO_OK = 0, MO_ERR_INVALID_ARG = 1, MO_ERR_DIM = 2, MO_ERR_NONFINITE = 3 };

typedef struct {
    double grad_norm, error_norm, empirical_q;
    int64_t update_nnz;
    double loss;
} mo_report; /* optim.hpp:32-38 StepReport */

/* Direct round-to-nearest-even of a double to bfloat16 (8 significant bits,
 * fp32 exponent range incl. subnormals, overflow to ±inf). Not in the
 * reference (it has no bf16); the device uses the same rule. */
double mo_bf16_round(double x) {
    if (!isfinite(x) || x == 0.0) return x;
    double ax = fabs(x);
    if (ax < 0x1p-126) {
        /* bf16 subnormal spacing 2^-133 */
        return nearbyint(x * 0x1p133) * 0x1p-133;
    }
    union { double d; uint64_t u; } v = {x};
    uint64_t lsb = (v.u >> 45) & 1u;
    v.u += ((uint64_t)1 << 44) - 1u + lsb;
    v.u &= ~(((uint64_t)1 << 45) - 1u);
    if (fabs(v.d) >= 0x1p128) return copysign(INFINITY, x);
    return v.d;
}

double mo_round(double x, int dtype) {
    switch (dtype) {
        case MO_F32: return (double)(float)x;
        case MO_BF16: return mo_bf16_round(x);
        default: return x;
    }
}

/* ---------------------------------------------------------------------------
 * L1 primitives
 * ------------------------------------------------------------------------- */

/* compress.cpp:19-33 BlockLayout::from_density: per_block_k = min(ceil(density*block), block). */
int64_t mo_per_block_k(int64_t block, double density) {
    int64_t k = (int64_t)ceil(density * (double)block);
    return k < block ? k : block;
}

static const double* g_sort_x; /* qsort has no context argument */

/* compress.cpp:39-53 comparator: |x| descending, ties toward the lower index. */
static int cmp_better(const void* pa, const void* pb) {
    int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    double ma = fabs(g_sort_x[a]), mb = fabs(g_sort_x[b]);
    if (ma != mb) return ma > mb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

static int cmp_i64(const void* pa, const void* pb) {
    int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* compress.cpp:39-53 topk_indices: the k first entries of [first,last) under
 * the total order above (nth_element + resize), returned ascending (sort).
 * A full sort yields the same set because the order is total. */
static void topk_indices(const double* x, int64_t first, int64_t last, int64_t k, int64_t* out,
                         int64_t* scratch) {
    int64_t n = last - first;
    for (int64_t i = 0; i < n; ++i) scratch[i] = first + i;
    g_sort_x = x;
    qsort(scratch, (size_t)n, sizeof(int64_t), cmp_better);
    memcpy(out, scratch, (size_t)k * sizeof(int64_t));
    qsort(out, (size_t)k, sizeof(int64_t), cmp_i64);
}

/* compress.cpp:73-85 topk_blockwise (+ gather :55-62). Returns the number of
 * selected entries; out_idx/out_val hold Σ_b min(per_block_k, len_b) entries. */
int64_t mo_topk_blockwise(const double* x, int64_t d, int64_t block, int64_t per_block_k,
                          int64_t* out_idx, double* out_val) {
    int64_t* scratch = (int64_t*)malloc((size_t)(block < d ? block : d) * sizeof(int64_t));
    int64_t n = 0;
    for (int64_t start = 0; start < d; start += block) {
        int64_t len = block < d - start ? block : d - start;
        int64_t k = per_block_k < len ? per_block_k : len;
        topk_indices(x, start, start + len, k, out_idx + n, scratch);
        n += k;
    }
    free(scratch);
    if (out_val)
        for (int64_t j = 0; j < n; ++j) out_val[j] = x[out_idx[j]];
    return n;
}

/* compress.cpp:66-71 topk_global == one block spanning d. */
int64_t mo_topk_global(const double* x, int64_t d, int64_t k, int64_t* out_idx, double* out_val) {
    return mo_topk_blockwise(x, d, d, k, out_idx, out_val);
}

/* quantize.cpp:7-13 QuantParams ctor: level = lo == hi ? 0 : (hi - lo) / (2^bits - 1). */
double mo_level(double lo, double hi, int bits) {
    return lo == hi ? 0.0 : (hi - lo) / (double)((1u << bits) - 1u);
}

/* quantize.cpp:15-24 quant_params: running std::min / std::max from x[0]. */
void mo_quant_params(const double* x, int64_t n, double* lo, double* hi) {
    double l = x[0], h = x[0];
    for (int64_t i = 0; i < n; ++i) {
        l = (x[i] < l) ? x[i] : l; /* std::min(l, x) */
        h = (h < x[i]) ? x[i] : h; /* std::max(h, x) */
    }
    *lo = l;
    *hi = h;
}

/* quantize.cpp:42-55 quantize_nearest: floor((x - lo)/level + 0.5) clamped to
 * [0, 2^bits - 1]; level 0 maps everything to code 0. */
uint32_t mo_quantize_nearest(double x, double lo, double level, int bits) {
    if (level == 0.0) return 0u;
    double v = floor((x - lo) / level + 0.5);
    double mx = (double)((1u << bits) - 1u);
    v = v < 0.0 ? 0.0 : (v > mx ? mx : v);
    return (uint32_t)v;
}

/* quantize.cpp:102-114 pack: bitstream, low bits first within each byte. */
void mo_pack(const uint32_t* codes, int64_t n, int bits, uint8_t* out) {
    int64_t nbytes = (n * bits + 7) / 8;
    memset(out, 0, (size_t)nbytes);
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int b = 0; b < bits; ++b, ++pos)
            if ((codes[i] >> b) & 1u) out[pos / 8] |= (uint8_t)(1u << (pos % 8));
}

/* quantize.cpp:116-128 unpack. */
void mo_unpack(const uint8_t* bytes, int64_t n, int bits, uint32_t* codes) {
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i) {
        codes[i] = 0;
        for (int b = 0; b < bits; ++b, ++pos)
            if ((bytes[pos / 8] >> (pos % 8)) & 1u) codes[i] |= 1u << b;
    }
}

/* quantize.cpp:142-162 QuantizedErrorBuffer::encode (nearest). */
void mo_encode(const double* x, int64_t d, int bits, int64_t bucket, uint8_t* codes, double* lo,
               double* hi) {
    uint32_t* all = (uint32_t*)malloc((size_t)d * sizeof(uint32_t));
    int64_t nb = (d + bucket - 1) / bucket;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t start = b * bucket;
        int64_t len = bucket < d - start ? bucket : d - start;
        mo_quant_params(x + start, len, &lo[b], &hi[b]);
        double level = mo_level(lo[b], hi[b], bits);
        for (int64_t i = 0; i < len; ++i)
            all[start + i] = mo_quantize_nearest(x[start + i], lo[b], level, bits);
    }
    mo_pack(all, d, bits, codes);
    free(all);
}

/* quantize.cpp:164-178 decode: e_i = double(code) * level + lo (separate
 * multiply and add; the reference build has no FMA). */
void mo_decode(const uint8_t* codes, const double* lo, const double* hi, int64_t d, int bits,
               int64_t bucket, double* out) {
    uint32_t* all = (uint32_t*)malloc((size_t)d * sizeof(uint32_t));
    mo_unpack(codes, d, bits, all);
    int64_t nb = (d + bucket - 1) / bucket;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t start = b * bucket;
        int64_t len = bucket < d - start ? bucket : d - start;
        double level = mo_level(lo[b], hi[b], bits);
        for (int64_t i = 0; i < len; ++i) {
            volatile double prod = (double)all[start + i] * level;
            out[start + i] = prod + lo[b];
        }
    }
    free(all);
}

/* window.cpp:28-46 adam_stats over rows in physical slot order. rows are
 * [m][row_width] (idx, val); stamps[m]; z has d entries. */
void mo_adam_stats(const int64_t* idx, const double* val, const int64_t* stamps, int64_t m,
                   int64_t row_width, int64_t filled, int64_t step, int64_t d, double beta,
                   int square, double* z) {
    (void)m;
    for (int64_t i = 0; i < d; ++i) z[i] = 0.0;
    for (int64_t r = 0; r < filled; ++r) {
        if (stamps[r] == 0) continue;
        double w = pow(beta, (double)(step - stamps[r]));
        for (int64_t j = 0; j < row_width; ++j) {
            double v = val[r * row_width + j];
            volatile double c = w * (square ? v * v : v);
            z[idx[r * row_width + j]] += c;
        }
    }
    double scale = (1.0 - beta) / (1.0 - pow(beta, (double)step));
    for (int64_t i = 0; i < d; ++i) z[i] *= scale;
}

static double norm2(const double* x, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s);
}

/* ---------------------------------------------------------------------------
 * L2: MicroAdamOptimizer (blockwise, quantized EF) — optim.cpp:127-190
 * ------------------------------------------------------------------------- */

typedef struct mo_opt {
    int64_t dim, m, block, bucket, per_block_k, row_width, nbuckets;
    double beta1, beta2, eps;
    int bits, param_dtype, value_dtype;
    double* theta;
    uint8_t* codes;
    double *lo, *hi;
    int64_t head, filled, step;
    int64_t* stamps;
    int64_t* win_idx; /* [m][row_width] global indices (window.hpp:11-15) */
    double* win_val;  /* stored values, rounded to value_dtype */
    int64_t* last_idx;
    double* last_val; /* exact a at the selection (compress.cpp:55-62) */
    double *a, *e, *r, *z1, *z2;
} mo_opt;

void mo_destroy(mo_opt* o) {
    if (!o) return;
    free(o->theta); free(o->codes); free(o->lo); free(o->hi); free(o->stamps);
    free(o->win_idx); free(o->win_val); free(o->last_idx); free(o->last_val);
    free(o->a); free(o->e); free(o->r); free(o->z1); free(o->z2);
    free(o);
}

/* optim.cpp:7-21 HyperParams::validate + :127-153 ctor (blockwise=true,
 * lossless=false). k <= 0 means "unset" (std::optional). Returns NULL and
 * sets *status on invalid input. */
mo_opt* mo_create(int64_t dim, const double* theta0, double beta1, double beta2, double eps,
                  double lr, int64_t window, double density, int64_t k, int bits, int64_t block,
                  int64_t bucket, int param_dtype, int value_dtype, int* status) {
    *status = MO_ERR_INVALID_ARG;
    if (!(beta1 > 0.0 && beta1 < 1.0) || !(beta2 > 0.0 && beta2 < 1.0)) return NULL;
    if (!(eps > 0.0) || !(lr > 0.0) || window < 1) return NULL;
    if (!(density > 0.0) || density > 1.0) return NULL;
    if (k != 0 && k < 1) return NULL;
    if (bits < 1 || bits > 24 || block < 1 || block > 32767 || bucket < 1) return NULL;
    if (dim < 1) return NULL;
    if (k > dim) return NULL; /* resolve_k, optim.cpp:23-30 */
    mo_opt* o = (mo_opt*)calloc(1, sizeof(mo_opt));
    o->dim = dim;
    o->m = window;
    o->beta1 = beta1;
    o->beta2 = beta2;
    o->eps = eps;
    o->bits = bits;
    o->bucket = bucket;
    o->param_dtype = param_dtype;
    o->value_dtype = value_dtype;
    double dens = k > 0 ? (double)k / (double)dim : density;
    if (!(dens > 0.0) || dens > 1.0) { free(o); return NULL; }
    o->block = block < dim ? block : dim;
    o->per_block_k = mo_per_block_k(o->block, dens);
    if (o->per_block_k < 1) { free(o); return NULL; }
    o->row_width = 0;
    for (int64_t s = 0; s < dim; s += o->block) {
        int64_t len = dim - s;
        o->row_width += o->per_block_k < len ? o->per_block_k : len;
    }
    o->nbuckets = (dim + bucket - 1) / bucket;
    o->theta = (double*)malloc((size_t)dim * sizeof(double));
    for (int64_t i = 0; i < dim; ++i) o->theta[i] = mo_round(theta0[i], param_dtype);
    o->codes = (uint8_t*)calloc((size_t)((dim * bits + 7) / 8), 1);
    o->lo = (double*)calloc((size_t)o->nbuckets, sizeof(double));
    o->hi = (double*)calloc((size_t)o->nbuckets, sizeof(double));
    o->stamps = (int64_t*)calloc((size_t)window, sizeof(int64_t));
    o->win_idx = (int64_t*)calloc((size_t)(window * o->row_width), sizeof(int64_t));
    o->win_val = (double*)calloc((size_t)(window * o->row_width), sizeof(double));
    o->last_idx = (int64_t*)calloc((size_t)o->row_width, sizeof(int64_t));
    o->last_val = (double*)calloc((size_t)o->row_width, sizeof(double));
    o->a = (double*)malloc((size_t)dim * sizeof(double));
    o->e = (double*)malloc((size_t)dim * sizeof(double));
    o->r = (double*)malloc((size_t)dim * sizeof(double));
    o->z1 = (double*)malloc((size_t)dim * sizeof(double));
    o->z2 = (double*)malloc((size_t)dim * sizeof(double));
    *status = MO_OK;
    return o;
}

/* optim.cpp:164-190 MicroAdamOptimizer::step (blockwise, quantized EF). */
int mo_step(mo_opt* o, const double* grad, double lr, mo_report* rep) {
    int64_t d = o->dim;
    /* optim.cpp:34-37 check_grad: finite before any mutation */
    for (int64_t i = 0; i < d; ++i)
        if (!isfinite(grad[i])) return MO_ERR_NONFINITE;
    /* :166-168 e = decode(error); a = g + e */
    mo_decode(o->codes, o->lo, o->hi, d, o->bits, o->bucket, o->e);
    for (int64_t i = 0; i < d; ++i) o->a[i] = grad[i] + o->e[i];
    for (int64_t i = 0; i < d; ++i)
        if (!isfinite(o->a[i])) return MO_ERR_NONFINITE; /* compress.cpp:76 check_finite */
    /* :169 topk_blockwise */
    mo_topk_blockwise(o->a, d, o->block, o->per_block_k, o->last_idx, o->last_val);
    /* :170 zero_selected (compress.cpp:95-102) */
    memcpy(o->r, o->a, (size_t)d * sizeof(double));
    for (int64_t j = 0; j < o->row_width; ++j) o->r[o->last_idx[j]] = 0.0;
    /* :174 encode (nearest) */
    mo_encode(o->r, d, o->bits, o->bucket, o->codes, o->lo, o->hi);
    /* :175 window push (window.cpp:14-26) */
    ++o->step;
    o->stamps[o->head] = o->step;
    for (int64_t j = 0; j < o->row_width; ++j) {
        o->win_idx[o->head * o->row_width + j] = o->last_idx[j];
        o->win_val[o->head * o->row_width + j] = mo_round(o->last_val[j], o->value_dtype);
    }
    o->head = (o->head + 1) % o->m;
    o->filled = o->step < o->m ? o->step : o->m;
    /* :176-177 adam_stats(β1,false), adam_stats(β2,true) */
    mo_adam_stats(o->win_idx, o->win_val, o->stamps, o->m, o->row_width, o->filled, o->step, d,
                  o->beta1, 0, o->z1);
    mo_adam_stats(o->win_idx, o->win_val, o->stamps, o->m, o->row_width, o->filled, o->step, d,
                  o->beta2, 1, o->z2);
    /* :178-182 report */
    mo_report rp;
    memset(&rp, 0, sizeof(rp));
    rp.grad_norm = norm2(grad, d);
    double na = norm2(o->a, d);
    rp.empirical_q = na > 0.0 ? norm2(o->r, d) / na : 0.0;
    mo_decode(o->codes, o->lo, o->hi, d, o->bits, o->bucket, o->e);
    rp.error_norm = norm2(o->e, d);
    /* :183-187 update */
    for (int64_t i = 0; i < d; ++i) {
        volatile double den = o->eps + sqrt(o->z2[i]);
        double u = o->z1[i] / den;
        if (u != 0.0) ++rp.update_nnz;
        volatile double step_ = lr * u;
        o->theta[i] = mo_round(o->theta[i] - step_, o->param_dtype);
    }
    if (rep) *rep = rp;
    return MO_OK;
}

/* ---- accessors (optim.hpp:109-115) ---- */
int64_t mo_dim(const mo_opt* o) { return o->dim; }
int64_t mo_row_width(const mo_opt* o) { return o->row_width; }
int64_t mo_per_block_k_of(const mo_opt* o) { return o->per_block_k; }
int64_t mo_block_of(const mo_opt* o) { return o->block; }
int64_t mo_num_buckets(const mo_opt* o) { return o->nbuckets; }
const double* mo_params(const mo_opt* o) { return o->theta; }
const uint8_t* mo_codes(const mo_opt* o) { return o->codes; }
const double* mo_lo(const mo_opt* o) { return o->lo; }
const double* mo_hi(const mo_opt* o) { return o->hi; }
const int64_t* mo_last_idx(const mo_opt* o) { return o->last_idx; }
const double* mo_last_val(const mo_opt* o) { return o->last_val; }
void mo_counters(const mo_opt* o, int64_t* step, int64_t* head, int64_t* filled) {
    *step = o->step;
    *head = o->head;
    *filled = o->filled;
}
const int64_t* mo_stamps(const mo_opt* o) { return o->stamps; }
const int64_t* mo_win_idx(const mo_opt* o) { return o->win_idx; }
const double* mo_win_val(const mo_opt* o) { return o->win_val; }

/* ---- synthetic inputs (include/ma_synth.h), rounded to a dtype ---- */
void mo_synth_fill(uint64_t seed, uint64_t step, int64_t offset, int64_t n, int dtype, int levels,
                   double* out) {
    for (int64_t i = 0; i < n; ++i) {
        double v = ma_synth_value(levels, seed, step, (uint64_t)(offset + i));
        out[i] = mo_round(v, dtype);
    }
}
