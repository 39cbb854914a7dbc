// ma_internal.h — shared between the C-ABI host code (ma_capi.cu) and the
// sm_100a kernels (ma_kernels.cu). Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ma {

constexpr int kMaxWindow = 1024;  // m supported on device (params carry m weights; 10-bit rows in dup lists)
constexpr int kMaxWindowGlobal = 256;  // m of the global Top-K mode (its stats kernel stages m row bounds)
constexpr int kMaxRanks = 8;     // gradient sources of a fused reduce-scatter step
constexpr int kMaxBlock = 8192;  // B_d of the register-resident kernels (fp64 block held on chip)
constexpr int kMaxBlockBig = 32767;  // B_d of the big-block kernel (the reference's BlockLayout limit)
constexpr int kCandCap = 128;    // exact-rank stage capacity of the Top-K select
constexpr int kReportFields = 5; // Σg², Σa², Σr², Σe_new², nnz per block

enum Dtype : int32_t { F64 = 0, F32 = 1, BF16 = 2 };

// One step over blocks [block_offset, block_offset + gridDim-covered) of the
// handle's shard. All pointers are shard-local (element 0 = first element of
// the shard); block b covers elements [b*block, min((b+1)*block, dim)).
struct StepArgs {
    const void* grads;
    void* params;
    uint8_t* codes;   // packed 4-bit EF codes, low nibble first (quantize.cpp:102-114)
    double2* meta;    // per-bucket (lo, hi) fp64
    int16_t* win_idx; // [num_blocks][m][kb_stride] block-relative indices
    void* win_val;    // [num_blocks][m][kb_stride] values (value dtype)
    unsigned int* flag;
    double* partials; // nullable: [num_blocks][kReportFields]
    uint32_t* thresh; // [num_blocks] Top-K fast-path threshold carried across steps (fast kernel)
    unsigned int* dbg;  // nullable diagnostics: [0] exact-select fallbacks, [1] exact-quotient
                        // elements, [2] threshold bisection probes (fast kernel)
    int64_t dim;
    int64_t num_blocks;
    int64_t block_offset;
    int64_t block_count;  // blocks [block_offset, block_offset + block_count) (persistent kernel)
    int32_t block, per_block_k, kb_stride, bucket;
    int32_t m, filled, slot, check_finite;
    int32_t g_dtype, p_dtype, v_dtype, force_exact;  // force_exact: warp kernel without the fp32 screen (A/B, tests)
    double eps, lr, scale1, scale2;
    double w1[kMaxWindow];
    double w2[kMaxWindow];
    // fp32 companions for the lean kernel's bf16-θ update screen (ma_warp.cu):
    // c1[r] = rn(w1[r] * scale1), c2[r] = rn(sqrt(w2[r] * scale2)), rn(eps), rn(lr)
    float c1[kMaxWindow];
    float c2[kMaxWindow];
    float eps32, lr32;
    // sparse-propagation front (lean kernel PH = 1): new rows also go to
    // stage_*[(b - stage_b0) * kb_stride + pos]
    int16_t* stage_idx;
    void* stage_val;
    int64_t stage_b0;
    // lossless error feedback (MicroAdamOptimizer(..., lossless_error = true),
    // optim.cpp:172-173): the residual kept dense in fp64 (generic kernel only)
    double* dense;
    int32_t bits;  // EF code width; the generic kernel handles 1..8, the others 4
    int32_t pad1;
    // fused gradient reduce-scatter (ma_step_reduce, lean kernel RS variant):
    // g = rn_gdt(((src_0 + src_1) + ...) * rs_scale) in fp32, written to grads
    // block by block before the step reads it; rs_n = 0 off
    const void* rs_src[kMaxRanks];
    int32_t rs_n;
    float rs_scale;
    // bucket-split mode (B_q does not divide B_d, quantize.cpp:142-162 buckets
    // the whole vector): the generic kernel skips the re-quantization and
    // marks its selection here (1 bit per element, zeroed before the step);
    // launch_requant_buckets then re-quantizes bucket by bucket
    uint32_t* split_sel;
};

// Global Top-K mode (ma_global.cu, blockwise = false with d > kMaxBlock).
struct GlobalArgs {
    const void* grads;
    void* params;
    uint8_t* codes;
    double2* meta;
    double* level;       // [nbuckets] level of the EF being decoded
    int64_t* win_idx;    // [m][row_stride] global indices (int64: d may exceed 2^31)
    void* win_val;       // [m][row_stride] values (v_dtype)
    uint16_t* selbits;   // selection bits, 16 elements per word
    uint32_t* hist;      // [2048] radix histogram
    int2* cnt;           // [chunks] (keys > K*, keys == K*)
    int2* sel_info;        // [chunks] (row offset, ties taken)
    unsigned long long* sel_state;  // radix select on device: [0] key prefix (K* at the end), [1] mask, [2] ties left
    uint64_t* cand;       // keys sharing the prefix after three digits (cand_cap entries)
    int64_t* cand_idx;    // their indices
    unsigned int* cand_n;
    unsigned int cand_cap;
    int32_t* bounds;     // [m][chunks + 1] first entry of each 4096-chunk per row
    int32_t* ovf_list;   // [chunks] chunks with more window entries than the staged path holds
    uint64_t* seg_key;    // carried bracket: per-CTA segments of collected keys (cand_cap entries)
    int64_t* seg_idx;     // their indices
    unsigned int* seg_n;  // [kBracketCtas] keys collected per segment
    int32_t* tiles;       // [chunks / 1024 + 1][4] g_alloc tile sums / carries
    unsigned int* ovf_n;
    double* partials;    // nullable: [chunks][kReportFields]
    unsigned int* flag;
    double* dense;       // lossless error feedback (optim.cpp:149-152): the fp64 residual, else null
    int64_t dim, nbuckets, bucket, k, row_stride;
    int32_t slot, g_dtype, p_dtype, v_dtype, check_finite, bucket_shift;
    double eps, lr, scale1, scale2;
};
constexpr int kBracketCtas = 148 * 8;  // g_bracket grid (one collection segment per CTA)
int64_t global_chunks(int64_t dim);
bool global_fused_emit(const GlobalArgs& a);  // G3 runs inside the re-quantization kernel
size_t global_requant_smem(int64_t bucket);
cudaError_t g_launch_levels(const GlobalArgs& a, cudaStream_t s);
cudaError_t g_launch_select(const GlobalArgs& a, cudaStream_t s);  // G1: six digit passes, no host sync
cudaError_t g_launch_count(const GlobalArgs& a, cudaStream_t s);  // G2 + row offsets / ties per chunk
cudaError_t g_launch_emit(const GlobalArgs& a, cudaStream_t s);
cudaError_t g_launch_requant(const GlobalArgs& a, cudaStream_t s);  // lossless: the residual itself
struct GWeights {
    double w1[kMaxWindowGlobal];
    double w2[kMaxWindowGlobal];
};
cudaError_t g_launch_stats_update(const GlobalArgs& a, const GWeights& w, int filled, bool all_bounds,
                                  cudaStream_t s);

struct Variant {
    int nt;   // threads per CTA
    int ept;  // elements per thread (even)
};

// Dynamic shared memory bytes needed by the step kernel for this shape.
size_t step_smem_bytes(int nt, int ept, int block, int bucket, int m, int kb_stride, int bits = 4);
// Smallest variant that holds `block` elements on chip; nt == 0 if none.
Variant pick_variant(int block);

cudaError_t launch_step(const StepArgs& a, Variant v, int64_t nblocks, cudaStream_t s);

// Fast persistent kernel (ma_fast.cu): full blocks only; B_q in {16, 32, 64},
// B_d in {1024, 2048, 4096, 8192}, m*kb_stride <= 65535. ept = 8 * groups per thread.
Variant pick_fast_variant(int block, int bucket, int m, int kb_stride, int g_dtype, int p_dtype,
                          int v_dtype);
size_t fast_smem_bytes(Variant v, int block, int bucket, int m, int kb_stride, int g_dtype,
                       int p_dtype, int v_dtype);
int fast_blocks_per_sm(Variant v, int bucket, size_t smem);
cudaError_t launch_step_fast(const StepArgs& a, Variant v, int grid, cudaStream_t s);
// Warp-per-block kernel (ma_warp.cu): full B_d = 4096 blocks, k_b <= 64.
bool warp_path_ok(int block, int bucket, int kb, int m, int kb_stride, int g_dtype, int p_dtype,
                  int v_dtype);
size_t warp_smem_bytes(int bucket);
cudaError_t launch_step_warp(const StepArgs& a, cudaStream_t s);
// Tile kernel (ma_tile.cu, the default): persistent 128-thread CTAs, one
// B_d = 4096 / B_q = 64 block at a time, TMA-fed double-buffered stages.
bool tile_ok(const StepArgs& a);
cudaError_t launch_step_tile(const StepArgs& a, cudaStream_t s);
// Whether the warp kernels run this step (the exact one needs k_b <= 64).
bool warp_can_run(const StepArgs& a);
// Lean kernel split for sparse parameter propagation (ph 1 = front, 2 = stats).
bool lean_phase_ok(const StepArgs& a);
cudaError_t launch_step_lean_phase(const StepArgs& a, int ph, cudaStream_t s);
cudaError_t launch_finite_scan(const void* g, int dtype, int64_t n, unsigned int* flag,
                               cudaStream_t s);
// STRICT finiteness of a = g + e for f64 gradients (reference: check_finite in
// topk_blockwise, compress.cpp:76), before any mutation.
cudaError_t launch_finite_scan_a(const double* g, const uint8_t* codes, const double2* meta, const double* dense,
                                 int64_t n, int64_t bucket, int bits, unsigned int* flag, cudaStream_t s);
cudaError_t launch_report_reduce(const double* partials, int64_t nblocks, double* out5,
                                 cudaStream_t s);
cudaError_t launch_gather_window_theta(const int16_t* win_idx, const void* theta, int pdt, void* out, int64_t b0,
                                      int64_t b1, int m, int kbs, int kb, int filled, int64_t block, int64_t dim,
                                      cudaStream_t s);
// g[e0, e1) = rn_gdt(((src_0 + src_1) + ...) * scale) (fp32 sums for bf16/f32
// gradients, fp64 for f64): the unfused reduce-scatter of ma_step_reduce.
cudaError_t launch_reduce_grads(const void* const* srcs, int nsrc, float scale, int gdt, void* dst, int64_t e0,
                                int64_t e1, cudaStream_t s);
// Blockwise Top-K blocks in (kMaxBlock, kMaxBlockBig] (ma_bigblock.cu): one CTA
// per block, a recomputed from global memory, EF re-quantized afterwards by
// launch_requant_buckets (the handle runs in bucket-split mode).
size_t big_block_smem_bytes(int block, int m, int kb_stride);
cudaError_t launch_step_big(const StepArgs& a, int64_t nblocks, cudaStream_t s);
// Bucket-split mode: per bucket q of the whole vector, a = g + decode(old
// codes, meta[q]) (codes_old), zero the elements marked in `sel`, exact
// (lo, hi), 4-bit codes by the guarded quotient into codes_new (zeroed before),
// meta[q] = (lo, hi); Σ e_new² added to *err2 when non-null (StepReport).
cudaError_t launch_requant_buckets(const void* grads, int gdt, const uint8_t* codes_old, uint8_t* codes_new,
                                   double2* meta, const uint32_t* sel, int64_t dim, int64_t bucket, double* err2,
                                   cudaStream_t s);
// lean kernel with the fused reduce (B_q = 64, k_b <= 64, bf16/bf16/bf16 or f32/f32/f32)
bool lean_rs_ok(const StepArgs& a);
cudaError_t launch_fill_synthetic(void* out, int dtype, int64_t n, uint64_t seed, uint64_t step,
                                  int64_t offset, int levels, cudaStream_t s);

}  // namespace ma

#include <string>

// NCCL entry points resolved at run time (ma_nccl.cpp). Opaque types keep this
// header free of nccl.h: comm = ncclComm_t, id = ncclUniqueId (128 bytes),
// enums passed as int (ncclDataType_t / ncclRedOp_t / ncclResult_t values).
namespace ma {
namespace nccl {
struct IdBytes {
    char internal[128];
};
using Comm = struct ncclComm*;
struct Api {
    int (*GetUniqueId)(IdBytes*);
    int (*CommInitRank)(Comm*, int, IdBytes, int);
    int (*CommDestroy)(Comm);
    int (*CommCount)(const Comm, int*);
    int (*CommUserRank)(const Comm, int*);
    int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t);
    int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
    int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
    int (*GroupStart)();
    int (*GroupEnd)();
    const char* (*GetErrorString)(int);
    int (*GetVersion)(int*);
};
constexpr int kUint8 = 1, kFloat64 = 8, kSum = 0;  // ncclUint8, ncclFloat64, ncclSum
// nullptr (and *err set) when no NCCL library can be loaded.
const Api* api(std::string* err);
std::string describe(const Api* a, int rc);
}  // namespace nccl
}  // namespace ma
