/*
 * microadam_cuda.h — C ABI of libmicroadam_cuda: the B200 (sm_100a) MicroAdam
 * optimizer step behind plain pointers and sizes (no C++ / torch types).
 *
 * It replaces, for the blockwise practical engine, the reference's
 *   microadam::MicroAdamOptimizer            (proj/include/microadam/optim.hpp:98-128,
 *                                             proj/src/optim.cpp:127-190)
 *   microadam::HyperParams / validate        (optim.hpp:15-30, optim.cpp:7-30)
 *   microadam::StepReport                    (optim.hpp:32-38)
 *   microadam::GradientWindow, QuantizedErrorBuffer state inspection
 *                                            (window.hpp:10-33, quantize.hpp:54-70)
 * Paths are relative to the reference root /root/reference. Each entry point
 * names the reference symbol it stands in for. INTEGRATION.md shows the
 * reference-side binding (a C++ Optimizer adapter and a ctypes stub).
 *
 * Error model: every call returns ma_status; the reference's throw sites map
 * to codes (std::invalid_argument -> MA_ERR_INVALID_ARG / MA_ERR_DIM /
 * MA_ERR_NONFINITE, std::logic_error -> MA_ERR_STATE). ma_last_error() gives
 * the message for the calling thread. No exception crosses the ABI.
 *
 * Threading: one handle is bound to one device; calls on one handle must be
 * serialized (the reference optimizer is not thread-safe either).
 */
#ifndef MICROADAM_CUDA_H
#define MICROADAM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MA_API __attribute__((visibility("default")))
#else
#define MA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MA_ABI_VERSION 1

typedef enum ma_status {
    MA_OK = 0,
    MA_ERR_INVALID_ARG = 1, /* HyperParams::validate / BlockLayout ctor throws (optim.cpp:7-21, compress.cpp:19-26) */
    MA_ERR_DIM = 2,         /* "step: gradient dim mismatch" (optim.cpp:34-35) */
    MA_ERR_NONFINITE = 3,   /* check_finite on the gradient (optim.cpp:36, vec.hpp:41-45) */
    MA_ERR_CUDA = 4,        /* CUDA runtime failure */
    MA_ERR_NCCL = 5,        /* collective failure (multi-GPU helpers) */
    MA_ERR_UNSUPPORTED = 6, /* legal reference config this build does not run on device */
    MA_ERR_STATE = 7        /* e.g. error_buffer() on a lossless engine (optim.cpp:155-158) */
} ma_status;

typedef enum ma_dtype { MA_F64 = 0, MA_F32 = 1, MA_BF16 = 2 } ma_dtype;

/* Non-finite gradient handling (reference: check_grad throws before any
 * mutation, optim.cpp:34-37). */
typedef enum ma_finite_mode {
    MA_FINITE_FLAG = 0,   /* fused check; flag read at ma_sync(); state undefined after a hit */
    MA_FINITE_STRICT = 1, /* pre-scan + host sync; rejects before mutation (reference-exact) */
    MA_FINITE_OFF = 2     /* no check */
} ma_finite_mode;

/* Mirrors microadam::HyperParams (optim.hpp:15-30). k <= 0 means "unset". */
typedef struct ma_hyperparams {
    double beta1;        /* 0.9 */
    double beta2;        /* 0.999 */
    double eps;          /* 1e-8 */
    double lr;           /* 1e-3 (used by ma_step_host; ma_step takes lr per call) */
    double weight_decay; /* 0; unused by the practical engine, as in the reference */
    int64_t window;      /* m = 10 */
    double density;      /* 0.01 */
    int64_t k;           /* explicit selection count, overrides density; <= 0 unset */
    int32_t bits;        /* 4 */
    int32_t reserved0;
    int64_t block;       /* B_d = 4096 */
    int64_t bucket;      /* B_q = 64 */
} ma_hyperparams;

typedef struct ma_config {
    ma_hyperparams hp;
    int32_t blockwise;      /* 1 (the device path); 0 = global Top-K, run as one block when d <= 8192 */
    int32_t lossless_error; /* 0 (quantized EF); 1 = dense fp64 residual (blockwise, generic kernel) */
    int32_t param_dtype;    /* ma_dtype of θ in device memory */
    int32_t grad_dtype;     /* ma_dtype of the gradient */
    int32_t value_dtype;    /* ma_dtype of window values (bf16 = the paper's layout) */
    int32_t finite_mode;    /* ma_finite_mode */
} ma_config;

/* Mirrors microadam::StepReport (optim.hpp:32-38). Norms are reduced in a
 * fixed tree order (≠ the reference's sequential sum: within 1e-12 relative);
 * update_nnz is exact. loss is left 0 (filled by run() in the reference). */
typedef struct ma_step_report {
    double grad_norm;
    double error_norm;
    double empirical_q;
    int64_t update_nnz;
    double loss;
} ma_step_report;

/* Derived layout (optim.cpp:137-144, compress.cpp:28-33, quantize.hpp:67). */
typedef struct ma_layout_info {
    int64_t dim;          /* parameters covered by this layout (shard length for shards) */
    int64_t block;        /* min(hp.block, global dim) */
    int64_t per_block_k;  /* min(ceil(density*block), block) */
    int64_t num_blocks;   /* blocks covered */
    int64_t row_width;    /* Σ_b min(per_block_k, len_b) = window row width k_ */
    int64_t num_buckets;  /* EF buckets covered */
    int64_t code_bytes;   /* packed EF bytes covered */
    int64_t kb_stride;    /* device window entries reserved per (block, slot) */
    int64_t state_bytes;  /* device optimizer-state bytes (EF codes + meta + window) */
} ma_layout_info;

typedef struct ma_handle ma_handle;

/* Defaults of HyperParams (optim.hpp:15-30) + device dtypes f32/f32/bf16, flag mode. */
MA_API void ma_config_default(ma_config* cfg);

/* HyperParams::validate (optim.cpp:7-21) + resolve_k (:23-30) + BlockLayout
 * checks + device support checks, without allocating anything. */
MA_API ma_status ma_validate(const ma_config* cfg, int64_t dim);

/* Layout for the whole vector (block_begin=0, block_end=-1) or a block range. */
MA_API ma_status ma_layout(const ma_config* cfg, int64_t dim, int64_t block_begin, int64_t block_end,
                    ma_layout_info* out);

/* MicroAdamOptimizer ctor (optim.cpp:127-153): zero EF buffer (quantize.cpp:130-140),
 * empty window (window.cpp:5-12). θ stays caller-owned (see ma_step). */
MA_API ma_status ma_create(const ma_config* cfg, int64_t dim, int device, ma_handle** out);

/* Same, owning only blocks [block_begin, block_end) of a dim-length vector
 * (block-aligned data-parallel shard). Pointers passed to
 * ma_step then address the shard's slice (element block_begin*block). */
MA_API ma_status ma_create_shard(const ma_config* cfg, int64_t dim, int64_t block_begin,
                          int64_t block_end, int device, ma_handle** out);

MA_API ma_status ma_destroy(ma_handle* h);

/* MicroAdamOptimizer::step (optim.cpp:164-190) on device memory:
 * d_params (param_dtype, updated in place) and d_grads (grad_dtype), both
 * covering the handle's range; lr replaces hp.lr; stream is a cudaStream_t
 * (NULL = legacy default). Asynchronous unless report != NULL or
 * finite_mode == MA_FINITE_STRICT. */
MA_API ma_status ma_step(ma_handle* h, void* d_params, const void* d_grads, double lr, void* stream,
                  ma_step_report* report);

/* Drop-in host path for Optimizer::step(const Vec&) + params(): h_grads and
 * h_params are HOST buffers (pinned or pageable, grad/param dtype). The handle
 * keeps a device copy of θ (uploaded from h_params on the first call or after
 * ma_set_params), streams the gradient up and the updated θ back in chunks
 * that overlap the step, and returns when h_params holds the new θ. The device
 * θ is authoritative between calls: modify θ only through ma_set_params. With
 * MA_HOST_SPARSE=1 in the environment only θ at the window coordinates comes
 * back (scattered by host threads) when h_params is the buffer of the
 * previous call; otherwise, and by default, the whole θ is copied back. */
MA_API ma_status ma_step_host(ma_handle* h, void* h_params, const void* h_grads, double lr,
                       ma_step_report* report);

/* Data-parallel step with the gradient reduce-scatter fused in (SURVEY.md
 * §8(f) rank 2; the step's input a = g + e is optim.cpp:166-168 with g the
 * reduced gradient). d_srcs[r] (r < nsrc <= 8) point at rank r's gradient for
 * THIS handle's element range — peer device pointers (CUDA IPC / symmetric
 * memory over NVLink) or local buffers — and must stay unmodified until the
 * step completes on `stream`. The step uses
 *     g = rn_grad_dtype(((src_0 + src_1) + ... + src_{nsrc-1}) * scale)
 * with fp32 sums and product for bf16/f32 gradients (fp64 for f64), written
 * into d_grads (may alias one source), and is then bit-identical to ma_step on
 * that g. The lean kernel reads the sources block by block inside the step
 * (B_q = 64, k_b <= 64, bf16/bf16/bf16 or f32/f32/f32, no report, finite mode
 * off/flag); other configurations run a reduce kernel, then ma_step. */
MA_API ma_status ma_step_reduce(ma_handle* h, void* d_params, void* d_grads, const void* const* d_srcs,
                                int32_t nsrc, float scale, double lr, void* stream, ma_step_report* report);

/* Wait for outstanding work; returns MA_ERR_NONFINITE if the fused check hit. */
MA_API ma_status ma_sync(ma_handle* h);

/* window().step / head / filled and the m row stamps (window.hpp:10-33). */
MA_API ma_status ma_get_counters(const ma_handle* h, int64_t* step, int64_t* head, int64_t* filled,
                          int64_t* stamps /* m entries, may be NULL */);

/* error_buffer() (optim.cpp:155-158): packed codes (code_bytes) and per-bucket
 * (lo, hi) as fp64 (num_buckets each), host buffers, for the handle's range. */
MA_API ma_status ma_read_error_buffer(ma_handle* h, uint8_t* codes, double* lo, double* hi);

/* error_vector() (optim.cpp:160-162): the dense error feedback in fp64 (dim
 * entries): the decoded 4-bit buffer, or the stored residual of a
 * lossless_error engine (for which ma_read_error_buffer returns MA_ERR_STATE,
 * like error_buffer() throwing std::logic_error, optim.cpp:155-158). */
MA_API ma_status ma_read_error_vector(ma_handle* h, double* out);

/* error_buffer() restricted to blocks [block_begin, block_end) of the handle:
 * their packed codes (elements [block_begin*block, min(block_end*block, dim)),
 * byte-aligned since block*bits is a multiple of 8) and their buckets' (lo, hi).
 * For parity checks of sampled block ranges of very large handles. On a
 * global Top-K handle (blockwise = 0) a "block" is a 4096-element chunk. */
MA_API ma_status ma_read_error_buffer_blocks(ma_handle* h, int64_t block_begin, int64_t block_end, uint8_t* codes,
                                             double* lo, double* hi);

/* window().rows[slot] restricted to blocks [block_begin, block_end): the
 * Σ min(per_block_k, len_b) entries of those blocks, global int64 indices
 * (ascending) and values widened to fp64. */
MA_API ma_status ma_read_window_blocks(ma_handle* h, int64_t slot, int64_t block_begin, int64_t block_end,
                                       int64_t* indices, double* values);

/* window().rows[slot] in the reference layout: row_width global int64 indices
 * (ascending) and values widened to fp64. Returns MA_ERR_INVALID_ARG for slot
 * out of range. An unwritten row reads back as zeros. */
MA_API ma_status ma_read_window_row(ma_handle* h, int64_t slot, int64_t* indices, double* values);

/* Restore state (checkpoint resume; inverse of the three readers above). */
MA_API ma_status ma_write_state(ma_handle* h, const uint8_t* codes, const double* lo, const double* hi,
                         int64_t step, int64_t head, const int64_t* stamps,
                         const int64_t* win_indices /* m*row_width */,
                         const double* win_values /* m*row_width */);

/* save_checkpoint / load_checkpoint (checkpoint.hpp:28-33, checkpoint.cpp:50-140):
 * the reference's MADM v1 file, written from / restored into this handle's
 * state. params (param_dtype, dim elements) is a device pointer when
 * params_on_device != 0, else a host pointer; on load it receives θ (may be
 * NULL to skip). θ and window values are stored as f64 (exact widening), the
 * EF as packed codes + fp64 (lo, hi). Whole-vector handles only
 * (MA_ERR_UNSUPPORTED for shards and lossless buffers). Note: the reference
 * loader itself rejects dim > 2^32 (checkpoint.cpp:101). */
MA_API ma_status ma_save_checkpoint(ma_handle* h, const void* params, int32_t params_on_device, const char* path);
MA_API ma_status ma_load_checkpoint(ma_handle* h, void* params, int32_t params_on_device, const char* path);

/* Sparse parameter propagation: MicroAdamOptimizer::step
 * (optim.cpp:164-190) split so data-parallel ranks exchange the new window rows
 * (int16 index + value per selected entry, ~0.04 B/param) instead of θ. Every
 * rank holds a whole-vector handle and a θ replica; per step:
 *   ma_step_front  on its block range [block_begin, block_end): EF decode, Top-K,
 *                  window row (also copied to d_stage_idx / d_stage_val, layout
 *                  [block_end - block_begin][kb_stride], int16 / value dtype),
 *                  EF re-quantization; advances the window counters. d_grads
 *                  holds the gradient of that block range only.
 *   (all-gather the stage buffers across ranks, e.g. ncclAllGather)
 *   ma_scatter_rows puts the gathered rows of [block_begin, block_end) into the
 *                  window ring at this step's slot.
 *   ma_step_stats  ADAM_STATS (window.cpp:28-46) + update (optim.cpp:183-187)
 *                  over all blocks into d_params (the rank's θ replica).
 * Whole 4096-blocks, B_q = 64, flag/off finiteness, lean-kernel dtypes;
 * front(all) + stats(all) is bit-identical to ma_step. MA_ERR_STATE if the
 * calls are out of order. */
MA_API ma_status ma_step_front(ma_handle* h, const void* d_grads, int64_t block_begin, int64_t block_end,
                        void* d_stage_idx, void* d_stage_val, void* stream);
MA_API ma_status ma_scatter_rows(ma_handle* h, const void* d_rows_idx, const void* d_rows_val,
                          int64_t block_begin, int64_t block_end, void* stream);
MA_API ma_status ma_step_stats(ma_handle* h, void* d_params, double lr, void* stream);

/* ---- Data-parallel collectives over NCCL ----------------
 * One process (or thread) per GPU, one shard handle per rank: rank r of N owns
 * blocks [r*per, min((r+1)*per, num_blocks)) with per = ceil(num_blocks / N)
 * (paper_2405_15593_b200/sharding.py), i.e. elements from r*per*block on. The
 * step itself exchanges nothing (the Top-K partitions by block,
 * compress.cpp:73-85; the replicated host counters keep the bias correction of
 * window.cpp:43 global), so a sharded run is bit-identical to the unsharded one.
 * NCCL is loaded at run time (libnccl.so.2 already in the process, e.g.
 * torch's, else the system one; MA_NCCL_LIB overrides); failures return
 * MA_ERR_NCCL. The reference has no distributed path. */
typedef struct ma_comm ma_comm;

/* ncclGetUniqueId: 128 bytes rank 0 hands to every rank (any out-of-band channel). */
MA_API ma_status ma_comm_unique_id(uint8_t* id /* 128 bytes */);
/* ncclCommInitRank on `device` (collective across the nranks callers). */
MA_API ma_status ma_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int device, ma_comm** out);
/* Use an existing ncclComm_t (not destroyed by ma_comm_destroy). */
MA_API ma_status ma_comm_wrap(void* nccl_comm, ma_comm** out);
MA_API ma_status ma_comm_destroy(ma_comm* comm);
MA_API ma_status ma_comm_info(const ma_comm* comm, int32_t* nranks, int32_t* rank);

/* The north star's ZeRO-1 step: ma_step on this rank's shard of the full θ
 * replica d_params_full (the shard starts at element r*per*block), then the
 * NCCL all-gather of the updated θ shards into every rank's replica, all on
 * `stream`. full_elems >= N*per*block (padded layout): one in-place
 * ncclAllGather; full_elems == dim: grouped in-place ncclBroadcast of each
 * rank's shard. d_grads covers this rank's shard only. With a report, the
 * StepReport sums are all-reduced first, so every rank gets the global one. */
MA_API ma_status ma_step_allgather(ma_handle* h, void* d_params_full, int64_t full_elems, const void* d_grads,
                                   double lr, ma_comm* comm, void* stream, ma_step_report* report);
/* The all-gather of ma_step_allgather alone. */
MA_API ma_status ma_allgather_params(ma_handle* h, void* d_params_full, int64_t full_elems, ma_comm* comm,
                                     void* stream);
/* Sparse parameter propagation's exchange (between ma_step_front and
 * ma_step_stats on whole-vector handles): ncclAllGather of every rank's stage
 * rows ([stage_blocks][kb_stride] int16 indices + values, stage_blocks =
 * ceil(num_blocks / N)) into d_rows_* ([N*stage_blocks][kb_stride]), then
 * ma_scatter_rows of all blocks into the window ring. */
MA_API ma_status ma_exchange_rows(ma_handle* h, const void* d_stage_idx, const void* d_stage_val,
                                  int64_t stage_blocks, void* d_rows_idx, void* d_rows_val, ma_comm* comm,
                                  void* stream);

/* For ma_step_host: replace the device copy of θ from a host buffer. */
MA_API ma_status ma_set_params(ma_handle* h, const void* h_params);

MA_API ma_status ma_get_layout(const ma_handle* h, ma_layout_info* out);

/* Number of step-kernel launches issued so far by this handle (all kernels). */
MA_API int64_t ma_kernel_launches(const ma_handle* h);

/* Diagnostics of the fast kernel, collected only when the handle was created
 * with MA_DEBUG_COUNTERS=1 in the environment (else zeros): out[0] blocks that
 * took the exact radix-select fallback, out[1] elements quantized through the
 * IEEE-division path, out[2] Top-K threshold bisection probes. */
MA_API ma_status ma_debug_counters(ma_handle* h, int64_t* out, int n);

MA_API const char* ma_last_error(void);
MA_API const char* ma_version(void);

/* Synthetic gradient generator on device (include/ma_synth.h stream rounded
 * to dtype), for benches: out[i] = round(value(seed, step, offset + i));
 * levels = 0 Gaussian-like, 1 the 16-level tie-heavy stream, 2 heavy-tailed
 * with per-block scales (ma_synth_heavy). */
MA_API ma_status ma_fill_synthetic(void* d_out, int32_t dtype, int64_t n, uint64_t seed, uint64_t step,
                            int64_t offset, int32_t levels, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MICROADAM_CUDA_H */
