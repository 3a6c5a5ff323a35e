/*
 * cdn.h -- C ABI of the B200-native compressed-DNN inference library
 * (arxiv 1711.00244, "inference from Deep-Compression models under memory
 * constraints").  Citations: P:Lnnn = /root/reference/PAPER.md line,
 * S:Lnnn = SPEC.md line, C-nn = reading listed in DESIGN.md.
 *
 * The calls follow the paper's statement of the problem (P:L754, L651,
 * L724-726): a user loads compressed layers once (the model stays resident,
 * P:L40, L173), sets a memory budget TOT and optionally a latency threshold,
 * and asks for inference of K inputs with maximum throughput.
 *
 * Conventions
 *  - Every function returns cdn_status: 0 = CDN_OK, negative = error.  No C++
 *    exception or abort crosses this boundary.  cdn_last_error() returns a
 *    thread-local message describing the last failure on the calling thread.
 *  - Pointers are plain host or device pointers as stated per argument.  The
 *    library never takes ownership of caller buffers; it copies what it keeps.
 *  - One call at a time per cdn_model handle; distinct handles are
 *    independent.  Loaded layers are immutable.
 *  - Floating point is fp32 (FC: fp32 FMA, fp32 accumulate; CONV: bf16 inputs,
 *    fp32 accumulate, config C4).
 *  - Device work runs on the stream given (NULL = the library's own stream, in
 *    which case the call returns with results complete).
 */
#ifndef CDN_H_
#define CDN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDN_ABI_VERSION 2

typedef int32_t cdn_status;
enum {
  CDN_OK = 0,
  CDN_E_ARG = -1,          /* bad argument (NULL, out of range)                        */
  CDN_E_MAGIC = -2,        /* CDNI magic is not "CDNI"                                 */
  CDN_E_VERSION = -3,      /* unknown CDNI version                                     */
  CDN_E_TRUNCATED = -4,    /* buffer shorter than the CDNI structure requires          */
  CDN_E_MALFORMED = -5,    /* Kraft violation, offsets non-monotone, val/gap token     */
                           /* counts differ, column >= cols, pad invariant broken      */
  CDN_E_UNSUPPORTED = -6,  /* code length > 32, r > 8, k > 8, blocked layout (bh != 1) */
  CDN_E_SHAPE = -7,        /* layer shapes do not chain / input shape mismatch         */
  CDN_E_OOM = -8,          /* device or host allocation failed                         */
  CDN_E_INFEASIBLE = -9,   /* no batch plan satisfies TOT / latency     */
  CDN_E_CUDA = -10,        /* CUDA runtime error (message has the CUDA error string)   */
  CDN_E_NCCL = -11,        /* NCCL error                                               */
  CDN_E_STATE = -12        /* call not valid in this state (no layers, concurrent use) */
};

typedef struct cdn_model cdn_model;

enum { CDN_LAYER_FC = 0, CDN_LAYER_CONV = 1 };

/* How a loaded weight matrix is used.  FC: b = W a + v (Eq. 1-2).
 * CONV: W has one row per filter and K = kh*kw*in_c/groups columns flattened
 * as (r, s, c), channel fastest (C-18); activations are NHWC. */
typedef struct {
  int32_t kind;                  /* CDN_LAYER_FC or CDN_LAYER_CONV                    */
  int32_t relu;                  /* 1: ReLU after the bias                             */
  int32_t in_c, in_h, in_w;      /* CONV input geometry (ignored for FC)               */
  int32_t kh, kw, stride, pad, groups;
  int32_t lrn;                   /* CONV: cross-channel LRN after ReLU (C-20)          */
  int32_t pool_k, pool_s;        /* CONV: max-pool after (0 = none)                    */
} cdn_layer_desc;

typedef struct {
  uint32_t rows, cols;           /* full layer geometry                               */
  uint32_t row_begin, row_end;   /* rows held by this rank (row-block shard)          */
  uint32_t k, r;                 /* relative-index bits, quantization bits            */
  uint32_t lanes_per_row;        /* G: decode lanes per row (column bands)             */
  uint32_t max_len_val, max_len_gap;
  uint64_t tokens;               /* tokens of this rank's rows, pads included         */
  uint64_t nnz;                  /* real (non-pad) tokens of this rank's rows         */
  uint64_t stream_bytes;         /* ceil(val bits/8) + ceil(gap bits/8) of the shard  */
  uint64_t algo_bytes_fixed;     /* stream + row_ptr + codebook + tables + bias bytes */
  uint64_t index_bytes;          /* every resident restart index (overhead): decode-  */
                                 /* lane records and token starts, interval indices,  */
                                 /* tensor-core list layout, merged-stream lanes      */
  uint64_t ws_bytes;             /* WS(i): device scratch the layer uses     */
  uint64_t in_features, out_features; /* per image                                     */
  uint64_t resident_bytes;       /* every device byte the loaded layer keeps resident */
                                 /* (streams, merged stream, indices, tables, bias)   */
  uint64_t call_index_bytes;     /* index bytes the small-batch kernel (k_fc_j) reads */
                                 /* per call (lane records + row starts)              */
  uint32_t col_begin, col_end;   /* input columns this rank multiplies (column-sharded */
                                 /* FC layers: the rank's K block; else 0, cols)       */
} cdn_layer_stats;

/* ---- library / errors ------------------------------------------------- */
int cdn_abi_version(void);
const char* cdn_last_error(void);

/* ---- multi-GPU bootstrap: rank 0 creates the 128-byte NCCL unique id;
 * the caller broadcasts it (e.g. with torch.distributed).  Errors: CDN_E_NCCL. */
cdn_status cdn_nccl_unique_id(uint8_t out[128]);

/* ---- model lifecycle --------------------------------------------------
 * device: CUDA ordinal; rank/world: this process's place in the row-block
 * sharding (world == 1: single GPU, nccl_id may be NULL).  world > 1 with
 * nccl_id == NULL creates a shard-only handle: it loads rank's row block and
 * serves cdn_layer_forward / cdn_layer_decode, but infer/plan return
 * CDN_E_STATE (used to test sharding on one GPU).  The library owns
 * its device memory, streams and NCCL communicator.  Errors: CDN_E_ARG,
 * CDN_E_CUDA, CDN_E_NCCL, CDN_E_OOM. */
cdn_status cdn_model_create(int device, int rank, int world, const uint8_t* nccl_id,
                            cdn_model** out);
void cdn_model_destroy(cdn_model* m); /* NULL-safe */

/* ---- load compressed layer (the stored model of Fig. 1e) ----
 * cdni/n: host buffer holding a CDNI container (format in DESIGN.md);
 * the bytes are copied, the caller may free them on return.  layer_in_file
 * selects one layer of a multi-layer file.  Layers are appended in network
 * order; shapes are validated against the previous layer.  Each rank keeps
 * only its block of output rows; the streams are sliced at row_ptr bit
 * offsets, never re-encoded.  Load builds the decode-lane index (DESIGN.md
 * "container") on the host and copies everything to the device once.
 * Errors: CDN_E_MAGIC, CDN_E_VERSION, CDN_E_TRUNCATED, CDN_E_MALFORMED,
 * CDN_E_UNSUPPORTED, CDN_E_SHAPE, CDN_E_OOM, CDN_E_CUDA. */
cdn_status cdn_model_load_layer(cdn_model* m, const void* cdni, size_t n, int layer_in_file,
                                const cdn_layer_desc* desc, int* layer_idx);

/* ---- memory budget (P:L651 TOT; P:L724-726 latency threshold) ----------
 * tot_bytes counts activations + workspace per GPU, EXCLUDING the resident
 * compressed model.  latency_ms <= 0: no threshold.  Invalidates the
 * cached plan.  Errors: CDN_E_ARG. */
cdn_status cdn_model_set_memory_budget(cdn_model* m, uint64_t tot_bytes, double latency_ms);

/* ---- plan: profiles Time(i,B) on the device for B = 1..K
 * (cached), runs the variable-batch DP and returns the per-layer batch sizes
 * of the first round (batch_per_layer has n_layers entries) and the predicted
 * total time for all K inputs including remainder re-plans.
 * Errors: CDN_E_INFEASIBLE, CDN_E_CUDA, CDN_E_STATE. */
cdn_status cdn_model_plan(cdn_model* m, int K, int* batch_per_layer, double* predicted_ms);

/* Use a fixed plan instead of the DP (batch sizes must form a divisor chain
 * B_1 | B_2 | ... | B_f).  n == 0 clears it. */
cdn_status cdn_model_set_plan(cdn_model* m, const int* batch_per_layer, int n);

/* ---- infer(batch) -> class scores --------------------------------------
 * input : fp32, image-major: [K][features] for FC-only nets, [K][H][W][C] NHWC
 *         for conv nets.  Host or device memory per on_device.
 * scores: fp32 [K][classes] raw (no softmax), host or device per on_device.
 * Runs the planned per-layer batches with B/b phases.  Under
 * world > 1 every rank calls it with the same input; only rank 0's scores are
 * written.  stream: cudaStream_t or NULL.  Errors: CDN_E_SHAPE,
 * CDN_E_INFEASIBLE, CDN_E_CUDA, CDN_E_NCCL, CDN_E_STATE. */
cdn_status cdn_model_infer(cdn_model* m, const float* input, int K, float* scores, int on_device,
                           void* stream);

/* ---- one layer on device-resident, feature-major activations ------------
 * x: device [in_features][ldx] fp32 (column b = image b), y: device
 * [rows of this rank][ldy] fp32.  B images.  The hot path of one layer
 * (parallel Huffman decode -> gap prefix sum -> codebook dequantize -> sparse
 * multiply -> bias -> ReLU) in the fused kernels; used by infer, the profiler,
 * parity tests and bench.  Errors: CDN_E_ARG, CDN_E_CUDA. */
cdn_status cdn_layer_forward(cdn_model* m, int layer, const float* x, int ldx, int B, float* y,
                             int ldy, void* stream);

/* ---- one CONV layer on a device-resident NHWC batch ----
 * x: device fp32 [B][in_h][in_w][in_c] (NHWC), y: device fp32
 * [B][out_h][out_w][rows] with out_* from cdn_layer_out_shape.  The layer's
 * compressed filters are Huffman-decoded to a dense bf16 matrix (RNE of the
 * codebook value, reading C-21), the input is unfolded to bf16 patches with K
 * order (r, s, c) per group (C-18), the contraction runs on tcgen05 tensor
 * cores with fp32 accumulation, then bias, ReLU, LRN (C-20) and max-pool as
 * the descriptor asks.  Every rank holds all filters
 * (CONV layers are replicated).  Errors: CDN_E_ARG (not a CONV layer),
 * CDN_E_CUDA, CDN_E_OOM. */
cdn_status cdn_conv_forward(cdn_model* m, int layer, const float* x, int B, float* y, void* stream);
/* Output geometry of a layer per image: CONV -> (out_h, out_w, filters) after
 * the optional pool; FC -> (1, 1, rows).  Errors: CDN_E_ARG. */
cdn_status cdn_layer_out_shape(const cdn_model* m, int layer, int* out_h, int* out_w, int* out_c);
/* Test hook of the tcgen05 GEMM: out[i*ldo + n] = act(sum_k A[i][k] Wt[n][k] + bias[n])
 * with A [M][Kpad], Wt [N][Kpad] bf16 (device, K contiguous, Kpad % 64 == 0),
 * bias [N] fp32, out fp32 (device).  Errors: CDN_E_ARG, CDN_E_CUDA. */
cdn_status cdn_debug_gemm_bf16(const void* A, int M, const void* Wt, int N, int Kpad, const float* bias, int relu,
                               float* out, int ldo, void* stream);
/* Number of CUDA kernels this library has launched since it was loaded (all
 * models, all threads; a host-side counter, no device work).  *out receives
 * the count.  Errors: CDN_E_ARG (null out). */
cdn_status cdn_debug_kernel_launches(uint64_t* out);
/* Kernel timer (measurement hook): enable != 0 starts recording, 0 stops;
 * either way the previous records are dropped.  While on, the library brackets
 * each launch of its main kernels (k_fc_tc, k_tc_list, k_split_x, k_fc_band,
 * k_fc_ms, k_fc_fold) with CUDA events on the launch stream.  Errors: none. */
cdn_status cdn_debug_kernel_timer(int enable);
/* Sum of the recorded durations of `kernel` (ms) and the number of launches
 * recorded; waits for the recorded events.  Errors: CDN_E_ARG, CDN_E_CUDA. */
cdn_status cdn_debug_kernel_timer_read(const char* kernel, double* total_ms, int* launches);

/* ---- FC kernel policy (tuning / parity hook) ---------------------------
 * tc_min_batch: batches B >= this run the tensor-core kernel (W tiles decoded
 * into shared memory, 3-pass bf16 split tcgen05 contraction, fp32 accumulate);
 * band_min_batch: batches B >= this (and below tc_min_batch) run the
 * warp-specialised CUDA-core band kernel (when x meets its TMA alignment rule:
 * ldx % 4 == 0, x 16-byte aligned); smaller batches the small-batch kernels.
 * <= 0 restores a default (env CDN_TC_MIN_B else off; env CDN_BAND_MIN_B else
 * 16).  All kernels compute the same layer; they differ in summation order and,
 * for the tensor-core kernel, in the 2^-16-level split of operands
 * (DESIGN.md §9).  Errors: CDN_E_ARG. */
cdn_status cdn_model_set_kernel_policy(cdn_model* m, int band_min_batch, int tc_min_batch);

/* ---- decode only (parity hook, kernel K2) -------------------------------
 * Writes every token of this rank's rows in row-major token order, pads
 * included: row, abs column (Alg. 1 l.7), val symbol, codebook value (l.8).
 * Device pointers; call first with all four NULL to get *n_tokens.
 * Errors: CDN_E_ARG, CDN_E_CUDA. */
cdn_status cdn_layer_decode(cdn_model* m, int layer, int32_t* row, int32_t* col, uint8_t* sym,
                            float* val, uint64_t* n_tokens, void* stream);

cdn_status cdn_model_num_layers(const cdn_model* m, int* n);
cdn_status cdn_layer_stats_get(const cdn_model* m, int layer, cdn_layer_stats* out);

/* ---- profiler: Time(i,B) for B = 1..Bmax, ms (median of reps), written to
 * time_ms[i*Bmax + (B-1)].  Errors: CDN_E_CUDA, CDN_E_STATE. */
cdn_status cdn_model_profile(cdn_model* m, int Bmax, int reps, double* time_ms);

/* ---- the planner's memory model for batches up to Bmax: per
 * layer IN and OUT bytes per image and WS(i) bytes (readings C-23, C-24), the
 * same numbers cdn_model_plan uses.  Arrays of n_layers.  Errors: CDN_E_ARG. */
cdn_status cdn_model_memory_model(cdn_model* m, int Bmax, uint64_t* in_bytes, uint64_t* out_bytes,
                                  uint64_t* ws_bytes);

/* ---- sharding of the FC layers across ranks (call before loading layers):
 * CDN_SHARD_ROWS (default): rank r keeps a contiguous block of
 * output rows; layer outputs are all-gathered.  CDN_SHARD_COLS (Megatron-style,
 * SURVEY §8(f) row 4): rank r multiplies a contiguous block of input columns
 * (K tiles of 64) for every output row; the partial sums are reduce-scattered
 * into the next layer's column blocks (bias and ReLU applied after the sum)
 * and reduced to rank 0 after the last layer -- the first layer reads only its
 * column block of the input.  Column-sharded layers run the tensor-core path;
 * cdn_layer_forward on such a layer returns the rank's partial sums (no bias,
 * no ReLU) from its column block of x ([col_end - col_begin][ldx]).
 * Errors: CDN_E_ARG, CDN_E_STATE (layers already loaded). */
#define CDN_SHARD_ROWS 0
#define CDN_SHARD_COLS 1
cdn_status cdn_model_set_sharding(cdn_model* m, int mode);

/* The column block [*k0, *k1) rank `rank` of `world` multiplies in a
 * column-sharded layer with `cols` input columns (host only). */
cdn_status cdn_col_block(uint32_t cols, int rank, int world, uint32_t* k0, uint32_t* k1);

/* ---- inference scratch (the memory TOT bounds: everything but the
 * resident compressed model -- level activation buffers, workspaces, per-call
 * decoded lists / filters, staging): bytes allocated now and the high-water
 * mark since the model was created or the peak last reset (reset_peak != 0
 * sets it to the current bytes after reading).  Under a memory budget the
 * planner only runs plans whose executor scratch fits TOT (reading C-36).
 * Either output may be NULL.  Errors: CDN_E_ARG. */
cdn_status cdn_model_scratch_bytes(cdn_model* m, uint64_t* current, uint64_t* peak, int reset_peak);

/* Free every inference-scratch buffer of the model (the next call allocates
 * what its plan needs); waits for the model's streams.  Errors: CDN_E_ARG,
 * CDN_E_STATE (a call in progress), CDN_E_CUDA. */
cdn_status cdn_model_release_scratch(cdn_model* m);

/* Name of the kernel a layer launches for batch B under the current policy
 * (after the first-use autotune at that B, if any): "k_fc_j" (B <= 4),
 * "k_fc_ms", "k_fc_fold", "k_fc_band<V>", "k_fc_tc", "k_gemm_bf16 (conv)" or
 * "k_gemm_bf16 (conv, implicit im2col)";
 * "" for bad arguments.  The string is static. */
const char* cdn_layer_kernel_name(const cdn_model* m, int layer, int B);

/* ---- host-only utilities (no device needed) ----------------------------- */

/* Compress a dense fp32 row-major rows x cols matrix: magnitude
 * prune to floor(density*rows*cols + 0.5) entries (C-10), r-bit linear
 * codebook (C-04/05/07), k-bit relative index with pads (C-01..03), Huffman
 * per stream (C-14..17).  bias may be NULL.  *out receives a malloc'd
 * single-layer CDNI buffer the caller frees with cdn_free.
 * Errors: CDN_E_ARG, CDN_E_UNSUPPORTED, CDN_E_OOM. */
cdn_status cdn_compress_dense(const float* W, const float* bias, uint32_t rows, uint32_t cols,
                              double density, int r, int k, void** out, size_t* out_len);
/* As cdn_compress_dense with a choice of quantizer and storage order.
 * quantizer: 0 = the linear codebook above (C-05), 1 = 1-D Lloyd k-means
 * refined from that grid (C-33: binary64 nearest-centre assignment with ties
 * to the smaller index, binary64 means in row-major order, <= 50 iterations or
 * until no centre moves by more than 1e-7 max(|lo|,|hi|)).
 * bh x bw: 1 x 0 (0 = cols) is the plain row-major container; otherwise the
 * block-contiguous container of Alg. 2 (C-34): rows % bh == 0,
 * cols % bw == 0, relative indexing / Huffman / row_ptr over the stored rows
 * of M' (block (bi, bj) flattened row-major = stored row bi*(cols/bw) + bj).
 * Errors: as above, CDN_E_ARG for another quantizer or a non-tiling block. */
cdn_status cdn_compress_dense_q(const float* W, const float* bias, uint32_t rows, uint32_t cols, double density,
                                int r, int k, int quantizer, uint32_t bh, uint32_t bw, void** out, size_t* out_len);
void cdn_free(void* p);

/* Variable-batch DP of P:L694-720 on a given table (host).  time_ms[i*Bmax + B-1]
 * = Time(i,B); in/out bytes per image; ws bytes per layer; tot; latency (<=0:
 * none); step: memory-axis granularity in bytes (A + IN rounded UP, C-25).
 * Outputs the batch per layer and OPT(f,B*,0).  Errors: CDN_E_INFEASIBLE. */
cdn_status cdn_plan_dp(const double* time_ms, const uint64_t* in_bytes, const uint64_t* out_bytes,
                       const uint64_t* ws_bytes, int f, int Bmax, uint64_t tot, double latency_ms,
                       uint64_t step, int* batches, double* opt_ms);

/* Parse + validate a CDNI layer and run the load-time host walk that builds
 * the decode-lane index; returns the tokens it walked (test hook for the
 * container builder; not used by inference).  Call with NULL outputs to get
 * *n_tokens.  row/col int32, sym uint8 (host). */
cdn_status cdn_debug_host_walk(const void* cdni, size_t n, int layer_in_file, int32_t* row,
                               int32_t* col, uint8_t* sym, uint64_t* n_tokens);

/* The same host walk on the row-block shard of `rank` out of `world`
 * (ceil(rows/world) rows per rank): the shard's stream bytes are
 * cut at word-aligned bit positions and its row_ptr rebased exactly as
 * cdn_model_load_layer does, then walked; rows are reported as global row
 * indices.  Host-only (multi-rank sharding logic is tested on CPU with it). */
cdn_status cdn_debug_host_walk_shard(const void* cdni, size_t n, int layer_in_file, int rank, int world,
                                     int32_t* row, int32_t* col, uint8_t* sym, uint64_t* n_tokens);

#ifdef __cplusplus
}
#endif
#endif /* CDN_H_ */
