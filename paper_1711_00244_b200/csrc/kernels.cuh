// Device-side data of one loaded FC/CONV weight matrix (a rank's row block)
// and the kernel launchers.  Layout rationale: DESIGN.md "Data layout in HBM".
#pragma once
#include <atomic>
#include <cstdint>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace cdn {

// kernels this library has launched (cdn_debug_kernel_launches): every launcher
// returns through launched(n) right after its n launches
extern std::atomic<unsigned long long> g_launches;
inline cudaError_t launched(int n = 1) {
  g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Debug kernel timer (cdn_debug_kernel_timer): when enabled, the launchers
// bracket their main kernel with CUDA events on the launch stream, so a caller
// can read each kernel's live duration inside its own workload.
void ktimer_begin(const char* kernel, cudaStream_t s);
void ktimer_end(const char* kernel, cudaStream_t s);
void ktimer_enable(bool on);  // (re)starts with no records
bool ktimer_active();
cudaError_t ktimer_read(const char* kernel, double* total_ms, int* launches);

constexpr int kLutMaxBits = 10;   // plain LUT width cap (decode kernel); longer codes take the canonical slow path
constexpr int kTcChunk = 8;       // max K tiles per decode task of the tensor-core path's list decoder
constexpr int kFoldLutBits = 11;  // pad-folding val LUT width (fused forward)
constexpr uint32_t kFoldSlow = 0xFFFFFFFFu;
constexpr int kMaxBatchTiles = 1024;

struct FcDev {
  const uint32_t* vw = nullptr;      // val stream as big-endian u32 words (bit i = bit 31-(i%32) of word i/32)
  const uint32_t* gw = nullptr;      // gap (col_ind) stream, same packing
  const uint32_t* rp = nullptr;      // 2*(nrows+1): (val bit, gap bit) at each local row start (row_ptr)
  const void* rec = nullptr;         // nrows*G lane records (u32 or u64, see host.hpp LaneIndex)
  const uint64_t* tok_start = nullptr;  // nrows*G+1 token index per lane (decode kernel only)
  const uint32_t* vlut = nullptr;    // 2^Lv entries: (len << 16) | sym, 0 = longer code
  const uint32_t* glut = nullptr;    // 2^Lg entries
  const uint32_t* vtab = nullptr;    // [0..32] first_code, [33..65] count, [66..98] first_index
  const uint32_t* gtab = nullptr;
  const uint16_t* vsorted = nullptr; // symbols in canonical order
  const uint16_t* gsorted = nullptr;
  const uint32_t* flut = nullptr;    // 2^Lf pad-folding entries: sym | len<<8 | pads<<13 | has<<18, or kFoldSlow
  int* ctr = nullptr;                // kMaxBatchTiles work counters (dynamic row scheduling)
  const float* codebook = nullptr;   // 2^r fp32 centres, [0] = 0.0 (pads)
  const float* bias = nullptr;       // nrows fp32 (zeros if absent)
  int nrows = 0, cols = 0;
  int G = 1, log2G = 0, W = 1;       // lanes per row, lane column width
  int k = 4, Lv = 1, Lg = 1, vmax = 0, gmax = 0;
  int ncb = 32, nvs = 0, ngs = 0;
  int rec64 = 0;
  int Lf = 1, Lpg = 0;               // folding LUT width; code length of the pad gap symbol 2^k-1
  // large-batch band kernel: interval restart index (host.hpp IntervalIndex),
  // nrows x NI entries: (val bit, gap bit) relative to the slice words, and
  // (dm1 | nnz << 8): previous column = i*Wi - (dm1+1), real tokens in interval
  const uint2* ivg = nullptr;
  const uint16_t* ivm = nullptr;
  int Wi = 64, NI = 0;               // interval width (= band width), intervals per row
  int Cint = 16;                     // intervals per decode chunk
  // tensor-core FC kernel (tc.cu): interval index with Wi = 64 (the K tile);
  // aliases ivg/ivm when the band index already uses Wi = 64
  const uint2* tivg = nullptr;
  const uint16_t* tivm = nullptr;
  int tNI = 0;                       // 64-column K tiles of the weight matrix (list blocks, contraction)
  int sNI = 0;                       // 64-position intervals per stored row
  int sNC = 0;                       // list-decoder chunks per stored row (tivg / tivm rows: the chunk starts)
  // Block-contiguous container (Alg. 2, C-34): nrows / cols above are the
  // STORED matrix's (blocks of M' when blocked); the weight matrix is
  // wrows x wcols in bh x bw blocks, stored row i = block (i / (wcols/bw),
  // i % (wcols/bw)).  Unblocked: bh = 1, bw = wcols = cols, wrows = nrows.
  int wrows = 0, wcols = 0, bh = 1, bw = 0;
  // decoded-entry list between the tensor-core path's two kernels: entry =
  // (column - 64 kt) | codebook index << 6, one per real token, in blocks of
  // (128-row tile rt, K tile kt) at tbase[rt * tNI + kt], rows in order inside,
  // row r at troff[(rt * tNI + kt) * 129 + r] ([128]: the block's count)
  const uint32_t* tbase = nullptr;
  const uint16_t* troff = nullptr;
  uint16_t* tlist = nullptr;
  int tch = kTcChunk;                // K tiles per list-decoder task (fewer for small / dense layers)
  // small-batch multi-symbol LUTs (small.cu): 2^msLv / 2^msLg entries
  const uint32_t* msv = nullptr;
  const uint32_t* msg = nullptr;
  int msLv = 12, msLg = 12;
  float tc_wsc = 1.f;                // tensor-core path: power-of-two weight scale of the fp16 split
  // merged-stream small-batch kernel (joint.cu; host.hpp JointIndex): words,
  // row start bits (nrows + 1), token-balanced lane records (nrows * G), joint LUT
  const uint32_t* jw = nullptr;
  const uint32_t* jrow = nullptr;
  const uint32_t* jlane = nullptr;
  // CONV filter decode (k_decode_conv): cG lanes per row of cols / cG columns,
  // per lane {val bit, gap bit, previous column + 1, tokens} (absolute restart
  // states: no prefix scan, so a row spreads over any number of threads), and
  // the dense-W position of each decoded K index (padded / space-to-depth order)
  const uint4* clane = nullptr;
  int cG = 0;
  const int* kmap = nullptr;
  const uint32_t* jlutr = nullptr;  // the same blob with the joint LUT in k_fc_j's entry layout (build_joint_lut_r),
  uint32_t jlhash = 0;               // entry of index i at i ^ ((i >> 5) & jlhash)
  const uint32_t* jlut = nullptr;   // the kernel's tables as one blob, laid out as in shared memory:
  int jL = 12;                       // [joint LUT 4<<jL | vlut | glut | vtab | gtab | vsorted | gsorted | codebook]
  uint32_t jo_vlut = 0, jo_glut = 0, jo_vtab = 0, jo_gtab = 0, jo_vs = 0, jo_gs = 0, jo_cb = 0, jblob = 0;
  uint32_t jsub = 0;                 // bytes of one row's staging sub-slot
  int jG = 1;                        // lanes per row of the merged-stream split
  int jQ = 1, jKq = 0;               // column groups of the lane split, group width (columns)
  float* jpart = nullptr;            // column-group partial sums [Q][nrows][BS]
  int* jctr = nullptr;               // per-warp-unit arrival counters (Q > 1), zero between calls
  // medium-batch split of the same stream (5 <= B <~ 128, joint.cu plan_fc_jm):
  // one lane per (row, column group), jmQ groups of jmKq columns, so a CTA's
  // x slice holds 32 images
  const uint32_t* jmlane = nullptr;  // nrows * jmQ lane records
  const uint16_t* jmperm = nullptr;  // [jmQ][nrows]: rows of each group by decreasing bits within blocks of
                                     // kJmSortRows (a warp's lanes then run about equally many steps)
  int jmQ = 0, jmKq = 0;
  int jmupc = 1;                     // warp units (32 rows) per CTA: rows sorted within these ranges
  uint32_t jmsub = 0;                // bytes of one (row, group) staging sub-slot
  const uint32_t* jmlut = nullptr;   // its table blob (the jlut layout with a narrower joint LUT, jmL bits:
  uint32_t jmblob = 0;               // small enough for two CTAs per SM)
  int jmL = 12;
  uint32_t jmo_vlut = 0, jmo_glut = 0, jmo_vtab = 0, jmo_gtab = 0, jmo_vs = 0, jmo_gs = 0, jmo_cb = 0;
};

// Launch plan of the merged-stream kernel for one (layer, B <= 4).
struct JPlan {
  bool ok = false;
  bool medium = false;  // the medium-batch split (jm*): image groups of BS on grid z, partials + k_j_reduce
  int BS = 1, Q = 1, GQ = 1, RPW = 1, units = 0, nw = 1, nrb = 0, nbg = 1, Bp = 1;
  int upc = 0;          // medium: warp units per CTA (its warps take them dynamically)
  bool jbig = false;    // medium: stages the small-batch kernel's table blob (wider joint LUT), else jmlut
  uint32_t sub = 0, off_x = 0, off_slot = 0;
  size_t smem = 0;
  std::vector<uint2> cta;  // Q == 1: per CTA (16-byte index of its rows' first bits, bytes to stage)
  int wpr = 1;             // k_fc_j: warps per row (G > 32)
};
bool j_supported(const FcDev& L);
// row_bit: the host copy of L.jrow (nrows + 1), for the per-CTA stream ranges
JPlan plan_fc_j(const FcDev& L, int B, int num_sms, const uint32_t* row_bit);
// part: medium plans with Q > 1, jm_part_bytes(L, p) of scratch (else unused)
cudaError_t launch_fc_j(const FcDev& L, const JPlan& p, const float* x, int ldx, int B, float* y, int ldy, int relu,
                        cudaStream_t s, float* part = nullptr);
bool jm_supported(const FcDev& L);
// part_cap: largest partial-sum buffer a launch may use (image groups beyond
// it run in further launches); the caller launches ceil(B / Bp) times
JPlan plan_fc_jm(const FcDev& L, int B, int num_sms, size_t part_cap);
size_t jm_part_bytes(const FcDev& L, const JPlan& p);

// Launch plan of the band kernel for one (layer, B, x) — ok == false means the
// inputs do not meet its alignment rules (the small-batch kernel then runs).
struct BandPlan {
  bool ok = false;
  int vec = 4, nbt = 1, S = 1, nchunks = 0, units = 0, tiles = 0, grid = 0, ipb = 1;
  size_t ws_floats = 0, smem = 0;
};
BandPlan plan_fc_band(const FcDev& L, const float* x, int ldx, int B, int num_sms);
cudaError_t launch_fc_band(const FcDev& L, const BandPlan& p, const float* x, int ldx, int B, float* y, int ldy,
                           int relu, float* ws, int* tctr, cudaStream_t s);
// Tensor-core FC kernel (tc.cu, B >= ~16): decode W tiles into tensor memory,
// 3-pass fp16 split (per-image / per-layer power-of-two scales) tcgen05 contraction.
struct TcPlan {
  bool ok = false;
  int nbt = 1, nrt = 1, nkt = 0, ldk = 0, tiles = 0, grid = 0, mpt = 1;  // mpt: max CTAs per tile
  int tn = 256;  // images per tile (UMMA N): 128 when the batch fits one
  int kbase = 0, kcols = 0;  // first K tile and K columns of the call (column-sharded layers: the rank's block)
  long W = 0;  // tile steps (stream-K split over `grid` CTAs)
  size_t ws_floats = 0, xsplit_elems = 0, smem = 0;
};
bool tc_supported(const FcDev& L);
// K tiles [kt0, kt1) only (kt1 < 0: all): a column-sharded layer's block
TcPlan plan_fc_tc(const FcDev& L, int B, int num_sms, int kt0 = 0, int kt1 = -1);
// list decoder of the tensor-core path (k_tc_list[_ms]): fills L.tlist from the
// compressed streams; launch_fc_tc reads it (the caller orders the two)
cudaError_t launch_tc_list(const FcDev& L, cudaStream_t s, int kt0 = 0, int kt1 = -1);
// xh / xl: fp16 hi / lo scratch [B][ldk]; scw: tc_scale_floats(B) floats (per-image split
// scales); xctr: >= B ints, zero at allocation (the kernels leave them zero)
size_t tc_scale_floats(int B);
cudaError_t launch_fc_tc(const FcDev& L, const TcPlan& p, const float* x, int ldx, int B, float* y, int ldy, int relu,
                         uint16_t* xh, uint16_t* xl, float* ws, float* scw, int* xctr, cudaStream_t s,
                         bool x_image_major, bool y_image_major,
                         const float* bias,
                         const float* xrg_in = nullptr, int nrg_in = 0, float* xrg_out = nullptr);  // x: [kcols][ldx] feature-major, or [B][ldx] image-major (the plan's K
                                              // columns); bias null: partial sums without bias / ReLU

// Small-batch multi-symbol kernel (B <= 8; r <= 5, k <= 4, 32-bit lane records).
bool ms_supported(const FcDev& L);
size_t ms_smem_bytes(const FcDev& L);  // dynamic smem of the multi-symbol LUT kernels
cudaError_t launch_fc_ms(const FcDev& L, const float* x, int ldx, int B, float* y, int ldy, int relu, cudaStream_t s,
                         int num_sms);
int band_rows_per_unit();
int band_list_capacity();
int band_max_chunk();

// y[r][b] = act( sum_j W_q[r][j] x[j][b] + v[r] ) for the rank's rows, B images,
// feature-major activations (x: [cols][ldx], y: [nrows][ldy]).
cudaError_t launch_fc_forward(const FcDev& L, const float* x, int ldx, int B, float* y, int ldy,
                              int relu, cudaStream_t s, int num_sms);

// Every token of the rank's rows (pads included) -> row (global index), column,
// val symbol, codebook value.  row_offset converts local to global rows.
cudaError_t launch_decode(const FcDev& L, int row_offset, int32_t* row, int32_t* col, uint8_t* sym,
                          float* val, cudaStream_t s, int num_sms);

// [B][K] image-major -> [K][ldo] feature-major (and the reverse).
cudaError_t launch_transpose(const float* in, int rows, int cols, int ldi, float* out, int ldo,
                             cudaStream_t s);

size_t fc_smem_bytes(const FcDev& L);

// dst[r][b] = act(src[r][b] + bias[r0 + r]) (bias rows >= nbias add 0): the
// reduce-scattered block of a column-sharded layer -> the next layer's input
cudaError_t launch_bias_act(const float* src, int rows, int B, int lds, const float* bias, int r0, int nbias, int relu,
                            float* dst, int ldd, cudaStream_t s);

// ---- CONV path (conv.cu)
// Decode the rank's rows into dense bf16 W[row][col] (zero-filled by caller).
// cg / cgp: channels per group and their padding per tap (implicit-GEMM layers;
// column (r*kw + s)*cg + c lands at (r*kw + s)*cgp + c); 0: no remap
cudaError_t launch_decode_dense(const FcDev& L, __nv_bfloat16* W, int ldw, cudaStream_t s, int num_sms, int cg = 0,
                                int cgp = 0, const int* kmap = nullptr);
// NHWC fp32 -> bf16 patches [B*Ho*Wo][Kpad] of channels [c0, c0+cg), k = (r*kw+s)*cg + c.
cudaError_t launch_im2col(const float* x, int B, int H, int W, int C, int kh, int kw, int stride, int pad, int c0,
                          int cg, int Ho, int Wo, int Kreal, int Kpad, __nv_bfloat16* out, cudaStream_t s,
                          int num_sms);
// tcgen05 GEMM: out[pos*ldo + col0 + n] = act(sum_k A[pos][k] Wt[n][k] + bias[n]); Kpad % 64 == 0.
int gemm_tile_n(int Nrows);  // N tile of the conv GEMM (<= 256)
cudaError_t launch_gemm_bf16(const __nv_bfloat16* A, int Mrows, const __nv_bfloat16* Wt, int Nrows, int Kpad,
                             const float* bias, int relu, float* out, int ldo, int col0, cudaStream_t s,
                             int lrn = 0, int groups = 1);
cudaError_t launch_lrn(const float* x, long npos, int C, float* y, cudaStream_t s, int num_sms);
// Implicit-GEMM CONV (stride 1, channel groups of cg padded to cgp = 64k):
// x fp32 NHWC [npix][C] -> bf16 [npix][G * cgp] (channels of a group padded with
// zeros), then the tcgen05 GEMM with its activation tiles loaded by TMA in
// im2col mode from that tensor (no patch matrix).
cudaError_t launch_to_bf16_pad(const float* x, long npix, int C, int G, int cg, int cgp, __nv_bfloat16* out,
                               cudaStream_t s);
// CONV filters decoded into dense bf16 W[row][kmap[col]] (the caller zero-fills
// W) over the per-lane restart states L.clane (a thread per lane)
cudaError_t launch_decode_conv(const FcDev& L, __nv_bfloat16* W, int ldw, cudaStream_t s);
// a one-warp kernel spinning ~ns nanoseconds on the GPU clock (autotune timing)
cudaError_t launch_spin(cudaStream_t s, long long ns);
// space-to-depth (strided CONV as a stride-1 one): x fp32 NHWC [B][H][W][C] ->
// bf16 [B][Hs][Ws][cgp], channel (dy * s + dx) * C + c of super-pixel (Y, X) =
// x[4Y+dy][4X+dx][c] for s = 4 (zero outside the image / past s*s*C)
cudaError_t launch_s2d_bf16(const float* x, int B, int H, int W, int C, int st, int Hs, int Ws, int cgp,
                            __nv_bfloat16* out, cudaStream_t s);
cudaError_t launch_gemm_implicit(const __nv_bfloat16* act, int B, int H, int W, int G, int cgp, int kh, int kw,
                                 int pad, int Ho, int Wo, const __nv_bfloat16* Wt, int Nrows, const float* bias,
                                 int relu, float* out, int ldo, cudaStream_t s, int lrn,
                                 __nv_bfloat16* out_bf = nullptr, int cg_real = 0);
// (cg_real: real channels per group, <= cgp; the filters' and the input's channels past it are zeros)
// whether the halo-tile kernel (the only one with a bf16 output: out_bf) takes the layer
bool conv_halo_applies(int G, int cgp, int kh, int kw, int pad, int Ho, int Wo, int Nrows, int lrn);
// max-pool (+ LRN ahead of it when lrn), 8 channels per thread; output fp32 NHWC
// (y) or, when yb, bf16 with G groups of cg channels padded to cgp (the next
// CONV layer's input).  pool8_ok: the shapes it takes (cg = 0: fp32 output)
bool pool8_ok(int C, int k, int cg, int cgp);
cudaError_t launch_pool8(const float* x, int B, int H, int W, int C, int k, int st, int lrn, float* y,
                         __nv_bfloat16* yb, int G, int cg, int cgp, cudaStream_t s, int num_sms);
cudaError_t launch_maxpool(const float* x, int B, int H, int W, int C, int k, int st, float* y, cudaStream_t s,
                           int num_sms);

}  // namespace cdn
