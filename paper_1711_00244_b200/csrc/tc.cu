// Tensor-core FC path for large batches, sm_100a:
// PAPER.md Alg. 1 lines 4-9, Eq. 1-2, as two kernels.
//
//  1. k_tc_list -- the bit-serial part (Huffman decode of both streams, gap
//     prefix sum), in parallel over (row, 8-tile chunk) tasks from the Wi = 64
//     restart index: one u16 entry (column - 64 kt) | codebook index << 6 per
//     real token, rows in order.  Done ONCE per call, whatever the batch
//     (the 2 B / nonzero list is per-call scratch; it is re-derived from the
//     compressed streams on every forward).
//  2. k_fc_tc -- dequantize + contraction: the W tile (128 rows x 64 K) is
//     rebuilt from the list in REGISTERS and stored straight into tensor
//     memory (tcgen05.st), where the UMMA reads it as its A operand; only the
//     activation tile goes through shared memory (TMA).  Shared-memory
//     bandwidth is the bound of an M = 128 UMMA pipeline, so keeping W out of
//     it (no zero fill, no scatter, no A-operand reads) is the point.
//
// At B >= 128 the sparse CUDA-core kernel is bound by one shared-memory load
// per FMA; the tensor cores run the DENSE tile product 25x faster per flop, so
// even at 4% density they win.  fp32 fidelity with 16-bit tensor cores: every
// weight (codebook value) and activation is split into two fp16 halves,
// hi = fp16(v s) and lo = fp16(v s - hi), after scaling by a power of two s
// (per layer for W, per image for X: max |v| s in [2^14, 2^15), so hi never
// overflows and lo stays normal for every value within 2^-17 of the maximum);
// D += Whi*Xhi + Whi*Xlo + Wlo*Xhi (three UMMAs per K step, kind::f16 with
// fp16 operands), and the epilogue multiplies by 1 / (s_W s_b) (exact).  A
// 2-way fp16 split keeps 22 significant bits; each product is within ~2^-21
// relative of the fp32 product (the dropped lo*lo term and the two splits),
// against 2^-15 for a bf16 split.
//   unit = (128 output rows, 256 images, K range), split in two K halves
//   ("streams") expanded concurrently; per 64-column K tile:
//     * 4 EXPAND warps per stream, one lane per row (= TMEM lane): the lane
//       walks its row's entries, builds each 8-column chunk of bf16 hi / lo in
//       4 + 4 registers and tcgen05.st's them into the stream's free W buffer
//       (2 per stream, 64 TMEM columns each: hi 32 | lo 32);
//     * warp 0 / lane 0: TMA of the Xhi / Xlo tiles [256 images][64 K] into a
//       3-stage shared-memory ring (consumption order);
//     * warp 1 / lane 0: 12 x tcgen05.mma.cta_group::1.kind::f16 (M=128,
//       N=256, K=16, A from TMEM) into the fp32 accumulator (TMEM columns
//       0-255); commits free the X stage and the W buffer;
//     * 4 EPILOGUE warps: tcgen05.ld -> + bias -> ReLU -> y (or a K-split
//       partial, reduced in fixed order by the last CTA of the tile).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dev_common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"
#include "tmap.hpp"

namespace cdn {

namespace {

using namespace dev;

constexpr int kTM = 128;            // rows per unit (UMMA M)
constexpr int kTN = 256;            // images per unit (UMMA N); 128 for B <= 128, 64 for B <= 64 (TN template)
constexpr int kTK = 64;             // K tile (= interval width of the TC index)
constexpr int kXStages = 3;         // X ring depth
constexpr int kEnt = 16;            // list entries per row tile carried in registers (the rest: loads)
constexpr int kRowBytes = 128;      // expand lane's private row: 64 bf16 (chunk-swizzled)
constexpr int kDecW = 4;            // expand warps per K stream: 4 lane quarters (x {bf16 hi, lo} if 8)
constexpr int kHalvesPerWarp = 8 / kDecW;  // bf16 halves (hi, lo) each expand warp builds
constexpr int kStreams = 2;         // K halves of a unit expanded concurrently
constexpr int kWBufs = 2;           // TMEM W buffers per stream
constexpr int kWCols = 64;          // TMEM columns per W buffer: hi 32 | lo 32
constexpr int kEpiW = 4;            // epilogue warps
constexpr int kTThreads = (2 + kStreams * kDecW + kEpiW) * 32;   // 448
constexpr int kTmemCols = 512;      // accumulator 256 + W buffers 4 x 64

struct TcArgs {
  float* y;
  int ldy, B, relu;
  float* ws;   // [tiles][mpt][TN / 4][128] float4 partials of split tiles, summed by k_tc_reduce
  int nbt, nrt, nkt, G, mpt;  // batch tiles, row tiles, K tiles, CTAs, max pieces per tile
  long W;                     // total tile steps = tiles * nkt (stream-K)
  unsigned long long* trace;    // debug (env CDN_TC_TRACE): CTA 0 event clocks [event][256], else null
  int yt;                       // 1: y image-major [B][ldy] (the class scores of the last layer), else [rows][ldy]
  const float* xsc;             // [2B] per-image power-of-two scales of the fp16 split and their inverses (k_xscale_*)
  float winv;                   // 1 / the layer's weight scale
  int kbase;                    // first K tile of this call (column-sharded layers: the rank's K block)
  const float* bias;            // added in the epilogue; null: partial sums (column-sharded layers)
  float* xrg;                   // non-null: max |y| per (32-row group, image), [row group][B], for the next split
};

__device__ __forceinline__ void tc_trace(const TcArgs& a, int ev, int i) {
  if (a.trace != nullptr && blockIdx.x == 0 && i < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[ev * 256 + i] = t;  // ns
  }
}

// List blocks of the intervals j0, j0+1, ... of stored row i, and the weight
// row's slot in each: block (row tile, K tile) of the weight matrix.
// Unblocked (bw = wcols): row i, K tile j.  Blocked (Alg. 2 l.11-12, C-34;
// bw % 64 == 0): block (bi, bj) = (i / nbj, i % nbj); position j*64 -> weight
// row bi*bh + j*64/bw, column bj*bw + j*64 % bw.  One division per task, then
// incremental steps (integer division is ~20 instructions).
template <bool BLOCKED>
struct ListMap {
  int g, kt, c64, bw64, ktb;  // weight row, K tile, 64-block inside the block row, bw/64, first K tile of bj
  __device__ __forceinline__ void init(const FcDev& L, int i, int j0) {
    if (!BLOCKED) {
      g = i;
      kt = j0;
      return;
    }
    const int nbj = L.wcols / L.bw;
    const int bi = i / nbj, bj = i - bi * nbj;
    bw64 = L.bw >> 6;
    const int r = j0 / bw64;
    c64 = j0 - r * bw64;
    g = bi * L.bh + r;
    ktb = bj * bw64;
    kt = ktb + c64;
  }
  __device__ __forceinline__ size_t block(const FcDev& L, int& rr) const {
    rr = g & 127;
    return (size_t)(g >> 7) * L.tNI + kt;
  }
  __device__ __forceinline__ void next() {
    if (!BLOCKED) {
      ++kt;
      return;
    }
    if (++c64 == bw64) {
      c64 = 0;
      ++g;
    }
    kt = ktb + c64;
  }
};

// Stream-K work split: the tiles x nkt tile steps are cut into G equal
// contiguous ranges, one per CTA; a CTA's range falls into one or more pieces
// (tile, K range).  A tile covered by several CTAs is summed by k_tc_reduce
// from ws[tile][i], i = CTA - first CTA of the tile (fixed order).
struct TUnit {
  int rt, bt, kt0, kt1, tile, slot, count;  // slot: index among the tile's pieces; count: pieces of the tile
};

__host__ __device__ __forceinline__ long sk_start(long c, long W, int G) { return c * W / G; }
// CTA whose range holds step x
__host__ __device__ __forceinline__ int sk_cta(long x, long W, int G) { return (int)(((x + 1) * G - 1) / W); }

__device__ __forceinline__ bool cta_piece(const TcArgs& a, int c, int p, TUnit& t) {
  const long s0 = sk_start(c, a.W, a.G), s1 = sk_start(c + 1, a.W, a.G);
  if (s1 <= s0) return false;
  const long tile = s0 / a.nkt + p;
  const long t0 = tile * a.nkt;
  if (t0 >= s1) return false;
  t.tile = (int)tile;
  t.rt = t.tile / a.nbt;
  t.bt = t.tile % a.nbt;
  t.kt0 = (int)((s0 > t0 ? s0 : t0) - t0);
  t.kt1 = (int)((s1 < t0 + a.nkt ? s1 : t0 + a.nkt) - t0);
  const int clo = sk_cta(t0, a.W, a.G);
  t.slot = c - clo;
  t.count = sk_cta(t0 + a.nkt - 1, a.W, a.G) - clo + 1;
  return true;
}

// byte offset of column c in a private row: 16-byte chunk c / 8 swizzled by the
// row, so the 32 lanes of a warp reading chunk j hit 8 distinct chunk slots
__device__ __forceinline__ uint32_t rsw_off(int r, uint32_t c) {
  return (((c >> 3) ^ (uint32_t)(r & 7)) << 4) + ((c & 7u) << 1);
}

__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}

__device__ __forceinline__ void st_u16_if(uint16_t* p, uint32_t v, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.u16 [%0], %1; }" ::"l"(p), "h"((unsigned short)v),
               "r"((uint32_t)pred)
               : "memory");
}

__device__ __forceinline__ void sts_u16_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }" ::"r"(a), "h"((unsigned short)v),
               "r"((uint32_t)p)
               : "memory");
}

__device__ __forceinline__ uint4 lds_u128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}

// stream q's K tiles of unit t: q = 0 the first half, q = 1 the second
__device__ __forceinline__ void stream_range(const TUnit& t, int q, int& k0, int& k1) {
  const int mid = t.kt0 + (t.kt1 - t.kt0 + 1) / 2;
  k0 = q == 0 ? t.kt0 : mid;
  k1 = q == 0 ? mid : t.kt1;
}

template <int TN>
__global__ void __launch_bounds__(kTThreads, 1)
    k_fc_tc(FcDev L, TcArgs a, const __grid_constant__ CUtensorMap txh, const __grid_constant__ CUtensorMap txl) {
  constexpr int kXTile = TN * kTK * 2;      // bf16 X tile [TN images][64 K]
  constexpr int kXStageBytes = 2 * kXTile;  // hi + lo
  extern __shared__ unsigned char smem_raw[];
  // align within the shared window (pointer arithmetic on smem_raw keeps the .shared address space)
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  unsigned char* xst = smem;  // [kXStages]{Xhi, Xlo}
  unsigned char* rows = smem + kXStages * kXStageBytes;  // [stream][128 rows] private zero rows
  uint64_t* xfull = reinterpret_cast<uint64_t*>(rows + kStreams * (kDecW / 4) * kTM * kRowBytes);
  uint64_t* xempty = xfull + kXStages;
  uint64_t* wfull = xempty + kXStages;      // [stream][buf]
  uint64_t* wempty = wfull + kStreams * kWBufs;
  uint64_t* tfull = wempty + kStreams * kWBufs;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  uint32_t* s_cbs = tmem_slot + 4;  // [ncb] bf16 hi | lo << 16
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tc_trace(a, 5, 0);
  {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < L.ncb; i += nt) {
      const float w = L.codebook[i] * L.tc_wsc;  // |w s_W| < 2^15 (power-of-two scale: exact)
      const __half hi = __float2half_rn(w);
      const __half lo = __float2half_rn(w - __half2float(hi));
      s_cbs[i] = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
    }
    if (tid == 0) {
      for (int s = 0; s < kXStages; ++s) {
        mbar_init(&xfull[s], 1);
        mbar_init(&xempty[s], 1);
      }
      for (int s = 0; s < kStreams * kWBufs; ++s) {
        mbar_init(&wfull[s], kDecW);
        mbar_init(&wempty[s], 1);
      }
      mbar_init(tfull, 1);
      mbar_init(tempty, kEpiW);
      mbar_fence_init();
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // zero the private rows once; each tile's entries are cleared after use
  for (int i = threadIdx.x; i < kStreams * (kDecW / 4) * kTM * kRowBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(rows)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // launched as a programmatic dependent of the split kernel: everything above
  // (TMEM, barriers, codebook) overlapped its tail; its output is read below
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // the reduce's blocks may take their slots
  const uint32_t tmem_w = tmem + TN;  // W buffers: column TN + (q * kWBufs + b) * kWCols

  // The MMA consumes the two streams' tiles alternately q = 0, 1, 0, 1, ...
  // (the longer first half finishes alone); the X producer loads in that order.
  if (warp == 0) {
    // ---------------------------------------------------------- X tile producer
    if (lane == 0) {
      uint32_t xc = 0;
      TUnit t;
      for (int pc = 0; cta_piece(a, blockIdx.x, pc, t); ++pc) {
        int a0, a1, b0, b1;
        stream_range(t, 0, a0, a1);
        stream_range(t, 1, b0, b1);
        for (int j = 0; j < a1 - a0; ++j)
#pragma unroll
          for (int q = 0; q < kStreams; ++q) {
            if (q == 1 && j >= b1 - b0) continue;
            const int kt = (q == 0 ? a0 : b0) + j;
            const int s = (int)(xc % kXStages);
            mbar_wait(&xempty[s], ((xc / kXStages) & 1) ^ 1);
            unsigned char* st = xst + s * kXStageBytes;
            mbar_arrive_expect_tx(&xfull[s], 2 * kXTile);
            tma2d(st, &txh, kt * kTK, t.bt * TN, &xfull[s]);
            tma2d(st + kXTile, &txl, kt * kTK, t.bt * TN, &xfull[s]);
            ++xc;
          }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      // kind::f16: D fp32 (bits 4-5 = 1), A and B fp16 (bits 7-9, 10-12 = 0), K-major, N / 8, M / 16
      const uint32_t idesc = (1u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
      uint32_t xc = 0, gq[kStreams] = {0, 0}, uc = 0;
      TUnit t;
      for (int pc = 0; cta_piece(a, blockIdx.x, pc, t); ++pc, ++uc) {
        mbar_wait(tempty, (uc & 1) ^ 1);  // the epilogue drained the accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        int a0, a1, b0, b1;
        stream_range(t, 0, a0, a1);
        stream_range(t, 1, b0, b1);
        int step = 0;
        for (int j = 0; j < a1 - a0; ++j)
#pragma unroll
          for (int q = 0; q < kStreams; ++q) {
            if (q == 1 && j >= b1 - b0) continue;
            const int wb = q * kWBufs + (int)(gq[q] % kWBufs);
            const int s = (int)(xc % kXStages);
            tc_trace(a, 8, step);
            mbar_wait(&wfull[wb], (gq[q] / kWBufs) & 1);
            tc_trace(a, 9, step);
            mbar_wait(&xfull[s], (xc / kXStages) & 1);
            tc_trace(a, 10, step);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            unsigned char* st = xst + s * kXStageBytes;
            const uint64_t xh = sw128_desc(smem_addr(st)), xl = sw128_desc(smem_addr(st + kXTile));
            const uint32_t ah = tmem_w + (uint32_t)(wb * kWCols), al = ah + kWCols / 2;
#pragma unroll
            for (int k = 0; k < kTK / 16; ++k) {
              const uint32_t acc = (step == 0 && k == 0) ? 0u : 1u;
              umma_bf16_ts(tmem, ah + 8 * k, xh + 2 * k, idesc, acc);
              umma_bf16_ts(tmem, ah + 8 * k, xl + 2 * k, idesc, 1u);
              umma_bf16_ts(tmem, al + 8 * k, xh + 2 * k, idesc, 1u);
            }
            umma_commit(&xempty[s]);
            umma_commit(&wempty[wb]);
            tc_trace(a, 11, step);
            ++xc;
            ++gq[q];
            ++step;
          }
        umma_commit(tfull);  // an empty K range leaves the accumulator untouched (epilogue writes zeros)
      }
    }
  } else if (warp < 2 + kStreams * kDecW) {
    // ------------------------------------------------------------ expand warps
    // one lane per row = TMEM lane (a warp reaches lanes 32 (warp % 4) ...);
    // the row's entries of K tile kt are the next nnz(kt) u16 of the list
    // (k_tc_list), in column order, read through L1 with the next one in flight
    const int q = (warp - 2) / kDecW;  // K stream of this warp group
    const int hsel = kHalvesPerWarp == 2 ? 0 : ((warp - 2) % kDecW) >> 2;  // warp's half (kDecW == 8)
    const int quarter = warp & 3;
    const int row_l = quarter * 32 + lane;
    const uint32_t tlane = (uint32_t)(quarter * 32) << 16;
    const uint32_t prow = smem_addr(rows) + (uint32_t)(((q * (kDecW / 4) + hsel) * kTM + row_l) * kRowBytes);  // private row
    uint32_t g = 0;  // tiles of this stream so far
    TUnit t;
    for (int pc = 0; cta_piece(a, blockIdx.x, pc, t); ++pc) {
      int k0, k1;
      stream_range(t, q, k0, k1);
      // tile kt's entries: block (rt, kt) of the list, this row's slice of it
      const size_t blk0 = (size_t)t.rt * L.tNI + a.kbase;
      // raw loads only: the base / count arithmetic happens a tile later, at use
      struct Off { uint32_t b, o0, o1; };
      auto offs = [&](int kt) -> Off {
        const size_t blk = blk0 + kt;
        return Off{L.tbase[blk], L.troff[blk * 129 + row_l], L.troff[blk * 129 + row_l + 1]};
      };
      if (k1 <= k0) continue;
      Off fc = offs(k0);                          // tile kt
      Off fn = offs(k0 + 1 < k1 ? k0 + 1 : k1 - 1);  // tile kt + 1 (loaded one tile ahead of use)
      uint32_t oc = fc.b + fc.o0, nc = fc.o1 - fc.o0;
      // the next tile's first kEnt entries ride in registers one tile ahead;
      // every per-entry loop below stops at the warp's largest count (uniform branch)
      uint32_t nx[kEnt];
      {
        const uint32_t wm = __reduce_max_sync(0xffffffffu, nc);
#pragma unroll
        for (int i = 0; i < kEnt; ++i) {
          if ((uint32_t)i >= wm) break;
          nx[i] = (uint32_t)i < nc ? __ldg(L.tlist + oc + i) : 0u;
        }
      }
      for (int kt = k0; kt < k1; ++kt, ++g) {
        const bool tr = quarter == 2 && hsel == 0 && lane == 0;
        if (tr) tc_trace(a, 0 + 4 * q, kt - k0);
        const uint32_t nnz = nc;
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, nnz);
        const uint16_t* cur = L.tlist + oc;
        uint32_t v[kEnt];
#pragma unroll
        for (int i = 0; i < kEnt; ++i) {
          if ((uint32_t)i >= wmax) break;
          v[i] = nx[i];
        }
        oc = fn.b + fn.o0;
        nc = fn.o1 - fn.o0;
        {
          const uint32_t wm = __reduce_max_sync(0xffffffffu, nc);
#pragma unroll
          for (int i = 0; i < kEnt; ++i) {
            if ((uint32_t)i >= wm) break;
            nx[i] = (uint32_t)i < nc ? __ldg(L.tlist + oc + i) : 0u;
          }
        }
        fn = offs(kt + 2 < k1 ? kt + 2 : k1 - 1);
        const int wb = q * kWBufs + (int)(g % kWBufs);
        mbar_wait(&wempty[wb], ((g / kWBufs) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tr) tc_trace(a, 2 + 4 * q, kt - k0);
        const uint32_t tw = tmem_w + (uint32_t)(wb * kWCols) + tlane;
        // per entry (predicated on i < nnz): this warp's bf16 half of C[sym] and
        // its slot in the lane's private zero row
        uint32_t hl[kEnt], ad[kEnt];
#pragma unroll
        for (int i = 0; i < kEnt; ++i) {
          if ((uint32_t)i >= wmax) break;
          hl[i] = s_cbs[(v[i] >> 6) & 255u];
          ad[i] = prow + rsw_off(row_l, v[i] & 63u);
        }
#pragma unroll
        for (int hh = 0; hh < kHalvesPerWarp; ++hh) {
          const int h = kHalvesPerWarp == 2 ? hh : hsel;  // 0: bf16 hi tile, 1: lo tile
          const uint32_t hsh = 16u * (uint32_t)h;
#pragma unroll
          for (int i = 0; i < kEnt; ++i) {
            if ((uint32_t)i >= wmax) break;
            sts_u16_if(ad[i], (hl[i] >> hsh) & 0xFFFFu, (uint32_t)i < nnz);
          }
          // a denser row tile: the rest in groups of 8 whose loads are all in
          // flight together (one at a time, each entry waited its full latency)
          for (uint32_t i0 = kEnt; i0 < wmax; i0 += 8) {
            uint32_t e[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) e[j] = i0 + j < nnz ? __ldg(cur + i0 + j) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              sts_u16_if(prow + rsw_off(row_l, e[j] & 63u), (s_cbs[e[j] >> 6] >> hsh) & 0xFFFFu, i0 + j < nnz);
          }
          {  // 8 conflict-free LDS.128 -> one tcgen05.st of 32 columns
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 w4 = lds_u128(prow + ((uint32_t)(j ^ (row_l & 7)) << 4));
              r[4 * j] = w4.x; r[4 * j + 1] = w4.y; r[4 * j + 2] = w4.z; r[4 * j + 3] = w4.w;
            }
            tmem_st32(tw + (uint32_t)(h * (kWCols / 2)), r);
          }
          // back to a zero row
#pragma unroll
          for (int i = 0; i < kEnt; ++i) {
            if ((uint32_t)i >= wmax) break;
            sts_u16_if(ad[i], 0u, (uint32_t)i < nnz);
          }
          for (uint32_t i0 = kEnt; i0 < wmax; i0 += 8) {
            uint32_t e[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) e[j] = i0 + j < nnz ? __ldg(cur + i0 + j) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) sts_u16_if(prow + rsw_off(row_l, e[j] & 63u), 0u, i0 + j < nnz);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (tr) tc_trace(a, 3 + 4 * q, kt - k0);
        if (lane == 0) mbar_arrive(&wfull[wb]);
      }
    }
  } else {

    // ---------------------------------------------------------- epilogue warps
    const int ew = warp - (2 + kStreams * kDecW);
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int row_l = q4 * 32 + lane;
    uint32_t uc = 0;
    TUnit t;
    for (int pc = 0; cta_piece(a, blockIdx.x, pc, t); ++pc, ++uc) {
      if (ew == 0 && lane == 0) tc_trace(a, 12, 0);
      mbar_wait(tfull, uc & 1);
      if (ew == 0 && lane == 0) tc_trace(a, 13, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = t.rt * kTM + row_l;
      const int b0 = t.bt * TN;
      const bool has = t.kt1 > t.kt0;
      const bool whole = t.count == 1;  // this CTA owns the tile's whole K range
      // partials: [tile][slot][TN / 4 column groups][128 rows] float4, so a warp's
      // 32 rows of one column group are 512 contiguous bytes (row-major 1 KB
      // rows made every store instruction 32 scattered half-sectors)
      float* const dst = whole ? (a.yt ? a.y : a.y + (size_t)row * a.ldy + b0)
                               : a.ws + ((size_t)t.tile * a.mpt + t.slot) * kTM * TN + (size_t)row_l * 4;
      const float bias = (whole && row < L.wrows && a.bias) ? a.bias[row] : 0.f;
      // y rows are contiguous over the batch: whole float4s where the tile is inside B
      const bool vec_ok = (a.ldy % 4) == 0 && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
      for (int c = 0; c < TN; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c, v);
        if (!has) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        } else {
          // undo the fp16 split's scales: D / (s_W s_b), exact (powers of two)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= a.winv * __ldg(a.xsc + a.B + min(b0 + c + i, a.B - 1));
        }
        if (whole) {
          if (row < L.wrows) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              v[i] += bias;
              if (a.relu) v[i] = fmaxf(v[i], 0.f);
            }
          }
          if (a.xrg) {  // the images' max |y| over the warp's 32 rows (the next layer's split scale)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t mx =
                  __reduce_max_sync(0xffffffffu, row < L.wrows ? __float_as_uint(fabsf(v[i])) : 0u);
              if (lane == 0 && b0 + c + i < a.B) a.xrg[(size_t)(t.rt * 4 + q4) * a.B + b0 + c + i] = __uint_as_float(mx);
            }
          }
          if (row < L.wrows) {
            if (a.yt) {  // image-major: a warp's 32 rows are 128 contiguous bytes per image
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (b0 + c + i < a.B) a.y[(size_t)(b0 + c + i) * a.ldy + row] = v[i];
            } else if (vec_ok && b0 + c + 16 <= a.B) {
#pragma unroll
              for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(dst + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (b0 + c + i < a.B) dst[c + i] = v[i];
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            __stcg(reinterpret_cast<float4*>(dst + (size_t)((c + i) >> 2) * (kTM * 4)),
                   make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      if (ew == 0 && lane == 0) tc_trace(a, 14, 0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// Per-image power-of-two scale of the fp16 split: s = 2^e with m s in
// [2^14, 2^15) for m = max_k |x[b][k]| (m == 0, inf or NaN: s = 1).
__device__ __forceinline__ float pow2_scale(float m) {
  if (!(m > 0.f) || isinf(m)) return 1.f;
  int E;
  frexpf(m, &E);  // m = f 2^E, f in [0.5, 1)
  return ldexpf(1.f, max(-120, min(120, 15 - E)));
}

// max |x| per image over a K chunk (blockIdx.y of KS) -> part[ks][b]; the last
// block of an image (arrival counter, reset by it) writes its scale sc[b].
// Feature-major x [K][ldx]: block = 32 images x 8 row groups (image-major
// input: k_scale_split_rows).
constexpr int kScaleChunks = 16;
// sc[b] = s_b, sc[B + b] = 1 / s_b (exact: a power of two)
__device__ __forceinline__ void scale_finish(float m, int b, int B, int nparts, float* part, int* ctr, float* sc) {
  part[(size_t)blockIdx.y * B + b] = m;
  __threadfence();
  if (atomicAdd(&ctr[b], 1) == nparts - 1) {
    __threadfence();
    float mm = 0.f;
    for (int i = 0; i < nparts; ++i) mm = fmaxf(mm, __ldcg(&part[(size_t)i * B + b]));
    const float s = pow2_scale(mm);
    sc[b] = s;
    sc[B + b] = 1.0f / s;
    ctr[b] = 0;
  }
}
__global__ void __launch_bounds__(256) k_xscale_cols(const float* __restrict__ x, int K, int ldx, int B,
                                                     float* part, int* ctr, float* sc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (a programmatic dependent of the producer of x)
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, b = blockIdx.x * 32 + tx;
  const int kc = (K + gridDim.y - 1) / gridDim.y, k0 = blockIdx.y * kc, k1 = min(K, k0 + kc);
  float m = 0.f;
  if (b < B) {
    int k = k0 + ty;
    for (; k + 56 < k1; k += 64) {  // eight rows in flight per thread
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(x + (size_t)(k + 8 * j) * ldx + b);
#pragma unroll
      for (int j = 0; j < 8; ++j) m = fmaxf(m, fabsf(v[j]));
    }
    for (; k < k1; k += 8) m = fmaxf(m, fabsf(__ldg(x + (size_t)k * ldx + b)));
  }
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && b < B) {
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i][tx]);
    scale_finish(m, b, B, gridDim.y, part, ctr, sc);
  }
}
// fp16 hi / lo of v * s (s a power of two: |v s| < 2^15), packed in pairs
__device__ __forceinline__ void split_pair(float v0, float v1, float s, uint32_t& h, uint32_t& l) {
  v0 *= s;
  v1 *= s;
  const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
  const __half l0 = __float2half_rn(v0 - __half2float(h0)), l1 = __float2half_rn(v1 - __half2float(h1));
  h = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
  l = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
}

// X fp32 feature-major [K][ldx] -> fp16 hi / lo of x s_b, image-major [B][ldk] (K contiguous).
// Tile = 64 k x 32 images: coalesced 128-byte row loads, then each thread
// converts 8 consecutive k of one image and writes them as one 16-byte store
// per half (8 lanes cover a 128-byte run of an image row).
constexpr int kSplitK = 64, kSplitB = 32;
__global__ void __launch_bounds__(256) k_split_x(const float* __restrict__ x, int K, int ldx, int B,
                                                 uint16_t* __restrict__ xh, uint16_t* __restrict__ xl, int ldk,
                                                 float* __restrict__ xsc, const float* __restrict__ xrg, int nrg) {
  // a programmatic dependent of the producer of x (its launch and prologue
  // overlap that kernel's tail); nothing of x, xrg, xh / xl is touched before
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // the contraction's prologue may start
  // xrg: the producer's max |x| per (32-row group, image) -- the fused scale (no
  // k_xscale_cols pass over x): every block reduces its 32 images' groups; the
  // first K block of an image group writes the scales for the contraction
  __shared__ float s_m[8][kSplitB + 1];
  __shared__ float s_sc[kSplitB];
  if (xrg) {
    const int bl = (int)(threadIdx.x & 31), b = blockIdx.y * kSplitB + bl;
    float mx = 0.f;
    if (b < B)
      for (int g = (int)(threadIdx.x >> 5); g < nrg; g += 8) mx = fmaxf(mx, __ldg(xrg + (size_t)g * B + b));
    s_m[threadIdx.x >> 5][bl] = mx;
    __syncthreads();
    if (threadIdx.x < kSplitB) {
      for (int i = 1; i < 8; ++i) mx = fmaxf(mx, s_m[i][bl]);
      const float sc = pow2_scale(mx);
      s_sc[bl] = sc;
      if (blockIdx.x == 0 && b < B) {
        xsc[b] = sc;
        xsc[B + b] = 1.0f / sc;
      }
    }
  }
  __shared__ float tile[kSplitK][kSplitB + 1];
  const int k0 = blockIdx.x * kSplitK, b0 = blockIdx.y * kSplitB;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
#pragma unroll
  for (int i = ty; i < kSplitK; i += 8) {
    const int k = k0 + i, b = b0 + tx;
    tile[i][tx] = (k < K && b < B) ? __ldg(x + (size_t)k * ldx + b) : 0.f;
  }
  __syncthreads();
  const int c = threadIdx.x & 7, bl = threadIdx.x >> 3;  // k chunk (8 values), image
  const int b = b0 + bl, k = k0 + 8 * c;
  if (b >= B || k >= ldk) return;
  const float sb = xrg ? s_sc[bl] : xsc[b];
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_pair(tile[8 * c + 2 * i][bl], tile[8 * c + 2 * i + 1][bl], sb, h[i], l[i]);
  uint16_t* ph = xh + (size_t)b * ldk + k;
  uint16_t* pl = xl + (size_t)b * ldk + k;
  if (k + 8 <= ldk) {  // ldk % 8 == 0 and k % 8 == 0: 16-byte aligned
    *reinterpret_cast<uint4*>(ph) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(pl) = make_uint4(l[0], l[1], l[2], l[3]);
  } else {
    for (int i = 0; i < 8 && k + i < ldk; ++i) {
      ph[i] = (uint16_t)(h[i >> 1] >> (16 * (i & 1)));
      pl[i] = (uint16_t)(l[i >> 1] >> (16 * (i & 1)));
    }
  }
}

// Split tiles (covered by several CTAs' ranges): y[row][b] = act(sum_i
// ws[tile][i][row][b] + bias), i in CTA order (deterministic); one thread per 4
// images of a row, coalesced, over every tile at once (whole tiles skip).
template <int TN>
__global__ void __launch_bounds__(256) k_tc_reduce(const float* __restrict__ ws, uint32_t W, int G, int nkt,
                                                   int mpt, int nbt, int nrows, int B, const float* __restrict__ bias,
                                                   int relu, float* __restrict__ y, int ldy, int vec_ok, int yt,
                                                   float* __restrict__ xrg) {
  // block = 32 rows x 8 float4 column groups of one tile.  Reads go row-fastest
  // (the partials are column-group major, [TN / 4][128] float4 per piece:
  // coalesced), the sums are transposed through shared memory, and the y
  // writes go column-fastest (128 contiguous bytes per row)
  constexpr int kC4 = TN / 4, kCC = kC4 / 8;
  __shared__ float4 s_t[32][9];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of the contraction
  asm volatile("griddepcontrol.launch_dependents;");  // the next layer's split may launch (it waits for us)
  const uint32_t tile = blockIdx.x / (4 * kCC);
  const int rg = (int)(blockIdx.x % (4 * kCC)) / kCC, cc = (int)(blockIdx.x % kCC);
  const uint32_t t0 = tile * (uint32_t)nkt;  // 32-bit: W = tiles * nkt < 2^32 / G (host-checked)
  const int count = (int)(((t0 + nkt) * (uint32_t)G - 1) / W) - (int)(((t0 + 1) * (uint32_t)G - 1) / W) + 1;
  if (count == 1) return;  // (uniform over the block)
  const int rt = (int)(tile / (uint32_t)nbt), bt = (int)(tile % (uint32_t)nbt);
  {
    const int r = rg * 32 + (int)(threadIdx.x & 31), g = (int)(threadIdx.x >> 5);
    const int c4 = cc * 8 + g;
    const int row = rt * kTM + r, b = bt * TN + 4 * c4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < nrows && b < B) {
      const float* p = ws + (size_t)tile * mpt * kTM * TN + ((size_t)c4 * kTM + r) * 4;
      float4 q[8];  // the partials' loads all in flight before the (ordered) sum
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < count) q[j] = __ldcg(reinterpret_cast<const float4*>(p + (size_t)j * kTM * TN));
      acc = q[0];
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (j < count) { acc.x += q[j].x; acc.y += q[j].y; acc.z += q[j].z; acc.w += q[j].w; }
      for (int j = 8; j < count; ++j) {  // rare: more than 8 CTAs on one tile
        const float4 e = __ldcg(reinterpret_cast<const float4*>(p + (size_t)j * kTM * TN));
        acc.x += e.x; acc.y += e.y; acc.z += e.z; acc.w += e.w;
      }
      const float bs = bias ? bias[row] : 0.f;
      acc.x += bs; acc.y += bs; acc.z += bs; acc.w += bs;
      if (relu) {
        acc.x = fmaxf(acc.x, 0.f); acc.y = fmaxf(acc.y, 0.f); acc.z = fmaxf(acc.z, 0.f); acc.w = fmaxf(acc.w, 0.f);
      }
    }
    if (xrg) {  // the images' max |y| over the warp's 32 rows (the next layer's split scale)
      const bool in = row < nrows && b < B;
      const float ov[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t mx = __reduce_max_sync(0xffffffffu, in ? __float_as_uint(fabsf(ov[k])) : 0u);
        if ((threadIdx.x & 31) == 0 && b + k < B) xrg[(size_t)(rt * 4 + rg) * B + b + k] = __uint_as_float(mx);
      }
    }
    if (yt) {  // image-major y (class scores): consecutive rows are consecutive floats
      if (row < nrows && b < B) {
        const float ov[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int k = 0; k < 4 && b + k < B; ++k) y[(size_t)(b + k) * ldy + row] = ov[k];
      }
      return;  // (yt is uniform: no block skips the barrier another one waits at)
    }
    s_t[threadIdx.x & 31][g] = acc;
  }
  __syncthreads();
  const int g = (int)(threadIdx.x & 7), r = rg * 32 + (int)(threadIdx.x >> 3);
  const int row = rt * kTM + r, b = bt * TN + 4 * (cc * 8 + g);
  if (row >= nrows || b >= B) return;
  const float4 o = s_t[threadIdx.x >> 3][g];
  float* yp = y + (size_t)row * ldy + b;
  if (vec_ok && b + 4 <= B) {
    *reinterpret_cast<float4*>(yp) = o;
  } else {
    const float ov[4] = {o.x, o.y, o.z, o.w};
    for (int k = 0; k < 4 && b + k < B; ++k) yp[k] = ov[k];
  }
}

size_t tc_smem_bytes(const FcDev&, int tn) {
  size_t b = 1024 + (size_t)kXStages * (2 * tn * kTK * 2) + (size_t)kStreams * (kDecW / 4) * kTM * kRowBytes + 8 * (2 * kXStages + 2 * kStreams * kWBufs + 2) + 16 + 4 * 256;
  return (b + 127) & ~(size_t)127;
}

// ---------------------------------------------------------------------------
// List decoder (first kernel of the tensor-core path): PAPER.md Alg. 1 lines
// 4-7 -- Huffman decode of both streams, gap prefix sum -- for
// every (row, 8-tile chunk) in parallel from the Wi = 64 restart index; each
// real token becomes one u16 entry (column - 64 kt) | codebook index << 6 in
// its (row tile, K tile) block of the list (tbase / troff, built at load).
// Pads (symbol 0, C-04) produce nothing.  One thread per task; the 128 rows of
// a row tile are consecutive threads, so their entry writes are adjacent.
constexpr int kListThreads = 256;

template <bool BLOCKED>
__global__ void __launch_bounds__(kListThreads) k_tc_list(FcDev L, int c0, int nchr) {
  __shared__ uint32_t s_flut[1 << kFoldLutBits];
  __shared__ uint32_t s_glut[1 << kLutMaxBits];
  __shared__ uint32_t s_vtab[99], s_gtab[99];
  __shared__ uint16_t s_vsorted[257], s_gsorted[257];
  for (int i = threadIdx.x; i < (1 << L.Lf); i += blockDim.x) s_flut[i] = L.flut[i];
  for (int i = threadIdx.x; i < (1 << L.Lg); i += blockDim.x) s_glut[i] = L.glut[i];
  for (int i = threadIdx.x; i < 99; i += blockDim.x) { s_vtab[i] = L.vtab[i]; s_gtab[i] = L.gtab[i]; }
  for (int i = threadIdx.x; i < L.nvs; i += blockDim.x) s_vsorted[i] = L.vsorted[i];
  for (int i = threadIdx.x; i < L.ngs; i += blockDim.x) s_gsorted[i] = L.gsorted[i];
  __syncthreads();
  // task = (row group, chunk of L.tch <= kTcChunk intervals, row in group): consecutive
  // threads write adjacent slices of the same blocks
  const int tch = L.tch;
  // chunks [c0, c0 + nchr) of the row's (column-sharded layers: the rank's K block)
  const size_t task = (size_t)blockIdx.x * kListThreads + threadIdx.x;
  // groups of 128 stored rows (a row tile: a warp's list slots are adjacent),
  // 32 when blocked (few long stored rows)
  constexpr int kGrp = BLOCKED ? 32 : 128, kGrpLog2 = BLOCKED ? 5 : 7;
  const int r = (int)(task & (kGrp - 1));
  const size_t rc = task >> kGrpLog2;
  const int rt = (int)(rc / nchr), kt0 = (c0 + (int)(rc % nchr)) * tch;
  const int row = rt * kGrp + r;
  if (row >= L.nrows) return;
  const int nk = L.sNI - kt0 < tch ? L.sNI - kt0 : tch;
  // output slot of this row's first entry in each of the chunk's tiles
  uint32_t p[kTcChunk], n = 0;
  ListMap<BLOCKED> lm;
  lm.init(L, row, kt0);
#pragma unroll
  for (int k = 0; k < kTcChunk; ++k) {
    p[k] = 0;
    if (k < nk) {
      int rr = r;
      size_t blk = (size_t)rt * L.tNI + kt0 + k;  // unblocked: row tile rt, K tile kt0 + k
      if constexpr (BLOCKED) {
        blk = lm.block(L, rr);
        lm.next();
      }
      const uint32_t o0 = L.troff[blk * 129 + rr], o1 = L.troff[blk * 129 + rr + 1];
      p[k] = L.tbase[blk] + o0;
      n += o1 - o0;
    }
  }
  if (n == 0) return;
  const size_t q = (size_t)row * L.sNC + kt0 / tch;  // (restart index: chunk starts only)
  const uint2 st = L.tivg[q];
  int col = kt0 * 64 - (int)(L.tivm[q] & 0xFFu) - 1;
  SReader vr, gr;
  vr.init(L.vw, st.x);
  gr.init(L.gw, st.y);
  int ck = -1;       // tile of the last entry written
  uint32_t pos = 0;  // its next slot
  const int fsh = 32 - L.Lf, gsh = 32 - L.Lg, kk = L.k;
  for (uint32_t i = 0; i < n;) {
    const uint32_t w = vr.peek();
    const uint32_t e = s_flut[w >> fsh];
    uint32_t len, sym, pads, pbits;
    if (e != kFoldSlow) {  // pads folded in front of the code (C-04), one lookup
      len = e >> 28;
      sym = e & 0xFFu;
      pads = (e >> 24) & 15u;
      pbits = (e >> 8) & 0xFFFFu;
    } else {
      const uint32_t r = slow_sym(w, L.Lf + 1, s_vtab, s_vsorted, L.vmax);
      len = r >> 16;
      sym = r & 0xFFu;
      pads = sym == 0;
      pbits = pads ? (uint32_t)L.Lpg : 0u;
    }
    vr.skip(len);
    col += (int)(pads << kk);  // a pad advances the column by 2^k (gap 2^k - 1, C-01)
    if (pbits <= 32) {
      gr.skip(pbits);
    } else {
      for (uint32_t z = 0; z < pads; ++z) gr.skip((uint32_t)L.Lpg);
    }
    if (sym) {
      const uint32_t gwin = gr.peek();
      uint32_t ge = s_glut[gwin >> gsh];
      if (ge == 0) ge = slow_sym(gwin, L.Lg + 1, s_gtab, s_gsorted, L.gmax);
      gr.skip(ge >> 16);
      col += (int)(ge & 0xFFFFu) + 1;  // c = prev + g + 1 (Alg. 1 l.7, C-01)
      const int k = (col >> 6) - kt0;
      if (k != ck) {  // entered the next tile of the chunk: its slot (register select)
        ck = k;
        pos = p[0];
#pragma unroll
        for (int j = 1; j < kTcChunk; ++j) pos = k == j ? p[j] : pos;
      }
      L.tlist[pos++] = (uint16_t)((col & 63) | (sym << 6));
      ++i;
    }
  }
}


// Multi-symbol variant of the list decoder (r <= 5, k <= 4: the layers the
// small-batch kernel's LUTs serve, small.cu): one lookup on the val stream
// yields up to 4 codes, one on the gap stream up to 6; the two queues are
// consumed up to 4 tokens per step, a pad being a token whose gap advances the
// column by 2^k and whose symbol 0 emits nothing (C-01, C-04).
template <bool BLOCKED>
__global__ void __launch_bounds__(kListThreads) k_tc_list_ms(FcDev L, int c0, int nchr) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* s_vl = sm;
  uint32_t* s_gl = s_vl + (1 << L.msLv);
  uint32_t* s_vtab = s_gl + (1 << L.msLg);
  uint32_t* s_gtab = s_vtab + 99;
  uint16_t* s_vsorted = reinterpret_cast<uint16_t*>(s_gtab + 99);
  uint16_t* s_gsorted = s_vsorted + (L.nvs + 1);
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_pos[kTcChunk * kListThreads];
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
    const uint32_t vb = 4u << L.msLv, gb = 4u << L.msLg;
    mbar_arrive_expect_tx(&s_bar, vb + gb);
    bulk_g2s(s_vl, L.msv, vb, &s_bar);
    bulk_g2s(s_gl, L.msg, gb, &s_bar);
  }
  for (int i = threadIdx.x; i < 99; i += blockDim.x) { s_vtab[i] = L.vtab[i]; s_gtab[i] = L.gtab[i]; }
  for (int i = threadIdx.x; i < L.nvs; i += blockDim.x) s_vsorted[i] = L.vsorted[i];
  for (int i = threadIdx.x; i < L.ngs; i += blockDim.x) s_gsorted[i] = L.gsorted[i];
  __syncthreads();
  mbar_wait(&s_bar, 0);
  const int tch = L.tch;
  // chunks [c0, c0 + nchr) of the row's (column-sharded layers: the rank's K block)
  const size_t task = (size_t)blockIdx.x * kListThreads + threadIdx.x;
  // groups of 128 stored rows (a row tile: a warp's list slots are adjacent),
  // 32 when blocked (few long stored rows)
  constexpr int kGrp = BLOCKED ? 32 : 128, kGrpLog2 = BLOCKED ? 5 : 7;
  const int r = (int)(task & (kGrp - 1));
  const size_t rc = task >> kGrpLog2;
  const int rt = (int)(rc / nchr), kt0 = (c0 + (int)(rc % nchr)) * tch;
  const int row = rt * kGrp + r;
  if (row >= L.nrows) return;
  const int nk = L.sNI - kt0 < tch ? L.sNI - kt0 : tch;
  // the decoder state first (its loads gate everything), the output slots meanwhile
  const size_t q = (size_t)row * L.sNC + kt0 / tch;  // (restart index: chunk starts only)
  const uint2 st = L.tivg[q];
  const uint32_t m0 = L.tivm[q];
  // this thread's first list slot in each tile of the chunk, in shared memory
  // ([k][thread]: conflict-free) so the emission below picks it without branches
  uint32_t left = 0;
  ListMap<BLOCKED> lm;
  lm.init(L, row, kt0);
#pragma unroll
  for (int k = 0; k < kTcChunk; ++k) {
    uint32_t pk = 0;
    if (k < nk) {
      int rr = r;
      size_t blk = (size_t)rt * L.tNI + kt0 + k;  // unblocked: row tile rt, K tile kt0 + k
      if constexpr (BLOCKED) {
        blk = lm.block(L, rr);
        lm.next();
      }
      const uint32_t o0 = L.troff[blk * 129 + rr], o1 = L.troff[blk * 129 + rr + 1];
      pk = L.tbase[blk] + o0;
      left += o1 - o0;
    }
    s_pos[k * kListThreads + threadIdx.x] = pk;
  }
  SReader vr, gr;
  vr.init(L.vw, st.x);
  gr.init(L.gw, st.y);
  if (left == 0) return;
  int col = kt0 * 64 - (int)(m0 & 0xFFu) - 1;
  const int vsh = 32 - L.msLv, gsh = 32 - L.msLg;
  uint64_t qv = 0, qg = 0;
  int cv = 0, cg = 0;
  int ck = -1;
  uint32_t pos = 0;
  while (left > 0) {
    {  // refill the symbol queue (up to 4 codes per lookup)
      const uint32_t w = vr.peek();
      const uint32_t e = s_vl[w >> vsh];
      uint32_t n = e & 7u, len = (e >> 3) & 31u, syms = e >> 8;
      if (n == 0) {
        const uint32_t x = slow_sym(w, L.msLv + 1, s_vtab, s_vsorted, L.vmax);
        n = 1;
        len = x >> 16;
        syms = x & 31u;
      }
      const bool room = cv <= 8;
      qv |= (uint64_t)(room ? syms : 0u) << (5 * cv);
      cv += room ? (int)n : 0;
      vr.skip(room ? len : 0u);
    }
    {  // refill the gap queue (up to 6 codes per lookup)
      const uint32_t w = gr.peek();
      const uint32_t e = s_gl[w >> gsh];
      uint32_t n = e & 7u, len = (e >> 3) & 31u, gaps = e >> 8;
      if (n == 0) {
        const uint32_t x = slow_sym(w, L.msLg + 1, s_gtab, s_gsorted, L.gmax);
        n = 1;
        len = x >> 16;
        gaps = x & 15u;
      }
      const bool room = cg <= 10;
      qg |= (uint64_t)(room ? gaps : 0u) << (4 * cg);
      cg += room ? (int)n : 0;
      gr.skip(room ? len : 0u);
    }
    const int pn = min(min(cv, cg), 4);
    const uint32_t qv32 = (uint32_t)qv, qg32 = (uint32_t)qg;
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // branch-free: every slot computes, only real tokens store
      const bool take = j < pn;
      col += take ? (int)((qg32 >> (4 * j)) & 15u) + 1 : 0;  // c = prev + g + 1 (Alg. 1 l.7, C-01)
      const uint32_t sym = (qv32 >> (5 * j)) & 31u;
      int k = (col >> 6) - kt0;
      k = k < kTcChunk - 1 ? k : kTcChunk - 1;  // tokens past the chunk never store
      const uint32_t pk = s_pos[k * kListThreads + threadIdx.x];
      pos = k != ck ? pk : pos;  // columns only grow: a tile is entered once
      ck = k;
      const bool em = take && sym != 0 && left > 0;
      st_u16_if(L.tlist + pos, (col & 63) | (sym << 6), em);
      pos += em;
      left -= em;
    }
    qv >>= 5 * pn;
    qg >>= 4 * pn;
    cv -= pn;
    cg -= pn;
  }
}

bool list_fold_forced() {
  static const bool v = [] {
    const char* e = std::getenv("CDN_TC_LIST");
    return e && e[0] == 'f';
  }();
  return v;
}

}  // namespace

// Image-major input (the public infer input / a conv trunk's output): one
// block per image finds max |x| over its K features, writes the power-of-two
// scale and its inverse, then splits the row (second read: L2-resident) into
// fp16 hi / lo of x s_b -- k_xscale_rows + k_split_rows in one launch.
__global__ void __launch_bounds__(512) k_scale_split_rows(const float* __restrict__ x, int K, int ldx, int B,
                                                          uint16_t* __restrict__ xh, uint16_t* __restrict__ xl,
                                                          int ldk, int vec, float* __restrict__ sc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (a programmatic dependent of the work before it)
  asm volatile("griddepcontrol.launch_dependents;");  // the contraction's prologue may start
  __shared__ float red[16];
  __shared__ float s_scale;
  const int b = blockIdx.x;
  const float* p = x + (size_t)b * ldx;
  float m = 0.f;
  if (vec) {
    const int k4 = K / 4;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    int k = threadIdx.x;
    for (; k + 3 * 512 < k4; k += 4 * 512) {  // four 16-byte loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldg(p4 + k + 512 * j);
#pragma unroll
      for (int j = 0; j < 4; ++j) m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
    }
    for (; k < k4; k += 512) {
      const float4 v = __ldg(p4 + k);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int kk = k4 * 4 + threadIdx.x; kk < K; kk += 512) m = fmaxf(m, fabsf(__ldg(p + kk)));
  } else {
    for (int kk = threadIdx.x; kk < K; kk += 512) m = fmaxf(m, fabsf(__ldg(p + kk)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 16; ++i) m = fmaxf(m, red[i]);
    const float s = pow2_scale(m);
    s_scale = s;
    sc[b] = s;
    sc[B + b] = 1.0f / s;
  }
  __syncthreads();
  const float sb = s_scale;
  for (int k8 = threadIdx.x; k8 * 8 < ldk; k8 += 512) {
    const int k = k8 * 8;
    float v[8];
    if (vec && k + 8 <= K) {
      const float4 a0 = __ldg(reinterpret_cast<const float4*>(p + k)), a1 = __ldg(reinterpret_cast<const float4*>(p + k + 4));
      v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = k + j < K ? p[k + j] : 0.f;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split_pair(v[2 * j], v[2 * j + 1], sb, h[j], l[j]);
    *reinterpret_cast<uint4*>(xh + (size_t)b * ldk + k) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(xl + (size_t)b * ldk + k) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

size_t tc_scale_floats(int B) { return (size_t)B * (kScaleChunks + 2); }

bool tc_supported(const FcDev& L) {
  return L.tivg && L.tivm && L.tNI > 0 && L.sNI > 0 && L.sNC > 0 && L.tbase && L.troff && L.ncb <= 256 && L.nvs <= 256 && L.ngs <= 256 &&
         L.Lf == kFoldLutBits && L.Lg <= kLutMaxBits;
}

TcPlan plan_fc_tc(const FcDev& L, int B, int num_sms, int kt0, int kt1) {
  TcPlan p;
  if (!tc_supported(L) || B <= 0) return p;
  if (kt1 < 0) kt1 = L.tNI;
  if (kt0 < 0 || kt1 > L.tNI || kt1 <= kt0 || ((kt0 > 0 || kt1 < L.tNI) && L.bw != L.wcols)) return p;
  // a 128-image tile when the batch fits one (half the tensor work of 256)
  p.tn = B <= 64 ? 64 : (B <= 128 ? 128 : kTN);
  p.nbt = (B + p.tn - 1) / p.tn;
  p.nrt = (L.wrows + kTM - 1) / kTM;
  p.kbase = kt0;
  p.nkt = kt1 - kt0;
  p.kcols = std::min(L.wcols, kt1 * kTK) - kt0 * kTK;
  p.ldk = (p.kcols + 7) & ~7;
  p.tiles = p.nrt * p.nbt;
  p.W = (long)p.tiles * p.nkt;
  long G;
  if (p.W >= 64L * num_sms) {
    // long shares: stream-K, every SM an equal contiguous share of the tile
    // steps (no wave quantisation; a share spans at most a few pieces)
    G = num_sms;
  } else {
    // short shares: each CTA one (tile, K/S range) piece (G = tiles * S, which
    // the stream-K formulas reduce to); the piece start-up (~16 steps' worth,
    // measured on C5) dominates, so S minimises waves * (nkt / S + 16)
    double best = 1e30;
    int bestS = 1;
    const int smax = p.nkt < 64 ? p.nkt : 64;
    for (int S = 1; S <= smax; ++S) {
      const long units = (long)p.tiles * S;
      const long waves = (units + num_sms - 1) / num_sms;
      const double cost = (double)waves * ((double)p.nkt / S + 16.0);
      if (cost < best * 0.98) { best = cost; bestS = S; }
    }
    G = (long)p.tiles * bestS;
  }
  p.grid = (int)G;
  const long per = p.W / G;  // >= 1
  p.mpt = (int)((p.nkt + per - 1) / per) + 1;
  if (p.mpt > (int)G) p.mpt = (int)G;
  p.ws_floats = (size_t)p.tiles * p.mpt * kTM * p.tn;
  p.xsplit_elems = (size_t)B * p.ldk;
  p.smem = tc_smem_bytes(L, p.tn);
  // 32-bit stream-K arithmetic in k_tc_reduce
  p.ok = p.smem <= 227 * 1024 && (uint64_t)(p.W + p.nkt) * (uint64_t)p.grid < (1ull << 32);
  return p;
}

cudaError_t launch_tc_list(const FcDev& L, cudaStream_t s, int kt0, int kt1) {
  cudaError_t e = cudaSuccess;
  const bool blocked = L.bw != L.wcols;
  const size_t grp = blocked ? 32 : 128;
  if (kt1 < 0 || kt1 > L.sNI) kt1 = L.sNI;
  // the chunks of L.tch K tiles that cover [kt0, kt1) (edge chunks decode a
  // few tiles outside the range into their own -- valid -- list blocks)
  const int c0 = kt0 / L.tch, c1 = (kt1 + L.tch - 1) / L.tch;
  const int nchr = std::max(1, c1 - c0);
  const size_t tasks = (size_t)((L.nrows + grp - 1) / grp) * nchr * grp;
  const unsigned lgrid = (unsigned)((tasks + kListThreads - 1) / kListThreads);
  if (ms_supported(L) && !list_fold_forced()) {
    const size_t lsm = ms_smem_bytes(L);
    static size_t set_lsm = 0;
    if (lsm > set_lsm) {
      for (auto kern : {k_tc_list_ms<false>, k_tc_list_ms<true>}) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
        if (e != cudaSuccess) return e;
      }
      set_lsm = lsm;
    }
    ktimer_begin("k_tc_list", s);
    if (blocked)
      k_tc_list_ms<true><<<lgrid, kListThreads, lsm, s>>>(L, c0, nchr);
    else
      k_tc_list_ms<false><<<lgrid, kListThreads, lsm, s>>>(L, c0, nchr);
  } else {
    ktimer_begin("k_tc_list", s);
    if (blocked)
      k_tc_list<true><<<lgrid, kListThreads, 0, s>>>(L, c0, nchr);
    else
      k_tc_list<false><<<lgrid, kListThreads, 0, s>>>(L, c0, nchr);
  }
  e = launched();
  ktimer_end("k_tc_list", s);
  return e;
}

// a launch as a programmatic dependent of the stream's previous kernel (the
// kernel waits on griddepcontrol before touching anything that kernel wrote)
template <typename... KArgs, typename... Args>
static cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_fc_tc(const FcDev& L, const TcPlan& p, const float* x, int ldx, int B, float* y, int ldy, int relu,
                         uint16_t* xh, uint16_t* xl, float* ws, float* scw, int* xctr, cudaStream_t s,
                         bool x_image_major, bool y_image_major, const float* bias, const float* xrg_in,
                         int nrg_in, float* xrg_out) {
  // per-image scales of the fp16 split: scw = [B scales | B inverse scales |
  // kScaleChunks x B partial maxima]; xctr: >= B arrival counters, zero between calls
  float* xsc = scw;
  float* xpart = scw + 2 * (size_t)B;
  ktimer_begin("k_split_x", s);
  if (x_image_major) {
    const int vec = (ldx % 4) == 0 && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    cudaError_t e0 = pdl_launch(k_scale_split_rows, dim3((unsigned)B), dim3(512), s, x, p.kcols, ldx, B, xh, xl, p.ldk,
                                vec, xsc);
    if (e0 != cudaSuccess) return e0;
  } else {
    cudaError_t e0 = cudaSuccess;
    if (!xrg_in)  // (no producer maxima: a separate pass over x)
      e0 = pdl_launch(k_xscale_cols, dim3((unsigned)((B + 31) / 32), kScaleChunks), dim3(256), s, x, p.kcols, ldx, B,
                      xpart, xctr, xsc);
    if (e0 != cudaSuccess) return e0;
    dim3 sg((p.ldk + kSplitK - 1) / kSplitK, (B + kSplitB - 1) / kSplitB);
    e0 = pdl_launch(k_split_x, sg, dim3(256), s, x, p.kcols, ldx, B, xh, xl, p.ldk, xsc, xrg_in, nrg_in);
    if (e0 != cudaSuccess) return e0;
  }
  cudaError_t e = launched(x_image_major || xrg_in ? 1 : 2);
  ktimer_end("k_split_x", s);
  if (e != cudaSuccess) return e;
  CUtensorMap th, tl;
  e = encode_tmap_2d(&th, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, xh, (uint64_t)p.ldk, (uint64_t)B, (uint64_t)p.ldk * 2,
                     kTK, (uint32_t)p.tn, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  e = encode_tmap_2d(&tl, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, xl, (uint64_t)p.ldk, (uint64_t)B, (uint64_t)p.ldk * 2,
                     kTK, (uint32_t)p.tn, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  static bool attr_set = false;
  if (!attr_set) {  // the largest footprint (256-image tiles) covers both
    for (auto kern : {k_fc_tc<64>, k_fc_tc<128>, k_fc_tc<256>}) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes(L, kTN));
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  static unsigned long long* trace = nullptr;
  const char* trace_path = getenv("CDN_TC_TRACE");
  if (trace_path && !trace) {
    e = cudaMalloc(&trace, 16 * 256 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
  }
  if (trace) cudaMemsetAsync(trace, 0, 16 * 256 * sizeof(unsigned long long), s);
  TcArgs a{y, ldy, B, relu, ws, p.nbt, p.nrt, p.nkt, p.grid, p.mpt, p.W, trace_path ? trace : nullptr,
           y_image_major ? 1 : 0, xsc, 1.0f / L.tc_wsc, p.kbase, bias, y_image_major ? nullptr : xrg_out};
  ktimer_begin("k_fc_tc", s);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.grid);
    cfg.blockDim = dim3(kTThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps the split
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (p.tn == 128)
      e = cudaLaunchKernelEx(&cfg, k_fc_tc<128>, L, a, th, tl);
    else if (p.tn == 64)
      e = cudaLaunchKernelEx(&cfg, k_fc_tc<64>, L, a, th, tl);
    else
      e = cudaLaunchKernelEx(&cfg, k_fc_tc<256>, L, a, th, tl);
    if (e != cudaSuccess) return e;
  }
  e = launched();
  ktimer_end("k_fc_tc", s);
  if (e == cudaSuccess && p.grid != p.tiles) {  // some tile is split over CTAs
    ktimer_begin("k_tc_reduce", s);
    const int vec_ok = (ldy % 4) == 0 && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.tiles * (p.tn / 8)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // launch latency hidden under the contraction
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const float* wsc = ws;
    const int yt = y_image_major ? 1 : 0;
    if (p.tn == 128)
      e = cudaLaunchKernelEx(&cfg, k_tc_reduce<128>, wsc, (uint32_t)p.W, p.grid, p.nkt, p.mpt, p.nbt, (int)L.wrows, B,
                             bias, relu, y, ldy, vec_ok, yt, yt ? nullptr : xrg_out);
    else if (p.tn == 64)
      e = cudaLaunchKernelEx(&cfg, k_tc_reduce<64>, wsc, (uint32_t)p.W, p.grid, p.nkt, p.mpt, p.nbt, (int)L.wrows, B,
                             bias, relu, y, ldy, vec_ok, yt, yt ? nullptr : xrg_out);
    else
      e = cudaLaunchKernelEx(&cfg, k_tc_reduce<256>, wsc, (uint32_t)p.W, p.grid, p.nkt, p.mpt, p.nbt, (int)L.wrows, B,
                             bias, relu, y, ldy, vec_ok, yt, yt ? nullptr : xrg_out);
    if (e == cudaSuccess) e = launched();
    ktimer_end("k_tc_reduce", s);
  }
  if (e == cudaSuccess && trace_path) {  // debug only: dump CTA 0's event clocks
    std::vector<unsigned long long> h(16 * 256);
    e = cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (FILE* fp = fopen(trace_path, "wb")) {
      fwrite(h.data(), sizeof(h[0]), h.size(), fp);
      fclose(fp);
    }
  }
  return e;
}

}  // namespace cdn
