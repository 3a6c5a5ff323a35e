// CONV path (Eq. 1 for a convolution layer in its
// im2col form): per call the layer's compressed filter matrix is
// Huffman-decoded straight into a dense bf16 matrix (kernels.cu
// k_decode_dense, L2-resident: <= 2.4 MB per AlexNet layer), the NHWC input is
// unfolded to bf16 patches (K order (r, s, c), channel fastest, reading C-18),
// and the contraction runs on the 5th-generation tensor cores:
//
//   k_gemm_bf16: D[pos][filter] = sum_k A[pos][k] * W[filter][k], every group
//   of the layer in one persistent launch (a CTA per SM walking the tiles)
//     * 128 positions x BN filters per tile, K in 64-element (128-byte) tiles;
//     * warp 0 / lane 0: TMA producer (cp.async.bulk.tensor 3D, 128B swizzle)
//       into a smem ring (~200 KB) on full/empty mbarriers, across tiles;
//     * warp 1 / lane 0: issues tcgen05.mma.cta_group::1.kind::f16 (bf16 x
//       bf16 -> fp32 accumulator in TMEM, two accumulator buffers), commits
//       to the stage's empty barrier and, after a tile's last K step, to that
//       buffer's ready barrier;
//     * warps 2-5: epilogue tcgen05.ld (32x32b) -> + bias -> ReLU (-> LRN) ->
//       fp32 NHWC, then release the buffer -- overlapping the next tile.
//   k_lrn, k_maxpool: the AlexNet norm / pool layers (C-19, C-20), NHWC fp32.
#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>

#include "dev_common.cuh"
#include "tc_common.cuh"
#include "kernels.cuh"
#include "tmap.hpp"

namespace cdn {

namespace {

using namespace dev;

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGMaxStages = 8;
constexpr int kGEpiWarps = 4;
constexpr int kGMaxBias = 4096;  // groups * filters per group staged in shared memory
constexpr int kGThreads = 64 + 32 * kGEpiWarps;  // TMA warp, MMA warp, epilogue warps

// out[pos * ldo + col0 + z * Nrows + n] = act( sum_k A_z[pos][k] W_z[n][k] + bias[z * Nrows + n] ),
// pos in [0, Mrows), n in [0, Nrows), z the group.  A: tensor map over
// [groups][Mrows][Kpad] bf16, W: over [groups][Nrows][Kpad] bf16; nk = Kpad / 64.
// Persistent: a CTA per SM walks the (m, n, z) tiles; the TMEM accumulator is
// double-buffered, so the epilogue of one tile overlaps the loads and MMAs of
// the next (warp 0 TMA, warp 1 MMA, warps 2-5 epilogue, TMEM lane quadrant =
// warp % 4).
__global__ void __launch_bounds__(kGThreads, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int Mrows, int Nrows,
                int nk, int BN, int tmem_cols, int kGStages, const float* __restrict__ bias,
                float* __restrict__ out, int ldo, int col0, int relu, int lrn, int groups, int4 imc, int4 imc2) {
  // imc = (im2col mode, Wo, Ho * Wo, pad), imc2 = (kw, channel chunks per tap, padded channels per group, -):
  // in im2col mode `ta` is an im2col map over the bf16 NHWC input and K tile kt
  // = (tap, chunk) = (r * kw + s, c / 64) of group z
  extern __shared__ unsigned char smem_raw[];
  // align within the shared window (pointer arithmetic on smem_raw keeps the .shared address space)
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int a_bytes = kBM * kBK * 2, b_bytes = BN * kBK * 2;
  unsigned char* sA = smem;
  unsigned char* sB = smem + kGStages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kGStages * b_bytes);
  uint64_t* empty = full + kGStages;
  uint64_t* acc_full = empty + kGStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // [groups * Nrows], 16-byte aligned (float4 reads): off the epilogue's load latency
  float* s_bias = reinterpret_cast<float*>(
      smem + ((reinterpret_cast<unsigned char*>(tmem_slot + 4) - smem + 15) & ~(ptrdiff_t)15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (Mrows + kBM - 1) / kBM, ntl = (Nrows + BN - 1) / BN;
  const int tiles = mt * ntl * groups;
  for (int i = threadIdx.x; i < groups * Nrows; i += blockDim.x) s_bias[i] = bias[i];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kGEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "r"(2 * tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer, the stage ring running on across tiles
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m = t % mt, n = (t / mt) % ntl, z = t / (mt * ntl);
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % kGStages;
          mbar_wait(&empty[s], ((it / kGStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(a_bytes + b_bytes));
          if (imc.x) {  // implicit GEMM: the 128 output pixels' tap (r, s) channels, straight from the input
            const int p0 = m * kBM, img = p0 / imc.z, rem = p0 - img * imc.z, oh = rem / imc.y, ow = rem - oh * imc.y;
            const int tap = kt / imc2.y, ch = kt - tap * imc2.y, r = tap / imc2.x, sx = tap - r * imc2.x;
            tma_im2col4d(sA + s * a_bytes, &ta, z * imc2.z + ch * kBK, ow - imc.w, oh - imc.w, img, sx, r, &full[s]);
          } else {
            tma3d(sA + s * a_bytes, &ta, kt * kBK, m * kBM, z, &full[s]);
          }
          tma3d(sB + s * b_bytes, &tb, kt * kBK, n * BN, z, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: 4 x (128 x BN x 16) per 64-wide K tile, into accumulator (local tile & 1)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(buf * tmem_cols);
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % kGStages;
          mbar_wait(&full[s], (it / kGStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128_desc(smem_addr(sA + s * a_bytes));
          const uint64_t bd = sw128_desc(smem_addr(sB + s * b_bytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) umma_bf16(acc, ad + 2 * k, bd + 2 * k, idesc, (kt | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---- epilogue warps: TMEM lane = position row (quadrant warp % 4), column = filter
    const int q = warp & 3;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int m = t % mt, n = (t / mt) % ntl, z = t / (mt * ntl);
      const int buf = i & 1;
      const int n0 = n * BN, c0z = col0 + z * Nrows;
      const float* bz = s_bias + z * Nrows;
      mbar_wait(&acc_full[buf], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * tmem_cols);
      const int row = m * kBM + q * 32 + lane;
      if (lrn) {
        // LRN fused (the tile holds all Nrows channels of its positions; one lane =
        // one position): y_c = a_c * (2 + 1e-4/5 * sum_{q=c-2..c+2} a_q^2)^-0.75,
        // a = act(conv + bias), summed in the order k_lrn uses (bit-identical).
        // Chunks of 16 channels slide with the 2 before and the 16 after.
        auto act = [&](float (&v)[16], int c) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int ch = c + u;
            float o = ch < Nrows ? v[u] + bz[ch] : 0.f;  // (uniform over the warp: smem broadcast)
            if (relu) o = fmaxf(o, 0.f);
            v[u] = o;
          }
        };
        float cur[16], nxt[16], p1 = 0.f, p2 = 0.f;  // p2 = a[c-2], p1 = a[c-1]
        tmem_ld16(tq, cur);
        act(cur, 0);
        for (int c = 0; c < Nrows; c += 16) {
          if (c + 16 < Nrows) {
            tmem_ld16(tq + (uint32_t)(c + 16), nxt);
            act(nxt, c + 16);
          } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) nxt[u] = 0.f;
          }
          float o[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int ch = c + u;
            // window a[ch-2 .. ch+2] clipped to [0, Nrows)
            float w[5];
            w[0] = u >= 2 ? cur[u - 2] : (u == 1 ? p1 : p2);
            w[1] = u >= 1 ? cur[u - 1] : p1;
            w[2] = cur[u];
            w[3] = u + 1 < 16 ? cur[u + 1] : nxt[u - 15];
            w[4] = u + 2 < 16 ? cur[u + 2] : nxt[u - 14];
            float sq = 0.f;
#pragma unroll
            for (int r = 0; r < 5; ++r) {
              const int cq = ch - 2 + r;
              if (cq >= 0 && cq < Nrows) sq = fmaf(w[r], w[r], sq);
            }
            o[u] = cur[u] * exp2f(-0.75f * __log2f(2.0f + (1e-4f / 5.0f) * sq));
          }
          if (row < Mrows) {
            float* op = out + (size_t)row * ldo + c0z + c;
            if (c + 16 <= Nrows && ((((uintptr_t)op) & 15) == 0)) {
#pragma unroll
              for (int r = 0; r < 4; ++r)
                reinterpret_cast<float4*>(op)[r] = make_float4(o[4 * r], o[4 * r + 1], o[4 * r + 2], o[4 * r + 3]);
            } else {
#pragma unroll
              for (int u = 0; u < 16; ++u)
                if (c + u < Nrows) op[u] = o[u];
            }
          }
          p2 = cur[14];
          p1 = cur[15];
#pragma unroll
          for (int u = 0; u < 16; ++u) cur[u] = nxt[u];
        }
      } else {
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(tq + (uint32_t)c, v);
          if (row < Mrows) {
            float* op = out + (size_t)row * ldo + c0z + n0 + c;
            if (n0 + c + 16 <= Nrows && ((((uintptr_t)op) & 15) == 0)) {
              const float4* bp = reinterpret_cast<const float4*>(bz + n0 + c);
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const float4 bq = bp[r];
                float4 o = make_float4(v[4 * r] + bq.x, v[4 * r + 1] + bq.y, v[4 * r + 2] + bq.z, v[4 * r + 3] + bq.w);
                if (relu) {
                  o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                }
                reinterpret_cast<float4*>(op)[r] = o;
              }
            } else {
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int ch = n0 + c + u;
                if (ch < Nrows) {
                  float o = v[u] + bz[ch];
                  if (relu) o = fmaxf(o, 0.f);
                  op[u] = o;
                }
              }
            }
          }
        }
      }
      // the accumulator buffer is free again once every epilogue warp has read it
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * tmem_cols) : "memory");
}

// Halo-tile implicit GEMM for stride-1 CONV layers (k_conv_halo), computed
// transposed: D[filter][position] = sum_k W[filter][k] * patch[position][k],
// filters on the M side (128 per tile, TMEM lanes) and up to 256 positions on
// the N side (TMEM columns) -- at N = 128 the 16-bit MMA reads its two smem
// operands about as fast as it computes (measured: 128-filter tiles ran the
// position-major form below the im2col GEMM), N up to 256 halves that.
// The K loop runs (64-channel chunk, tap (r, s)); per chunk the CTA stages
// ONCE the input rows its positions and their kh x kw windows need -- a
// "halo", one 4D tiled TMA box, padding and edges from the TMA's
// out-of-bounds zeros -- and every tap's B operand is that halo seen from a
// shifted start.  Positions are flattened at the pitch P = Wo + kw - 1
// (f = y P + x; positions with x >= Wo are computed and dropped), so the input
// of position f for tap (r, s) sits at halo row (f - y_s P) + r P + s:
// consecutive positions stay 128 bytes apart, i.e. the K-major 128B-swizzle
// layout (8-row groups 1024 B apart) from an unaligned start, the swizzle
// following the shared-memory address as the TMA wrote it (measured: the
// descriptor's base-offset field must stay 0).  The im2col TMA it replaces
// re-read each input pixel from L2 once per tap (kh kw = 9-25 times).
// Tile = (image, position block of NT, 128-filter block, group); persistent,
// double-buffered TMEM accumulator; warp 0 TMA, warp 1 MMA, warps 2-9 the
// epilogue (two per TMEM lane quadrant, each half of the columns; lane =
// filter: + bias, ReLU, each store a warp's 32 consecutive channels of one
// position; the position walks (y, x) incrementally -- a division per column
// had made the epilogue, not the MMA, the bound).
struct HaloArgs {
  int B, Ho, Wo, P, HR, kh, kw, pad, nch, cgp, Nrows, NT, spi, mtl, G, tiles;
  int halo_bytes, SA, SB, talloc, relu, ldo;
  const float* bias;
  float* out;
};

constexpr int kHEpiWarps = 8;
constexpr int kHThreads = 64 + 32 * kHEpiWarps;

__global__ void __launch_bounds__(kHThreads, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap th, const __grid_constant__ CUtensorMap tb, const HaloArgs h) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  constexpr int f_bytes = kBM * kBK * 2;  // one filter tile (128 filters x 64 K)
  unsigned char* sH = smem;                   // halo stages
  unsigned char* sF = smem + h.SA * h.halo_bytes;  // filter stages
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sF + h.SB * f_bytes);
  uint64_t* hempty = hfull + h.SA;
  uint64_t* ffull = hempty + h.SA;
  uint64_t* fempty = ffull + h.SB;
  uint64_t* acc_full = fempty + h.SB;  // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < h.SA; ++s) {
      mbar_init(&hfull[s], 1);
      mbar_init(&hempty[s], 1);
    }
    for (int s = 0; s < h.SB; ++s) {
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kHEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "r"(h.talloc)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int nsub = h.B * h.spi, taps = h.kh * h.kw;
  // tile t: position block u (image u / spi), filter block m, group z
  auto decode = [&](int t, int& img, int& f0, int& ys, int& m, int& z) {
    const int u = t % nsub, rest = t / nsub;
    m = rest % h.mtl;
    z = rest / h.mtl;
    img = u / h.spi;
    f0 = (u - img * h.spi) * h.NT;
    ys = f0 / h.P;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: per chunk the halo, then one filter tile per tap
      int ai = 0, bi = 0;
      for (int t = blockIdx.x; t < h.tiles; t += gridDim.x) {
        int img, f0, ys, m, z;
        decode(t, img, f0, ys, m, z);
        for (int ch = 0; ch < h.nch; ++ch, ++ai) {
          const int sa = ai % h.SA;
          mbar_wait(&hempty[sa], ((ai / h.SA) & 1) ^ 1);
          mbar_arrive_expect_tx(&hfull[sa], (uint32_t)(h.HR * h.P * 128));
          tma4d(sH + sa * h.halo_bytes, &th, z * h.cgp + ch * kBK, -h.pad, ys - h.pad, img, &hfull[sa]);
          for (int tap = 0; tap < taps; ++tap, ++bi) {
            const int sb = bi % h.SB;
            mbar_wait(&fempty[sb], ((bi / h.SB) & 1) ^ 1);
            mbar_arrive_expect_tx(&ffull[sb], (uint32_t)f_bytes);
            tma3d(sF + sb * f_bytes, &tb, (tap * h.nch + ch) * kBK, m * kBM, z, &ffull[sb]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: per tap 4 x (128 filters x NT positions x 16)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(h.NT >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      int ai = 0, bi = 0, i = 0;
      for (int t = blockIdx.x; t < h.tiles; t += gridDim.x, ++i) {
        int img, f0, ys, m, z;
        decode(t, img, f0, ys, m, z);
        const int off0 = f0 - ys * h.P;
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(buf * h.NT);
        for (int ch = 0; ch < h.nch; ++ch, ++ai) {
          const int sa = ai % h.SA;
          mbar_wait(&hfull[sa], (ai / h.SA) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t hbase = smem_addr(sH + sa * h.halo_bytes);
          for (int tap = 0; tap < taps; ++tap, ++bi) {
            const int r = tap / h.kw, sx = tap - r * h.kw;
            const int sb = bi % h.SB;
            mbar_wait(&ffull[sb], (bi / h.SB) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad = sw128_desc(smem_addr(sF + sb * f_bytes));
            const uint64_t bd = sw128_desc(hbase + (uint32_t)(off0 + r * h.P + sx) * 128u);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) umma_bf16(acc, ad + 2 * k, bd + 2 * k, idesc, (ch | tap | k) != 0);
            umma_commit(&fempty[sb]);
          }
          umma_commit(&hempty[sa]);
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---- epilogue warps: TMEM lane = filter (quadrant warp % 4), column = flattened
    // position; the quadrant's two warps take the two halves of the columns
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int c_lo = half ? ((h.NT / 2 + 15) & ~15) : 0, c_hi = half ? h.NT : ((h.NT / 2 + 15) & ~15);
    int i = 0;
    for (int t = blockIdx.x; t < h.tiles; t += gridDim.x, ++i) {
      int img, f0, ys, m, z;
      decode(t, img, f0, ys, m, z);
      const int buf = i & 1;
      const int fl = m * kBM + q * 32 + lane;  // this lane's filter in the group
      const bool fok = fl < h.Nrows;
      const float bv = fok ? h.bias[z * h.Nrows + fl] : 0.f;
      float* obase = h.out + (size_t)img * h.Ho * h.Wo * h.ldo + z * h.Nrows + fl;
      // the first column's position, then stepped (uniform over the warp)
      int y = (f0 + c_lo) / h.P, x = f0 + c_lo - y * h.P;
      mbar_wait(&acc_full[buf], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * h.NT);
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        tmem_ld16(tq + (uint32_t)c, v);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (fok && y < h.Ho && x < h.Wo) {
            float o = v[u] + bv;
            if (h.relu) o = fmaxf(o, 0.f);
            obase[(size_t)(y * h.Wo + x) * h.ldo] = o;
          }
          if (++x == h.P) {
            x = 0;
            ++y;
          }
        }
      }
      // the accumulator buffer is free again once every epilogue warp has read it
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(h.talloc) : "memory");
}

// NHWC fp32 -> bf16 (RNE) patches [pos][Kpad] of channels [c0, c0+cg):
// k = (r*kw + s)*cg + c, zero for padding taps and k >= kh*kw*cg.
template <bool VEC8>
__global__ void k_im2col(const float* __restrict__ x, int B, int H, int W, int C, int kh, int kw, int stride, int pad,
                         int c0, int cg, int Ho, int Wo, int Kreal, int Kpad, __nv_bfloat16* __restrict__ out) {
  const int kq = Kpad / 8;
  // 32-bit indexing (the launcher checks B * Ho * Wo * Kpad / 8 < 2^31): 64-bit
  // division here cost more than the copy itself
  const uint32_t total = (uint32_t)B * Ho * Wo * kq;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t pos = idx / kq;
    const int k0 = (int)(idx - pos * kq) * 8;
    const int b = (int)(pos / (uint32_t)(Ho * Wo));
    const int rem = (int)(pos - (uint32_t)b * (Ho * Wo));
    const int oh = rem / Wo, ow = rem - oh * Wo;
    __align__(16) __nv_bfloat16 v[8];
    if (VEC8) {
      // cg % 8 == 0: the 8 k's are 8 consecutive channels of one (r, s) tap
      float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (k0 < Kreal) {
        const int c = k0 % cg, rs = k0 / cg;
        const int s = rs % kw, r = rs / kw;
        const int ih = oh * stride - pad + r, iw = ow * stride - pad + s;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
          const float4* px = reinterpret_cast<const float4*>(x + (((size_t)b * H + ih) * W + iw) * C + c0 + c);
          const float4 a0 = __ldg(px), a1 = __ldg(px + 1);
          f[0] = a0.x; f[1] = a0.y; f[2] = a0.z; f[3] = a0.w;
          f[4] = a1.x; f[5] = a1.y; f[6] = a1.z; f[7] = a1.w;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn(f[j]);
    } else {
      // one (c, s, r) decomposition per thread, then incremental steps
      int c = k0 % cg, rs = k0 / cg;
      int sx = rs % kw, r = rs / kw;
      const float* xb = x + (size_t)b * H * W * C + c0;
      const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float f = 0.f;
        if (k0 + j < Kreal) {
          const int ih = ih0 + r, iw = iw0 + sx;
          if (ih >= 0 && ih < H && iw >= 0 && iw < W) f = __ldg(xb + ((size_t)ih * W + iw) * C + c);
        }
        v[j] = __float2bfloat16_rn(f);
        if (++c == cg) {
          c = 0;
          if (++sx == kw) {
            sx = 0;
            ++r;
          }
        }
      }
    }
    *reinterpret_cast<uint4*>(out + (size_t)pos * Kpad + k0) = *reinterpret_cast<const uint4*>(v);
  }
}

// Cross-channel LRN (reading C-20: n = 5, alpha = 1e-4, beta = 0.75, k = 2,
// alpha/n scaling, window clipped at the channel ends), NHWC fp32.
__global__ void k_lrn(const float* __restrict__ x, long npos, int C, float* __restrict__ y) {
  const long total = npos * C;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const float* px = x + (i - c);
    float s = 0.f;
    const int lo = max(0, c - 2), hi = min(C - 1, c + 2);
    for (int q = lo; q <= hi; ++q) s = fmaf(px[q], px[q], s);
    // base in [2, 2 + 2e-5 * sum a^2]: exp2/log2 intrinsics are ~1e-7 relative here
    y[i] = px[c] * exp2f(-0.75f * __log2f(2.0f + (1e-4f / 5.0f) * s));
  }
}

// k x k / stride s max-pool, no padding, NHWC fp32.
__global__ void k_maxpool(const float* __restrict__ x, int B, int H, int W, int C, int k, int s, int Ho, int Wo,
                          float* __restrict__ y) {
  const long total = (long)B * Ho * Wo * C;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    long p = i / C;
    const int ow = (int)(p % Wo);
    p /= Wo;
    const int oh = (int)(p % Ho);
    const int b = (int)(p / Ho);
    float m = -INFINITY;
    for (int r = 0; r < k; ++r)
      for (int q = 0; q < k; ++q)
        m = fmaxf(m, x[(((size_t)b * H + oh * s + r) * W + ow * s + q) * C + c]);
    y[i] = m;
  }
}

// 4 channels per thread (C % 4 == 0, 16-byte aligned), 32-bit indexing: the
// common AlexNet case of the two kernels above.
__global__ void k_maxpool4(const float4* __restrict__ x, int B, int H, int W, int C4, int k, int s, int Ho, int Wo,
                           float4* __restrict__ y) {
  const int total = B * Ho * Wo * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C4;
    int p = i / C4;
    const int ow = p % Wo;
    p /= Wo;
    const int oh = p % Ho, b = p / Ho;
    float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    const float4* xb = x + ((size_t)(b * H + oh * s) * W + ow * s) * C4 + c;
    if (k == 3) {  // AlexNet's 3x3 (C-19): the nine loads in flight together
      float4 v[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) v[j] = __ldg(xb + ((size_t)(j / 3) * W + (j % 3)) * C4);
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        m.x = fmaxf(m.x, v[j].x); m.y = fmaxf(m.y, v[j].y); m.z = fmaxf(m.z, v[j].z); m.w = fmaxf(m.w, v[j].w);
      }
    } else {
      for (int r = 0; r < k; ++r)
        for (int q = 0; q < k; ++q) {
          const float4 v = __ldg(xb + ((size_t)r * W + q) * C4);
          m.x = fmaxf(m.x, v.x); m.y = fmaxf(m.y, v.y); m.z = fmaxf(m.z, v.z); m.w = fmaxf(m.w, v.w);
        }
    }
    y[i] = m;
  }
}

__global__ void k_lrn4(const float* __restrict__ x, int npos, int C, float* __restrict__ y) {
  const int C4 = C >> 2, total = npos * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c0 = (i % C4) * 4;
    const float* px = x + (size_t)(i / C4) * C;
    float a[8];  // channels c0-2 .. c0+5 (0 outside, never summed)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 - 2 + j;
      a[j] = (c >= 0 && c < C) ? __ldg(px + c) : 0.f;
    }
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + j;
      float sq = 0.f;
      // the same order as k_lrn: q from max(0, c-2) to min(C-1, c+2)
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int cq = c - 2 + q;
        if (cq >= 0 && cq < C) sq = fmaf(a[j + q], a[j + q], sq);
      }
      o[j] = a[j + 2] * exp2f(-0.75f * __log2f(2.0f + (1e-4f / 5.0f) * sq));
    }
    *reinterpret_cast<float4*>(y + (size_t)(i / C4) * C + c0) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

int grid_for(long work, int threads, int num_sms) {
  const long g = (work + threads - 1) / threads;
  const long cap = (long)num_sms * 16;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

}  // namespace

int gemm_tile_n(int Nrows) {
  static const int cap = [] {  // (experiment knob: widest filter tile)
    const char* e = std::getenv("CDN_GEMM_BN");
    return e ? std::max(16, std::min(256, std::atoi(e))) : 256;
  }();
  int tiles = (Nrows + cap - 1) / cap;
  int bn = (Nrows + tiles - 1) / tiles;
  return (bn + 15) & ~15;
}

// Pipeline depth: as many stages as fit ~200 KB (one persistent CTA per SM;
// its double-buffered accumulator overlaps the epilogue with the next tile).
int gemm_stages(int BN) {
  const int per = kBM * kBK * 2 + BN * kBK * 2;
  int st = (200 * 1024) / per;
  return st < 2 ? 2 : (st > kGMaxStages ? kGMaxStages : st);
}

size_t gemm_smem_bytes(int BN) {
  const int st = gemm_stages(BN);
  return 1024 + (size_t)st * (kBM * kBK * 2 + BN * kBK * 2) + (2 * st + 4) * 8 + 32 + 4 * kGMaxBias;
}

cudaError_t launch_gemm_bf16(const __nv_bfloat16* A, int Mrows, const __nv_bfloat16* Wt, int Nrows, int Kpad,
                             const float* bias, int relu, float* out, int ldo, int col0, cudaStream_t s, int lrn,
                             int groups) {
  if (Mrows <= 0 || Nrows <= 0 || groups <= 0) return cudaSuccess;
  if ((long)groups * Nrows > kGMaxBias) return cudaErrorInvalidValue;
  if (Kpad % kBK) return cudaErrorInvalidValue;
  const int BN = gemm_tile_n(Nrows);
  if (lrn && BN < Nrows) return cudaErrorInvalidValue;  // the fused LRN needs every channel in one tile
  int tcols = 32;
  while (tcols < BN) tcols <<= 1;
  // groups stacked as planes: A [groups][Mrows][Kpad], W [groups][Nrows][Kpad]
  CUtensorMap ta, tb;
  cudaError_t e = encode_tmap_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, A, (uint64_t)Kpad, (uint64_t)Mrows,
                                 (uint64_t)groups, (uint64_t)Kpad * 2, (uint64_t)Kpad * 2 * Mrows, kBK, kBM,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  e = encode_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Wt, (uint64_t)Kpad, (uint64_t)Nrows, (uint64_t)groups,
                     (uint64_t)Kpad * 2, (uint64_t)Kpad * 2 * Nrows, kBK, (uint32_t)BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  const size_t smem = gemm_smem_bytes(BN);
  static thread_local size_t set_smem = 0;
  if (smem > set_smem) {
    e = cudaFuncSetAttribute(k_gemm_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  ktimer_begin("k_gemm_bf16", s);
  const long tiles = (long)((Mrows + kBM - 1) / kBM) * ((Nrows + BN - 1) / BN) * groups;
  int num_sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);
  k_gemm_bf16<<<grid, kGThreads, smem, s>>>(ta, tb, Mrows, Nrows, Kpad / kBK, BN, tcols, gemm_stages(BN), bias, out,
                                            ldo, col0, relu, lrn, groups, make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0));
  const cudaError_t e_ = launched();
  ktimer_end("k_gemm_bf16", s);
  return e_;
}

// Launch geometry of k_conv_halo for one stride-1 layer; false: it does not
// apply (the im2col-TMA GEMM runs: fused LRN, halos over the smem budget).
// Position blocks: an image's Ho P flattened positions in spi equal blocks of
// NT <= 256 (multiple of 16); two halo stages, as many filter stages as fit.
static bool halo_plan(int B, int G, int cgp, int kh, int kw, int pad, int Ho, int Wo, int Nrows, int lrn, HaloArgs& h,
                      size_t& smem) {
  static const int mode = [] {  // CDN_CONV_HALO=0: off (A/B knob)
    const char* e = std::getenv("CDN_CONV_HALO");
    return e ? std::atoi(e) : 1;
  }();
  if (!mode || lrn || cgp % kBK) return false;
  h = HaloArgs{};
  h.B = B; h.Ho = Ho; h.Wo = Wo; h.kh = kh; h.kw = kw; h.pad = pad; h.G = G; h.cgp = cgp; h.Nrows = Nrows;
  h.P = Wo + kw - 1;
  const int flat = Ho * h.P;
  h.spi = (flat + 255) / 256;
  h.NT = ((flat + h.spi - 1) / h.spi + 15) & ~15;
  h.HR = (h.NT - 1) / h.P + 2 + kh - 1;  // a block's output rows (<= (NT-1)/P + 2) + kh - 1
  if (h.P > 256 || h.HR > 256) return false;
  const int rows_alloc = std::max(h.HR * h.P, (kh - 1) * h.P + kw + h.P + h.NT);  // + the dropped positions' overreach
  h.halo_bytes = (rows_alloc * 128 + 1023) & ~1023;
  h.nch = cgp / kBK;
  h.mtl = (Nrows + kBM - 1) / kBM;
  h.talloc = 32;
  while (h.talloc < 2 * h.NT) h.talloc <<= 1;
  h.SA = 2;
  const size_t fixed = 1024 + 256;
  const long left = 225L * 1024 - (long)fixed - (long)h.SA * h.halo_bytes;
  h.SB = (int)std::min<long>(8, left / (kBM * kBK * 2));
  if (h.SB < 3 || h.talloc > 512) return false;
  h.tiles = B * h.spi * h.mtl * G;
  smem = fixed + (size_t)h.SA * h.halo_bytes + (size_t)h.SB * kBM * kBK * 2;
  return smem <= 227 * 1024;
}

cudaError_t launch_gemm_implicit(const __nv_bfloat16* act, int B, int H, int W, int G, int cgp, int kh, int kw,
                                 int pad, int Ho, int Wo, const __nv_bfloat16* Wt, int Nrows, const float* bias,
                                 int relu, float* out, int ldo, cudaStream_t s, int lrn) {
  const int Mrows = B * Ho * Wo;
  if (Mrows <= 0 || Nrows <= 0 || G <= 0) return cudaSuccess;
  if ((long)G * Nrows > kGMaxBias || cgp % kBK || kh != kw || Ho != H + 2 * pad - kh + 1 || Wo != W + 2 * pad - kw + 1)
    return cudaErrorInvalidValue;
  {
    HaloArgs h;
    size_t smem = 0;
    if (halo_plan(B, G, cgp, kh, kw, pad, Ho, Wo, Nrows, lrn, h, smem)) {
      h.relu = relu;
      h.ldo = ldo;
      h.bias = bias;
      h.out = out;
      CUtensorMap th, tb;
      cudaError_t e = encode_tmap_nhwc4d(&th, act, (uint64_t)G * cgp, (uint64_t)W, (uint64_t)H, (uint64_t)B, kBK,
                                         (uint32_t)h.P, (uint32_t)h.HR);
      if (e != cudaSuccess) return e;
      const int Kpad = kh * kw * cgp;
      e = encode_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Wt, (uint64_t)Kpad, (uint64_t)Nrows, (uint64_t)G,
                         (uint64_t)Kpad * 2, (uint64_t)Kpad * 2 * Nrows, kBK, (uint32_t)kBM, CU_TENSOR_MAP_SWIZZLE_128B);
      if (e != cudaSuccess) return e;
      static thread_local size_t set_smem = 0;
      if (smem > set_smem) {
        e = cudaFuncSetAttribute(k_conv_halo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        set_smem = smem;
      }
      int num_sms = 148;
      {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
      }
      ktimer_begin("k_conv_halo", s);
      k_conv_halo<<<std::min(h.tiles, num_sms), kHThreads, smem, s>>>(th, tb, h);
      const cudaError_t e_ = launched();
      ktimer_end("k_conv_halo", s);
      return e_;
    }
  }
  const int BN = gemm_tile_n(Nrows);
  if (lrn && BN < Nrows) return cudaErrorInvalidValue;
  int tcols = 32;
  while (tcols < BN) tcols <<= 1;
  const int nch = cgp / kBK, Kpad = kh * kw * cgp;
  CUtensorMap ta, tb;
  cudaError_t e = encode_tmap_im2col4d(&ta, act, (uint64_t)G * cgp, (uint64_t)W, (uint64_t)H, (uint64_t)B, -pad,
                                       pad - (kh - 1), kBK, kBM);
  if (e != cudaSuccess) return e;
  e = encode_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Wt, (uint64_t)Kpad, (uint64_t)Nrows, (uint64_t)G,
                     (uint64_t)Kpad * 2, (uint64_t)Kpad * 2 * Nrows, kBK, (uint32_t)BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  const size_t smem = gemm_smem_bytes(BN);
  static thread_local size_t set_smem = 0;
  if (smem > set_smem) {
    e = cudaFuncSetAttribute(k_gemm_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  ktimer_begin("k_gemm_bf16", s);
  const long tiles = (long)((Mrows + kBM - 1) / kBM) * ((Nrows + BN - 1) / BN) * G;
  int num_sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);
  k_gemm_bf16<<<grid, kGThreads, smem, s>>>(ta, tb, Mrows, Nrows, Kpad / kBK, BN, tcols, gemm_stages(BN), bias, out,
                                            ldo, 0, relu, lrn, G, make_int4(1, Wo, Ho * Wo, pad),
                                            make_int4(kw, nch, cgp, 0));
  const cudaError_t e_ = launched();
  ktimer_end("k_gemm_bf16", s);
  return e_;
}

// x fp32 NHWC [npix][C] (G groups of cg channels) -> bf16 (RNE, reading C-21)
// [npix][G * cgp], each group's channels padded with zeros to cgp: the
// implicit GEMM's TMA im2col reads 64-channel (128-byte) runs per tap.
__global__ void k_to_bf16_pad(const float* __restrict__ x, long npix, int C, int G, int cg, int cgp,
                              __nv_bfloat16* __restrict__ out) {
  const int cp = G * cgp, q = cp / 2;  // channel pairs per pixel
  const long n = npix * q;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long p = i / q;
    const int c2 = (int)(i - p * q) * 2, z = c2 / cgp, c = c2 - z * cgp;
    const float* xp = x + p * C + z * cg;
    const float a = c < cg ? xp[c] : 0.f, b = c + 1 < cg ? xp[c + 1] : 0.f;
    reinterpret_cast<__nv_bfloat162*>(out)[i] = __floats2bfloat162_rn(a, b);
  }
}

// The same conversion 8 channels per thread (two 16-byte loads, one 16-byte
// store) when every group's channels come in whole 8-channel runs (cg % 8 ==
// 0: AlexNet conv2-5) -- the pair-per-thread form ran at ~2 TB/s
__global__ void __launch_bounds__(256) k_to_bf16_pad8(const float* __restrict__ x, long npix, int C, int G, int cg,
                                                      int cgp, __nv_bfloat16* __restrict__ out) {
  const int q = G * cgp / 8;  // 8-channel chunks per output pixel
  const long n = npix * q;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long p = i / q;
    const int c8 = (int)(i - p * q) * 8, z = c8 / cgp, c = c8 - z * cgp;
    float v[8];
    if (c < cg) {  // (cg % 8 == 0: a chunk is all real or all padding)
      const float4* xp = reinterpret_cast<const float4*>(x + p * C + z * cg + c);
      const float4 a = __ldg(xp), b = __ldg(xp + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
    }
    __nv_bfloat162 h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    reinterpret_cast<uint4*>(out)[i] = *reinterpret_cast<const uint4*>(h);
  }
}

cudaError_t launch_to_bf16_pad(const float* x, long npix, int C, int G, int cg, int cgp, __nv_bfloat16* out,
                               cudaStream_t s) {
  if (npix <= 0) return cudaSuccess;
  if (cgp % 2) return cudaErrorInvalidValue;
  ktimer_begin("k_to_bf16_pad", s);
  if (cg % 8 == 0 && cgp % 8 == 0 && C % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const long n = npix * G * cgp / 8;
    const int grid = (int)std::min<long>((n + 255) / 256, 148L * 16);
    k_to_bf16_pad8<<<grid, 256, 0, s>>>(x, npix, C, G, cg, cgp, out);
  } else {
    const long n = npix * G * cgp / 2;
    const int grid = (int)std::min<long>((n + 255) / 256, 148L * 16);
    k_to_bf16_pad<<<grid, 256, 0, s>>>(x, npix, C, G, cg, cgp, out);
  }
  const cudaError_t e_ = launched();
  ktimer_end("k_to_bf16_pad", s);
  return e_;
}

// Space-to-depth of a strided CONV's input (conv1: 227 x 227 x 3, stride 4 ->
// 57 x 57 x 48 padded to 64 channels): the layer becomes a stride-1 CONV with
// a ceil(kh / s)-square kernel, whose filters are decoded into the matching K
// order (api.cpp s2d_kmap) -- the same products, so the implicit GEMM's TMA
// im2col path (>= 64-channel runs) serves it with no patch matrix.  A thread
// per super-pixel: its s input row runs of s*C floats (adjacent threads read
// adjacent runs) and one 2*cgp-byte row of 16-byte stores.
template <int ST, int C>
__global__ void __launch_bounds__(256) k_s2d_bf16(const float* __restrict__ x, int B, int H, int W, int Hs, int Ws,
                                                  int cgp, __nv_bfloat16* __restrict__ out) {
  constexpr int RUN = ST * C, NV = ST * RUN;  // floats per input row run, values per super-pixel
  const long n = (long)B * Hs * Ws;
  for (long p = (long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
    const int X = (int)(p % Ws);
    const long t = p / Ws;
    const int Y = (int)(t % Hs), b = (int)(t / Hs);
    float v[NV];
#pragma unroll
    for (int dy = 0; dy < ST; ++dy) {
      const int yy = Y * ST + dy;
      const float* row = x + (((size_t)b * H + yy) * W + (size_t)X * ST) * C;
#pragma unroll
      for (int i = 0; i < RUN; ++i) {
        const int xx = X * ST + i / C;
        v[dy * RUN + i] = (yy < H && xx < W) ? __ldg(row + i) : 0.f;
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)p * cgp);
#pragma unroll
    for (int c8 = 0; c8 < (NV + 7) / 8; ++c8) {
      __nv_bfloat162 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = c8 * 8 + 2 * k;
        h[k] = __floats2bfloat162_rn(c < NV ? v[c] : 0.f, c + 1 < NV ? v[c + 1] : 0.f);
      }
      dst[c8] = *reinterpret_cast<const uint4*>(h);
    }
    for (int c8 = (NV + 7) / 8; c8 < cgp / 8; ++c8) dst[c8] = make_uint4(0u, 0u, 0u, 0u);
  }
}

cudaError_t launch_s2d_bf16(const float* x, int B, int H, int W, int C, int st, int Hs, int Ws, int cgp,
                            __nv_bfloat16* out, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (cgp % 8 || st * st * C > cgp) return cudaErrorInvalidValue;
  const long n = (long)B * Hs * Ws;
  const int grid = (int)std::min<long>((n + 255) / 256, 148L * 16);
  ktimer_begin("k_s2d_bf16", s);
  if (st == 4 && C == 3) k_s2d_bf16<4, 3><<<grid, 256, 0, s>>>(x, B, H, W, Hs, Ws, cgp, out);
  else if (st == 2 && C == 3) k_s2d_bf16<2, 3><<<grid, 256, 0, s>>>(x, B, H, W, Hs, Ws, cgp, out);
  else if (st == 2 && C == 4) k_s2d_bf16<2, 4><<<grid, 256, 0, s>>>(x, B, H, W, Hs, Ws, cgp, out);
  else if (st == 4 && C == 4) k_s2d_bf16<4, 4><<<grid, 256, 0, s>>>(x, B, H, W, Hs, Ws, cgp, out);
  else return cudaErrorInvalidValue;
  const cudaError_t e_ = launched();
  ktimer_end("k_s2d_bf16", s);
  return e_;
}

// im2col for small channel groups (conv1: 3 channels, K = 11*11*3): a warp per
// output position, lanes along K, so a warp reads the window's contiguous
// (s, c) runs and writes 64 contiguous bytes per step; the (r, s, c) of every k
// is tabled in shared memory once per block (no per-element division).
constexpr int kIm2colMaxK = 4096;
__global__ void __launch_bounds__(256) k_im2col_warp(const float* __restrict__ x, int B, int H, int W, int C, int kh,
                                                     int kw, int stride, int pad, int c0, int cg, int Ho, int Wo,
                                                     int Kreal, int Kpad, __nv_bfloat16* __restrict__ out) {
  __shared__ int s_off[kIm2colMaxK];             // (r * W + s) * C + c, -1 past Kreal
  __shared__ unsigned char s_r[kIm2colMaxK], s_s[kIm2colMaxK];
  for (int k = threadIdx.x; k < Kpad; k += blockDim.x) {
    if (k < Kreal) {
      const int c = k % cg, rs = k / cg, sx = rs % kw, r = rs / kw;
      s_off[k] = (r * W + sx) * C + c;
      s_r[k] = (unsigned char)r;
      s_s[k] = (unsigned char)sx;
    } else {
      s_off[k] = -1;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int npos = B * Ho * Wo;
  for (int pos = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pos < npos; pos += warps) {
    const int b = pos / (Ho * Wo), rem = pos - b * (Ho * Wo);
    const int oh = rem / Wo, ow = rem - oh * Wo;
    const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
    const bool inside = ih0 >= 0 && iw0 >= 0 && ih0 + kh <= H && iw0 + kw <= W;  // no padding taps
    const float* xw = x + (((size_t)b * H + ih0) * W + iw0) * C + c0;            // window origin (maybe outside)
    // lane: 2 consecutive k per step (one 4-byte store; 128 contiguous bytes per warp)
    uint32_t* o = reinterpret_cast<uint32_t*>(out + (size_t)pos * Kpad);
    auto tap = [&](int k) -> float {
      const int off = s_off[k];
      if (off < 0) return 0.f;
      if (!inside) {
        const int ih = ih0 + s_r[k], iw = iw0 + s_s[k];
        if (ih < 0 || ih >= H || iw < 0 || iw >= W) return 0.f;
      }
      return __ldg(xw + off);
    };
#pragma unroll 2
    for (int k = 2 * lane; k < Kpad; k += 64) {
      const float f0 = tap(k), f1 = tap(k + 1);
      const __nv_bfloat162 h = __floats2bfloat162_rn(f0, f1);
      o[k >> 1] = *reinterpret_cast<const uint32_t*>(&h);
    }
  }
}

// im2col for small channel groups (conv1: 3 channels, 11x11 taps, stride 4):
// a block per output row (b, oh).  The kh input rows it reads are staged once
// in shared memory as bf16 (padding columns and rows as zeros), so each input
// element is fetched from L2 once per block instead of once per tap that
// covers it (~(kh/stride)^2 = 7.6x for conv1); patches are then built from
// shared memory, a lane per 8 consecutive k (one 16-byte store, 512 contiguous
// bytes per warp instruction), through a per-k offset table.
constexpr int kIm2colRowsMaxSmem = 40 * 1024;
__global__ void __launch_bounds__(256) k_im2col_rows(const float* __restrict__ x, int B, int H, int W, int C, int kh,
                                                     int kw, int stride, int pad, int c0, int cg, int Ho, int Wo,
                                                     int Kreal, int Kpad, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char ir_smem[];
  const int Wp = W + 2 * pad;
  const int plane = kh * Wp * cg;                                       // staged rows, + one zero slot
  int* s_off = reinterpret_cast<int*>(ir_smem);                         // [Kpad]
  __nv_bfloat16* s_x = reinterpret_cast<__nv_bfloat16*>(ir_smem + 4 * Kpad);  // [kh][Wp][cg], [plane] = 0
  const int b = blockIdx.x / Ho, oh = blockIdx.x - b * Ho;
  const int ih0 = oh * stride - pad;
  for (int k = threadIdx.x; k < Kpad; k += blockDim.x) {
    int off = plane;  // the zero slot
    if (k < Kreal) {
      const int c = k % cg, rs = k / cg, sx = rs % kw, r = rs / kw;
      off = (r * Wp + sx) * cg + c;
    }
    s_off[k] = off;
  }
  // stage the kh input rows (cg == C: a pixel row is one contiguous run of W * C
  // floats), padding columns and out-of-image rows as zeros; no division
  // (eight independent loads in flight per thread: the staging is latency-bound otherwise)
  const int rowlen = Wp * cg, lo = pad * cg, hi = (pad + W) * cg;
  const float* xb = x + (size_t)b * H * W * C - lo;
  for (int i0 = threadIdx.x; i0 < plane; i0 += 8 * blockDim.x) {
    int r = i0 / rowlen, j = i0 - r * rowlen;
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int ih = ih0 + r;
      const bool ok = i0 + u * (int)blockDim.x < plane && ih >= 0 && ih < H && j >= lo && j < hi;
      v[u] = ok ? __ldg(xb + (size_t)ih * W * C + j) : 0.f;
      j += blockDim.x;  // rowlen >= blockDim.x (launcher): at most one wrap
      if (j >= rowlen) {
        j -= rowlen;
        ++r;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * (int)blockDim.x < plane) s_x[i0 + u * blockDim.x] = __float2bfloat16_rn(v[u]);
  }
  if (threadIdx.x == 0) s_x[plane] = __float2bfloat16_rn(0.f);
  __syncthreads();
  const int nq = Kpad >> 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned short* sx16 = reinterpret_cast<const unsigned short*>(s_x);
  for (int ow = warp; ow < Wo; ow += nw) {
    const int base = ow * stride * cg;
    uint4* o = reinterpret_cast<uint4*>(out + ((size_t)blockIdx.x * Wo + ow) * Kpad);
    for (int q = lane; q < nq; q += 32) {
      const int4 oa = *reinterpret_cast<const int4*>(&s_off[8 * q]);
      const int4 ob = *reinterpret_cast<const int4*>(&s_off[8 * q + 4]);
      auto at = [&](int off) -> uint32_t { return sx16[off == plane ? plane : base + off]; };
      uint4 v;
      v.x = at(oa.x) | (at(oa.y) << 16);
      v.y = at(oa.z) | (at(oa.w) << 16);
      v.z = at(ob.x) | (at(ob.y) << 16);
      v.w = at(ob.z) | (at(ob.w) << 16);
      o[q] = v;
    }
  }
}

static size_t im2col_rows_smem(int kh, int W, int pad, int cg, int Kpad) {
  return (size_t)4 * Kpad + 2 * ((size_t)kh * (W + 2 * pad) * cg + 1);
}

// im2col for channel groups of 8k (conv2-5): a warp per output position, a
// lane per 8-channel chunk of K (two float4 loads, one 16-byte store, 512
// contiguous bytes per warp step); the (r, s, c) of every chunk is tabled in
// shared memory once per block, so the per-chunk work is a table read and the
// bounds test -- no integer division (the per-thread decomposition of
// k_im2col<true> made that kernel issue-bound at ~3x the HBM time).
constexpr int kIm2colMaxChunks = 1024;
__global__ void __launch_bounds__(256) k_im2col_warp8(const float* __restrict__ x, int B, int H, int W, int C, int kh,
                                                      int kw, int stride, int pad, int c0, int cg, int Ho, int Wo,
                                                      int Kreal, int Kpad, __nv_bfloat16* __restrict__ out) {
  __shared__ int s_off[kIm2colMaxChunks];  // (r * W + s) * C + c of the chunk's first channel, -1 past Kreal
  __shared__ unsigned char s_r[kIm2colMaxChunks], s_s[kIm2colMaxChunks];
  const int nq = Kpad >> 3;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    const int k = q << 3;
    if (k < Kreal) {
      const int c = k % cg, rs = k / cg, sx = rs % kw, r = rs / kw;
      s_off[q] = (r * W + sx) * C + c;
      s_r[q] = (unsigned char)r;
      s_s[q] = (unsigned char)sx;
    } else {
      s_off[q] = -1;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int npos = B * Ho * Wo;
  for (int pos = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pos < npos; pos += warps) {
    const int b = pos / (Ho * Wo), rem = pos - b * (Ho * Wo);
    const int oh = rem / Wo, ow = rem - oh * Wo;
    const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
    const bool inside = ih0 >= 0 && iw0 >= 0 && ih0 + kh <= H && iw0 + kw <= W;
    const float* xw = x + ((ptrdiff_t)((size_t)b * H + ih0) * W + iw0) * C + c0;  // window origin (maybe outside)
    // a lane per half chunk (4 channels): the two lanes of a chunk read its 32
    // contiguous bytes in ONE load instruction (whole sectors; a lane reading
    // both halves took two instructions on half sectors each), 8-byte stores
    uint2* o = reinterpret_cast<uint2*>(out + (size_t)pos * Kpad);
#pragma unroll 4
    for (int q2 = lane; q2 < 2 * nq; q2 += 32) {
      const int q = q2 >> 1;
      const int off = s_off[q];
      bool ok = off >= 0;
      if (ok && !inside) {
        const int ih = ih0 + s_r[q], iw = iw0 + s_s[q];
        ok = ih >= 0 && ih < H && iw >= 0 && iw < W;
      }
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) a = __ldg(reinterpret_cast<const float4*>(xw + off + 4 * (q2 & 1)));
      const __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
      o[q2] = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
    }
  }
}

cudaError_t launch_im2col(const float* x, int B, int H, int W, int C, int kh, int kw, int stride, int pad, int c0,
                          int cg, int Ho, int Wo, int Kreal, int Kpad, __nv_bfloat16* out, cudaStream_t s,
                          int num_sms) {
  const long work = (long)B * Ho * Wo * (Kpad / 8);
  if (work >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing in the kernels
  const bool vec8 = (cg % 8 == 0) && (C % 4 == 0) && (c0 % 4 == 0) && (((uintptr_t)x & 15) == 0);
  ktimer_begin("k_im2col", s);
  if (vec8 && Kpad / 8 <= kIm2colMaxChunks && (long)B * Ho * Wo < (1L << 31) && kh < 256 && kw < 256)
    k_im2col_warp8<<<grid_for((long)B * Ho * Wo * 32, 256, num_sms), 256, 0, s>>>(x, B, H, W, C, kh, kw, stride, pad,
                                                                                 c0, cg, Ho, Wo, Kreal, Kpad, out);
  else if (vec8)
    k_im2col<true><<<grid_for(work, 256, num_sms), 256, 0, s>>>(x, B, H, W, C, kh, kw, stride, pad, c0, cg, Ho, Wo,
                                                                Kreal, Kpad, out);
  else if (cg == C && c0 == 0 && (W + 2 * pad) * cg >= 256 && im2col_rows_smem(kh, W, pad, cg, Kpad) <= kIm2colRowsMaxSmem && (long)B * Ho < (1L << 31) &&
           (long)B * Ho * Wo * Kpad < (1L << 40))
    k_im2col_rows<<<(unsigned)((long)B * Ho), 256, im2col_rows_smem(kh, W, pad, cg, Kpad), s>>>(
        x, B, H, W, C, kh, kw, stride, pad, c0, cg, Ho, Wo, Kreal, Kpad, out);
  else if (Kpad <= kIm2colMaxK && (long)B * Ho * Wo < (1L << 31) && (long)B * H * W * C < (1L << 40))
    k_im2col_warp<<<grid_for((long)B * Ho * Wo * 32, 256, num_sms), 256, 0, s>>>(x, B, H, W, C, kh, kw, stride, pad,
                                                                                c0, cg, Ho, Wo, Kreal, Kpad, out);
  else
    k_im2col<false><<<grid_for(work, 256, num_sms), 256, 0, s>>>(x, B, H, W, C, kh, kw, stride, pad, c0, cg, Ho, Wo,
                                                                 Kreal, Kpad, out);
  const cudaError_t e_ = launched();
  ktimer_end("k_im2col", s);
  return e_;
}

cudaError_t launch_lrn(const float* x, long npos, int C, float* y, cudaStream_t s, int num_sms) {
  ktimer_begin("k_lrn", s);
  if (C % 4 == 0 && npos * C < (1L << 31) && (((uintptr_t)x | (uintptr_t)y) & 15) == 0)
    k_lrn4<<<grid_for(npos * C / 4, 256, num_sms), 256, 0, s>>>(x, (int)npos, C, y);
  else
    k_lrn<<<grid_for(npos * C, 256, num_sms), 256, 0, s>>>(x, npos, C, y);
  const cudaError_t e_ = launched();
  ktimer_end("k_lrn", s);
  return e_;
}

cudaError_t launch_maxpool(const float* x, int B, int H, int W, int C, int k, int st, float* y, cudaStream_t s,
                           int num_sms) {
  const int Ho = (H - k) / st + 1, Wo = (W - k) / st + 1;
  ktimer_begin("k_maxpool", s);
  if (C % 4 == 0 && (long)B * H * W * C < (1L << 31) && (((uintptr_t)x | (uintptr_t)y) & 15) == 0)
    k_maxpool4<<<grid_for((long)B * Ho * Wo * C / 4, 256, num_sms), 256, 0, s>>>(
        reinterpret_cast<const float4*>(x), B, H, W, C / 4, k, st, Ho, Wo, reinterpret_cast<float4*>(y));
  else
    k_maxpool<<<grid_for((long)B * Ho * Wo * C, 256, num_sms), 256, 0, s>>>(x, B, H, W, C, k, st, Ho, Wo, y);
  const cudaError_t e_ = launched();
  ktimer_end("k_maxpool", s);
  return e_;
}

}  // namespace cdn
