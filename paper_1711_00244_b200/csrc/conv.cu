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

// A launch as a programmatic dependent of the stream's previous kernel: the
// kernel's CTAs may be scheduled while that kernel drains (launch latency and
// prologue hidden); it touches nothing the stream's earlier work wrote before
// pdl_wait().  Off by default (CDN_CONV_PDL=1 turns it on): measured slower on
// AlexNet at B = 64 (C4 0.456 -> 0.476 ms) -- the dependents' CTAs (the halo
// GEMM's hold ~200 KB of shared memory each) take SM slots from the kernel
// still running and then sit in griddepcontrol.wait.
template <typename... KArgs, typename... Args>
cudaError_t conv_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  static const int mode = [] {
    const char* e = std::getenv("CDN_CONV_PDL");
    return e ? std::atoi(e) : 0;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = mode ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

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

__device__ __forceinline__ void store_out(float* p, float o) { *p = o; }
__device__ __forceinline__ void store_out(__nv_bfloat16* p, float o) { *p = __float2bfloat16_rn(o); }

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
  int TP;     // filter taps per pipeline stage (the most, <= kHTPMax, that leaves two stages)
  int klast;  // K16 slices of a group's last 64-channel chunk that hold real channels (the rest multiply zeros)
  const float* bias;
  float* out;
  __nv_bfloat16* out_bf;  // non-null: the output as bf16 (RNE), the next CONV layer's input (ldo = its channels)
};

constexpr int kHEpiWarps = 16;
constexpr int kHTPMax = 4;  // most filter taps per pipeline stage (HaloArgs::TP)
constexpr int kHThreads = 64 + 32 * kHEpiWarps;

__global__ void __launch_bounds__(kHThreads, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap th, const __grid_constant__ CUtensorMap tb, const HaloArgs h) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  constexpr int f_bytes = kBM * kBK * 2;  // one filter tile (128 filters x 64 K)
  // TP taps per filter stage: one barrier round (wait, fence, commit -- ~300
  // clocks of the MMA thread's serial time) per TP taps instead of per tap
  const int kHTP = h.TP, s_bytes = kHTP * f_bytes;
  unsigned char* sH = smem;                   // halo stages
  unsigned char* sF = smem + h.SA * h.halo_bytes;  // filter stages
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sF + h.SB * s_bytes);
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
  pdl_wait();  // (barriers and tensor memory were set up under the previous kernel's tail)
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
      // (Both single-thread roles step their ring slot, phase, tap coordinates and
      // descriptors instead of dividing per tap: one thread's dependent
      // instructions issue ~4 clocks apart, and ~100 of them per tap -- three
      // divisions by run-time values among them -- had set the kernel's pace at
      // ~1000 clocks per tap whatever the tile size, ring depth or MMA count.)
      const int SA = h.SA, SB = h.SB, nch = h.nch;
      int sa = 0, pa = 1, sb = 0, pb = 1;  // ring slots and the parity their empty barriers are waited on
      for (int t = blockIdx.x; t < h.tiles; t += gridDim.x) {
        int img, f0, ys, m, z;
        decode(t, img, f0, ys, m, z);
        const int c_ch = z * h.cgp, m0 = m * kBM;
        for (int ch = 0; ch < nch; ++ch) {
          mbar_wait(&hempty[sa], (uint32_t)pa);
          mbar_arrive_expect_tx(&hfull[sa], (uint32_t)(h.HR * h.P * 128));
          tma4d(sH + sa * h.halo_bytes, &th, c_ch + ch * kBK, -h.pad, ys - h.pad, img, &hfull[sa]);
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
          int kc = ch * kBK;  // K coordinate of (tap, ch): (tap * nch + ch) * 64
          for (int tap = 0; tap < taps; tap += kHTP) {
            const int n = taps - tap < kHTP ? taps - tap : kHTP;  // taps of this stage
            mbar_wait(&fempty[sb], (uint32_t)pb);
            mbar_arrive_expect_tx(&ffull[sb], (uint32_t)(n * f_bytes));
            for (int j = 0; j < n; ++j, kc += nch * kBK) tma3d(sF + sb * s_bytes + j * f_bytes, &tb, kc, m0, z, &ffull[sb]);
            if (++sb == SB) {
              sb = 0;
              pb ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: per tap 4 x (128 filters x NT positions x 16)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(h.NT >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      const int SA = h.SA, SB = h.SB, nch = h.nch, kw = h.kw, klast = h.klast;
      const uint64_t fdesc0 = sw128_desc(smem_addr(sF));
      const uint32_t fstep = (uint32_t)(f_bytes >> 4);               // descriptor units (16 B) per filter tile
      const uint32_t rstep = (uint32_t)((h.P - kw) * 8);             // B start: next kernel row (after kw taps of +8)
      int sa = 0, pa = 0, sb = 0, pb = 0, i = 0;
      uint64_t ad = fdesc0;
      for (int t = blockIdx.x; t < h.tiles; t += gridDim.x, ++i) {
        int img, f0, ys, m, z;
        decode(t, img, f0, ys, m, z);
        const int off0 = f0 - ys * h.P;
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(buf * h.NT);
        uint32_t first = 0;  // 0 for the tile's first MMA (overwrites the accumulator)
        for (int ch = 0; ch < nch; ++ch) {
          mbar_wait(&hfull[sa], (uint32_t)pa);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // tap (r, s) reads the halo from row off0 + r P + s: +8 units per s, + rstep more per r
          uint64_t bd = sw128_desc(smem_addr(sH + sa * h.halo_bytes) + (uint32_t)off0 * 128u);
          // (a last chunk padded from 48 to 64 channels -- conv1's super-pixels,
          // conv2's groups -- issues 3 of the 4 K16 slices: the 4th is zeros x zeros)
          const int nk = ch + 1 == nch ? klast : kBK / 16;
          int sx = 0;
          for (int tap = 0; tap < taps; tap += kHTP) {
            const int n = taps - tap < kHTP ? taps - tap : kHTP;
            mbar_wait(&ffull[sb], (uint32_t)pb);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int j = 0; j < n; ++j) {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                if (k < nk) {
                  umma_bf16(acc, ad + j * fstep + 2 * k, bd + 2 * k, idesc, first);
                  first = 1;
                }
              bd += 8;
              if (++sx == kw) {
                sx = 0;
                bd += rstep;
              }
            }
            umma_commit(&fempty[sb]);
            ad += kHTP * fstep;
            if (++sb == SB) {
              sb = 0;
              pb ^= 1;
              ad = fdesc0;
            }
          }
          umma_commit(&hempty[sa]);
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---- epilogue warps: TMEM lane = filter (quadrant warp % 4), column = flattened
    // position; the quadrant's two warps take the two halves of the columns
    // (kHEpiWarps / 4 warps per quadrant, each a share of the columns in whole 16-column chunks)
    constexpr int kParts = kHEpiWarps / 4;
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int chunks = h.NT / 16;
    const int c_lo = (chunks * part / kParts) * 16, c_hi = (chunks * (part + 1) / kParts) * 16;
    int i = 0;
    for (int t = blockIdx.x; t < h.tiles; t += gridDim.x, ++i) {
      int img, f0, ys, m, z;
      decode(t, img, f0, ys, m, z);
      const int buf = i & 1;
      const int fl = m * kBM + q * 32 + lane;  // this lane's filter in the group
      const bool fok = fl < h.Nrows;
      const float bv = fok ? h.bias[z * h.Nrows + fl] : 0.f;
      const size_t o0 = (size_t)img * h.Ho * h.Wo * h.ldo + z * h.Nrows + fl;
      // (y0, x0) = the position of a 16-column chunk's first column (uniform over
      // the warp).  Within the chunk every column derives its own position from
      // that alone -- at most two row wraps in 16 columns (P >= 8) -- so the 16
      // stores carry no serial chain: stepping (x, y) column by column had the
      // epilogue warps latency-bound at ~150 clocks per column (conv1: 20 k clocks
      // per tile against ~5 k of MMAs).
      int y0 = (f0 + c_lo) / h.P, x0 = f0 + c_lo - y0 * h.P;
      const int drop = h.P - h.Wo;
      mbar_wait(&acc_full[buf], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * h.NT);
      auto cols = [&](auto* out) {
        // (a quadrant past the layer's filters -- conv1: 96 of 128 -- only releases the buffer)
        for (int c = c_lo; c < c_hi && __any_sync(0xffffffffu, fok); c += 16) {
          float v[16];
          tmem_ld16(tq + (uint32_t)c, v);
          auto* pc = out + o0 + (size_t)(y0 * h.Wo + x0) * h.ldo;
          if (x0 + 16 <= h.Wo && y0 < h.Ho) {  // the chunk inside one output row: no per-column tests
            if (fok) {
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                float o = v[u] + bv;
                if (h.relu) o = fmaxf(o, 0.f);
                store_out(pc + (ptrdiff_t)u * h.ldo, o);
              }
            }
            x0 += 16;
            continue;
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int wraps = (x0 + u >= h.P) + (x0 + u >= 2 * h.P);
            const int xu = x0 + u - wraps * h.P, yu = y0 + wraps;
            float o = v[u] + bv;
            if (h.relu) o = fmaxf(o, 0.f);
            if (fok && xu < h.Wo && yu < h.Ho) store_out(pc + (ptrdiff_t)(u - wraps * drop) * h.ldo, o);
          }
          x0 += 16;
          while (x0 >= h.P) {
            x0 -= h.P;
            ++y0;
          }
        }
      };
      if (h.out_bf) cols(h.out_bf);
      else cols(h.out);
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

// Max-pool, optionally with the cross-channel LRN ahead of it in the same pass
// (AlexNet conv2: the LRN output is never written), 8 channels per thread; the
// result as fp32 NHWC, or (BF) as the next CONV layer's bf16 input -- G groups
// of cg channels padded with zeros to cgp (rounding is monotonic, so the max
// of the rounded values is the rounded max; reading C-21).  LRN is evaluated
// per window position (2.25 x per input value for 3 x 3 / 2): the same
// expression and summation order as k_lrn4.
template <bool LRN, bool BF>
__global__ void __launch_bounds__(256) k_pool8(const float* __restrict__ x, int B, int H, int W, int C, int k, int st,
                                               int Ho, int Wo, float* __restrict__ yf, __nv_bfloat16* __restrict__ yb,
                                               int G, int cg, int cgp) {
  pdl_wait();
  const int Q = (BF ? G * cgp : C) / 8;
  const long total = (long)B * Ho * Wo * Q;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % Q) * 8;
    long p = i / Q;
    const int ow = (int)(p % Wo);
    const long t = p / Wo;
    const int oh = (int)(t % Ho), b = (int)(t / Ho);
    int cin = c8;
    if (BF) {
      const int z = c8 / cgp, c = c8 - z * cgp;
      if (c >= cg) {  // (cg % 8 == 0: a chunk is all real or all padding)
        reinterpret_cast<uint4*>(yb)[i] = make_uint4(0u, 0u, 0u, 0u);
        continue;
      }
      cin = z * cg + c;
    }
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
    const float* xb = x + (((size_t)b * H + (size_t)oh * st) * W + (size_t)ow * st) * C + cin;
    for (int r = 0; r < k; ++r) {
#pragma unroll 3
      for (int q = 0; q < k; ++q) {
        const float4* px = reinterpret_cast<const float4*>(xb + ((size_t)r * W + q) * C);
        if (LRN) {
          float a[16];  // channels cin - 4 .. cin + 11 (0 outside: adds nothing to a window sum)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int c = cin - 4 + 4 * v;
            const float4 f = (c >= 0 && c < C) ? __ldg(px - 1 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
            a[4 * v] = f.x; a[4 * v + 1] = f.y; a[4 * v + 2] = f.z; a[4 * v + 3] = f.w;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float sq = 0.f;
#pragma unroll
            for (int w = 0; w < 5; ++w) {
              const int cq = cin + j - 2 + w;
              if (cq >= 0 && cq < C) sq = fmaf(a[j + 2 + w], a[j + 2 + w], sq);
            }
            m[j] = fmaxf(m[j], a[j + 4] * exp2f(-0.75f * __log2f(2.0f + (1e-4f / 5.0f) * sq)));
          }
        } else {
          const float4 f0 = __ldg(px), f1 = __ldg(px + 1);
          m[0] = fmaxf(m[0], f0.x); m[1] = fmaxf(m[1], f0.y); m[2] = fmaxf(m[2], f0.z); m[3] = fmaxf(m[3], f0.w);
          m[4] = fmaxf(m[4], f1.x); m[5] = fmaxf(m[5], f1.y); m[6] = fmaxf(m[6], f1.z); m[7] = fmaxf(m[7], f1.w);
        }
      }
    }
    if (BF) {
      __nv_bfloat162 h[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(m[2 * j], m[2 * j + 1]);
      reinterpret_cast<uint4*>(yb)[i] = *reinterpret_cast<const uint4*>(h);
    } else {
      float4* dst = reinterpret_cast<float4*>(yf + p * C + c8);
      dst[0] = make_float4(m[0], m[1], m[2], m[3]);
      dst[1] = make_float4(m[4], m[5], m[6], m[7]);
    }
  }
}

// (2 + 1e-4/5 * sq)^-0.75 (reading C-20) through lg2 / ex2 without the library
// wrappers' denormal branches: the argument is >= 2 and the exponent within
// [-96, -0.75], where exp2f(-0.75f * __log2f(t)) returns the same bits.
__device__ __forceinline__ float lrn_scale(float sq) {
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(fmaf(1e-4f / 5.0f, sq, 2.0f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-0.75f * l));
  return r;
}

// LRN + max-pool with every LRN value computed once per pooled row: a CTA takes
// one (image, pooled row) at a time, evaluates LRN over the k input rows under it
// (contiguous in NHWC: k * W * C floats) into shared memory -- fp32, or already
// rounded to bf16 when the output is the next CONV layer's input (rounding is
// monotonic: the max of the rounded values is the rounded max) -- then pools
// from there.  k_pool8<true> re-evaluated LRN per window position (k * k / st^2
// = 2.25 x) and was bound by it (conv2: 39 us); here rows overlap only
// vertically (k / st = 1.5 x).  The same expression and summation order as
// k_lrn4.  Output layouts as k_pool8.
template <bool BF>
__global__ void __launch_bounds__(256) k_lrn_pool_rows(const float* __restrict__ x, int B, int H, int W, int C, int k,
                                                       int st, int Ho, int Wo, float* __restrict__ yf,
                                                       __nv_bfloat16* __restrict__ yb, int G, int cg, int cgp, int R) {
  // R pooled rows per item: (R - 1) st + k input rows, each evaluated once per item
  extern __shared__ __align__(16) unsigned char sm_lp[];
  float* sf = reinterpret_cast<float*>(sm_lp);
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(sm_lp);
  pdl_wait();
  const int Q8 = C / 8, HoR = (Ho + R - 1) / R;
  const int Co = BF ? G * cgp : C, Qo = Co / 8;
  for (int it = blockIdx.x; it < B * HoR; it += gridDim.x) {
    const int b = it / HoR, oh = (it - b * HoR) * R;
    const int Rc = min(R, Ho - oh);
    const int n1 = ((Rc - 1) * st + k) * W * Q8, n2 = Rc * Wo * Qo;
    const float* xr = x + ((size_t)b * H + (size_t)oh * st) * W * C;
    // two items per thread per round (the eight 16-byte loads issued before either
    // is used); (pixel, chunk) of item j stepped, not divided, from round to round
    int pixs[2], c8s[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = threadIdx.x + e * blockDim.x;
      pixs[e] = j / Q8;
      c8s[e] = j - pixs[e] * Q8;  // (chunk index; * 8 = first channel)
    }
    const int dpix = 2 * blockDim.x / Q8, dq = 2 * blockDim.x - dpix * Q8;
    float4 f[2][4];
    // slot e's next item: channels c8 - 4 .. c8 + 11 (0 outside: adds nothing to a window sum)
    auto load = [&](int e, bool in) {
      const int c8 = c8s[e] * 8;
      const float4* px = reinterpret_cast<const float4*>(xr + (size_t)pixs[e] * C + c8);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = c8 - 4 + 4 * v;
        f[e][v] = (in && c >= 0 && c < C) ? __ldg(px - 1 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto comp = [&](int e, bool in) {
      if (in) {
        const float a[16] = {f[e][0].x, f[e][0].y, f[e][0].z, f[e][0].w, f[e][1].x, f[e][1].y, f[e][1].z, f[e][1].w,
                             f[e][2].x, f[e][2].y, f[e][2].z, f[e][2].w, f[e][3].x, f[e][3].y, f[e][3].z, f[e][3].w};
        float o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // q from c - 2 to c + 2 in k_lrn4's order; channels outside [0, C) hold 0 and fma(0, 0, sq) = sq
          float sq = 0.f;
#pragma unroll
          for (int w = 0; w < 5; ++w) sq = fmaf(a[u + 2 + w], a[u + 2 + w], sq);
          o[u] = a[u + 4] * lrn_scale(sq);
        }
        const size_t so = (size_t)pixs[e] * C + c8s[e] * 8;
        if (BF) {
          __nv_bfloat162 h[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) h[u] = __floats2bfloat162_rn(o[2 * u], o[2 * u + 1]);
          *reinterpret_cast<uint4*>(sb + so) = *reinterpret_cast<const uint4*>(h);
        } else {
          float4* d = reinterpret_cast<float4*>(sf + so);
          d[0] = make_float4(o[0], o[1], o[2], o[3]);
          d[1] = make_float4(o[4], o[5], o[6], o[7]);
        }
      }
      pixs[e] += dpix;
      c8s[e] += dq;
      if (c8s[e] >= Q8) {
        c8s[e] -= Q8;
        ++pixs[e];
      }
    };
    // the loads of one slot stay in flight while the other slot is evaluated
    const int bd = blockDim.x;
    load(0, (int)threadIdx.x < n1);
    for (int j0 = threadIdx.x; j0 < n1; j0 += 2 * bd) {
      load(1, j0 + bd < n1);
      comp(0, true);
      load(0, j0 + 2 * bd < n1);
      comp(1, j0 + bd < n1);
    }
    __syncthreads();
    const size_t orow = ((size_t)b * Ho + oh) * Wo;  // (the item's pooled rows are consecutive: orow + rr * Wo + ow)
    for (int j = threadIdx.x; j < n2; j += blockDim.x) {
      const int pw = j / Qo, c8 = (j - pw * Qo) * 8;  // pw = rr * Wo + ow
      const int rr = pw / Wo, ow = pw - rr * Wo;
      const size_t s0 = ((size_t)rr * st * W + (size_t)ow * st) * C;
      if (BF) {
        uint4* dst = reinterpret_cast<uint4*>(yb + (orow + pw) * Co + c8);
        const int z = c8 / cgp, c = c8 - z * cgp;
        if (c >= cg) {  // (cg % 8 == 0: a chunk is all real or all padding)
          *dst = make_uint4(0u, 0u, 0u, 0u);
          continue;
        }
        const __nv_bfloat16* p0 = sb + s0 + z * cg + c;
        uint4 m4 = *reinterpret_cast<const uint4*>(p0);
        __nv_bfloat162* m = reinterpret_cast<__nv_bfloat162*>(&m4);
        for (int r = 0; r < k; ++r)
          for (int q = 0; q < k; ++q) {
            const uint4 v4 = *reinterpret_cast<const uint4*>(p0 + ((size_t)r * W + q) * C);
            const __nv_bfloat162* v = reinterpret_cast<const __nv_bfloat162*>(&v4);
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = __hmax2(m[u], v[u]);
          }
        *dst = m4;
      } else {
        const float* p0 = sf + s0 + c8;
        float m[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m[u] = -INFINITY;
        for (int r = 0; r < k; ++r)
          for (int q = 0; q < k; ++q) {
            const float4* v = reinterpret_cast<const float4*>(p0 + ((size_t)r * W + q) * C);
            const float4 f0 = v[0], f1 = v[1];
            m[0] = fmaxf(m[0], f0.x); m[1] = fmaxf(m[1], f0.y); m[2] = fmaxf(m[2], f0.z); m[3] = fmaxf(m[3], f0.w);
            m[4] = fmaxf(m[4], f1.x); m[5] = fmaxf(m[5], f1.y); m[6] = fmaxf(m[6], f1.z); m[7] = fmaxf(m[7], f1.w);
          }
        float4* dst = reinterpret_cast<float4*>(yf + (orow + pw) * C + c8);
        dst[0] = make_float4(m[0], m[1], m[2], m[3]);
        dst[1] = make_float4(m[4], m[5], m[6], m[7]);
      }
    }
    __syncthreads();  // the next item overwrites the rows
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
  static const int nt_cap = [] {  // CDN_HALO_NT: widest position block (experiment knob, <= 256)
    const char* e = std::getenv("CDN_HALO_NT");
    return e ? std::max(16, std::min(256, std::atoi(e))) : 256;
  }();
  h.spi = (flat + nt_cap - 1) / nt_cap;
  h.NT = ((flat + h.spi - 1) / h.spi + 15) & ~15;
  h.HR = (h.NT - 1) / h.P + 2 + kh - 1;  // a block's output rows (<= (NT-1)/P + 2) + kh - 1
  if (h.P > 256 || h.HR > 256 || h.P < 8) return false;  // (P >= 8: the epilogue allows two row wraps per 16 columns)
  const int rows_alloc = std::max(h.HR * h.P, (kh - 1) * h.P + kw + h.P + h.NT);  // + the dropped positions' overreach
  h.halo_bytes = (rows_alloc * 128 + 1023) & ~1023;
  h.nch = cgp / kBK;
  h.mtl = (Nrows + kBM - 1) / kBM;
  h.talloc = 32;
  while (h.talloc < 2 * h.NT) h.talloc <<= 1;
  h.SA = 2;
  const size_t fixed = 1024 + 256;
  const long left = 225L * 1024 - (long)fixed - (long)h.SA * h.halo_bytes;
  static const int sb_cap = [] {  // CDN_HALO_SB: filter stages cap (experiment knob)
    const char* e = std::getenv("CDN_HALO_SB");
    return e ? std::max(3, std::atoi(e)) : 8;
  }();
  static const int tp_cap = [] {  // CDN_HALO_TP: taps per stage cap (experiment knob)
    const char* e = std::getenv("CDN_HALO_TP");
    return e ? std::max(1, std::min(kHTPMax, std::atoi(e))) : 3;  // (4 on conv3-5, two stages: 35.1 / 30.0 / 19.5 vs 34.2 / 29.5 / 18.8 us)
  }();
  h.TP = std::min(tp_cap, kh * kw);
  while (h.TP > 1 && left / (h.TP * kBM * kBK * 2) < 2) --h.TP;
  h.SB = (int)std::min<long>(sb_cap, left / (h.TP * kBM * kBK * 2));
  if (h.SB < 2 || h.talloc > 512) return false;
  h.tiles = B * h.spi * h.mtl * G;
  smem = fixed + (size_t)h.SA * h.halo_bytes + (size_t)h.SB * h.TP * kBM * kBK * 2;
  return smem <= 227 * 1024;
}

bool conv_halo_applies(int G, int cgp, int kh, int kw, int pad, int Ho, int Wo, int Nrows, int lrn) {
  HaloArgs h;
  size_t smem = 0;
  return kh == kw && halo_plan(1, G, cgp, kh, kw, pad, Ho, Wo, Nrows, lrn, h, smem);
}

cudaError_t launch_gemm_implicit(const __nv_bfloat16* act, int B, int H, int W, int G, int cgp, int kh, int kw,
                                 int pad, int Ho, int Wo, const __nv_bfloat16* Wt, int Nrows, const float* bias,
                                 int relu, float* out, int ldo, cudaStream_t s, int lrn, __nv_bfloat16* out_bf,
                                 int cg_real) {
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
      h.out_bf = out_bf;
      h.klast = kBK / 16;
      if (cg_real > 0 && cg_real <= cgp && cg_real > cgp - kBK) h.klast = (cg_real - (cgp - kBK) + 15) / 16;
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
      e = conv_launch(k_conv_halo, dim3(std::min(h.tiles, num_sms)), dim3(kHThreads), smem, s, th, tb, h);
      if (e != cudaSuccess) return e;
      const cudaError_t e_ = launched();
      ktimer_end("k_conv_halo", s);
      return e_;
    }
  }
  if (out_bf) return cudaErrorInvalidValue;  // (bf16 output: the halo kernel only, conv_halo_applies)
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
  pdl_wait();
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
  if (st == 4 && C == 3) {
    const cudaError_t e = conv_launch(k_s2d_bf16<4, 3>, dim3(grid), dim3(256), 0, s, x, B, H, W, Hs, Ws, cgp, out);
    if (e != cudaSuccess) return e;
  }
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

bool pool8_ok(int C, int k, int cg, int cgp) { return C % 8 == 0 && k >= 1 && (cg == 0 || (cg % 8 == 0 && cgp % 8 == 0)); }

cudaError_t launch_pool8(const float* x, int B, int H, int W, int C, int k, int st, int lrn, float* y,
                         __nv_bfloat16* yb, int G, int cg, int cgp, cudaStream_t s, int num_sms) {
  const int Ho = (H - k) / st + 1, Wo = (W - k) / st + 1;
  if (B <= 0 || Ho <= 0 || Wo <= 0) return cudaSuccess;
  if (!pool8_ok(C, k, yb ? cg : 0, cgp) || (yb && G * cg != C) ||
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(yb)) & 15))
    return cudaErrorInvalidValue;
  const long work = (long)B * Ho * Wo * ((yb ? G * cgp : C) / 8);
  const int grid = grid_for(work, 256, num_sms);
  ktimer_begin(lrn ? "k_lrn_pool" : "k_maxpool", s);
  static const int rows_mode = [] {  // CDN_LRN_POOL_ROWS=0: the per-window kernel (A/B knob)
    const char* e = std::getenv("CDN_LRN_POOL_ROWS");
    return e ? std::atoi(e) : 1;
  }();
  // pooled rows per item: one.  Two (1.25 x LRN evaluations per input value instead
  // of 1.5 x for 3 x 3 / 2) measured slower -- conv1 34 -> 38 us, conv2 23 -> 29 us:
  // half as many, larger CTAs (CDN_LRN_POOL_R, A/B knob)
  const size_t row_bytes = (size_t)W * C * (yb ? 2 : 4);
  static const int r_env = [] {
    const char* e = std::getenv("CDN_LRN_POOL_R");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  const int R = (size_t)((r_env - 1) * st + k) * row_bytes <= 160 * 1024 ? r_env : 1;
  const size_t smem = (size_t)((R - 1) * st + k) * row_bytes;
  if (lrn && rows_mode && smem <= 160 * 1024 && (long)B * Ho < (1L << 30)) {
    static thread_local size_t set_bf = 0, set_f = 0;
    size_t& set = yb ? set_bf : set_f;
    if (smem > 48 * 1024 && smem > set) {
      const cudaError_t e = yb ? cudaFuncSetAttribute(k_lrn_pool_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                               : cudaFuncSetAttribute(k_lrn_pool_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      set = smem;
    }
    // resident CTAs, then a grid every CTA of which takes the same number of (image, row) items
    int per_sm = 0;
    if (yb) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lrn_pool_rows<true>, 256, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lrn_pool_rows<false>, 256, smem);
    per_sm = std::max(per_sm, 1);
    const long items = (long)B * ((Ho + R - 1) / R), resident = (long)num_sms * per_sm;
    const long rounds = (items + resident - 1) / resident;
    const int g = (int)((items + rounds - 1) / rounds);
    const cudaError_t e = yb ? conv_launch(k_lrn_pool_rows<true>, dim3(g), dim3(256), smem, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp, R)
                             : conv_launch(k_lrn_pool_rows<false>, dim3(g), dim3(256), smem, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp, R);
    if (e != cudaSuccess) return e;
  } else {
    const cudaError_t e =
        lrn && yb ? conv_launch(k_pool8<true, true>, dim3(grid), dim3(256), 0, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp)
        : lrn     ? conv_launch(k_pool8<true, false>, dim3(grid), dim3(256), 0, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp)
        : yb      ? conv_launch(k_pool8<false, true>, dim3(grid), dim3(256), 0, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp)
                  : conv_launch(k_pool8<false, false>, dim3(grid), dim3(256), 0, s, x, B, H, W, C, k, st, Ho, Wo, y, yb, G, cg, cgp);
    if (e != cudaSuccess) return e;
  }
  const cudaError_t e_ = launched();
  ktimer_end(lrn ? "k_lrn_pool" : "k_maxpool", s);
  return e_;
}

}  // namespace cdn
