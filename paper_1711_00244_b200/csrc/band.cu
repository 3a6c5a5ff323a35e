// Large-batch fused FC kernel (sm_100a): parallel Huffman decode -> gap prefix
// sum -> codebook dequantize -> sparse multiply -> bias -> ReLU, PAPER.md
// Alg. 1 lines 4-9 and Eq. 1-2, for B >= ~16 images.
//
// At large batch the layer is bound by the fp32 FMA / shared-memory datapath,
// not by the compressed bytes: every nonzero w_ij multiplies a
// contiguous batch vector x[j][b0:b0+BT].  Design:
//   * work unit = (block of R = 128 output rows, batch tile of BT = 32*VEC
//     images, range of column chunks).  Units are independent; K-split
//     partials are reduced in a fixed order (deterministic).
//   * the load-time interval index (host.hpp IntervalIndex) gives, for every
//     (row, interval of Wi columns), the decoder state at the interval start
//     AND the number of real tokens in it.  So all (row, interval) decode
//     tasks of a chunk are independent and know where their output goes:
//       - DECODE phase: all 16 worker warps, one lane per (row, interval):
//         pad-folding val LUT + gap LUT in shared memory, c += g + 1 (Alg. 1
//         l.7, reading C-01), w = C[sym] (l.8); (w, smem offset of x[c])
//         entries written at the row's exclusive nnz prefix (a segmented
//         shuffle scan of the per-interval counts);
//       - FMA phase: per band (= interval) the same warps, 8 rows each and
//         lanes over the batch tile: one broadcast LDS.128 per two entries +
//         VEC-wide LDS of x + VEC FMAs into register accumulators (l.9).
//   * a PRODUCER warp streams the activation bands x[i*Wi:(i+1)*Wi][b0:b0+BT]
//     into a 3-stage shared-memory ring with 2D TMA (UTMALDG) on full/empty
//     mbarriers, running ahead across chunk and unit boundaries.
//   * decoded weights never leave the SM (no HBM materialisation).
#include <cuda.h>

#include "dev_common.cuh"
#include "kernels.cuh"
#include "tmap.hpp"

namespace cdn {

namespace {

using namespace dev;

constexpr int kR = 128;                          // rows per unit
constexpr int kWorkWarps = 16;                   // FMA warps
constexpr int kWorkers = kWorkWarps * 32;
constexpr int kDecWarps = 8;                     // decode warps
constexpr int kDecoders = kDecWarps * 32;
constexpr int kThreads = kWorkers + kDecoders + 32;  // + 1 producer warp
constexpr int kRowsPerWarp = kR / kWorkWarps;    // 8
constexpr int kLC = 32;                          // list entries per row per chunk
constexpr int kMaxCint = 16;
constexpr int kStages = 2;                       // activation-band ring
constexpr int kLBufs = 2;                        // decoded-list ring
constexpr int kXStageBytes = 64 * 1024;
constexpr int kWorkBar = 1;                      // named barrier of the 16 FMA warps

struct BandArgs {
  const float* x;
  int ldx, B;
  float* y;
  int ldy, relu;
  float* ws;   // [tiles][S][kR][BT] split partials (S > 1)
  int* tctr;   // [tiles] arrival counters, zero between launches
  int S, nbt, units, nch;
  int ipb;     // intervals per band (one band = one X stage)
};

template <int VEC>
__device__ __forceinline__ void load_x(const unsigned char* p, float (&v)[VEC]) {
  if constexpr (VEC == 8) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    const float4 u = *reinterpret_cast<const float4*>(p + 512);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    v[4] = u.x; v[5] = u.y; v[6] = u.z; v[7] = u.w;
  } else if constexpr (VEC == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (VEC == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = *reinterpret_cast<const float*>(p);
  }
}

// 2D tensor copy (SASS UTMALDG) of an activation band box x[c0:c0+Wi][b0:b0+BT]
// into shared memory; out-of-range rows / images are zero-filled by the TMA.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c_inner, int c_outer,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_addr(dst)), "l"(map), "r"(c_inner), "r"(c_outer), "r"(smem_addr(bar))
      : "memory");
}

struct UnitCoord {
  int tile, sp, rb, bt, i0, i1;  // intervals [i0, i1)
};

__device__ __forceinline__ UnitCoord unit_coord(const FcDev& L, const BandArgs& a, int u) {
  UnitCoord c;
  c.sp = u % a.S;
  c.tile = u / a.S;
  c.rb = c.tile / a.nbt;
  c.bt = c.tile % a.nbt;
  const int ch0 = (int)(((long)c.sp * a.nch) / a.S), ch1 = (int)(((long)(c.sp + 1) * a.nch) / a.S);
  c.i0 = ch0 * L.Cint;
  c.i1 = min(L.NI, ch1 * L.Cint);
  return c;
}

// Task-local MSB-first reader: three words loaded up front (an interval's
// codes usually fit), later words on demand.
struct TReader {
  const uint32_t* p;
  uint32_t off, w0, w1, w2;
  __device__ __forceinline__ void init(const uint32_t* words, uint32_t bit) {
    p = words + (bit >> 5);
    off = bit & 31;
    w0 = ldg_u32(p);
    w1 = ldg_u32(p + 1);
    w2 = ldg_u32(p + 2);
    p += 3;
  }
  __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, off); }
  __device__ __forceinline__ void skip(uint32_t n) {  // n <= 32
    off += n;
    if (off >= 32) {
      off -= 32;
      w0 = w1;
      w1 = w2;
      w2 = ldg_u32(p);
      ++p;
    }
  }
};

// Batch column of accumulator v of a lane: lanes cover 16-byte quads so every
// LDS.128 of x is one contiguous 512-byte warp access (VEC 8 = two of them).
template <int VEC>
__device__ __forceinline__ int bcol(int lane, int v) {
  if constexpr (VEC == 8) return (v >> 2) * 128 + lane * 4 + (v & 3);
  else return lane * VEC + v;
}

struct Task {
  int rl, j;
  size_t q;
  uint32_t m, off;
  uint2 st;
  TReader vr, gr;
};

template <int VEC>
__global__ void __launch_bounds__(kThreads, 1)
    k_fc_band(FcDev L, BandArgs a, const __grid_constant__ CUtensorMap tmx) {
  constexpr int BT = 32 * VEC;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* xs = smem;                                                  // [kStages][ipb*Wi][BT] fp32
  float2* lists = reinterpret_cast<float2*>(smem + kStages * kXStageBytes);  // [kLBufs][kR][kLC] (w, x offset)
  uint32_t* bse = reinterpret_cast<uint32_t*>(lists + kLBufs * kR * kLC);   // [kLBufs][kR][kMaxCint]
  uint64_t* full = reinterpret_cast<uint64_t*>(bse + kLBufs * kR * kMaxCint);
  uint64_t* empty = full + kStages;
  uint64_t* lfull = empty + kStages;
  uint64_t* lempty = lfull + kLBufs;
  int* meta = reinterpret_cast<int*>(lempty + kLBufs);                      // [kLBufs][4]: ni | flags, tile, sp
  int* s_last = meta + kLBufs * 4;                                          // [4]
  uint32_t* s_flut = reinterpret_cast<uint32_t*>(s_last + 4);
  uint32_t* s_glut = s_flut + (1 << L.Lf);
  float* s_cb = reinterpret_cast<float*>(s_glut + (1 << L.Lg));
  uint32_t* s_vtab = reinterpret_cast<uint32_t*>(s_cb + L.ncb);
  uint32_t* s_gtab = s_vtab + 99;
  uint16_t* s_vsorted = reinterpret_cast<uint16_t*>(s_gtab + 99);
  uint16_t* s_gsorted = s_vsorted + (L.nvs + 1);
  {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < (1 << L.Lf); i += nt) s_flut[i] = L.flut[i];
    for (int i = tid; i < (1 << L.Lg); i += nt) s_glut[i] = L.glut[i];
    for (int i = tid; i < L.ncb; i += nt) s_cb[i] = L.codebook[i];
    for (int i = tid; i < 99; i += nt) { s_vtab[i] = L.vtab[i]; s_gtab[i] = L.gtab[i]; }
    for (int i = tid; i < L.nvs; i += nt) s_vsorted[i] = L.vsorted[i];
    for (int i = tid; i < L.ngs; i += nt) s_gsorted[i] = L.gsorted[i];
    if (tid == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], kWorkWarps);
      }
      for (int b = 0; b < kLBufs; ++b) {
        mbar_init(&lfull[b], kDecWarps);
        mbar_init(&lempty[b], kWorkWarps);
      }
      mbar_fence_init();
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ipb = a.ipb;
  const uint32_t xstage_bytes = (uint32_t)(L.Wi * ipb) * BT * 4;
  const int Cint = L.Cint;

  if (warp == kWorkWarps + kDecWarps) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      uint32_t g = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const UnitCoord c = unit_coord(L, a, u);
        for (int ib = c.i0; ib < c.i1; ib += Cint) {
          const int ni = min(Cint, c.i1 - ib);
          for (int b0 = 0; b0 < ni; b0 += ipb, ++g) {
            const int s = g % kStages;
            mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], xstage_bytes);
            tma_load_2d(xs + s * kXStageBytes, &tmx, c.bt * BT, (ib + b0) * L.Wi, &full[s]);
          }
        }
      }
    }
    return;
  }

  if (warp >= kWorkWarps) {
    // ------------------------------------------------------------ decode warps
    // one lane per (row, interval) task of a chunk; known output offsets (the
    // interval index carries each interval's real-token count)
    const int dtid = threadIdx.x - kWorkers;
    const int dwarp = warp - kWorkWarps;
    const int fsh = 32 - L.Lf, gsh = 32 - L.Lg, k = L.k;
    const int npass = (kR * Cint + kDecoders - 1) / kDecoders;
    uint32_t c = 0;  // chunk counter (list ring position)
    for (int u = blockIdx.x;; u += gridDim.x) {
      const bool done = u >= a.units;
      UnitCoord uc{};
      if (!done) uc = unit_coord(L, a, u);
      // every unit emits >= 1 chunk (an empty K-split still flushes its partial)
      for (int ib = uc.i0;; ib += Cint, ++c) {
        const int lb = c % kLBufs;
        mbar_wait(&lempty[lb], ((c / kLBufs) & 1) ^ 1);
        if (done) {
          if (dwarp == 0 && lane == 0) meta[lb * 4] = 1 << 30;
          __syncwarp();
          if (lane == 0) mbar_arrive(&lfull[lb]);
          ++c;
          break;
        }
        const int ni = max(0, min(Cint, uc.i1 - ib));
        const bool last_chunk = ib + Cint >= uc.i1;
        float2* lst = lists + (size_t)lb * kR * kLC;
        uint32_t* bs = bse + (size_t)lb * kR * kMaxCint;
        for (int pass = 0; pass < npass; pass += 2) {
          Task tk[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = (pass + h) * kDecoders + dtid;
            tk[h].rl = t / Cint;
            tk[h].j = t % Cint;
            const int row = uc.rb * kR + tk[h].rl;
            const bool valid = pass + h < npass && tk[h].rl < kR && row < L.nrows && tk[h].j < ni;
            tk[h].q = (size_t)row * L.NI + ib + tk[h].j;
            tk[h].m = valid ? (uint32_t)L.ivm[tk[h].q] : 0u;
            tk[h].st = valid ? L.ivg[tk[h].q] : make_uint2(0, 0);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t nnz = tk[h].m >> 8;
            uint32_t off = nnz;  // inclusive scan over the Cint lanes of this row
            for (int o = 1; o < Cint; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, off, o, Cint);
              if (tk[h].j >= o) off += y;
            }
            off -= nnz;
            tk[h].off = off;
            if (pass + h < npass && tk[h].rl < kR) bs[tk[h].rl * kMaxCint + tk[h].j] = off | ((off + nnz) << 16);
            if (nnz) {
              tk[h].vr.init(L.vw, tk[h].st.x);
              tk[h].gr.init(L.gw, tk[h].st.y);
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t nnz = tk[h].m >> 8;
            if (!nnz) continue;
            const int iv = ib + tk[h].j;
            const int bstart = (ib + (tk[h].j / ipb) * ipb) * L.Wi;  // first column of the band's X stage
            int col = iv * L.Wi - (int)(tk[h].m & 0xFFu) - 1;
            float2* dst = lst + tk[h].rl * kLC + tk[h].off;
            TReader& vr = tk[h].vr;
            TReader& gr = tk[h].gr;
            uint32_t ndone = 0;
            while (ndone < nnz) {
              const uint32_t w = vr.peek();
              const uint32_t e = s_flut[w >> fsh];
              uint32_t len, sym, pads, pbits;
              if (e != kFoldSlow) {
                len = e >> 28;
                sym = e & 0xFFu;
                pads = (e >> 24) & 15u;
                pbits = (e >> 8) & 0xFFFFu;
              } else {
                const uint32_t r = slow_sym(w, L.Lf + 1, s_vtab, s_vsorted, L.vmax);
                len = r >> 16;
                sym = r & 0xFFu;
                pads = sym == 0;  // a long pad code (C-04: symbol 0 <=> pad)
                pbits = pads ? (uint32_t)L.Lpg : 0u;
              }
              vr.skip(len);
              col += (int)(pads << k);
              if (pbits <= 32) {
                gr.skip(pbits);
              } else {
                for (uint32_t z = 0; z < pads; ++z) gr.skip((uint32_t)L.Lpg);  // long pad codes (rare)
              }
              if (sym) {
                const uint32_t gwin = gr.peek();
                uint32_t ge = s_glut[gwin >> gsh];
                if (ge == 0) ge = slow_sym(gwin, L.Lg + 1, s_gtab, s_gsorted, L.gmax);
                gr.skip(ge >> 16);
                col += (int)(ge & 0xFFFFu) + 1;
                dst[ndone++] = make_float2(s_cb[sym], __uint_as_float((uint32_t)(col - bstart) * (BT * 4)));
              }
            }
          }
        }
        if (dwarp == 0 && lane == 0) {
          meta[lb * 4 + 0] = ni | (last_chunk ? (1 << 29) : 0);  // bit 29: last chunk of the unit
          meta[lb * 4 + 1] = uc.tile;
          meta[lb * 4 + 2] = uc.sp;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&lfull[lb]);
        if (last_chunk) {
          ++c;
          break;
        }
      }
      if (done) break;
    }
    return;
  }

  // ---------------------------------------------------------------- FMA warps
  const int tid = threadIdx.x;
  float acc[kRowsPerWarp][VEC];
#pragma unroll
  for (int rr = 0; rr < kRowsPerWarp; ++rr)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[rr][v] = 0.f;
  const unsigned char* xl = xs + lane * (VEC == 8 ? 16 : VEC * 4);
  uint32_t g = 0;
  for (uint32_t c = 0;; ++c) {
    const int lb = c % kLBufs;
    mbar_wait(&lfull[lb], (c / kLBufs) & 1);
    const int m0 = meta[lb * 4 + 0];
    if (m0 & (1 << 30)) break;
    const int ni = m0 & 0xFFFF;
    const bool last = (m0 >> 29) & 1;
    const int tile = meta[lb * 4 + 1], sp = meta[lb * 4 + 2];
    const float2* lst = lists + (size_t)lb * kR * kLC;
    const uint32_t* bs = bse + (size_t)lb * kR * kMaxCint;
    for (int j0 = 0; j0 < ni; j0 += ipb, ++g) {
      const int s = g % kStages;
      const int j1 = min(ni, j0 + ipb) - 1;
      mbar_wait(&full[s], (g / kStages) & 1);
      const unsigned char* xb = xl + s * kXStageBytes;
      int eb[kRowsPerWarp], ee[kRowsPerWarp];  // all 8 rows' entry ranges up front
#pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int rl = warp + kWorkWarps * rr;
        eb[rr] = (int)(bs[rl * kMaxCint + j0] & 0xFFFFu);
        ee[rr] = (int)(bs[rl * kMaxCint + j1] >> 16);
      }
#pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int rl = warp + kWorkWarps * rr;
        const int e0 = eb[rr], e1 = ee[rr];
        const float2* lr = lst + rl * kLC;
        // one broadcast LDS.64 (w, x offset) + one VEC-wide LDS of x per entry
#pragma unroll 4
        for (int e = e0; e < e1; ++e) {
          const float2 p = lr[e];
          float xv[VEC];
          load_x<VEC>(xb + __float_as_uint(p.y), xv);
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[rr][v] = fmaf(p.x, xv[v], acc[rr][v]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&lempty[lb]);
    if (!last) continue;

    // ---- unit complete: bias + ReLU (S == 1) or split partial + ordered reduction
    const int rb0 = tile / a.nbt, bt = tile % a.nbt;
    const int nb = min(BT, a.B - bt * BT);
    if (a.S == 1) {
#pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int row = rb0 * kR + warp + kWorkWarps * rr;
        if (row < L.nrows) {
          const float bias = L.bias[row];
          float* yp = a.y + (size_t)row * a.ldy + bt * BT;
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int b = bcol<VEC>(lane, v);
            float o = acc[rr][v] + bias;
            if (a.relu) o = fmaxf(o, 0.f);
            if (b < nb) yp[b] = o;
          }
        }
      }
    } else {
      float* slab = a.ws + ((size_t)tile * a.S + sp) * kR * BT;
#pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        float* p = slab + (size_t)(warp + kWorkWarps * rr) * BT;
#pragma unroll
        for (int v = 0; v < VEC; ++v) __stcg(p + bcol<VEC>(lane, v), acc[rr][v]);
      }
      __threadfence();
      named_bar_sync(kWorkBar, kWorkers);
      if (tid == 0) {
        const int old = atomicAdd(&a.tctr[tile], 1);
        const int is_last = old == a.S - 1;
        if (is_last) a.tctr[tile] = 0;
        s_last[0] = is_last;
      }
      named_bar_sync(kWorkBar, kWorkers);
      if (s_last[0]) {
        __threadfence();
        const float* base = a.ws + (size_t)tile * a.S * kR * BT;
#pragma unroll
        for (int rr = 0; rr < kRowsPerWarp; ++rr) {
          const int rl = warp + kWorkWarps * rr;
          const int row = rb0 * kR + rl;
          if (row >= L.nrows) continue;
          float sum[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) sum[v] = 0.f;
          for (int jj = 0; jj < a.S; ++jj) {
            const float* p = base + ((size_t)jj * kR + rl) * BT;
#pragma unroll
            for (int v = 0; v < VEC; ++v) sum[v] += __ldcg(p + bcol<VEC>(lane, v));
          }
          const float bias = L.bias[row];
          float* yp = a.y + (size_t)row * a.ldy + bt * BT;
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int b = bcol<VEC>(lane, v);
            float o = sum[v] + bias;
            if (a.relu) o = fmaxf(o, 0.f);
            if (b < nb) yp[b] = o;
          }
        }
      }
      named_bar_sync(kWorkBar, kWorkers);  // s_last is rewritten by the next flush
    }
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[rr][v] = 0.f;
  }
}

size_t band_smem_bytes(const FcDev& L) {
  size_t b = (size_t)kStages * kXStageBytes + sizeof(float2) * kLBufs * kR * kLC +
             sizeof(uint32_t) * kLBufs * kR * kMaxCint + sizeof(uint64_t) * 2 * (kStages + kLBufs) +
             sizeof(int) * (kLBufs * 4 + 4);
  b += (sizeof(uint32_t) << L.Lf) + (sizeof(uint32_t) << L.Lg) + sizeof(float) * L.ncb + 2 * 99 * sizeof(uint32_t) +
       sizeof(uint16_t) * (L.nvs + 1) + sizeof(uint16_t) * (L.ngs + 1);
  return (b + 127) & ~(size_t)127;
}

template <int VEC>
cudaError_t launch_band_t(const FcDev& L, const BandPlan& p, const BandArgs& a, const CUtensorMap& tmx,
                          cudaStream_t s) {
  auto kern = k_fc_band<VEC>;
  static thread_local size_t set_smem = 0;
  if (p.smem > set_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    set_smem = p.smem;
  }
  ktimer_begin("k_fc_band", s);
  kern<<<p.grid, kThreads, p.smem, s>>>(L, a, tmx);
  const cudaError_t e_ = launched();
  ktimer_end("k_fc_band", s);
  return e_;
}

}  // namespace

int band_rows_per_unit() { return kR; }
int band_list_capacity() { return kLC; }
int band_max_chunk() { return kMaxCint; }

BandPlan plan_fc_band(const FcDev& L, const float* x, int ldx, int B, int num_sms) {
  BandPlan p;
  if (B <= 0 || L.nrows <= 0 || L.Cint <= 0) return p;  // (L.ivg: uploaded at first use, api.cpp)
  const int vec = B > 64 ? 4 : (B > 32 ? 2 : 1);
  const int BT = 32 * vec;
  if ((ldx & 3) || ldx < B || ((uintptr_t)x & 15)) return p;  // TMA: 16-byte row pitch and base
  if ((size_t)L.Wi * BT * 4 > (size_t)kXStageBytes) return p;
  p.vec = vec;
  p.ipb = 1;
  while (p.ipb * 2 <= L.Cint && (size_t)L.Wi * (p.ipb * 2) * BT * 4 <= (size_t)kXStageBytes &&
         L.Wi * p.ipb * 2 <= 256)
    p.ipb *= 2;
  p.nbt = (B + BT - 1) / BT;
  p.nchunks = (L.NI + L.Cint - 1) / L.Cint;
  const int tiles = ((L.nrows + kR - 1) / kR) * p.nbt;
  // K-splits over chunks: cost ~ waves / S (unit time ~ 1/S) plus a 3% charge
  // per extra split (each writes and re-reads an R x BT partial slab); the
  // smallest S within 2% of the best wins.
  double best = 1e30;
  int bestS = 1;
  const int smax = p.nchunks < 64 ? p.nchunks : 64;
  for (int S = 1; S <= smax; ++S) {
    const long units = (long)tiles * S;
    const long waves = (units + num_sms - 1) / num_sms;
    const double cost = (double)waves / S * (1.0 + 0.03 * (S - 1));  // split partials cost HBM traffic
    if (cost < best * 0.98) { best = cost; bestS = S; }
  }
  p.S = bestS;
  p.units = tiles * p.S;
  p.tiles = tiles;
  p.grid = p.units < num_sms ? p.units : num_sms;
  p.ws_floats = p.S > 1 ? (size_t)tiles * p.S * kR * BT : 0;
  p.smem = band_smem_bytes(L);
  p.ok = true;
  return p;
}

cudaError_t launch_fc_band(const FcDev& L, const BandPlan& p, const float* x, int ldx, int B, float* y, int ldy,
                           int relu, float* ws, int* tctr, cudaStream_t s) {
  BandArgs a{x, ldx, B, y, ldy, relu, ws, tctr, p.S, p.nbt, p.units, p.nchunks, p.ipb};
  // Tensor map of x viewed as [cols][B] fp32 with row pitch ldx; box [Wi][BT].
  // Encoding is host work: cache the last few (same buffers every step).
  struct Entry { const float* x; int ldx, B, cols, bt, wi; CUtensorMap m; };
  const int box_rows = L.Wi * p.ipb;
  static thread_local Entry cache[8];
  static thread_local int ncache = 0, next = 0;
  const int BT = 32 * p.vec;
  const CUtensorMap* map = nullptr;
  for (int i = 0; i < ncache; ++i) {
    const Entry& e = cache[i];
    if (e.x == x && e.ldx == ldx && e.B == B && e.cols == L.cols && e.bt == BT && e.wi == box_rows) { map = &e.m; break; }
  }
  if (!map) {
    Entry& e = cache[next];
    next = (next + 1) % 8;
    if (ncache < 8) ++ncache;
    e = Entry{x, ldx, B, L.cols, BT, box_rows, {}};
    if (encode_tmap_2d(&e.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, (uint64_t)B, (uint64_t)L.cols,
                       (uint64_t)ldx * sizeof(float), (uint32_t)BT, (uint32_t)box_rows,
                       CU_TENSOR_MAP_SWIZZLE_NONE) != cudaSuccess) {
      e.x = nullptr;
      return cudaErrorInvalidValue;
    }
    map = &e.m;
  }
  switch (p.vec) {
    case 4: return launch_band_t<4>(L, p, a, *map, s);
    case 2: return launch_band_t<2>(L, p, a, *map, s);
    default: return launch_band_t<1>(L, p, a, *map, s);
  }
}

}  // namespace cdn
