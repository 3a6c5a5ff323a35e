// Small-batch fused FC kernel (B <= 8, sm_100a): the decode-bound regime
// where the layer is nominally bound by HBM on the compressed bytes (SURVEY
// §8(d)).  Alg. 1 lines 4-9, Eq. 1-2.
//
// Decoding is the work here, so the kernel minimises instructions per token:
//   * multi-symbol LUTs in shared memory: one lookup on the next Lv bits of the
//     val (codebook index) stream yields up to 4 complete codes, one lookup on
//     the next Lg bits of the col_ind (gap) stream up to 6; codes longer than
//     the window take the canonical slow path (rare: < 0.1% of val tokens);
//   * the two streams are decoded independently into small register queues
//     (5-bit symbols / 4-bit gaps packed in 64-bit words) and consumed four
//     tokens per step in lockstep: c += g + 1 (Alg. 1 l.7, reading C-01),
//     w = C[sym] by a lane shuffle of the register-resident codebook (l.8),
//     acc += w * x[c] (l.9).  Pads (symbol 0 <=> C[0] = 0, C-04) need no
//     branch: they advance the column like any token and their load / FMA is
//     predicated off;
//   * G lanes per row at the load-time decode-lane index restart points
//     (host.hpp LaneIndex), static row assignment (no work counter), a fixed
//     shuffle tree reduces the G partial sums (deterministic).
// Used when r <= 5 (<= 32 codebook entries) and k <= 4 (gap symbols < 16).
#include "dev_common.cuh"
#include "kernels.cuh"

namespace cdn {

namespace {

using namespace dev;

constexpr int kMsThreads = 256;

// Multi-symbol entry layouts (built in api.cpp):
//   val: n (3) | len (5) << 3 | sym_i (5 bits each) << (8 + 5 i), i < 4; n == 0: slow path
//   gap: n (3) | len (5) << 3 | g_i (4 bits each) << (8 + 4 i), i < 6;   n == 0: slow path

template <int BS, bool VEC>
__global__ void __launch_bounds__(kMsThreads, 4) k_fc_ms(FcDev L, const float* __restrict__ x, int ldx, int B,
                                                          float* __restrict__ y, int ldy, int relu) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* s_vl = sm;
  uint32_t* s_gl = s_vl + (1 << L.msLv);
  uint32_t* s_vtab = s_gl + (1 << L.msLg);
  uint32_t* s_gtab = s_vtab + 99;
  uint16_t* s_vsorted = reinterpret_cast<uint16_t*>(s_gtab + 99);
  uint16_t* s_gsorted = s_vsorted + (L.nvs + 1);
  __shared__ float s_cb[32];
  if (threadIdx.x < 32) s_cb[threadIdx.x] = threadIdx.x < L.ncb ? L.codebook[threadIdx.x] : 0.f;
  // The two LUTs (24 KB) arrive by bulk async copy (UBLKCP) at full bandwidth
  // instead of a latency-bound load/store loop; the small canonical tables by
  // plain loads meanwhile.
  __shared__ __align__(8) uint64_t s_bar;
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

  const int lane = threadIdx.x & 31;
  const int lj = lane & (L.G - 1);
  const int rows_per_warp = 32 >> L.log2G;
  const int warp_g = (blockIdx.x * kMsThreads + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * kMsThreads) >> 5;
  const int b0 = blockIdx.y * BS;
  const int nb = min(BS, B - b0);
  x += b0;
  y += b0;
  const int vsh = 32 - L.msLv, gsh = 32 - L.msLg;

  for (int unit = warp_g; unit * rows_per_warp < L.nrows; unit += nwarps) {
    const int row = unit * rows_per_warp + (lane >> L.log2G);
    const bool active = row < L.nrows;
    uint32_t vlen = 0, glen = 0, dm1 = 0;
    if (active) {
      const uint32_t r = reinterpret_cast<const uint32_t*>(L.rec)[(size_t)row * L.G + lj];
      vlen = r & 0xFFFu;
      glen = (r >> 12) & 0xFFFu;
      dm1 = r >> 24;
    }
    uint32_t vs = vlen, gs = glen;
    for (int o = 1; o < L.G; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, vs, o, L.G);
      const uint32_t b = __shfl_up_sync(0xffffffffu, gs, o, L.G);
      if (lj >= o) { vs += a; gs += b; }
    }
    // Pull the unit's stream lines into L1 while the lanes set up: the unit's
    // rows are consecutive, so their val / gap bits are two contiguous ranges.
    {
      const int r0 = unit * rows_per_warp, r1 = min(L.nrows, r0 + rows_per_warp);
      const uint32_t v0 = L.rp[2 * r0] >> 10, v1 = (L.rp[2 * r1] + 1023) >> 10;  // 128-byte lines
      const uint32_t g0 = L.rp[2 * r0 + 1] >> 10, g1 = (L.rp[2 * r1 + 1] + 1023) >> 10;
      for (uint32_t l = v0 + lane; l < v1; l += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(L.vw + (size_t)l * 32));
      for (uint32_t l = g0 + lane; l < g1; l += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(L.gw + (size_t)l * 32));
    }
    int ntok = 0;
    SReader vr, gr;
    int col = lj * L.W - (int)(dm1 + 1);
    if (active && vlen) {
      const size_t q = (size_t)row * L.G + lj;
      ntok = (int)(L.tok_start[q + 1] - L.tok_start[q]);
      vr.init(L.vw, L.rp[2 * row] + vs - vlen);
      gr.init(L.gw, L.rp[2 * row + 1] + gs - glen);
    } else {
      // idle lane: the refill code still runs (uncommitted); keep the readers
      // in a state whose skip(0) never loads
      vr.p = L.vw;
      vr.off = vr.w0 = vr.w1 = vr.n1 = vr.n2 = vr.n3 = vr.n4 = 0;
      gr = vr;
    }
    float acc[BS];
#pragma unroll
    for (int b = 0; b < BS; ++b) acc[b] = 0.f;
    uint64_t qv = 0, qg = 0;
    int cv = 0, cg = 0;
    float pw[4] = {0.f, 0.f, 0.f, 0.f}, px[4] = {0.f, 0.f, 0.f, 0.f};  // pipelined products (BS == 1)
    const float* xcur = x + (ptrdiff_t)col * ldx;  // x row of the current column (BS == 1)
    while (__any_sync(0xffffffffu, ntok > 0)) {
      {  // refill the symbol queue (up to 4 codes per lookup); always look up, commit if room
        const uint32_t w = vr.peek();
        const uint32_t e = s_vl[w >> vsh];
        uint32_t n = e & 7u, len = (e >> 3) & 31u, syms = e >> 8;
        if (n == 0) {
          const uint32_t r = slow_sym(w, L.msLv + 1, s_vtab, s_vsorted, L.vmax);
          n = 1;
          len = r >> 16;
          syms = r & 31u;
        }
        const bool room = cv <= 8 && ntok > 0;
        qv |= (uint64_t)(room ? syms : 0u) << (5 * cv);
        cv += room ? (int)n : 0;
        vr.skip(room ? len : 0u);
      }
      {  // refill the gap queue (up to 6 codes per lookup)
        const uint32_t w = gr.peek();
        const uint32_t e = s_gl[w >> gsh];
        uint32_t n = e & 7u, len = (e >> 3) & 31u, gaps = e >> 8;
        if (n == 0) {
          const uint32_t r = slow_sym(w, L.msLg + 1, s_gtab, s_gsorted, L.gmax);
          n = 1;
          len = r >> 16;
          gaps = r & 15u;
        }
        const bool room = cg <= 10 && ntok > 0;
        qg |= (uint64_t)(room ? gaps : 0u) << (4 * cg);
        cg += room ? (int)n : 0;
        gr.skip(room ? len : 0u);
      }
      const int p = ntok > 0 ? min(min(cv, cg), min(ntok, 4)) : 0;
      if constexpr (BS == 1) {
        // one step of software pipelining: the products of the previous step
        // (whose x loads have had a whole decode step to arrive) first
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[0] = fmaf(pw[j], px[j], acc[0]);
        const uint32_t qv32 = (uint32_t)qv, qg32 = (uint32_t)qg;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t sym = (qv32 >> (5 * j)) & 31u;
          const bool take = j < p;
          xcur += take ? (int)(((qg32 >> (4 * j)) & 15u) + 1) * ldx : 0;
          const bool use = take && sym != 0;
          float wv = 0.f, xv = 0.f;
          if (use) {  // predicated: xcur may sit one column before the row's first
            wv = s_cb[sym];
            xv = __ldg(xcur);
          }
          pw[j] = wv;
          px[j] = xv;
        }
      } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t sym = (uint32_t)(qv >> (5 * j)) & 31u;
        const float wv = s_cb[sym];
        if (j < p) {
          col += (int)((qg >> (4 * j)) & 15u) + 1;
          if (sym) {
            const float* xp = x + (size_t)col * ldx;
            if (VEC && BS >= 4) {
#pragma unroll
              for (int b = 0; b < BS; b += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(xp + b));
                acc[b] = fmaf(wv, v.x, acc[b]);
                acc[b + 1] = fmaf(wv, v.y, acc[b + 1]);
                acc[b + 2] = fmaf(wv, v.z, acc[b + 2]);
                acc[b + 3] = fmaf(wv, v.w, acc[b + 3]);
              }
            } else {
#pragma unroll
              for (int b = 0; b < BS; ++b)
                if (b < nb) acc[b] = fmaf(wv, __ldg(xp + b), acc[b]);
            }
          }
        }
      }
      }
      qv >>= 5 * p;
      qg >>= 4 * p;
      cv -= p;
      cg -= p;
      ntok -= p;
    }
    if constexpr (BS == 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[0] = fmaf(pw[j], px[j], acc[0]);
    }
#pragma unroll
    for (int b = 0; b < BS; ++b)
      for (int o = L.G >> 1; o > 0; o >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o, L.G);
    if (active && lj == 0) {
      const float v = L.bias[row];
#pragma unroll
      for (int b = 0; b < BS; ++b) {
        if (b < nb) {
          float o = acc[b] + v;
          if (relu) o = fmaxf(o, 0.f);
          y[(size_t)row * ldy + b] = o;
        }
      }
    }
  }
}


template <int BS, bool VEC>
cudaError_t launch_ms_t(const FcDev& L, const float* x, int ldx, int B, float* y, int ldy, int relu, cudaStream_t s,
                        int num_sms) {
  auto kern = k_fc_ms<BS, VEC>;
  const size_t smem = ms_smem_bytes(L);
  static thread_local size_t set_smem = 0;
  if (smem > 48 * 1024 && smem > set_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  const int rows_per_warp = 32 / L.G;
  const int units = (L.nrows + rows_per_warp - 1) / rows_per_warp;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMsThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int need = (units + kMsThreads / 32 - 1) / (kMsThreads / 32);
  const int cap = per_sm * num_sms;
  dim3 grid(need < cap ? need : cap, (B + BS - 1) / BS);
  ktimer_begin("k_fc_ms", s);
  kern<<<grid, kMsThreads, smem, s>>>(L, x, ldx, B, y, ldy, relu);
  const cudaError_t e_ = launched();
  ktimer_end("k_fc_ms", s);
  return e_;
}

template <int BS>
cudaError_t launch_ms_bs(const FcDev& L, const float* x, int ldx, int B, float* y, int ldy, int relu, cudaStream_t s,
                         int num_sms) {
  const bool vec = (BS % 4 == 0) && (ldx % 4 == 0) && (((uintptr_t)x & 15) == 0) && (B % BS == 0);
  if (vec) return launch_ms_t<BS, true>(L, x, ldx, B, y, ldy, relu, s, num_sms);
  return launch_ms_t<BS, false>(L, x, ldx, B, y, ldy, relu, s, num_sms);
}

}  // namespace

size_t ms_smem_bytes(const FcDev& L) {
  size_t b = (sizeof(uint32_t) << L.msLv) + (sizeof(uint32_t) << L.msLg) + 2 * 99 * sizeof(uint32_t) +
             sizeof(uint16_t) * (L.nvs + 1) + sizeof(uint16_t) * (L.ngs + 1);
  return (b + 15) & ~(size_t)15;
}

bool ms_supported(const FcDev& L) {
  return L.msv && L.msg && L.ncb <= 32 && L.k <= 4 && !L.rec64;
}

cudaError_t launch_fc_ms(const FcDev& L, const float* x, int ldx, int B, float* y, int ldy, int relu, cudaStream_t s,
                         int num_sms) {
  if (B <= 0 || L.nrows <= 0) return cudaSuccess;
  if (B <= 1) return launch_ms_bs<1>(L, x, ldx, B, y, ldy, relu, s, num_sms);
  if (B <= 2) return launch_ms_bs<2>(L, x, ldx, B, y, ldy, relu, s, num_sms);
  if (B <= 4) return launch_ms_bs<4>(L, x, ldx, B, y, ldy, relu, s, num_sms);
  return launch_ms_bs<8>(L, x, ldx, B, y, ldy, relu, s, num_sms);
}

}  // namespace cdn
