// Small-batch fused FC kernel on the merged token stream (sm_100a): the
// decode-bound regime, nominally HBM-bound on the compressed bytes (SURVEY
// §8(d)).  PAPER.md Alg. 1 lines 4-9, Eq. 1-2.
//
// One table lookup per real token:
//   * the row's val (codebook index) and col_ind (gap) Huffman codes are
//     resident interleaved token by token (host.hpp JointIndex, reading C-35),
//     so a lane runs ONE MSB-first reader: a two-word register window refilled
//     from the row's bits, which a bulk async copy (UBLKCP) staged in shared
//     memory;
//   * one lookup of the next jL bits in the joint LUT (shared memory) decodes
//     the leading padding tokens (val symbol 0, C-04) together with the real
//     token that follows: 4 x its codebook index, the bits consumed and the
//     column advance sum(g + 1) (Alg. 1 l.7, reading C-01) as a byte offset
//     into x; a window whose first token is longer than jL bits yields 0, a
//     no-op step that leaves the inner loop for a code-by-code slow path
//     (plain LUTs + canonical tables);
//   * w = C[sym] from the 32-entry codebook in shared memory (conflict-free:
//     equal indices broadcast, distinct ones sit in distinct banks; l.8) and
//     acc += w * x[c] with x staged in shared memory (l.9).
// Lanes: thread = (row, lane j) of the lane split recorded at load (start bit,
// previous column; lanes split at the kernel's lookup steps, so every lane runs
// the same number of lookups +-1).  A lane ends at its last column (record
// j + 1).  The G lanes of a row are reduced by a fixed shuffle tree, and rows
// of G > 32 lanes (short layers: VGG fc8) over several warps in warp order
// (deterministic).
// A programmatic dependent launch: the table / stream copies are issued at
// entry, x (the previous layer's output) right after griddepcontrol.wait,
// before the lane records are consumed.
// Measured bound (ncu, C5 fc6 at B = 1, profiles/r02_k_fc_j_*): during the
// decode the shared-memory data path runs at ~90% of its one wavefront per
// clock -- per lookup ~3.5 wavefronts of joint-LUT gather, ~3.3 of x gather
// (random columns), ~2 of stream refills, 1 of codebook -- with instruction
// issue at ~70%; the staging of tables + x (~165 KB per SM from L2) takes
// ~2.3 us of the ~11.5 us launch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dev_common.cuh"
#include "kernels.cuh"

namespace cdn {

namespace {

using namespace dev;

constexpr int kJMaxWarps = 32;
constexpr int kJMaxCta = 148;  // CTAs whose rows are staged as one stream range (one per SM)
constexpr int kJPieces = 4;    // a CTA's stream bits arrive in this many pieces (warps start on their own)

struct JArgs {
  const float* x;
  int ldx;
  float* y;
  int ldy;
  int relu;
  int B;
  int Q, GQ, RPW, nw, units;
  const uint32_t* lanes;  // lane records (nrows * G) of the split this launch runs
  int G, Kq;              // lanes per row, column-group width
  float* part;            // Q > 1: partial sums [Q][nrows][Bp]
  int* ctr;               // Q > 1 and !sep: per-warp-unit arrival counters
  int Bp, sep;            // padded batch (image groups x BS); sep: partials only (k_j_reduce adds them)
  const uint16_t* perm;   // GQ == 1: per column group, the row of each warp-unit slot (null: identity)
  const uint32_t* blob;   // the tables, one bulk copy (FcDev jlut / jmlut) and their offsets
  uint32_t blob_bytes;
  int jL;                 // joint LUT width of this blob
  uint32_t o_vlut, o_glut, o_vtab, o_gtab, o_vs, o_gs, o_cb;
  int lanecopy;           // GQ == 1: each lane stages its own stream piece (no bulk copies)
  int upc;                // k_fc_jm: warp units per CTA (taken dynamically by its warps)
  uint32_t sub;       // bytes of one row's staging sub-slot (16-aligned)
  uint32_t off_x, off_slot;  // dynamic smem offsets (the table blob sits at 0)
  int xbulk;          // 1: x contiguous (ldx == 1, B == 1) and 16-byte aligned
  unsigned long long* trace;  // debug (env CDN_J_TRACE): per CTA 8 globaltimer stamps, else null
  int ncta;           // Q == 1: CTAs whose stream ranges are in cta_a / cta_n (the rest stage per warp)
  int wpr;            // warps per row (k_fc_j, G > 32: a row's lanes span wpr warps of one CTA; else 1)
  uint32_t lhash;     // k_fc_j: joint LUT entry of index i at i ^ ((i >> 5) & lhash) (spreads the banks)
  // Q == 1, per CTA and piece: 16-byte index of the piece's first bits and bytes to stage; piece p =
  // the CTA's warps [pw(p), pw(p + 1)), pw(p) = (p nw / P) rounded down to whole rows (j_piece_warp)
  uint32_t cta_a[kJMaxCta * kJPieces];
  uint16_t cta_n[kJMaxCta * kJPieces];
};
static_assert(sizeof(JArgs) <= 4000, "k_fc_j parameters must stay under 4 KB");

__host__ __device__ __forceinline__ int j_piece_warp(int p, int nw, int wpr) { return (p * nw / kJPieces) / wpr * wpr; }

__device__ __forceinline__ void jtrace(const JArgs& A, int ev) {
  if (A.trace != nullptr && (threadIdx.x & 31) == 0 && threadIdx.x < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + ev] = t;
  }
}

// shared-window address of a shared-memory object, computed once (volatile:
// the compiler would otherwise rematerialise it inside the hot loop)
static __device__ __forceinline__ uint32_t saddr(const void* p) {
  uint32_t a;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
  return a;
}
static __device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
static __device__ __forceinline__ float ldsf(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
// if (off >= 32) { off -= 32; w0 = w1; w1 = word at sp; sp += 4; } -- the load
// lands straight in w1 (no temporary the compiler would wait on)
static __device__ __forceinline__ void refill(uint32_t& w0, uint32_t& w1, uint32_t& off, uint32_t& sp) {
  asm volatile(
      "{ .reg .pred p; setp.ge.u32 p, %2, 32; @p mov.b32 %0, %1; @p ld.shared.u32 %1, [%3]; "
      "@p add.u32 %3, %3, 4; @p sub.u32 %2, %2, 32; }"
      : "+r"(w0), "+r"(w1), "+r"(off), "+r"(sp));
}

template <int BS>
__host__ __device__ constexpr int log2_bs() { return BS == 1 ? 0 : BS == 2 ? 1 : BS == 4 ? 2 : BS == 8 ? 3 : BS == 16 ? 4 : 5; }
// BS >= 8: a column's BS values are BS / 4 16-byte chunks, row c at c * 4 BS
// bytes.  Lane l reads its column's chunks in the rotated order (j + l) mod
// (BS / 4), so the eight lanes of a quarter warp hit distinct 16-byte bank
// groups whatever their columns (BS = 32: conflict-free, 4 wavefronts per
// 128-bit load); its accumulators hold the images in the same rotated order.
template <int BS>
__device__ __forceinline__ void gather_fma(float (&acc)[BS], float w, uint32_t xa, uint32_t rot16) {
  if constexpr (BS >= 8) {
#pragma unroll
    for (int j = 0; j < BS / 4; ++j) {
      float a, b, cc, d;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(a), "=f"(b), "=f"(cc), "=f"(d)
                   : "r"(xa + ((((uint32_t)j << 4) + rot16) & (uint32_t)(BS * 4 - 1))));
      acc[4 * j] = fmaf(w, a, acc[4 * j]);
      acc[4 * j + 1] = fmaf(w, b, acc[4 * j + 1]);
      acc[4 * j + 2] = fmaf(w, cc, acc[4 * j + 2]);
      acc[4 * j + 3] = fmaf(w, d, acc[4 * j + 3]);
    }
  } else if constexpr (BS == 1) {
    acc[0] = fmaf(w, ldsf(xa), acc[0]);
  } else if constexpr (BS == 2) {
    float a, b;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(xa));
    acc[0] = fmaf(w, a, acc[0]);
    acc[1] = fmaf(w, b, acc[1]);
  } else {
    float a, b, c, d;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(xa));
    acc[0] = fmaf(w, a, acc[0]);
    acc[1] = fmaf(w, b, acc[1]);
    acc[2] = fmaf(w, c, acc[2]);
    acc[3] = fmaf(w, d, acc[3]);
  }
}

// One lane's decode (Alg. 1 l.4-9 over the lane's tokens): the merged-stream
// reader over bits [lb, le) staged at shared address sp (the 32-bit word
// holding bit lb), x gathered at xa (shared address of the lane's previous
// column), acc = sum of w * x over the lane's real tokens.  sb: the tables'
// shared base (A's blob layout).
template <int BS>
__device__ __forceinline__ void j_lane(const FcDev& L, const JArgs& A, uint32_t sb, uint32_t sp, uint32_t lb,
                                       uint32_t le, uint32_t xa, uint32_t rot16, float (&acc)[BS]) {
  constexpr int LBS = log2_bs<BS>();
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t* s_vtab = reinterpret_cast<const uint32_t*>(smem + A.o_vtab);
  const uint32_t* s_gtab = reinterpret_cast<const uint32_t*>(smem + A.o_gtab);
  const uint16_t* s_vs = reinterpret_cast<const uint16_t*>(smem + A.o_vs);
  const uint16_t* s_gs = reinterpret_cast<const uint16_t*>(smem + A.o_gs);
  const uint32_t lut = sb;
  const uint32_t cbase = sb + A.o_cb;
  const int jsh = 32 - A.jL;
  const int vsh = 32 - L.Lv, gsh = 32 - L.Lg;
#pragma unroll
  for (int b = 0; b < BS; ++b) acc[b] = 0.f;
  int nrem = (int)lb - (int)le;  // -(bits left in the lane)
  uint32_t off = lb & 31;
  uint32_t w0 = 0, w1 = 0;
  if (nrem < 0) {  // (lanes with bits only: the others never load)
    w0 = lds32(sp);
    w1 = lds32(sp + 4);
  }
  sp += 8;
  while (nrem < 0) {  // one lookup per (padding run +) real token
    const uint32_t win = __funnelshift_l(w1, w0, off);
    uint32_t e = lds32(lut + ((win >> jsh) << 2));
    if (e == 0) {
      // slow path, taken by this lane alone (the others wait a few dozen
      // instructions, not until their lanes end): one token whose codes did
      // not fit the window, code by code through the plain LUTs (canonical
      // tables for codes longer than those)
      const uint32_t ev = lds32(sb + A.o_vlut + ((win >> vsh) << 2));
      uint32_t vl, vsym;
      if (ev) { vl = ev >> 16; vsym = ev & 0xffffu; }
      else { const uint32_t r = slow_sym(win, L.Lv + 1, s_vtab, s_vs, L.vmax); vl = r >> 16; vsym = r & 0xffffu; }
      off += vl;
      nrem += (int)vl;
      refill(w0, w1, off, sp);
      const uint32_t win2 = __funnelshift_l(w1, w0, off);
      const uint32_t eg = lds32(sb + A.o_glut + ((win2 >> gsh) << 2));
      uint32_t gl, gsym;
      if (eg) { gl = eg >> 16; gsym = eg & 0xffffu; }
      else { const uint32_t r = slow_sym(win2, L.Lg + 1, s_gtab, s_gs, L.gmax); gl = r >> 16; gsym = r & 0xffffu; }
      off += gl;
      nrem += (int)gl;
      refill(w0, w1, off, sp);
      // an entry as the LUT would have built it, both codes already consumed
      e = (vsym * 4u) | (((gsym + 1) * 4u) << 10);
    }
    off += e >> 27;
    nrem += (int)(e >> 27);
    refill(w0, w1, off, sp);
    const uint32_t ca = e & 0x3fcu;
    const float w = ldsf(cbase + ca);
    xa += ((e & 0x07fffc00u) >> 10) << LBS;
    if (ca) gather_fma<BS>(acc, w, xa, rot16);
  }
}

// threads per CTA: BS accumulators per thread beside the decoder state
template <int BS>
__host__ __device__ constexpr int j_max_warps() { return BS >= 32 ? 16 : BS >= 16 ? 24 : kJMaxWarps; }

// if (R & 32) { w0 = w1; w1 = word at sp; sp += 4; R -= 32; } -- the refill
// of the small-batch kernel's lane, whose bit offset is R's low 5 bits
static __device__ __forceinline__ void refill_r(uint32_t& w0, uint32_t& w1, uint32_t& R, uint32_t& sp) {
  asm volatile(
      "{ .reg .pred p; .reg .b32 t; and.b32 t, %2, 32; setp.ne.u32 p, t, 0; @p mov.b32 %0, %1; "
      "@p ld.shared.u32 %1, [%3]; @p add.u32 %3, %3, 4; @p sub.u32 %2, %2, 32; }"
      : "+r"(w0), "+r"(w1), "+r"(R), "+r"(sp));
}

// One lane of the small-batch kernel (Alg. 1 l.4-9 over the lane's tokens) on
// the entry layout of build_joint_lut_r: one register R = (x offset << 6) |
// refill flag (bit 5) | bit offset (bits 0-4) -- an entry's (e >> 10) adds the
// bits consumed to the offset and the column advance (x 4 bytes) to the x
// offset in a single add, the funnel shift reads the offset from R's low bits,
// and the lane ends when the x offset reaches its last column (lanes cover
// whole steps; the column only grows).  BS == 1: R's x offset is the x
// address itself.  sp: shared address of the word holding bit lb; xa0: shared
// address of x at the lane's previous column; span = last - previous column.
template <int BS>
__device__ __forceinline__ void j_lane_r(const FcDev& L, const JArgs& A, uint32_t sb, uint32_t sp, uint32_t lb,
                                         uint32_t xa0, uint32_t span, float (&acc)[BS]) {
  constexpr int LBS = log2_bs<BS>();
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t* s_vtab = reinterpret_cast<const uint32_t*>(smem + A.o_vtab);
  const uint32_t* s_gtab = reinterpret_cast<const uint32_t*>(smem + A.o_gtab);
  const uint16_t* s_vs = reinterpret_cast<const uint16_t*>(smem + A.o_vs);
  const uint16_t* s_gs = reinterpret_cast<const uint16_t*>(smem + A.o_gs);
  const uint32_t lut = sb;
  const uint32_t cbase = sb + A.o_cb;
  const int jsh = 32 - A.jL;
  const int vsh = 32 - L.Lv, gsh = 32 - L.Lg;
#pragma unroll
  for (int b = 0; b < BS; ++b) acc[b] = 0.f;
  const uint32_t x0 = BS == 1 ? xa0 : 0u;
  uint32_t R = (x0 << 6) | (lb & 31);
  const uint32_t Rend = (x0 + span * 4u) << 6;
  uint32_t w0 = 0, w1 = 0;
  if (R < Rend) {  // (lanes with tokens only: the others never load)
    w0 = lds32(sp);
    w1 = lds32(sp + 4);
  }
  sp += 8;
  while (R < Rend) {  // one lookup per (padding run +) real token
    const uint32_t win = __funnelshift_l(w1, w0, R);
    const uint32_t li = win >> jsh;
    uint32_t e = lds32(lut + ((li ^ ((li >> 5) & A.lhash)) << 2));  // (bank bits hashed, j_lut_pos)
    if (e == 0) {
      // slow path, this lane alone: one token whose codes did not fit the
      // window, code by code (plain LUTs, canonical tables for longer codes)
      const uint32_t ev = lds32(sb + A.o_vlut + ((win >> vsh) << 2));
      uint32_t vl, vsym;
      if (ev) { vl = ev >> 16; vsym = ev & 0xffffu; }
      else { const uint32_t r = slow_sym(win, L.Lv + 1, s_vtab, s_vs, L.vmax); vl = r >> 16; vsym = r & 0xffffu; }
      R += vl;
      refill_r(w0, w1, R, sp);
      const uint32_t win2 = __funnelshift_l(w1, w0, R);
      const uint32_t eg = lds32(sb + A.o_glut + ((win2 >> gsh) << 2));
      uint32_t gl, gsym;
      if (eg) { gl = eg >> 16; gsym = eg & 0xffffu; }
      else { const uint32_t r = slow_sym(win2, L.Lg + 1, s_gtab, s_gs, L.gmax); gl = r >> 16; gsym = r & 0xffffu; }
      R += gl;
      refill_r(w0, w1, R, sp);
      // an entry as the LUT would have built it, both codes already consumed
      e = (vsym * 4u) | (((gsym + 1) * 4u) << 16);
    }
    R += e >> 10;  // bits consumed (offset) and column advance (x offset), one add
    const uint32_t ca = e & 0x3fcu;
    const float w = ldsf(cbase + ca);
    const uint32_t xa = BS == 1 ? (R >> 6) : xa0 + ((R >> 6) << LBS);
    if (ca) gather_fma<BS>(acc, w, xa, 0u);
    refill_r(w0, w1, R, sp);
  }
}

template <int BS>
__global__ void __launch_bounds__(j_max_warps<BS>() * 32, 1) k_fc_j(FcDev L, const __grid_constant__ JArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_w, bar_x;
  __shared__ __align__(8) uint64_t bar_s[kJMaxWarps];
  __shared__ float s_red[kJMaxWarps][BS];  // rows spanning several warps: each warp's sum
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  jtrace(A, 0);
  asm volatile("griddepcontrol.launch_dependents;");

  const int G = A.G, GQ = A.GQ, q = blockIdx.y, WPR = A.wpr;
  const int xc0 = q * A.Kq, xcols = max(0, min(A.Kq, L.cols - xc0));  // this column group's slice of x
  const int u = blockIdx.x * A.nw + warp;  // warp unit: RPW rows, or 1 / WPR of a row
  int row, j, jj;                          // row, lane of the row (of G), lane of the row in this group (of GQ)
  if (WPR > 1) {
    row = u / WPR;
    jj = (u - row * WPR) * 32 + lane;
    j = jj;
  } else {
    const int rr = lane / GQ;
    jj = lane - rr * GQ;
    row = u * A.RPW + rr;
    j = q * GQ + jj;
  }
  const bool ok = u < A.units && row < L.nrows;
  // lane records (G + 1 per row: lane j's end is record j + 1) and the row's
  // first bit: the loads fly while the copies are issued and x is requested
  const bool whole = A.Q == 1 && (int)blockIdx.x < A.ncta;  // the CTA's rows in kJPieces copies
  // the copies first, from several threads at once (each initialises the
  // barrier it arms): the tables from thread 0, the CTA's stream pieces from
  // threads 32 .. 32 + kJPieces - 1 (C2 fc6 at B = 1: 8.96 -> 8.71 us against
  // one thread issuing every copy after initialising every barrier)
  if (tid == 0) {
    mbar_init(&bar_w, 1);
    mbar_init(&bar_x, 1);
    mbar_fence_init();
    // every table in one bulk copy (host-built blob in this layout)
    mbar_arrive_expect_tx(&bar_w, A.blob_bytes);
    bulk_g2s(smem, A.blob, A.blob_bytes, &bar_w);
    jtrace(A, 7);
    if (!whole) {
      for (int w = 0; w < A.nw; ++w) mbar_init(&bar_s[w], 1);
      mbar_fence_init();
    }
  }
  if (whole && tid >= 32 && tid < 32 + kJPieces) {
    const int pc = tid - 32;
    const uint32_t base = A.cta_a[blockIdx.x * kJPieces];
    const uint32_t a = A.cta_a[blockIdx.x * kJPieces + pc], n = A.cta_n[blockIdx.x * kJPieces + pc];
    mbar_init(&bar_s[pc], 1);
    mbar_fence_init();
    mbar_arrive_expect_tx(&bar_s[pc], n);
    if (n)
      bulk_g2s(smem + A.off_slot + (a - base) * 16u, reinterpret_cast<const uint8_t*>(L.jw) + (size_t)a * 16u, n,
               &bar_s[pc]);
  }
  uint32_t r0 = 0, rec = 0, nxt = 0;
  if (ok) {
    r0 = L.jrow[row];
    rec = A.lanes[(size_t)row * (G + 1) + j];
    nxt = A.lanes[(size_t)row * (G + 1) + j + 1];
  }
  jtrace(A, 1);

  // ---- activations (after the producer of x finished), requested before the
  // lane records are needed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  jtrace(A, 2);
  float* xs = reinterpret_cast<float*>(smem + A.off_x);
  const int K = xcols;
  constexpr int LBS = log2_bs<BS>();
  if (A.xbulk) {  // x contiguous: ldx == BS == B (the slice is one range)
    const int nb = (K * 4 * BS) & ~15;
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar_x, (uint32_t)nb);
      if (nb) bulk_g2s(xs, A.x + (size_t)xc0 * BS, (uint32_t)nb, &bar_x);
    }
    for (int i = nb / 4 + tid; i < K * BS; i += blockDim.x) xs[i] = A.x[(size_t)xc0 * BS + i];
  } else {
    if (tid == 0) mbar_arrive(&bar_x);
    // eight loads in flight per thread before their stores (small CTAs would
    // otherwise pay one memory latency per element)
    const int n = K * BS, step = blockDim.x;
    for (int i0 = tid; i0 < n; i0 += 8 * step) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * step, c = i >> LBS, b = i & (BS - 1);
        v[k] = (i < n && b < A.B) ? A.x[(size_t)(xc0 + c) * A.ldx + b] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k * step < n) xs[i0 + k * step] = v[k];
    }
  }

  const uint32_t lb = ok ? r0 + (rec & 0xffffu) : 0u;  // lane's bits from lb
  const int prev = (int)(rec >> 16) - 1;                // lane's previous column
  const int last = ok ? (int)(nxt >> 16) - 1 : prev;    // its last token's column
  uint32_t rs, slot_off;  // staged bits start (128-bit aligned) and its shared-memory offset
  if (whole) {
    rs = A.cta_a[blockIdx.x * kJPieces] * 128u;
    slot_off = A.off_slot;
  } else {
    // per warp (WPR == 1): each row's range of this column group [first lane's start, last lane's end)
    const uint32_t le = ok ? r0 + (nxt & 0xffffu) : 0u;
    const uint32_t g0 = __shfl_sync(0xffffffffu, lb, (lane / GQ) * GQ);
    const uint32_t g1 = __shfl_sync(0xffffffffu, le, (lane / GQ) * GQ + GQ - 1);
    rs = (g0 >> 7) << 7;
    slot_off = A.off_slot + ((uint32_t)warp * A.RPW + (uint32_t)(lane / GQ)) * A.sub;
    const uint32_t bytes = ok ? (((g1 + 127) >> 7) - (g0 >> 7)) * 16u + 16u : 0u;
    uint32_t tot = jj == 0 ? bytes : 0u;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    __syncthreads();  // the barriers are initialised
    if (lane == 0) mbar_arrive_expect_tx(&bar_s[warp], tot);
    __syncwarp();
    if (jj == 0 && bytes)
      bulk_g2s(smem + slot_off, reinterpret_cast<const uint8_t*>(L.jw) + (size_t)(g0 >> 7) * 16u, bytes,
               &bar_s[warp]);
  }
  __syncthreads();
  mbar_wait(&bar_w, 0);
  mbar_wait(&bar_x, 0);
  jtrace(A, 3);

  const uint32_t sb = saddr(smem);
  const uint32_t xbase = sb + A.off_x;
  float acc[BS];
#pragma unroll
  for (int b = 0; b < BS; ++b) acc[b] = 0.f;
  if (u < A.units) {
    // the piece holding this warp's rows: the last whose first warp is <= warp
    int pc = 0;
    if (whole) {
      for (int k = 1; k < kJPieces; ++k)
        if (j_piece_warp(k, A.nw, WPR) <= warp) pc = k;
    }
    mbar_wait(&bar_s[whole ? pc : warp], 0);
    jtrace(A, 4);
    if (ok)
      j_lane_r<BS>(L, A, sb, sb + slot_off + ((lb - rs) >> 5) * 4u, lb,
                   xbase + (uint32_t)((prev - xc0) * 4 * BS), (uint32_t)(last - prev), acc);
    // lanes of a row: fixed shuffle tree (deterministic)
    const int width = WPR > 1 ? 32 : GQ;
#pragma unroll
    for (int b = 0; b < BS; ++b)
      for (int o = width >> 1; o > 0; o >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o, width);
  }
  if (WPR > 1) {
    // a row's warps: their sums in warp order (deterministic)
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < BS; ++b) s_red[warp][b] = acc[b];
    }
    __syncthreads();
    if (lane == 0 && ok && (u % WPR) == 0) {
      const float v = L.bias[row];
#pragma unroll
      for (int b = 0; b < BS; ++b) {
        float t = 0.f;
        for (int k = 0; k < WPR; ++k) t += s_red[warp + k][b];
        if (b < A.B) {
          float o = t + v;
          if (A.relu) o = fmaxf(o, 0.f);
          A.y[(size_t)row * A.ldy + b] = o;
        }
      }
    }
  } else if (u < A.units) {
    if (A.Q == 1) {
      if (jj == 0 && row < L.nrows) {
        const float v = L.bias[row];
#pragma unroll
        for (int b = 0; b < BS; ++b) {
          if (b < A.B) {
            float o = acc[b] + v;
            if (A.relu) o = fmaxf(o, 0.f);
            A.y[(size_t)row * A.ldy + b] = o;
          }
        }
      }
    } else {
      // column groups: the last of the unit's Q CTAs adds the Q partial sums in
      // group order (deterministic) and applies bias / ReLU
      if (jj == 0 && row < L.nrows) {
#pragma unroll
        for (int b = 0; b < BS; ++b) __stcg(&A.part[((size_t)q * L.nrows + row) * A.Bp + b], acc[b]);
      }
      __threadfence();
      __syncwarp();
      int lst = 0;
      if (lane == 0) lst = atomicAdd(&A.ctr[u], 1) == A.Q - 1;
      lst = __shfl_sync(0xffffffffu, lst, 0);
      if (lst) {
        __threadfence();
        if (jj == 0 && row < L.nrows) {
          const float v = L.bias[row];
#pragma unroll
          for (int b = 0; b < BS; ++b) {
            if (b < A.B) {
              float sum = 0.f;
              for (int qq = 0; qq < A.Q; ++qq) sum += __ldcg(&A.part[((size_t)qq * L.nrows + row) * A.Bp + b]);
              float o = sum + v;
              if (A.relu) o = fmaxf(o, 0.f);
              A.y[(size_t)row * A.ldy + b] = o;
            }
          }
        }
        if (lane == 0) A.ctr[u] = 0;
      }
    }
  }
  jtrace(A, 5);
  __syncthreads();
  jtrace(A, 6);
}

// Medium-batch kernel (FC, one launch per group of <= 32 images): the same
// lane decode over the medium split -- one lane per (row, column group), the
// CTA = one column group (its x slice, BS images per column) x a range of
// upc warp units (32 rows each, taken in the group's row order, longest
// first).  Its warps take the units dynamically (the first nw in order, staged
// before griddepcontrol.wait; the rest from a shared counter), so the CTA's
// warps finish together however the lanes' lengths vary; each lane stages its
// own piece of the stream in its sub-slot before decoding a unit.  Output:
// the column group's partial sums (Q > 1; k_j_reduce adds them in group
// order) or y itself (Q == 1).
template <int BS>
__global__ void __launch_bounds__(j_max_warps<BS>() * 32, 1) k_fc_jm(FcDev L, const __grid_constant__ JArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_w, bar_x;
  __shared__ int s_next;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  jtrace(A, 0);
  asm volatile("griddepcontrol.launch_dependents;");
  const int q = blockIdx.y;
  const int b0 = blockIdx.z * BS;  // image group of this CTA
  const int xc0 = q * A.Kq, K = max(0, min(A.Kq, L.cols - xc0));
  const int u0 = blockIdx.x * A.upc, u1 = min(A.units, u0 + A.upc);
  if (tid == 0) {
    mbar_init(&bar_w, 1);
    mbar_init(&bar_x, 1);
    mbar_fence_init();
    s_next = A.nw;
    mbar_arrive_expect_tx(&bar_w, A.blob_bytes);
    bulk_g2s(smem, A.blob, A.blob_bytes, &bar_w);
  }
  const uint32_t sb = saddr(smem);
  const uint32_t sub_off = A.off_slot + ((uint32_t)warp * 32u + (uint32_t)lane) * A.sub;
  const uint32_t rot = (uint32_t)lane & (uint32_t)(BS / 4 - 1);
  uint32_t lb = 0, le = 0;
  int prev = 0, row = L.nrows;
  // lane of unit u: its row (the group's order), bits [lb, le), previous
  // column; its piece (16-byte blocks + one of read-ahead) into the sub-slot
  auto setup = [&](int u) {
    const int slot = u * 32 + lane;
    lb = le = 0;
    prev = 0;
    row = L.nrows;
    if (slot < L.nrows) {
      row = A.perm ? (int)A.perm[(size_t)q * L.nrows + slot] : slot;
      const uint32_t r0 = L.jrow[row], r1 = L.jrow[row + 1];
      const uint32_t rec = A.lanes[(size_t)row * A.G + q];
      const uint32_t nxt = q + 1 < A.G ? A.lanes[(size_t)row * A.G + q + 1] : 0u;
      lb = r0 + (rec & 0xffffu);
      le = r0 + (q + 1 < A.G ? (nxt & 0xffffu) : r1 - r0);
      prev = (int)(rec >> 16) - 1;
      if (le > lb) {
        const uint32_t n16 = ((le + 127) >> 7) - (lb >> 7) + 1;
        const uint4* src = reinterpret_cast<const uint4*>(L.jw) + (lb >> 7);
        uint4* dst = reinterpret_cast<uint4*>(smem + sub_off);
        for (uint32_t i0 = 0; i0 < n16; i0 += 8) {
          uint4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (i0 + k < n16) v[k] = __ldg(src + i0 + k);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (i0 + k < n16) dst[i0 + k] = v[k];
        }
      }
    }
  };
  int u = u0 + warp;
  if (u < u1) setup(u);
  jtrace(A, 1);

  // ---- activations (after the producer of x finished)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  jtrace(A, 2);
  float* xs = reinterpret_cast<float*>(smem + A.off_x);
  if (A.xbulk) {  // x contiguous: ldx == BS == B (the slice is one range)
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar_x, (uint32_t)(K * 4 * BS));
      if (K) bulk_g2s(xs, A.x + (size_t)xc0 * BS, (uint32_t)(K * 4 * BS), &bar_x);
    }
  } else {
    // (image group b0: columns' images b0 .. b0 + BS - 1)
    if (tid == 0) mbar_arrive(&bar_x);
    // 16-byte chunks (4 images of a column), eight loads in flight per thread
    constexpr int NCH = BS / 4;
    const int n = K * NCH, step = blockDim.x;
    const bool v4 = (A.ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(A.x) & 15) == 0;
    for (int i0 = tid; i0 < n; i0 += 8 * step) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * step, c = i / NCH, b = b0 + 4 * (i - c * NCH);
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n) {
          const float* src = A.x + (size_t)(xc0 + c) * A.ldx + b;
          if (v4 && b + 3 < A.B) {
            v[k] = *reinterpret_cast<const float4*>(src);
          } else {
            if (b < A.B) v[k].x = src[0];
            if (b + 1 < A.B) v[k].y = src[1];
            if (b + 2 < A.B) v[k].z = src[2];
            if (b + 3 < A.B) v[k].w = src[3];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k * step < n) reinterpret_cast<float4*>(xs)[i0 + k * step] = v[k];
    }
  }
  __syncthreads();
  mbar_wait(&bar_w, 0);
  mbar_wait(&bar_x, 0);
  jtrace(A, 3);
  const uint32_t xbase = sb + A.off_x;
  auto img = [&](int b) { return (int)((((uint32_t)(b >> 2) + rot) & (uint32_t)(BS / 4 - 1)) << 2) + (b & 3); };
  while (u < u1) {
    float acc[BS];
    j_lane<BS>(L, A, sb, sb + sub_off + ((lb & 127u) >> 5) * 4u, lb, le, xbase + (uint32_t)((prev - xc0) * 4 * BS),
               rot << 4, acc);
    if (row < L.nrows) {
      if (A.Q == 1) {
        const float v = L.bias[row];
#pragma unroll
        for (int b = 0; b < BS; ++b) {
          const int bi = b0 + img(b);
          if (bi < A.B) {
            float o = acc[b] + v;
            if (A.relu) o = fmaxf(o, 0.f);
            A.y[(size_t)row * A.ldy + bi] = o;
          }
        }
      } else {
        float* dst = A.part + ((size_t)q * L.nrows + row) * A.Bp + b0;
#pragma unroll
        for (int b = 0; b < BS; b += 4)
          __stcg(reinterpret_cast<float4*>(dst + img(b)), make_float4(acc[b], acc[b + 1], acc[b + 2], acc[b + 3]));
      }
    }
    int nu = 0;
    if (lane == 0) nu = atomicAdd(&s_next, 1);
    u = u0 + __shfl_sync(0xffffffffu, nu, 0);
    if (u < u1) setup(u);
  }
  jtrace(A, 5);
}

// Column-group partial sums of the medium-batch split (A.sep): y = act(sum over
// the Q groups, in group order, + bias) -- Alg. 1 l.9 completed across groups.
// Thread per output (row, image), consecutive images on consecutive threads.
__global__ void __launch_bounds__(256) k_j_reduce(const float* __restrict__ part, int Q, int N, int Bp, int B,
                                                  const float* __restrict__ bias, int relu, float* __restrict__ y,
                                                  int ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const size_t n = (size_t)N * B, plane = (size_t)N * Bp;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / B), b = (int)(i - (size_t)row * B);
    const float* p = part + (size_t)row * Bp + b;
    float v[8];
    float sum = 0.f;
    int q = 0;
    for (; q + 8 <= Q; q += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + (size_t)(q + k) * plane);
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += v[k];
    }
    for (; q < Q; ++q) sum += __ldcg(p + (size_t)q * plane);
    float o = sum + bias[row];
    if (relu) o = fmaxf(o, 0.f);
    y[(size_t)row * ldy + b] = o;
  }
}

}  // namespace

bool j_supported(const FcDev& L) { return L.jw && L.jlutr && L.ncb <= 32 && L.jG <= 128 && L.jG >= 1; }

JPlan plan_fc_j(const FcDev& L, int B, int num_sms, const uint32_t* row_bit) {
  JPlan p;
  if (!j_supported(L) || B < 1 || B > 4 || L.nrows <= 0) return p;
  p.BS = B <= 1 ? 1 : (B <= 2 ? 2 : 4);
  p.Q = L.jQ;
  p.GQ = L.jG / p.Q;
  if (p.GQ > 32) {  // a row's lanes span wpr warps (one column group only)
    if (p.Q != 1 || p.GQ % 32) return p;
    p.wpr = p.GQ / 32;
    p.RPW = 1;
    p.units = L.nrows * p.wpr;
  } else {
    p.wpr = 1;
    p.RPW = 32 / p.GQ;
    p.units = (L.nrows + p.RPW - 1) / p.RPW;
  }
  // one CTA per SM (Q column groups of a row block side by side), every
  // warp one unit of RPW rows (or 1 / wpr of a row); a CTA holds whole rows
  const int rb = std::max(1, num_sms / p.Q);
  auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
  const size_t off_x = al(L.jblob);
  const size_t off_slot = al(off_x + (size_t)4 * p.BS * L.jKq);
  int nw0 = std::min(kJMaxWarps, std::max(1, (p.units + rb - 1) / rb));
  nw0 = std::min(kJMaxWarps, (nw0 + p.wpr - 1) / p.wpr * p.wpr);  // whole rows per CTA (rounded up: <= one wave)
  for (p.nw = nw0; p.nw >= p.wpr; p.nw -= p.wpr) {
    p.nrb = (p.units + p.nw - 1) / p.nw;
    p.cta.clear();
    size_t slot = (size_t)p.nw * p.RPW * L.jsub;  // per-warp row slots
    const bool whole = p.Q == 1 && row_bit && p.nrb <= kJMaxCta && p.nw >= kJPieces;
    if (whole) {
      // the CTA's rows are contiguous: one range of the merged stream, staged
      // in kJPieces copies of whole rows (pieces overlap by at most the
      // 16-byte blocks of a shared boundary, copied twice)
      size_t mx = 0;
      const int rows_cta = p.nw * p.RPW / p.wpr;
      for (int c = 0; c < p.nrb; ++c) {
        const int cr0 = c * rows_cta;
        uint32_t first = 0;
        for (int pc = 0; pc < kJPieces; ++pc) {
          const int w0 = j_piece_warp(pc, p.nw, p.wpr), w1 = pc + 1 < kJPieces ? j_piece_warp(pc + 1, p.nw, p.wpr) : p.nw;
          const int r0 = std::min(L.nrows, cr0 + w0 * p.RPW / p.wpr), r1 = std::min(L.nrows, cr0 + w1 * p.RPW / p.wpr);
          const uint32_t a = row_bit[r0] >> 7, e = (row_bit[r1] + 127) >> 7;
          const uint32_t bytes = r1 > r0 ? (e - a) * 16u + 16u : 0u;  // + 16 bytes of read-ahead
          if (pc == 0) first = a;
          p.cta.push_back(make_uint2(a, bytes));
          mx = std::max<size_t>(mx, (size_t)(a - first) * 16u + bytes);
        }
      }
      slot = mx;
    } else if (p.wpr > 1) {
      continue;  // (per-warp staging serves whole-row warp units only)
    }
    p.off_x = (uint32_t)off_x;
    p.off_slot = (uint32_t)off_slot;
    p.sub = L.jsub;
    p.smem = off_slot + slot;
    if (p.smem <= 227 * 1024 - 1024 && (!whole || std::all_of(p.cta.begin(), p.cta.end(), [](const uint2& c) {
          return c.y < 65536u;
        })))
      break;
  }
  p.ok = p.nw >= p.wpr && p.smem <= 227 * 1024 - 1024 && (p.Q == 1 || (L.jpart && L.jctr));
  return p;
}

int j_max_warps_host(int BS) { return BS >= 32 ? j_max_warps<32>() : BS >= 16 ? j_max_warps<16>() : j_max_warps<8>(); }

bool jm_supported(const FcDev& L) { return L.jw && L.jmlut && L.jmlane && L.ncb <= 32 && L.jmQ >= 1; }

JPlan plan_fc_jm(const FcDev& L, int B, int num_sms, size_t part_cap) {
  (void)num_sms;  // (the CTA geometry is the load-time split's: L.jmupc)
  JPlan p;
  if (!jm_supported(L) || B < 1 || L.nrows <= 0) return p;
  p.medium = true;
  p.BS = B <= 8 ? 8 : (B <= 16 ? 16 : 32);
  // image groups of BS on grid z, as many per launch as the partial sums
  // (Q x rows x groups x BS floats) fit in part_cap (at least one)
  const int groups = (B + p.BS - 1) / p.BS;
  const size_t per_group = sizeof(float) * (size_t)std::max(1, L.jmQ) * L.nrows * p.BS;
  p.nbg = L.jmQ > 1 ? (int)std::max<size_t>(1, std::min<size_t>(groups, part_cap / per_group)) : groups;
  p.Bp = p.nbg * p.BS;
  p.Q = L.jmQ;
  p.GQ = 1;
  p.RPW = 32;
  p.units = (L.nrows + 31) / 32;
  p.upc = std::max(1, L.jmupc);
  p.nrb = (p.units + p.upc - 1) / p.upc;
  auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
  // warps per CTA: up to the register budget of BS accumulators, no more than
  // the CTA's units; the small-batch kernel's tables (the wider joint LUT:
  // fewer lookups) when they fit beside the x slice and the staging
  // sub-slots, else the narrow-LUT blob, and fewer warps while even that
  // does not fit
  const int nw0 = std::min(j_max_warps_host(p.BS), p.upc);
  const size_t xb = (size_t)4 * p.BS * L.jmKq, sl = (size_t)nw0 * 32 * L.jmsub;
  p.jbig = L.jlut && al(al(L.jblob) + xb) + sl <= 227 * 1024 - 1024;
  const size_t off_x = al(p.jbig ? L.jblob : L.jmblob);
  const size_t off_slot = al(off_x + xb);
  int nw = nw0;
  while (nw >= 1 && off_slot + (size_t)nw * 32 * L.jmsub > 227 * 1024 - 1024) --nw;
  p.nw = nw;
  p.smem = nw >= 1 ? off_slot + (size_t)nw * 32 * L.jmsub : 0;
  p.off_x = (uint32_t)off_x;
  p.off_slot = (uint32_t)off_slot;
  p.sub = L.jmsub;
  p.ok = nw >= 1 && p.nrb < 65535 && p.Q < 65535 && p.nbg < 65535;
  return p;
}

size_t jm_part_bytes(const FcDev& L, const JPlan& p) {
  return p.medium && p.Q > 1 ? sizeof(float) * (size_t)p.Q * L.nrows * p.Bp : 0;
}

cudaError_t launch_fc_j(const FcDev& L, const JPlan& p, const float* x, int ldx, int B, float* y, int ldy, int relu,
                        cudaStream_t s, float* part) {
  if (!p.ok) return cudaErrorInvalidValue;
  if (p.medium && p.Q > 1 && !part) return cudaErrorInvalidValue;
  JArgs a{};
  a.x = x;
  a.ldx = ldx;
  a.y = y;
  a.ldy = ldy;
  a.relu = relu;
  a.B = B;
  a.Q = p.Q;
  a.GQ = p.GQ;
  a.RPW = p.RPW;
  a.nw = p.nw;
  a.units = p.units;
  if (p.medium) {
    a.lanes = L.jmlane;
    a.G = L.jmQ;
    a.Kq = L.jmKq;
    a.part = part;
    a.ctr = nullptr;
    a.Bp = p.Bp;
    a.sep = 1;
    a.perm = L.jmperm;
    a.lanecopy = 1;
    a.upc = p.upc;
    if (p.jbig) {
      a.blob = L.jlut;
      a.blob_bytes = L.jblob;
      a.jL = L.jL;
      a.o_vlut = L.jo_vlut; a.o_glut = L.jo_glut; a.o_vtab = L.jo_vtab; a.o_gtab = L.jo_gtab;
      a.o_vs = L.jo_vs; a.o_gs = L.jo_gs; a.o_cb = L.jo_cb;
    } else {
      a.blob = L.jmlut;
      a.blob_bytes = L.jmblob;
      a.jL = L.jmL;
      a.o_vlut = L.jmo_vlut; a.o_glut = L.jmo_glut; a.o_vtab = L.jmo_vtab; a.o_gtab = L.jmo_gtab;
      a.o_vs = L.jmo_vs; a.o_gs = L.jmo_gs; a.o_cb = L.jmo_cb;
    }
  } else {
    a.lanes = L.jlane;
    a.G = L.jG;
    a.Kq = L.jKq;
    a.part = L.jpart;
    a.ctr = L.jctr;
    a.Bp = p.BS;
    a.sep = 0;
    a.perm = nullptr;
    a.lanecopy = 0;
    a.blob = L.jlutr;
    a.blob_bytes = L.jblob;
    a.jL = L.jL;
    a.o_vlut = L.jo_vlut; a.o_glut = L.jo_glut; a.o_vtab = L.jo_vtab; a.o_gtab = L.jo_gtab;
    a.o_vs = L.jo_vs; a.o_gs = L.jo_gs; a.o_cb = L.jo_cb;
  }
  a.sub = p.sub;
  a.off_x = p.off_x;
  a.off_slot = p.off_slot;
  a.ncta = (int)std::min<size_t>(p.cta.size() / kJPieces, kJMaxCta);
  for (int i = 0; i < a.ncta * kJPieces; ++i) {
    a.cta_a[i] = p.cta[i].x;
    a.cta_n[i] = (uint16_t)p.cta[i].y;
  }
  a.wpr = p.wpr;
  a.lhash = p.medium ? 0u : L.jlhash;
  static unsigned long long* trace = nullptr;
  static const char* trace_path = getenv("CDN_J_TRACE");
  const size_t ntr = (size_t)p.nrb * p.Q * p.nbg * 8;
  static size_t trace_n = 0;
  if (trace_path && trace_n < ntr) {
    if (trace) cudaFree(trace);
    if (cudaMalloc(&trace, ntr * sizeof(unsigned long long)) != cudaSuccess) return cudaErrorMemoryAllocation;
    trace_n = ntr;
  }
  if (trace_path) cudaMemsetAsync(trace, 0, ntr * sizeof(unsigned long long), s);
  a.trace = trace_path ? trace : nullptr;
  a.xbulk = (ldx == p.BS && B == p.BS && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && a.Kq % 4 == 0) ? 1 : 0;
  cudaError_t e = cudaSuccess;
  static thread_local size_t set_smem[6] = {0, 0, 0, 0, 0, 0};
  auto run = [&](auto kern, int bi) {
    if (p.smem > 48 * 1024 && p.smem > set_smem[bi]) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      if (e != cudaSuccess) return;
      set_smem[bi] = p.smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.nrb, (unsigned)p.Q, (unsigned)p.nbg);
    cfg.blockDim = dim3((unsigned)(p.nw * 32));
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // LUT / stream staging overlaps the producer of x
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, L, a);
  };
  if (!p.medium) {
    ktimer_begin("k_fc_j", s);
    if (p.BS == 1) run(k_fc_j<1>, 0);
    else if (p.BS == 2) run(k_fc_j<2>, 1);
    else run(k_fc_j<4>, 2);
    if (e == cudaSuccess) e = launched();
    ktimer_end("k_fc_j", s);
  } else {
    ktimer_begin("k_fc_jm", s);
    if (p.BS == 8) run(k_fc_jm<8>, 3);
    else if (p.BS == 16) run(k_fc_jm<16>, 4);
    else run(k_fc_jm<32>, 5);
    if (e == cudaSuccess) e = launched();
    ktimer_end("k_fc_jm", s);
  }
  if (e == cudaSuccess && p.medium && p.Q > 1) {
    cudaLaunchConfig_t cfg = {};
    const size_t n = (size_t)L.nrows * B;
    cfg.gridDim = dim3((unsigned)std::min<size_t>((n + 255) / 256, 8 * 148));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ktimer_begin("k_j_reduce", s);
    e = cudaLaunchKernelEx(&cfg, k_j_reduce, (const float*)part, p.Q, L.nrows, p.Bp, B, L.bias, relu, y, ldy);
    if (e == cudaSuccess) e = launched();
    ktimer_end("k_j_reduce", s);
  }
  if (e == cudaSuccess && trace_path) {  // debug only: append this launch's stamps
    std::vector<unsigned long long> h(ntr);
    e = cudaMemcpyAsync(h.data(), trace, ntr * sizeof(h[0]), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (FILE* fp = fopen(trace_path, "ab")) {
      const unsigned long long n = ntr;
      fwrite(&n, sizeof(n), 1, fp);
      fwrite(h.data(), sizeof(h[0]), h.size(), fp);
      fclose(fp);
    }
  }
  return e;
}

}  // namespace cdn
