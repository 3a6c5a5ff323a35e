// Device helpers shared by the decode / FC kernels (sm_100a): non-coherent
// stream loads, the canonical-Huffman slow path, a prefetching MSB-first bit
// reader, and the mbarrier / bulk-copy / named-barrier PTX wrappers used by the
// warp-specialised band kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cdn {
namespace dev {

static __device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// if (pred) v = *p, with the load targeting v's own register
static __device__ __forceinline__ void ldg_u32_if(uint32_t& v, const uint32_t* p, uint32_t pred) {
  asm("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.global.nc.u32 %0, [%1]; }" : "+r"(v) : "l"(p), "r"(pred));
}

// Canonical decode of a code longer than the LUT width (rare).  tab[0..32] =
// first_code per length, tab[33..65] = count, tab[66..98] = first index into
// the canonically sorted symbols.  Returns (len << 16) | sym.
static __device__ __noinline__ uint32_t slow_sym(uint32_t w, int from, const uint32_t* tab,
                                                 const uint16_t* sorted, int maxlen) {
  for (int l = from; l <= maxlen; ++l) {
    const uint32_t c = (l == 32) ? w : (w >> (32 - l));
    const uint32_t off = c - tab[l];
    if (off < tab[33 + l]) return ((uint32_t)l << 16) | sorted[tab[66 + l] + off];
  }
  return 32u << 16;  // unreachable for a validated container
}

// MSB-first reader over big-endian packed words with the word after the
// current pair already in flight, so a one-word advance never waits on memory.
// peek() = the 32 bits starting `off` bits into w0; skip(n) takes any n.
struct PReader {
  const uint32_t* base;
  uint32_t cur, off, w0, w1, w2;
  __device__ __forceinline__ void init(const uint32_t* words, uint32_t bit) {
    base = words;
    cur = bit >> 5;
    off = bit & 31;
    w0 = ldg_u32(base + cur);
    w1 = ldg_u32(base + cur + 1);
    w2 = ldg_u32(base + cur + 2);
  }
  __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, off); }
  __device__ __forceinline__ void skip(uint32_t n) {
    off += n;
    const uint32_t adv = off >> 5;
    off &= 31;
    if (adv == 1) {
      ++cur;
      w0 = w1;
      w1 = w2;
      w2 = ldg_u32(base + cur + 2);
    } else if (adv > 1) {
      cur += adv;
      w0 = ldg_u32(base + cur);
      w1 = ldg_u32(base + cur + 1);
      w2 = ldg_u32(base + cur + 2);
    }
  }
};

// Lean MSB-first reader for decode lanes: a two-word window (w0:w1) plus
// four words in flight, so the word moved into the window on an advance was
// requested four advances (~128 bits, tens of tokens) earlier -- a shallower
// queue lets the predicated register rotation wait on L2 latency every few
// steps.  skip(n) for n <= 32.  Requires >= 6 words of tail padding.
struct SReader {
  const uint32_t* p;  // next word to prefetch
  uint32_t off, w0, w1, n1, n2, n3, n4;
  __device__ __forceinline__ void init(const uint32_t* words, uint32_t bit) {
    p = words + (bit >> 5);
    off = bit & 31;
    w0 = ldg_u32(p);
    w1 = ldg_u32(p + 1);
    n1 = ldg_u32(p + 2);
    n2 = ldg_u32(p + 3);
    n3 = ldg_u32(p + 4);
    n4 = ldg_u32(p + 5);
    p += 6;
  }
  __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, off); }
  __device__ __forceinline__ void skip(uint32_t n) {
    off += n;
    const uint32_t adv = off >= 32;
    if (adv) {
      off -= 32;
      w0 = w1;
      w1 = n1;
      n1 = n2;
      n2 = n3;
      n3 = n4;
    }
    // predicated load straight into n4: a plain `n4 = ldg(p)` lets the compiler
    // load into a temporary and MOV it into n4 a few instructions later, which
    // waits for the load there and defeats the prefetch
    ldg_u32_if(n4, p, adv);
    p += adv;
  }
};

static __device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

static __device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
static __device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
static __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
static __device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// Stream reader whose words arrive through a per-lane 4-block (64 B) ring in
// shared memory filled by cp.async (LDGSTS) three blocks ahead of the cursor:
// the decode chain only ever waits on shared-memory latency.  Ring layout per
// warp and stream: [slot 0..3][lane 0..31][16 B], so a warp's reads spread over
// the banks.  Requires 16-byte aligned word arrays with >= 16 words of tail
// padding.  Two readers of one thread share its cp.async group sequence: a
// block is waited for with wait_group(2), which holds because every block is
// followed by at least two later groups of its own stream before it is read.
struct RReader {
  const uint4* g;   // 16-byte blocks of the stream
  uint32_t ring;    // smem address of (slot 0, this lane)
  uint32_t wi, off, w0, w1, fb;
  __device__ __forceinline__ uint32_t slot_addr(uint32_t blk) const { return ring + (blk & 3) * 512; }
  __device__ __forceinline__ uint32_t word(uint32_t w) const { return lds_u32(slot_addr(w >> 2) + (w & 3) * 4); }
  // start at `bit`; issues the 4 block fetches (call fill_wait before peek).
  __device__ __forceinline__ void start(const uint32_t* words, uint32_t ring_addr, uint32_t bit) {
    g = reinterpret_cast<const uint4*>(words);
    ring = ring_addr;
    wi = bit >> 5;
    off = bit & 31;
    const uint32_t cb = wi >> 2;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      cp_async16(slot_addr(cb + i), g + cb + i);
      cp_async_commit();
    }
    fb = cb + 4;
  }
  __device__ __forceinline__ void fill_done() {
    w0 = word(wi);
    w1 = word(wi + 1);
  }
  __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, off); }
  __device__ __forceinline__ void skip(uint32_t n) {  // n <= 32
    off += n;
    if (off >= 32) {
      off -= 32;
      ++wi;
      w0 = w1;
      if ((wi & 3) == 0) {  // entered a new block: refill the slot of the one left
        cp_async16(slot_addr(fb), g + fb);
        cp_async_commit();
        ++fb;
      }
      if (((wi + 1) & 3) == 0) cp_async_wait<2>();
      w1 = word(wi + 1);
    }
  }
};

static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

static __device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

static __device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

static __device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

static __device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

// Bulk (non-tensor) async copy global -> shared, completing on an mbarrier
// (SASS UBLKCP).  bytes % 16 == 0, both addresses 16-byte aligned.
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

static __device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace dev
}  // namespace cdn
