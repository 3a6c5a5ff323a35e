// Host side of the library: CDNI container, canonical Huffman tables, the
// load-time decode-lane index (container row a1 of SURVEY §8(a)), the
// product-side compressor and the variable-batch DP.  No CUDA here.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cdn.h"

namespace cdn {

struct Error : std::runtime_error {
  cdn_status code;
  Error(cdn_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Canonical Huffman code rebuilt from (symbol, length) pairs (C-17).
struct HuffCode {
  int n = 0;
  int max_len = 0;
  std::vector<uint16_t> syms;     // ascending symbol order (as stored)
  std::vector<uint8_t> lens;
  std::vector<uint16_t> sorted;   // canonical order: (length, symbol)
  uint32_t count[33] = {0};
  uint32_t first_code[33] = {0};
  uint32_t first_index[33] = {0};
  std::vector<uint32_t> code_of;  // per symbol (alphabet-sized), encode side
  std::vector<uint8_t> len_of;

  // Validates lengths (1..32 else UNSUPPORTED/MALFORMED), symbol range, Kraft
  // equality (complete code for n >= 2; a single symbol has length 1).
  void build(int alphabet, const char* what);
  // Decode one symbol from a 32-bit left-aligned window.  false: no code.
  bool decode(uint32_t window, uint32_t& sym, uint32_t& len) const;
};

struct HostLayer {
  // rows x cols = the STORED matrix the streams and row_ptr index: the weight
  // matrix, or for the block-contiguous container of Alg. 2 (C-34) its M'
  // (one stored row per bh x bw block, flattened row-major)
  uint32_t rows = 0, cols = 0, bh = 1, bw = 0, k = 0, r = 0;
  uint32_t wrows = 0, wcols = 0;  // the weight matrix (bias has wrows entries)
  bool blocked() const { return !(bh == 1 && bw == wcols); }
  std::vector<float> codebook;
  HuffCode val, gap;
  std::vector<uint64_t> rp;       // 2*(rows+1): (val bit, gap bit) per row start
  std::vector<uint8_t> vbytes, gbytes;  // streams, + 8 zero bytes of padding
  uint64_t vbits = 0, gbits = 0;
  bool has_bias = false;
  std::vector<float> bias;
};

// Parse layer `idx` of a CDNI buffer (format in DESIGN.md).
HostLayer parse_cdni_layer(const uint8_t* p, size_t n, int idx, int* n_layers_out = nullptr);

// Decode-lane index for rows [r0, r1) of a layer.
// G lanes per row; lane j owns the tokens whose absolute column falls in
// [j*W, (j+1)*W), W = ceil(cols/G).  Record per (row, lane): the lane's bit
// lengths in both streams and delta = j*W - (column of the previous token),
// 1 <= delta <= 2^k (pads bound every gap by 2^k).
struct LaneIndex {
  int G = 1, log2G = 0;
  uint32_t W = 1;
  bool rec64 = false;
  std::vector<uint32_t> rec32;
  std::vector<uint64_t> rec64v;
  std::vector<uint64_t> tok_start;  // (rows*G + 1) token index of each lane's first token
  // Absolute decoder state at every lane start (val bit, gap bit, previous
  // column): the restart points of the large-batch band kernel's K-splits.
  std::vector<uint64_t> start_v, start_g;
  std::vector<int32_t> start_prev;
  uint64_t tokens = 0, nnz = 0;
};

struct Token { int32_t row, col; uint8_t sym; };

// Host walk of rows [r0, r1): validates the streams (both end exactly at the
// next row_ptr, equal token counts, columns < cols, pad invariant C-06) and
// fills the lane index.  tokens_out, if non-null, receives every token.
void build_lane_index(const HostLayer& L, uint32_t r0, uint32_t r1, int G, LaneIndex& out,
                      std::vector<Token>* tokens_out = nullptr);

// Merged token stream of the small-batch kernel (k_fc_j, joint.cu; reading
// C-35): the row's two Huffman code streams interleaved token by token --
// val code, then its gap code -- so one MSB-first reader and one lookup serve
// both (a bit permutation of the same codes: the same number of bits).
// Decode lanes: G per row in Q column groups (group q = G/Q lanes holding the
// columns [q Kq, (q+1) Kq), so a CTA of group q stages only that slice of x);
// inside a group the lanes are split at the kernel's joint-LUT steps (lane j
// starts at the group's step ~j S_q Q/G: every lane runs the same number of
// lookups, +-1); group boundaries are moved back over padding tokens so no
// lookup folds a group's padding into the next group's first real token (a
// row never ends with padding: padding precedes a real token, C-02).  A lane record = bit offset of its first
// token from the row start (u16) | (previous column + 1) << 16 (u16).
struct JointIndex {
  int G = 1, Q = 1;                // lanes per row; column groups (lanes [q G/Q, (q+1) G/Q) hold columns [q Kq, (q+1) Kq))
  uint32_t Kq = 0;
  std::vector<uint32_t> words;     // big-endian u32 words (bit i = bit 31-(i%32) of word i/32), >= 8 words padding
  std::vector<uint32_t> row_bit;   // nr+1: start bit of each local row (relative to the slice)
  std::vector<uint32_t> lane;      // nr*G records
  uint64_t bits = 0;
  uint32_t max_row_bits = 0;
};
// false (nothing built) when a row has >= 2^16 bits or cols > 65535
// lut / Lb: the joint LUT the kernel will use (build_joint_lut): lanes start
// at the kernel's lookup steps, so they are balanced in steps
// tail: one more record per row (index G: the row's bit length | (last column + 1) << 16), so
// lane j's end (bits and last column) is always record j + 1 (the small-batch kernel's layout)
bool build_joint_index(const HostLayer& L, uint32_t r0, uint32_t r1, int G, int Q, const std::vector<uint32_t>& lut,
                       int Lb, JointIndex& out, bool tail = false);
// Joint LUT over the next Lb bits of the merged stream: the leading padding
// tokens (val symbol 0 with its gap code) and then one real token, when they
// lie inside the window.  Entry: 4 * val symbol (bits 0-9) | 4 * column
// advance << 10 (17 bits) | total bits << 27 (5 bits); 0 = the first token is
// longer than the window (the kernel's slow path decodes it code by code).
std::vector<uint32_t> build_joint_lut(const HuffCode& val, const HuffCode& gap, int Lb);
// The same lookups in the small-batch kernel's entry layout: 4 * val symbol
// (bits 0-9) | total bits << 10 (5 bits) | 0 (bit 15) | 4 * column advance << 16
// (16 bits) -- (entry >> 10) adds the bits to a lane's bit offset and the
// advance to the x offset above it in one add (joint.cu); 0 = slow path.
std::vector<uint32_t> build_joint_lut_r(const HuffCode& val, const HuffCode& gap, int Lb);

// Restart index of the large-batch band kernel: every row split into NI
// intervals of W columns; per (row, interval) the decoder state before the
// first token whose column is >= i*W (bit offsets in both streams, previous
// column = i*W - (dm1+1)), and the number of real (non-pad) tokens whose
// column lies in the interval.  Built by the load-time host walk (SURVEY §8(a)
// a1: chunk start-bit offsets and row boundaries).
struct IntervalIndex {
  uint32_t W = 16, NI = 0;
  std::vector<uint64_t> v, g;     // absolute start bits, rows*NI
  std::vector<uint8_t> dm1, nnz;  // rows*NI
};
void build_interval_index(const HostLayer& L, uint32_t r0, uint32_t r1, uint32_t W, IntervalIndex& out);

// Row-block shard of a rank: rows [row0, row1) with
// ceil(rows/world) rows per rank, and the word-aligned bit positions where the
// rank's slices of the val / gap streams start (streams are cut, never
// re-encoded).  replicate: every rank keeps all rows (CONV layers).
struct ShardSlice {
  uint32_t row0 = 0, row1 = 0;
  uint64_t vbase = 0, gbase = 0;
};
ShardSlice shard_slice(const HostLayer& H, int rank, int world, bool replicate);
// A standalone layer holding only the shard's rows: stream bytes cut at the
// slice bases, row_ptr rebased, bias sliced.  Decoding it must give exactly the
// shard's rows of the full layer (the invariant row-block sharding relies on).
HostLayer slice_rows(const HostLayer& H, const ShardSlice& s);

int choose_lanes_per_row(const HostLayer& L, uint32_t r0, uint32_t r1, int target_tokens);

// Product-side compressor (independent of oracle/, same readings).
std::vector<uint8_t> compress_dense(const float* W, const float* bias, uint32_t rows, uint32_t cols,
                                    double density, int r, int k, int quantizer = 0, uint32_t bh = 1,
                                    uint32_t bw = 0);  // bw = 0: cols (unblocked)

// Variable-batch DP with memory axis granularity `step` bytes.
struct PlanResult {
  bool feasible = false;
  std::vector<int> batches;
  double opt = 0.0;
};
PlanResult plan_dp(const double* time_ms, const uint64_t* in_b, const uint64_t* out_b,
                   const uint64_t* ws, int f, int Bmax, uint64_t tot, double latency, uint64_t step);

}  // namespace cdn
