// Host side: CDNI parse/validate, canonical Huffman, load-time lane index,
// product-side compressor, variable-batch DP.  See host.hpp.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <queue>
#include <unordered_map>

namespace cdn {

// ------------------------------------------------------------------ Huffman

void HuffCode::build(int alphabet, const char* what) {
  n = (int)syms.size();
  std::memset(count, 0, sizeof(count));
  max_len = 0;
  for (int i = 0; i < n; ++i) {
    if (lens[i] == 0) throw Error(CDN_E_MALFORMED, std::string(what) + ": zero code length");
    if (lens[i] > 32) throw Error(CDN_E_UNSUPPORTED, std::string(what) + ": code length > 32");
    if (syms[i] >= alphabet) throw Error(CDN_E_MALFORMED, std::string(what) + ": symbol out of range");
    if (i > 0 && syms[i] <= syms[i - 1])
      throw Error(CDN_E_MALFORMED, std::string(what) + ": symbols not strictly ascending");
    count[lens[i]]++;
    max_len = std::max<int>(max_len, lens[i]);
  }
  if (n == 1 && lens[0] != 1) throw Error(CDN_E_MALFORMED, std::string(what) + ": single symbol needs length 1");
  if (n >= 2) {
    uint64_t kraft = 0;  // sum 2^(32-len) must equal 2^32 (complete prefix code)
    for (int i = 0; i < n; ++i) kraft += (uint64_t)1 << (32 - lens[i]);
    if (kraft != ((uint64_t)1 << 32)) throw Error(CDN_E_MALFORMED, std::string(what) + ": Kraft sum != 1");
  }
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return lens[a] != lens[b] ? lens[a] < lens[b] : syms[a] < syms[b];
  });
  sorted.resize(n);
  for (int i = 0; i < n; ++i) sorted[i] = syms[order[i]];
  uint64_t code = 0;
  uint32_t idx = 0;
  for (int L = 1; L <= 32; ++L) {
    first_code[L] = (uint32_t)code;
    first_index[L] = idx;
    code = (code + count[L]) << 1;
    idx += count[L];
  }
  code_of.assign(alphabet, 0);
  len_of.assign(alphabet, 0);
  for (int i = 0; i < n; ++i) {
    int L = lens[order[i]];
    code_of[sorted[i]] = first_code[L] + (uint32_t)(i - first_index[L]);
    len_of[sorted[i]] = (uint8_t)L;
  }
}

bool HuffCode::decode(uint32_t w, uint32_t& sym, uint32_t& len) const {
  for (int L = 1; L <= max_len; ++L) {
    uint32_t c = (L == 32) ? w : (w >> (32 - L));
    uint32_t off = c - first_code[L];
    if (off < count[L]) {
      sym = sorted[first_index[L] + off];
      len = (uint32_t)L;
      return true;
    }
  }
  return false;
}

// -------------------------------------------------------------------- CDNI

namespace {
struct Rd {
  const uint8_t* p;
  size_t n, pos = 0;
  void need(size_t k) {
    if (pos + k > n) throw Error(CDN_E_TRUNCATED, "CDNI truncated at byte " + std::to_string(pos));
  }
  template <class T> T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p + pos, sizeof(T));  // little-endian host (x86/aarch64)
    pos += sizeof(T);
    return v;
  }
  const uint8_t* take(size_t k) {
    need(k);
    const uint8_t* q = p + pos;
    pos += k;
    return q;
  }
};

void read_table(Rd& rd, HuffCode& h) {
  uint16_t cnt = rd.get<uint16_t>();
  h.syms.resize(cnt);
  h.lens.resize(cnt);
  for (int i = 0; i < cnt; ++i) {
    h.syms[i] = rd.get<uint16_t>();
    h.lens[i] = rd.get<uint8_t>();
  }
}

HostLayer read_layer(Rd& rd, bool keep) {
  HostLayer L;
  L.rows = rd.get<uint32_t>();
  L.cols = rd.get<uint32_t>();
  L.bh = rd.get<uint32_t>();
  L.bw = rd.get<uint32_t>();
  L.k = rd.get<uint8_t>();
  L.r = rd.get<uint8_t>();
  uint16_t ncb = rd.get<uint16_t>();
  const uint8_t* cb = rd.take(4ull * ncb);
  read_table(rd, L.val);
  read_table(rd, L.gap);
  if (L.rows == 0 || L.cols == 0) throw Error(CDN_E_MALFORMED, "empty layer geometry");
  if (L.bh == 0 || L.bw == 0 || L.rows % L.bh || L.cols % L.bw)
    throw Error(CDN_E_MALFORMED, "block " + std::to_string(L.bh) + "x" + std::to_string(L.bw) +
                                     " does not tile the matrix (C-34)");
  L.wrows = L.rows;
  L.wcols = L.cols;
  if (L.blocked()) {  // the streams index M' (Alg. 2)
    const uint64_t nst = (uint64_t)(L.wrows / L.bh) * (L.wcols / L.bw), sc = (uint64_t)L.bh * L.bw;
    if (nst >= (1ull << 31) || sc >= (1ull << 31)) throw Error(CDN_E_UNSUPPORTED, "blocked layer too large");
    L.rows = (uint32_t)nst;
    L.cols = (uint32_t)sc;
  }
  const uint8_t* rp = rd.take(16ull * (L.rows + 1ull));
  L.rp.resize(2ull * (L.rows + 1));
  std::memcpy(L.rp.data(), rp, 16ull * (L.rows + 1ull));
  L.vbits = L.rp[2ull * L.rows];
  L.gbits = L.rp[2ull * L.rows + 1];
  const uint8_t* vb = rd.take((L.vbits + 7) / 8);
  const uint8_t* gb = rd.take((L.gbits + 7) / 8);
  uint8_t hb = rd.get<uint8_t>();
  const uint8_t* bias = hb ? rd.take(4ull * L.wrows) : nullptr;
  if (!keep) return L;
  if (L.k < 1 || L.k > 8 || L.r < 1 || L.r > 8) throw Error(CDN_E_UNSUPPORTED, "k and r must be in 1..8");
  if (ncb != (1u << L.r)) throw Error(CDN_E_MALFORMED, "codebook size != 2^r");
  if (hb > 1) throw Error(CDN_E_MALFORMED, "bias flag");
  L.codebook.resize(ncb);
  std::memcpy(L.codebook.data(), cb, 4ull * ncb);
  if (L.rp[0] != 0 || L.rp[1] != 0) throw Error(CDN_E_MALFORMED, "row_ptr[0] != (0,0)");
  for (uint32_t i = 0; i < L.rows; ++i)
    if (L.rp[2ull * i + 2] < L.rp[2ull * i] || L.rp[2ull * i + 3] < L.rp[2ull * i + 1])
      throw Error(CDN_E_MALFORMED, "row_ptr not monotone at row " + std::to_string(i));
  L.val.build(1 << L.r, "val table");
  L.gap.build(1 << L.k, "gap table");
  L.vbytes.assign(vb, vb + (L.vbits + 7) / 8);
  L.gbytes.assign(gb, gb + (L.gbits + 7) / 8);
  L.vbytes.resize(L.vbytes.size() + 8, 0);
  L.gbytes.resize(L.gbytes.size() + 8, 0);
  L.has_bias = hb != 0;
  if (bias) {
    L.bias.resize(L.wrows);
    std::memcpy(L.bias.data(), bias, 4ull * L.wrows);
  }
  return L;
}
}  // namespace

HostLayer parse_cdni_layer(const uint8_t* p, size_t n, int idx, int* n_layers_out) {
  Rd rd{p, n};
  rd.need(4);
  if (std::memcmp(p, "CDNI", 4) != 0) throw Error(CDN_E_MAGIC, "bad CDNI magic");
  rd.pos = 4;
  uint16_t ver = rd.get<uint16_t>();
  if (ver != 1) throw Error(CDN_E_VERSION, "CDNI version " + std::to_string(ver));
  uint32_t nl = rd.get<uint32_t>();
  if (n_layers_out) *n_layers_out = (int)nl;
  if (idx < 0 || (uint32_t)idx >= nl) throw Error(CDN_E_ARG, "layer_in_file out of range");
  HostLayer out;
  for (uint32_t i = 0; i < nl; ++i) {
    HostLayer L = read_layer(rd, (int)i == idx);
    if ((int)i == idx) out = std::move(L);
  }
  if (rd.pos != n) throw Error(CDN_E_MALFORMED, "trailing bytes after last layer");
  return out;
}

// ------------------------------------------------------------ lane index

static inline uint32_t window32(const std::vector<uint8_t>& b, uint64_t pos) {
  uint64_t byte = pos >> 3;
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v = (v << 8) | b[byte + i];  // padded by 8 bytes
  return (uint32_t)((v << (pos & 7)) >> 32);
}

int choose_lanes_per_row(const HostLayer& L, uint32_t r0, uint32_t r1, int target) {
  // Expected val code length of an optimal code ~ sum len * 2^-len (Kraft).
  double el = 0;
  for (int i = 0; i < L.val.n; ++i) el += L.val.lens[i] * std::ldexp(1.0, -L.val.lens[i]);
  if (el <= 0) el = 1;
  double bits = (double)(L.rp[2ull * r1] - L.rp[2ull * r0]);
  double per_row = r1 > r0 ? bits / el / (double)(r1 - r0) : 0.0;
  int G = 1;
  while (G < 32 && per_row / G > target) G <<= 1;
  return G;
}

void build_lane_index(const HostLayer& L, uint32_t r0, uint32_t r1, int G, LaneIndex& out,
                      std::vector<Token>* toks) {
  out.G = G;
  out.log2G = 0;
  while ((1 << out.log2G) < G) out.log2G++;
  out.W = (L.cols + G - 1) / G;
  const uint32_t W = out.W;
  const uint32_t nr = r1 - r0;
  const uint32_t padsym = (1u << L.k) - 1;
  std::vector<uint32_t> vlen((size_t)nr * G), glen((size_t)nr * G), dl((size_t)nr * G);
  out.tok_start.assign((size_t)nr * G + 1, 0);
  out.start_v.assign((size_t)nr * G, 0);
  out.start_g.assign((size_t)nr * G, 0);
  out.start_prev.assign((size_t)nr * G, -1);
  bool need64 = false;
  uint64_t t = 0, nnz = 0;
  std::vector<uint64_t> vs(G + 1), gs(G + 1);
  std::vector<int64_t> pc(G);
  for (uint32_t i = r0; i < r1; ++i) {
    uint64_t vpos = L.rp[2ull * i], gpos = L.rp[2ull * i + 1];
    const uint64_t vend = L.rp[2ull * i + 2], gend = L.rp[2ull * i + 3];
    int64_t prev = -1;
    int next = 1;
    vs[0] = vpos; gs[0] = gpos; pc[0] = -1;
    out.tok_start[(size_t)(i - r0) * G] = t;
    while (vpos < vend) {
      uint32_t vsym, vl, gsym, gl;
      if (!L.val.decode(window32(L.vbytes, vpos), vsym, vl) || vpos + vl > vend)
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": bad val code");
      if (gpos >= gend)
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": val/gap token counts differ");
      if (!L.gap.decode(window32(L.gbytes, gpos), gsym, gl) || gpos + gl > gend)
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": bad gap code");
      int64_t c = prev + (int64_t)gsym + 1;
      if (c >= (int64_t)L.cols)
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": column >= cols");
      if (vsym == 0 && gsym != padsym)
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": pad without gap 2^k-1 (C-06)");
      int lane = (int)std::min<int64_t>(c / W, G - 1);
      while (next <= lane) {
        vs[next] = vpos; gs[next] = gpos; pc[next] = prev;
        out.tok_start[(size_t)(i - r0) * G + next] = t;
        ++next;
      }
      if (toks) toks->push_back(Token{(int32_t)i, (int32_t)c, (uint8_t)vsym});
      vpos += vl;
      gpos += gl;
      prev = c;
      ++t;
      nnz += vsym != 0;
    }
    if (gpos != gend) throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": val/gap token counts differ");
    while (next < G) {
      vs[next] = vend; gs[next] = gend; pc[next] = prev;
      out.tok_start[(size_t)(i - r0) * G + next] = t;
      ++next;
    }
    vs[G] = vend; gs[G] = gend;
    for (int j = 0; j < G; ++j) {
      size_t q = (size_t)(i - r0) * G + j;
      out.start_v[q] = vs[j];
      out.start_g[q] = gs[j];
      out.start_prev[q] = (int32_t)pc[j];
      vlen[q] = (uint32_t)(vs[j + 1] - vs[j]);
      glen[q] = (uint32_t)(gs[j + 1] - gs[j]);
      int64_t d = (int64_t)j * W - pc[j];
      if (vlen[q] == 0) d = 1;
      if (d < 1 || d > (int64_t)(1u << L.k))
        throw Error(CDN_E_MALFORMED, "internal: lane delta out of range");
      dl[q] = (uint32_t)(d - 1);
      if (vlen[q] >= 4096 || glen[q] >= 4096 || dl[q] >= 256) need64 = true;
    }
  }
  out.tok_start[(size_t)nr * G] = t;
  out.tokens = t;
  out.nnz = nnz;
  out.rec64 = need64;
  if (!need64) {
    out.rec32.resize((size_t)nr * G);
    for (size_t q = 0; q < out.rec32.size(); ++q) out.rec32[q] = vlen[q] | (glen[q] << 12) | (dl[q] << 24);
  } else {
    out.rec64v.resize((size_t)nr * G);
    for (size_t q = 0; q < out.rec64v.size(); ++q) {
      if (vlen[q] >= (1u << 24) || glen[q] >= (1u << 24))
        throw Error(CDN_E_UNSUPPORTED, "lane longer than 2^24 bits");
      out.rec64v[q] = (uint64_t)vlen[q] | ((uint64_t)glen[q] << 24) | ((uint64_t)dl[q] << 48);
    }
  }
}

void build_interval_index(const HostLayer& L, uint32_t r0, uint32_t r1, uint32_t W, IntervalIndex& out) {
  out.W = W;
  const uint32_t NI = (L.cols + W - 1) / W;
  out.NI = NI;
  const size_t n = (size_t)(r1 - r0) * NI;
  out.v.assign(n, 0);
  out.g.assign(n, 0);
  out.dm1.assign(n, 0);
  out.nnz.assign(n, 0);
  for (uint32_t i = r0; i < r1; ++i) {
    const size_t base = (size_t)(i - r0) * NI;
    uint64_t vpos = L.rp[2ull * i], gpos = L.rp[2ull * i + 1];
    const uint64_t vend = L.rp[2ull * i + 2];
    int64_t prev = -1;
    uint32_t next = 0;  // next interval whose start is not yet recorded
    auto record = [&](uint32_t upto) {  // intervals [next, upto] start here
      for (; next <= upto && next < NI; ++next) {
        out.v[base + next] = vpos;
        out.g[base + next] = gpos;
        const int64_t d = (int64_t)next * W - prev;
        out.dm1[base + next] = (uint8_t)std::min<int64_t>(std::max<int64_t>(d - 1, 0), 255);
      }
    };
    while (vpos < vend) {
      uint32_t vsym, vl, gsym, gl;
      if (!L.val.decode(window32(L.vbytes, vpos), vsym, vl) || !L.gap.decode(window32(L.gbytes, gpos), gsym, gl))
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": bad code (interval index)");
      const int64_t c = prev + (int64_t)gsym + 1;
      const uint32_t iv = (uint32_t)std::min<int64_t>(c / W, NI - 1);
      record(iv);
      if (vsym != 0) out.nnz[base + iv]++;
      vpos += vl;
      gpos += gl;
      prev = c;
    }
    record(NI - 1);  // trailing empty intervals start at the row end
  }
}

// ------------------------------------------------- merged token stream

bool build_joint_index(const HostLayer& L, uint32_t r0, uint32_t r1, int G, int Q, const std::vector<uint32_t>& lut,
                       int Lb, JointIndex& out, bool tail) {
  const uint32_t nr = r1 - r0;
  const int GS = G + (tail ? 1 : 0);  // records per row
  if (L.cols > 65535 || G < 1 || Q < 1 || G % Q) return false;
  uint64_t total = 0;
  uint32_t mx = 0;
  for (uint32_t i = r0; i < r1; ++i) {
    const uint64_t rb = (L.rp[2ull * i + 2] - L.rp[2ull * i]) + (L.rp[2ull * i + 3] - L.rp[2ull * i + 1]);
    if (rb >= 65536) return false;
    mx = std::max<uint32_t>(mx, (uint32_t)rb);
    total += rb;
  }
  if (total >= (1ull << 32) - 1024) return false;
  const int GQ = G / Q;
  const uint32_t Kq = (uint32_t)(((L.cols + Q - 1) / Q + 3) & ~3u);  // column group width (16-byte x slices)
  out.G = G;
  out.Q = Q;
  out.Kq = Kq;
  out.bits = total;
  out.max_row_bits = mx;
  out.words.assign((size_t)((total + 31) / 32) + 8, 0u);
  out.row_bit.assign((size_t)nr + 1, 0u);
  out.lane.assign((size_t)nr * GS, 0u);
  uint64_t pos = 0;
  auto put = [&](uint32_t code, uint32_t len) {  // MSB-first, len <= 32
    for (uint32_t b = 0; b < len; ++b) {
      if ((code >> (len - 1 - b)) & 1u) out.words[pos >> 5] |= 0x80000000u >> (pos & 31);
      ++pos;
    }
  };
  std::vector<uint32_t> tbit;   // bit offset (from the row start) of each token
  std::vector<int32_t> tprev;   // previous column before each token
  std::vector<int32_t> tcol;    // column of each token
  std::vector<uint8_t> tpad;    // token is padding
  for (uint32_t i = r0; i < r1; ++i) {
    const size_t li = i - r0;
    out.row_bit[li] = (uint32_t)pos;
    tbit.clear();
    tprev.clear();
    tcol.clear();
    tpad.clear();
    uint64_t vpos = L.rp[2ull * i], gpos = L.rp[2ull * i + 1];
    const uint64_t vend = L.rp[2ull * i + 2];
    int32_t prev = -1;
    while (vpos < vend) {
      uint32_t vs, vl, gs, gl;
      if (!L.val.decode(window32(L.vbytes, vpos), vs, vl) || !L.gap.decode(window32(L.gbytes, gpos), gs, gl))
        throw Error(CDN_E_MALFORMED, "row " + std::to_string(i) + ": bad code (merged stream)");
      tbit.push_back((uint32_t)(pos - out.row_bit[li]));
      tprev.push_back(prev);
      tpad.push_back(vs == 0);
      put(L.val.code_of[vs], vl);
      put(L.gap.code_of[gs], gl);
      prev += (int32_t)gs + 1;
      tcol.push_back(prev);
      vpos += vl;
      gpos += gl;
    }
    const size_t T = tbit.size();
    // the kernel's steps over tokens [a, b): from a, one joint-LUT lookup per
    // step consumes the padding run and the real token after it (or, for a
    // window the LUT cannot resolve, one token through the slow path)
    auto window_at = [&](uint64_t bit) {
      const uint64_t w = bit >> 5, o = bit & 31;
      const uint64_t v = ((uint64_t)out.words[w] << 32) | out.words[w + 1];
      return (uint32_t)(v >> (32 - o));
    };
    std::vector<size_t> step_at;
    auto steps = [&](size_t a, size_t b) {
      step_at.clear();
      size_t t = a;
      while (t < b) {
        step_at.push_back(t);
        const uint32_t e = lut[window_at(out.row_bit[li] + tbit[t]) >> (32 - Lb)];
        if (e == 0) {
          ++t;
        } else {
          const uint32_t end = tbit[t] + (e >> 27);
          while (t < b && tbit[t] < end) ++t;
        }
      }
    };
    // column group q = the tokens from the first with column >= q*Kq, moved
    // back over the padding before it (a group never ends with padding, so no
    // lookup folds padding into the next group's first real token); inside a
    // group, lane j starts at the kernel's step ~j*S_q/GQ of the group (S_q
    // steps), so every lane runs the same number of lookups (+-1) and ends
    // exactly at a step boundary
    size_t bprev = 0;
    for (int q = 0; q < Q; ++q) {
      size_t gb = 0;  // group's first token
      if (q > 0) {
        while (gb < T && tcol[gb] < (int64_t)q * Kq) ++gb;
        gb = std::max(gb, bprev);
        while (gb > bprev && tpad[gb - 1]) --gb;
      }
      size_t ge = T;  // next group's first token
      if (q + 1 < Q) {
        ge = 0;
        while (ge < T && tcol[ge] < (int64_t)(q + 1) * Kq) ++ge;
        ge = std::max(ge, gb);
        while (ge > gb && tpad[ge - 1]) --ge;
      }
      steps(gb, ge);
      const size_t S = step_at.size();
      for (int jj = 0; jj < GQ; ++jj) {
        const size_t bb = jj == 0 ? gb : (S ? step_at[(uint64_t)jj * S / (uint64_t)GQ] : ge);
        const uint32_t off = bb < T ? tbit[bb] : (uint32_t)(pos - out.row_bit[li]);
        const int32_t pc = bb < T ? tprev[bb] : prev;
        out.lane[li * GS + q * GQ + jj] = off | ((uint32_t)(pc + 1) << 16);
      }
      bprev = ge;
    }
    if (tail) out.lane[li * GS + G] = (uint32_t)(pos - out.row_bit[li]) | ((uint32_t)(prev + 1) << 16);
  }
  out.row_bit[nr] = (uint32_t)pos;
  if (pos != total) throw Error(CDN_E_MALFORMED, "internal: merged stream length");
  return true;
}

std::vector<uint32_t> build_joint_lut(const HuffCode& val, const HuffCode& gap, int Lb) {
  std::vector<uint32_t> lut((size_t)1 << Lb, 0u);
  for (uint32_t w = 0; w < (1u << Lb); ++w) {
    const uint32_t win = w << (32 - Lb);
    uint32_t pos = 0, adv = 0, sym = 0;
    bool any = false;
    for (;;) {
      uint32_t vs, vl, gs, gl;
      if (pos >= (uint32_t)Lb || !val.decode(win << pos, vs, vl) || pos + vl > (uint32_t)Lb) break;
      if (pos + vl >= 32 || !gap.decode(win << (pos + vl), gs, gl) || pos + vl + gl > (uint32_t)Lb) break;
      pos += vl + gl;
      adv += gs + 1;
      any = true;
      if (vs != 0) {  // a real token ends the entry; padding tokens (symbol 0, C-04) fold into it
        sym = vs;
        break;
      }
    }
    if (!any || pos > 31 || adv * 4 >= (1u << 17) || sym > 255) continue;  // slow path
    lut[w] = (sym * 4) | ((adv * 4) << 10) | (pos << 27);
  }
  return lut;
}

std::vector<uint32_t> build_joint_lut_r(const HuffCode& val, const HuffCode& gap, int Lb) {
  const std::vector<uint32_t> a = build_joint_lut(val, gap, Lb);
  std::vector<uint32_t> lut(a.size(), 0u);
  for (size_t w = 0; w < a.size(); ++w) {
    const uint32_t e = a[w];
    if (e == 0) continue;
    const uint32_t sym4 = e & 0x3ffu, adv4 = (e >> 10) & 0x1ffffu, len = e >> 27;
    if (adv4 >= (1u << 16)) continue;  // (slow path)
    lut[w] = sym4 | (len << 10) | (adv4 << 16);
  }
  return lut;
}

ShardSlice shard_slice(const HostLayer& H, int rank, int world, bool replicate) {
  ShardSlice sl;
  const uint32_t rb = replicate ? H.rows : (H.rows + (uint32_t)world - 1) / (uint32_t)world;
  sl.row0 = replicate ? 0 : std::min<uint64_t>(H.rows, (uint64_t)rb * (uint32_t)rank);
  sl.row1 = std::min<uint32_t>(H.rows, sl.row0 + rb);
  sl.vbase = (H.rp[2ull * sl.row0] >> 5) << 5;
  sl.gbase = (H.rp[2ull * sl.row0 + 1] >> 5) << 5;
  return sl;
}

HostLayer slice_rows(const HostLayer& H, const ShardSlice& sl) {
  if (H.blocked()) throw Error(CDN_E_UNSUPPORTED, "row shards of a blocked layer");
  HostLayer S;
  S.rows = sl.row1 - sl.row0;
  S.cols = H.cols;
  S.wrows = S.rows;
  S.wcols = H.wcols;
  S.bh = H.bh;
  S.bw = H.bw;
  S.k = H.k;
  S.r = H.r;
  S.codebook = H.codebook;
  S.val = H.val;
  S.gap = H.gap;
  const uint64_t v1 = H.rp[2ull * sl.row1], g1 = H.rp[2ull * sl.row1 + 1];
  auto cut = [](const std::vector<uint8_t>& b, uint64_t base_bit, uint64_t end_bit) {
    const uint64_t b0 = base_bit >> 3, b1 = (end_bit + 7) >> 3;
    std::vector<uint8_t> out(b.begin() + (ptrdiff_t)b0, b.begin() + (ptrdiff_t)std::min<uint64_t>(b.size(), b1));
    out.resize(out.size() + 8, 0);  // read-ahead padding (window32 reads 8 bytes)
    return out;
  };
  S.vbytes = cut(H.vbytes, sl.vbase, v1);
  S.gbytes = cut(H.gbytes, sl.gbase, g1);
  S.vbits = v1 - sl.vbase;
  S.gbits = g1 - sl.gbase;
  S.rp.resize(2ull * (S.rows + 1));
  for (uint32_t i = 0; i <= S.rows; ++i) {
    S.rp[2ull * i] = H.rp[2ull * (sl.row0 + i)] - sl.vbase;
    S.rp[2ull * i + 1] = H.rp[2ull * (sl.row0 + i) + 1] - sl.gbase;
  }
  S.has_bias = H.has_bias;
  if (H.has_bias) S.bias.assign(H.bias.begin() + sl.row0, H.bias.begin() + sl.row1);
  return S;
}

// -------------------------------------------------------------- compressor

namespace {
struct BitWriter {
  std::vector<uint8_t> bytes;
  uint64_t nbits = 0;
  void put(uint32_t code, int len) {
    for (int b = len - 1; b >= 0; --b) {
      if ((nbits & 7) == 0) bytes.push_back(0);
      if ((code >> b) & 1) bytes.back() |= (uint8_t)(0x80u >> (nbits & 7));
      ++nbits;
    }
  }
};

// Huffman code lengths with the (count, smallest symbol) merge rule (C-15).
std::vector<uint8_t> huffman_lengths(const std::vector<uint64_t>& freq) {
  const int A = (int)freq.size();
  std::vector<uint8_t> len(A, 0);
  struct Node { uint64_t c; int minsym; int id; };
  auto cmp = [](const Node& a, const Node& b) {
    return a.c != b.c ? a.c > b.c : a.minsym > b.minsym;
  };
  std::priority_queue<Node, std::vector<Node>, decltype(cmp)> pq(cmp);
  std::vector<int> parent;
  std::vector<int> leaf_sym;
  for (int s = 0; s < A; ++s)
    if (freq[s] > 0) {
      int id = (int)parent.size();
      parent.push_back(-1);
      leaf_sym.push_back(s);
      pq.push(Node{freq[s], s, id});
    }
  const int nleaf = (int)parent.size();
  if (nleaf == 0) return len;
  if (nleaf == 1) {
    len[leaf_sym[0]] = 1;
    return len;
  }
  while (pq.size() > 1) {
    Node a = pq.top(); pq.pop();
    Node b = pq.top(); pq.pop();
    int id = (int)parent.size();
    parent.push_back(-1);
    parent[a.id] = id;
    parent[b.id] = id;
    pq.push(Node{a.c + b.c, std::min(a.minsym, b.minsym), id});
  }
  for (int i = 0; i < nleaf; ++i) {
    int d = 0;
    for (int p = parent[i]; p != -1; p = parent[p]) ++d;
    if (d > 32) throw Error(CDN_E_UNSUPPORTED, "Huffman code longer than 32 bits");
    len[leaf_sym[i]] = (uint8_t)d;
  }
  return len;
}

template <class T> void put(std::vector<uint8_t>& o, T v) {
  uint8_t b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  o.insert(o.end(), b, b + sizeof(T));
}
}  // namespace

std::vector<uint8_t> compress_dense(const float* W, const float* bias, uint32_t rows, uint32_t cols,
                                    double density, int r, int k, int quantizer, uint32_t bh, uint32_t bw) {
  if (quantizer != 0 && quantizer != 1) throw Error(CDN_E_ARG, "quantizer must be 0 (linear) or 1 (k-means)");
  if (bw == 0) bw = cols;
  if (bh == 0 || rows % bh || cols % bw) throw Error(CDN_E_ARG, "block does not tile the matrix (C-34)");
  if (!W || rows == 0 || cols == 0) throw Error(CDN_E_ARG, "empty matrix");
  if (r < 1 || r > 8 || k < 1 || k > 8) throw Error(CDN_E_UNSUPPORTED, "k and r must be in 1..8");
  if (!(density >= 0.0 && density <= 1.0)) throw Error(CDN_E_ARG, "density must be in [0,1]");
  const uint64_t n = (uint64_t)rows * cols;
  // prune (C-10): exact count, ties -> lower row-major index
  double nk = std::floor(density * (double)n + 0.5);
  uint64_t n_keep = nk <= 0 ? 0 : (nk >= (double)n ? n : (uint64_t)nk);
  std::vector<uint8_t> keep(n, 0);
  if (n_keep == n) {
    std::fill(keep.begin(), keep.end(), 1);
  } else if (n_keep > 0) {
    std::vector<float> a(n);
    for (uint64_t i = 0; i < n; ++i) a[i] = std::fabs(W[i]);
    std::nth_element(a.begin(), a.begin() + (n - n_keep), a.end());
    const float t = a[n - n_keep];
    uint64_t above = 0;
    for (uint64_t i = 0; i < n; ++i)
      if (std::fabs(W[i]) > t) { keep[i] = 1; ++above; }
    uint64_t need = n_keep - above;
    for (uint64_t i = 0; i < n && need; ++i)
      if (std::fabs(W[i]) == t) { keep[i] = 1; --need; }
  }
  // quantize (C-04/05/07)
  const int ncb = 1 << r;
  std::vector<float> cb(ncb, 0.0f);
  double lo = 0, hi = 0;
  bool any = false;
  for (uint64_t i = 0; i < n; ++i)
    if (keep[i]) {
      double v = (double)W[i];
      if (!any) { lo = hi = v; any = true; }
      lo = std::min(lo, v);
      hi = std::max(hi, v);
    }
  if (any) {
    const double denom = ncb > 2 ? (double)(ncb - 2) : 1.0;
    for (int j = 1; j < ncb; ++j) cb[j] = (float)(lo + (hi - lo) * (double)(j - 1) / denom);
    if (quantizer == 1) {
      // 1-D Lloyd k-means from the same grid (C-33): nearest centre in binary64
      // (ties -> smaller index), move non-empty centres to the binary64 mean of
      // their weights summed in row-major order, <= 50 iterations or until no
      // centre moves by more than 1e-7 * max(|lo|, |hi|)
      const int nc = ncb - 1;
      std::vector<double> c(nc), sum(nc);
      std::vector<uint64_t> cnt(nc);
      for (int j = 0; j < nc; ++j) c[j] = lo + (hi - lo) * (double)j / denom;
      const double eps = 1e-7 * std::max(std::fabs(lo), std::fabs(hi));
      for (int it = 0; it < 50; ++it) {
        std::fill(sum.begin(), sum.end(), 0.0);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (uint64_t i = 0; i < n; ++i) {
          if (!keep[i]) continue;
          const double v = (double)W[i];
          int best = 0;
          double bd = std::fabs(v - c[0]);
          for (int j = 1; j < nc; ++j) {
            const double d = std::fabs(v - c[j]);
            if (d < bd) { bd = d; best = j; }
          }
          sum[best] += v;
          cnt[best]++;
        }
        double moved = 0.0;
        for (int j = 0; j < nc; ++j) {
          if (!cnt[j]) continue;
          const double nv = sum[j] / (double)cnt[j];
          moved = std::max(moved, std::fabs(nv - c[j]));
          c[j] = nv;
        }
        if (moved <= eps) break;
      }
      for (int j = 0; j < nc; ++j) cb[j + 1] = (float)c[j];
    }
  }
  // relative index (C-01..03) + token streams, over the stored
  // rows: the weight rows, or the blocks of M' (Alg. 2, C-34) flattened
  // row-major (position p of block (bi, bj) = weight (bi*bh + p/bw, bj*bw + p%bw))
  const uint32_t cap = (1u << k) - 1;
  const bool blocked = !(bh == 1 && bw == cols);
  const uint32_t nbj = cols / bw;
  const uint32_t srows = blocked ? (rows / bh) * nbj : rows, scols = blocked ? bh * bw : cols;
  std::vector<uint8_t> vt, gt;
  std::vector<uint64_t> row_tok(srows + 1, 0);
  for (uint32_t i = 0; i < srows; ++i) {
    row_tok[i] = vt.size();
    int64_t prev = -1;
    const uint32_t bi = i / nbj, bj = i % nbj;
    for (uint32_t c = 0; c < scols; ++c) {
      const uint64_t idx = blocked ? (uint64_t)(bi * bh + c / bw) * cols + bj * bw + c % bw
                                   : (uint64_t)i * cols + c;
      if (!keep[idx]) continue;
      const double w = (double)W[idx];
      int best = 1;
      double bd = std::fabs(w - (double)cb[1]);
      for (int j = 2; j < ncb; ++j) {
        double d = std::fabs(w - (double)cb[j]);
        if (d < bd) { bd = d; best = j; }
      }
      int64_t g = (int64_t)c - prev - 1;
      while (g > (int64_t)cap) {
        vt.push_back(0);
        gt.push_back((uint8_t)cap);
        prev += (int64_t)1 << k;
        g -= (int64_t)1 << k;
      }
      vt.push_back((uint8_t)best);
      gt.push_back((uint8_t)g);
      prev = c;
    }
  }
  row_tok[srows] = vt.size();
  // Huffman per stream (C-14..17)
  std::vector<uint64_t> fv(ncb, 0), fg(1u << k, 0);
  for (uint8_t s : vt) fv[s]++;
  for (uint8_t s : gt) fg[s]++;
  HuffCode hv, hg;
  auto lv = huffman_lengths(fv), lg = huffman_lengths(fg);
  for (int s = 0; s < ncb; ++s)
    if (lv[s]) { hv.syms.push_back((uint16_t)s); hv.lens.push_back(lv[s]); }
  for (int s = 0; s < (1 << k); ++s)
    if (lg[s]) { hg.syms.push_back((uint16_t)s); hg.lens.push_back(lg[s]); }
  hv.build(ncb, "val");
  hg.build(1 << k, "gap");
  BitWriter bv, bg;
  std::vector<uint64_t> rp(2ull * (srows + 1));
  for (uint32_t i = 0; i < srows; ++i) {
    rp[2ull * i] = bv.nbits;
    rp[2ull * i + 1] = bg.nbits;
    for (uint64_t t = row_tok[i]; t < row_tok[i + 1]; ++t) {
      bv.put(hv.code_of[vt[t]], hv.len_of[vt[t]]);
      bg.put(hg.code_of[gt[t]], hg.len_of[gt[t]]);
    }
  }
  rp[2ull * srows] = bv.nbits;
  rp[2ull * srows + 1] = bg.nbits;
  // serialize
  std::vector<uint8_t> o;
  o.insert(o.end(), {'C', 'D', 'N', 'I'});
  put<uint16_t>(o, 1);
  put<uint32_t>(o, 1);
  put<uint32_t>(o, rows); put<uint32_t>(o, cols); put<uint32_t>(o, bh); put<uint32_t>(o, bw);
  put<uint8_t>(o, (uint8_t)k); put<uint8_t>(o, (uint8_t)r);
  put<uint16_t>(o, (uint16_t)ncb);
  for (float v : cb) put<float>(o, v);
  for (HuffCode* h : {&hv, &hg}) {
    put<uint16_t>(o, (uint16_t)h->syms.size());
    for (size_t i = 0; i < h->syms.size(); ++i) { put<uint16_t>(o, h->syms[i]); put<uint8_t>(o, h->lens[i]); }
  }
  for (uint64_t v : rp) put<uint64_t>(o, v);
  o.insert(o.end(), bv.bytes.begin(), bv.bytes.end());
  o.insert(o.end(), bg.bytes.begin(), bg.bytes.end());
  if (bias) {
    put<uint8_t>(o, 1);
    for (uint32_t i = 0; i < rows; ++i) put<float>(o, bias[i]);
  } else {
    put<uint8_t>(o, 0);
  }
  return o;
}

// --------------------------------------------------------------------- DP

PlanResult plan_dp(const double* T, const uint64_t* inb, const uint64_t* outb, const uint64_t* ws,
                   int f, int Bmax, uint64_t tot, double lat, uint64_t step) {
  const double INF = std::numeric_limits<double>::infinity();
  if (f <= 0 || Bmax <= 0) throw Error(CDN_E_ARG, "empty planning problem");
  if (Bmax >= (1 << 18)) throw Error(CDN_E_ARG, "Bmax too large");
  if (step == 0) step = 1;
  std::unordered_map<uint64_t, std::pair<double, int>> memo;
  std::vector<std::vector<int>> divs(Bmax + 1);
  for (int B = 1; B <= Bmax; ++B)
    for (int b = B; b >= 1; --b)
      if (B % b == 0) divs[B].push_back(b);  // descending: C-26 larger b first
  auto feasible = [&](int i, int B, uint64_t A) {
    return A <= tot && A + inb[i] * (uint64_t)B + ws[i] + outb[i] * (uint64_t)B <= tot;
  };
  std::function<std::pair<double, int>(int, int, uint64_t)> opt = [&](int i, int B, uint64_t A) {
    if (!feasible(i, B, A)) return std::make_pair(INF, 0);
    uint64_t key = ((uint64_t)i << 58) | ((uint64_t)B << 40) | A;
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    double v;
    int bb = 0;
    if (i == 0) {
      v = T[(size_t)0 * Bmax + (B - 1)];
    } else {
      double best = INF;
      for (int b : divs[B]) {
        uint64_t A2 = A + inb[i] * (uint64_t)(B - b);
        A2 = (A2 + step - 1) / step * step;  // C-25: round up
        auto sub = opt(i - 1, b, A2);
        double cand = (double)(B / b) * sub.first;
        if (cand < best) { best = cand; bb = b; }
      }
      v = best < INF ? T[(size_t)i * Bmax + (B - 1)] + best : INF;
    }
    if (lat > 0 && v > lat) v = INF;
    auto r = std::make_pair(v, bb);
    memo.emplace(key, r);
    return r;
  };
  PlanResult res;
  double best_per = INF;
  for (int B = Bmax; B >= 1; --B) {
    auto v = opt(f - 1, B, 0);
    if (v.first == INF) continue;
    double per = v.first / (double)B;
    if (!res.feasible || per < best_per) {
      res.feasible = true;
      best_per = per;
      res.opt = v.first;
      std::vector<int> bs{B};
      uint64_t A = 0;
      int Bi = B;
      for (int i = f - 1; i >= 1; --i) {
        int b = opt(i, Bi, A).second;
        A = A + inb[i] * (uint64_t)(Bi - b);
        A = (A + step - 1) / step * step;
        Bi = b;
        bs.push_back(b);
      }
      std::reverse(bs.begin(), bs.end());
      res.batches = bs;
    }
  }
  return res;
}

}  // namespace cdn
