// decode.cu -- K8: chunk-parallel Huffman decode fused with the dual-quant
// dequantiser, plus the v1 (reference stream) compat decoder.
//
// Replaces pipeline._parse_sz_stream (pipeline.py:203-223) ->
// encode.huffman_decode (encode.py:242-261) -> K.huff_decode
// (_kernels.py:348-374) and quantize.dequantize_field -> K.sz_dequantize
// (_kernels.py:126-147).
//
// v2 (kind 3) decode: chunks are self-contained (the dual-quant chain
// restarts at every 16384-symbol chunk and escape values sit inline in the
// bitstream), so one WARP decodes one chunk with no cross-chunk traffic:
//   1. persistent CTAs, one field each, stage a 2^16-entry code-length table
//      and the canonical symbol table in shared memory once;
//   2. each lane takes 1/32 of the chunk's bits and walks it from an
//      arbitrary bit with a 64-bit register bit-reader (code lengths only):
//      Huffman codes resynchronise within a few codewords, so the walk's end
//      is the true codeword boundary after the slice;
//   3. lane l decodes from lane l-1's end, counting codewords and summing
//      the lattice deltas (reset at escapes); lanes whose start moved
//      repeat until no end moves;
//   4. warp scans give each lane its output offset and incoming lattice
//      index; lanes decode their slice once more and write
//      recon = f32(k * 2b) or the inline escape value.
// Status words: INVALID_CODE / TRUNCATED / BAD_STREAM -> DecodeError.
#include <cstdio>
#include <cstdlib>

#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kDWarps = 24;        // warps per CTA, each decodes one chunk at a time
constexpr int kDThreads = kDWarps * 32;
constexpr int kLutBits = 16;       // code-length table index bits (u8 entries, 64 KiB)
constexpr int kSmemSyms = 16384;   // sorted-symbol table staged in smem up to this k
constexpr int kTpcBits = 15;       // thread-per-chunk fused table index bits (i32, 128 KiB)
#ifndef NBZG_LV_RING
#define NBZG_LV_RING 16
#endif
// decode_lv_kernel's per-thread word ring (8 or 16 words; 16 leaves room for
// two 16-byte stream blocks in flight per lane, at the cost of half the
// long-code table)
constexpr int kLvRing = NBZG_LV_RING;
constexpr int kLvRingMask = kLvRing - 1;
// secondary (long-code) table entries that always fit beside a full primary
// table (12800: with the 48 KiB ring and 768 B of static shared memory the
// CTA sits 256 bytes under the 227 KiB limit)
constexpr int kTpc2Cap = kLvRing == 16 ? 12800 : 16384;
constexpr int kTpcMaxThreads = 704;
constexpr int kLvMaxThreads = 768;  // decode_lv_kernel: 80 registers x 768 fit the register file
constexpr int kRingStride = 1024;  // words between ring slots (power of two, >= threads)
// decode_lv_kernel's ring: slot stride = its thread cap
constexpr int kLvStride = NBZG_LV_RING == 16 ? 768 : kRingStride;
constexpr int kTpcTab = (1 << kTpcBits) + kTpc2Cap;
constexpr int kLut2Stride = 2 << kTpcBits;  // global fused table per field: primary | long entries
#ifndef NBZG_CANON_MASS
#define NBZG_CANON_MASS 0.996
#endif
constexpr double kCanonMass = NBZG_CANON_MASS;  // fused-table coverage below which the canonical mode decodes
constexpr int kCanonMaxK = 65536;     // its symbol table: u16 by canonical rank, <= 128 KiB
constexpr int kCanonBits = 12;        // first-length table index bits (8-byte entries: 32 KiB)
#ifndef NBZG_CANON_COST
#define NBZG_CANON_COST 1.5
#endif
constexpr double kCanonCost = NBZG_CANON_COST, kCanonCostBits = 12.5;  // host-side CTA split

struct DParsed {
  uint64_t n_esc, k, total_bits;
  uint64_t index_off, bits_off, esc_off;
  uint32_t min_len, max_len;
  uint32_t status;
  uint32_t esc_len;   // code length of symbol 0 (escape), 0 if absent
  uint64_t esc_code;  // its canonical code word: first_code[esc_len] (rank 0)
  uint64_t t2_r0;     // thread-per-chunk secondary table: window start,
  uint32_t t2_w, t2_n;  // resolution bits and entry count (0 = none)
  uint32_t use_canon;   // thread-per-chunk decoder: canonical mode (large alphabets)
  uint64_t first_code[64];
  uint32_t first_idx[64];
  uint32_t counts[64];
};

struct DArgs {
  DField f[6];
  int nf;
  int64_t n, nchunks, nbins;
  int half;
  DParsed* parsed;     // [nf]
  uint32_t* lut;       // [nf][2^16] u8 code lengths
  int32_t* lut2;       // [nf][2^15] fused (delta, length) entries, 0 = slow path
  uint32_t* ssyms;     // [nf][nbins] sorted (len, sym) symbols
  uint64_t* choff;     // [nf][nchunks+1] chunk bit offsets
  uint64_t* lb;        // [nf][2][nchunks]
  uint32_t* tickets;   // [nf]
  uint32_t* status;    // global status word
  int cta0[7];         // decode_lv_kernel: first CTA of each field (cta0[nf] = grid)
};

NBZG_DEV uint32_t ld_u32_bytes(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
NBZG_DEV uint64_t ld_u64_bytes(const uint8_t* p) {
  return (uint64_t)ld_u32_bytes(p) | ((uint64_t)ld_u32_bytes(p + 4) << 32);
}
NBZG_DEV void fail(uint32_t* status, uint32_t code) { atomicCAS(status, 0u, code); }

// ---------------------------------------------------------------- D0: parse
// Validates the table (HuffmanTable.__post_init__, encode.py:105-121 and
// deserialize 182-196) and builds the canonical decode tables.
__device__ void chunk_offsets_body(const DArgs& a, int fi);
NBZG_DEV void parse_body(const DArgs& a, int fi);
// grid (nf, 2): row 0 parses the tables, row 1 scans the chunk index (it
// re-derives the few header fields it needs, so the two run side by side)
__global__ void __launch_bounds__(1024) parse_kernel(DArgs a) {
  if (blockIdx.y == 0) parse_body(a, (int)blockIdx.x);
  else chunk_offsets_body(a, (int)blockIdx.x);
}
NBZG_DEV void parse_body(const DArgs& a, int fi) {
  const DField& F = a.f[fi];
  DParsed& P = a.parsed[fi];
  uint8_t* lut = reinterpret_cast<uint8_t*>(a.lut) + fi * (1 << kLutBits);
  uint32_t* ss = a.ssyms + fi * a.nbins;
  __shared__ uint32_t s_bad, s_cbl[64], s_max, s_min;
  __shared__ uint32_t scan_tmp[33];
  __shared__ uint64_t s_fc[64];
  __shared__ uint32_t s_fi[64];
  __shared__ uint32_t s_lim16[kLutBits + 1];
  __shared__ uint32_t s_wcnt[32 * 64];  // [warp][length] counters of the canonical ranking
  const int tid = threadIdx.x;
  const uint8_t* p = F.payload;
  const int64_t L = F.payload_len;
  if (tid == 0) {
    s_bad = 0;
    s_max = 0;
    s_min = 255;
  }
  if (tid < 64) s_cbl[tid] = 0;
  for (int i = tid; i < (1 << kLutBits) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(lut)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (L < 8) {
    if (tid == 0) P.status = NBZG_TRUNCATED, fail(a.status, NBZG_TRUNCATED);
    return;
  }
  const uint64_t n_esc = ld_u32_bytes(p), k = ld_u32_bytes(p + 4);
  if (k == 0 || 8 + 5 * k > (uint64_t)L || k > (uint64_t)a.nbins) {
    if (tid == 0) P.status = NBZG_TRUNCATED, fail(a.status, NBZG_TRUNCATED);
    return;
  }
  // validate symbols / lengths
  for (uint64_t i = tid; i < k; i += blockDim.x) {
    const uint8_t* e = p + 8 + 5 * i;
    uint32_t s = ld_u32_bytes(e), l = e[4];
    // v1 codes span [0, interval_count]; v2 codes [0, interval_count-1]
    bool bad = l < 1 || l > kMaxCodeLen || s >= (uint64_t)a.nbins - ((F.kind & 15) == 3 ? 1 : 0);
    if (i > 0 && ld_u32_bytes(e - 5) >= s) bad = true;
    if (bad) atomicOr(&s_bad, 1u);
    else {
      atomicAdd(&s_cbl[l], 1u);
      atomicMax(&s_max, l);
      atomicMin(&s_min, l);
    }
  }
  __syncthreads();
  const int max_len = (int)s_max;
  if (tid == 0 && !s_bad) {
    // Kraft inequality, exact in integers (encode.py:117-120)
    unsigned __int128 kraft = 0;
    for (int l = 1; l <= max_len; l++) kraft += (unsigned __int128)s_cbl[l] << (max_len - l);
    if (kraft > ((unsigned __int128)1 << max_len)) s_bad = 1;
    uint64_t code = 0;
    uint32_t idx = 0;
    for (int l = 1; l <= max_len; l++) {
      s_fc[l] = code;
      s_fi[l] = idx;
      P.first_code[l] = code;
      P.first_idx[l] = idx;
      P.counts[l] = s_cbl[l];
      code = (code + s_cbl[l]) << 1;
      idx += s_cbl[l];
    }
    for (int l = max_len + 1; l < 64; l++) P.counts[l] = 0;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) P.status = NBZG_BAD_STREAM, fail(a.status, NBZG_BAD_STREAM);
    return;
  }
  // canonical order: rank within length class, ascending symbol.  Warp w owns
  // the table entries [w B, (w + 1) B), 32 consecutive ones per round;
  // MATCH.ANY groups the lanes of equal length.  Pass 1 counts per (warp,
  // length), 64 threads scan the warps, pass 2 replays the rounds with the
  // running counters as ranks (same scheme as the encoder's codebook).
  {
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int i = tid; i < 32 * 64; i += blockDim.x) s_wcnt[i] = 0;
    __syncthreads();
    const uint64_t RB = (k + blockDim.x - 1) / blockDim.x;  // rounds per warp
    const uint64_t wbase = (uint64_t)warp * RB * 32;
    for (uint64_t r = 0; r < RB; r++) {
      const uint64_t i = wbase + r * 32 + lane;
      const bool valid = i < k;
      const uint32_t l = valid ? (uint32_t)p[8 + 5 * i + 4] : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      if (valid && (peers & lanemask_lt()) == 0) s_wcnt[warp * 64 + l] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (tid < 64) {
      uint32_t run = 0;
      for (int w = 0; w < nw; w++) {
        const uint32_t c = s_wcnt[w * 64 + tid];
        s_wcnt[w * 64 + tid] = run;
        run += c;
      }
    }
    __syncthreads();
    for (uint64_t r = 0; r < RB; r++) {
      const uint64_t i = wbase + r * 32 + lane;
      const bool valid = i < k;
      const uint32_t l = valid ? (uint32_t)p[8 + 5 * i + 4] : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      const uint32_t lt = peers & lanemask_lt();
      uint32_t rank = 0;
      if (valid) rank = s_wcnt[warp * 64 + l] + __popc(lt);
      __syncwarp();
      if (valid && lt == 0) s_wcnt[warp * 64 + l] += __popc(peers);
      __syncwarp();
      if (valid) ss[s_fi[l] + rank] = ld_u32_bytes(p + 8 + 5 * i);
    }
  }
  // length table: entry e (16-bit prefix) -> smallest l with e.. < limit[l]
  // (canonical order), 0xFE when the code is longer than 16 bits, 0 = invalid.
  // The limits rise with l, so a thread walks its run of consecutive entries
  // with one monotone length cursor and stores 16 entries per instruction.
  if (tid <= kLutBits) {
    const int l = tid;  // s_lim16[l]: first 16-bit prefix past the codes of length <= l
    s_lim16[l] = (l >= 1 && l <= max_len) ? (uint32_t)((s_fc[l] + s_cbl[l]) << (kLutBits - l)) : 0u;
  }
  __syncthreads();
  {
    constexpr int kPer = (1 << kLutBits) / 1024;  // entries per thread (block of 1024)
    static_assert(kPer % 16 == 0, "16 entries per store");
    const int e0 = tid * kPer;
    int l = 1;
    uint4* dst = reinterpret_cast<uint4*>(lut + e0);
#pragma unroll 1
    for (int g = 0; g < kPer / 16; g++) {
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const uint32_t e = (uint32_t)(e0 + 16 * g + j);
        while (l <= max_len && l <= kLutBits && e >= s_lim16[l]) l++;
        const uint32_t len = l > max_len ? 0u : (l > kLutBits ? 0xFEu : (uint32_t)l);
        w[j >> 2] |= len << (8 * (j & 3));
      }
      dst[g] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __syncthreads();  // ss (global) complete for the fused table
  // fused tables for the thread-per-chunk decoder.  Entry: bits 0-5 code
  // length, bit 6 escape, bits 7-31 lattice delta; 64 = unresolved
  // sym - bias.  Primary: 15-bit prefix, codes <= 15 bits.  Secondary: the
  // canonical tail (32-bit window value >= R0, i.e. codes > 15 bits) at W-bit
  // resolution, W <= 24 chosen so the tail fits kTpc2Cap entries.
  if ((F.kind & 15) == 3) {
    int32_t* lut2 = a.lut2 + (size_t)fi * kLut2Stride;
    const int bias = a.half + 1;
    auto entry = [&](int l, uint64_t u) -> int32_t {  // u: 32-bit window value
      const uint32_t idx = s_fi[l] + (uint32_t)((u >> (32 - l)) - s_fc[l]);
      const int sym = (int)ss[idx];
      return sym == 0 ? (int32_t)(l | 64) : (int32_t)(((uint32_t)(sym - bias) << 7) | (uint32_t)l);
    };
    for (int e = tid; e < (1 << kTpcBits); e += blockDim.x) {
      const int l = lut[e << (kLutBits - kTpcBits)];
      lut2[e] = (l >= 1 && l <= kTpcBits) ? entry(l, (uint64_t)e << (32 - kTpcBits)) : 64;
    }
    uint64_t R0 = 1ull << 32;
    int W = 0;
    uint32_t n2 = 0;
    if (max_len > kTpcBits && max_len <= 32) {
      R0 = (s_fc[kTpcBits] + s_cbl[kTpcBits]) << (32 - kTpcBits);
      for (int w = min(max_len, 24); w > kTpcBits; w--) {
        const uint64_t cnt = ((1ull << 32) - R0 + (1ull << (32 - w)) - 1) >> (32 - w);
        // decode_lv_kernel stores only the primary entries below R0, so what
        // the long codes take from the primary table is theirs again
        // (decode_tpc_kernel, sz-lcf, keeps the full primary table)
        const uint64_t room = F.kind == 3
                                  ? min((uint64_t)kTpcTab - (R0 >> (32 - kTpcBits)), (uint64_t)1 << kTpcBits)
                                  : (uint64_t)kTpc2Cap;
        if (cnt <= room) {
          W = w;
          n2 = (uint32_t)cnt;
          break;
        }
      }
    }
    for (uint32_t j = tid; j < n2; j += blockDim.x) {
      const uint64_t u = R0 + ((uint64_t)j << (32 - W));
      int l = 0;
      for (int m = max_len; m > kTpcBits; m--)
        if (u < ((s_fc[m] + s_cbl[m]) << (32 - m))) l = m;
      lut2[(1 << kTpcBits) + j] = (l > 0 && l <= W) ? entry(l, u) : 64;
    }
    if (tid == 0) {
      P.t2_r0 = R0;
      P.t2_w = (uint32_t)W;
      P.t2_n = n2;
      // Share of the symbols the fused tables resolve, estimated from the
      // code lengths (a Huffman code of length l has probability ~2^-l): the
      // codes of <= max(15, W) bits.  One unresolved symbol replays its whole
      // 8-symbol group on the exact path for every lane of the warp.  The
      // canonical mode (symbols by rank in shared memory, three or four
      // dependent lookups per symbol, no replays) costs ~2.5x a clean fused
      // decode; measured at 2^26 particles: coverage 0.9985 -> fused 2.5 ms,
      // canonical 4.5 ms; 0.9971 -> equal (6.9 ms); 0.94 -> fused 13.1 ms,
      // canonical 4.6 ms.
      const int lres = n2 ? max(W, kTpcBits) : kTpcBits;
      double mass = 0.0;
      for (int l = 1; l <= min(max_len, lres); l++) mass += ldexp((double)s_cbl[l], -l);
      P.use_canon = (mass < kCanonMass && k <= (uint64_t)kCanonMaxK && max_len <= 32) ? 1u : 0u;
#ifdef NBZG_CANON_DEBUG
      printf("parse field %d k %llu max_len %d W %d n2 %u resolved mass %.6f canon %u\n", fi,
             (unsigned long long)k, max_len, W, n2, mass, P.use_canon);
#endif
    }
  } else if (tid == 0) {
    P.use_canon = 0;
  }
  if (tid == 0) {
    const uint64_t table_end = 8 + 5 * k;
    const bool has_esc = ld_u32_bytes(p + 8) == 0;  // ascending symbols: 0 is first
    P.esc_len = has_esc ? p[12] : 0;
    P.esc_code = has_esc ? s_fc[p[12]] : 0;
    P.n_esc = n_esc;
    P.k = k;
    P.min_len = s_min;
    P.max_len = s_max;
    uint32_t st = 0;
    if (table_end + 8 > (uint64_t)L) st = NBZG_TRUNCATED;
    else {
      P.total_bits = ld_u64_bytes(p + table_end);
      if ((F.kind & 15) == 3) {  // escapes inline: the bitstream ends the payload
        P.index_off = table_end + 8;
        P.bits_off = (P.index_off + 4 * (uint64_t)a.nchunks + 3) & ~3ull;
        P.esc_off = P.bits_off + 4 * ((P.total_bits + 31) / 32);
        if (P.esc_off != (uint64_t)L) st = NBZG_TRUNCATED;
      } else {
        P.index_off = 0;
        P.bits_off = table_end + 8;
        P.esc_off = P.bits_off + (P.total_bits + 7) / 8;
        if (P.esc_off + 4 * n_esc > (uint64_t)L) st = NBZG_TRUNCATED;  // pipeline.py:213-214
      }
    }
    P.status = st;
    if (st) fail(a.status, st);
  }
}

// ---------------------------------------------------------------- D1: chunk offsets
// Exclusive scan of the v2 chunk index (u32 bit counts, unaligned in the
// payload).  Independent of parse_body: the index position follows from the
// header's symbol count; a malformed header is parse_body's to report.
__device__ void chunk_offsets_body(const DArgs& a, int fi) {
  const DField& F = a.f[fi];
  if ((F.kind & 15) != 3) return;
  const uint8_t* p = F.payload;
  const uint64_t L = (uint64_t)F.payload_len;
  if (L < 8) return;
  const uint64_t k = ld_u32_bytes(p + 4);
  const uint64_t table_end = 8 + 5 * k;
  if (k == 0 || k > (uint64_t)a.nbins || table_end + 8 + 4 * (uint64_t)a.nchunks > L) return;
  const uint64_t total_bits = ld_u64_bytes(p + table_end);
  __shared__ unsigned long long scan_tmp[33];
  const uint8_t* idx = p + table_end + 8;
  uint64_t* off = a.choff + fi * (a.nchunks + 1);
  const int R = (int)((a.nchunks + blockDim.x - 1) / blockDim.x);
  constexpr int kReg = 16;  // index entries per thread held in registers
  uint32_t v[kReg];
  unsigned long long s = 0;
  if (R <= kReg) {
#pragma unroll
    for (int r = 0; r < kReg; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      v[r] = (r < R && c < a.nchunks) ? ld_u32_bytes(idx + 4 * c) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kReg; r++) s += v[r];
  } else {
    for (int r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) s += ld_u32_bytes(idx + 4 * c);
    }
  }
  unsigned long long tot;
  unsigned long long ex = block_excl_scan<unsigned long long>(s, scan_tmp, &tot);
  if (R <= kReg) {
#pragma unroll
    for (int r = 0; r < kReg; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (r < R && c < a.nchunks) off[c] = ex;
      ex += v[r];
    }
  } else {
    for (int r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) {
        off[c] = ex;
        ex += ld_u32_bytes(idx + 4 * c);
      }
    }
  }
  if (threadIdx.x == 0) {
    off[a.nchunks] = tot;
    if (tot != total_bits) fail(a.status, NBZG_BAD_STREAM);
  }
}

// ---------------------------------------------------------------- decode step
// MSB-first bit reader: two current words + one prefetched raw word; a
// 32-bit window is one funnel shift, a refill never waits on its own load.
struct BitReader {
  const uint4* g4;   // 16-byte aligned view of the stream
  uint32_t w0, w1;   // current words (byte-swapped)
  uint4 qa;          // next raw words, consumed from .x; nq of them valid
  uint4 qb;          // the next aligned uint4, already in flight
  uint32_t nq;
  uint32_t off;      // bit offset into w0 (0..31)
  uint32_t vi;       // next uint4 index to load
};

NBZG_DEV uint32_t bswap32(uint32_t w) { return __byte_perm(w, 0, 0x0123); }

// pos: bit position relative to the 16-byte aligned base
NBZG_DEV void br_init(BitReader& R, const uint4* g4, uint64_t pos) {
  const uint32_t w = (uint32_t)(pos >> 5);  // word index
  const uint32_t* g = reinterpret_cast<const uint32_t*>(g4);
  R.g4 = g4;
  R.off = (uint32_t)(pos & 31);
  R.w0 = bswap32(__ldg(g + w));
  R.w1 = bswap32(__ldg(g + w + 1));
  const uint32_t n = w + 2, v = n >> 2, s = n & 3;
  uint4 A = __ldg(g4 + v);
  if (s == 1) A = make_uint4(A.y, A.z, A.w, 0u);
  else if (s == 2) A = make_uint4(A.z, A.w, 0u, 0u);
  else if (s == 3) A = make_uint4(A.w, 0u, 0u, 0u);
  R.qa = A;
  R.nq = 4 - s;
  R.qb = __ldg(g4 + v + 1);
  R.vi = v + 2;
}
NBZG_DEV uint32_t br_peek(const BitReader& R) { return __funnelshift_l(R.w1, R.w0, R.off); }
// predicated in-place 16-byte load: the destination registers ARE the
// queue slot, so no register copy waits on the load (a plain conditional
// load makes the compiler merge the result with a move right after it).
NBZG_DEV void ldg_v4_if(uint4& q, const uint4* p, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n"
      " @p ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%5];\n}\n"
      : "+r"(q.x), "+r"(q.y), "+r"(q.z), "+r"(q.w)
      : "r"((uint32_t)pred), "l"(p));
}
NBZG_DEV void ldg_v8_if_l2(uint4& q, uint4& r, const uint4* p, bool pred) {  // 32 bytes per lane
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %8, 0;\n"
      " @p ld.global.nc.L2::256B.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%9];\n}\n"
      : "+r"(q.x), "+r"(q.y), "+r"(q.z), "+r"(q.w), "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "r"((uint32_t)pred), "l"(p));
}
NBZG_DEV void ldg_v4_if_l2(uint4& q, const uint4* p, bool pred) {  // 256-byte L2 fill on a miss
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n"
      " @p ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%5];\n}\n"
      : "+r"(q.x), "+r"(q.y), "+r"(q.z), "+r"(q.w)
      : "r"((uint32_t)pred), "l"(p));
}
NBZG_DEV void br_skip(BitReader& R, uint32_t l) {  // l <= 32
  R.off += l;
  const bool adv = R.off >= 32;
  bool refill = false;
  if (adv) {
    R.off -= 32;
    R.w0 = R.w1;
    R.w1 = bswap32(R.qa.x);
    R.qa.x = R.qa.y;
    R.qa.y = R.qa.z;
    R.qa.z = R.qa.w;
    refill = --R.nq == 0;
    if (refill) {
      R.qa = R.qb;
      R.nq = 4;
    }
  }
  ldg_v4_if(R.qb, R.g4 + R.vi, refill);
  R.vi += refill ? 1u : 0u;
}

// segmented (reset, k) scan element: a later reset wins, otherwise values add
struct KSeg {
  int r;
  long long v;
};
NBZG_DEV KSeg kseg_op(KSeg a, KSeg b) { return b.r ? b : KSeg{a.r, a.v + b.v}; }

NBZG_DEV long long esc_k(float v, const DField& F) {
  bool fast;
  double kd = lattice_index<false>(v, F.inv32, F.inv, F.twob, fast);
  if (!fast) kd = fmin(fmax(kd, -kDqKmax), kDqKmax);
  return (long long)kd;
}

// Decode symbols from `pos` until the position reaches `stop`: counts
// codewords and accumulates the segmented lattice sum.  Returns the end
// position (first codeword start >= stop), or ~0 on an invalid code.
struct WalkOut {
  uint64_t end;
  uint32_t cnt;
  KSeg agg;
  uint64_t last_reset;  // position of the last escape codeword (or 0)
};

// bit-serial canonical decode of one symbol straight from global bytes
// (v1 compat path and pathological > 32-bit codes).
NBZG_DEV int decode_serial(const uint8_t* bits, uint64_t& bp, uint64_t total, const DParsed& P,
                           const uint32_t* ss, uint32_t& sym) {
  uint64_t code = 0;
  int len = 0;
  while (true) {
    if (bp >= total) return -NBZG_TRUNCATED;
    uint32_t bit = (bits[bp >> 3] >> (7 - (bp & 7))) & 1u;
    bp++;
    code = (code << 1) | bit;
    len++;
    if (len > (int)P.max_len) return -NBZG_INVALID_CODE;
    if (len >= (int)P.min_len && P.counts[len] > 0) {
      uint64_t fc = P.first_code[len];
      if (code >= fc && code - fc < P.counts[len]) {
        sym = ss[P.first_idx[len] + (uint32_t)(code - fc)];
        return len;
      }
    }
  }
}

// ---------------------------------------------------------------- D2: decode
template <bool SMALL_K>
NBZG_DEV uint32_t sym_of(uint32_t v, int l, const int32_t* base, const uint16_t* SS,
                         const uint32_t* ss) {
  uint32_t idx = (uint32_t)(base[l] + (int32_t)(v >> (32 - l)));
  return SMALL_K ? (uint32_t)SS[idx] : __ldg(ss + idx);
}

// one decode step shared by all phases: returns bits consumed (0 = invalid);
// escapes (symbol 0) consume their inline 32-bit value and reset the sum
template <bool SMALL_K>
NBZG_DEV uint32_t dstep(BitReader& R, const uint8_t* LL, const uint64_t* limit,
                        const int32_t* base, const uint16_t* SS, const uint32_t* ss,
                        int max_len, int bias, const DField& F, KSeg& agg, uint32_t& sym,
                        float& ev) {
  uint32_t v = br_peek(R);
  int l = LL[v >> (32 - kLutBits)];
  if (l >= 0xFE) {
    int r = 0;
#pragma unroll 1
    for (int len = max_len; len > kLutBits; len--) r = ((uint64_t)v < limit[len]) ? len : r;
    l = r;
    if (l == 0) return 0;
  }
  sym = sym_of<SMALL_K>(v, l, base, SS, ss);
  br_skip(R, (uint32_t)l);
  if (sym == 0) {
    ev = __uint_as_float(br_peek(R));
    br_skip(R, 32);
    agg = KSeg{1, esc_k(ev, F)};
    return (uint32_t)l + 32;
  }
  agg.v += (long long)((int)sym - bias);
  return (uint32_t)l;
}

template <bool SMALL_K>
__global__ void __launch_bounds__(kDThreads, 1) decode_kernel(DArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* LL = smem;                                                  // [1 << kLutBits]
  uint16_t* SS = reinterpret_cast<uint16_t*>(smem + (1 << kLutBits));  // [kSmemSyms]
  __shared__ uint64_t s_limit[64];
  __shared__ int32_t s_base[64];
  __shared__ int s_next;

  const int fi = blockIdx.x % a.nf;
  const int grp = blockIdx.x / a.nf, ngrp = gridDim.x / a.nf;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if (F.kind != 3 || P.status || *a.status || P.max_len > 32) return;
  if (SMALL_K != (P.k <= (uint64_t)kSmemSyms)) return;
  const int64_t cb = (a.nchunks * grp) / ngrp, ce = (a.nchunks * (grp + 1)) / ngrp;
  if (cb >= ce) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t* ss = a.ssyms + fi * a.nbins;

  // ---- stage the decode tables once per CTA
  {
    const uint4* gl = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(a.lut) +
                                                     (size_t)fi * (1 << kLutBits));
    uint4* sl = reinterpret_cast<uint4*>(LL);
    for (int i = tid; i < (1 << kLutBits) / 16; i += kDThreads) sl[i] = gl[i];
  }
  if (SMALL_K)
    for (uint32_t i = tid; i < (uint32_t)P.k; i += kDThreads) SS[i] = (uint16_t)ss[i];
  if (tid < 64) {
    const int l = tid;
    uint64_t lim = 0;
    int32_t bs = 0;
    if (l >= 1 && l <= 32 && l <= (int)P.max_len) {
      lim = (P.first_code[l] + P.counts[l]) << (32 - l);
      bs = (int32_t)P.first_idx[l] - (int32_t)P.first_code[l];
    }
    s_limit[l] = l > (int)P.max_len ? ~0ull : lim;
    s_base[l] = bs;
  }
  if (tid == 0) s_next = (int)cb;
  __syncthreads();

  const uintptr_t bits_addr = reinterpret_cast<uintptr_t>(F.payload + P.bits_off);
  const uint4* G = reinterpret_cast<const uint4*>(bits_addr & ~uintptr_t(15));
  const uint32_t a0 = (uint32_t)(bits_addr & 15) * 8;
  const uint64_t* choff = a.choff + fi * (a.nchunks + 1);
  const int bias = a.half + 1;
  const int max_len = (int)P.max_len;

#define DSTEP(R, agg, sym, ev) \
  dstep<SMALL_K>(R, LL, s_limit, s_base, SS, ss, max_len, bias, F, agg, sym, ev)

  while (true) {
    int c32 = 0;
    if (lane == 0) c32 = atomicAdd(&s_next, 1);
    const int64_t c = __shfl_sync(0xffffffffu, c32, 0);
    if (c >= ce) break;
    const uint64_t B = choff[c];
    const uint32_t Tb = (uint32_t)(choff[c + 1] - B);
    const int64_t c0 = c * kChunk;
    const int mc = (int)min((int64_t)kChunk, a.n - c0);
    // lane slice [rs0, rs1), chunk-relative bit positions (< 2^32)
    const uint32_t rs0 = (uint32_t)(((uint64_t)Tb * lane) / 32);
    const uint32_t rs1 = (uint32_t)(((uint64_t)Tb * (lane + 1)) / 32);
    int err = 0;

    // ---- phase 1: full decode from an arbitrary start (count + lattice sum),
    // remembering checkpoints after 16, 32, 48, 64 codewords
    constexpr int kCp = 4;
    uint32_t cp_pos[kCp], cp_cnt[kCp];
    long long cp_v[kCp];
    int ncp = 0;
    uint32_t cnt = 0, next_cp = 16;
    KSeg agg{0, 0};
    uint32_t last_reset = 0;  // 1 + position of the last escape codeword (0: none)
    uint32_t end;
    {
      BitReader R;
      br_init(R, G, a0 + B + rs0);
      uint32_t pos = rs0;
      while (__any_sync(0xffffffffu, pos < rs1)) {
        if (pos < rs1) {
          if (cnt >= next_cp) {
            if (ncp < kCp) {
#pragma unroll
              for (int j = 0; j < kCp; j++)
                if (j == ncp) {
                  cp_pos[j] = pos;
                  cp_cnt[j] = cnt;
                  cp_v[j] = agg.v;
                }
              ncp++;
            }
            next_cp += 16;
          }
          uint32_t sym;
          float ev;
          uint32_t l = DSTEP(R, agg, sym, ev);
          if (l == 0) {  // garbage from a wrong start (incomplete codes): step a bit
            pos += 1;
            br_init(R, G, a0 + B + pos);
          } else {
            if (sym == 0) last_reset = pos + 1;
            pos += l;
            cnt++;
          }
        }
      }
      end = pos;
    }
    // ---- phase 2: lane l re-walks from lane l-1's end (its true start once
    // l-1 is synchronised) until it meets one of its checkpoints, then
    // splices the phase-1 totals; lanes that never meet one redo the slice.
    uint32_t start = rs0;
    for (int iter = 0; iter < 33; iter++) {
      uint32_t s = __shfl_up_sync(0xffffffffu, end, 1);
      if (lane == 0) s = 0;
      const bool redo = (s != start) && !err;
      bool active = redo;
      bool changed = false;
      BitReader R;
      br_init(R, G, a0 + B + (active ? s : rs0));
      uint32_t q = s;
      uint32_t steps = 0;
      KSeg wagg{0, 0};
      uint32_t wlast = 0;
      int hit = -1;
      bool full = false;  // past the last checkpoint: walking the whole slice
      while (__any_sync(0xffffffffu, active)) {
        if (active) {
          if (!full) {
#pragma unroll
            for (int j = 0; j < kCp; j++)
              if (j < ncp && cp_pos[j] == q) hit = j;
            if (hit < 0 && (ncp == 0 || q > cp_pos[ncp - 1])) full = true;
          }
          if (hit >= 0 || q >= rs1) {
            active = false;
          } else {
            uint32_t sym;
            float ev;
            uint32_t l = DSTEP(R, wagg, sym, ev);
            if (l == 0) {
              err = NBZG_INVALID_CODE;
              active = false;
            } else {
              if (sym == 0) wlast = q + 1;
              q += l;
              steps++;
            }
          }
        }
      }
      if (redo) {
        if (hit >= 0) {
          uint32_t hc = 0, hp = 0;
          long long hv = 0;
#pragma unroll
          for (int j = 0; j < kCp; j++)
            if (j == hit) {
              hc = cp_cnt[j];
              hp = cp_pos[j];
              hv = cp_v[j];
            }
          // phase-1 suffix from the checkpoint: a reset after it wins
          KSeg suf = (last_reset > hp) ? KSeg{1, agg.v} : KSeg{0, agg.v - hv};
          cnt = steps + (cnt - hc);
          agg = kseg_op(wagg, suf);
          last_reset = (last_reset > hp) ? last_reset : wlast;
        } else if (!err) {
          cnt = steps;
          agg = wagg;
          last_reset = wlast;
          if (q != end) changed = true;
          end = q;
        }
        ncp = 0;  // checkpoints before the splice point are stale
        start = s;
      }
      if (!__any_sync(0xffffffffu, changed)) break;
    }

    // ---- offsets, incoming lattice index, validation
    uint32_t o = warp_incl_scan<uint32_t>(cnt) - cnt;
    uint32_t tot = __shfl_sync(0xffffffffu, o + cnt, 31);
    KSeg inc = agg;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      KSeg u;
      u.r = __shfl_up_sync(0xffffffffu, inc.r, dd);
      u.v = __shfl_up_sync(0xffffffffu, inc.v, dd);
      if (lane >= dd) inc = kseg_op(u, inc);
    }
    long long k = __shfl_up_sync(0xffffffffu, inc.v, 1);
    if (lane == 0) k = 0;  // chunk start: k_{-1} = 0, so the prefix value is the index
    uint32_t last_end = __shfl_sync(0xffffffffu, end, 31);
    err = (int)__reduce_max_sync(0xffffffffu, (unsigned)err);
    if (!err && (tot != (uint32_t)mc || last_end != Tb))
      err = tot < (uint32_t)mc ? NBZG_TRUNCATED : NBZG_BAD_STREAM;
    if (err) {
      if (lane == 0) fail(a.status, (uint32_t)err);
      continue;
    }

    // ---- phase 3: decode from the true start and write
    {
      uint32_t s = __shfl_up_sync(0xffffffffu, end, 1);
      if (lane == 0) s = 0;
      BitReader R;
      br_init(R, G, a0 + B + s);
      float* dst = F.out + c0 + o;
      const double twob = F.twob;
      const uint32_t maxcnt = __reduce_max_sync(0xffffffffu, cnt);
      for (uint32_t i = 0; i < maxcnt; i++) {
        if (i < cnt) {
          uint32_t v = br_peek(R);
          int l = LL[v >> (32 - kLutBits)];
          if (l >= 0xFE) {
            int r = 0;
#pragma unroll 1
            for (int len = max_len; len > kLutBits; len--)
              r = ((uint64_t)v < s_limit[len]) ? len : r;
            l = r;
          }
          uint32_t sym = sym_of<SMALL_K>(v, l, s_base, SS, ss);
          br_skip(R, (uint32_t)l);
          float outv;
          if (sym == 0) {
            outv = __uint_as_float(br_peek(R));
            br_skip(R, 32);
            k = esc_k(outv, F);
          } else {
            k += (long long)((int)sym - bias);
            outv = (float)__dmul_rn((double)k, twob);
          }
          dst[i] = outv;
        }
      }
    }
  }
#undef DSTEP
}

// ---------------------------------------------------------------- D2': thread per chunk
// When a field has many chunks (>= kTpcMinChunks) every THREAD decodes one
// whole chunk serially: no resynchronisation and one pass over the bits
// instead of the warp decoder's two and a half.  The fused 2^15-entry table
// (128 KiB of shared memory) turns a common step into one LDS: peek 32 bits,
// look up (delta, length), add the delta to the lattice index, write
// f32(k * 2b).  Outputs are buffered 8 at a time and written as two 16-byte
// stores (one full sector per lane).  Escapes and codes longer than 15 bits
// take the canonical slow path (limits + symbol table, also in smem).
// A thread's chunk takes ~1.4-3 ms whatever the input size, the warp decoder's
// time grows with n: measured crossover (scripts/path_crossover.py, HACC-like
// slabs, eb 1e-4) between 1536 and 2048 chunks per field (1024: 1.24 vs
// 2.09 ms, 2048: 2.30 vs 2.04 ms).
constexpr int kTpcMinChunks = 1792;

// Per-lane bit reader of the thread-per-chunk decoder.  The window (w0, w1)
// lives in registers; the words after it come from an 8-word ring per lane
// in shared memory (word-major, so lanes never conflict).  Refills happen
// only at 8-symbol group boundaries: the 16-byte block loaded at the
// previous boundary is stored into the ring and the next block's load is
// issued.  A register that is the target of an in-flight load is therefore
// read once per group, 8 symbols after its load was issued -- never inside
// the decode step (the register scoreboard is per warp: a per-step refill
// by any lane would stall every lane).  A lane that outruns its ring reads
// the word straight from global memory (rare: > 4 words in 8 symbols).
struct TpcReader {
  uint32_t w0, w1, off;  // window: bits [off, off+32) of w0:w1
  uint32_t wi;           // stream word index of w1
  uint32_t wr;           // first stream word not in the ring (multiple of 4)
  uint4 qs;              // block wr/4, loaded at the last boundary
};

// one 32-byte streaming store (sm_100 256-bit STG): a whole sector per lane
NBZG_DEV void st_v8_cs(float* p, const float (&o)[8]) {
#ifdef NBZG_DEC_NOSTORE  // timing experiment only: values consumed, nothing stored
  float s = ((o[0] + o[1]) + (o[2] + o[3])) + ((o[4] + o[5]) + (o[6] + o[7]));
  if (s == 1234.5678f) *p = s;
#else
  asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(o[0]),
               "f"(o[1]), "f"(o[2]), "f"(o[3]), "f"(o[4]), "f"(o[5]), "f"(o[6]), "f"(o[7])
               : "memory");
#endif
}

NBZG_DEV void tpc_init(TpcReader& R, const uint4* G, uint32_t* ring, int nthr, uint64_t bitpos,
                       uint32_t vmax) {
  const uint32_t gw0 = (uint32_t)(bitpos >> 5);
  const uint32_t blk = gw0 >> 2;
  const uint4 A = ldg_l2fill(G + min(blk, vmax)), B = ldg_l2fill(G + min(blk + 1, vmax));
  const uint32_t s0 = (4 * blk) & 7, s1 = s0 ^ 4;  // word 4 blk + i -> slot (4 blk + i) & 7
  ring[(s0 + 0) * nthr] = bswap32(A.x);  // words stored byte-swapped
  ring[(s0 + 1) * nthr] = bswap32(A.y);
  ring[(s0 + 2) * nthr] = bswap32(A.z);
  ring[(s0 + 3) * nthr] = bswap32(A.w);
  ring[(s1 + 0) * nthr] = bswap32(B.x);
  ring[(s1 + 1) * nthr] = bswap32(B.y);
  ring[(s1 + 2) * nthr] = bswap32(B.z);
  ring[(s1 + 3) * nthr] = bswap32(B.w);
  R.off = (uint32_t)(bitpos & 31);
  R.w0 = ring[(gw0 & 7) * nthr];
  R.w1 = ring[((gw0 + 1) & 7) * nthr];
  R.wi = gw0 + 1;
  R.wr = 4 * (blk + 2);
  R.qs = make_uint4(0, 0, 0, 0);
  ldg_v4_if_l2(R.qs, G + min(blk + 2, vmax), true);
}

// consume l <= 32 bits.  The next ring word is read unconditionally (its
// address depends only on wi, so the load overlaps the table lookup) and the
// window advances through selects; only a lane that outran its ring takes
// the branch to global memory.
NBZG_DEV void tpc_skip(TpcReader& R, uint32_t l, const uint32_t* ring, int nthr,
                       const uint32_t* G32, uint32_t wmax, uint32_t nw) {
  R.off += l;
  const bool cross = R.off >= 32;
  if (cross && (int32_t)(R.wr - (R.wi + 1)) <= 0) {  // outran the ring (rare)
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(nw) : "l"(G32 + min(R.wi + 1, wmax)));
    nw = bswap32(nw);
  }
  R.w0 = cross ? R.w1 : R.w0;
  R.w1 = cross ? nw : R.w1;
  R.wi += cross ? 1u : 0u;
  R.off -= cross ? 32u : 0u;
}
NBZG_DEV uint32_t tpc_next(const TpcReader& R, const uint32_t* ring, int nthr) {
  return ring[((R.wi + 1) & 7) * nthr];
}

NBZG_DEV void tpc_refill(TpcReader& R, uint32_t* ring, int nthr, const uint4* G, uint32_t vmax) {
  const bool room = (int32_t)(R.wr - R.wi) <= 5;
  if (room) {
    const uint32_t s = R.wr & 7;  // 0 or 4
    ring[(s + 0) * nthr] = bswap32(R.qs.x);
    ring[(s + 1) * nthr] = bswap32(R.qs.y);
    ring[(s + 2) * nthr] = bswap32(R.qs.z);
    ring[(s + 3) * nthr] = bswap32(R.qs.w);
    R.wr += 4;
  }
  ldg_v4_if_l2(R.qs, G + min(R.wr >> 2, vmax), room);
}

// Lattice-index state of one chunk.  LV: k_i = k_{i-1} + q_i, kept in FP64
// (exact: |k| <= 2^52).  LCF (sz-lcf): k_i = q_i + 2 k_{i-1} - k_{i-2} with
// pred_1 = k_0 (both history slots hold k_0 after the first symbol), int64.
template <bool LCF>
struct KState;
template <>
struct KState<false> {
  double kd = 0.0;
  NBZG_DEV float apply(int32_t q, double twob) {
    kd += (double)q;
    return (float)__dmul_rn(kd, twob);
  }
  NBZG_DEV void escape(long long k) { kd = (double)k; }
};
template <>
struct KState<true> {
  long long k1 = 0, k2 = 0;
  bool first = true;
  NBZG_DEV void push(long long k) {
    k2 = first ? k : k1;
    k1 = k;
    first = false;
  }
  NBZG_DEV float apply(int32_t q, double twob) {
    const long long k = (long long)q + 2 * k1 - k2;
    push(k);
    return (float)__dmul_rn((double)k, twob);
  }
  NBZG_DEV void escape(long long k) { push(k); }
};

template <bool LCF>
__global__ void __launch_bounds__(kTpcMaxThreads, 1) decode_tpc_kernel(DArgs a, int ctas_per_field) {
  extern __shared__ __align__(16) uint8_t dsm2[];
  int32_t* LT = reinterpret_cast<int32_t*>(dsm2);  // [2^15 + t2_n]
  __shared__ uint64_t s_limit[64];
  __shared__ int32_t s_base[64];
  const int fi = blockIdx.y;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if (F.kind != (LCF ? 3 + NBZG_KIND_LCF : 3) || P.status || *a.status || P.max_len > 32) return;
  const int64_t cb = (a.nchunks * blockIdx.x) / ctas_per_field;
  const int64_t ce = (a.nchunks * (blockIdx.x + 1)) / ctas_per_field;
  if (cb >= ce) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  uint32_t* ring = reinterpret_cast<uint32_t*>(dsm2 + 4 * kTpcTab) + tid;  // [8][kRingStride]
  const uint32_t* ss = a.ssyms + fi * a.nbins;
  const uint32_t n2 = P.t2_n;
  {
    const int32_t* gl = a.lut2 + (size_t)fi * kLut2Stride;
    const uint32_t nv = ((1u << kTpcBits) + n2 + 3) / 4;
    for (uint32_t i = tid; i < nv; i += nthr)
      reinterpret_cast<uint4*>(LT)[i] = __ldg(reinterpret_cast<const uint4*>(gl) + i);
  }
  if (tid < 64) {
    const int l = tid;
    uint64_t lim = 0;
    int32_t bs = 0;
    if (l >= 1 && l <= 32 && l <= (int)P.max_len) {
      lim = (P.first_code[l] + P.counts[l]) << (32 - l);
      bs = (int32_t)P.first_idx[l] - (int32_t)P.first_code[l];
    }
    s_limit[l] = l > (int)P.max_len ? ~0ull : lim;
    s_base[l] = bs;
  }
  __syncthreads();

  const uintptr_t bits_addr = reinterpret_cast<uintptr_t>(F.payload + P.bits_off);
  const uint4* G = reinterpret_cast<const uint4*>(bits_addr & ~uintptr_t(15));
  const uint32_t* G32 = reinterpret_cast<const uint32_t*>(G);
  const uint32_t a0 = (uint32_t)(bits_addr & 15) * 8;
  // last 16-byte block / word the stream may touch (payload + 64-byte slack)
  const uint32_t vmax = (uint32_t)((a0 / 8 + 4 * ((P.total_bits + 31) / 32) + 16) / 16);
  const uint32_t wmax = 4 * vmax + 3;
  const uint64_t* choff = a.choff + fi * (a.nchunks + 1);
  const int bias = a.half + 1;
  const int max_len = (int)P.max_len;
  const double twob = F.twob;
  const bool vec = (reinterpret_cast<uintptr_t>(F.out) & 31) == 0;  // 32-byte stores
  const uint32_t r0 = (uint32_t)min(P.t2_r0, (uint64_t)0xFFFFFFFFu);
  const uint32_t sh2 = 32u - P.t2_w;
  const int32_t* LT2 = LT + (1 << kTpcBits);
  const uint32_t n2m1 = n2 ? n2 - 1 : 0;

  for (int64_t c = cb + tid; c < ce; c += nthr) {
    const uint64_t b0 = choff[c];
    const uint64_t Tb = choff[c + 1] - b0;
    const int64_t i0 = c * kChunk;
    const int mc = (int)min((int64_t)kChunk, a.n - i0);
    const uint64_t B = a0 + b0;
    TpcReader R;
    tpc_init(R, G, ring, kRingStride, B, vmax);
    KState<LCF> ks;
    int err = 0;
    float* dst = F.out + i0;
    // bits consumed so far
    auto consumed = [&]() -> uint64_t { return ((uint64_t)(R.wi - 1) << 5) + R.off - B; };
    // canonical decode of the symbol at the window (any length <= 32):
    // returns the fused entry (length | escape flag | delta)
    auto resolve = [&](uint32_t v) -> int32_t {
      int32_t e = LT[v >> (32 - kTpcBits)];
      if ((e & 63) == 0) {
        const uint32_t j = (v - r0) >> sh2;
        e = (v >= r0 && j < n2) ? LT2[j] : 0;
        if ((e & 63) == 0) {
          int r = 0;
#pragma unroll 1
          for (int len = max_len; len >= 1; len--) r = ((uint64_t)v < s_limit[len]) ? len : r;
          if (r == 0) {
            err = NBZG_INVALID_CODE;
            e = 1;
          } else {
            const uint32_t sym = __ldg(ss + (uint32_t)(s_base[r] + (int32_t)(v >> (32 - r))));
            e = sym == 0 ? (r | 64) : (int32_t)(((uint32_t)((int)sym - bias) << 7) | (uint32_t)r);
          }
        }
      }
      return e;
    };
    // exact step (ring or global words): escapes, slow codes, replays, tails
    auto safe_step = [&](float& o) {
      const int32_t e = resolve(__funnelshift_l(R.w1, R.w0, R.off));
      const uint32_t l = (uint32_t)e & 63u;
      if (e & 64) {
        tpc_skip(R, l, ring, kRingStride, G32, wmax, tpc_next(R, ring, kRingStride));
        o = __uint_as_float(__funnelshift_l(R.w1, R.w0, R.off));
        ks.escape(esc_k(o, F));
        tpc_skip(R, 32, ring, kRingStride, G32, wmax, tpc_next(R, ring, kRingStride));
      } else {
        o = ks.apply(e >> 7, twob);
        tpc_skip(R, l, ring, kRingStride, G32, wmax, tpc_next(R, ring, kRingStride));
      }
    };
    // common step: table hit (primary or secondary), no escape; the window
    // advances from the ring speculatively and `under` records a lane that
    // needed a word the ring did not hold yet (the group is then replayed)
    auto fast_step = [&](float& o) {
      const uint32_t v = __funnelshift_l(R.w1, R.w0, R.off);
      const uint32_t nw = tpc_next(R, ring, kRingStride);
      int32_t e = LT[v >> (32 - kTpcBits)];
      const uint32_t j = min((v - r0) >> sh2, n2m1);
      const int32_t e2 = LT2[j];
      if ((e & 63) == 0) e = (v >= r0 && ((v - r0) >> sh2) < n2) ? e2 : 0;
      if ((uint32_t)((e & 127) - 1) >= 63u) {  // unresolved (length 0) or escape
        safe_step(o);
        return;
      }
      o = ks.apply(e >> 7, twob);
      R.off += (uint32_t)e & 63u;
      const bool cross = R.off >= 32;
      R.w0 = cross ? R.w1 : R.w0;
      R.w1 = cross ? nw : R.w1;
      R.wi += cross ? 1u : 0u;
      R.off -= cross ? 32u : 0u;
    };
    // 8 symbols; replayed exactly if any window word came from past the ring
    auto group = [&](float (&o)[8]) {
      const TpcReader S = R;
      const KState<LCF> ks0 = ks;
#pragma unroll
      for (int q = 0; q < 8; q++) fast_step(o[q]);
      // the largest word index read in the group is the final wi
      if ((int32_t)(R.wr - R.wi) <= 0) {
        R = S;
        ks = ks0;
#pragma unroll 1
        for (int q = 0; q < 8; q++) {
          float t;
          safe_step(t);
#pragma unroll
          for (int u = 0; u < 8; u++) o[u] = (u == q) ? t : o[u];
        }
      }
      tpc_refill(R, ring, kRingStride, G, vmax);
    };
    int i = 0;
    if (vec) {
      // two register sets: a set's 16-byte stores are issued one group
      // before the set is rewritten (pinned live meanwhile), so the decode
      // never waits for the store queue to read its source registers
      float oa[8], ob[8];
#pragma unroll
      for (int u = 0; u < 8; u++) ob[u] = 0.0f;
      for (; i + 16 <= mc; i += 16) {
        group(oa);
        asm volatile("" ::"f"(ob[0]), "f"(ob[1]), "f"(ob[2]), "f"(ob[3]), "f"(ob[4]),
                     "f"(ob[5]), "f"(ob[6]), "f"(ob[7]));
        st_v8_cs(dst + i, oa);
        group(ob);
        asm volatile("" ::"f"(oa[0]), "f"(oa[1]), "f"(oa[2]), "f"(oa[3]), "f"(oa[4]),
                     "f"(oa[5]), "f"(oa[6]), "f"(oa[7]));
        st_v8_cs(dst + i + 8, ob);
        if (consumed() > Tb) break;  // corrupt: stop early, reported below
      }
    }
    for (; i < mc && consumed() <= Tb; i++) {
      float o;
      safe_step(o);
      if ((i & 7) == 7) tpc_refill(R, ring, kRingStride, G, vmax);
      dst[i] = o;
    }
    const uint64_t pos = consumed();
    if (!err && pos != Tb) err = pos > Tb ? NBZG_TRUNCATED : NBZG_BAD_STREAM;
    if (err) fail(a.status, (uint32_t)err);
  }
}

// ---------------------------------------------------------------- D2'': LV thread per chunk, 64-bit buffer
// The sz-lv / sz-lv-prx decoder.  Same work split, tables and ring as
// decode_tpc_kernel, but a shorter dependent chain per symbol: the next bits
// sit left-aligned in a 64-bit register buffer (hi:lo), so a step is
//   lookup(hi) -> l -> hi:lo <<= l
// with the long-code table read speculatively beside the primary one (no
// branch), one buffer refill from the ring per symbol PAIR (>= 32 valid bits
// before an even symbol, an odd one checks l <= cnt), and the lattice index
// accumulated in int64 as the oracle does (orc_dq_dequantize_p).  Anything
// the fast step cannot take -- escape, unresolved code, too few buffered
// bits, a ring word not yet loaded -- marks the lane and its 8-symbol group
// is replayed with exact steps from the saved state.  Stream blocks are read
// with a 256-byte L2 fill hint: one DRAM burst serves a lane's next 16
// refills (the 96000 per-chunk streams otherwise miss L2 one sector at a
// time; -7% kernel time at C2).
struct BufReader {
  uint32_t hi, lo;  // next stream bits, MSB first (bit 31 of hi is the next bit)
  uint32_t cnt;     // valid bits in hi:lo (the bits after them are zero)
  uint32_t wi;      // next stream word to enter the buffer
  uint32_t wr;      // first stream word not in the ring (multiple of 4)
  uint4 qs;         // block wr/4, loaded at the last refill
#if NBZG_LV_RING == 16
  uint4 qs2;        // block wr/4 + 1
#endif
};

NBZG_DEV uint32_t shl_c(uint32_t x, uint32_t s) {  // s >= 32 -> 0
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
NBZG_DEV uint32_t shr_c(uint32_t x, uint32_t s) {  // s >= 32 -> 0
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
NBZG_DEV void bb_take(BufReader& R, uint32_t l) {  // l <= 32
  R.hi = __funnelshift_lc(R.lo, R.hi, l);
  R.lo = shl_c(R.lo, l);
  R.cnt -= l;
}
NBZG_DEV void bb_fill(BufReader& R, uint32_t nw) {  // cnt <= 32
  R.hi |= shr_c(nw, R.cnt);
  R.lo |= shl_c(nw, 32u - R.cnt);
  R.cnt += 32;
  R.wi += 1;
}
NBZG_DEV void ring_put(uint32_t* ring, uint32_t s, const uint4& q) {
  ring[(s + 0) * kLvStride] = bswap32(q.x);
  ring[(s + 1) * kLvStride] = bswap32(q.y);
  ring[(s + 2) * kLvStride] = bswap32(q.z);
  ring[(s + 3) * kLvStride] = bswap32(q.w);
}
#if NBZG_LV_RING == 16
// 16-word ring refilled 8 words at a time: one 32-byte load per lane (half
// the L1 wavefronts of 16-byte loads) that has several groups to land.
// Stream blocks are 32-byte aligned here: G8 = the 32-byte block index.
NBZG_DEV void bb_init(BufReader& R, const uint4* G, uint32_t* ring, uint64_t bitpos,
                      uint32_t vmax) {
  const uint32_t gw0 = (uint32_t)(bitpos >> 5);
  const uint32_t blk = gw0 >> 3;  // 8-word block
  const uint32_t v8 = vmax >> 1;
  uint4 A0 = make_uint4(0, 0, 0, 0), A1 = A0, B0 = A0, B1 = A0;
  ldg_v8_if_l2(A0, A1, G + 2 * min(blk, v8), true);
  ldg_v8_if_l2(B0, B1, G + 2 * min(blk + 1, v8), true);
  const uint32_t s0 = (8 * blk) & 15, s1 = s0 ^ 8;
  ring_put(ring, s0, A0);
  ring_put(ring, s0 + 4, A1);
  ring_put(ring, s1, B0);
  ring_put(ring, s1 + 4, B1);
  const uint32_t off = (uint32_t)(bitpos & 31);
  const uint32_t w0 = ring[(gw0 & 15) * kLvStride], w1 = ring[((gw0 + 1) & 15) * kLvStride];
  R.hi = __funnelshift_l(w1, w0, off);
  R.lo = shl_c(w1, off);
  R.cnt = 64 - off;
  R.wi = gw0 + 2;
  R.wr = 8 * (blk + 2);
  R.qs = make_uint4(0, 0, 0, 0);
  R.qs2 = make_uint4(0, 0, 0, 0);
  ldg_v8_if_l2(R.qs, R.qs2, G + 2 * min(blk + 2, v8), true);
}
// group boundary: when 8 ring slots are consumed, move the 32-byte block
// loaded at the last such refill into the ring and issue the next load
NBZG_DEV void bb_refill(BufReader& R, uint32_t* ring, const uint4* G, uint32_t vmax) {
  const bool room = (int32_t)(R.wr - R.wi) <= 8;
  if (room) {
    const uint32_t s = R.wr & 15;  // 0 or 8
    ring_put(ring, s, R.qs);
    ring_put(ring, s + 4, R.qs2);
    R.wr += 8;
  }
  ldg_v8_if_l2(R.qs, R.qs2, G + 2 * min(R.wr >> 3, vmax >> 1), room);
}
#else
NBZG_DEV void bb_init(BufReader& R, const uint4* G, uint32_t* ring, uint64_t bitpos,
                      uint32_t vmax) {
  const uint32_t gw0 = (uint32_t)(bitpos >> 5);
  const uint32_t blk = gw0 >> 2;
  const uint4 A = ldg_l2fill(G + min(blk, vmax)), B = ldg_l2fill(G + min(blk + 1, vmax));
  const uint32_t s0 = (4 * blk) & 7, s1 = s0 ^ 4;  // word w -> slot w & 7
  ring[(s0 + 0) * kRingStride] = bswap32(A.x);
  ring[(s0 + 1) * kRingStride] = bswap32(A.y);
  ring[(s0 + 2) * kRingStride] = bswap32(A.z);
  ring[(s0 + 3) * kRingStride] = bswap32(A.w);
  ring[(s1 + 0) * kRingStride] = bswap32(B.x);
  ring[(s1 + 1) * kRingStride] = bswap32(B.y);
  ring[(s1 + 2) * kRingStride] = bswap32(B.z);
  ring[(s1 + 3) * kRingStride] = bswap32(B.w);
  const uint32_t off = (uint32_t)(bitpos & 31);
  const uint32_t w0 = ring[(gw0 & 7) * kRingStride], w1 = ring[((gw0 + 1) & 7) * kRingStride];
  R.hi = __funnelshift_l(w1, w0, off);
  R.lo = shl_c(w1, off);
  R.cnt = 64 - off;
  R.wi = gw0 + 2;
  R.wr = 4 * (blk + 2);
  R.qs = make_uint4(0, 0, 0, 0);
  ldg_v4_if_l2(R.qs, G + min(blk + 2, vmax), true);
}
// group boundary: move the block loaded at the last boundary into the ring
// when its slots are consumed, and issue the next block's load
NBZG_DEV void bb_refill(BufReader& R, uint32_t* ring, const uint4* G, uint32_t vmax) {
  const bool room = (int32_t)(R.wr - R.wi) <= 4;
  if (room) {
    const uint32_t s = R.wr & 7;  // 0 or 4
    ring[(s + 0) * kRingStride] = bswap32(R.qs.x);
    ring[(s + 1) * kRingStride] = bswap32(R.qs.y);
    ring[(s + 2) * kRingStride] = bswap32(R.qs.z);
    ring[(s + 3) * kRingStride] = bswap32(R.qs.w);
    R.wr += 4;
  }
  ldg_v4_if_l2(R.qs, G + min(R.wr >> 2, vmax), room);
}
#endif

// constants of one field's decode, shared by the chunk lanes of a thread
struct LvCtx {
  const int32_t* LT;
  const uint64_t* s_limit;
  const int32_t* s_base;
  const uint32_t* ss;
  const uint4* G;
  const uint32_t* G32;
  const DField* F;
  double twob;
  uint32_t vmax, wmax, r0m1, r0, sh2, lt_s;
  uint32_t rlim, m2;  // table index of window v: hi(min(v, rlim) * 2^15) + hi((v - min) * m2)
  uint32_t p15;       // first long-code entry (= r0 >> 17 when long codes exist)
  uint32_t lt_n;      // entries in the shared table (checked build)
  int lmin, max_len, bias;
};
// one chunk being decoded
struct LvChunk {
  BufReader R;
  long long k;     // lattice index of the last symbol
  uint64_t B, Tb;  // first bit (from the aligned base) and bit length
  float* dst;
  uint32_t* ring;  // this chunk's ring column
  uint32_t ring_s;
  int mc, err;
};
struct LvSnap {
  uint32_t hi, lo, cnt, wi;
  long long k;
};

NBZG_DEV uint64_t lv_consumed(const LvChunk& S) {
  return ((uint64_t)S.R.wi << 5) - S.R.cnt - S.B;
}
// exact refill to > 32 valid bits (ring, or global words past it)
NBZG_DEV void lv_fill_safe(const LvCtx& X, LvChunk& S) {
#pragma unroll 1
  while (S.R.cnt <= 32) {
    uint32_t nw;
    if ((int32_t)(S.R.wr - S.R.wi) > 0) {
      nw = S.ring[(S.R.wi & kLvRingMask) * kLvStride];
    } else {
      asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(nw) : "l"(X.G32 + min(S.R.wi, X.wmax)));
      nw = bswap32(nw);
    }
    bb_fill(S.R, nw);
  }
}
// Index of window v in the shared table: codes <= 15 bits resolve in the
// primary entries [0, P) (P = r0 >> 17: the 15-bit prefixes below the first
// long code), longer codes in the long-code entries [P, P + n2) at 2^sh2
// resolution.  Branch- and select-free, mostly on the FMA pipe (two
// IMAD.HI): min(v, r0) >> 17 is the prefix of a short code and P for a long
// one; (v - min(v, r0)) >> sh2 is 0 for a short code.
NBZG_DEV uint32_t lv_index(const LvCtx& X, uint32_t v) {
#ifdef NBZG_DEC_LVINDEX  // (measured slower: the IMAD.HI chain lengthens the critical path)
  const uint32_t m = min(v, X.rlim);
  return __umulhi(m, 1u << kTpcBits) + __umulhi(v - m, X.m2);
#else
  return v > X.r0m1 ? X.p15 + ((v - X.r0) >> X.sh2) : v >> (32 - kTpcBits);
#endif
}
// canonical decode of the symbol at v (any length <= 32)
NBZG_DEV int32_t lv_resolve(const LvCtx& X, LvChunk& S, uint32_t v) {
  int32_t e = X.LT[lv_index(X, v)];
  {
    if ((e & 63) == 0) {  // longer than the tables resolve, or invalid
      int r = 0;
#pragma unroll 1
      for (int len = X.max_len; len > X.lmin; len--) r = ((uint64_t)v < X.s_limit[len]) ? len : r;
      if (r == 0) {
        S.err = NBZG_INVALID_CODE;
        e = 1;
      } else {
        const uint32_t sym = __ldg(X.ss + (uint32_t)(X.s_base[r] + (int32_t)(v >> (32 - r))));
        e = sym == 0 ? (r | 64) : (int32_t)(((uint32_t)((int)sym - X.bias) << 7) | (uint32_t)r);
      }
    }
  }
  return e;
}
NBZG_DEV void lv_safe_step(const LvCtx& X, LvChunk& S, float& o) {
  lv_fill_safe(X, S);
  const int32_t e = lv_resolve(X, S, S.R.hi);
  bb_take(S.R, (uint32_t)e & 63u);
  if (e & 64) {
    lv_fill_safe(X, S);
    o = __uint_as_float(S.R.hi);
    S.k = esc_k(o, *X.F);
    bb_take(S.R, 32);
  } else {
    S.k += (long long)(e >> 7);
    o = (float)__dmul_rn((double)S.k, X.twob);
  }
}
// 8 symbols, straight-line (no branch: the steps of two chunks interleave);
// returns true when the group must be replayed exactly.  The 64-bit buffer
// is topped up to > 32 bits every RF symbols: every 2 for long codes, every
// 4 for short ones (a field's mean code length below 6 bits) -- a window
// that outruns the buffer wraps `cnt` and the group is replayed.
template <int RF>
NBZG_DEV bool lv_fast8(const LvCtx& X, LvChunk& S, float (&o)[8], LvSnap& sn) {
  BufReader& R = S.R;
  sn.hi = R.hi;
  sn.lo = R.lo;
  sn.cnt = R.cnt;
  sn.wi = R.wi;
  sn.k = S.k;
  // int32 lattice index inside the group: 8 deltas move it < 2^19
  int32_t k32 = (int32_t)S.k;
  uint32_t flags = (unsigned long long)(S.k + (1ll << 30)) >> 31 ? 64u : 0u;  // |k| >= 2^30
#pragma unroll
  for (int q = 0; q < 8; q++) {
    if ((q & (RF - 1)) == 0) {  // > 32 valid bits before every RF-th symbol (branch-free:
      // both shifts are 0 when cnt > 32)
      const uint32_t nw = S.ring[(R.wi & kLvRingMask) * kLvStride];
      R.hi |= shr_c(nw, R.cnt);
      R.lo |= shl_c(nw, 32u - R.cnt);
      const uint32_t t = R.cnt <= 32 ? 32u : 0u;
      R.cnt += t;
      R.wi += t >> 5;
    }
    const uint32_t v = R.hi;
    NBZG_CHECK(lv_index(X, v) < X.lt_n);
    const int32_t e = X.LT[lv_index(X, v)];
    flags |= (uint32_t)e;  // bit 6: escape or unresolved
    bb_take(R, (uint32_t)e & 63u);
    k32 += e >> 7;
#ifdef NBZG_DEC_MAGIC
    // f32(k * 2b) with k exact in double: 2^52 + 2^31 + k, minus the bias
    const double kd =
        __hiloint2double(0x43300000, (int32_t)((uint32_t)k32 ^ 0x80000000u)) - 4503601774854144.0;
#else
    const double kd = (double)k32;  // I2F.F64 (exact): one conversion-pipe op
#endif
    o[q] = (float)__dmul_rn(kd, X.twob);
  }
  S.k = k32;
  // replay when: a flagged entry; an odd symbol longer than the buffered
  // bits (cnt wrapped: it then stays > 64); a ring word past the ring
  return (flags & 64u) || R.cnt > 64 || (int32_t)(R.wi - R.wr) > 0;
}
NBZG_DEV void lv_fix(const LvCtx& X, LvChunk& S, float (&o)[8], const LvSnap& sn, bool bad) {
  if (bad) {
    S.R.hi = sn.hi;
    S.R.lo = sn.lo;
    S.R.cnt = sn.cnt;
    S.R.wi = sn.wi;
    S.k = sn.k;
#pragma unroll 1
    for (int q = 0; q < 8; q++) {
      float t;
      lv_safe_step(X, S, t);
#pragma unroll
      for (int u = 0; u < 8; u++) o[u] = (u == q) ? t : o[u];
    }
  }
  bb_refill(S.R, S.ring, X.G, X.vmax);
}
NBZG_DEV void lv_start(const LvCtx& X, const DArgs& a, const uint64_t* choff, uint32_t a0,
                       int64_t c, uint32_t* ring, LvChunk& S) {
  const uint64_t b0 = choff[c];
  S.Tb = choff[c + 1] - b0;
  const int64_t i0 = c * kChunk;
  S.mc = (int)min((int64_t)kChunk, a.n - i0);
  S.B = a0 + b0;
  S.ring = ring;
  S.ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  bb_init(S.R, X.G, ring, S.B, X.vmax);
  S.k = 0;
  S.err = 0;
  S.dst = X.F->out + i0;
}
// symbols [i, mc) one exact step at a time, then the end-of-chunk checks
NBZG_DEV void lv_finish(const LvCtx& X, const DArgs& a, LvChunk& S, int i) {
  for (; i < S.mc && lv_consumed(S) <= S.Tb; i++) {
    float o;
    lv_safe_step(X, S, o);
    if ((i & 7) == 7) bb_refill(S.R, S.ring, X.G, X.vmax);
    S.dst[i] = o;
  }
  const uint64_t pos = lv_consumed(S);
  if (!S.err && pos != S.Tb) S.err = pos > S.Tb ? NBZG_TRUNCATED : NBZG_BAD_STREAM;
  if (S.err) fail(a.status, (uint32_t)S.err);
}

// the chunks [cb, ce) of one field, a chunk per thread
template <int RF>
NBZG_DEV void lv_chunks(const LvCtx& X, const DArgs& a, const uint64_t* choff, uint32_t a0,
                        int64_t cb, int64_t ce, uint32_t* ring, bool vec) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int64_t c = cb + tid; c < ce; c += nthr) {
    LvChunk A;
    lv_start(X, a, choff, a0, c, ring, A);
    int i = 0;
    if (vec) {
      float oa[8], ob[8];
      LvSnap sa;
#pragma unroll
      for (int u = 0; u < 8; u++) ob[u] = 0.0f;
      for (; i + 16 <= A.mc; i += 16) {
        NBZG_CHECK(A.dst + i + 16 <= X.F->out + a.n);
        lv_fix(X, A, oa, sa, lv_fast8<RF>(X, A, oa, sa));
        // two register sets: a set's stores are issued one group before the
        // set is rewritten (pinned live meanwhile)
        asm volatile("" ::"f"(ob[0]), "f"(ob[1]), "f"(ob[2]), "f"(ob[3]), "f"(ob[4]),
                     "f"(ob[5]), "f"(ob[6]), "f"(ob[7]));
        st_v8_cs(A.dst + i, oa);
        lv_fix(X, A, ob, sa, lv_fast8<RF>(X, A, ob, sa));
        asm volatile("" ::"f"(oa[0]), "f"(oa[1]), "f"(oa[2]), "f"(oa[3]), "f"(oa[4]),
                     "f"(oa[5]), "f"(oa[6]), "f"(oa[7]));
#ifndef NBZG_DEC_STHALF  // timing experiment: half the stores
        st_v8_cs(A.dst + i + 8, ob);
#else
        if (ob[0] == 1234.5f) A.dst[i] = ob[1];
#endif
        if (lv_consumed(A) > A.Tb) {
          i += 16;
          break;  // corrupt: stop early, reported below
        }
      }
    }
    lv_finish(X, a, A, i);
  }
}


// ---- canonical mode of the thread-per-chunk decoder (large alphabets) ----
// When most codes are longer than the fused tables resolve (k ~ 2^15-2^16
// symbols at tight error bounds: code lengths 14-18), every group would be
// replayed on the exact path, whose symbol lookup is a global load.  This
// mode keeps the canonical decode (encode.py:242-261) entirely in shared
// memory instead: the symbols by canonical rank (u16, <= 128 KiB), the
// left-aligned limits and rank bases per length, and a 2^12-entry table with
// the first length possible for a 12-bit prefix (and its rank base).  A symbol is
//   (l, base) = first[v >> 20];  unless the prefix holds one length only:
//   while (v >= limit[l]) l++;  base = base_of[l];
//   sym = syms[base + (v >> (32 - l))]
// i.e. two dependent shared-memory reads for most symbols (a 12-bit prefix of
// 14-18-bit codes rarely straddles two lengths) and no speculation.
struct CanonCtx {
  const uint16_t* syms;
  const uint2* first;     // [2^kCanonBits]: .x = rank base of length l, .y = l | unique << 8
  const uint64_t* limit;  // [l]: first window value past the codes of length <= l (<= 2^32)
  const int32_t* base;    // [l]: rank of the first code of length l minus its code value
  int max_len, bias;
};

NBZG_DEV void canon_step(const LvCtx& X, const CanonCtx& C, LvChunk& S, float& o) {
  lv_fill_safe(X, S);
  const uint32_t v = S.R.hi;
  const uint2 e = C.first[v >> (32 - kCanonBits)];
  int l = (int)(e.y & 0xffu);
  int32_t bs = (int32_t)e.x;
  if (!(e.y & 0x100u)) {  // the prefix spans several lengths: walk the limits
    while (l <= C.max_len && (uint64_t)v >= C.limit[l]) l++;
    if (l > C.max_len) {  // outside the code (incomplete table)
      S.err = NBZG_INVALID_CODE;
      bb_take(S.R, 1);
      o = 0.0f;
      return;
    }
    bs = C.base[l];
  }
  const uint32_t sym = C.syms[bs + (int32_t)(v >> (32 - l))];
  bb_take(S.R, (uint32_t)l);
  if (sym == 0) {  // escape: the raw f32 follows
    lv_fill_safe(X, S);
    o = __uint_as_float(S.R.hi);
    S.k = esc_k(o, *X.F);
    bb_take(S.R, 32);
  } else {
    S.k += (long long)((int)sym - C.bias);
    o = (float)__dmul_rn((double)S.k, X.twob);
  }
}

NBZG_DEV void canon_chunks(const LvCtx& X, const CanonCtx& C, const DArgs& a, const uint64_t* choff,
                           uint32_t a0, int64_t cb, int64_t ce, uint32_t* ring, bool vec) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int64_t c = cb + tid; c < ce; c += nthr) {
    LvChunk A;
    lv_start(X, a, choff, a0, c, ring, A);
    int i = 0;
    if (vec) {
      for (; i + 8 <= A.mc && lv_consumed(A) <= A.Tb; i += 8) {
        float o[8];
#pragma unroll
        for (int q = 0; q < 8; q++) canon_step(X, C, A, o[q]);
        bb_refill(A.R, A.ring, X.G, X.vmax);
        st_v8_cs(A.dst + i, o);
      }
    }
    for (; i < A.mc && lv_consumed(A) <= A.Tb; i++) {
      float o;
      canon_step(X, C, A, o);
      if ((i & 7) == 7) bb_refill(A.R, A.ring, X.G, X.vmax);
      A.dst[i] = o;
    }
    const uint64_t pos = lv_consumed(A);
    if (!A.err && pos != A.Tb) A.err = pos > A.Tb ? NBZG_TRUNCATED : NBZG_BAD_STREAM;
    if (A.err) fail(a.status, (uint32_t)A.err);
  }
}


__global__ void __launch_bounds__(kLvMaxThreads, 1) decode_lv_kernel(DArgs a) {
  extern __shared__ __align__(16) uint8_t dsm2[];
  int32_t* LT = reinterpret_cast<int32_t*>(dsm2);  // [2^15 + t2_n]
  __shared__ uint64_t s_limit[64];
  __shared__ int32_t s_base[64];
  // fields own contiguous CTA ranges sized by their decode cost (host)
  int fi = 0;
  while (fi + 1 < a.nf && (int)blockIdx.x >= a.cta0[fi + 1]) fi++;
  const int gj = (int)blockIdx.x - a.cta0[fi], gn = a.cta0[fi + 1] - a.cta0[fi];
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if (F.kind != 3 || P.status || *a.status || P.max_len > 32) return;
  const int64_t cb = (a.nchunks * gj) / gn;
  const int64_t ce = (a.nchunks * (gj + 1)) / gn;
  if (cb >= ce) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
#ifdef NBZG_LV_PROF  // timing experiment: cycles of the first CTA of every field
  const long long lv_t0 = clock64();
  struct LvProf {
    long long t0;
    int fi, gn, canon;
    int64_t nch;
    __device__ ~LvProf() {
      __syncthreads();
      if (threadIdx.x == 0 && t0) printf("decode_lv field %d canon %d ctas %d chunks/cta %lld cycles %lld\n", fi, canon, gn, (long long)nch, clock64() - t0);
    }
  } lv_prof{lv_t0, fi, gn, (int)P.use_canon, ce - cb};
  if (gj != 0) lv_prof.t0 = 0;
#endif
  uint32_t* ring = reinterpret_cast<uint32_t*>(dsm2 + 4 * kTpcTab) + tid;  // [kLvRing][kRingStride]
  if (P.use_canon) {
    // shared layout: syms u16[k] | first uint2[2^12] (both inside the fused
    // table's 180 KiB), then the ring as in the fused mode
    uint16_t* c_syms = reinterpret_cast<uint16_t*>(dsm2);
    uint2* c_first = reinterpret_cast<uint2*>(dsm2 + 2 * (size_t)kCanonMaxK);
    const uint32_t* gs = a.ssyms + fi * a.nbins;
    for (uint32_t i = tid; i < (uint32_t)P.k; i += nthr) c_syms[i] = (uint16_t)__ldg(gs + i);
    if (tid < 64) {
      const int l = tid;
      uint64_t lim = 0;
      int32_t bs = 0;
      if (l >= 1 && l <= 32 && l <= (int)P.max_len) {
        lim = (P.first_code[l] + P.counts[l]) << (32 - l);
        bs = (int32_t)P.first_idx[l] - (int32_t)P.first_code[l];
      }
      s_limit[l] = lim;
      s_base[l] = bs;
    }
    __syncthreads();
    for (uint32_t pfx = tid; pfx < (1u << kCanonBits); pfx += nthr) {
      // length of the first and of the last window value of the prefix
      const uint64_t v0 = (uint64_t)pfx << (32 - kCanonBits);
      const uint64_t v1 = v0 + ((1ull << (32 - kCanonBits)) - 1);
      int l0 = 1;
      while (l0 <= (int)P.max_len && v0 >= s_limit[l0]) l0++;
      int l1 = l0;
      while (l1 <= (int)P.max_len && v1 >= s_limit[l1]) l1++;
      const bool unique = l0 == l1 && l0 <= (int)P.max_len;
      c_first[pfx] = make_uint2((uint32_t)s_base[min(l0, 63)], (uint32_t)min(l0, 33) | (unique ? 0x100u : 0u));
    }
    __syncthreads();
    LvCtx X{};
    const uintptr_t bits_addr = reinterpret_cast<uintptr_t>(F.payload + P.bits_off);
    constexpr uintptr_t kAl = NBZG_LV_RING == 16 ? 31 : 15;
    X.G = reinterpret_cast<const uint4*>(bits_addr & ~kAl);
    X.G32 = reinterpret_cast<const uint32_t*>(X.G);
    const uint32_t a0 = (uint32_t)(bits_addr & kAl) * 8;
    X.vmax = (uint32_t)((a0 / 8 + 4 * ((P.total_bits + 31) / 32) + 16) / 16);
    X.wmax = 4 * X.vmax + 3;
    X.F = &F;
    X.twob = F.twob;
    CanonCtx C{c_syms, c_first, s_limit, s_base, (int)P.max_len, a.half + 1};
    const bool vec = (reinterpret_cast<uintptr_t>(F.out) & 31) == 0;
    canon_chunks(X, C, a, a.choff + fi * (a.nchunks + 1), a0, cb, ce, ring, vec);
    return;
  }
  const uint32_t n2 = P.t2_n;
  // shared table: the primary entries of the 15-bit prefixes below r0, then
  // the long-code entries (lv_index); one unresolved entry when long codes
  // exist but their table is empty
  const bool has_long = P.t2_r0 < ((uint64_t)1 << 32);
  const uint32_t P15 = has_long ? (uint32_t)(P.t2_r0 >> (32 - kTpcBits)) : (1u << kTpcBits);
  {
    const int32_t* gl = a.lut2 + (size_t)fi * kLut2Stride;
    for (uint32_t i = tid; i < P15; i += nthr) LT[i] = __ldg(gl + i);
    for (uint32_t i = tid; i < n2; i += nthr) LT[P15 + i] = __ldg(gl + (1 << kTpcBits) + i);
    if (tid < 2 && has_long && n2 == 0) LT[P15 + tid] = 64;  // (v - r0) >> 31 is 0 or 1
  }
  __syncthreads();
  if (tid < 64) {
    const int l = tid;
    uint64_t lim = 0;
    int32_t bs = 0;
    if (l >= 1 && l <= 32 && l <= (int)P.max_len) {
      lim = (P.first_code[l] + P.counts[l]) << (32 - l);
      bs = (int32_t)P.first_idx[l] - (int32_t)P.first_code[l];
    }
    s_limit[l] = l > (int)P.max_len ? ~0ull : lim;
    s_base[l] = bs;
  }
  __syncthreads();

  LvCtx X;
  X.LT = LT;
  X.s_limit = s_limit;
  X.s_base = s_base;
  X.ss = a.ssyms + fi * a.nbins;
  const uintptr_t bits_addr = reinterpret_cast<uintptr_t>(F.payload + P.bits_off);
  // stream base aligned to the refill load size (the bit offset a0 absorbs
  // the rest; the payload's table precedes its bitstream, so the aligned
  // base stays inside the payload)
  constexpr uintptr_t kAl = NBZG_LV_RING == 16 ? 31 : 15;
  X.G = reinterpret_cast<const uint4*>(bits_addr & ~kAl);
  X.G32 = reinterpret_cast<const uint32_t*>(X.G);
  const uint32_t a0 = (uint32_t)(bits_addr & kAl) * 8;
  // last 16-byte block / word the stream may touch (payload + 64-byte slack)
  X.vmax = (uint32_t)((a0 / 8 + 4 * ((P.total_bits + 31) / 32) + 16) / 16);
  X.wmax = 4 * X.vmax + 3;
  X.F = &F;
  X.twob = F.twob;
  X.bias = a.half + 1;
  X.max_len = (int)P.max_len;
  // table index of window v: codes <= 15 bits fill [0, r0) and resolve in
  // the primary table; the rest index the long-code table, which covers
  // [r0, 2^32) at 2^sh2 resolution (two unresolved entries when it is empty)
  X.r0m1 = (uint32_t)(min(P.t2_r0, (uint64_t)1 << 32) - 1);
  X.r0 = X.r0m1 + 1;
  X.sh2 = n2 ? 32u - P.t2_w : 31u;
  X.rlim = has_long ? (uint32_t)P.t2_r0 : 0xffffffffu;
  X.p15 = P15;
  X.lt_n = P15 + max(n2, 2u);
  X.m2 = n2 ? (1u << P.t2_w) : 0u;
  X.lmin = n2 ? (int)P.t2_w : kTpcBits;  // longer codes: canonical search
  X.lt_s = (uint32_t)__cvta_generic_to_shared(LT);
  const uint64_t* choff = a.choff + fi * (a.nchunks + 1);
  const bool vec = (reinterpret_cast<uintptr_t>(F.out) & 31) == 0;  // 32-byte stores

#ifndef NBZG_DEC_RF4
#define NBZG_DEC_RF4 0
#endif
  // refill cadence by the field's mean code length (bits per symbol)
  const bool rf4 = NBZG_DEC_RF4 && 8 * F.payload_len < 6 * a.n;
  if (rf4) lv_chunks<4>(X, a, choff, a0, cb, ce, ring, vec);
  else lv_chunks<2>(X, a, choff, a0, cb, ce, ring, vec);
}

// v2 streams with codes longer than 32 bits (pathological alphabets):
// serial decode per chunk (one thread per chunk), same semantics.
template <bool LCF>
__device__ void decode_v2_serial_body(const DArgs& a, const DField& F, const DParsed& P, int fi);
__global__ void decode_v2_serial_kernel(DArgs a) {
  const int fi = blockIdx.y;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if ((F.kind & 15) != 3 || P.status || P.max_len <= 32) return;
  if (F.kind & NBZG_KIND_LCF) decode_v2_serial_body<true>(a, F, P, fi);
  else decode_v2_serial_body<false>(a, F, P, fi);
}
template <bool LCF>
__device__ void decode_v2_serial_body(const DArgs& a, const DField& F, const DParsed& P, int fi) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nchunks) return;
  const uint64_t* choff = a.choff + fi * (a.nchunks + 1);
  const uint8_t* bits = F.payload + P.bits_off;
  uint64_t bp = choff[c], endp = choff[c + 1];
  const uint32_t* ss = a.ssyms + fi * a.nbins;
  const int64_t c0 = c * kChunk, c1 = min(a.n, c0 + kChunk);
  KState<LCF> ks;
  for (int64_t i = c0; i < c1; i++) {
    uint32_t sym = 0;
    int l = decode_serial(bits, bp, endp, P, ss, sym);
    if (l < 0) {
      fail(a.status, (uint32_t)(-l));
      return;
    }
    float outv;
    if (sym == 0) {
      if (bp + 32 > endp) {
        fail(a.status, NBZG_TRUNCATED);
        return;
      }
      uint32_t u = 0;
      for (int b = 0; b < 32; b++, bp++) u = (u << 1) | ((bits[bp >> 3] >> (7 - (bp & 7))) & 1u);
      outv = __uint_as_float(u);
      ks.escape(esc_k(outv, F));
    } else {
      outv = ks.apply((int)sym - a.half - 1, F.twob);
    }
    F.out[i] = outv;
  }
  if (bp != endp) fail(a.status, NBZG_BAD_STREAM);
}

// ---------------------------------------------------------------- v1 compat
// Reference SZ_FIELD streams: bit-serial decode + the exact sequential chain
// (_kernels.py:126-147), one thread per field.  Compatibility path only.
__global__ void decode_v1_kernel(DArgs a) {
  const int fi = blockIdx.x;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if ((F.kind & 15) != 0 || P.status || threadIdx.x != 0) return;
  const bool lcf = F.kind & NBZG_KIND_LCF;  // sz-lcf: pred = 2*h1 - h2 from i = 2
  const uint8_t* bits = F.payload + P.bits_off;
  const uint8_t* escp = F.payload + P.esc_off;
  const uint32_t* ss = a.ssyms + fi * a.nbins;
  const int half = a.half;
  uint64_t bp = 0, ei = 0;
  double h1 = 0.0, h2 = 0.0;
  for (int64_t i = 0; i < a.n; i++) {
    uint32_t sym = 0;
    int l = decode_serial(bits, bp, P.total_bits, P, ss, sym);
    if (l < 0) {
      fail(a.status, (uint32_t)(-l));
      return;
    }
    float r;
    if (sym == 0) {
      if (ei >= P.n_esc) {
        fail(a.status, NBZG_BAD_STREAM);
        return;
      }
      r = __uint_as_float(ld_u32_bytes(escp + 4 * ei));
      ei++;
    } else {
      double pred = i == 0 ? 0.0 : (lcf && i >= 2 ? __dsub_rn(2.0 * h1, h2) : h1);
      double q = (double)((int)sym - half - 1);
      r = (float)__dadd_rn(pred, __dmul_rn(q, F.twob));
    }
    F.out[i] = r;
    h2 = h1;
    h1 = (double)r;
  }
  if (ei != P.n_esc) fail(a.status, NBZG_BAD_STREAM);
}

// ---------------------------------------------------------------- parity hook
// K.huff_decode (_kernels.py:348-374): canonical decode of n symbols from a
// raw MSB-first bitstream, one thread, the reference's exact walk and
// statuses (0 ok, NBZG_INVALID_CODE, NBZG_TRUNCATED).
__global__ void huff_decode_hook_kernel(const uint8_t* bits, uint64_t total, int64_t n,
                                        DParsed P, const uint32_t* ss, uint32_t* out,
                                        uint32_t* status) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t bp = 0;
  for (int64_t i = 0; i < n; i++) {
    uint32_t sym = 0;
    const int l = decode_serial(bits, bp, total, P, ss, sym);
    if (l < 0) {
      *status = (uint32_t)(-l);
      return;
    }
    out[i] = sym;
  }
  *status = 0;
}

int launch_huff_decode_hook(const uint8_t* bits, uint64_t total, int64_t n, int min_len,
                            int max_len, const uint64_t* first_code, const uint32_t* counts,
                            const uint32_t* first_idx, const uint32_t* ss, uint32_t* out,
                            uint32_t* status, cudaStream_t st) {
  if (min_len < 1 || max_len > 63 || min_len > max_len) return NBZG_BAD_ARG;
  DParsed P{};
  P.min_len = (uint32_t)min_len;
  P.max_len = (uint32_t)max_len;
  for (int l = 0; l < 64; l++) {
    P.first_code[l] = first_code[l];
    P.counts[l] = counts[l];
    P.first_idx[l] = first_idx[l];
  }
  count_launch();
  huff_decode_hook_kernel<<<1, 32, 0, st>>>(bits, total, n, P, ss, out, status);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// deinterleave3 (_kernels.py:789-798): key bit 3j+2 -> x bit j, 3j+1 -> y, 3j -> z
NBZG_DEV uint64_t compact3_hook(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v | (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v | (v >> 8)) & 0x1F0000FF0000FFull;
  v = (v | (v >> 16)) & 0x1F00000000FFFFull;
  v = (v | (v >> 32)) & 0x1FFFFFull;
  return v;
}
__global__ void deinterleave3_kernel(const uint64_t* keys, int64_t n, int64_t* x, int64_t* y,
                                     int64_t* z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  x[i] = (int64_t)compact3_hook(k >> 2);
  y[i] = (int64_t)compact3_hook(k >> 1);
  z[i] = (int64_t)compact3_hook(k);
}
int launch_deinterleave3(const uint64_t* keys, int64_t n, int64_t* x, int64_t* y, int64_t* z,
                         cudaStream_t st) {
  if (n > 0) {
    count_launch();
    deinterleave3_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(keys, n, x, y, z);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// ---------------------------------------------------------------- launcher
// NBZG_DECODE=warp|thread forces one v2 decoder (tests cover both).
static bool use_tpc(int64_t nchunks) {
  const char* e = getenv("NBZG_DECODE");
  if (e && e[0] == 't') return true;
  if (e && e[0] == 'w') return false;
  return nchunks >= kTpcMinChunks;
}

size_t decompress_ws(int nf, int64_t n, int64_t nbins) {
  int64_t nchunks = (n + kChunk - 1) / kChunk;
  size_t s = 0;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  s += al(sizeof(DParsed) * nf);
  s += al((size_t)nf * (1 << kLutBits));
  s += al((size_t)nf * 4 * kLut2Stride);
  s += al(sizeof(uint32_t) * nf * nbins);
  s += al(sizeof(uint64_t) * nf * (nchunks + 1));
  s += al(sizeof(uint64_t) * nf * 2 * (nchunks + 1));
  s += al(sizeof(uint32_t) * 16);
  return s;
}

int launch_decompress(const DField* fields, int nf, int64_t n, int64_t interval_count, void* ws,
                      size_t ws_bytes, uint32_t* status, cudaStream_t st) {
  if (nf < 1 || nf > 6) return NBZG_BAD_ARG;
  if (interval_count < 2 || interval_count > 65536 || (interval_count & 1)) return NBZG_UNSUPPORTED;
  int64_t nbins = interval_count + 1;  // v1 codes reach interval_count
  if (ws_bytes < decompress_ws(nf, n, nbins)) return NBZG_BAD_ARG;
  DArgs a{};
  for (int i = 0; i < nf; i++) a.f[i] = fields[i];
  a.nf = nf;
  a.n = n;
  a.nchunks = (n + kChunk - 1) / kChunk;
  a.nbins = nbins;
  a.half = (int)(interval_count / 2);
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  a.parsed = reinterpret_cast<DParsed*>(p);
  p += al(sizeof(DParsed) * nf);
  a.lut = reinterpret_cast<uint32_t*>(p);
  p += al((size_t)nf * (1 << kLutBits));
  a.lut2 = reinterpret_cast<int32_t*>(p);
  p += al((size_t)nf * 4 * kLut2Stride);
  a.ssyms = reinterpret_cast<uint32_t*>(p);
  p += al(sizeof(uint32_t) * nf * nbins);
  a.choff = reinterpret_cast<uint64_t*>(p);
  p += al(sizeof(uint64_t) * nf * (a.nchunks + 1));
  a.lb = reinterpret_cast<uint64_t*>(p);
  p += al(sizeof(uint64_t) * nf * 2 * (a.nchunks + 1));
  a.tickets = reinterpret_cast<uint32_t*>(p);
  a.status = status;
  if (n == 0) return NBZG_OK;
  cudaMemsetAsync(a.lb, 0, sizeof(uint64_t) * nf * 2 * a.nchunks, st);
  cudaMemsetAsync(a.tickets, 0, sizeof(uint32_t) * 16, st);
  count_launch();
  parse_kernel<<<dim3(nf, 2), 1024, 0, st>>>(a);
  trace_mark("dq_parse", st);
  size_t sm = (1 << kLutBits) + kSmemSyms * 2;
  smem_attr((const void*)decode_kernel<true>, (int)sm);
  smem_attr((const void*)decode_kernel<false>, (int)sm);
  bool any_v2 = false, any_v2_lcf = false, any_v1 = false;
  for (int i = 0; i < nf; i++) {
    any_v2 |= (fields[i].kind & 15) == 3;
    any_v2_lcf |= fields[i].kind == 3 + NBZG_KIND_LCF;
    any_v1 |= (fields[i].kind & 15) == 0;
  }
  if (any_v2) {
    int groups = max(1, sm_count() / nf);
    if (groups > a.nchunks) groups = (int)a.nchunks;
    const int per = (int)((a.nchunks + groups - 1) / groups);
    const int thr = min(kTpcMaxThreads, (per + 31) / 32 * 32);
    const size_t sm2 = 4 * kTpcTab + 32 * (size_t)kRingStride;
    {  // sized for the largest launch
      const int smax = 4 * kTpcTab + 4 * max(kLvRing * kLvStride, 8 * kRingStride);
      smem_attr((const void*)decode_tpc_kernel<false>, smax);
      smem_attr((const void*)decode_tpc_kernel<true>, smax);
      smem_attr((const void*)decode_lv_kernel, smax);
    }
    if (any_v2_lcf) {  // sz-lcf streams: thread-per-chunk decoder only
      count_launch();
      decode_tpc_kernel<true><<<dim3(groups, nf), thr, sm2, st>>>(a, groups);
    }
    if (use_tpc(a.nchunks)) {
      count_launch();
      // CTAs per field in proportion to an estimated decode cost per chunk
      // (a fixed per-symbol part plus the stream bits: at C2 a 10-bit
      // velocity symbol costs ~1.25x a 3.5-bit coordinate one), at most
      // kLvMaxThreads chunks per CTA, one CTA per SM
      const int sms = sm_count();
      double w[6], wsum = 0;
      int gmin[6], g[6], gtot = 0;
      for (int f = 0; f < nf; f++) {
        const double bits = a.n ? 8.0 * (double)fields[f].payload_len / (double)a.n : 0.0;
        w[f] = fields[f].kind == 3 ? 1.0 + bits / 26.0 : 0.0;
        // (streams this dense usually decode in the canonical mode: two or
        // three dependent lookups per symbol instead of one)
        if (bits >= kCanonCostBits) w[f] *= kCanonCost;
        wsum += w[f];
        gmin[f] = fields[f].kind == 3 ? (int)((a.nchunks + kLvMaxThreads - 1) / kLvMaxThreads) : 1;
        gmin[f] = max(1, gmin[f]);
      }
      for (int f = 0; f < nf; f++) {
        g[f] = wsum > 0 ? max(gmin[f], (int)((double)sms * w[f] / wsum)) : 1;
        if (g[f] > a.nchunks) g[f] = (int)max((int64_t)1, a.nchunks);
        gtot += g[f];
      }
      while (gtot > sms) {  // trim the fields with the most slack
        int best = -1;
        for (int f = 0; f < nf; f++)
          if (g[f] > gmin[f] && (best < 0 || g[f] * w[best] > g[best] * w[f])) best = f;
        if (best < 0) break;
        g[best]--;
        gtot--;
      }
      int thr_lv = 32;
      a.cta0[0] = 0;
      for (int f = 0; f < nf; f++) {
        a.cta0[f + 1] = a.cta0[f] + g[f];
        thr_lv = max(thr_lv, (int)min((int64_t)kLvMaxThreads, ((a.nchunks + g[f] - 1) / g[f] + 31) / 32 * 32));
      }
      decode_lv_kernel<<<a.cta0[nf], thr_lv, 4 * kTpcTab + 4 * kLvRing * (size_t)kLvStride, st>>>(a);
    } else {
      count_launch();
      decode_kernel<true><<<groups * nf, kDThreads, sm, st>>>(a);
      count_launch();
      decode_kernel<false><<<groups * nf, kDThreads, sm, st>>>(a);
    }
    count_launch();
    decode_v2_serial_kernel<<<dim3((unsigned)((a.nchunks + 63) / 64), nf), 64, 0, st>>>(a);
    trace_mark("dq_decode", st);
  }
  if (any_v1) {
    count_launch();
    decode_v1_kernel<<<nf, 32, 0, st>>>(a);
    trace_mark("dq_decode_v1", st);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
