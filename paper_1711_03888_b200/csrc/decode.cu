// decode.cu -- K8: chunk-parallel Huffman decode fused with the dual-quant
// dequantiser, plus the v1 (reference stream) compat decoder.
//
// Replaces pipeline._parse_sz_stream (pipeline.py:203-223) ->
// encode.huffman_decode (encode.py:242-261) -> K.huff_decode
// (_kernels.py:348-374) and quantize.dequantize_field -> K.sz_dequantize
// (_kernels.py:126-147).
//
// v2 (kind 3) decode, one CTA per 16384-symbol chunk located by the chunk
// index:
//   1. stage the chunk's bits in shared memory, re-aligned so bit 0 is the
//      MSB of word 0 (any payload alignment);
//   2. self-synchronising parallel Huffman decode: every thread decodes its
//      slice (>= 192 bits) from an arbitrary bit, counting codewords and
//      remembering its first 8 codeword starts in registers, then re-walks
//      from its predecessor's true end until it lands on a remembered start
//      (Huffman codes resynchronise within a few codewords) and corrects its
//      count; a 2^16-entry code-length table in shared memory decodes;
//   3. decode again from the true starts into shared memory;
//   4. dequantise: escape offsets and the lattice index k carried into the
//      chunk come from two decoupled look-backs; recon = f32(k * 2b) or the
//      verbatim escape; 16 floats per thread written with 128-bit stores.
// Status words: INVALID_CODE / TRUNCATED / BAD_STREAM -> DecodeError.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kDThreads = 1024;
constexpr int kDPer = kChunk / kDThreads;  // 16 symbols per thread (dequant)
constexpr int kDBufWords = 8192;           // 262144 bits of stream per chunk in smem
constexpr int kLutBits = 16;       // length LUT index bits (u8 entries, 64 KiB)
constexpr int kRec = 8;            // phase-1 codeword starts remembered per thread
constexpr int kSmemSyms = 16384;  // sorted-symbol table staged in smem up to this k
constexpr int kSegBits = 192;      // minimum bits per decoding thread (limits sync cascades)

struct DParsed {
  uint64_t n_esc, k, total_bits;
  uint64_t index_off, bits_off, esc_off;
  uint32_t min_len, max_len;
  uint32_t status;
  uint32_t pad;
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
  uint32_t* lut;       // [nf][4096]
  uint32_t* ssyms;     // [nf][nbins] sorted (len, sym) symbols
  uint64_t* choff;     // [nf][nchunks+1] chunk bit offsets
  uint64_t* lb;        // [nf][2][nchunks]
  uint32_t* tickets;   // [nf]
  uint32_t* status;    // global status word
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
__global__ void __launch_bounds__(1024) parse_kernel(DArgs a) {
  const int fi = blockIdx.x;
  const DField& F = a.f[fi];
  DParsed& P = a.parsed[fi];
  uint8_t* lut = reinterpret_cast<uint8_t*>(a.lut) + fi * (1 << kLutBits);
  uint32_t* ss = a.ssyms + fi * a.nbins;
  __shared__ uint32_t s_bad, s_cbl[64], s_max, s_min;
  __shared__ uint32_t scan_tmp[33];
  __shared__ uint64_t s_fc[64];
  __shared__ uint32_t s_fi[64];
  const int tid = threadIdx.x;
  const uint8_t* p = F.payload;
  const int64_t L = F.payload_len;
  if (tid == 0) {
    s_bad = 0;
    s_max = 0;
    s_min = 255;
  }
  if (tid < 64) s_cbl[tid] = 0;
  for (int i = tid; i < (1 << kLutBits); i += blockDim.x) lut[i] = 0;
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
    bool bad = l < 1 || l > kMaxCodeLen || s >= (uint64_t)a.nbins - (F.kind == 3 ? 1 : 0);
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
  // canonical order: rank within length class, ascending symbol
  const int RK = (int)((k + blockDim.x - 1) / blockDim.x);
  for (int l = 1; l <= max_len; l++) {
    if (s_cbl[l] == 0) continue;
    uint32_t c = 0;
    for (int r = 0; r < RK; r++) {
      uint64_t i = (uint64_t)tid * RK + r;
      if (i < k && p[8 + 5 * i + 4] == l) c++;
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan<uint32_t>(c, scan_tmp, &tot);
    for (int r = 0; r < RK; r++) {
      uint64_t i = (uint64_t)tid * RK + r;
      if (i < k && p[8 + 5 * i + 4] == l) {
        uint32_t sym = ld_u32_bytes(p + 8 + 5 * i);
        uint32_t pos = s_fi[l] + ex;
        ss[pos] = sym;
        ex++;
      }
    }
  }
  // length table: entry e (16-bit prefix) -> smallest l with e.. < limit[l]
  // (canonical order), 0xFE when the code is longer than 16 bits, 0 = invalid
  for (int e = tid; e < (1 << kLutBits); e += blockDim.x) {
    uint8_t len = 0;
    for (int l = 1; l <= max_len; l++) {
      if (l <= kLutBits) {
        uint64_t lim = (s_fc[l] + s_cbl[l]) << (kLutBits - l);  // limit in 16-bit units
        if ((uint64_t)e < lim) {
          len = (uint8_t)l;
          break;
        }
      } else {
        len = 0xFE;
        break;
      }
    }
    lut[e] = len;
  }
  if (tid == 0) {
    const uint64_t table_end = 8 + 5 * k;
    P.n_esc = n_esc;
    P.k = k;
    P.min_len = s_min;
    P.max_len = s_max;
    uint32_t st = 0;
    if (table_end + 8 > (uint64_t)L) st = NBZG_TRUNCATED;
    else {
      P.total_bits = ld_u64_bytes(p + table_end);
      if (F.kind == 3) {
        P.index_off = table_end + 8;
        P.bits_off = (P.index_off + 4 * (uint64_t)a.nchunks + 3) & ~3ull;
        P.esc_off = P.bits_off + 4 * ((P.total_bits + 31) / 32);
        if (P.esc_off + 4 * n_esc != (uint64_t)L) st = NBZG_TRUNCATED;
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
__global__ void __launch_bounds__(1024) chunk_offsets_kernel(DArgs a) {
  const int fi = blockIdx.x;
  const DParsed& P = a.parsed[fi];
  if (P.status || a.f[fi].kind != 3) return;
  __shared__ unsigned long long scan_tmp[33];
  const uint8_t* idx = a.f[fi].payload + P.index_off;
  uint64_t* off = a.choff + fi * (a.nchunks + 1);
  const int R = (int)((a.nchunks + blockDim.x - 1) / blockDim.x);
  unsigned long long s = 0;
  for (int r = 0; r < R; r++) {
    int64_t c = (int64_t)threadIdx.x * R + r;
    if (c < a.nchunks) s += ld_u32_bytes(idx + 4 * c);
  }
  unsigned long long tot;
  unsigned long long ex = block_excl_scan<unsigned long long>(s, scan_tmp, &tot);
  for (int r = 0; r < R; r++) {
    int64_t c = (int64_t)threadIdx.x * R + r;
    if (c < a.nchunks) {
      off[c] = ex;
      ex += ld_u32_bytes(idx + 4 * c);
    }
  }
  if (threadIdx.x == 0) {
    off[a.nchunks] = tot;
    if (tot != P.total_bits) fail(a.status, NBZG_BAD_STREAM);
  }
}

// ---------------------------------------------------------------- decode step
// Shared-memory tables: a 2^12-entry code-LENGTH table (0 = invalid prefix,
// 0xFE = longer code) and the canonical left-justified limits
// (encode.py:133-139): a codeword's length is the smallest l with
// window < limit[l], its symbol ss[base[l] + (window >> (32 - l))].
struct DecTab {
  const uint8_t* ll;         // smem [1 << kLutBits]
  const uint64_t* limit;     // smem [64]
  const int32_t* base;       // smem [64] first_idx[l] - first_code[l]
  const uint16_t* ss16;      // smem sorted symbols (k <= kSmemSyms) or null
  const uint32_t* ss;        // global sorted symbols
  int max_len;
};

NBZG_DEV uint32_t peek32(const uint32_t* W, uint32_t p) {
  uint32_t i = p >> 5, s = p & 31;
  return __funnelshift_l(W[i + 1], W[i], s);
}

// length of the codeword whose left-justified bits are v (0 = invalid)
NBZG_DEV int code_len(uint32_t v, const DecTab& T) {
  int l = T.ll[v >> (32 - kLutBits)];
  if (l < 0xFE) return l;
#pragma unroll 1
  for (int len = kLutBits + 1; len <= T.max_len; len++)
    if ((uint64_t)v < T.limit[len]) return len;
  return 0;
}

NBZG_DEV uint32_t code_sym(uint32_t v, int len, const DecTab& T) {
  uint32_t idx = (uint32_t)(T.base[len] + (int32_t)(v >> (32 - len)));
  return T.ss16 ? T.ss16[idx] : T.ss[idx];
}

// segmented (reset, k) scan element
struct KSeg {
  int r;
  long long v;
};
NBZG_DEV KSeg kseg_op(KSeg a, KSeg b) { return b.r ? b : KSeg{a.r, a.v + b.v}; }

// bit-serial canonical decode of one symbol straight from global bytes
// (fallback for chunks too large for the shared buffer, and the v1 path).
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
// Error handling rule: once a CTA holds a chunk ticket it ALWAYS publishes
// both look-back values (successors spin on them); failures only set the
// status word.
__global__ void __launch_bounds__(kDThreads) decode_kernel(DArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* W = reinterpret_cast<uint32_t*>(smem);                 // [kDBufWords + 4]
  uint16_t* S = reinterpret_cast<uint16_t*>(W + kDBufWords + 4);  // [16384]
  uint16_t* SS = S + kChunk;                                       // [kSmemSyms]
  uint8_t* LL = reinterpret_cast<uint8_t*>(SS + kSmemSyms);        // [1 << kLutBits]
  __shared__ uint64_t s_limit[64];
  __shared__ int32_t s_base[64];
  __shared__ uint32_t ends[kDThreads];
  __shared__ uint32_t scan_tmp[33];
  __shared__ KSeg kscan[33];
  __shared__ int64_t s_c;
  __shared__ unsigned long long s_eoff;
  __shared__ long long s_carry;
  __shared__ uint32_t s_err;

  const int fi = blockIdx.y;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if (F.kind != 3 || P.status || *a.status) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    s_c = atomicAdd(&a.tickets[fi], 1u);
    s_err = 0;
  }
  __syncthreads();
  const int64_t c = s_c;
  if (c >= a.nchunks) return;
  const uint64_t* choff = a.choff + fi * (a.nchunks + 1);
  const uint64_t B = choff[c];
  const uint32_t Lb = (uint32_t)(choff[c + 1] - B);
  const int64_t c0 = c * kChunk;
  const int mc = (int)min((int64_t)kChunk, a.n - c0);
  const int half = a.half;
  const uint32_t* ss = a.ssyms + fi * a.nbins;

  DecTab T;
  T.ll = LL;
  T.limit = s_limit;
  T.base = s_base;
  T.ss = ss;
  T.ss16 = P.k <= (uint64_t)kSmemSyms ? SS : nullptr;
  T.max_len = (int)P.max_len;
  {
    const uint32_t* gl = reinterpret_cast<const uint32_t*>(
        reinterpret_cast<const uint8_t*>(a.lut) + fi * (1 << kLutBits));
    uint32_t* sl = reinterpret_cast<uint32_t*>(LL);
    for (int i = tid; i < (1 << kLutBits) / 4; i += kDThreads) sl[i] = gl[i];
  }
  if (T.ss16)
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
  const bool big = (uint64_t)Lb + 64 > (uint64_t)kDBufWords * 32 || P.max_len > 32;
  if (big) {
    // rare: > 16 bits/symbol on average in this chunk -- sequential decode
    if (tid == 0) {
      uint64_t bp = B, total = B + Lb;
      for (int i = 0; i < mc; i++) {
        uint32_t sym = 0;
        int l = decode_serial(F.payload + P.bits_off, bp, total, P, ss, sym);
        if (l < 0) {
          s_err = (uint32_t)(-l);
          sym = 1;
        }
        S[i] = (uint16_t)sym;
      }
      if (bp != total && !s_err) s_err = NBZG_BAD_STREAM;
    }
    __syncthreads();
  } else {
    // ---- 1. stage bits: W[j] = 32 stream bits starting at chunk bit 32j (MSB-first)
    {
      const uint8_t* bits = F.payload + P.bits_off;
      const uint64_t byte0 = B >> 3;
      const uintptr_t addr = reinterpret_cast<uintptr_t>(bits) + byte0;
      const uint32_t* g = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
      const uint32_t sh = (uint32_t)((addr & 3) * 8 + (B & 7));
      const int nw = (int)((Lb + 31) / 32) + 2;
      const uint64_t avail_bytes =
          (uint64_t)(reinterpret_cast<uintptr_t>(F.payload + F.payload_len + 16) -
                     reinterpret_cast<uintptr_t>(g));
      for (int j = tid; j < nw; j += kDThreads) {
        uint32_t w0 = (4ull * j + 4 <= avail_bytes) ? __byte_perm(g[j], 0, 0x0123) : 0u;
        uint32_t w1 = (4ull * j + 8 <= avail_bytes) ? __byte_perm(g[j + 1], 0, 0x0123) : 0u;
        uint32_t v = sh ? __funnelshift_l(w1, w0, sh) : w0;
        int64_t endbit = (int64_t)Lb - 32ll * j;  // zero bits past the chunk end
        if (endbit <= 0) v = 0;
        else if (endbit < 32) v &= ~(0xffffffffu >> endbit);
        W[j] = v;
      }
    }
    __syncthreads();

    // ---- 2. self-synchronising decode over T_dec threads (>= kSegBits bits each).
    // Phase 1: every thread decodes its slice from an arbitrary bit, counting
    // codewords and remembering the first kRec codeword starts (registers).
    int tdec = (int)min((uint32_t)kDThreads, max(32u, ((Lb / kSegBits) + 31u) & ~31u));
    const bool active = tid < tdec;
    const uint32_t seg0 = active ? (uint32_t)(((uint64_t)Lb * tid) / tdec) : Lb;
    const uint32_t seg1 = active ? (uint32_t)(((uint64_t)Lb * (tid + 1)) / tdec) : Lb;
    uint32_t rec[kRec];
    int nrec = 0;
    uint32_t cnt = 0;
    uint32_t start = seg0;
    auto walk_full = [&](uint32_t s) -> uint32_t {  // decode [s, seg1): count + record
      uint32_t p = s;
      cnt = 0;
      nrec = 0;
      while (p < seg1) {
        int l = code_len(peek32(W, p), T);
        if (l == 0) {  // garbage from a wrong start (incomplete codes only): step a bit
          p += 1;
          continue;
        }
#pragma unroll
        for (int r = 0; r < kRec; r++)
          if (r == nrec) rec[r] = p;
        nrec = min(nrec + 1, kRec);
        cnt++;
        p += l;
      }
      return p;
    };
    if (active) ends[tid] = walk_full(seg0);
    __syncthreads();
    // Phase 2: thread t re-walks from its predecessor's true end until it lands
    // on one of its remembered starts (resynchronised: later codewords agree).
    int invalid = 0;
    for (int iter = 0; iter <= kDThreads; iter++) {
      int changed = 0;
      if (active && tid > 0) {
        uint32_t s = ends[tid - 1];
        if (s != start) {
          uint32_t q = s;
          int steps = 0, sync_j = -1;
          while (q < seg1) {
            int j = -1;
#pragma unroll
            for (int r = 0; r < kRec; r++)
              if (r < nrec && rec[r] == q) j = r;
            if (j >= 0) {
              sync_j = j;
              break;
            }
            if (nrec == kRec && q > rec[kRec - 1]) break;  // past the remembered window
            int l = code_len(peek32(W, q), T);
            if (l == 0) {
              invalid = 1;
              break;
            }
            q += l;
            steps++;
          }
          if (sync_j >= 0) {
            cnt = cnt - (uint32_t)sync_j + (uint32_t)steps;
            // refresh the remembered starts along the true path
            uint32_t p = s;
            int nr = 0;
            for (int r = 0; r < kRec && p < seg1; r++) {
              int l = code_len(peek32(W, p), T);
              if (l == 0) break;
#pragma unroll
              for (int r2 = 0; r2 < kRec; r2++)
                if (r2 == nr) rec[r2] = p;
              nr++;
              p += l;
            }
            nrec = nr;
          } else if (!invalid) {
            uint32_t e = walk_full(s);
            if (ends[tid] != e) changed = 1;
            ends[tid] = e;
          }
          start = s;
        }
      }
      if (!__syncthreads_or(changed)) break;
    }
    if (__syncthreads_or(invalid) && tid == 0) s_err = NBZG_INVALID_CODE;
    // ---- 3. output offsets and the final decode into shared memory
    uint32_t tot;
    uint32_t o = block_excl_scan<uint32_t>(active ? cnt : 0u, scan_tmp, &tot);
    if (tid == 0 && (tot != (uint32_t)mc || ends[tdec - 1] != Lb) && !s_err)
      s_err = tot < (uint32_t)mc ? NBZG_TRUNCATED : NBZG_BAD_STREAM;
    __syncthreads();
    if (!s_err && active) {
      uint32_t p = tid == 0 ? 0 : ends[tid - 1];
      int bad = 0;
      for (uint32_t i = 0; i < cnt; i++) {
        uint32_t v = peek32(W, p);
        int l = code_len(v, T);
        if (l == 0) {
          bad = 1;
          break;
        }
        if (o + i < (uint32_t)kChunk) S[o + i] = (uint16_t)code_sym(v, l, T);
        p += l;
      }
      if (bad) atomicCAS(&s_err, 0u, (uint32_t)NBZG_INVALID_CODE);
    }
    __syncthreads();
    if (s_err)
      for (int i = tid; i < mc; i += kDThreads) S[i] = 1;  // keep going: publish look-backs
    __syncthreads();
  }

  // ---- 4. dequantise (orc_dq_dequantize)
  const int q0 = tid * kDPer;
  const int qn = max(0, min(kDPer, mc - q0));
  uint32_t my_esc = 0;
  for (int j = 0; j < qn; j++) my_esc += S[q0 + j] == 0;
  uint32_t etot;
  uint32_t eo = block_excl_scan<uint32_t>(my_esc, scan_tmp, &etot);
  if (tid < 32) {
    uint64_t eo2 = lookback_sum(a.lb + (fi * 2 + 0) * a.nchunks, c, etot);
    if (tid == 0) s_eoff = eo2;
  }
  __syncthreads();
  const uint8_t* escp = F.payload + P.esc_off;
  const uint64_t e_idx = s_eoff + eo;
  const bool esc_ok = e_idx + my_esc <= P.n_esc;
  if (!esc_ok) atomicCAS(&s_err, 0u, (uint32_t)NBZG_BAD_STREAM);
  KSeg agg{0, 0};
  {
    uint64_t ei = e_idx;
    for (int j = 0; j < qn; j++) {
      uint32_t code = S[q0 + j];
      if (code == 0) {
        float v = esc_ok ? __uint_as_float(ld_u32_bytes(escp + 4 * ei)) : 0.0f;
        ei++;
        bool fast;
        double kd = lattice_index<false>(v, F.inv32, F.inv, F.twob, fast);
        if (!fast) kd = fmin(fmax(kd, -kDqKmax), kDqKmax);
        agg = KSeg{1, (long long)kd};
      } else {
        agg.v += (long long)((int)code - half - 1);
      }
    }
  }
  // block-wide exclusive segmented scan of agg
  KSeg inc = agg;
#pragma unroll
  for (int o2 = 1; o2 < 32; o2 <<= 1) {
    KSeg u;
    u.r = __shfl_up_sync(0xffffffffu, inc.r, o2);
    u.v = __shfl_up_sync(0xffffffffu, inc.v, o2);
    if (lane >= o2) inc = kseg_op(u, inc);
  }
  if (lane == 31) kscan[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    KSeg wi = kscan[lane];
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
      KSeg u;
      u.r = __shfl_up_sync(0xffffffffu, wi.r, o2);
      u.v = __shfl_up_sync(0xffffffffu, wi.v, o2);
      if (lane >= o2) wi = kseg_op(u, wi);
    }
    KSeg ex;
    ex.r = __shfl_up_sync(0xffffffffu, wi.r, 1);
    ex.v = __shfl_up_sync(0xffffffffu, wi.v, 1);
    if (lane == 0) ex = KSeg{0, 0};
    __syncwarp();
    kscan[lane] = ex;
    if (lane == 31) kscan[32] = wi;  // chunk aggregate
  }
  __syncthreads();
  KSeg exw;
  exw.r = __shfl_up_sync(0xffffffffu, inc.r, 1);
  exw.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
  if (lane == 0) exw = KSeg{0, 0};
  KSeg before = kseg_op(kscan[wid], exw);
  if (tid < 32) {
    KSeg ca = kscan[32];
    long long cr = lookback_kcarry(a.lb + (fi * 2 + 1) * a.nchunks, c, ca.r != 0, ca.v);
    if (tid == 0) {
      s_carry = cr;
      if (s_err) fail(a.status, s_err);
    }
  }
  __syncthreads();
  long long k = before.r ? before.v : s_carry + before.v;
  float outv[kDPer];
  {
    uint64_t ei = e_idx;
#pragma unroll
    for (int j = 0; j < kDPer; j++) {
      outv[j] = 0.0f;
      if (j < qn) {
        uint32_t code = S[q0 + j];
        if (code == 0) {
          float v = esc_ok ? __uint_as_float(ld_u32_bytes(escp + 4 * ei)) : 0.0f;
          ei++;
          bool fast;
          double kd = lattice_index<false>(v, F.inv32, F.inv, F.twob, fast);
          if (!fast) kd = fmin(fmax(kd, -kDqKmax), kDqKmax);
          k = (long long)kd;
          outv[j] = v;
        } else {
          k += (long long)((int)code - half - 1);
          outv[j] = (float)__dmul_rn((double)k, F.twob);
        }
      }
    }
  }
  float* dst = F.out + c0 + q0;
  if (qn == kDPer && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; q++)
      d4[q] = make_float4(outv[4 * q], outv[4 * q + 1], outv[4 * q + 2], outv[4 * q + 3]);
  } else {
    for (int j = 0; j < qn; j++) dst[j] = outv[j];
  }
}

// ---------------------------------------------------------------- v1 compat
// Reference SZ_FIELD streams: bit-serial decode + the exact sequential chain
// (_kernels.py:126-147), one thread per field.  Compatibility path only.
__global__ void decode_v1_kernel(DArgs a) {
  const int fi = blockIdx.x;
  const DField& F = a.f[fi];
  const DParsed& P = a.parsed[fi];
  if (F.kind != 0 || P.status || threadIdx.x != 0) return;
  const uint8_t* bits = F.payload + P.bits_off;
  const uint8_t* escp = F.payload + P.esc_off;
  const uint32_t* ss = a.ssyms + fi * a.nbins;
  const int half = a.half;
  uint64_t bp = 0, ei = 0;
  double h1 = 0.0;
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
      double pred = i == 0 ? 0.0 : h1;
      double q = (double)((int)sym - half - 1);
      r = (float)__dadd_rn(pred, __dmul_rn(q, F.twob));
    }
    F.out[i] = r;
    h1 = (double)r;
  }
  if (ei != P.n_esc) fail(a.status, NBZG_BAD_STREAM);
}

// ---------------------------------------------------------------- launcher
size_t decompress_ws(int nf, int64_t n, int64_t nbins) {
  int64_t nchunks = (n + kChunk - 1) / kChunk;
  size_t s = 0;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  s += al(sizeof(DParsed) * nf);
  s += al((size_t)nf * (1 << kLutBits));
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
  parse_kernel<<<nf, 1024, 0, st>>>(a);
  trace_mark("dq_parse", st);
  count_launch();
  chunk_offsets_kernel<<<nf, 1024, 0, st>>>(a);
  trace_mark("dq_offsets", st);
  size_t sm = (kDBufWords + 4) * 4 + kChunk * 2 + kSmemSyms * 2 + (1 << kLutBits);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  bool any_v2 = false, any_v1 = false;
  for (int i = 0; i < nf; i++) {
    any_v2 |= fields[i].kind == 3;
    any_v1 |= fields[i].kind == 0;
  }
  if (any_v2) {
    count_launch();
    decode_kernel<<<dim3((unsigned)a.nchunks, nf), kDThreads, sm, st>>>(a);
  }
  if (any_v2) trace_mark("dq_decode", st);
  if (any_v1) {
    count_launch();
    decode_v1_kernel<<<nf, 32, 0, st>>>(a);
    trace_mark("dq_decode_v1", st);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
