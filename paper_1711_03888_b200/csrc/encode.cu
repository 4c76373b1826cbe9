// encode.cu -- K6/K7: v2 SZ_DQ payload writer and the warp-per-chunk Huffman
// encoder.  Replaces encode.huffman_encode (encode.py:222-239) ->
// K.huff_encode (_kernels.py:304-345) and the stream framing of
// pipeline._build_sz_stream (pipeline.py:188-200).
//
// Payload (all little-endian):
//   u32 n_esc | u32 k | k x (u32 sym, u8 len) | u64 bit_length
//   | u32 chunk_bits[ceil(n/16384)] | pad to 4 | bitstream (MSB-first,
//   padded to 4 bytes; every escape code is followed inline by the 32 bits
//   of the escaped float32)
//
// Encoder: one WARP per 16384-code chunk (per-field ticket order), 8 warps
// per CTA, many CTAs per SM so look-back waits are hidden.  Lane l owns
// codes [512 l, 512 l + 512) of the chunk:
//   1. bit count of its codes (u64 LUT (len << 57) | word, +32 per escape);
//   2. warp scan -> lane bit offsets; the chunk total is published at once
//      and a warp-parallel decoupled look-back gives the chunk's global bit
//      offset;
//   3. each lane streams its codes through a 64-bit accumulator and stores
//      every complete big-endian 32-bit word it owns directly; its first and
//      last partial words go to per-warp shared slots and are OR-merged with
//      the neighbours' parts.  A word belongs to the chunk holding its first
//      bit; a chunk ending mid-word appends the first bits of the next chunk
//      (encoded on the spot), so every word is written exactly once -- no
//      zero fill, no global atomics.
#include <cstdio>
#include <cstdlib>

#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kEWarps = 8;
constexpr int kEThreads = kEWarps * 32;
constexpr int kELane = kChunk / 32;  // 512 codes per lane

NBZG_DEV void put_u32_bytes(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v;
  p[1] = (uint8_t)(v >> 8);
  p[2] = (uint8_t)(v >> 16);
  p[3] = (uint8_t)(v >> 24);
}
NBZG_DEV void put_u64_bytes(uint8_t* p, uint64_t v) {
  put_u32_bytes(p, (uint32_t)v);
  put_u32_bytes(p + 4, (uint32_t)(v >> 32));
}

// ---------------------------------------------------------------- table writer
struct TArgs {
  nbzg_meta* meta;
  uint8_t* arena;
  const uint32_t* sym;  // [6][nbins]
  const uint8_t* len;   // [6][nbins]
  int64_t nbins;
  int64_t nchunks;
  int64_t n;
  int f0;               // CTA b -> field f0 + b
};

__global__ void table_writer_kernel(TArgs a) {
  const int field = a.f0 + (int)blockIdx.x;
  const nbzg_field_meta& m = a.meta->f[field];
  if (m.is_const || a.n == 0 || a.meta->status) return;
  uint8_t* p = a.arena + m.payload_off;
  const uint32_t* sym = a.sym + field * a.nbins;
  const uint8_t* len = a.len + field * a.nbins;
  if (threadIdx.x == 0) {
    put_u32_bytes(p, (uint32_t)m.n_esc);
    put_u32_bytes(p + 4, m.k);
    put_u64_bytes(p + 8 + 5 * (uint64_t)m.k, m.total_bits);
    for (uint64_t q = m.index_off + 4 * (uint64_t)a.nchunks; q < m.bits_off; q++) p[q] = 0;
  }
  for (uint32_t i = threadIdx.x; i < m.k; i += blockDim.x) {
    uint8_t* e = p + 8 + 5 * (uint64_t)i;
    put_u32_bytes(e, sym[i]);
    e[4] = len[i];
  }
}

// ---------------------------------------------------------------- encoder
struct EArgs {
  nbzg_meta* meta;
  uint8_t* arena;
  const uint16_t* codes;  // [6][code_stride]
  int64_t code_stride;
  const uint64_t* lut;    // [6][nbins]
  const uint32_t* twin;   // [6][kEncWin] (payload path: staged in smem)
  const uint8_t* tlen8;   // [6][nbins] code lengths (chunk bit counts)
  int64_t nbins;
  int64_t n, nchunks;
  const float* f[6];
  const uint16_t* perm;   // null if unsorted
  int64_t tile;
  uint64_t* lb;           // [6][nchunks]
  uint32_t* tickets;      // [6]
  int inline_esc;         // 1: payload mode (escape values inline); 0: raw hook
  int f0;                 // field of blockIdx.y (or .x) 0 (field groups)
  // parity-hook mode: raw bitstream output instead of a payload
  uint8_t* raw_out;
  uint32_t* raw_chunk_bits;
};

NBZG_DEV uint32_t esc_value_bits(const EArgs& a, int field, int64_t pos) {
  int64_t src = a.perm ? (pos / a.tile) * a.tile + a.perm[pos] : pos;
  return __float_as_uint(a.f[field][src]);
}

// 64-bit MSB-aligned bit accumulator
struct Acc {
  uint64_t acc;
  int nacc;
};

template <typename Emit>
NBZG_DEV void acc_put(Acc& A, uint64_t v, int nb, Emit&& emit) {
  while (nb > 0) {
    int take = nb < 32 ? nb : 32;
    uint64_t piece = (v >> (nb - take)) & ((1ull << take) - 1);
    A.acc |= piece << (64 - A.nacc - take);
    A.nacc += take;
    nb -= take;
    if (A.nacc >= 32) {
      emit((uint32_t)(A.acc >> 32));
      A.acc <<= 32;
      A.nacc -= 32;
    }
  }
}

// code-word lookup through the global u64 LUT (hook path; slow path of the
// payload encoder)
struct CodeTab {
  const uint64_t* lut;
};
template <bool FAST>
NBZG_DEV uint32_t code_len(const CodeTab& T, uint32_t code) {
  return (uint32_t)(__ldg(&T.lut[code]) >> 57);
}
template <bool FAST>
NBZG_DEV uint64_t code_word(const CodeTab& T, uint32_t code, uint32_t& l) {
  const uint64_t e = __ldg(&T.lut[code]);
  l = (uint32_t)(e >> 57);
  return e & ((1ull << 57) - 1);
}

// first `need` (1..31) bits of chunk c1's stream, MSB-aligned (serial, one lane)
template <bool FAST>
NBZG_DEV uint32_t chunk_head_bits(const EArgs& a, int field, const uint16_t* codes,
                                  const CodeTab& T, int64_t c1, int need) {
  const int64_t s0 = c1 * kChunk, s1 = min(a.n, s0 + kChunk);
  uint64_t acc = 0;
  int nacc = 0;
  for (int64_t i = s0; i < s1 && nacc < need; i++) {
    uint32_t code = codes[i];
    uint32_t lu;
    uint64_t w = code_word<FAST>(T, code, lu);
    int l = (int)lu;
    if (l > 32) {  // only the leading bits can still land in the window
      w >>= (l - 32);
      l = 32;
    }
    acc |= (w << (64 - l)) >> nacc;
    nacc += l;
    if (code == 0 && a.inline_esc && nacc < need) {
      acc |= ((uint64_t)esc_value_bits(a, field, i) << 32) >> nacc;
      nacc += 32;
    }
  }
  uint32_t top = (uint32_t)(acc >> 32);
  return top & ~(0xffffffffu >> need);
}

// one chunk, one warp (see the file comment)
template <bool FAST>
NBZG_DEV void encode_chunk(const EArgs& a, int field, int64_t c, const CodeTab& T,
                           long long* s_idx, uint32_t* s_bits) {
  const int lane = threadIdx.x & 31;
  const bool raw = a.raw_out != nullptr;
  const nbzg_field_meta* mp = raw ? nullptr : &a.meta->f[field];
  const uint16_t* codes = a.codes + field * a.code_stride;
  uint8_t* payload = raw ? nullptr : a.arena + mp->payload_off;
  uint32_t* outw = raw ? reinterpret_cast<uint32_t*>(a.raw_out)
                       : reinterpret_cast<uint32_t*>(payload + mp->bits_off);
  const int64_t c0 = c * kChunk;
  const int mc = (int)min((int64_t)kChunk, a.n - c0);
  const int lo = lane * kELane;
  const int cnt = max(0, min(kELane, mc - lo));
  const uint16_t* cp = codes + c0 + lo;
  const bool vec = ((reinterpret_cast<uintptr_t>(cp) & 15) == 0);

  // ---- 1. bits of this lane's codes
  uint32_t bits = 0;
  for (int j = 0; j < cnt; j += 8) {
    uint16_t cv[8];
    if (vec && j + 8 <= cnt) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(cp + j));
      uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 8; q++) cv[q] = (uint16_t)(w4[q >> 1] >> ((q & 1) * 16));
    } else {
#pragma unroll
      for (int q = 0; q < 8; q++) cv[q] = j + q < cnt ? cp[j + q] : (uint16_t)0xffff;
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (j + q < cnt) {
        bits += code_len<FAST>(T, cv[q]);
        if (cv[q] == 0 && a.inline_esc) bits += 32;
      }
    }
  }
  const uint32_t incl = warp_incl_scan<uint32_t>(bits);
  const uint32_t off = incl - bits;
  const uint32_t Tt = __shfl_sync(0xffffffffu, incl, 31);

  // ---- 2. publish, look back for the chunk's global bit offset
  uint64_t* lbb = a.lb + field * a.nchunks;
  if (lane == 0 && c > 0) lb_store(&lbb[c], kFlagAgg | Tt);
  const uint64_t B = lookback_sum(lbb, c, Tt);
  if (lane == 0) {
    if (raw) a.raw_chunk_bits[c] = Tt;
    else put_u32_bytes(payload + mp->index_off + 4 * c, Tt);
  }

  // ---- 3. pack
  const uint64_t g0 = B + off;
  uint64_t widx = g0 >> 5;
  Acc A{0ull, (int)(g0 & 31)};
  bool head_pending = (g0 & 31) != 0;
  long long head_idx = -1, tail_idx = -1;
  uint32_t head_bits = 0, tail_bits = 0;
  auto emit = [&](uint32_t w) {
    if (head_pending) {
      head_idx = (long long)widx;
      head_bits = w;
      head_pending = false;
    } else {
#ifdef NBZG_BOUNDS
      if (!raw && widx * 4 + mp->bits_off + 4 > mp->payload_len) {
        printf("OOB emit field %d chunk %lld lane %d widx %llu B %llu off %u bits %u T %u plen %llu boff %llu\n", field, (long long)c, lane, (unsigned long long)widx, (unsigned long long)B, off, bits, Tt, (unsigned long long)mp->payload_len, (unsigned long long)mp->bits_off);
        __trap();
      }
#endif
      outw[widx] = __byte_perm(w, 0, 0x0123);
    }
    widx++;
  };
  for (int j = 0; j < cnt; j += 8) {
    uint16_t cv[8];
    if (vec && j + 8 <= cnt) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(cp + j));
      uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 8; q++) cv[q] = (uint16_t)(w4[q >> 1] >> ((q & 1) * 16));
    } else {
#pragma unroll
      for (int q = 0; q < 8; q++) cv[q] = j + q < cnt ? cp[j + q] : (uint16_t)0xffff;
    }
    uint64_t e[8];
    uint32_t el[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      el[q] = 0;
      e[q] = j + q < cnt ? code_word<FAST>(T, cv[q], el[q]) : 0ull;
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (j + q < cnt) {
        acc_put(A, e[q], (int)el[q], emit);
        if (cv[q] == 0 && a.inline_esc)
          acc_put(A, esc_value_bits(a, field, c0 + lo + j + q), 32, emit);
      }
    }
  }
  if (bits > 0 && A.nacc > 0) {
    // final partial word (also the first word when the lane never filled one)
    tail_idx = (long long)widx;
    tail_bits = (uint32_t)(A.acc >> 32);
  }
  __syncwarp();
  s_idx[2 * lane] = head_idx;
  s_bits[2 * lane] = head_bits;
  s_idx[2 * lane + 1] = tail_idx;
  s_bits[2 * lane + 1] = tail_bits;
  __syncwarp();

  // ---- 4. merge boundary words (lane 0): OR the parts of each word
  if (lane == 0 && Tt > 0) {
    const uint64_t Bend = B + Tt;
    const long long first_owned = (long long)((B + 31) >> 5);
    const long long last_word = (long long)((Bend - 1) >> 5);
    long long cur = -1;
    uint32_t acc = 0;
    auto flush = [&](long long idx, uint32_t w) {
      if (idx < first_owned) return;  // belongs to the previous chunk
      if (idx == last_word && (Bend & 31) && c + 1 < a.nchunks) {
        int need = 32 - (int)(Bend & 31);
        w |= chunk_head_bits<FAST>(a, field, codes, T, c + 1, need) >> (Bend & 31);
      }
#ifdef NBZG_BOUNDS
      if (!raw && idx * 4 + mp->bits_off + 4 > mp->payload_len) {
        printf("OOB merge field %d chunk %lld idx %lld B %llu T %u\n", field, (long long)c, idx, (unsigned long long)B, Tt);
        __trap();
      }
#endif
      outw[idx] = __byte_perm(w, 0, 0x0123);
    };
    for (int s = 0; s < 64; s++) {
      long long idx = s_idx[s];
      if (idx < 0) continue;
      if (idx == cur) {
        acc |= s_bits[s];
      } else {
        if (cur >= 0) flush(cur, acc);
        cur = idx;
        acc = s_bits[s];
      }
    }
    if (cur >= 0) flush(cur, acc);
  }
}

// hook path: one warp per ticketed chunk, global LUT
__global__ void __launch_bounds__(kEThreads) encode_kernel(EArgs a) {
  __shared__ long long s_idx[kEWarps][64];
  __shared__ uint32_t s_bits[kEWarps][64];
  const int field = a.f0 + (int)blockIdx.y;
  const bool raw = a.raw_out != nullptr;
  if (!raw && (a.meta->f[field].is_const || a.n == 0 || a.meta->status)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t c = 0;
  if (lane == 0) c = atomicAdd(&a.tickets[field], 1u);
  c = __shfl_sync(0xffffffffu, c, 0);
  if (c >= a.nchunks) return;
  CodeTab T{a.lut + field * a.nbins};
  encode_chunk<false>(a, field, c, T, s_idx[warp], s_bits[warp]);
}

// ---- payload path.  Code words of the codes nearest the centre (deltas in
// [-8192, 8191], length <= 26: all but a few per mille of the codes) come
// from a 64 KiB shared-memory window table, one LDS per code; the rest from
// the global LUT.  Code loads are software-pipelined one 8-code group ahead.
struct WinTab {
  const uint32_t* win;  // smem [kEncWin]
  uint32_t wlo;         // code of win[0]
  const uint64_t* lut;  // global fallback
};
NBZG_DEV uint32_t win_len(const WinTab& T, uint32_t code) {
  const uint32_t wi = code - T.wlo;
  const uint32_t e = wi < (uint32_t)kEncWin ? T.win[wi] : 0u;
  return e ? (e & 63u) : (uint32_t)(__ldg(&T.lut[code]) >> 57);
}
// (word, len); returns false when the word came from the global LUT
NBZG_DEV bool win_word(const WinTab& T, uint32_t code, uint64_t& w, uint32_t& l) {
  const uint32_t wi = code - T.wlo;
  const uint32_t e = wi < (uint32_t)kEncWin ? T.win[wi] : 0u;
  if (e) {
    l = e & 63u;
    w = (e & ~63u) >> (32 - l);  // entries hold the MSB-aligned word
    return true;
  }
  const uint64_t g = __ldg(&T.lut[code]);
  l = (uint32_t)(g >> 57);
  w = g & ((1ull << 57) - 1);
  return false;
}

NBZG_DEV uint32_t chunk_head_bits_w(const EArgs& a, int field, const uint16_t* codes,
                                    const WinTab& T, int64_t c1, int need) {
  const int64_t s0 = c1 * kChunk, s1 = min(a.n, s0 + kChunk);
  uint64_t acc = 0;
  int nacc = 0;
  for (int64_t i = s0; i < s1 && nacc < need; i++) {
    const uint32_t code = codes[i];
    uint64_t w;
    uint32_t lu;
    win_word(T, code, w, lu);
    int l = (int)lu;
    if (l > 32) {
      w >>= (l - 32);
      l = 32;
    }
    acc |= (w << (64 - l)) >> nacc;
    nacc += l;
    if (code == 0 && nacc < need) {
      acc |= ((uint64_t)esc_value_bits(a, field, i) << 32) >> nacc;
      nacc += 32;
    }
  }
  return (uint32_t)(acc >> 32) & ~(0xffffffffu >> need);
}

NBZG_DEV void st_pred_u32(uint32_t* p, uint32_t v, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.global.u32 [%0], %1;\n}\n" ::"l"(p),
      "r"(v), "r"((uint32_t)pred)
      : "memory");
}

NBZG_DEV void st_pred_v4(uint32_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %5, 0;\n"
      " @p st.global.v4.u32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(p),
      "r"(a), "r"(b), "r"(c), "r"(d), "r"((uint32_t)pred)
      : "memory");
}

NBZG_DEV void st_pred_v8(uint32_t* p, const uint32_t (&q)[7], uint32_t w, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %9, 0;\n"
      " @p st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n}\n" ::"l"(p),
      "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(w),
      "r"((uint32_t)pred)
      : "memory");
}

NBZG_DEV void unpack8(uint4 u, uint32_t (&cv)[8]) {
  cv[0] = u.x & 0xffffu; cv[1] = u.x >> 16;
  cv[2] = u.y & 0xffffu; cv[3] = u.y >> 16;
  cv[4] = u.z & 0xffffu; cv[5] = u.z >> 16;
  cv[6] = u.w & 0xffffu; cv[7] = u.w >> 16;
}

NBZG_DEV void encode_chunk_fast(const EArgs& a, int field, int64_t c, const WinTab& T,
                                long long* s_idx, uint32_t* s_bits, uint32_t* s_headw) {
  const int lane = threadIdx.x & 31;
  const nbzg_field_meta* mp = &a.meta->f[field];
  const uint16_t* codes = a.codes + field * a.code_stride;
  uint8_t* payload = a.arena + mp->payload_off;
  uint32_t* outw = reinterpret_cast<uint32_t*>(payload + mp->bits_off);
  const int64_t c0 = c * kChunk;
  const int mc = (int)min((int64_t)kChunk, a.n - c0);
  const int lo = lane * kELane;
  const int cnt = max(0, min(kELane, mc - lo));
  const int cnt8 = cnt & ~7;  // full 8-code groups (codes are 16-byte aligned)
  const uint16_t* cp = codes + c0 + lo;
  const uint4* cp4 = reinterpret_cast<const uint4*>(cp);

  // ---- 1. bits of this lane's codes (per 8-code group: window lookups,
  // and the global LUT only for a group holding a miss)
  uint32_t bits = 0;
  const int ng = cnt8 >> 3;  // 8-code groups; loads run 3 groups ahead
  {
    uint4 n0 = ng > 0 ? __ldg(cp4) : make_uint4(0, 0, 0, 0);
    uint4 n1 = ng > 1 ? __ldg(cp4 + 1) : make_uint4(0, 0, 0, 0);
    uint4 n2 = ng > 2 ? __ldg(cp4 + 2) : make_uint4(0, 0, 0, 0);
    for (int j = 0; j < cnt8; j += 8) {
      const uint4 cur = n0;
      n0 = n1;
      n1 = n2;
      if ((j >> 3) + 3 < ng) n2 = __ldg(cp4 + (j >> 3) + 3);
      uint32_t cv[8], e[8];
      unpack8(cur, cv);
      bool hit = true;
      uint32_t gb = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint32_t wi = cv[q] - T.wlo;
        e[q] = wi < (uint32_t)kEncWin ? T.win[wi] : 0u;
        hit &= e[q] != 0;
        gb += e[q] & 63u;
      }
      if (!hit) {
        gb = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) gb += win_len(T, cv[q]) + (cv[q] == 0 ? 32u : 0u);
      }
      bits += gb;
    }
    for (int j = cnt8; j < cnt; j++) {
      const uint32_t code = cp[j];
      bits += win_len(T, code) + (code == 0 ? 32u : 0u);
    }
  }
  const uint32_t incl = warp_incl_scan<uint32_t>(bits);
  const uint32_t off = incl - bits;
  const uint32_t Tt = __shfl_sync(0xffffffffu, incl, 31);

  // ---- 2. publish, look back for the chunk's global bit offset
  uint64_t* lbb = a.lb + field * a.nchunks;
  if (lane == 0 && c > 0) lb_store(&lbb[c], kFlagAgg | Tt);
  const uint64_t B = lookback_sum(lbb, c, Tt);
  if (lane == 0) put_u32_bytes(payload + mp->index_off + 4 * c, Tt);

  // ---- 3. pack: 64-bit MSB-aligned accumulator, nacc < 32 between codes.
  // Completed words go to consecutive addresses through a running pointer;
  // a lane starting mid-word sends its first (partial) word to a shared
  // slot instead (it is OR-merged with the neighbour's bits in step 4).
  const uint64_t g0 = B + off;
  const uint64_t widx0 = g0 >> 5;
  uint64_t acc = 0;
  uint32_t nacc = (uint32_t)(g0 & 31);
  const bool head_partial = nacc != 0;
  uint32_t* wp = head_partial ? s_headw + lane : outw + widx0;  // generic pointer
  uint32_t* wn = outw + widx0 + 1;
  uint32_t nemit = 0;
  auto emit = [&](uint32_t w) {
    *wp = __byte_perm(w, 0, 0x0123);
    wp = wn;
    wn++;
    nemit++;
  };
  auto append = [&](uint32_t w, uint32_t l) {  // l <= 26
    acc |= (uint64_t)w << (64 - nacc - l);
    nacc += l;
    if (nacc >= 32) {
      emit((uint32_t)(acc >> 32));
      acc <<= 32;
      nacc -= 32;
    }
  };
  // slow append of up to 57 bits (long codes, escapes)
  auto put_slow = [&](uint64_t v, uint32_t nb) {
    Acc A{acc, (int)nacc};
    acc_put(A, v, (int)nb, emit);
    acc = A.acc;
    nacc = (uint32_t)A.nacc;
  };
  auto put_code = [&](uint32_t code, int64_t pos) {
    uint64_t w;
    uint32_t l;
    win_word(T, code, w, l);
    put_slow(w, l);
    if (code == 0) put_slow(esc_value_bits(a, field, pos), 32);
  };
  {
    uint4 n0 = ng > 0 ? __ldg(cp4) : make_uint4(0, 0, 0, 0);
    uint4 n1 = ng > 1 ? __ldg(cp4 + 1) : make_uint4(0, 0, 0, 0);
    uint4 n2 = ng > 2 ? __ldg(cp4 + 2) : make_uint4(0, 0, 0, 0);
    for (int j = 0; j < cnt8; j += 8) {
      const uint4 cur = n0;
      n0 = n1;
      n1 = n2;
      if ((j >> 3) + 3 < ng) n2 = __ldg(cp4 + (j >> 3) + 3);
      uint32_t cv[8], e[8];
      unpack8(cur, cv);
      bool hit = true;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint32_t wi = cv[q] - T.wlo;
        e[q] = wi < (uint32_t)kEncWin ? T.win[wi] : 0u;
        hit &= e[q] != 0;
      }
      if (hit) {
#pragma unroll
        for (int q = 0; q < 8; q++) append((e[q] & ~63u) >> (32 - (e[q] & 63u)), e[q] & 63u);
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) put_code(cv[q], c0 + lo + j + q);
      }
    }
    for (int j = cnt8; j < cnt; j++) put_code(cp[j], c0 + lo + j);
  }
  long long head_idx = -1, tail_idx = -1;
  uint32_t head_bits = 0, tail_bits = 0;
  __syncwarp();
  if (head_partial && nemit > 0) {
    head_idx = (long long)widx0;
    head_bits = __byte_perm(s_headw[lane], 0, 0x0123);
  }
  if (bits > 0 && nacc > 0) {
    // final partial word (also the first word when the lane never filled one)
    tail_idx = (long long)(widx0 + nemit);
    tail_bits = (uint32_t)(acc >> 32);
  }
  __syncwarp();
  s_idx[2 * lane] = head_idx;
  s_bits[2 * lane] = head_bits;
  s_idx[2 * lane + 1] = tail_idx;
  s_bits[2 * lane + 1] = tail_bits;
  __syncwarp();

  // ---- 4. merge boundary words (lane 0)
  if (lane == 0 && Tt > 0) {
    const uint64_t Bend = B + Tt;
    const long long first_owned = (long long)((B + 31) >> 5);
    const long long last_word = (long long)((Bend - 1) >> 5);
    long long cur = -1;
    uint32_t accw = 0;
    auto flush = [&](long long idx, uint32_t w) {
      if (idx < first_owned) return;  // belongs to the previous chunk
      if (idx == last_word && (Bend & 31) && c + 1 < a.nchunks) {
        const int need = 32 - (int)(Bend & 31);
        w |= chunk_head_bits_w(a, field, codes, T, c + 1, need) >> (Bend & 31);
      }
      outw[idx] = __byte_perm(w, 0, 0x0123);
    };
    for (int s = 0; s < 64; s++) {
      const long long idx = s_idx[s];
      if (idx < 0) continue;
      if (idx == cur) {
        accw |= s_bits[s];
      } else {
        if (cur >= 0) flush(cur, accw);
        cur = idx;
        accw = s_bits[s];
      }
    }
    if (cur >= 0) flush(cur, accw);
  }
}

// payload path: persistent CTAs (one field each) stage the field's window
// table in shared memory, then each warp encodes ticketed chunks until the
// field is done
constexpr int kEFWarps = 16;
__global__ void __launch_bounds__(kEFWarps * 32, 2) encode_fast_kernel(EArgs a) {
  extern __shared__ __align__(16) uint8_t esm[];
  uint32_t* s_win = reinterpret_cast<uint32_t*>(esm);                 // [kEncWin]
  long long* s_idx = reinterpret_cast<long long*>(s_win + kEncWin);  // [warps][64]
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_idx + kEFWarps * 64);
  uint32_t* s_headw = s_bits + kEFWarps * 64;                         // [warps][32]
  const int field = a.f0 + (int)blockIdx.y;
  if (a.meta->f[field].is_const || a.n == 0 || a.meta->status) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const uint4* g = reinterpret_cast<const uint4*>(a.twin + (size_t)field * kEncWin);
    for (int i = threadIdx.x; i < kEncWin / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(s_win)[i] = __ldg(g + i);
  }
  __syncthreads();
  const WinTab T{s_win, (uint32_t)(a.nbins / 2 + 1 - kEncWin / 2), a.lut + field * a.nbins};
  while (true) {
    int64_t c = 0;
    if (lane == 0) c = atomicAdd(&a.tickets[field], 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= a.nchunks) return;
    encode_chunk_fast(a, field, c, T, s_idx + warp * 64, s_bits + warp * 64, s_headw + warp * 32);
  }
}

// ---- block-parallel payload encoder (>= kTpcEncMinChunks chunks/field).
// A chunk's 16384 codes are 32 blocks of 512.  E1 counts every block's bits
// (one warp per chunk, coalesced code loads, 64 KiB smem length table); E2
// scans them per field into block bit offsets (and writes the v2 chunk
// index); E3 packs each block with ONE thread at its known offset: no
// look-back, no merges.  A block writes the words whose first bit it holds;
// its last, partial word is completed with the leading bits of the stream
// after it (a few codes of lookahead).  With the field-group overlap this
// path wins from 128 chunks per field up (whole compress 0.44 vs 0.47 ms at
// 128, 0.91 vs 1.06 ms at 1024, 2.47 vs 2.83 ms at 4096 chunks; equal at 64:
// scripts/path_crossover.py).
constexpr int kTpcEncMinChunks = 128;
constexpr int kBlk = 512;                  // codes per block (= warp encoder's lane share)
constexpr int kBlkPerChunk = kChunk / kBlk;
constexpr int kE1Warps = 16;

// leading `need` (1..31) bits of the stream from code s0 on, MSB-aligned
NBZG_DEV uint32_t head_bits_from(const EArgs& a, int field, const uint16_t* codes,
                                 const WinTab& T, int64_t s0, int need) {
  uint64_t acc = 0;
  int nacc = 0;
  for (int64_t i = s0; i < a.n && nacc < need; i++) {
    const uint32_t code = codes[i];
    uint64_t w;
    uint32_t lu;
    win_word(T, code, w, lu);
    int l = (int)lu;
    if (l > 32) {
      w >>= (l - 32);
      l = 32;
    }
    acc |= (w << (64 - l)) >> nacc;
    nacc += l;
    if (code == 0 && nacc < need) {
      acc |= ((uint64_t)esc_value_bits(a, field, i) << 32) >> nacc;
      nacc += 32;
    }
  }
  return (uint32_t)(acc >> 32) & ~(0xffffffffu >> need);
}

__global__ void __launch_bounds__(kE1Warps * 32, 2) chunk_bits_kernel(EArgs a, uint32_t* bbits,
                                                                      uint32_t* ctot,
                                                                      int ctas_per_field) {
  extern __shared__ __align__(16) uint8_t e1sm[];
  uint8_t* s_len = e1sm;  // [nbins]
  const int field = a.f0 + (int)blockIdx.y;
  if (a.meta->f[field].is_const || a.n == 0 || a.meta->status) return;
  {
    const uint4* g = reinterpret_cast<const uint4*>(a.tlen8 + (size_t)field * a.nbins);
    for (int i = threadIdx.x; i < (int)(a.nbins / 16); i += blockDim.x)
      reinterpret_cast<uint4*>(s_len)[i] = __ldg(g + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * kE1Warps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)ctas_per_field * kE1Warps;
  const uint16_t* codes = a.codes + field * a.code_stride;
  uint32_t* bb = bbits + (size_t)field * a.nchunks * kBlkPerChunk;
  for (int64_t c = wg; c < a.nchunks; c += nw) {
    const int64_t c0 = c * kChunk;
    const int mc = (int)min((int64_t)kChunk, a.n - c0);
    const uint4* cp4 = reinterpret_cast<const uint4*>(codes + c0);
    uint32_t mine = 0;  // lane b keeps block b's count
    if (mc == kChunk) {
      // full chunk: four blocks per step, their eight 16-byte loads per lane
      // issued before any is consumed
#pragma unroll 1
      for (int b = 0; b < kBlkPerChunk; b += 4) {
        uint4 q[8];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          q[2 * u] = __ldg(cp4 + (b + u) * (kBlk / 8) + lane);
          q[2 * u + 1] = __ldg(cp4 + (b + u) * (kBlk / 8) + 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          uint32_t bits = 0;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            uint32_t cv[8];
            unpack8(q[2 * u + h], cv);
#pragma unroll
            for (int qq = 0; qq < 8; qq++) bits += s_len[cv[qq]] + (cv[qq] == 0 ? 32u : 0u);
          }
          bits = warp_sum(bits);
          mine = lane == b + u ? bits : mine;
        }
      }
    } else
#pragma unroll 2
    for (int b = 0; b < kBlkPerChunk; b++) {
      const int lo = b * kBlk;
      uint32_t bits = 0;
      if (lo + kBlk <= mc) {  // full block: 64 uint4, two per lane
        uint32_t cv[8];
        unpack8(__ldg(cp4 + lo / 8 + lane), cv);
#pragma unroll
        for (int q = 0; q < 8; q++) bits += s_len[cv[q]] + (cv[q] == 0 ? 32u : 0u);
        unpack8(__ldg(cp4 + lo / 8 + 32 + lane), cv);
#pragma unroll
        for (int q = 0; q < 8; q++) bits += s_len[cv[q]] + (cv[q] == 0 ? 32u : 0u);
      } else {
        for (int i = lo + lane; i < min(mc, lo + kBlk); i += 32) {
          const uint32_t code = codes[c0 + i];
          bits += s_len[code] + (code == 0 ? 32u : 0u);
        }
      }
      bits = warp_sum(bits);
      mine = lane == b ? bits : mine;
    }
    const uint32_t incl = warp_incl_scan<uint32_t>(mine);
    bb[c * kBlkPerChunk + lane] = incl - mine;  // in-chunk exclusive prefix
    if (lane == 31) ctot[field * a.nchunks + c] = incl;
  }
}

// E2: per field exclusive scan of chunk bits -> chunk bit offsets; v2 index
__global__ void __launch_bounds__(1024) chunk_scan_kernel(EArgs a, const uint32_t* ctot,
                                                          uint64_t* coff) {
  const int field = a.f0 + (int)blockIdx.x;
  const nbzg_field_meta& m = a.meta->f[field];
  if (m.is_const || a.n == 0 || a.meta->status) return;
  __shared__ unsigned long long scan_tmp[33];
  const uint32_t* ct = ctot + (size_t)field * a.nchunks;
  uint64_t* off = coff + (size_t)field * (a.nchunks + 1);
  uint8_t* idx = a.arena + m.payload_off + m.index_off;
  const int64_t R = (a.nchunks + blockDim.x - 1) / blockDim.x;
  constexpr int kReg = 16;  // chunk totals per thread held in registers (one pass over ctot)
  uint32_t v[kReg];
  unsigned long long s = 0;
  if (R <= kReg) {
#pragma unroll
    for (int r = 0; r < kReg; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      v[r] = (r < R && c < a.nchunks) ? ct[c] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kReg; r++) s += v[r];
  } else {
    for (int64_t r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) s += ct[c];
    }
  }
  unsigned long long tot;
  unsigned long long ex = block_excl_scan<unsigned long long>(s, scan_tmp, &tot);
  if (R <= kReg) {
#pragma unroll
    for (int r = 0; r < kReg; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (r < R && c < a.nchunks) {
        off[c] = ex;
        put_u32_bytes(idx + 4 * c, v[r]);
      }
      ex += v[r];
    }
  } else {
    for (int64_t r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) {
        off[c] = ex;
        put_u32_bytes(idx + 4 * c, ct[c]);
        ex += ct[c];
      }
    }
  }
  if (threadIdx.x == 0) {
    off[a.nchunks] = tot;
    if (tot != m.total_bits) atomicCAS(&a.meta->status, 0u, (uint32_t)NBZG_BAD_STREAM);
  }
}

// E3: one thread packs one 512-code block at its known bit offset.  Completed
// words go to a per-thread 16-word ring in shared memory (word-major, so the
// lanes of a warp never conflict) with one predicated STS per code step --
// no divergent register shuffling -- and every 8 codes the thread flushes the
// 32-byte aligned 8-word groups it has completed with one 256-bit store.  The
// words before the block's first aligned group go out as scalar stores; the
// block's first partial word belongs to the block before (which completes it
// with this block's leading bits).
constexpr int kE3Threads = 384;
constexpr int kE3Ring = 16;  // words per thread

NBZG_DEV void st_v8_u32(uint32_t* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__global__ void __launch_bounds__(kE3Threads, 2) encode_tpc_kernel(EArgs a, const uint64_t* coff,
                                                                   const uint32_t* bpre,
                                                                   int ctas_per_field) {
  extern __shared__ __align__(16) uint8_t e3sm[];
  uint32_t* s_win = reinterpret_cast<uint32_t*>(e3sm);  // [kEncWin]
  const int field = a.f0 + (int)blockIdx.y;
  const nbzg_field_meta* mp = &a.meta->f[field];
  if (mp->is_const || a.n == 0 || a.meta->status) return;
  {
    const uint4* g = reinterpret_cast<const uint4*>(a.twin + (size_t)field * kEncWin);
    for (int i = threadIdx.x; i < kEncWin / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(s_win)[i] = __ldg(g + i);
  }
  __syncthreads();
  // ring word j of this thread at ring_s + 4 * j * blockDim.x
  const uint32_t ring_s = sh_addr(s_win + kEncWin) + 4u * threadIdx.x;
  uint32_t win_s;  // opaque copy: no per-lookup generic-to-shared conversion
  asm volatile("mov.u32 %0, %1;" : "=r"(win_s) : "r"(sh_addr(s_win)));
  const uint32_t rstride = 4u * blockDim.x;
  const WinTab T{s_win, (uint32_t)(a.nbins / 2 + 1 - kEncWin / 2), a.lut + field * a.nbins};
  const int64_t nb = a.nchunks * kBlkPerChunk;
  const uint16_t* codes = a.codes + field * a.code_stride;
  uint32_t* outw = reinterpret_cast<uint32_t*>(a.arena + mp->payload_off + mp->bits_off);
  const uint64_t* off = coff + (size_t)field * (a.nchunks + 1);
  const uint32_t* bp = bpre + (size_t)field * nb;
  const uint64_t ow = (reinterpret_cast<uintptr_t>(outw) >> 2) & 7;  // word phase of outw
  const int64_t stride = (int64_t)ctas_per_field * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += stride) {
    const int64_t s0 = k * kBlk;
    if (s0 >= a.n) continue;  // empty tail blocks of the last chunk
    const int mc = (int)min((int64_t)kBlk, a.n - s0);
    const int64_t c = k / kBlkPerChunk;
    const uint64_t B = off[c] + bp[k];
    const uint64_t Bend = (k + 1) % kBlkPerChunk ? off[c] + bp[k + 1] : off[c + 1];
    const uint4* cp4 = reinterpret_cast<const uint4*>(codes + s0);
    // 32-bit MSB-aligned pending word `cur` holding `nacc` < 32 bits; every
    // completed word goes to the ring with one predicated STS (no branch)
    uint32_t cur = 0;
    uint32_t nacc = (uint32_t)(B & 31);
    uint64_t widx = B >> 5;
    const uint64_t fo = (B + 31) >> 5;                  // first owned word
    const uint64_t va = ((fo + ow + 7) & ~7ull) - ow;  // first 32-byte aligned owned word
    uint64_t fl = widx;                                 // next ring word to flush
    // ring slot of stream word u: (u + ow) & 15, so 32-byte aligned groups
    // occupy slots 0-7 or 8-15; `rs` = slot counter of the next word
    uint32_t rs = (uint32_t)(widx + ow);
    // l in [1, 32]: append the l bits of the MSB-aligned word wl
    auto put_msb = [&](uint32_t wl, uint32_t l) {
      cur |= wl >> nacc;
      const uint32_t spill = __funnelshift_lc(0u, wl, 32 - nacc);  // wl << (32 - nacc), 0 at 32
      const uint32_t t = nacc + l;
      const bool full = t >= 32;
      const uint32_t slot = ring_s + rstride * (rs & (kE3Ring - 1));
      asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u32 [%0], %1;\n}\n" ::"r"(slot),
                   "r"(__byte_perm(cur, 0, 0x0123)), "r"((uint32_t)full)
                   : "memory");
      rs += full ? 1u : 0u;
      cur = full ? spill : cur;
      nacc = t & 31u;
    };
    auto put32 = [&](uint32_t v, uint32_t l) { put_msb(v << (32 - l), l); };  // low l bits of v
    auto put64 = [&](uint64_t v, uint32_t l) {  // l <= 64
      if (l > 32) {
        put32((uint32_t)(v >> 32), l - 32);
        put32((uint32_t)v, 32);
      } else if (l) {
        put32((uint32_t)v, l);
      }
    };
    auto ring_at = [&](uint64_t u) {
      return lds_u32(ring_s + rstride * ((uint32_t)(u + ow) & (kE3Ring - 1)));
    };
    auto flush = [&]() {  // head words one by one, then complete aligned 8-word groups
      widx = (B >> 5) + (uint32_t)(rs - (uint32_t)((B >> 5) + ow));
      while (fl < widx) {
        if (fl < va) {
          NBZG_CHECK(fl < (mp->payload_len - mp->bits_off) / 4);
          if (fl >= fo) outw[fl] = ring_at(fl);
          fl++;
        } else if (fl + 8 <= widx) {
          const uint32_t base = ring_s + rstride * ((uint32_t)(fl + ow) & 8u);
          uint32_t v[8];
#pragma unroll
          for (int u = 0; u < 8; u++) v[u] = lds_u32(base + rstride * u);
          NBZG_CHECK(fl + 8 <= (mp->payload_len - mp->bits_off + 3) / 4 + 8);
          st_v8_u32(outw + fl, v);
          fl += 8;
        } else {
          break;
        }
      }
    };
    auto put_code = [&](uint32_t code, int64_t pos) {
      uint64_t w;
      uint32_t l;
      win_word(T, code, w, l);
      put64(w, l);
      if (code == 0) put32(esc_value_bits(a, field, pos), 32);
    };
    const int ng = mc >> 3;
    uint4 n0 = ng > 0 ? __ldg(cp4) : make_uint4(0, 0, 0, 0);
    uint4 n1 = ng > 1 ? __ldg(cp4 + 1) : make_uint4(0, 0, 0, 0);
    uint4 n2 = ng > 2 ? __ldg(cp4 + 2) : make_uint4(0, 0, 0, 0);
    for (int g = 0; g < ng; g++) {
      const uint4 cu = n0;
      n0 = n1;
      n1 = n2;
      if (g + 3 < ng) n2 = __ldg(cp4 + g + 3);
      uint32_t cv[8], e[8];
      unpack8(cu, cv);
      bool hit = true;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint32_t wi = cv[q] - T.wlo;
        uint32_t v = 0;
        if (wi < (uint32_t)kEncWin)
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(win_s + 4u * wi));
        e[q] = v;
        hit &= v != 0;
      }
      if (hit) {
        // <= 8 x 26 bits: at most 7 new words; the ring (16) holds < 8 after a flush
#pragma unroll
        for (int q = 0; q < 8; q++) put_msb(e[q] & ~63u, e[q] & 63u);
      } else {
        // Long codes, codes outside the window, escapes.  The serial loop
        // below reads one global LUT entry (and, for an escape, perm and the
        // value) per miss; touch them all first so those dependent reads hit
        // L1 instead of paying an L2 round trip each (large alphabets: most
        // groups come here).
        {
          uint32_t sink = 0;
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (e[q] == 0) sink ^= (uint32_t)__ldg(&T.lut[cv[q]]);
            if (cv[q] == 0) sink ^= esc_value_bits(a, field, s0 + 8 * g + q);
          }
          asm volatile("" ::"r"(sink));
        }
        // codes re-extracted from the packed group (no dynamically indexed array)
        const uint64_t lo = ((uint64_t)cu.y << 32) | cu.x, hi = ((uint64_t)cu.w << 32) | cu.z;
#pragma unroll 1
        for (int q = 0; q < 8; q++) {
          const uint32_t code = (uint32_t)(((q < 4 ? lo : hi) >> (16 * (q & 3))) & 0xffffu);
          put_code(code, s0 + 8 * g + q);
          flush();  // long codes and escapes: up to 3 words per code
        }
      }
      flush();
    }
    for (int j = 8 * ng; j < mc; j++) {
      put_code(codes[s0 + j], s0 + j);
      flush();
    }
    // ring words of the last (incomplete) aligned group
    widx = (B >> 5) + (uint32_t)(rs - (uint32_t)((B >> 5) + ow));
    for (uint64_t u = fl; u < widx; u++) {
      NBZG_CHECK(u < (mp->payload_len - mp->bits_off) / 4);
      if (u >= fo) outw[u] = ring_at(u);
    }
    // final partial word: completed with the leading bits that follow
    if (nacc > 0 && (Bend >> 5) >= fo) {
      uint32_t w = cur;
      if (s0 + mc < a.n) w |= head_bits_from(a, field, codes, T, s0 + mc, 32 - (int)nacc) >> nacc;
      outw[widx] = __byte_perm(w, 0, 0x0123);
    }
  }
}

bool encode_uses_tpc(const Plan& p) {
  const char* ev = getenv("NBZG_ENCODE");
  const bool tpc = ev ? ev[0] == 't' : p.nchunks >= kTpcEncMinChunks;
  return p.nbins == 65536 && tpc;
}

// fields f0 .. f0+nf-1 (the TPC path may run in field groups; the other
// encoders always take all six fields)
int launch_encode(const Plan& p, cudaStream_t st, int f0, int nf) {
  if (p.n == 0) return NBZG_OK;
  TArgs t{p.meta, p.arena, p.cb_sym, p.cb_len, p.nbins, p.nchunks, p.n, f0};
  count_launch();
  table_writer_kernel<<<nf, 256, 0, st>>>(t);
  EArgs a{};
  a.meta = p.meta;
  a.arena = p.arena;
  a.codes = p.codes;
  a.code_stride = (p.n + 7) & ~int64_t(7);
  a.lut = p.lut;
  a.nbins = p.nbins;
  a.n = p.n;
  a.nchunks = p.nchunks;
  for (int f = 0; f < 6; f++) a.f[f] = p.f[f];
  a.perm = p.sorted ? p.perm : nullptr;
  a.tile = p.tile;
  a.lb = p.lb;
  a.tickets = p.counters;
  a.inline_esc = 1;
  a.twin = p.enc_win;
  a.tlen8 = p.enc_len8;
  a.f0 = f0;
  const bool tpc = encode_uses_tpc(p);
  if (!tpc) {  // look-back words and tickets of the warp encoders (all six fields)
    cudaMemsetAsync(p.lb, 0, sizeof(uint64_t) * 6 * p.nchunks, st);
    cudaMemsetAsync(p.counters, 0, sizeof(uint32_t) * 8, st);
  }
  if (tpc) {
    // E1 -> E2 -> E3: chunk offsets, then in-chunk block prefixes, chunk totals
    const int64_t nb = p.nchunks * kBlkPerChunk;
    uint64_t* coff = p.enc_boff;
    uint32_t* bpre = reinterpret_cast<uint32_t*>(p.enc_boff + 6 * (p.nchunks + 1));
    uint32_t* ctot = bpre + 6 * nb;
    smem_attr((const void*)chunk_bits_kernel, 65536);
    smem_attr((const void*)encode_tpc_kernel, 4 * kEncWin + 4 * kE3Ring * kE3Threads);
    int g1 = max(1, 2 * sm_count() / nf);
    if (g1 > (p.nchunks + kE1Warps - 1) / kE1Warps) g1 = (int)((p.nchunks + kE1Warps - 1) / kE1Warps);
    count_launch();
    chunk_bits_kernel<<<dim3(g1, nf), kE1Warps * 32, (size_t)p.nbins, st>>>(a, bpre, ctot, g1);
    count_launch();
    chunk_scan_kernel<<<nf, 1024, 0, st>>>(a, ctot, coff);
    int g3 = max(1, 2 * sm_count() / nf);
    if (g3 > (nb + kE3Threads - 1) / kE3Threads) g3 = (int)((nb + kE3Threads - 1) / kE3Threads);
    count_launch();
    encode_tpc_kernel<<<dim3(g3, nf), kE3Threads, 4 * kEncWin + 4 * kE3Ring * kE3Threads, st>>>(
        a, coff, bpre, g3);
  } else if (p.nbins == 65536) {
    const size_t sm = 4 * kEncWin + kEFWarps * 64 * 12 + kEFWarps * 32 * 4;
    smem_attr((const void*)encode_fast_kernel, (int)sm);
    int groups = max(1, 2 * sm_count() / 6);
    const int64_t need = (p.nchunks + kEFWarps - 1) / kEFWarps;
    if (groups > need) groups = (int)need;
    count_launch();
    encode_fast_kernel<<<dim3(groups, 6), kEFWarps * 32, sm, st>>>(a);
  } else {
    dim3 grid((unsigned)((p.nchunks + kEWarps - 1) / kEWarps), 6);
    count_launch();
    encode_kernel<<<grid, kEThreads, 0, st>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// parity hook: raw MSB-first bitstream of u16 symbols (K.huff_encode); no
// inline escapes (the reference's v1 bit layout)
int launch_huff_encode_raw(const uint16_t* syms, int64_t n, const uint64_t* lut, uint8_t* out,
                           uint32_t* chunk_bits, uint64_t* lb, uint32_t* tickets,
                           cudaStream_t st) {
  if (n == 0) return NBZG_OK;
  EArgs a{};
  a.codes = syms;
  a.code_stride = 0;
  a.lut = lut;
  a.nbins = 0;
  a.n = n;
  a.nchunks = (n + kChunk - 1) / kChunk;
  a.lb = lb;
  a.tickets = tickets;
  a.inline_esc = 0;
  a.raw_out = out;
  a.raw_chunk_bits = chunk_bits;
  cudaMemsetAsync(lb, 0, sizeof(uint64_t) * a.nchunks, st);
  cudaMemsetAsync(tickets, 0, sizeof(uint32_t), st);
  dim3 grid((unsigned)((a.nchunks + kEWarps - 1) / kEWarps), 1);
  count_launch();
  encode_kernel<<<grid, kEThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
