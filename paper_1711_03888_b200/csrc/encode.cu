// encode.cu -- K6/K7: v2 SZ_DQ payload writer and the chunk-parallel Huffman
// encoder.  Replaces encode.huffman_encode (encode.py:222-239) ->
// K.huff_encode (_kernels.py:304-345) and the stream framing of
// pipeline._build_sz_stream (pipeline.py:188-200).
//
// Payload (all little-endian):
//   u32 n_esc | u32 k | k x (u32 sym, u8 len) | u64 bit_length
//   | u32 chunk_bits[ceil(n/16384)] | pad to 4 | bitstream (MSB-first,
//   padded to 4 bytes) | f32 escapes[n_esc]
//
// Encoder: one CTA per 16384-code chunk (ticket-ordered).  Code lengths come
// from the u64 LUT (len << 57 | word); a block scan gives every thread's bit
// offset inside the chunk and a decoupled look-back over chunks gives the
// chunk's global bit offset and escape offset (u64).  Threads OR their code
// words into a shared-memory word buffer, which is written out as
// big-endian 32-bit words.  Word ownership: a word belongs to the chunk that
// holds its first bit; a chunk finishing mid-word encodes the first few codes
// of the next chunk itself to complete it, so every output word is written
// exactly once, with no zero-fill pass and no global atomics.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kEThreads = 512;
constexpr int kEPer = kChunk / kEThreads;  // 32 codes per thread
constexpr int kEBufWords = 8192;           // 262144 bits per round

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
};

__global__ void table_writer_kernel(TArgs a) {
  const int field = blockIdx.x;
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
  int64_t nbins;
  int64_t n, nchunks;
  const float* f[6];
  const uint16_t* perm;   // null if unsorted
  int64_t tile;
  uint64_t* lb;           // [6][2][nchunks]
  uint32_t* tickets;      // [6]
  // parity-hook mode: raw bitstream output instead of a payload
  uint8_t* raw_out;
  uint32_t* raw_chunk_bits;
};

// Encode the first codes of chunk `c1` (warp-wide) until `need` bits are
// produced; returns them MSB-aligned in a u32 (remaining bits zero).
NBZG_DEV uint32_t lookahead_bits(const uint16_t* codes, int64_t c1, int64_t n, const uint64_t* lut,
                                 int need) {
  const int lane = threadIdx.x & 31;
  int64_t i = c1 * kChunk + lane;
  uint64_t e = i < n ? __ldg(&lut[codes[i]]) : 0;
  uint32_t l = (uint32_t)(e >> 57);
  uint64_t w = e & ((1ull << 57) - 1);
  uint32_t incl = warp_incl_scan<uint32_t>(l);
  uint32_t start = incl - l;
  // contribution of this lane to bits [0, 32): word bits [start, start+l)
  uint32_t out = 0;
  if (l && start < 32) {
    // place w (l bits) at MSB offset `start` of a 32-bit window
    int sh = 32 - (int)start - (int)l;  // may be negative (code crosses the window)
    uint32_t part = sh >= 0 ? (uint32_t)(w << sh) : (uint32_t)(w >> (-sh));
    out = part;
  }
  // OR-reduce across the warp
#pragma unroll
  for (int o = 16; o; o >>= 1) out |= __shfl_xor_sync(0xffffffffu, out, o);
  // keep only `need` leading bits
  return need >= 32 ? out : (out & ~(0xffffffffu >> need));
}

__global__ void __launch_bounds__(kEThreads, 2) encode_kernel(EArgs a) {
  __shared__ uint32_t buf[kEBufWords + 2];
  __shared__ uint32_t scan_tmp[33];
  __shared__ unsigned long long s_boff, s_eoff;
  __shared__ uint32_t s_tail;
  const int field = blockIdx.y;
  const nbzg_field_meta& m = a.meta->f[field];
  const bool raw = a.raw_out != nullptr;
  if (!raw && (m.is_const || a.n == 0 || a.meta->status)) return;
  __shared__ int64_t s_c;
  if (threadIdx.x == 0) s_c = atomicAdd(&a.tickets[field], 1u);
  __syncthreads();
  const int64_t c = s_c;
  if (c >= a.nchunks) return;
  const int tid = threadIdx.x;
  const uint16_t* codes = a.codes + field * a.code_stride;
  const uint64_t* lut = a.lut + field * a.nbins;
  uint8_t* payload = raw ? nullptr : a.arena + m.payload_off;
  uint32_t* bits_w = raw ? reinterpret_cast<uint32_t*>(a.raw_out)
                         : reinterpret_cast<uint32_t*>(payload + m.bits_off);
  const int64_t c0 = c * kChunk;
  const int mc = (int)min((int64_t)kChunk, a.n - c0);

  // ---- load 32 codes (packed pairs), lengths, escape flags
  uint32_t cw[kEPer / 2];
  const int p0 = tid * kEPer;
  const int cnt = max(0, min(kEPer, mc - p0));
  if (cnt == kEPer && ((reinterpret_cast<uintptr_t>(codes + c0 + p0) & 15) == 0)) {
    const uint4* s4 = reinterpret_cast<const uint4*>(codes + c0 + p0);
#pragma unroll
    for (int q = 0; q < kEPer / 8; q++) {
      uint4 u = s4[q];
      cw[4 * q] = u.x;
      cw[4 * q + 1] = u.y;
      cw[4 * q + 2] = u.z;
      cw[4 * q + 3] = u.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kEPer / 2; j++) {
      uint32_t lo = 2 * j < cnt ? codes[c0 + p0 + 2 * j] : 0u;
      uint32_t hi = 2 * j + 1 < cnt ? codes[c0 + p0 + 2 * j + 1] : 0u;
      cw[j] = lo | (hi << 16);
    }
  }
#define CODE_AT(j) ((cw[(j) >> 1] >> (((j) & 1) * 16)) & 0xffffu)
  uint32_t tbits = 0, tesc = 0;
#pragma unroll
  for (int j = 0; j < kEPer; j++) {
    if (j < cnt) {
      uint32_t cv = CODE_AT(j);
      tbits += (uint32_t)(__ldg(&lut[cv]) >> 57);
      tesc += cv == 0;
    }
  }
  uint32_t chunk_bits, chunk_esc;
  uint32_t my_off = block_excl_scan<uint32_t>(tbits, scan_tmp, &chunk_bits);
  uint32_t my_esc = block_excl_scan<uint32_t>(tesc, scan_tmp, &chunk_esc);
  uint64_t* lbb = a.lb + (field * 2 + 0) * a.nchunks;
  uint64_t* lbe = a.lb + (field * 2 + 1) * a.nchunks;
  // publish the local aggregates at once so successors' look-backs never wait on our packing
  if (tid == 0 && c > 0) {
    lb_store(&lbb[c], kFlagAgg | chunk_bits);
    if (!raw) lb_store(&lbe[c], kFlagAgg | chunk_esc);
  }

  // ---- decoupled look-back: global bit / escape offsets of this chunk
  if (tid < 32) {
    uint64_t bo = lookback_sum(lbb, c, chunk_bits);
    uint64_t eo = raw ? 0 : lookback_sum(lbe, c, chunk_esc);
    if (tid == 0) {
      s_boff = bo;
      s_eoff = eo;
      if (raw) a.raw_chunk_bits[c] = chunk_bits;
      else put_u32_bytes(payload + m.index_off + 4 * c, chunk_bits);
    }
  }
  __syncthreads();
  const uint64_t B = s_boff;
  const uint64_t Bend = B + chunk_bits;

  // ---- escapes: verbatim f32 values in position order
  if (!raw && tesc) {
    float* esc = reinterpret_cast<float*>(payload + m.esc_off);
    uint64_t e = s_eoff + my_esc;
    for (int j = 0; j < cnt; j++) {
      if (CODE_AT(j) == 0) {
        int64_t pos = c0 + p0 + j;
        int64_t src = a.perm ? (pos / a.tile) * a.tile + a.perm[pos] : pos;
        esc[e++] = a.f[field][src];
      }
    }
  }

  // ---- pack words.  Rounds of 256 threads (4096 codes) when the chunk's
  // bits exceed the buffer; word 0 of each round is the carried partial word.
  const bool one_round = (uint64_t)chunk_bits + 64 <= (uint64_t)kEBufWords * 32;
  const int rounds = one_round ? 1 : 4;
  const int per_round = kEThreads / rounds;
  uint64_t round_start = B;  // global bit at which this round's buffer word 0 begins (aligned down)
  uint32_t carry = 0;
  const uint64_t first_owned = (B + 31) >> 5;  // first word whose first bit is in the chunk
  for (int r = 0; r < rounds; r++) {
    const uint64_t wbase = round_start >> 5;
    // bits of this round: threads [r*per_round, (r+1)*per_round)
    uint32_t rb_end_local;
    {
      // end offset of this round (chunk-relative) = offset of the first thread of the next round
      __shared__ uint32_t s_rend;
      if (tid == min(kEThreads - 1, (r + 1) * per_round - 1)) s_rend = my_off + tbits;
      __syncthreads();
      rb_end_local = s_rend;
    }
    const uint64_t rend = B + rb_end_local;
    const int nwords = (int)(((rend + 31) >> 5) - wbase);
    for (int i = tid; i < nwords + 1; i += kEThreads) buf[i] = 0;
    __syncthreads();
    if (tid == 0) buf[0] = carry;
    __syncthreads();
    if (tid >= r * per_round && tid < (r + 1) * per_round) {
      uint64_t pos = B + my_off - (wbase << 5);  // bit offset within buffer
#pragma unroll
      for (int j = 0; j < kEPer; j++) {
        if (j < cnt) {
          uint64_t e = __ldg(&lut[CODE_AT(j)]);
          int l = (int)(e >> 57);
          uint64_t w = e & ((1ull << 57) - 1);
          // write l bits of w starting at bit `pos` (MSB-first)
          while (l > 0) {
            int wi = (int)(pos >> 5), bo = (int)(pos & 31);
            int take = min(l, 32 - bo);
            uint32_t piece = (uint32_t)((w >> (l - take)) & ((1ull << take) - 1));
            atomicOr(&buf[wi], piece << (32 - bo - take));
            pos += take;
            l -= take;
          }
        }
      }
    }
    __syncthreads();
    // write complete words of this round; the last partial word carries on
    const bool last_round = r == rounds - 1;
    const int full = last_round ? nwords : (int)((rend >> 5) - wbase);
    for (int i = tid; i < full; i += kEThreads) {
      uint64_t gw = wbase + i;
      if (gw < first_owned) continue;                 // owned by the previous chunk
      if (last_round && i == nwords - 1 && (Bend & 31)) continue;  // completed below
      bits_w[gw] = __byte_perm(buf[i], 0, 0x0123);
    }
    if (!last_round) {
      __syncthreads();
      carry = buf[full];
      round_start = (wbase + full) << 5;
      __syncthreads();
    }
    if (last_round) {
      // final partial word (owned if its first bit lies inside this chunk)
      if ((Bend & 31) && nwords > 0) {
        uint64_t gw = wbase + nwords - 1;
        uint32_t word = buf[nwords - 1];
        if (c + 1 < a.nchunks) {
          int need = 32 - (int)(Bend & 31);
          uint32_t la = 0;
          if (tid < 32) la = lookahead_bits(codes, c + 1, a.n, lut, need);
          if (tid == 0) word |= la >> (32 - need) ;
        }
        if (tid == 0 && gw >= first_owned) bits_w[gw] = __byte_perm(word, 0, 0x0123);
      }
    }
  }
  (void)s_tail;
#undef CODE_AT
}

int launch_encode(const Plan& p, cudaStream_t st) {
  if (p.n == 0) return NBZG_OK;
  TArgs t{p.meta, p.arena, p.cb_sym, p.cb_len, p.nbins, p.nchunks, p.n};
  count_launch();
  table_writer_kernel<<<6, 256, 0, st>>>(t);
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
  cudaMemsetAsync(p.lb, 0, sizeof(uint64_t) * 12 * p.nchunks, st);
  cudaMemsetAsync(p.counters, 0, sizeof(uint32_t) * 8, st);
  dim3 grid((unsigned)p.nchunks, 6);
  count_launch();
  encode_kernel<<<grid, kEThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// parity hook: raw MSB-first bitstream of u16 symbols (K.huff_encode)
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
  a.raw_out = out;
  a.raw_chunk_bits = chunk_bits;
  cudaMemsetAsync(lb, 0, sizeof(uint64_t) * 2 * a.nchunks, st);
  cudaMemsetAsync(tickets, 0, sizeof(uint32_t), st);
  dim3 grid((unsigned)a.nchunks, 1);
  count_launch();
  encode_kernel<<<grid, kEThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
