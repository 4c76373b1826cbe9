// v1.cu -- opt-in reference-readable SZ streams (container version 1,
// stream kind SZ_FIELD): archives the unmodified reference decodes
// (io.py:128-211 -> pipeline._parse_sz_stream, pipeline.py:203-223).
//
// The reference's quantiser is a loop-carried FP64 chain (_kernels.py:
// 150-184: pred = recon[i-1], qf = rint((x - pred) * inv), recon =
// f32(pred + qf * 2b), escape when out of range or off by more than b).
// Restarting the chain with a FORCED ESCAPE every 16384 values (SURVEY.md
// Appendix B) makes every chunk independent -- the escape's recon is the
// exact value, so the next prediction no longer depends on the previous
// chunk -- while the stream stays an ordinary SZ_FIELD stream: the
// reference's dequantiser replays the same chain and reconstructs every
// value within its bound.  Cost: one escape per 16384 values (~+0.01%).
//
//   G  (sorted modes) gather the six fields into sorted order (a tile's
//      reads stay in its 64 KB window);
//   Q  one thread per 16384-value chunk runs the exact chain: u32 codes
//      (0 = escape, qf + half + 1 in [1, 2 half]), the chunk's escape values
//      at its chunk start in a scratch array, the escape count;
//   H  code histogram, nbins = interval_count + 1 (a shared-memory window
//      around the centre, global atomics outside it);
//   codebook (K4, v1 sizes) and layout as for v2;
//   B  bits per chunk (thread per chunk), S per-field scans of chunk bits
//      and escape counts, P pack (thread per chunk; interior words plain
//      stores, the chunk's boundary words atomicOr into a zeroed scratch),
//   E  the payload: u32 n_esc | u32 k | k x (u32 sym, u8 len) | u64 bits |
//      MSB-first bytes (ceil(bits/8)) | f32 escapes in position order.
// Mirrors oracle/nbz_oracle.c orc_sz_quantize_r + orc_sz_payload (fmt 1).
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kV1Threads = 128;  // threads per CTA of the thread-per-chunk kernels
constexpr int kV1Win = 16384;    // histogram window bins

struct V1Args {
  const float* f[6];
  const uint16_t* perm;
  int64_t tile;
  int sorted;
  int64_t n, nchunks, xs;  // xs: stride of the sorted-field / code / escape arrays
  int half;
  nbzg_meta* meta;
  float* xsort;      // [6][xs] sorted fields (sorted modes)
  uint32_t* codes;   // [6][xs]
  float* esc;        // [6][xs] chunk c's escapes from c * 16384
  uint32_t* esc_cnt; // [6][nchunks]
  uint32_t* cbits;   // [6][nchunks]
  uint64_t* boff;    // [6][nchunks + 1]
  uint64_t* eoff;    // [6][nchunks + 1]
  uint32_t* words;   // [6][wstride] packed bitstream scratch
  int64_t wstride;
  uint32_t* hist;    // [6][nbins]
  int64_t nbins;
  const uint8_t* len8;    // [6][nbins] code length by symbol
  const uint64_t* lut;    // [6][nbins] (len << 57) | word
  const uint32_t* cb_sym; // [6][nbins] ascending symbols
  const uint8_t* cb_len;  // [6][nbins] lengths by rank
  uint8_t* arena;
};

NBZG_DEV bool v1_active(const V1Args& a, int field) {
  return !a.meta->f[field].is_const && !a.meta->status && a.n > 0;
}

// ---- G: sorted order, one CTA per (tile, field); a tile's reads stay in
// one 64 KB window (L1-resident)
__global__ void __launch_bounds__(1024) v1_gather_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t t0 = (int64_t)blockIdx.x * a.tile;
  const int m = (int)min(a.tile, a.n - t0);
  const float* x = a.f[field] + t0;
  float* out = a.xsort + field * a.xs + t0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = __ldg(x + min((int)a.perm[t0 + i], m - 1));
}

// ---- Q: the exact chain, one thread per chunk (restart = forced escape)
__global__ void __launch_bounds__(kV1Threads) v1_quantize_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nchunks) return;
  const nbzg_field_meta& fm = a.meta->f[field];
  const int64_t i0 = c * kChunk, i1 = min(a.n, i0 + kChunk);
  const float* x = a.sorted ? a.xsort + field * a.xs : a.f[field];
  uint32_t* codes = a.codes + field * a.xs;
  float* esc = a.esc + field * a.xs + i0;
  const double b = fm.bound, twob = fm.twob, inv = fm.inv;  // inv = 1.0 / twob (resolve_kernel)
  const double hi_f = (double)(a.half - 1), lo_f = -(double)a.half;
  double h1 = 0.0;
  uint32_t ne = 0;
  for (int64_t i = i0; i < i1; i++) {
    const float xf = x[i];
    const double xv = (double)xf;
    uint32_t code = 0;
    float rec = xf;
    if (i != i0) {  // the chunk's first value: forced escape (chain restart)
      const double pred = h1;
      const double qf = rint(__dmul_rn(__dsub_rn(xv, pred), inv));
      if (lo_f <= qf && qf <= hi_f) {
        const float r32 = __double2float_rn(__dadd_rn(pred, __dmul_rn(qf, twob)));
        if (fabs(xv - (double)r32) <= b) {
          code = (uint32_t)((int32_t)qf + a.half + 1);
          rec = r32;
        }
      }
    }
    if (code == 0) esc[ne++] = xf;
    codes[i] = code;
    h1 = (double)rec;
  }
  a.esc_cnt[field * a.nchunks + c] = ne;
}

// ---- H: histogram of the u32 codes (window of kV1Win bins around the centre)
__global__ void __launch_bounds__(1024) v1_hist_kernel(V1Args a) {
  extern __shared__ uint32_t hw[];  // [kV1Win]
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t wlo = (int64_t)a.half + 1 - kV1Win / 2;
  for (int i = threadIdx.x; i < kV1Win; i += blockDim.x) hw[i] = 0;
  __syncthreads();
  const uint32_t* codes = a.codes + field * a.xs;
  uint32_t* hist = a.hist + field * a.nbins;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const uint32_t c = codes[i];
    const uint64_t w = (uint64_t)((int64_t)c - wlo);
    if (w < (uint64_t)kV1Win) atomicAdd(&hw[w], 1u);
    else atomicAdd(&hist[c], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kV1Win; i += blockDim.x) {
    const int64_t s = wlo + i;
    if (hw[i] && s >= 0 && s < a.nbins) atomicAdd(&hist[s], hw[i]);
  }
}

// ---- B: bits per chunk
__global__ void __launch_bounds__(kV1Threads) v1_bits_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nchunks) return;
  const int64_t i0 = c * kChunk, i1 = min(a.n, i0 + kChunk);
  const uint32_t* codes = a.codes + field * a.xs;
  const uint8_t* len = a.len8 + field * a.nbins;
  uint32_t s = 0;
  for (int64_t i = i0; i < i1; i++) s += len[codes[i]];
  a.cbits[field * a.nchunks + c] = s;
}

// ---- S: per-field exclusive scans (chunk bit offsets, escape offsets)
__global__ void __launch_bounds__(1024) v1_scan_kernel(V1Args a) {
  const int field = blockIdx.x;
  if (!v1_active(a, field)) return;
  __shared__ unsigned long long tmp[33];
  const int R = (int)((a.nchunks + blockDim.x - 1) / blockDim.x);
  for (int pass = 0; pass < 2; pass++) {
    const uint32_t* in = (pass ? a.esc_cnt : a.cbits) + field * a.nchunks;
    uint64_t* out = (pass ? a.eoff : a.boff) + field * (a.nchunks + 1);
    unsigned long long s = 0;
    for (int r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) s += in[c];
    }
    unsigned long long tot;
    unsigned long long ex = block_excl_scan<unsigned long long>(s, tmp, &tot);
    for (int r = 0; r < R; r++) {
      const int64_t c = (int64_t)threadIdx.x * R + r;
      if (c < a.nchunks) {
        out[c] = ex;
        ex += in[c];
      }
    }
    if (threadIdx.x == 0) {
      out[a.nchunks] = tot;
      const nbzg_field_meta& m = a.meta->f[field];
      if (tot != (pass ? m.n_esc : m.total_bits)) atomicCAS(&a.meta->status, 0u, (uint32_t)NBZG_BAD_STREAM);
    }
  }
}

// ---- P: pack one chunk's codes MSB-first from its bit offset
__global__ void __launch_bounds__(kV1Threads) v1_pack_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nchunks) return;
  const int64_t i0 = c * kChunk, i1 = min(a.n, i0 + kChunk);
  const uint32_t* codes = a.codes + field * a.xs;
  const uint64_t* lut = a.lut + field * a.nbins;
  uint32_t* words = a.words + field * a.wstride;
  const uint64_t b0 = a.boff[field * (a.nchunks + 1) + c];
  const uint64_t b1 = a.boff[field * (a.nchunks + 1) + c + 1];
  if (b1 == b0) return;
  const uint64_t w_first = b0 >> 5, w_last = (b1 - 1) >> 5;
  // acc holds `nb` pending bits left-aligned; wi = index of the word they start
  uint64_t acc = 0;
  uint32_t nb = (uint32_t)(b0 & 31);  // bits of the first word owned by earlier chunks (zeros)
  uint64_t wi = w_first;
  auto emit = [&](uint32_t word) {
    NBZG_CHECK(wi <= w_last && wi < (uint64_t)a.wstride);
    if (wi == w_first || wi == w_last) atomicOr(&words[wi], word);
    else words[wi] = word;
    wi++;
  };
  for (int64_t i = i0; i < i1; i++) {
    const uint64_t e = lut[codes[i]];
    const uint32_t l = (uint32_t)(e >> 57);
    const uint64_t w = e & ((1ull << 57) - 1);
    // append l bits (l <= 57): split so the 64-bit accumulator never overflows
    uint32_t rem = l;
    while (rem) {
      const uint32_t take = min(rem, 32u);
      const uint64_t part = (w >> (rem - take)) & ((1ull << take) - 1);
      acc |= part << (64 - nb - take);
      nb += take;
      rem -= take;
      if (nb >= 32) {
        emit((uint32_t)(acc >> 32));
        acc <<= 32;
        nb -= 32;
      }
    }
  }
  if (nb) emit((uint32_t)(acc >> 32));  // trailing partial word (zero padded)
}

// ---- E: payload bytes.  CTA (blk, field): the table, the bitstream bytes
// and the escapes of one field; blk strides over the byte ranges.
NBZG_DEV void put_u32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v;
  p[1] = (uint8_t)(v >> 8);
  p[2] = (uint8_t)(v >> 16);
  p[3] = (uint8_t)(v >> 24);
}
__global__ void __launch_bounds__(256) v1_emit_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const nbzg_field_meta& m = a.meta->f[field];
  uint8_t* p = a.arena + m.payload_off;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  if (gt == 0) {
    put_u32(p, (uint32_t)m.n_esc);
    put_u32(p + 4, m.k);
    const uint64_t tb = m.total_bits;
    put_u32(p + 8 + 5 * (uint64_t)m.k, (uint32_t)tb);
    put_u32(p + 12 + 5 * (uint64_t)m.k, (uint32_t)(tb >> 32));
  }
  const uint32_t* sym = a.cb_sym + field * a.nbins;
  const uint8_t* len = a.cb_len + field * a.nbins;
  for (int64_t i = gt; i < (int64_t)m.k; i += gs) {
    put_u32(p + 8 + 5 * i, sym[i]);
    p[8 + 5 * i + 4] = len[i];
  }
  const uint32_t* words = a.words + field * a.wstride;
  const int64_t nbytes = (int64_t)((m.total_bits + 7) / 8);
  uint8_t* bits = p + m.bits_off;
  for (int64_t j = gt; j < nbytes; j += gs) bits[j] = (uint8_t)(words[j >> 2] >> (24 - 8 * (j & 3)));
}

// escapes of one chunk, at the field's escape area in position order
__global__ void __launch_bounds__(kV1Threads) v1_esc_kernel(V1Args a) {
  const int field = blockIdx.y;
  if (!v1_active(a, field)) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.nchunks) return;
  const nbzg_field_meta& m = a.meta->f[field];
  const uint32_t ne = a.esc_cnt[field * a.nchunks + c];
  const uint64_t e0 = a.eoff[field * (a.nchunks + 1) + c];
  const float* esc = a.esc + field * a.xs + c * kChunk;
  uint8_t* dst = a.arena + m.payload_off + m.esc_off + 4 * e0;
  NBZG_CHECK(m.esc_off + 4 * (e0 + ne) <= m.payload_len);
  for (uint32_t j = 0; j < ne; j++) put_u32(dst + 4 * j, __float_as_uint(esc[j]));
}

int launch_v1(const Plan& p, cudaStream_t st) {
  if (p.n == 0) return NBZG_OK;
  V1Args a;
  for (int f = 0; f < 6; f++) a.f[f] = p.f[f];
  a.perm = p.perm;
  a.tile = p.tile;
  a.sorted = p.sorted;
  a.n = p.n;
  a.nchunks = p.nchunks;
  a.xs = p.v1_stride;
  a.half = p.half;
  a.meta = p.meta;
  a.xsort = p.v1_xsort;
  a.codes = p.v1_codes;
  a.esc = p.v1_esc;
  a.esc_cnt = p.v1_esc_cnt;
  a.cbits = p.v1_cbits;
  a.boff = p.v1_boff;
  a.eoff = p.v1_eoff;
  a.words = p.v1_words;
  a.wstride = p.v1_wstride;
  a.hist = p.hist;
  a.nbins = p.nbins;
  a.len8 = p.enc_len8;
  a.lut = p.lut;
  a.cb_sym = p.cb_sym;
  a.cb_len = p.cb_len;
  a.arena = p.arena;
  const dim3 gc((unsigned)((p.nchunks + kV1Threads - 1) / kV1Threads), 6);
  if (p.sorted) {
    count_launch();
    v1_gather_kernel<<<dim3((unsigned)p.ntiles, 6), 1024, 0, st>>>(a);
  }
  count_launch();
  v1_quantize_kernel<<<gc, kV1Threads, 0, st>>>(a);
  trace_mark("quantize", st);
  cudaMemsetAsync(p.hist, 0, sizeof(uint32_t) * 6 * p.nbins, st);
  smem_attr((const void*)v1_hist_kernel, 4 * kV1Win);
  count_launch();
  v1_hist_kernel<<<dim3((unsigned)max(1, 2 * sm_count() / 6), 6), 1024, 4 * kV1Win, st>>>(a);
  if (int rc = launch_codebook(p, st)) return rc;
  trace_mark("codebook", st);
  if (int rc = launch_layout(p, st)) return rc;
  count_launch();
  v1_bits_kernel<<<gc, kV1Threads, 0, st>>>(a);
  count_launch();
  v1_scan_kernel<<<6, 1024, 0, st>>>(a);
  cudaMemsetAsync(p.v1_words, 0, sizeof(uint32_t) * 6 * p.v1_wstride, st);
  count_launch();
  v1_pack_kernel<<<gc, kV1Threads, 0, st>>>(a);
  count_launch();
  v1_emit_kernel<<<dim3((unsigned)max(1, 4 * sm_count() / 6), 6), 256, 0, st>>>(a);
  count_launch();
  v1_esc_kernel<<<gc, kV1Threads, 0, st>>>(a);
  trace_mark("encode", st);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
