// rindex.cu -- K2: R-index keys + segment-local stable radix sort.
//
// Replaces rindex.build_r_indices (rindex.py:164-198), K.interleave3
// (_kernels.py:778-786) and rindex.prx_sort -> K.prx_order
// (_kernels.py:887-927) for the coordinate variant.
//
// One CTA per tile (whole segments, <= 16384 particles).  Per segment:
//   1. exact f32 min/max of the three coordinates (block reduce); because
//      rint(f64(x)/2b) is monotone in x, the integerised minima/maxima are the
//      integerised min/max -- six exact FP64 divisions per segment give the
//      per-segment minima, `need`, `bits` and the 21-bit clamp drop;
//   2. per particle: exact integerise (FP32 fast path, FP64 fallback), shift,
//      and interleave ONLY the bits the sort looks at: key >> 3*min(k,bits)
//      == interleave(v_t >> (drop + min(k,bits))) with w = bits - min(k,bits)
//      bits per field (3w <= 32 -> u32 keys);
//   3. stable LSD radix sort of the tile-local indices by that key, 8-bit
//      digits, warp-level __match_any_sync ranking + per-warp shared-memory
//      digit histograms (digit-major/warp-minor scan keeps it stable).
// Output: u16 tile-local source index per sorted position, u8 bits/segment.
// Tiles whose masked keys need more than 32 bits are flagged and redone by
// the u64-key instantiation.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kSortThreads = 512;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kRadix = 256;

struct RArgs {
  const float* x[6];      // key fields (coord / vel: 3, coord+vel: 6)
  int fbase;              // meta index of x[0] (0, or 3 for the velocity variant)
  int64_t n, S, tile, ntiles;
  int ig;
  const nbzg_meta* meta;
  uint16_t* perm;
  uint8_t* seg_bits;
  uint32_t* tile_flags;
  uint32_t* status;
  int pass;  // 0 = u32 main pass, 1 = u64 pass over flagged tiles
  int no_clamp;     // CPC modes: allow_key_clamp=False (rindex.py:185-190)
  int64_t* minima;  // CPC modes: 3 segment minima per segment (io.py:115-117), else null
  const float* seg_mm;  // [nseg][3][2] key-field min/max per segment from K1, or null
  uint16_t* keys16;     // [n] compacted keys (split compact sort)
  uint8_t* seg_cw;      // [nseg] compacted key width, 255 = general kernel
};

NBZG_DEV void set_status(uint32_t* status, uint32_t code) { atomicCAS(status, 0u, code); }

struct SegParams {
  int64_t mn[3];
  float amax[3];  // max |x| over the segment, per coordinate
  int shift;  // drop + eff
  int w;      // key bits per field after masking
  int bits;
  int bad;
};

// exact integerize of one float (quantize.py:117-128 semantics)
NBZG_DEV int64_t integerize1(float x, const nbzg_field_meta& m) {
  bool fast;
  double k = lattice_index<true>(x, m.inv32, m.inv, m.twob, fast);
  return (int64_t)k;
}

template <typename KeyT>
NBZG_DEV KeyT make_key(uint64_t u0, uint64_t u1, uint64_t u2);
template <>
NBZG_DEV uint32_t make_key<uint32_t>(uint64_t u0, uint64_t u1, uint64_t u2) {
  return (spread3_32((uint32_t)u0) << 2) | (spread3_32((uint32_t)u1) << 1) |
         spread3_32((uint32_t)u2);
}
template <>
NBZG_DEV uint64_t make_key<uint64_t>(uint64_t u0, uint64_t u1, uint64_t u2) {
  return (spread3_64(u0) << 2) | (spread3_64(u1) << 1) | spread3_64(u2);
}

// Stable LSD sort of perm[lo, lo+m) by keys[perm[.]] over sort_bits bits.
// All shared accesses use 32-bit shared-window addresses.
template <typename KeyT, bool FULL>
NBZG_DEV void block_sort_range_t(const KeyT* keys, uint16_t* perm, int lo, int m, int sort_bits,
                                 uint16_t* whist, uint32_t* scan_tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // FULL: m == kTileMax, every warp owns exactly 32 full rows (no bounds checks)
  const int E = FULL ? kTileMax / kSortWarps
                     : ((m + kSortWarps * 32 - 1) / (kSortWarps * 32)) * 32;  // per-warp span
  const int J = E / 32;
  const int base = w * E;
  const uint32_t keys_s = sh_addr(keys), perm_s = sh_addr(perm) + 2u * (uint32_t)lo;
  const uint32_t whist_s = sh_addr(whist), wh_s = whist_s + 2u * (uint32_t)(w * kRadix);
  for (int sh = 0; sh < sort_bits; sh += 8) {
    for (int i = threadIdx.x; i < kSortWarps * kRadix / 2; i += kSortThreads)
      sts_u32(whist_s + 4u * (uint32_t)i, 0u);
    __syncthreads();
    uint32_t packed[32];
#pragma unroll
    for (int j = 0; j < 32; j++) {
      if (j < J) {
        int pos = base + j * 32 + lane;
        bool valid = FULL || pos < m;
        uint32_t idx = valid ? lds_u16(perm_s + 2u * (uint32_t)pos) : 0u;
        uint32_t d = valid ? (uint32_t)((lds_key<KeyT>(keys_s + (uint32_t)sizeof(KeyT) * idx) >> sh) & 0xff)
                           : 0x100u;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t lt = __popc(peers & lanemask_lt());
        uint32_t cnt = valid ? lds_u16(wh_s + 2u * d) : 0u;
        __syncwarp();
        if (valid && lt == 0) sts_u16(wh_s + 2u * d, cnt + __popc(peers));
        __syncwarp();
        packed[j] = idx | ((cnt + lt) << 14) | (d << 24);
      }
    }
    __syncthreads();
    // digit-major / warp-minor exclusive scan of the per-warp histograms
    {
      const int t = threadIdx.x;
      const int d = t >> 1, w0 = (t & 1) * (kSortWarps / 2);
      uint32_t c[kSortWarps / 2];
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < kSortWarps / 2; q++) {
        c[q] = whist[(w0 + q) * kRadix + d];
        s += c[q];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(s, scan_tmp, &tot);
#pragma unroll
      for (int q = 0; q < kSortWarps / 2; q++) {
        whist[(w0 + q) * kRadix + d] = (uint16_t)ex;
        ex += c[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j++) {
      if (j < J && (FULL || base + j * 32 + lane < m)) {
        uint32_t v = packed[j];
        uint32_t idx = v & 0x3fff, r = (v >> 14) & 0x3ff, d = v >> 24;
        sts_u16(perm_s + 2u * (lds_u16(wh_s + 2u * d) + r), idx);
      }
    }
    __syncthreads();
  }
}

template <typename KeyT>
NBZG_DEV void block_sort_range(const KeyT* keys, uint16_t* perm, int lo, int m, int sort_bits,
                               uint16_t* whist, uint32_t* scan_tmp) {
  if (m == kTileMax) block_sort_range_t<KeyT, true>(keys, perm, lo, m, sort_bits, whist, scan_tmp);
  else block_sort_range_t<KeyT, false>(keys, perm, lo, m, sort_bits, whist, scan_tmp);
}

// Masked keys of one segment into keys[lo, lo + m) (rindex.py:164-198 +
// _kernels.py:757-786): exact integerised coordinates minus the segment
// minima, shifted by drop + ignored groups, bit-interleaved.  Split keys
// (3w > 32 in a u32 array): part 0 = the low 32 key bits, 1 = the rest.
template <typename KeyT>
__device__ __noinline__ void gen_keys(const float* __restrict__ x0p, const float* __restrict__ x1p,
                                      const float* __restrict__ x2p, const nbzg_field_meta* fm,
                                      const SegParams* sp, KeyT* keys, int lo, int m, int64_t s0,
                                      bool split, int part) {
  const int shift = sp->shift;
  const int64_t m0 = sp->mn[0], m1 = sp->mn[1], m2 = sp->mn[2];
  // Segment-wide FP32 path (same margin argument as quantize_kernel):
  // with tmax = max |x| * inv32 over the segment, |t - rint(t)| < c_c
  // proves rint(fl(x * inv32)) == rint(f64(x) / 2b); otherwise the exact
  // FP64 division.  Needs every |t| < 2^22 (32-bit indices).
  float cm[3];
  bool small = true;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const float tmax = sp->amax[c] * fm[c].inv32;
    small &= tmax < 4194304.0f;
    cm[c] = 0.5f - __fmaf_ru(tmax, 2.384185791015625e-07f, 9.5367431640625e-07f);
  }
  const float i0 = fm[0].inv32, i1 = fm[1].inv32, i2 = fm[2].inv32;
  auto mk = [&](uint64_t u0, uint64_t u1, uint64_t u2) -> KeyT {
    if (sizeof(KeyT) == 8) return (KeyT)make_key<uint64_t>(u0, u1, u2);
    if (!split) return (KeyT)make_key<uint32_t>(u0, u1, u2);
    const uint64_t k = make_key<uint64_t>(u0, u1, u2);
    return (KeyT)(part ? (k >> 32) : k);
  };
  auto key_fast = [&](float x0, float x1, float x2) -> KeyT {
    const float xv[3] = {x0, x1, x2};
    const float iv[3] = {i0, i1, i2};
    uint32_t u[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const float t = xv[c] * iv[c];
      const float r = t + 12582912.0f;
      const float d = t - (r - 12582912.0f);
      int32_t k = __float_as_int(r) - 0x4B400000;
      if (!(fabsf(d) < cm[c])) k = (int32_t)rint(__ddiv_rn((double)xv[c], fm[c].twob));
      const int32_t mm = (int32_t)(c == 0 ? m0 : (c == 1 ? m1 : m2));
      u[c] = (uint32_t)(k - mm) >> shift;
    }
    return mk(u[0], u[1], u[2]);
  };
  auto key_of = [&](float x0, float x1, float x2) -> KeyT {
    const float xv[3] = {x0, x1, x2};
    uint64_t u[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      int64_t iv = fm[c].is_const ? 0 : integerize1(xv[c], fm[c]);
      int64_t mm = c == 0 ? m0 : (c == 1 ? m1 : m2);
      u[c] = (uint64_t)(iv - mm) >> shift;
    }
    return mk(u[0], u[1], u[2]);
  };
  const int m4 = (s0 & 3) ? 0 : m >> 2;  // float4 path needs 16-byte aligned segments
  const float4* x4[3] = {reinterpret_cast<const float4*>(x0p + s0),
                         reinterpret_cast<const float4*>(x1p + s0),
                         reinterpret_cast<const float4*>(x2p + s0)};
    if (small && sizeof(KeyT) == 4) {
#pragma unroll 2
      for (int v = threadIdx.x; v < m4; v += kSortThreads) {
        const float4 q0 = __ldg(x4[0] + v), q1 = __ldg(x4[1] + v), q2 = __ldg(x4[2] + v);
        KeyT* kd = keys + lo + 4 * v;
        kd[0] = key_fast(q0.x, q1.x, q2.x);
        kd[1] = key_fast(q0.y, q1.y, q2.y);
        kd[2] = key_fast(q0.z, q1.z, q2.z);
        kd[3] = key_fast(q0.w, q1.w, q2.w);
      }
    } else {
#pragma unroll 2
      for (int v = threadIdx.x; v < m4; v += kSortThreads) {
        const float4 q0 = __ldg(x4[0] + v), q1 = __ldg(x4[1] + v), q2 = __ldg(x4[2] + v);
        KeyT* kd = keys + lo + 4 * v;
        kd[0] = key_of(q0.x, q1.x, q2.x);
        kd[1] = key_of(q0.y, q1.y, q2.y);
        kd[2] = key_of(q0.z, q1.z, q2.z);
        kd[3] = key_of(q0.w, q1.w, q2.w);
      }
    }
    for (int i = 4 * m4 + threadIdx.x; i < m; i += kSortThreads)
      keys[lo + i] = key_of(x0p[s0 + i], x1p[s0 + i], x2p[s0 + i]);
    __syncthreads();
}

template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads, 2) rindex_sort_kernel(RArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  KeyT* keys = reinterpret_cast<KeyT*>(smem);
  uint16_t* perm = reinterpret_cast<uint16_t*>(keys + kTileMax);
  uint16_t* whist = perm + kTileMax;
  __shared__ uint32_t scan_tmp[33];
  __shared__ float red[2][3][kSortWarps];
  __shared__ SegParams sp;

  const int64_t t = blockIdx.x;
  if (a.pass >= 1 && a.tile_flags[t] != (uint32_t)a.pass) return;
  const int64_t t0 = t * a.tile;
  const int64_t t1 = min(a.n, t0 + a.tile);
  const int mt = (int)(t1 - t0);
  const nbzg_field_meta* fm = a.meta->f + a.fbase;

  for (int i = threadIdx.x; i < mt; i += kSortThreads) perm[i] = (uint16_t)i;

  for (int64_t s0 = t0; s0 < t1; s0 += a.S) {
    const int lo = (int)(s0 - t0);
    const int m = (int)(min(t1, s0 + a.S) - s0);
    // ---- 1. per-segment min / max of the coordinates
    float mn[3], mx[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      mn[c] = __int_as_float(0x7f800000);
      mx[c] = -__int_as_float(0x7f800000);
    }
    if (a.seg_mm) {
      // K1 already reduced this segment: every thread takes the values, so
      // the block reduction below returns them unchanged
      const float* sm = a.seg_mm + 6 * (s0 / a.S);
#pragma unroll
      for (int c = 0; c < 3; c++) {
        mn[c] = sm[2 * c];
        mx[c] = sm[2 * c + 1];
      }
    } else {
      // float4 loads, 4 x 3 in flight per thread (segments start 16-byte aligned)
      const int m4 = (s0 & 3) ? 0 : m >> 2;  // float4 path needs 16-byte aligned segments
      const float4* x4[3] = {reinterpret_cast<const float4*>(a.x[0] + s0),
                             reinterpret_cast<const float4*>(a.x[1] + s0),
                             reinterpret_cast<const float4*>(a.x[2] + s0)};
#pragma unroll 4
      for (int v = threadIdx.x; v < m4; v += kSortThreads) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float4 q = __ldg(x4[c] + v);
          mn[c] = fminf(mn[c], fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
          mx[c] = fmaxf(mx[c], fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
        }
      }
      for (int i = 4 * m4 + threadIdx.x; i < m; i += kSortThreads) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float v = a.x[c][s0 + i];
          mn[c] = fminf(mn[c], v);
          mx[c] = fmaxf(mx[c], v);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
        mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
      }
      if ((threadIdx.x & 31) == 0) {
        red[0][c][threadIdx.x >> 5] = mn[c];
        red[1][c][threadIdx.x >> 5] = mx[c];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = 0, bad = 0;
      for (int c = 0; c < 3; c++) {
        float a0 = red[0][c][0], b0 = red[1][c][0];
        for (int q = 1; q < kSortWarps; q++) {
          a0 = fminf(a0, red[0][c][q]);
          b0 = fmaxf(b0, red[1][c][q]);
        }
        sp.amax[c] = fmaxf(fabsf(a0), fabsf(b0));
        if (fm[c].is_const) {
          sp.mn[c] = 0;
          continue;
        }
        double qa = __ddiv_rn((double)a0, fm[c].twob), qb = __ddiv_rn((double)b0, fm[c].twob);
        if (fabs(qa) > kIntLimit || fabs(qb) > kIntLimit) bad = 1;
        int64_t ia = (int64_t)rint(qa), ib = (int64_t)rint(qb);
        sp.mn[c] = ia;
        int bl = bitlen64((uint64_t)(ib - ia));
        need = max(need, bl);
      }
      int bits = min(need, 21);
      int drop = need > 21 ? need - 21 : 0;  // allow_key_clamp=True for sz-lv-prx (pipeline.py:463)
      if (a.no_clamp && need > 21) bad = 1;   // CPC: BoundTooSmallError (rindex.py:185-190)
      int eff = min(a.ig, bits);
      sp.bits = bits;
      sp.shift = drop + eff;
      sp.w = bits - eff;
      sp.bad = bad;
    }
    __syncthreads();
    if (sp.bad) {
      if (threadIdx.x == 0) set_status(a.status, NBZG_BOUND_TOO_SMALL);
      return;
    }
    const int w = sp.w;
    // u32 keys hold 3w <= 32 bits; wider keys (the CPC modes' full keys,
    // ignored groups 0) are sorted in two LSD phases over the same u32
    // array: the low 32 key bits first, then the key's high bits
    // (recomputed from the coordinates) -- stable passes, so the result is
    // the full-key order and the tile keeps 2 CTAs per SM.
    const bool split = sizeof(KeyT) == 4 && 3 * w > 32;
    if (threadIdx.x == 0) {
      a.seg_bits[(s0) / a.S] = (uint8_t)sp.bits;
      if (a.minima)
        for (int c = 0; c < 3; c++) a.minima[3 * (s0 / a.S) + c] = sp.mn[c];
    }
    if (w > 0) {
      // ---- 3. stable radix sort over 3w bits (one call site: one inlined copy)
      for (int ph = 0; ph < (split ? 2 : 1); ph++) {
        // ---- 2. masked keys (not inlined: none of its state stays live
        // across the sort, whose rank loop needs the registers)
        gen_keys<KeyT>(a.x[0], a.x[1], a.x[2], a.meta->f + a.fbase, &sp, keys, lo, m, s0, split,
                       ph);
        const int nbits = split ? (ph == 0 ? 32 : 3 * w - 32) : 3 * w;
        block_sort_range<KeyT>(keys, perm, lo, m, nbits, whist, scan_tmp);
      }
    }
    __syncthreads();
  }
  // ---- write the tile's permutation (coalesced)
  for (int i = threadIdx.x; i < mt; i += kSortThreads) a.perm[t0 + i] = perm[i];
}

// Six-field coord+velocity keys (RIndexVariant.COORD_VELOCITY): group
// width 6, at most 10 bits per field (max_bits_per_field, rindex.py:42-44),
// bit j of field t at key bit 6j + 5 - t (interleave_any, _kernels.py:801).
// Scalar loads and a bit loop: a rarely used variant, kept simple.
template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads, 2) rindex_sort6_kernel(RArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  KeyT* keys = reinterpret_cast<KeyT*>(smem);
  uint16_t* perm = reinterpret_cast<uint16_t*>(keys + kTileMax);
  uint16_t* whist = perm + kTileMax;
  __shared__ uint32_t scan_tmp[33];
  __shared__ float red[2][6][kSortWarps];
  __shared__ int64_t s_mn[6];
  __shared__ int s_shift, s_w, s_bits, s_bad;

  const int64_t t = blockIdx.x;
  if (a.pass >= 1 && a.tile_flags[t] != (uint32_t)a.pass) return;
  const int64_t t0 = t * a.tile;
  const int64_t t1 = min(a.n, t0 + a.tile);
  const int mt = (int)(t1 - t0);
  const nbzg_field_meta* fm = a.meta->f;
  for (int i = threadIdx.x; i < mt; i += kSortThreads) perm[i] = (uint16_t)i;
  for (int64_t s0 = t0; s0 < t1; s0 += a.S) {
    const int lo = (int)(s0 - t0);
    const int m = (int)(min(t1, s0 + a.S) - s0);
    float mn[6], mx[6];
#pragma unroll
    for (int c = 0; c < 6; c++) {
      mn[c] = __int_as_float(0x7f800000);
      mx[c] = -__int_as_float(0x7f800000);
    }
    for (int i = threadIdx.x; i < m; i += kSortThreads)
#pragma unroll
      for (int c = 0; c < 6; c++) {
        const float v = a.x[c][s0 + i];
        mn[c] = fminf(mn[c], v);
        mx[c] = fmaxf(mx[c], v);
      }
#pragma unroll
    for (int c = 0; c < 6; c++) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
        mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
      }
      if ((threadIdx.x & 31) == 0) {
        red[0][c][threadIdx.x >> 5] = mn[c];
        red[1][c][threadIdx.x >> 5] = mx[c];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = 0, bad = 0;
      for (int c = 0; c < 6; c++) {
        float a0 = red[0][c][0], b0 = red[1][c][0];
        for (int q = 1; q < kSortWarps; q++) {
          a0 = fminf(a0, red[0][c][q]);
          b0 = fmaxf(b0, red[1][c][q]);
        }
        if (fm[c].is_const) {
          s_mn[c] = 0;
          continue;
        }
        double qa = __ddiv_rn((double)a0, fm[c].twob), qb = __ddiv_rn((double)b0, fm[c].twob);
        if (fabs(qa) > kIntLimit || fabs(qb) > kIntLimit) bad = 1;
        int64_t ia = (int64_t)rint(qa), ib = (int64_t)rint(qb);
        s_mn[c] = ia;
        need = max(need, bitlen64((uint64_t)(ib - ia)));
      }
      const int cap = 10;
      const int bits = min(need, cap);
      const int drop = need > cap ? need - cap : 0;
      const int eff = min(a.ig, bits);
      s_bits = bits;
      s_shift = drop + eff;
      s_w = bits - eff;
      s_bad = bad;
    }
    __syncthreads();
    if (s_bad) {
      if (threadIdx.x == 0) set_status(a.status, NBZG_BOUND_TOO_SMALL);
      return;
    }
    const int w = s_w;
    if (sizeof(KeyT) == 4 && 6 * w > 32) {
      if (threadIdx.x == 0) a.tile_flags[t] = 2;
      return;  // redone by the u64 pass
    }
    if (threadIdx.x == 0) a.seg_bits[s0 / a.S] = (uint8_t)s_bits;
    if (w > 0) {
      const int shift = s_shift;
      for (int i = threadIdx.x; i < m; i += kSortThreads) {
        KeyT key = 0;
#pragma unroll
        for (int c = 0; c < 6; c++) {
          const int64_t iv = fm[c].is_const ? 0 : integerize1(a.x[c][s0 + i], fm[c]);
          const uint64_t u = (uint64_t)(iv - s_mn[c]) >> shift;
          for (int j = 0; j < w; j++) key |= (KeyT)((u >> j) & 1u) << (6 * j + 5 - c);
        }
        keys[lo + i] = key;
      }
      __syncthreads();
      block_sort_range<KeyT>(keys, perm, lo, m, 6 * w, whist, scan_tmp);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < mt; i += kSortThreads) a.perm[t0 + i] = perm[i];
}

// ---------------------------------------------------------------- compact-key sort
// The stable order by the masked key K is unchanged when K is replaced by
// any strictly increasing function of the keys present in the segment.  Bits
// that are zero in every key of the segment are such a function's free
// choice: field t's masked value u_t = (k_t - mn_t) >> shift lies in
// [0, umax_t] with umax_t = (hi_t - lo_t) >> shift known from the segment's
// integerised min / max, so only its low w_t = bitlen(umax_t) bits can be
// set.  The compacted key keeps exactly those bits, in the interleaved
// order (group j high to low, x before y before z within a group): bit j of
// field t goes to position P_t(j) = sum_t' min(j, w_t') + #{t' > t : j < w_t'}.
// Per segment, byte-wise tables T[t][b][v] give each field's contribution,
// so a key costs three table reads instead of three bit-spreads.  At config
// 2 (eb 1e-4) the masked keys carry 21 bits but only ~9 vary: one radix pass
// with 2^cw bins sorts the segment.  Segments whose compacted key exceeds 16
// bits are flagged for the general kernel (rindex_sort_kernel, pass 1).
// rint(f64(x) / 2b) by the exact division (quantize.py:122): the near-tie
// fallback of the compact-key sort, kept out of line (one copy of the
// division code, executed only by the lanes that need it)
__device__ __noinline__ int32_t exact_index(float x, const nbzg_field_meta* m) {
  return m->is_const ? 0 : (int32_t)rint(__ddiv_rn((double)x, m->twob));
}

#ifdef NBZG_CS_PROF  // timing experiment: per-phase clock totals of CTA 0, printed at exit
#define CS_T(i) do { if (threadIdx.x == 0) { long long _c = clock64(); cs_t[i] += _c - cs_last; cs_last = _c; } } while (0)
#else
#define CS_T(i) do { } while (0)
#endif
constexpr int kCsKeyThreads = 256;  // K2a block
constexpr int kCsMaxBits = 16;  // compacted key bits handled here (u16 keys)
constexpr int kCsOneBits = 10;  // <= this: a single pass with 2^cw bins
constexpr int kCsJ = kTileMax / kSortThreads;  // elements per thread (32)

struct CsSeg {
  int64_t mn[3];
  float amax[3];
  int shift, w, bits, bad, cw, wmax;
  int wt[3];
};

// one stable counting pass over m <= 16384 elements: digit of element
// (warp-major position pos) = (key >> sh) & (2^D - 1), key = keys[src(pos)],
// src = pos (FIRST) or perm[pos]; output perm[dst] = src, in place.
// Values in perm are tile-local (segment start lo + segment index).
template <bool FIRST>
NBZG_DEV void cs_pass(const uint16_t* keys, uint16_t* perm, int lo, int m, int sh, int D,
                      uint16_t* whist, uint32_t* scan_tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = 1 << D;
  const uint32_t msk = (uint32_t)nb - 1;
  const uint32_t keys_s = sh_addr(keys), perm_s = sh_addr(perm);
  const uint32_t wh_s = sh_addr(whist) + 2u * (uint32_t)(w * nb);
  for (int i = threadIdx.x; i < kSortWarps * nb / 2; i += kSortThreads)
    sts_u32(sh_addr(whist) + 4u * (uint32_t)i, 0u);
  __syncthreads();
  const int base = w * (kTileMax / kSortWarps);
  // per element: FIRST -> rank (16 bits, two per register); else idx | rank << 14 | d << 24
  uint32_t packed[FIRST ? kCsJ / 2 : kCsJ];
#pragma unroll
  for (int j = 0; j < kCsJ; j++) {
    const int pos = base + j * 32 + lane;
    const bool valid = pos < m;
    const uint32_t src =
        FIRST ? (uint32_t)pos : (valid ? lds_u16(perm_s + 2u * (uint32_t)pos) - (uint32_t)lo : 0u);
    const uint32_t d = valid ? ((lds_u16(keys_s + 2u * src) >> sh) & msk) : 0x10000u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t lt = __popc(peers & lanemask_lt());
    const uint32_t cnt = valid ? lds_u16(wh_s + 2u * d) : 0u;
    __syncwarp();
    if (valid && lt == 0) sts_u16(wh_s + 2u * d, cnt + __popc(peers));
    __syncwarp();
    const uint32_t r = cnt + lt;
    if (FIRST) {
      if (j & 1) packed[j >> 1] |= r << 16;
      else packed[j >> 1] = r;
    } else {
      packed[j] = src | (r << 14) | (d << 24);
    }
  }
  __syncthreads();
  // digit-major / warp-minor exclusive scan of the per-warp counts: counter
  // q = d * 16 + w; thread t owns counters [t*ipt, (t+1)*ipt)
  {
    const int C = kSortWarps * nb;
    const int ipt = (C + kSortThreads - 1) / kSortThreads;  // 1 .. 32
    const int q0 = threadIdx.x * ipt;
    uint32_t s = 0;
    for (int q = q0; q < min(C, q0 + ipt); q++) s += whist[(q & 15) * nb + (q >> 4)];
    uint32_t tot;
    uint32_t ex = block_excl_scan<uint32_t>(s, scan_tmp, &tot);
    for (int q = q0; q < min(C, q0 + ipt); q++) {
      const int a = (q & 15) * nb + (q >> 4);
      const uint32_t c = whist[a];
      whist[a] = (uint16_t)ex;
      ex += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kCsJ; j++) {
    const int pos = base + j * 32 + lane;
    if (pos < m) {
      uint32_t src, r, d;
      if (FIRST) {
        src = (uint32_t)pos;
        r = (packed[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        d = (lds_u16(keys_s + 2u * src) >> sh) & msk;
      } else {
        src = packed[j] & 0x3fffu;
        r = (packed[j] >> 14) & 0x3ffu;
        d = packed[j] >> 24;
      }
      NBZG_CHECK(lds_u16(wh_s + 2u * d) + r < (uint32_t)m && src < (uint32_t)m);
      sts_u16(perm_s + 2u * (lds_u16(wh_s + 2u * d) + r), src + (uint32_t)lo);
    }
  }
  __syncthreads();
}

// the second pass of a two-pass segment (rare: ~5% of config-2 segments),
// out of line so its 32-register packed state does not weigh on the kernel
__device__ __noinline__ void cs_pass_next(const uint16_t* keys, uint16_t* perm, int lo, int m,
                                          int sh, int D, uint16_t* whist, uint32_t* scan_tmp) {
  cs_pass<false>(keys, perm, lo, m, sh, D, whist, scan_tmp);
}

// MODE 0: keys and sort in one kernel (keys in shared memory); MODE 1:
// segment parameters + compacted keys to HBM (u16, 2 B/particle) and the
// per-segment key width; MODE 2: the sort, keys loaded from HBM.  The split
// (1 + 2) streams the coordinates at high occupancy instead of holding a
// 105 KB sort CTA idle on them.
template <int MODE>
NBZG_DEV void csort_body(const RArgs& a) {
  extern __shared__ __align__(16) uint8_t csm[];
  uint16_t* keys = reinterpret_cast<uint16_t*>(csm);          // [kTileMax] segment-local
  uint16_t* perm = keys + kTileMax;                           // [kTileMax] tile-local values
  uint16_t* whist = perm + kTileMax;                          // [16][2^10]
  uint32_t(*lut)[3][256] = reinterpret_cast<uint32_t(*)[3][256]>(
      MODE == 1 ? csm : reinterpret_cast<uint8_t*>(whist + (kSortWarps << kCsOneBits)));
  constexpr int NT = MODE == 1 ? kCsKeyThreads : kSortThreads;
  __shared__ uint32_t scan_tmp[33];
  __shared__ float red[2][3][kSortWarps];
  __shared__ CsSeg sp;
  __shared__ float cs_v[6];     // segment (min, max) per key field
  __shared__ int64_t cs_q[6];   // their lattice indices
  __shared__ int cs_big[6];

  const nbzg_field_meta* fm = a.meta->f + a.fbase;
#ifdef NBZG_CS_PROF
  long long cs_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cs_last = clock64();
#endif
  // persistent CTAs (2 per SM), tiles strided by the grid.  (An L2 bulk
  // prefetch of the next tile's coordinates was measured: the lines were
  // evicted before use -- twice the DRAM reads -- and the tile got slower.)
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
  const int64_t t0 = t * a.tile;
  const int64_t t1 = min(a.n, t0 + a.tile);
  const int mt = (int)(t1 - t0);
  bool flagged = false;
  if (MODE == 2 && a.tile_flags[t]) continue;  // the general kernel sorts this tile

  for (int64_t s0 = t0; s0 < t1; s0 += a.S) {
    const int lo = (int)(s0 - t0);
    const int m = (int)(min(t1, s0 + a.S) - s0);
    if (MODE == 2) {
      const int cw = a.seg_cw[s0 / a.S];
      if (cw == 0) {
        for (int i = threadIdx.x; i < m; i += NT) perm[lo + i] = (uint16_t)(lo + i);
        __syncthreads();
        continue;
      }
      // the segment's compacted keys (K2a), coalesced 16-byte loads
      const uint16_t* src = a.keys16 + s0;
      const int m8 = (s0 & 7) ? 0 : m >> 3;
      for (int i = threadIdx.x; i < m8; i += NT)
        reinterpret_cast<uint4*>(keys)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
      for (int i = 8 * m8 + threadIdx.x; i < m; i += NT) keys[i] = src[i];
      __syncthreads();
      const int d1 = cw <= kCsOneBits ? cw : cw >> 1;
      cs_pass<true>(keys, perm + lo, lo, m, 0, d1, whist, scan_tmp);
      if (cw > d1) cs_pass_next(keys, perm + lo, lo, m, d1, cw - d1, whist, scan_tmp);
      continue;
    }
    // ---- 1. segment parameters (rindex.py:164-198): with K1's per-segment
    // min / max, six threads integerise them in parallel; else the CTA
    // reduces the segment first
    if (a.seg_mm) {
      if (threadIdx.x < 6) {
        const int c = threadIdx.x >> 1;
        const float v = a.seg_mm[6 * (s0 / a.S) + threadIdx.x];
        cs_v[threadIdx.x] = v;
        if (!fm[c].is_const) {
          const double q = __ddiv_rn((double)v, fm[c].twob);
          cs_q[threadIdx.x] = (int64_t)rint(q);
          cs_big[threadIdx.x] = fabs(q) > kIntLimit;
        }
      }
    } else {
      float mn[3], mx[3];
#pragma unroll
      for (int c = 0; c < 3; c++) {
        mn[c] = __int_as_float(0x7f800000);
        mx[c] = -__int_as_float(0x7f800000);
      }
      for (int i = threadIdx.x; i < m; i += NT) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float v = a.x[c][s0 + i];
          mn[c] = fminf(mn[c], v);
          mx[c] = fmaxf(mx[c], v);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; c++) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
          mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
        if ((threadIdx.x & 31) == 0) {
          red[0][c][threadIdx.x >> 5] = mn[c];
          red[1][c][threadIdx.x >> 5] = mx[c];
        }
      }
      __syncthreads();
      if (threadIdx.x < 6) {
        const int c = threadIdx.x >> 1, hiw = threadIdx.x & 1;
        float v = red[hiw][c][0];
        for (int q = 1; q < NT / 32; q++)
          v = hiw ? fmaxf(v, red[1][c][q]) : fminf(v, red[0][c][q]);
        cs_v[threadIdx.x] = v;
        if (!fm[c].is_const) {
          const double q = __ddiv_rn((double)v, fm[c].twob);
          cs_q[threadIdx.x] = (int64_t)rint(q);
          cs_big[threadIdx.x] = fabs(q) > kIntLimit;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = 0, bad = 0;
      int64_t rng[3];
      for (int c = 0; c < 3; c++) {
        sp.amax[c] = fmaxf(fabsf(cs_v[2 * c]), fabsf(cs_v[2 * c + 1]));
        rng[c] = 0;
        if (fm[c].is_const) {
          sp.mn[c] = 0;
          continue;
        }
        bad |= cs_big[2 * c] | cs_big[2 * c + 1];
        sp.mn[c] = cs_q[2 * c];
        rng[c] = cs_q[2 * c + 1] - cs_q[2 * c];
        need = max(need, bitlen64((uint64_t)rng[c]));
      }
      const int bits = min(need, 21);
      const int drop = need > 21 ? need - 21 : 0;  // allow_key_clamp (pipeline.py:463)
      if (a.no_clamp && need > 21) bad = 1;       // CPC: BoundTooSmallError (rindex.py:185-190)
      const int eff = min(a.ig, bits);
      sp.bits = bits;
      sp.shift = drop + eff;
      sp.w = bits - eff;
      sp.bad = bad;
      int cw = 0, wmax = 0;
      for (int c = 0; c < 3; c++) {
        const int wt = sp.w > 0 ? bitlen64((uint64_t)rng[c] >> sp.shift) : 0;
        sp.wt[c] = wt;
        cw += wt;
        wmax = max(wmax, wt);
      }
      sp.cw = cw;
      sp.wmax = wmax;
    }
    __syncthreads();
    if (sp.bad) {
      if (threadIdx.x == 0) set_status(a.status, NBZG_BOUND_TOO_SMALL);
      return;
    }
    if (threadIdx.x == 0) {
      a.seg_bits[s0 / a.S] = (uint8_t)sp.bits;
      if (a.minima)
        for (int c = 0; c < 3; c++) a.minima[3 * (s0 / a.S) + c] = sp.mn[c];
    }
    const int cw = sp.cw;
    if (MODE == 1 && threadIdx.x == 0) a.seg_cw[s0 / a.S] = (uint8_t)(cw > kCsMaxBits ? 255 : cw);
    if (cw > kCsMaxBits) {  // the general kernel redoes this tile
      flagged = true;
      continue;
    }
    if (flagged) continue;  // (seg_bits / minima still written for every segment)
    if (cw == 0) {
      if (MODE == 0) {
        for (int i = threadIdx.x; i < m; i += NT) perm[lo + i] = (uint16_t)(lo + i);
        __syncthreads();
      }
      continue;
    }
    CS_T(0);  // segment parameters
    // ---- 2. compaction tables: T[t][b][v] = sum_i bit_i(v) << P_t(8b + i)
    const int nbyte = (sp.wmax + 7) >> 3;
    for (int e = threadIdx.x; e < 3 * nbyte * 256; e += NT) {
      const int tt = e / (nbyte * 256), b = (e >> 8) % nbyte, v = e & 255;
      uint32_t out = 0;
      for (int i = 0; i < 8; i++) {
        const int j = 8 * b + i;
        if (!((v >> i) & 1) || j >= sp.wt[tt]) continue;
        int pos = 0;
#pragma unroll
        for (int c = 0; c < 3; c++) pos += min(j, sp.wt[c]) + ((c > tt && j < sp.wt[c]) ? 1 : 0);
        out |= 1u << pos;
      }
      lut[tt][b][v] = out;
    }
    __syncthreads();
    CS_T(1);  // tables
    // ---- 3. compacted keys.  Exact integerisation rint(f64(x) / 2b)
    // (quantize.py:117-128) from the FP64 product t = x * (1/2b): |t - x/2b|
    // <= |t| 2^-51, so unless t is within tmax 2^-50 of a half-integer,
    // rint(t) equals the reference's rint of the rounded quotient; those
    // near-ties (probability ~2^-40) take the exact division out of line.
    // rint(t) = low word of t + 1.5 * 2^52 (|t| < 2^31).
    {
      const int shift = sp.shift;
      const int32_t m0 = (int32_t)sp.mn[0], m1 = (int32_t)sp.mn[1], m2 = (int32_t)sp.mn[2];
      const uint32_t lut_s = sh_addr(&lut[0][0][0]);
      uint16_t* kdst = MODE == 1 ? a.keys16 + s0 : keys;  // K2a: to HBM (s0 % 4 == 0)
      const double iv0 = fm[0].inv, iv1 = fm[1].inv, iv2 = fm[2].inv;
      bool small = true;
      double tie = 0.0;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const double tmax = (double)sp.amax[c] * fm[c].inv;
        small &= tmax < 1073741824.0 || fm[c].is_const;  // |k| < 2^30
        tie = fmax(tie, tmax * 8.881784197001252e-16);  // 2^-50
      }
      const double cut = 0.5 - tie;
      // one component: lattice index minus the segment minimum (near-ties
      // flagged in `slow`, fixed after a warp vote)
      auto comp = [&](float x, double inv, int32_t mn, uint32_t& slow, int bit) -> int32_t {
        const double t = __dmul_rn((double)x, inv);
        const double r = __dadd_rn(t, 6755399441055744.0);
        if (!(fabs(__dsub_rn(t, __dsub_rn(r, 6755399441055744.0))) < cut)) slow |= 1u << bit;
        return __double2loint(r) - mn;
      };
      auto lut3 = [&](uint32_t u0, uint32_t u1, uint32_t u2) -> uint32_t {
        uint32_t key = lds_u32(lut_s + 4u * (u0 & 255u)) | lds_u32(lut_s + 4u * (768u + (u1 & 255u))) |
                       lds_u32(lut_s + 4u * (1536u + (u2 & 255u)));
        if (nbyte > 1)
          key |= lds_u32(lut_s + 4u * (256u + ((u0 >> 8) & 255u))) |
                 lds_u32(lut_s + 4u * (1024u + ((u1 >> 8) & 255u))) |
                 lds_u32(lut_s + 4u * (1792u + ((u2 >> 8) & 255u)));
        if (nbyte > 2)
          key |= lds_u32(lut_s + 4u * (512u + ((u0 >> 16) & 255u))) |
                 lds_u32(lut_s + 4u * (1280u + ((u1 >> 16) & 255u))) |
                 lds_u32(lut_s + 4u * (2048u + ((u2 >> 16) & 255u)));
        return key;
      };
      auto key_of = [&](float x0, float x1, float x2) -> uint32_t {
        uint32_t slow = 0;
        int32_t d[3] = {comp(x0, iv0, m0, slow, 0), comp(x1, iv1, m1, slow, 1),
                        comp(x2, iv2, m2, slow, 2)};
        if (slow) {
          const float xv[3] = {x0, x1, x2};
          const int32_t mv[3] = {m0, m1, m2};
#pragma unroll
          for (int c = 0; c < 3; c++)
            if (slow & (1u << c)) d[c] = exact_index(xv[c], fm + c) - mv[c];
        }
        return lut3((uint32_t)d[0] >> shift, (uint32_t)d[1] >> shift, (uint32_t)d[2] >> shift);
      };
      if (!small) {  // indices beyond 2^30: the general kernel redoes the tile
        flagged = true;
        continue;
      }
      const int m4 = (s0 & 3) ? 0 : m >> 2;
      const float4* x4[3] = {reinterpret_cast<const float4*>(a.x[0] + s0),
                             reinterpret_cast<const float4*>(a.x[1] + s0),
                             reinterpret_cast<const float4*>(a.x[2] + s0)};
      // FP32 bucket path.  u = (rint(Q) - mn) >> s = floor(g) with
      // g = (Q - mn + 0.5) / 2^s, Q = f64(x) / 2b -- exactly, unless Q sits on
      // a bucket boundary (g an integer; a rint tie there is where rint's
      // half-even rule matters).  g32 = fma(x, fl32(inv/2^s), -(mn - 0.5)/2^s)
      // is within (gmax + tmax/2^s + 1) 2^-22 of g, so a fractional part of
      // g32 farther than that from 0 and 1 decides floor(g); the others (a
      // bucket edge per 2^s lattice units: ~2^-14 of the values here) take
      // the exact division.  Needs s >= 4, |mn| < 2^22 (mn - 0.5 exact in
      // FP32) and g < 2^21 (g + 1.5 2^23 rounded down is 1.5 2^23 + floor(g)).
      bool f32 = shift >= 4;
      float invs[3], cs[3];
      float lim = 0.5f;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const double sc = ldexp(1.0, -shift);
        invs[c] = (float)(fm[c].inv * sc);
        cs[c] = (float)(((double)sp.mn[c] - 0.5) * sc);
        f32 &= fm[c].is_const || (sp.mn[c] > -4194304 && sp.mn[c] < 4194304);
        const double tmax = (double)sp.amax[c] * fm[c].inv;
        const double eps = (ldexp(1.0, sp.w) + tmax * sc + 1.0) * 2.384185791015625e-07;  // 2^-22
        lim = fminf(lim, (float)(0.5 - 2.0 * eps));
      }
      f32 &= lim > 0.25f;
      if (f32) {
#pragma unroll 2  // two iterations' loads in flight
        for (int v = threadIdx.x; v < m4; v += NT) {
          const float4 q0 = __ldg(x4[0] + v), q1 = __ldg(x4[1] + v), q2 = __ldg(x4[2] + v);
          const float xv[12] = {q0.x, q1.x, q2.x, q0.y, q1.y, q2.y, q0.z, q1.z, q2.z, q0.w, q1.w, q2.w};
          uint32_t u[12];
          bool fine = true;  // one predicate accumulates; the edge set is rebuilt on the rare path
#pragma unroll
          for (int e = 0; e < 12; e++) {
            const float g = __fmaf_rn(xv[e], invs[e % 3], -cs[e % 3]);
            const float r = __fadd_rd(g, 12582912.0f);
            const float fr = __fsub_rn(g, __fsub_rn(r, 12582912.0f));
            fine = fine && (fabsf(__fsub_rn(fr, 0.5f)) < lim);
            u[e] = (uint32_t)(__float_as_int(r) - 0x4B400000);
          }
          if (__any_sync(__activemask(), !fine)) {  // bucket edges
            uint32_t slow = 0;
#pragma unroll
            for (int e = 0; e < 12; e++) {
              const float g = __fmaf_rn(xv[e], invs[e % 3], -cs[e % 3]);
              const float r = __fadd_rd(g, 12582912.0f);
              const float fr = __fsub_rn(g, __fsub_rn(r, 12582912.0f));
              if (!(fabsf(__fsub_rn(fr, 0.5f)) < lim)) slow |= 1u << e;
            }
#pragma unroll 1
            for (uint32_t sl = slow; sl; sl &= sl - 1) {
              const int e = __ffs(sl) - 1;
              float x = xv[0];
              int32_t mm = m0;
#pragma unroll
              for (int q = 0; q < 12; q++)
                if (q == e) x = xv[q], mm = (q % 3 == 0 ? m0 : (q % 3 == 1 ? m1 : m2));
              const uint32_t ue = (uint32_t)(exact_index(x, fm + e % 3) - mm) >> shift;
#pragma unroll
              for (int q = 0; q < 12; q++)
                if (q == e) u[q] = ue;
            }
          }
          uint32_t kk[4];
#pragma unroll
          for (int j = 0; j < 4; j++) kk[j] = lut3(u[3 * j], u[3 * j + 1], u[3 * j + 2]);
          *reinterpret_cast<uint2*>(kdst + 4 * v) =
              make_uint2(kk[0] | (kk[1] << 16), kk[2] | (kk[3] << 16));
        }
      } else
#pragma unroll 2  // two iterations' loads in flight
      for (int v = threadIdx.x; v < m4; v += NT) {
        const float4 q0 = __ldg(x4[0] + v), q1 = __ldg(x4[1] + v), q2 = __ldg(x4[2] + v);
        const float xv[12] = {q0.x, q1.x, q2.x, q0.y, q1.y, q2.y, q0.z, q1.z, q2.z, q0.w, q1.w, q2.w};
        const double ivs[3] = {iv0, iv1, iv2};
        const int32_t mvs[3] = {m0, m1, m2};
        uint32_t slow = 0;
        int32_t d[12];
#pragma unroll
        for (int e = 0; e < 12; e++) d[e] = comp(xv[e], ivs[e % 3], mvs[e % 3], slow, e);
        // (a ragged segment leaves some lanes of a warp outside this loop)
        if (__any_sync(__activemask(), slow != 0)) {  // near-ties: ~2^-40 per value
#pragma unroll 1
          for (uint32_t sl = slow; sl; sl &= sl - 1) {
            const int e = __ffs(sl) - 1;
            float x = xv[0];
            int32_t mm = m0;
#pragma unroll
            for (int q = 0; q < 12; q++)
              if (q == e) x = xv[q], mm = mvs[q % 3];
            const int32_t de = exact_index(x, fm + e % 3) - mm;
#pragma unroll
            for (int q = 0; q < 12; q++)
              if (q == e) d[q] = de;
          }
        }
        uint32_t kk[4];
#pragma unroll
        for (int j = 0; j < 4; j++)
          kk[j] = lut3((uint32_t)d[3 * j] >> shift, (uint32_t)d[3 * j + 1] >> shift,
                       (uint32_t)d[3 * j + 2] >> shift);
        *reinterpret_cast<uint2*>(kdst + 4 * v) = make_uint2(kk[0] | (kk[1] << 16), kk[2] | (kk[3] << 16));
      }
      for (int i = 4 * m4 + threadIdx.x; i < m; i += NT)
        kdst[i] = (uint16_t)key_of(a.x[0][s0 + i], a.x[1][s0 + i], a.x[2][s0 + i]);
    }
    __syncthreads();
    CS_T(2);  // keys
    // ---- 4. stable LSD over cw bits, output into this segment's perm range
    if (MODE == 0) {
      const int d1 = cw <= kCsOneBits ? cw : cw >> 1;  // one pass, or two balanced digits
      cs_pass<true>(keys, perm + lo, lo, m, 0, d1, whist, scan_tmp);
      if (cw > d1) cs_pass_next(keys, perm + lo, lo, m, d1, cw - d1, whist, scan_tmp);
    }
    CS_T(3);  // sort
  }
  if (flagged) {
    if (MODE != 2 && threadIdx.x == 0) a.tile_flags[t] = 1;
  } else if (MODE != 1) {
    // ---- write the tile's permutation (coalesced, 16 bytes per lane: tiles
    // start at multiples of 8 elements whenever the tile size is one)
    const int m8 = (t0 & 7) ? 0 : mt >> 3;
    for (int i = threadIdx.x; i < m8; i += NT)
      reinterpret_cast<uint4*>(a.perm + t0)[i] = reinterpret_cast<const uint4*>(perm)[i];
    for (int i = 8 * m8 + threadIdx.x; i < mt; i += NT) a.perm[t0 + i] = perm[i];
  }
  __syncthreads();  // perm is reused by the next tile
  CS_T(4);  // write-out
  }
#ifdef NBZG_CS_PROF
  if (threadIdx.x == 0 && blockIdx.x < 2)
    printf("csort CTA %d cycles: params %lld tables %lld keys %lld sort %lld out %lld\n", blockIdx.x,
           cs_t[0], cs_t[1], cs_t[2], cs_t[3], cs_t[4]);
#endif
}

__global__ void __launch_bounds__(kSortThreads, 2) rindex_csort_kernel(RArgs a) { csort_body<0>(a); }
__global__ void __launch_bounds__(kCsKeyThreads, 4) rindex_ckeys_kernel(RArgs a) { csort_body<1>(a); }
__global__ void __launch_bounds__(kSortThreads, 2) rindex_crank_kernel(RArgs a) { csort_body<2>(a); }

int launch_rindex_sort(const Plan& p, cudaStream_t st) {
  if (p.n == 0) return NBZG_OK;
  RArgs a;
  const int nk = p.variant == 2 ? 6 : 3;
  a.fbase = p.variant == 1 ? 3 : 0;
  for (int c = 0; c < 6; c++) a.x[c] = c < nk ? p.f[a.fbase + c] : nullptr;
  a.n = p.n;
  a.S = p.S;
  a.tile = p.tile;
  a.ntiles = p.ntiles;
  a.ig = p.ig;
  a.meta = p.meta;
  a.perm = p.perm;
  a.seg_bits = p.seg_bits;
  a.tile_flags = p.tile_flags;
  a.status = &p.meta->status;
  a.no_clamp = p.cpc ? 1 : 0;
  a.minima = p.cpc ? p.minima : nullptr;
  a.seg_mm = p.seg_mm;
  a.keys16 = p.keys16;
  a.seg_cw = p.seg_cw;
  size_t sm32 = kTileMax * (4 + 2) + kSortWarps * kRadix * 2;
  size_t sm64 = kTileMax * (8 + 2) + kSortWarps * kRadix * 2;
  size_t smc = kTileMax * (2 + 2) + (kSortWarps << kCsOneBits) * 2 + 3 * 3 * 256 * 4;
  smem_attr((const void*)rindex_csort_kernel, (int)smc);
  smem_attr((const void*)rindex_crank_kernel, (int)smc);
  const size_t smk = 3 * 3 * 256 * 4;  // K2a: the compaction tables only
  smem_attr((const void*)rindex_sort_kernel<uint32_t>, (int)sm32);
  smem_attr((const void*)rindex_sort_kernel<uint64_t>, (int)sm64);
  smem_attr((const void*)rindex_sort6_kernel<uint32_t>, (int)sm32);
  smem_attr((const void*)rindex_sort6_kernel<uint64_t>, (int)sm64);
  cudaMemsetAsync(p.tile_flags, 0, sizeof(uint32_t) * p.ntiles, st);
  if (nk == 6) {
    a.pass = 0;
    count_launch();
    rindex_sort6_kernel<uint32_t><<<(unsigned)p.ntiles, kSortThreads, sm32, st>>>(a);
    a.pass = 2;  // tiles whose 6-field keys exceed 32 bits
    count_launch();
    rindex_sort6_kernel<uint64_t><<<(unsigned)p.ntiles, kSortThreads, sm64, st>>>(a);
  } else {
    // compact-key sort; tiles with a segment of more than 16 varying key
    // bits (flag 1) are redone by the general kernel
    a.pass = 0;
    const unsigned gcs = (unsigned)min(p.ntiles, (int64_t)2 * sm_count());
#ifdef NBZG_CS_SPLIT
    // K2a: segment parameters + compacted keys, streamed at 4 CTAs/SM;
    // K2b: the counting sort from the u16 keys.  Measured at config 2:
    // 0.82 + 1.01 ms, the same as the fused kernel (1.82 ms): the sort
    // itself is the limiter, so the fused kernel (no key round trip) is the
    // default
    count_launch();
    rindex_ckeys_kernel<<<(unsigned)min(p.ntiles, (int64_t)4 * sm_count()), kCsKeyThreads, smk, st>>>(a);
    count_launch();
    rindex_crank_kernel<<<gcs, kSortThreads, smc, st>>>(a);
#else
    count_launch();
    rindex_csort_kernel<<<gcs, kSortThreads, smc, st>>>(a);
#endif
    a.pass = 1;
    count_launch();
    rindex_sort_kernel<uint32_t><<<(unsigned)p.ntiles, kSortThreads, sm32, st>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// ---------------------------------------------------------------- parity hooks
// Full 63-bit keys (rindex.py:164-198 + _kernels.py:778-786), one CTA per
// segment; used by nbzg_rindex_keys for bit-exact key parity.
struct KArgs {
  const float* x[3];
  int64_t n, S;
  double twob[3];
  double inv[3];
  float inv32[3];
  int is_const[3];
  uint64_t* keys;
  uint8_t* seg_bits;
  uint32_t* status;
};

__global__ void __launch_bounds__(256) rindex_keys_kernel(KArgs a) {
  const int64_t s0 = (int64_t)blockIdx.x * a.S;
  const int64_t s1 = min(a.n, s0 + a.S);
  __shared__ float red[2][3][8];
  __shared__ int64_t smn[3];
  __shared__ int sdrop, sbad;
  float mn[3], mx[3];
  for (int c = 0; c < 3; c++) {
    mn[c] = __int_as_float(0x7f800000);
    mx[c] = -__int_as_float(0x7f800000);
  }
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x)
    for (int c = 0; c < 3; c++) {
      float v = a.x[c][i];
      mn[c] = fminf(mn[c], v);
      mx[c] = fmaxf(mx[c], v);
    }
  for (int c = 0; c < 3; c++) {
    for (int o = 16; o; o >>= 1) {
      mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][c][threadIdx.x >> 5] = mn[c];
      red[1][c][threadIdx.x >> 5] = mx[c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int need = 0, bad = 0;
    for (int c = 0; c < 3; c++) {
      float a0 = red[0][c][0], b0 = red[1][c][0];
      for (int q = 1; q < 8; q++) {
        a0 = fminf(a0, red[0][c][q]);
        b0 = fmaxf(b0, red[1][c][q]);
      }
      if (a.is_const[c]) {
        smn[c] = 0;
        continue;
      }
      double qa = __ddiv_rn((double)a0, a.twob[c]), qb = __ddiv_rn((double)b0, a.twob[c]);
      if (fabs(qa) > kIntLimit || fabs(qb) > kIntLimit) bad = 1;
      int64_t ia = (int64_t)rint(qa), ib = (int64_t)rint(qb);
      smn[c] = ia;
      need = max(need, bitlen64((uint64_t)(ib - ia)));
    }
    int bits = min(need, 21);
    sdrop = need > 21 ? need - 21 : 0;
    sbad = bad;
    a.seg_bits[blockIdx.x] = (uint8_t)bits;
  }
  __syncthreads();
  if (sbad) {
    if (threadIdx.x == 0) set_status(a.status, NBZG_BOUND_TOO_SMALL);
    return;
  }
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    uint64_t u[3];
    for (int c = 0; c < 3; c++) {
      int64_t iv = 0;
      if (!a.is_const[c]) {
        bool fast;
        iv = (int64_t)lattice_index<true>(a.x[c][i], a.inv32[c], a.inv[c], a.twob[c], fast);
      }
      u[c] = (uint64_t)(iv - smn[c]) >> sdrop;
    }
    a.keys[i] = make_key<uint64_t>(u[0], u[1], u[2]);
  }
}

int launch_rindex_keys(const float* x, const float* y, const float* z, int64_t n,
                       const double* bounds3, int64_t S, uint64_t* keys, uint8_t* seg_bits,
                       uint32_t* status, cudaStream_t st) {
  KArgs a;
  a.x[0] = x;
  a.x[1] = y;
  a.x[2] = z;
  a.n = n;
  a.S = S;
  for (int c = 0; c < 3; c++) {
    a.is_const[c] = bounds3[c] <= 0.0;
    a.twob[c] = 2.0 * bounds3[c];
    a.inv[c] = a.is_const[c] ? 0.0 : 1.0 / a.twob[c];
    a.inv32[c] = (float)a.inv[c];
  }
  a.keys = keys;
  a.seg_bits = seg_bits;
  a.status = status;
  int64_t nseg = (n + S - 1) / S;
  if (nseg > 0) {
    count_launch();
    rindex_keys_kernel<<<(unsigned)nseg, 256, 0, st>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// prx_order parity hook on full keys (_kernels.py:887-927): one CTA per
// segment, masked key = key >> 3*min(k,bits), up to 63 bits (u64 smem keys).
struct OArgs {
  const uint64_t* keys;
  int64_t n, S;
  const uint8_t* seg_bits;
  int ig;
  int64_t* order;
};

__global__ void __launch_bounds__(kSortThreads) prx_order_kernel(OArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint16_t* perm = reinterpret_cast<uint16_t*>(keys + kTileMax);
  uint16_t* whist = perm + kTileMax;
  __shared__ uint32_t scan_tmp[33];
  const int64_t s0 = (int64_t)blockIdx.x * a.S;
  const int m = (int)(min(a.n, s0 + a.S) - s0);
  const int bits = a.seg_bits[blockIdx.x];
  const int eff = min(a.ig, bits);
  const int sort_bits = 3 * bits - 3 * eff;
  for (int i = threadIdx.x; i < m; i += kSortThreads) {
    perm[i] = (uint16_t)i;
    keys[i] = a.keys[s0 + i] >> (3 * eff);
  }
  __syncthreads();
  if (sort_bits > 0) block_sort_range<uint64_t>(keys, perm, 0, m, sort_bits, whist, scan_tmp);
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += kSortThreads) a.order[s0 + i] = s0 + perm[i];
}

int launch_prx_order(const uint64_t* keys, int64_t n, int64_t S, const uint8_t* seg_bits, int ig,
                     int64_t* order, cudaStream_t st) {
  if (S > kTileMax) return NBZG_UNSUPPORTED;
  OArgs a{keys, n, S, seg_bits, ig, order};
  size_t sm = kTileMax * (8 + 2) + kSortWarps * kRadix * 2;
  smem_attr((const void*)prx_order_kernel, (int)sm);
  int64_t nseg = (n + S - 1) / S;
  if (nseg > 0) {
    count_launch();
    prx_order_kernel<<<(unsigned)nseg, kSortThreads, sm, st>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// tile-local u16 permutation -> global int64 order (CompressResult.order)
__global__ void order_expand_kernel(const uint16_t* perm, int64_t n, int64_t tile,
                                    int64_t* order) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) order[i] = (i / tile) * tile + perm[i];
}

int launch_order_expand(const uint16_t* perm, int64_t n, int64_t tile, int64_t* order,
                        cudaStream_t st) {
  if (n > 0) {
    count_launch();
    order_expand_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(perm, n, tile, order);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
