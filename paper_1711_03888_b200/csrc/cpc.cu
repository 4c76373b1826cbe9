// cpc.cu -- CPC2000-family streams (Mode.SZ_CPC2000, Mode.CPC2000).
//
// Replaces pipeline._build_coord_stream / _parse_coord_stream
// (pipeline.py:316-375) with K.cpc_encode_keys / K.cpc_decode_keys
// (_kernels.py:566-601, 623-645), pipeline._build_vel_stream /
// _parse_vel_stream (pipeline.py:378-428) with K.vlc_encode_segmented /
// K.vlc_decode_segmented (_kernels.py:604-620, 648-660), the per-segment
// scheme choice pipeline._choose_schemes (pipeline.py:275-300) and
// pipeline._float32_corrections (pipeline.py:230-249).  The payload layout
// is the reference's:
//     ids[nseg] | u64 total_bits | bitstream (MSB-first bytes) | corrections
// (coordinate stream: three lists, x y z; velocity stream: one list; a list
// is u32 count + count x (u64 pos, f32 val)).  Archives written here (v2)
// append u32 seg_len_bits[nseg] -- the bit length of every segment -- so the
// decoder runs one thread per segment instead of walking the whole stream.
//
// Everything is segment-parallel: the full-key sort (K2 with k = 0 and no
// key clamp) left the tile-local permutation, seg bits and minima; here one
// CTA per (segment, stream) recomputes each sorted value's integer index
// exactly (FP32 fast path under a field-wide margin, else the FP64 division
// of quantize.integerize), forms the key delta (coordinates: interleaved
// min-subtracted indices) or zigzag magnitude (velocities), and
//   plan:  sums the VLC cost under both candidate schemes and counts
//          correction records -> per-segment bits / scheme / counts, then
//          per-stream scans (exclusive offsets, totals);
//   pack:  emits every value at its bit offset (block scan of code lengths
//          inside the segment) and writes the correction records in order.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

void trace_mark(const char* name, cudaStream_t st);  // capi.cu (bench stage trace)

constexpr int kCThreads = 512;
constexpr int kCSub = 1024;  // values per decode sub-block (v2 segment index)
__host__ __device__ inline int64_t cpc_subs(int64_t S) { return (S + kCSub - 1) / kCSub; }

__constant__ uint8_t c_vlcw[4][8] = {{2, 4, 6, 8, 12, 16, 24, 33},
                                     {4, 8, 16, 24, 32, 40, 48, 64},
                                     {2, 4, 6, 8, 12, 16, 24, 33},
                                     {4, 8, 16, 24, 32, 40, 48, 64}};

// bucket of magnitude m under scheme sid (encode.py:324-339); 8 = no bucket
NBZG_DEV int vlc_bucket(uint64_t m, int sid) {
#pragma unroll
  for (int b = 0; b < 8; b++) {
    const int w = c_vlcw[sid][b];
    if (w >= 64 || m < (1ull << w)) return b;
  }
  return 8;
}
// inverse of spread3_64: bits 0, 3, 6, ... -> 0, 1, 2, ... (21 bits)
NBZG_DEV uint64_t compact3_64(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v | (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v | (v >> 8)) & 0x1F0000FF0000FFull;
  v = (v | (v >> 16)) & 0x1F00000000FFFFull;
  v = (v | (v >> 32)) & 0x1FFFFFull;
  return v;
}
NBZG_DEV int vlc_len(int b, int sid) { return (b < 7 ? b + 1 : 7) + c_vlcw[sid][b]; }

// Shared-memory tables of a CPC CTA: VLC bucket and code length by the
// magnitude's bit length (m < 2^w  <=>  bitlen(m) <= w), bucket widths, and
// the 11-bit 3-way bit spread for key interleaving (interleave3,
// _kernels.py:757-786: bit j of a field -> key bit 3j).
struct CTabs {
  uint8_t bkt[4][65];   // bucket, 8 = no bucket
  uint8_t len[4][65];   // prefix + payload bits, 0 = no bucket
  uint8_t w[4][8];
  uint32_t sp11[2048];
};
NBZG_DEV void ctabs_init(CTabs& T) {
  for (int i = threadIdx.x; i < 4 * 65; i += blockDim.x) {
    const int sid = i / 65, bl = i % 65;
    int b = 8;
    for (int bb = 0; bb < 8; bb++)
      if (c_vlcw[sid][bb] >= 64 || bl <= c_vlcw[sid][bb]) {
        b = bb;
        break;
      }
    T.bkt[sid][bl] = (uint8_t)b;
    T.len[sid][bl] = (uint8_t)(b < 8 ? vlc_len(b, sid) : 0);
  }
  for (int i = threadIdx.x; i < 32; i += blockDim.x) T.w[i >> 3][i & 7] = c_vlcw[i >> 3][i & 7];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) T.sp11[i] = spread3_32((uint32_t)i);
}
NBZG_DEV int bitlen_u64(uint64_t m) { return 64 - __clzll((long long)m); }
NBZG_DEV uint64_t spread21(const CTabs& T, uint64_t v) {
  return (uint64_t)T.sp11[v & 0x7ffu] | ((uint64_t)T.sp11[(v >> 11) & 0x3ffu] << 33);
}

struct CStream {
  // per stream (0 coordinates, 1..3 velocity fields 3..5)
  uint64_t* seg_cost;  // [nseg] bits of the segment (raw key included)
  uint8_t* seg_id;     // [nseg]
  uint64_t* seg_off;   // [nseg + 1] exclusive bit offsets
  uint32_t* corr_cnt;  // [3][nseg] correction records per list
  uint32_t* corr_off;  // [3][nseg + 1]
  uint32_t* run_bits;  // [2][nseg][kCThreads] bits of each thread's run per candidate
};

struct CArgs {
  const float* f[6];
  int64_t n, S, tile, nseg;
  const uint16_t* perm;
  const uint8_t* seg_bits;
  const int64_t* minima;
  const nbzg_meta* meta;
  int nstreams;  // 1 (sz-cpc2000) or 4 (cpc2000)
  CStream st[4];
  nbzg_cpc_meta* cm;
  uint8_t* arena;   // pack: payloads at cm->off[s]
};

// field-wide FP32 margin (same argument as quantize_kernel); negative = never fast
NBZG_DEV float field_margin(const nbzg_field_meta& fm) {
  const float tmax = fmaxf(fabsf(fm.lo), fabsf(fm.hi)) * fm.inv32;
  if (!(tmax < 4194304.0f)) return -1.0f;
  return 0.5f - __fmaf_ru(tmax, 2.384185791015625e-07f, 9.5367431640625e-07f);
}
// quantize.integerize (quantize.py:117-128): rint(f64(x) / 2b)
NBZG_DEV int64_t integerize_m(float x, const nbzg_field_meta& fm, float cm, bool& big) {
  const float t = x * fm.inv32;
  const float r = t + 12582912.0f;
  const float d = t - (r - 12582912.0f);
  if (fabsf(d) < cm) return (int64_t)(__float_as_int(r) - 0x4B400000);
  const double q = __ddiv_rn((double)x, fm.twob);
  if (fabs(q) > kIntLimit) big = true;
  return (int64_t)rint(q);
}
// _float32_corrections test (pipeline.py:230-237)
NBZG_DEV bool needs_corr(float x, int64_t iv, const nbzg_field_meta& fm) {
  const float r = (float)__dmul_rn((double)iv, fm.twob);
  return fabs((double)x - (double)r) > fm.bound;
}

struct SegPos {
  int64_t lo, hi, tb;  // segment [lo, hi), tile base
  int s;
};
NBZG_DEV SegPos seg_pos(const CArgs& a, int64_t s) {
  SegPos p;
  p.s = (int)s;
  p.lo = s * a.S;
  p.hi = min(a.n, p.lo + a.S);
  p.tb = (p.lo / a.tile) * a.tile;
  return p;
}
NBZG_DEV int64_t src_of(const CArgs& a, const SegPos& p, int64_t i) { return p.tb + a.perm[i]; }

// a stream whose field(s) are constant has no payload (pipeline.py:482, 487)
NBZG_DEV bool stream_absent(const CArgs& a, int sidx) {
  return sidx == 0 ? (a.meta->mask & 7u) == 7u : ((a.meta->mask >> (2 + sidx)) & 1u) != 0;
}

template <int ST>
struct Eval;
// coordinates: key of position i (interleave3 of min-subtracted indices)
template <>
struct Eval<0> {
  float cm[3];
  uint32_t cmask;  // constant coordinates
  const CTabs* tabs;
  NBZG_DEV void init(const CArgs& a, const CTabs* t) {
    tabs = t;
    cmask = a.meta->mask & 7u;
    for (int c = 0; c < 3; c++) cm[c] = field_margin(a.meta->f[c]);
  }
  template <bool CORR = true>
  NBZG_DEV uint64_t key(const CArgs& a, const SegPos& p, int64_t i, uint32_t& corr, bool& big) {
    const int64_t src = src_of(a, p, i);
    uint64_t k = 0;
    corr = 0;
#pragma unroll
    for (int c = 0; c < 3; c++) {
      if (cmask & (1u << c)) continue;
      const nbzg_field_meta& fm = a.meta->f[c];
      const float x = a.f[c][src];
      const int64_t iv = integerize_m(x, fm, cm[c], big);
      k |= spread21(*tabs, (uint64_t)(iv - a.minima[3 * p.s + c])) << (2 - c);
      if (CORR && needs_corr(x, iv, fm)) corr |= 1u << c;
    }
    return k;
  }
};

template <int ST>
NBZG_DEV void vel_init(const CArgs& a, float& cm) { cm = field_margin(a.meta->f[2 + ST]); }
template <int ST, bool CORR = true>
NBZG_DEV uint64_t vel_mag(const CArgs& a, const SegPos& p, int64_t i, float cm, uint32_t& corr,
                          bool& big) {
  const int fi = 2 + ST;
  const nbzg_field_meta& fm = a.meta->f[fi];
  const float x = a.f[fi][src_of(a, p, i)];
  const int64_t iv = integerize_m(x, fm, cm, big);
  corr = CORR && needs_corr(x, iv, fm) ? 1u : 0u;
  return ((uint64_t)iv << 1) ^ (uint64_t)(iv >> 63);  // zigzag, encode.py:309-312
}

// ---------------------------------------------------------------- plan
// grid (nseg, nstreams): per segment bits under both candidates -> choice
__global__ void __launch_bounds__(kCThreads) cpc_plan_kernel(CArgs a) {
  const int sidx = blockIdx.y;
  if (stream_absent(a, sidx)) return;
  __shared__ CTabs tabs;
  ctabs_init(tabs);
  __syncthreads();
  const SegPos p = seg_pos(a, blockIdx.x);
  const int64_t m = p.hi - p.lo;
  const int64_t cpt = (m + kCThreads - 1) / kCThreads;
  const int64_t i0 = p.lo + threadIdx.x * cpt, i1 = min(p.hi, i0 + cpt);
  const int c0 = sidx == 0 ? 2 : 0;  // unsigned (coordinate deltas) / signed candidates
  uint64_t cost0 = 0, cost1 = 0;
  uint32_t bad0 = 0, bad1 = 0, nc[3] = {0, 0, 0};
  bool big = false;
  if (i0 < i1) {
    if (sidx == 0) {
      Eval<0> E;
      E.init(a, &tabs);
      uint32_t cr;
      uint64_t prev = i0 > p.lo ? E.key(a, p, i0 - 1, cr, big) : 0;
      for (int64_t i = i0; i < i1; i++) {
        const uint64_t k = E.key(a, p, i, cr, big);
#pragma unroll
        for (int c = 0; c < 3; c++) nc[c] += (cr >> c) & 1u;
        if (i > p.lo) {
          const int bl = bitlen_u64(k - prev);
          const uint32_t l0 = tabs.len[c0][bl], l1 = tabs.len[c0 + 1][bl];
          bad0 |= l0 == 0;
          bad1 |= l1 == 0;
          cost0 += l0;
          cost1 += l1;
        }
        prev = k;
      }
    } else {
      float cm;
      if (sidx == 1) vel_init<1>(a, cm);
      else if (sidx == 2) vel_init<2>(a, cm);
      else vel_init<3>(a, cm);
      for (int64_t i = i0; i < i1; i++) {
        uint32_t cr;
        const uint64_t ms = sidx == 1 ? vel_mag<1>(a, p, i, cm, cr, big)
                            : sidx == 2 ? vel_mag<2>(a, p, i, cm, cr, big)
                                        : vel_mag<3>(a, p, i, cm, cr, big);
        nc[0] += cr;
        const int bl = bitlen_u64(ms);
        const uint32_t l0 = tabs.len[c0][bl], l1 = tabs.len[c0 + 1][bl];
        bad0 |= l0 == 0;
        bad1 |= l1 == 0;
        cost0 += l0;
        cost1 += l1;
      }
    }
  }
  {
    // per-thread run bits under both candidates (pack needs no length pass)
    const uint32_t raw = (i0 < i1 && i0 == p.lo && sidx == 0) ? 3u * a.seg_bits[p.s] : 0u;
    uint32_t* rb = a.st[sidx].run_bits + (size_t)p.s * kCThreads + threadIdx.x;
    rb[0] = (uint32_t)cost0 + raw;
    rb[(size_t)a.nseg * kCThreads] = (uint32_t)cost1 + raw;
  }
  __shared__ uint64_t r64[2][kCThreads / 32];
  __shared__ uint32_t r32[5][kCThreads / 32];
  cost0 = warp_sum<uint64_t>(cost0);
  cost1 = warp_sum<uint64_t>(cost1);
  uint32_t v[5] = {bad0, bad1, nc[0], nc[1], nc[2]};
#pragma unroll
  for (int q = 0; q < 5; q++) v[q] = warp_sum(v[q]);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    r64[0][w] = cost0;
    r64[1][w] = cost1;
#pragma unroll
    for (int q = 0; q < 5; q++) r32[q][w] = v[q];
  }
  if (big) atomicCAS(&a.cm->status, 0u, (uint32_t)NBZG_BOUND_TOO_SMALL);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s0 = 0, s1 = 0;
    uint32_t t[5] = {0, 0, 0, 0, 0};
    for (int q = 0; q < kCThreads / 32; q++) {
      s0 += r64[0][q];
      s1 += r64[1][q];
      for (int u = 0; u < 5; u++) t[u] += r32[u][q];
    }
    // cheaper candidate wins, ties to the first (pipeline.py:294-296)
    int id;
    uint64_t best;
    if (!t[0] && (t[1] || s0 <= s1)) {
      id = c0;
      best = s0;
    } else if (!t[1]) {
      id = c0 + 1;
      best = s1;
    } else {
      atomicCAS(&a.cm->status, 0u, (uint32_t)NBZG_CODE_TOO_LONG);  // EncodeError
      id = c0;
      best = 0;
    }
    const CStream& S = a.st[sidx];
    S.seg_cost[p.s] = best + (sidx == 0 ? 3ull * a.seg_bits[p.s] : 0ull);
    S.seg_id[p.s] = (uint8_t)id;
    const int nl = sidx == 0 ? 3 : 1;
    for (int c = 0; c < nl; c++) S.corr_cnt[(size_t)c * a.nseg + p.s] = t[2 + c];
  }
}

// per stream: exclusive scans of segment bits and correction counts; totals
__global__ void __launch_bounds__(1024) cpc_scan_kernel(CArgs a) {
  const int sidx = blockIdx.x;
  if (stream_absent(a, sidx)) return;
  const CStream& S = a.st[sidx];
  __shared__ unsigned long long tmp[33];
  const int64_t R = (a.nseg + blockDim.x - 1) / blockDim.x;
  const int nl = sidx == 0 ? 3 : 1;
  for (int list = -1; list < nl; list++) {
    unsigned long long s = 0;
    for (int64_t r = 0; r < R; r++) {
      const int64_t i = (int64_t)threadIdx.x * R + r;
      if (i < a.nseg) s += list < 0 ? S.seg_cost[i] : S.corr_cnt[(size_t)list * a.nseg + i];
    }
    unsigned long long tot;
    unsigned long long ex = block_excl_scan<unsigned long long>(s, tmp, &tot);
    for (int64_t r = 0; r < R; r++) {
      const int64_t i = (int64_t)threadIdx.x * R + r;
      if (i < a.nseg) {
        if (list < 0) {
          S.seg_off[i] = ex;
          ex += S.seg_cost[i];
        } else {
          S.corr_off[(size_t)list * (a.nseg + 1) + i] = (uint32_t)ex;
          ex += S.corr_cnt[(size_t)list * a.nseg + i];
        }
      }
    }
    if (threadIdx.x == 0) {
      if (list < 0) {
        S.seg_off[a.nseg] = tot;
        a.cm->total_bits[sidx] = tot;
      } else {
        S.corr_off[(size_t)list * (a.nseg + 1) + a.nseg] = (uint32_t)tot;
        a.cm->corr[sidx][list] = tot;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint64_t len = (uint64_t)a.nseg + 8 + (a.cm->total_bits[sidx] + 7) / 8 +
                   4ull * a.nseg * (uint64_t)cpc_subs(a.S);
    for (int c = 0; c < nl; c++) len += 4 + 12 * a.cm->corr[sidx][c];
    a.cm->len[sidx] = len;
  }
}

// ---------------------------------------------------------------- pack
// bit sink over the payload's 16-byte aligned bit region (zeroed): words are
// stored byte-swapped (MSB-first bytes); the first and last word of a
// thread's run can be shared with its neighbours and go out with atomicOr
struct BitSink {
  // 32-bit MSB-aligned pending word `cur` holding `nacc` < 32 bits; words
  // are stored byte-swapped (MSB-first bytes); the first word of a thread's
  // run (and the last, in finish) can be shared with a neighbour: atomicOr
  uint32_t* words;
  uint32_t cur;
  uint32_t nacc;
  uint64_t wi;     // word index of the pending word
  bool first;
  NBZG_DEV void init(uint32_t* w, uint64_t bitpos) {
    words = w;
    wi = bitpos >> 5;
    nacc = (uint32_t)(bitpos & 31);
    cur = 0;
    first = true;
  }
  NBZG_DEV void emit(uint32_t v) {
    const uint32_t be = __byte_perm(v, 0, 0x0123);
    if (first) atomicOr(words + wi, be);
    else words[wi] = be;
    first = false;
    wi++;
  }
  NBZG_DEV void put_msb(uint32_t wl, uint32_t l) {  // l in [1, 32], wl MSB-aligned
    cur |= wl >> nacc;
    const uint32_t spill = __funnelshift_lc(0u, wl, 32 - nacc);  // wl << (32 - nacc)
    const uint32_t t = nacc + l;
    if (t >= 32) {
      emit(cur);
      cur = spill;
    }
    nacc = t & 31u;
  }
  NBZG_DEV void put(uint64_t v, int nb) {  // nb <= 32, v < 2^nb
    if (nb > 0) put_msb((uint32_t)v << (32 - nb), (uint32_t)nb);
  }
  NBZG_DEV void put64(uint64_t v, int nb) {
    if (nb > 32) {
      put(v >> 32, nb - 32);
      put(v & 0xffffffffull, 32);
    } else {
      put(v, nb);
    }
  }
  NBZG_DEV void finish() {
    if (nacc > 0) atomicOr(words + wi, __byte_perm(cur, 0, 0x0123));
  }
};

// one VLC code (_kernels.py:604-620): unary bucket prefix + payload; a code
// of <= 32 bits goes in with one append
NBZG_DEV void vlc_emit(BitSink& B, uint64_t m, int sid, const CTabs& T) {
  const int b = T.bkt[sid][bitlen_u64(m)];
  const uint32_t plen = b < 7 ? (uint32_t)b + 1 : 7u;
  const uint32_t pval = b < 7 ? (1u << (b + 1)) - 2 : 127u;
  const uint32_t w = T.w[sid][b];
  const uint32_t tot = plen + w;
  if (tot <= 32) {
    B.put_msb((pval << (32 - plen)) | (uint32_t)(m << (32 - tot)), tot);
  } else {
    B.put(pval, (int)plen);
    B.put64(m, (int)w);
  }
}

// grid (nseg, nstreams): the bitstream of every segment
__global__ void __launch_bounds__(kCThreads) cpc_pack_kernel(CArgs a) {
  const int sidx = blockIdx.y;
  if (stream_absent(a, sidx)) return;
  __shared__ CTabs tabs;
  ctabs_init(tabs);
  __syncthreads();
  const SegPos p = seg_pos(a, blockIdx.x);
  const CStream& S = a.st[sidx];
  const int sid = S.seg_id[p.s];
  const int64_t m = p.hi - p.lo;
  const int64_t cpt = (m + kCThreads - 1) / kCThreads;
  const int64_t i0 = p.lo + threadIdx.x * cpt, i1 = min(p.hi, i0 + cpt);
  const int kb = sidx == 0 ? 3 * a.seg_bits[p.s] : 0;
  bool big = false;
  Eval<0> E;
  float cm = 0.0f;
  if (sidx == 0) E.init(a, &tabs);
  else if (sidx == 1) vel_init<1>(a, cm);
  else if (sidx == 2) vel_init<2>(a, cm);
  else vel_init<3>(a, cm);
  auto value = [&](int64_t i, uint32_t& cr) -> uint64_t {
    return sidx == 1 ? vel_mag<1, false>(a, p, i, cm, cr, big)
           : sidx == 2 ? vel_mag<2, false>(a, p, i, cm, cr, big)
                       : vel_mag<3, false>(a, p, i, cm, cr, big);
  };
  // bits of this thread's run under the chosen scheme (from the plan)
  const int cand = sid - (sidx == 0 ? 2 : 0);
  const uint64_t L = S.run_bits[((size_t)cand * a.nseg + p.s) * kCThreads + threadIdx.x];
  uint64_t prev = 0;
  uint32_t cr;
  if (i0 < i1 && sidx == 0) prev = i0 > p.lo ? E.key<false>(a, p, i0 - 1, cr, big) : 0;
  __shared__ unsigned long long tmp[33];
  unsigned long long tot;
  const uint64_t o = S.seg_off[p.s] + block_excl_scan<unsigned long long>(L, tmp, &tot);
  if (i0 < i1) {
    uint8_t* pay = a.arena + a.cm->off[sidx];
    uint32_t* words = reinterpret_cast<uint32_t*>(pay + a.nseg + 8);
    // v2 sub-block index: bit offset (from the segment start) of every
    // kCSub-th value, after the u32 segment lengths
    const int64_t subs = cpc_subs(a.S);
    uint8_t* sub = pay + a.cm->len[sidx] - 4 * (uint64_t)a.nseg * subs + 4 * a.nseg +
                   4 * (uint64_t)p.s * (subs - 1);
    const uint64_t seg0 = S.seg_off[p.s];
    auto mark = [&](int64_t i, const BitSink& B) {
      const int64_t r = i - p.lo;
      if (r > 0 && (r & (kCSub - 1)) == 0) {
        const uint32_t v = (uint32_t)(B.wi * 32 + B.nacc - seg0);
        uint8_t* d = sub + 4 * (r / kCSub - 1);
        for (int b = 0; b < 4; b++) d[b] = (uint8_t)(v >> (8 * b));
      }
    };
    BitSink B;
    B.init(words, o);
    if (sidx == 0) {
      uint64_t pv = prev;
      for (int64_t i = i0; i < i1; i++) {
        const uint64_t k = E.key<false>(a, p, i, cr, big);
        mark(i, B);
        if (i == p.lo) B.put64(k, kb);
        else vlc_emit(B, k - pv, sid, tabs);
        pv = k;
      }
    } else {
      for (int64_t i = i0; i < i1; i++) {
        mark(i, B);
        vlc_emit(B, value(i, cr), sid, tabs);
      }
    }
    B.finish();
  }
}

// correction records in position order: (u64 pos, f32 val), 12 bytes each
NBZG_DEV void put_rec(uint8_t* d, uint64_t pos, float v) {
  const uint32_t u = __float_as_uint(v);
#pragma unroll
  for (int b = 0; b < 8; b++) d[b] = (uint8_t)(pos >> (8 * b));
#pragma unroll
  for (int b = 0; b < 4; b++) d[8 + b] = (uint8_t)(u >> (8 * b));
}

// grid (nseg, nstreams): correction records (after the bit packing, so no
// plain byte store races an atomicOr on the bit region's last word)
__global__ void __launch_bounds__(kCThreads) cpc_corr_kernel(CArgs a) {
  const int sidx = blockIdx.y;
  if (stream_absent(a, sidx)) return;
  __shared__ CTabs tabs;
  const SegPos p = seg_pos(a, blockIdx.x);
  const CStream& S = a.st[sidx];
  const int nl = sidx == 0 ? 3 : 1;
  bool any = false;
  for (int c = 0; c < nl; c++) any |= S.corr_cnt[(size_t)c * a.nseg + p.s] != 0;
  if (!any) return;  // block-uniform
  ctabs_init(tabs);
  __syncthreads();
  const int64_t m = p.hi - p.lo;
  const int64_t cpt = (m + kCThreads - 1) / kCThreads;
  const int64_t i0 = p.lo + threadIdx.x * cpt, i1 = min(p.hi, i0 + cpt);
  bool big = false;
  Eval<0> E;
  float cm = 0.0f;
  if (sidx == 0) E.init(a, &tabs);
  else if (sidx == 1) vel_init<1>(a, cm);
  else if (sidx == 2) vel_init<2>(a, cm);
  else vel_init<3>(a, cm);
  uint32_t cnt[3] = {0, 0, 0};
  uint32_t cr;
  for (int64_t i = i0; i < i1; i++) {
    if (sidx == 0) E.key(a, p, i, cr, big);
    else if (sidx == 1) vel_mag<1>(a, p, i, cm, cr, big);
    else if (sidx == 2) vel_mag<2>(a, p, i, cm, cr, big);
    else vel_mag<3>(a, p, i, cm, cr, big);
    for (int c = 0; c < nl; c++) cnt[c] += (cr >> c) & 1u;
  }
  __shared__ unsigned long long tmp[33];
  uint8_t* pay = a.arena + a.cm->off[sidx];
  uint64_t base = (uint64_t)a.nseg + 8 + (a.cm->total_bits[sidx] + 7) / 8;
  uint32_t rank[3];
  for (int c = 0; c < nl; c++) {
    unsigned long long tot;
    rank[c] = S.corr_off[(size_t)c * (a.nseg + 1) + p.s] +
              (uint32_t)block_excl_scan<unsigned long long>(cnt[c], tmp, &tot);
    __syncthreads();
  }
  uint64_t lbase[3];
  for (int c = 0; c < nl; c++) {
    lbase[c] = base + 4;
    base += 4 + 12 * a.cm->corr[sidx][c];
  }
  for (int64_t i = i0; i < i1; i++) {
    int64_t src = src_of(a, p, i);
    if (sidx == 0) E.key(a, p, i, cr, big);
    else if (sidx == 1) vel_mag<1>(a, p, i, cm, cr, big);
    else if (sidx == 2) vel_mag<2>(a, p, i, cm, cr, big);
    else vel_mag<3>(a, p, i, cm, cr, big);
    for (int c = 0; c < nl; c++) {
      if ((cr >> c) & 1u) {
        const int fi = sidx == 0 ? c : 2 + sidx;
        put_rec(pay + lbase[c] + 12ull * rank[c], (uint64_t)i, a.f[fi][src]);
        rank[c]++;
      }
    }
  }
}

// per stream: ids, total_bits, list counts, segment index trailer
__global__ void cpc_frame_kernel(CArgs a) {
  const int sidx = blockIdx.x;
  if (stream_absent(a, sidx)) return;
  const CStream& S = a.st[sidx];
  uint8_t* pay = a.arena + a.cm->off[sidx];
  const uint64_t total = a.cm->total_bits[sidx];
  for (int64_t s = threadIdx.x; s < a.nseg; s += blockDim.x) pay[s] = S.seg_id[s];
  const int nl = sidx == 0 ? 3 : 1;
  uint64_t base = (uint64_t)a.nseg + 8 + (total + 7) / 8;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; b++) pay[a.nseg + b] = (uint8_t)(total >> (8 * b));
    for (int c = 0; c < nl; c++) {
      const uint64_t cnt = a.cm->corr[sidx][c];
      for (int b = 0; b < 4; b++) pay[base + b] = (uint8_t)(cnt >> (8 * b));
      base += 4 + 12 * cnt;
    }
  }
  if (threadIdx.x != 0) {
    for (int c = 0; c < nl; c++) base += 4 + 12 * a.cm->corr[sidx][c];
  }
  const int64_t subs = cpc_subs(a.S);
  for (int64_t s = threadIdx.x; s < a.nseg; s += blockDim.x) {
    const uint32_t v = (uint32_t)S.seg_cost[s];
    uint8_t* d = pay + base + 4 * s;
    for (int b = 0; b < 4; b++) d[b] = (uint8_t)(v >> (8 * b));
    // sub-blocks past a short segment's end repeat its length
    const int64_t m = min(a.S, a.n - s * a.S);
    for (int64_t k = (m + kCSub - 1) / kCSub; k < subs; k++) {
      uint8_t* e = pay + base + 4 * a.nseg + 4 * (s * (subs - 1) + k - 1);
      for (int b = 0; b < 4; b++) e[b] = (uint8_t)(v >> (8 * b));
    }
  }
}

// ---------------------------------------------------------------- decode
struct KArgsD {
  const uint8_t* pay;
  int64_t len, n, S, nseg;
  int kind;  // 2 coordinates (RINDEX), 1 velocity (VLC_FIELD)
  const uint8_t* seg_bits;
  const int64_t* minima;
  double twob[3];
  float* out[3];
  uint64_t* seg_off;  // [nseg + 1]
  uint32_t* status;
  uint64_t total;
  int64_t bits_at;  // payload offset of the bit region
  int64_t tr_bytes; // v2 segment index bytes at the payload end (0 for v1)
  int64_t subs;     // sub-blocks per segment
};

NBZG_DEV uint32_t ld_u32_le(const uint8_t* d) {
  return (uint32_t)d[0] | ((uint32_t)d[1] << 8) | ((uint32_t)d[2] << 16) | ((uint32_t)d[3] << 24);
}

// sequential bit reader over the MSB-first bytes (4-byte aligned loads)
struct BitSrc {
  // 16-byte blocks, one prefetched ahead: the refill of the 64-bit window
  // takes words from the current block and a block's load is issued four
  // words before it is needed, so the decode chain rarely waits on memory
  const uint4* g;     // 16-byte aligned base
  uint64_t cur;       // MSB-aligned window
  int nv;             // valid bits in cur
  uint32_t q0, q1, q2, q3;  // current block (byte-swapped), qn words left (from q0)
  int qn;
  uint4 nq;           // next block (raw), loaded ahead
  uint64_t nb;        // index of the block after nq
  NBZG_DEV void take_block() {
    q0 = __byte_perm(nq.x, 0, 0x0123);
    q1 = __byte_perm(nq.y, 0, 0x0123);
    q2 = __byte_perm(nq.z, 0, 0x0123);
    q3 = __byte_perm(nq.w, 0, 0x0123);
    qn = 4;
    nq = __ldg(g + nb);
    nb++;
  }
  NBZG_DEV uint32_t take_word() {
    if (qn == 0) take_block();
    const uint32_t v = q0;
    q0 = q1;
    q1 = q2;
    q2 = q3;
    qn--;
    return v;
  }
  NBZG_DEV void init(const uint8_t* p, uint64_t bitpos) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    g = reinterpret_cast<const uint4*>(base);
    const uint64_t pos = bitpos + 8 * (reinterpret_cast<uintptr_t>(p) & 15);
    const uint64_t blk = pos >> 7;
    nq = __ldg(g + blk);
    nb = blk + 1;
    take_block();
    for (int k = (int)((pos >> 5) & 3); k > 0; k--) take_word();
    cur = 0;
    nv = 0;
    fill();
    const int skip = (int)(pos & 31);
    cur <<= skip;
    nv -= skip;
    fill();
  }
  NBZG_DEV void fill() {
    while (nv <= 32) {
      cur |= (uint64_t)take_word() << (32 - nv);
      nv += 32;
    }
  }
  NBZG_DEV uint64_t get(int nb2) {  // nb2 <= 32
    if (nb2 <= 0) return 0;
    const uint64_t v = cur >> (64 - nb2);
    cur <<= nb2;
    nv -= nb2;
    fill();
    return v;
  }
  NBZG_DEV uint64_t get64(int nb2) {
    if (nb2 > 32) {
      const uint64_t hi = get(nb2 - 32);
      return (hi << 32) | get(32);
    }
    return get(nb2);
  }
  NBZG_DEV int ones7() {  // leading ones of the window, capped at 7
    const int o = __clz(~(uint32_t)(cur >> 32));
    return o < 7 ? o : 7;
  }
};

// per segment bit lengths (u32 trailer) -> exclusive offsets
__global__ void __launch_bounds__(1024) cpc_dec_offsets_kernel(KArgsD a) {
  __shared__ unsigned long long tmp[33];
  const int64_t R = (a.nseg + blockDim.x - 1) / blockDim.x;
  const uint8_t* tr = a.pay + a.len - a.tr_bytes;
  unsigned long long s = 0;
  auto rd = [&](int64_t i) -> uint32_t {
    const uint8_t* d = tr + 4 * i;
    return (uint32_t)d[0] | ((uint32_t)d[1] << 8) | ((uint32_t)d[2] << 16) | ((uint32_t)d[3] << 24);
  };
  for (int64_t r = 0; r < R; r++) {
    const int64_t i = (int64_t)threadIdx.x * R + r;
    if (i < a.nseg) s += rd(i);
  }
  unsigned long long tot;
  unsigned long long ex = block_excl_scan<unsigned long long>(s, tmp, &tot);
  for (int64_t r = 0; r < R; r++) {
    const int64_t i = (int64_t)threadIdx.x * R + r;
    if (i < a.nseg) {
      a.seg_off[i] = ex;
      ex += rd(i);
    }
  }
  if (threadIdx.x == 0) {
    a.seg_off[a.nseg] = tot;
    if (tot != a.total) atomicCAS(a.status, 0u, (uint32_t)NBZG_BAD_STREAM);
  }
}

// reference (v1) streams carry no segment index: one thread walks the
// stream once, skipping values (_kernels.py:566-601 / 604-620 order)
__global__ void cpc_dec_walk_kernel(KArgsD a, const uint8_t* ids) {
  if (threadIdx.x || blockIdx.x) return;
  BitSrc B;
  B.init(a.pay + a.bits_at, 0);
  uint64_t pos = 0;
  for (int64_t s = 0; s < a.nseg; s++) {
    a.seg_off[s] = pos;
    const int64_t lo = s * a.S, hi = min(a.n, lo + a.S);
    const int sid = ids[s];
    int64_t i = lo;
    if (a.kind == 2) {
      const int kb = 3 * a.seg_bits[s];
      B.get64(kb);
      pos += kb;
      i++;
    }
    for (; i < hi; i++) {
      const int o = B.ones7();
      const int pl = o < 7 ? o + 1 : 7;
      B.get(pl);
      const int w = c_vlcw[sid][o];
      B.get64(w);
      pos += pl + w;
      if (pos > a.total) {
        atomicCAS(a.status, 0u, (uint32_t)NBZG_TRUNCATED);
        return;
      }
    }
  }
  a.seg_off[a.nseg] = pos;
}

// one thread per segment: raw first key + VLC deltas (coordinates) or VLC
// magnitudes (velocities); writes the reconstructed floats
__global__ void __launch_bounds__(128) cpc_dec_kernel(KArgsD a, const uint8_t* ids) {
  __shared__ uint8_t sw[4][8];  // bucket widths (per-thread scheme: no divergent constant loads)
  if (threadIdx.x < 32) sw[threadIdx.x >> 3][threadIdx.x & 7] = c_vlcw[threadIdx.x >> 3][threadIdx.x & 7];
  __syncthreads();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nseg) return;
  const int64_t lo = s * a.S, hi = min(a.n, lo + a.S);
  const int sid = ids[s];
  if (sid > 3) {
    atomicCAS(a.status, 0u, (uint32_t)NBZG_BAD_STREAM);
    return;
  }
  const uint64_t b0 = a.seg_off[s], b1 = a.seg_off[s + 1];
  if (b1 > a.total || b0 > b1) {
    atomicCAS(a.status, 0u, (uint32_t)NBZG_TRUNCATED);
    return;
  }
  BitSrc B;
  B.init(a.pay + a.bits_at, b0);
  uint64_t pos = b0;
  if (a.kind == 2) {
    const int kb = 3 * a.seg_bits[s];
    uint64_t key = B.get64(kb);
    pos += kb;
    const int64_t m0 = a.minima[3 * s], m1 = a.minima[3 * s + 1], m2 = a.minima[3 * s + 2];
    for (int64_t i = lo; i < hi; i++) {
      if (i > lo) {
        const int o = B.ones7();
        const int pl = o < 7 ? o + 1 : 7;
        B.get(pl);
        const int w = sw[sid][o];
        key += B.get64(w);
        pos += pl + w;
      }
      if (a.out[0]) a.out[0][i] = (float)__dmul_rn((double)((int64_t)compact3_64(key >> 2) + m0), a.twob[0]);
      if (a.out[1]) a.out[1][i] = (float)__dmul_rn((double)((int64_t)compact3_64(key >> 1) + m1), a.twob[1]);
      if (a.out[2]) a.out[2][i] = (float)__dmul_rn((double)((int64_t)compact3_64(key) + m2), a.twob[2]);
    }
  } else {
    for (int64_t i = lo; i < hi; i++) {
      const int o = B.ones7();
      const int pl = o < 7 ? o + 1 : 7;
      B.get(pl);
      const int w = sw[sid][o];
      const uint64_t mm = B.get64(w);
      pos += pl + w;
      const int64_t h = (int64_t)(mm >> 1);
      const int64_t v = (mm & 1) ? -h - 1 : h;
      a.out[0][i] = (float)__dmul_rn((double)v, a.twob[0]);
    }
  }
  if (pos != b1) atomicCAS(a.status, 0u, (uint32_t)(pos > b1 ? NBZG_TRUNCATED : NBZG_BAD_STREAM));
}

// v2 streams: one thread per sub-block (kCSub values) from the segment
// index.  Coordinates take two passes: PHASE 0 sums each sub-block's key
// deltas (sub-block 0 also records the raw first key), PHASE 1 starts each
// sub-block from the raw key plus the sums before it and writes the floats.
// Velocities have no carried state: PHASE 1 only.  Every sub-block must end
// exactly where the next one starts.
template <int PHASE>
__global__ void __launch_bounds__(128) cpc_dec_sub_kernel(KArgsD a, const uint8_t* ids,
                                                          uint64_t* sums, uint64_t* k0) {
  __shared__ uint8_t sw[4][8];
  if (threadIdx.x < 32) sw[threadIdx.x >> 3][threadIdx.x & 7] = c_vlcw[threadIdx.x >> 3][threadIdx.x & 7];
  __syncthreads();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gt >= a.nseg * a.subs) return;
  const int64_t s = gt / a.subs, k = gt % a.subs;
  const int64_t seg_lo = s * a.S, seg_hi = min(a.n, seg_lo + a.S);
  const int64_t lo = seg_lo + k * kCSub;
  if (lo >= seg_hi) return;
  const int64_t hi = min(seg_hi, lo + kCSub);
  const int sid = ids[s];
  if (sid > 3) {
    atomicCAS(a.status, 0u, (uint32_t)NBZG_BAD_STREAM);
    return;
  }
  const uint8_t* subtab = a.pay + a.len - a.tr_bytes + 4 * a.nseg + 4 * s * (a.subs - 1);
  const uint64_t s0 = a.seg_off[s], s1 = a.seg_off[s + 1];
  const uint64_t b0 = s0 + (k == 0 ? 0 : ld_u32_le(subtab + 4 * (k - 1)));
  const uint64_t b1 = hi == seg_hi ? s1 : s0 + ld_u32_le(subtab + 4 * k);
  if (b1 > a.total || b0 > b1 || s1 > a.total) {
    atomicCAS(a.status, 0u, (uint32_t)NBZG_TRUNCATED);
    return;
  }
  BitSrc B;
  B.init(a.pay + a.bits_at, b0);
  uint64_t pos = b0;
  auto vlc = [&]() -> uint64_t {
    const int o = B.ones7();
    const int pl = o < 7 ? o + 1 : 7;
    B.get(pl);
    const int w = sw[sid][o];
    pos += pl + w;
    return B.get64(w);
  };
  const bool vec = (a.S & 3) == 0;  // sub-blocks start 16-byte aligned
  if (a.kind == 2) {
    const int kb = 3 * a.seg_bits[s];
    uint64_t key = 0;
    int64_t i = lo;
    if (k == 0) {
      key = B.get64(kb);
      pos += kb;
      i++;
    }
    if (PHASE == 0) {
      uint64_t sum = 0;
      for (; i < hi; i++) sum += vlc();
      sums[s * a.subs + k] = sum;
      if (k == 0) k0[s] = key;
    } else {
      if (k > 0) {
        key = k0[s];
        for (int64_t j = 0; j < k; j++) key += sums[s * a.subs + j];
      }
      const int64_t m0 = a.minima[3 * s], m1 = a.minima[3 * s + 1], m2 = a.minima[3 * s + 2];
      float ob[3][4];
      int nb = 0;
      auto out = [&](int64_t at) {
        const float v0 = (float)__dmul_rn((double)((int64_t)compact3_64(key >> 2) + m0), a.twob[0]);
        const float v1 = (float)__dmul_rn((double)((int64_t)compact3_64(key >> 1) + m1), a.twob[1]);
        const float v2 = (float)__dmul_rn((double)((int64_t)compact3_64(key) + m2), a.twob[2]);
        if (!vec) {
          if (a.out[0]) a.out[0][at] = v0;
          if (a.out[1]) a.out[1][at] = v1;
          if (a.out[2]) a.out[2][at] = v2;
          return;
        }
        ob[0][nb] = v0;
        ob[1][nb] = v1;
        ob[2][nb] = v2;
        if (++nb == 4) {
          for (int c = 0; c < 3; c++)
            if (a.out[c])
              *reinterpret_cast<float4*>(a.out[c] + at - 3) =
                  make_float4(ob[c][0], ob[c][1], ob[c][2], ob[c][3]);
          nb = 0;
        }
      };
      if (k == 0) out(lo);
      for (; i < hi; i++) {
        key += vlc();
        out(i);
      }
      for (int q = 0; q < nb; q++)
        for (int c = 0; c < 3; c++)
          if (a.out[c]) a.out[c][hi - nb + q] = ob[c][q];
    }
  } else {
    float ob[4];
    int nb = 0;
    for (int64_t i = lo; i < hi; i++) {
      const uint64_t mm = vlc();
      const int64_t h = (int64_t)(mm >> 1);
      const int64_t v = (mm & 1) ? -h - 1 : h;
      const float f = (float)__dmul_rn((double)v, a.twob[0]);
      if (!vec) {
        a.out[0][i] = f;
        continue;
      }
      ob[nb] = f;
      if (++nb == 4) {
        *reinterpret_cast<float4*>(a.out[0] + i - 3) = make_float4(ob[0], ob[1], ob[2], ob[3]);
        nb = 0;
      }
    }
    for (int q = 0; q < nb; q++) a.out[0][hi - nb + q] = ob[q];
  }
  if (pos != b1) atomicCAS(a.status, 0u, (uint32_t)(pos > b1 ? NBZG_TRUNCATED : NBZG_BAD_STREAM));
}

// correction lists (pipeline.py:240-260): one CTA per list, records applied
// in parallel after a serial walk of the list headers
__global__ void cpc_dec_corr_kernel(KArgsD a) {
  const int nl = a.kind == 2 ? 3 : 1;
  int64_t off = a.bits_at + (int64_t)((a.total + 7) / 8);
  const int64_t end = a.len - a.tr_bytes;  // the segment index follows the corrections
  for (int c = 0; c < nl; c++) {
    if (off + 4 > end) {
      if (threadIdx.x == 0) atomicCAS(a.status, 0u, (uint32_t)NBZG_TRUNCATED);
      return;
    }
    const uint8_t* h = a.pay + off;
    const uint32_t cnt = (uint32_t)h[0] | ((uint32_t)h[1] << 8) | ((uint32_t)h[2] << 16) |
                         ((uint32_t)h[3] << 24);
    off += 4;
    if (off + 12 * (int64_t)cnt > end) {
      if (threadIdx.x == 0) atomicCAS(a.status, 0u, (uint32_t)NBZG_TRUNCATED);
      return;
    }
    if ((int)blockIdx.x == c && a.out[c]) {
      for (uint32_t r = threadIdx.x; r < cnt; r += blockDim.x) {
        const uint8_t* d = a.pay + off + 12ull * r;
        uint64_t pos = 0;
        uint32_t u = 0;
        for (int b = 0; b < 8; b++) pos |= (uint64_t)d[b] << (8 * b);
        for (int b = 0; b < 4; b++) u |= (uint32_t)d[8 + b] << (8 * b);
        if (pos >= (uint64_t)a.n) atomicCAS(a.status, 0u, (uint32_t)NBZG_BAD_STREAM);
        else a.out[c][pos] = __uint_as_float(u);
      }
    }
    off += 12 * (int64_t)cnt;
  }
}

// ---------------------------------------------------------------- host side
static size_t r256(size_t b) { return (b + 255) & ~size_t(255); }
size_t cpc_ws(int64_t nseg) {
  // per stream (carved in this order, 256-byte aligned): seg_cost u64,
  // seg_off u64 (+1), ids u8, corr cnt 3 x u32, corr off 3 x u32 (+1)
  const size_t per = r256(8 * nseg) + r256(8 * (nseg + 1)) + r256(nseg) + r256(12 * nseg) +
                     r256(12 * (nseg + 1)) + r256(8 * (size_t)kCThreads * nseg);
  return 4 * per + 256;
}

static void carve(CArgs& a, void* ws, int64_t nseg) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  auto take = [&](size_t b) {
    uint8_t* r = p;
    p += r256(b);
    return r;
  };
  for (int s = 0; s < 4; s++) {
    a.st[s].seg_cost = reinterpret_cast<uint64_t*>(take(8 * nseg));
    a.st[s].seg_off = reinterpret_cast<uint64_t*>(take(8 * (nseg + 1)));
    a.st[s].seg_id = take(nseg);
    a.st[s].corr_cnt = reinterpret_cast<uint32_t*>(take(12 * nseg));
    a.st[s].corr_off = reinterpret_cast<uint32_t*>(take(12 * (nseg + 1)));
    a.st[s].run_bits = reinterpret_cast<uint32_t*>(take(8 * (size_t)kCThreads * nseg));
  }
}

static int fill_args(CArgs& a, const nbzg_cpc_args* g) {
  if (!g || !g->meta || !g->cmeta || g->n < 0 || g->segment_size < 1 ||
      g->segment_size > kTileMax || (g->mode != 1 && g->mode != 2))
    return NBZG_BAD_ARG;
  for (int f = 0; f < 6; f++) a.f[f] = g->fields[f];
  a.n = g->n;
  a.S = g->segment_size;
  a.tile = a.S < kTileMax ? (kTileMax / a.S) * a.S : a.S;
  a.nseg = (a.n + a.S - 1) / a.S;
  a.perm = g->perm;
  a.seg_bits = g->seg_bits;
  a.minima = g->seg_minima;
  a.meta = g->meta;
  a.nstreams = g->mode == 2 ? 4 : 1;
  a.cm = g->cmeta;
  a.arena = g->arena;
  if (g->workspace_bytes < cpc_ws(a.nseg)) return NBZG_BAD_ARG;
  carve(a, g->workspace, a.nseg);
  return NBZG_OK;
}

}  // namespace nbzg

using namespace nbzg;

extern "C" {

size_t nbzg_cpc_workspace_size(int64_t n, int64_t segment_size) {
  if (segment_size < 1) return 0;
  return cpc_ws((n + segment_size - 1) / segment_size);
}

int nbzg_cpc_plan(const nbzg_cpc_args* g, void* stream) {
  CArgs a;
  int rc = fill_args(a, g);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(g->cmeta, 0, sizeof(nbzg_cpc_meta), st);
  if (a.n == 0) return NBZG_OK;
  // the coordinate stream exists unless all three coordinates are constant
  // (pipeline.py:482); the plan still runs, the caller drops the stream
  count_launch();
  cpc_plan_kernel<<<dim3((unsigned)a.nseg, a.nstreams), kCThreads, 0, st>>>(a);
  count_launch();
  cpc_scan_kernel<<<a.nstreams, 1024, 0, st>>>(a);
  trace_mark("cpc_plan", st);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

int nbzg_cpc_pack(const nbzg_cpc_args* g, void* stream) {
  CArgs a;
  int rc = fill_args(a, g);
  if (rc) return rc;
  if (!a.arena) return NBZG_BAD_ARG;
  if (a.n == 0) return NBZG_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  trace_mark(nullptr, st);
  count_launch();
  cpc_pack_kernel<<<dim3((unsigned)a.nseg, a.nstreams), kCThreads, 0, st>>>(a);
  count_launch();
  cpc_frame_kernel<<<a.nstreams, 256, 0, st>>>(a);
  count_launch();
  cpc_corr_kernel<<<dim3((unsigned)a.nseg, a.nstreams), kCThreads, 0, st>>>(a);
  trace_mark("cpc_pack", st);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

size_t nbzg_cpc_decode_workspace_size(int64_t n, int64_t segment_size) {
  if (segment_size < 1) return 0;
  const size_t nseg = (size_t)((n + segment_size - 1) / segment_size);
  return 8 * (nseg + 1) + 8 * nseg * (size_t)cpc_subs(segment_size) + 8 * nseg + 256;
}

int nbzg_cpc_decode(const nbzg_cpc_decode_args* g, void* stream) {
  if (!g || g->n < 0 || g->segment_size < 1 || (g->kind != 1 && g->kind != 2) || !g->status)
    return NBZG_BAD_ARG;
  if (g->n == 0) return NBZG_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  KArgsD a;
  a.pay = g->payload;
  a.len = g->payload_len;
  a.n = g->n;
  a.S = g->segment_size;
  a.nseg = (a.n + a.S - 1) / a.S;
  a.kind = g->kind;
  a.seg_bits = g->seg_bits;
  a.minima = g->seg_minima;
  for (int c = 0; c < 3; c++) {
    a.twob[c] = 2.0 * g->bound[c];
    a.out[c] = g->out[c];
  }
  if (g->workspace_bytes < nbzg_cpc_decode_workspace_size(g->n, g->segment_size))
    return NBZG_BAD_ARG;
  a.seg_off = reinterpret_cast<uint64_t*>(g->workspace);
  a.status = g->status;
  a.bits_at = a.nseg + 8;
  // header fields the host already validated: ids, total bits (host passes)
  a.total = g->total_bits;
  a.subs = cpc_subs(a.S);
  a.tr_bytes = g->indexed ? 4 * a.nseg * a.subs : 0;
  const int64_t need = a.nseg + 8 + (int64_t)((a.total + 7) / 8) + a.tr_bytes;
  if (need > a.len) return NBZG_TRUNCATED;
  const uint8_t* ids = a.pay;
  trace_mark(nullptr, st);
  if (!g->indexed) {
    count_launch();
    cpc_dec_walk_kernel<<<1, 32, 0, st>>>(a, ids);
    count_launch();
    cpc_dec_kernel<<<(unsigned)((a.nseg + 127) / 128), 128, 0, st>>>(a, ids);
  } else {
    uint64_t* sums = a.seg_off + (a.nseg + 1);       // [nseg][subs]
    uint64_t* k0 = sums + a.nseg * a.subs;            // [nseg]
    const int64_t nt = a.nseg * a.subs;
    const unsigned grid = (unsigned)((nt + 127) / 128);
    count_launch();
    cpc_dec_offsets_kernel<<<1, 1024, 0, st>>>(a);
    if (a.kind == 2) {
      count_launch();
      cpc_dec_sub_kernel<0><<<grid, 128, 0, st>>>(a, ids, sums, k0);
    }
    count_launch();
    cpc_dec_sub_kernel<1><<<grid, 128, 0, st>>>(a, ids, sums, k0);
  }
  count_launch();
  cpc_dec_corr_kernel<<<a.kind == 2 ? 3 : 1, 256, 0, st>>>(a);
  trace_mark("cpc_decode", st);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // extern "C"
