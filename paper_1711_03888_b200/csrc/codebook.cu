// codebook.cu -- K4: on-device canonical Huffman codebook, bit-exact with
// encode.huffman_build (encode.py:199-219) -> K.huffman_lengths
// (_kernels.py:204-238) and HuffmanTable._build_tables (encode.py:123-152).
//
// One CTA per field:
//   A. compact the non-zero bins of the code histogram (ascending symbol);
//   B. order leaves by (count, symbol) -- identical to the reference's stable
//      argsort by count -- with a bitonic sort of (count << 16 | rank) keys;
//   C. the exact two-queue merge (leaf wins ties, _kernels.py:218,224) run by
//      one thread over shared memory, parents stored in place;
//   D. depths by parallel pointer jumping; lengths > 57 -> CODE_TOO_LONG;
//   E. canonical code words in (length, symbol) order and the u64 encode LUT
//      (len << 57) | word; payload sizes of the v2 stream.
// Leaf arrays live in shared memory for k <= 16384 symbols and in global
// scratch (L2-resident) above that.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kCBThreads = 1024;
constexpr int kCBSmemK = 16384;

struct CBArgs {
  const uint32_t* hist;
  int64_t nbins;
  uint32_t* sym;      // [6][nbins] ascending symbols
  uint8_t* len;       // [6][nbins] lengths by rank
  uint64_t* lut;      // [6][nbins] by symbol
  uint32_t* scratch;  // [6][5*nbins]
  nbzg_meta* meta;
  int64_t n;
  int64_t nchunks;
  int single_field;   // >= 0: only this field (parity hook), meta->f[0] receives
  uint32_t* twin;     // [6][kEncWin] encoder window table (may be null): code
                      // half+1-kEncWin/2+i -> MSB-aligned word | len (len <= 26, else 0)
  uint8_t* tlen8;     // [6][nbins] code length by symbol (may be null)
  int f0;             // first field of this launch (CTA b -> field f0 + b)
  int v1;             // payload sizes of a v1 SZ_FIELD stream (escapes after the bits)
};

NBZG_DEV void bitonic_sort_u64(uint64_t* a, int N) {
  for (int size = 2; size <= N; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = (lo & size) == 0;
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
}

// Stable LSD radix sort (4-bit digits) of the k leaves (w, idx) by weight,
// ping-pong between the A and B arrays, result in A.  Thread t owns the
// contiguous run [t RK, (t + 1) RK): it counts its digits in registers, eight
// u64 block scans (two digits each) turn the counts into digit-major /
// thread-major offsets, and the run is scattered in order -- stable, so equal
// counts stay in ascending symbol order like the reference's stable argsort.
NBZG_DEV void radix_sort_leaves(uint32_t* wA, uint16_t* iA, uint32_t* wB, uint16_t* iB, int k,
                                int bits, unsigned long long* scan_tmp) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int RK = (k + nt - 1) / nt;
  const int i0 = min(k, tid * RK), i1 = min(k, i0 + RK);
  int passes = max(2, (bits + 3) / 4);
  passes += passes & 1;  // even: the result lands in A
  for (int p = 0; p < passes; p++) {
    const uint32_t* sw = (p & 1) ? wB : wA;
    const uint16_t* si = (p & 1) ? iB : iA;
    uint32_t* dw = (p & 1) ? wA : wB;
    uint16_t* di = (p & 1) ? iA : iB;
    const int sh = 4 * p;
    uint32_t c[16];
#pragma unroll
    for (int d = 0; d < 16; d++) c[d] = 0;
    for (int i = i0; i < i1; i++) {
      const uint32_t d = sh < 32 ? (sw[i] >> sh) & 15u : 0u;
#pragma unroll
      for (int dd = 0; dd < 16; dd++) c[dd] += d == (uint32_t)dd ? 1u : 0u;
    }
    uint32_t base[16], run = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      unsigned long long tot;
      const unsigned long long ex = block_excl_scan<unsigned long long>(
          (unsigned long long)c[2 * q] | ((unsigned long long)c[2 * q + 1] << 32), scan_tmp, &tot);
      base[2 * q] = run + (uint32_t)ex;
      run += (uint32_t)tot;
      base[2 * q + 1] = run + (uint32_t)(ex >> 32);
      run += (uint32_t)(tot >> 32);
    }
    for (int i = i0; i < i1; i++) {
      const uint32_t w = sw[i];
      const uint16_t id = si[i];
      const uint32_t d = sh < 32 ? (w >> sh) & 15u : 0u;
      uint32_t pos = 0;
#pragma unroll
      for (int dd = 0; dd < 16; dd++) {
        if (d == (uint32_t)dd) {
          pos = base[dd];
          base[dd]++;
        }
      }
      dw[pos] = w;
      di[pos] = id;
    }
    __syncthreads();
  }
}

// The same sort for leaves in global scratch (k > 16384): elements are read
// in order, 1024 per round and coalesced; MATCH.ANY ranks equal digits inside
// a warp, u16 counters per (round, warp, digit) in shared memory are scanned
// digit-major, and the second sweep scatters.  cnt: R * 32 * 16 u16.
NBZG_DEV void radix_sort_leaves_striped(uint32_t* wA, uint16_t* iA, uint32_t* wB, uint16_t* iB, int k,
                                        int bits, uint16_t* cnt, uint32_t* scan_tmp) {
  const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (k + nt - 1) / nt;
  const int RW = R * 32;       // (round, warp) slots; counters digit-major: cnt[d * RW + r * 32 + warp]
  const int C = RW * 16;
  int passes = max(2, (bits + 3) / 4);
  passes += passes & 1;
  for (int p = 0; p < passes; p++) {
    const uint32_t* sw = (p & 1) ? wB : wA;
    const uint16_t* si = (p & 1) ? iB : iA;
    uint32_t* dw = (p & 1) ? wA : wB;
    uint16_t* di = (p & 1) ? iA : iB;
    const int sh = 4 * p;
    for (int r0 = 0; r0 < R; r0 += 4) {  // four rounds' loads in flight
      uint32_t wv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int i = (r0 + u) * nt + tid;
        wv[u] = (r0 + u < R && i < k) ? sw[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int r = r0 + u;
        if (r >= R) break;  // uniform
        const bool valid = r * nt + tid < k;
        const uint32_t d = valid ? (sh < 32 ? (wv[u] >> sh) & 15u : 0u) : 16u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint16_t* c = cnt + r * 32 + warp;
        if (lane < 16) c[lane * RW] = 0;
        __syncwarp();
        if (valid && (peers & lanemask_lt()) == 0) c[d * RW] = (uint16_t)__popc(peers);
      }
    }
    __syncthreads();
    {  // exclusive scan of the digit-major counters
      const int per = (C + nt - 1) / nt;
      const int q0 = min(C, tid * per), q1 = min(C, q0 + per);
      uint32_t sum = 0;
      for (int q = q0; q < q1; q++) sum += cnt[q];
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(sum, scan_tmp, &tot);
      for (int q = q0; q < q1; q++) {
        const uint32_t v = cnt[q];
        cnt[q] = (uint16_t)ex;
        ex += v;
      }
    }
    __syncthreads();
    for (int r0 = 0; r0 < R; r0 += 4) {
      uint32_t wv[4];
      uint16_t iv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int i = (r0 + u) * nt + tid;
        const bool ok = r0 + u < R && i < k;
        wv[u] = ok ? sw[i] : 0u;
        iv[u] = ok ? si[i] : (uint16_t)0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int r = r0 + u;
        if (r >= R) break;  // uniform
        const bool valid = r * nt + tid < k;
        const uint32_t d = valid ? (sh < 32 ? (wv[u] >> sh) & 15u : 0u) : 16u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid) {
          const uint32_t pos = (uint32_t)cnt[d * RW + r * 32 + warp] + __popc(peers & lanemask_lt());
          dw[pos] = wv[u];
          di[pos] = iv[u];
        }
      }
    }
    __syncthreads();
  }
}

// Two-queue Huffman (_kernels.py:213-232) over ascending leaf weights
// Lw[0..k), run by the whole CTA in batched rounds.  The reference picks,
// 2 (k - 1) times, the smaller head of the leaf queue and of the FIFO queue of
// internal nodes (the leaf on ties) and joins consecutive picks in pairs.
// Internal nodes are created in non-decreasing weight order, so the pick
// sequence is the stable merge (leaves first on ties) of the leaves with the
// node queue, and a node created now is never smaller than a node that already
// exists.  One round therefore settles, in parallel, every pick up to the last
// EXISTING node: with wmax that node's weight, the cL leaves of weight <= wmax
// and the e live nodes merge by rank (one binary search per element: a leaf's
// rank = its index + #nodes < it, a node's = its index + #leaves <= it), the
// pick left unpaired by the previous round goes in front, consecutive
// positions pair up into new nodes (weights by atomicAdd) and an odd last
// pick -- always the node of weight wmax -- is carried over.  Every live node
// is consumed in the round after its creation, so the number of rounds is at
// most about twice the tree height (<= 57, else CODE_TOO_LONG), whatever k.
// Outputs: PL[i] / PI[j] = internal index of leaf i's / node j's parent
// (root k-2: 0xffff).  Iw: k u32 of scratch (node weights).
struct TQState {
  int leaf, node, nI;      // next leaf, first live node, nodes created
  int carry;               // 0 none, 1 a leaf, 2 a node: picked, not yet paired
  int carry_idx;
  uint32_t carry_w;
  int ncarry_idx;          // the node left over by this round (or -1)
};

NBZG_DEV int tq_upper(const uint32_t* a, int n, uint32_t w) {  // #elements <= w (a ascending)
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= w) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
NBZG_DEV int tq_lower(const uint32_t* a, int n, uint32_t w) {  // #elements < w
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < w) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

NBZG_DEV void two_queue(const uint32_t* Lw, uint32_t* Iw, uint16_t* PL, uint16_t* PI, int k,
                        TQState* st) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < k; i += nt) Iw[i] = 0;
  if (tid == 0) {
    st->leaf = 0;
    st->node = 0;
    st->nI = 0;
    st->carry = 0;
    st->ncarry_idx = -1;
  }
  __syncthreads();
  while (true) {
    const int leaf = st->leaf, node = st->node, nI = st->nI, carry = st->carry;
    if (nI >= k - 1) break;
    const int e = nI - node;
    if (e == 0) {
      // no live node: the carried pick (if any) and the next leaves make one pair
      if (tid == 0) {
        uint32_t sum = 0;
        int lf = leaf;
        if (carry == 1) PL[st->carry_idx] = (uint16_t)nI, sum += st->carry_w;
        else if (carry == 2) PI[st->carry_idx] = (uint16_t)nI, sum += st->carry_w;
        for (int c = carry ? 1 : 0; c < 2; c++) {
          sum += Lw[lf];
          PL[lf] = (uint16_t)nI;
          lf++;
        }
        Iw[nI] = sum;
        st->leaf = lf;
        st->nI = nI + 1;
        st->carry = 0;
      }
      __syncthreads();
      continue;
    }
    const uint32_t wmax = Iw[nI - 1];
    const int cL = tq_upper(Lw + leaf, k - leaf, wmax);
    const int T = cL + e, c = carry ? 1 : 0;
    const bool odd = (T + c) & 1;
    if (tid == 0 && carry) {  // the carried pick opens the sequence: position 0
      if (carry == 1) PL[st->carry_idx] = (uint16_t)nI;
      else PI[st->carry_idx] = (uint16_t)nI;
      atomicAdd(&Iw[nI], st->carry_w);
    }
    for (int t = tid; t < T; t += nt) {
      if (t < cL) {
        const uint32_t w = Lw[leaf + t];
        const int pos = t + tq_lower(Iw + node, e, w) + c;
        PL[leaf + t] = (uint16_t)(nI + (pos >> 1));
        atomicAdd(&Iw[nI + (pos >> 1)], w);
      } else {
        const int j = t - cL;
        const uint32_t w = Iw[node + j];
        const int pos = j + tq_upper(Lw + leaf, cL, w) + c;
        if (odd && pos == T + c - 1) {
          st->ncarry_idx = node + j;  // (one thread: the last pick is the last node)
        } else {
          PI[node + j] = (uint16_t)(nI + (pos >> 1));
          atomicAdd(&Iw[nI + (pos >> 1)], w);
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      st->leaf = leaf + cL;
      st->node = nI;
      st->nI = nI + ((T + c) >> 1);
      if (odd) {
        st->carry = 2;
        st->carry_idx = st->ncarry_idx;
        st->carry_w = Iw[st->ncarry_idx];
      } else {
        st->carry = 0;
      }
    }
    __syncthreads();
  }
  if (tid == 0) PI[k - 2] = 0xffff;
  __syncthreads();
}

// Depth of every internal node (root = ni-1, parent index in P[j], parent >
// child): level-synchronous passes until no node changes (<= 58 passes).
NBZG_DEV void node_depths(const uint16_t* P, uint8_t* D, int ni) {
  for (int j = threadIdx.x; j < ni; j += blockDim.x) D[j] = (j == ni - 1) ? 0 : 0xff;
  __syncthreads();
  while (true) {
    int changed = 0;
    for (int j = threadIdx.x; j < ni; j += blockDim.x) {
      if (D[j] == 0xff) {
        uint8_t dp = D[P[j]];
        if (dp != 0xff) {
          D[j] = (uint8_t)min(dp + 1, 254);
          changed = 1;
        }
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
}

#ifdef NBZG_CB_PROF  // timing experiment: per-phase clocks of every CTA, printed at exit
#define CB_T(i) do { __syncthreads(); if (threadIdx.x == 0) { long long _c = clock64(); cb_t[i] = _c - cb_last; cb_last = _c; } } while (0)
#else
#define CB_T(i) do { } while (0)
#endif

__global__ void __launch_bounds__(kCBThreads) codebook_kernel(CBArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
#ifdef NBZG_CB_PROF
  long long cb_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cb_last = clock64();
#endif
  __shared__ uint32_t scan_u32[33];
  __shared__ unsigned long long scan_u64[33];
  __shared__ uint32_t s_cbl[64];
  __shared__ uint64_t s_fc[64];
  __shared__ uint32_t s_max, s_min;
  const int field = a.single_field >= 0 ? a.single_field : a.f0 + (int)blockIdx.x;
  const int mslot = a.single_field >= 0 ? 0 : field;
  nbzg_field_meta& fm = a.meta->f[mslot];
  if (a.single_field < 0 && (fm.is_const || a.n == 0)) return;
  const uint32_t* hist = a.hist + (a.single_field >= 0 ? 0 : field * a.nbins);
  uint32_t* sym = a.sym + field * a.nbins;
  uint8_t* lenr = a.len + field * a.nbins;
  uint64_t* lut = a.lut + field * a.nbins;
  uint32_t* scr = a.scratch + field * 5 * a.nbins;
  const int tid = threadIdx.x;
  const int64_t nb = a.nbins;

  // ---- A. compact non-zero bins, ascending symbol: warp w owns the bins
  // [w * per, (w + 1) * per), read 32 at a time (coalesced) and ranked by
  // ballot; a block scan of the warp totals gives each warp's output base
  uint32_t* cnt = scr;  // compact counts (global scratch, k entries)
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t per = ((nb + kCBThreads - 1) / kCBThreads) * 32;  // bins per warp (multiple of 32)
  const int64_t b0 = (int64_t)warp * per, b1 = min(nb, b0 + per);
  uint32_t mine = 0;
#pragma unroll 8
  for (int64_t bb = b0; bb < b1; bb += 32) {
    const int64_t bin = bb + lane;
    const uint32_t c = bin < b1 ? hist[bin] : 0u;
    mine += __popc(__ballot_sync(0xffffffffu, c != 0));
  }
  uint32_t ktot;
  uint32_t off = block_excl_scan<uint32_t>(lane == 0 ? mine : 0u, scan_u32, &ktot);
  off = __shfl_sync(0xffffffffu, off, 0);
#pragma unroll 8
  for (int64_t bb = b0; bb < b1; bb += 32) {
    const int64_t bin = bb + lane;
    const uint32_t c = bin < b1 ? hist[bin] : 0u;
    const uint32_t m = __ballot_sync(0xffffffffu, c != 0);
    if (c) {
      const uint32_t o = off + __popc(m & ((1u << lane) - 1u));
      sym[o] = (uint32_t)bin;
      cnt[o] = c;
    }
    off += __popc(m);
  }
  const int k = (int)ktot;
  CB_T(0);  // compaction
  if (tid == 0) {
    fm.k = (uint32_t)k;
    fm.n_esc = hist[0];
  }
  __syncthreads();
  if (k == 0) return;
  if (k > 65536) {  // ranks are 16-bit (only a v1 alphabet of 2^16 + 1 symbols can get here)
    if (tid == 0) atomicCAS(&a.meta->status, 0u, (uint32_t)NBZG_UNSUPPORTED);
    return;
  }

  // memory for the sort and the merge: shared for k <= 16384, else global
  // scratch (L2-resident).  Layout (N = pow2 >= k), byte offsets:
  //   sort   A: L u32 @8N, order u16 @12N     B: tmp u32 @0, tmp u16 @4N
  //   merge  Iw u32 @0, PL u16 @4N, PI u16 @6N, L @8N
  // Depths and the canonical-code pass then run out of shared memory in both
  // cases: D u8[k] and a copy of the lengths by rank (s_len) overlay dead
  // arrays; the large-k case first copies PI into the (otherwise unused)
  // shared memory.
  const bool small = k <= kCBSmemK;
  uint8_t* base = small ? smem : reinterpret_cast<uint8_t*>(scr + a.nbins);  // after cnt
  int N = 1;
  while (N < k) N <<= 1;
  uint32_t* L = reinterpret_cast<uint32_t*>(base + 8 * (size_t)N);
  uint16_t* order = reinterpret_cast<uint16_t*>(base + 12 * (size_t)N);
  uint32_t* Iw = reinterpret_cast<uint32_t*>(base);
  uint16_t* PL = reinterpret_cast<uint16_t*>(base + 4 * (size_t)N);
  uint16_t* PI = reinterpret_cast<uint16_t*>(base + 6 * (size_t)N);
  uint16_t* PIs = small ? PI : reinterpret_cast<uint16_t*>(smem);  // parents, shared
  uint8_t* D = small ? smem : smem + 2 * (size_t)N;                 // node depths, shared
  uint8_t* s_len = small ? smem + (size_t)N : smem;                 // lengths by rank, shared
  __shared__ TQState tq_state;
  __shared__ uint32_t s_wmax;

  if (k == 1) {
    if (tid == 0) lenr[0] = 1, s_len[0] = 1;  // _kernels.py:207-209
  } else {
    // ---- B. sort leaves by (count, rank) = the reference's stable argsort by
    // count.  Measured (C3, cycles): bitonic on (count << 16 | rank) keys 16 K
    // at N = 512, 146 K at N = 8192; the stable radix sort 55 K and 102 K.
    // Radix for N >= 8192 (per-thread runs in shared memory; the striped
    // variant for the global-scratch case), bitonic below.
    if (N >= 8192) {
      if (tid == 0) s_wmax = 0;
      __syncthreads();
      uint32_t mx = 0;
      for (int i = tid; i < k; i += kCBThreads) {
        const uint32_t c = cnt[i];
        L[i] = c;
        order[i] = (uint16_t)i;
        mx = max(mx, c);
      }
      atomicMax(&s_wmax, mx);
      __syncthreads();
      if (!small)
        radix_sort_leaves_striped(L, order, Iw, PL, k, 32 - __clz(s_wmax),
                                  reinterpret_cast<uint16_t*>(smem), scan_u32);
      else
      radix_sort_leaves(L, order, Iw, PL, k, 32 - __clz(s_wmax), scan_u64);
    } else {
      uint64_t* keys = reinterpret_cast<uint64_t*>(base);
      for (int i = tid; i < N; i += kCBThreads)
        keys[i] = i < k ? (((uint64_t)cnt[i] << 16) | (uint64_t)i) : ~0ull;
      __syncthreads();
      bitonic_sort_u64(keys, N);
      for (int i = tid; i < k; i += kCBThreads) {
        uint64_t kv = keys[i];
        L[i] = (uint32_t)(kv >> 16);
        order[i] = (uint16_t)(kv & 0xffff);
      }
      __syncthreads();
    }
    CB_T(1);  // sort
    // ---- C. two-queue merge (exact; batched rounds, whole CTA)
    two_queue(L, Iw, PL, PI, k, &tq_state);
    CB_T(2);  // merge
    // ---- D. depths (shared memory)
    if (!small) {
      for (int i = tid; i < k - 1; i += kCBThreads) PIs[i] = PI[i];
      __syncthreads();
    }
    node_depths(PIs, D, k - 1);
    // leaf depth = depth(parent) + 1, scattered to ascending-symbol rank
    // (s_len overlays only arrays that are dead by now: Iw, or the PI copy)
    for (int i = tid; i < k; i += kCBThreads) {
      const uint32_t d = (uint32_t)D[PL[i]] + 1;
      const uint8_t d8 = (uint8_t)min(d, 255u);
      lenr[order[i]] = d8;
      s_len[order[i]] = d8;
    }
  }
  __syncthreads();
  CB_T(3);  // depths

  // ---- E. canonical codes (encode.py:123-152): a symbol's code is
  // first_code[len] + its rank among the symbols of that length, ascending
  // symbol.  Warp w owns the symbols [w B, (w + 1) B), 32 consecutive ones per
  // round; MATCH.ANY groups the lanes of equal length, so a round costs one
  // counter update per distinct length.  Pass 1 counts per (warp, length), 64
  // threads scan the warps, pass 2 replays the rounds with the running
  // counters as ranks.
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem + 131072);  // [32 warps][64 lengths]
  if (tid == 0) {
    s_max = 0;
    s_min = 255;
  }
  for (int i = tid; i < 32 * 64; i += kCBThreads) wcnt[i] = 0;
  __syncthreads();
  const int RB = (k + kCBThreads - 1) / kCBThreads;  // rounds per warp
  const int wbase = warp * RB * 32;
  {
    uint32_t lmax = 0, lmin = 255;
    for (int r = 0; r < RB; r++) {
      const int i = wbase + r * 32 + lane;
      const bool valid = i < k;
      const uint32_t l = valid ? (uint32_t)s_len[i] : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      if (valid) {
        lmax = max(lmax, l);
        lmin = min(lmin, l);
        if ((peers & lanemask_lt()) == 0) wcnt[warp * 64 + min(l, 63u)] += __popc(peers);
      }
      __syncwarp();
    }
    atomicMax(&s_max, lmax);
    atomicMin(&s_min, lmin);
  }
  __syncthreads();
  if (tid < 64) {  // exclusive prefix over the warps, per length
    uint32_t run = 0;
    for (int w = 0; w < 32; w++) {
      const uint32_t c = wcnt[w * 64 + tid];
      wcnt[w * 64 + tid] = run;
      run += c;
    }
    s_cbl[tid] = run;
  }
  __syncthreads();
  const int max_len = (int)s_max;
  if (max_len > kMaxCodeLen) {
    if (tid == 0) atomicCAS(&a.meta->status, 0u, (uint32_t)NBZG_CODE_TOO_LONG);
    return;
  }
  if (tid == 0) {
    uint64_t code = 0;
    for (int l = 1; l <= max_len; l++) {
      s_fc[l] = code;
      code = (code + s_cbl[l]) << 1;
    }
    fm.min_len = s_min;
    fm.max_len = s_max;
  }
  __syncthreads();
  for (int r = 0; r < RB; r++) {
    const int i = wbase + r * 32 + lane;
    const bool valid = i < k;
    const uint32_t l = valid ? (uint32_t)s_len[i] : 0x100u;
    const uint32_t peers = __match_any_sync(0xffffffffu, l);
    const uint32_t lt = peers & lanemask_lt();
    uint32_t rank = 0;
    if (valid) rank = wcnt[warp * 64 + l] + __popc(lt);
    __syncwarp();
    if (valid && lt == 0) wcnt[warp * 64 + l] += __popc(peers);
    __syncwarp();
    if (valid) {
      const uint32_t sy = sym[i];
      const uint64_t word = s_fc[l] + rank;
      lut[sy] = ((uint64_t)l << 57) | word;
      if (a.tlen8) a.tlen8[field * a.nbins + sy] = (uint8_t)l;
      if (a.twin) {
        const uint32_t wi = sy - (uint32_t)(a.nbins / 2 + 1 - kEncWin / 2);
        if (wi < (uint32_t)kEncWin)
          // MSB-aligned code word | length (l <= 26 leaves the low 6 bits free)
          a.twin[field * kEncWin + wi] = l <= 26 ? ((uint32_t)word << (32 - l)) | (uint32_t)l : 0u;
      }
    }
  }
  CB_T(4);  // canonical codes + tables
  // ---- sizes: total bits = sum count * len
  unsigned long long tb = 0;
  for (int i = tid; i < k; i += kCBThreads) tb += (unsigned long long)cnt[i] * s_len[i];
  unsigned long long tbits;
  block_excl_scan<unsigned long long>(tb, scan_u64, &tbits);
  if (tid == 0) {
    const uint64_t table_end = 8 + 5 * (uint64_t)k;
    if (a.v1) {  // pipeline.py:188-200: table | u64 bits | bytes | f32 escapes
      fm.total_bits = tbits;
      fm.index_off = 0;
      fm.bits_off = table_end + 8;
      fm.esc_off = fm.bits_off + (tbits + 7) / 8;
      fm.payload_len = fm.esc_off + 4 * fm.n_esc;
    } else {
      tbits += 32ull * fm.n_esc;  // v2: escape values ride inline in the bitstream
      fm.total_bits = tbits;
      fm.index_off = table_end + 8;
      fm.bits_off = (fm.index_off + 4 * (uint64_t)a.nchunks + 3) & ~3ull;
      fm.esc_off = fm.bits_off + 4 * ((tbits + 31) / 32);  // == payload end (no escape area)
      fm.payload_len = fm.esc_off;
    }
  }
#ifdef NBZG_CB_PROF
  CB_T(5);
  if (tid == 0)
    printf("codebook field %d k %d cycles: compact %lld sort %lld merge %lld depths %lld codes %lld sizes %lld\n",
           field, k, cb_t[0], cb_t[1], cb_t[2], cb_t[3], cb_t[4], cb_t[5]);
#endif
}

int launch_codebook_impl(const uint32_t* hist, int64_t nbins, uint32_t* sym, uint8_t* len,
                         uint64_t* lut, uint32_t* scratch, nbzg_meta* meta, int64_t n,
                         int64_t nchunks, int single_field, cudaStream_t st,
                         uint32_t* twin, uint8_t* tlen8, int f0, int nf, int v1) {
  CBArgs a{hist, nbins, sym, len, lut, scratch, meta, n, nchunks, single_field, twin, tlen8, f0,
           v1};
  size_t sm = 14 * (size_t)kCBSmemK;  // keys u64 | L u32 | order u16
  smem_attr((const void*)codebook_kernel, (int)sm);
  count_launch();
  codebook_kernel<<<single_field >= 0 ? 1 : nf, kCBThreads, sm, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

int launch_codebook(const Plan& p, cudaStream_t st, int f0, int nf) {
  if (p.n == 0) return NBZG_OK;
  return launch_codebook_impl(p.hist, p.nbins, p.cb_sym, p.cb_len, p.lut, p.cb_scratch, p.meta,
                              p.n, p.nchunks, -1, st, p.fmt == 1 ? nullptr : p.enc_win,
                              p.enc_len8, f0, nf, p.fmt == 1 ? 1 : 0);
}

// ---- parity hook: K.huffman_lengths on sorted counts (one CTA)
__global__ void __launch_bounds__(kCBThreads) huffman_lengths_kernel(const uint32_t* counts,
                                                                     int k, uint8_t* lengths,
                                                                     uint32_t* scr,
                                                                     uint32_t* status) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ TQState tq_state;
  const bool small = k <= kCBSmemK;
  int N = 1;
  while (N < k) N <<= 1;
  uint8_t* base = small ? smem : reinterpret_cast<uint8_t*>(scr);
  uint32_t* Iw = reinterpret_cast<uint32_t*>(base);
  uint16_t* PL = reinterpret_cast<uint16_t*>(base + 4 * (size_t)N);
  uint16_t* PI = reinterpret_cast<uint16_t*>(base + 6 * (size_t)N);
  uint8_t* D = base;
  uint32_t* L = reinterpret_cast<uint32_t*>(base + 8 * (size_t)N);
  const int tid = threadIdx.x;
  if (k == 1) {
    if (tid == 0) lengths[0] = 1;
    return;
  }
  for (int i = tid; i < k; i += kCBThreads) L[i] = counts[i];
  __syncthreads();
  two_queue(L, Iw, PL, PI, k, &tq_state);
  node_depths(PI, D, k - 1);
  for (int i = tid; i < k; i += kCBThreads) {
    uint32_t d = (uint32_t)D[PL[i]] + 1;
    lengths[i] = (uint8_t)min(d, 255u);
    if (d > kMaxCodeLen) atomicCAS(status, 0u, (uint32_t)NBZG_CODE_TOO_LONG);
  }
}

int launch_huffman_lengths(const uint32_t* counts, int64_t k, uint8_t* lengths, uint32_t* scr,
                           uint32_t* status, cudaStream_t st) {
  if (k <= 0 || k > 65536) return NBZG_BAD_ARG;
  size_t sm = 12 * (size_t)kCBSmemK;
  smem_attr((const void*)huffman_lengths_kernel, (int)sm);
  count_launch();
  huffman_lengths_kernel<<<1, kCBThreads, sm, st>>>(counts, (int)k, lengths, scr, status);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// ---- K5: payload layout (offsets of the non-constant fields, field order)
// fields f0 .. f1-1, placed after the fields before f0 (whose layout ran first)
__global__ void layout_kernel(nbzg_meta* meta, int64_t n, int f0, int f1, int first) {
  if (threadIdx.x != 0) return;
  uint64_t off = first ? 0 : meta->arena_used;
  for (int f = f0; f < f1; f++) {
    nbzg_field_meta& m = meta->f[f];
    m.payload_off = off;
    if (m.is_const || n == 0) {
      m.payload_len = 0;
      continue;
    }
    off += m.payload_len;
  }
  meta->arena_used = off;
}

int launch_layout(const Plan& p, cudaStream_t st, int f0, int nf, bool first) {
  count_launch();
  layout_kernel<<<1, 32, 0, st>>>(p.meta, p.n, f0, f0 + nf, first ? 1 : 0);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
