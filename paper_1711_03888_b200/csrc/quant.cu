// quant.cu -- K3: permutation gather + dual-quant + code histogram.
//
// Replaces the gather (pipeline.py:466), quantize.quantize_field ->
// K.sz_quantize (_kernels.py:150-184) and np.bincount (pipeline.py:191).
// The reference's reconstruct-and-predict chain is sequential; this kernel
// computes the parallel "pre-quantise then difference" restatement
// (oracle/nbz_oracle.c orc_dq_quantize):
//     k_i = rint(x_i / 2b) (lattice index), q_i = k_i - k_{i-1} (k_{-1} = 0
//     at every 16384-symbol chunk start, so v2 chunks decode independently),
//     code_i = q_i + half + 1 if q_i in [-half, half-2] and
//              |x_i - f32(k_i * 2b)| <= b, else 0 (escape).
//
// Persistent CTAs, each owning ONE field and a contiguous range of tiles, so
// a CTA keeps one shared-memory histogram window for its whole range and
// flushes it once (out-of-window codes go straight to global atomics).
// Tiles (field values + the tile-local permutation) are staged into shared
// memory with TMA bulk copies (cp.async.bulk + mbarrier), double buffered,
// so the next tile streams in while the current one is gathered.
#include <cstdlib>

#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kQThreads = 1024;
constexpr int kQPer = kTileMax / kQThreads;  // 16 positions per thread
constexpr uint32_t kQFarBudget = 65536u;  // far codes a CTA counts with global atomics (NBZG_Q_FAR_BUDGET overrides: tests)
constexpr int kQWin = 4096;                  // histogram window (bins)

struct QArgs {
  const float* f[6];
  int64_t n, tile, ntiles;
  const uint16_t* perm;  // tile-local source index per sorted position (null: identity)
  const nbzg_meta* meta;
  int half;
  uint16_t* codes;  // 6 x code_stride
  int64_t code_stride;
  uint32_t* hist;  // 6 x nbins
  int64_t nbins;
  int groups;
  int use_tma;
  int f0, nf;  // field group: fields f0 .. f0+nf-1
  uint32_t far_budget;  // far codes a CTA counts with global atomics before deferring
};

NBZG_DEV uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
NBZG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
NBZG_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
NBZG_DEV bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
NBZG_DEV void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
NBZG_DEV uint32_t ld_shared_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
NBZG_DEV float ld_shared_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
NBZG_DEV void red_shared_add1(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}
NBZG_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// dual-quant lattice index, clamped (orc_dq_quantize: dq_k)
NBZG_DEV int64_t dq_index(float x, const nbzg_field_meta& m, bool& fast) {
  double k = lattice_index<false>(x, m.inv32, m.inv, m.twob, fast);
  if (!fast) k = fmin(fmax(k, -kDqKmax), kDqKmax);
  return (int64_t)k;
}

// Same result as dq_index, FP32/int32 on the fast path: adding 1.5*2^23
// rounds t to the nearest integer (ties to even, = rintf) for |t| < 2^22 and
// leaves it in the low mantissa bits, so no conversion instructions are
// needed; the FP64 slow path is taken only when the fast test fails.
NBZG_DEV int64_t dq_index_fast(float x, float inv32, const nbzg_field_meta& m, bool& fast) {
  const float t = x * inv32;
  const float r = t + 12582912.0f;
  const float kf = r - 12582912.0f;
  const float d = fabsf(t - kf);
  const float thr = fabsf(t) * 9.5367431640625e-07f + 9.5367431640625e-07f;
  fast = (0.5f - d) > thr && fabsf(t) < 4194304.0f;
  if (fast) return (int64_t)(__float_as_int(r) - 0x4B400000);
  double k = rint(__dmul_rn((double)x, m.inv));
  k = fmin(fmax(k, -kDqKmax), kDqKmax);
  return (int64_t)k;
}

template <bool SORTED>
__global__ void __launch_bounds__(kQThreads, 1) quantize_kernel(QArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* xbuf = reinterpret_cast<float*>(smem);                      // [2][16384]
  uint16_t* pbuf = reinterpret_cast<uint16_t*>(xbuf + 2 * kTileMax);  // [2][16384]
  uint32_t* hw = reinterpret_cast<uint32_t*>(pbuf + 2 * kTileMax);    // [kQWin + 1]: window + escapes
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int64_t s_carry2[2];
  __shared__ uint32_t s_far;      // far codes this CTA sent to global atomics so far
  __shared__ uint32_t s_budget;   // next count at which the far-code rate is examined
  __shared__ long long s_dstart;  // first deferred tile (te: none)

  const int field = a.f0 + (int)(blockIdx.x % a.nf);
  const int g = (int)(blockIdx.x / a.nf);
  const nbzg_field_meta& fm = a.meta->f[field];
  if (fm.is_const || a.n == 0 || a.meta->status) return;  // e.g. BOUND_TOO_SMALL in K2
  const int64_t tb = (a.ntiles * g) / a.groups, te = (a.ntiles * (g + 1)) / a.groups;
  if (tb >= te) return;
  const float* __restrict__ x = a.f[field];
  uint16_t* __restrict__ codes = a.codes + field * a.code_stride;
  uint32_t* __restrict__ hist = a.hist + field * a.nbins;
  const int half = a.half;
  const int wlo = half + 1 - kQWin / 2;
  const double b = fm.bound, twob = fm.twob;
  const float inv32 = fm.inv32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // Field-wide FP32 margin.  t32 = fl(x * fl(inv)) is within |t| 2^-23 (1 +
  // 2^-23) of the FP64 product x * inv, and |t| <= tmax for every value, so
  // |t32 - rint(t32)| < cmargin = 0.5 - (tmax 2^-22 + 2^-20) puts the FP64
  // product on the same side of every half-integer: rint agrees, and the
  // remaining distance to the cell edge (> |x| 2^-22) exceeds the f32
  // rounding of k * 2b (<= |x| 2^-24), so the reconstruction check holds.
  // `small` = every |t| < 2^22 (the 32-bit chain applies).
  const float tmax = fmaxf(fabsf(fm.lo), fabsf(fm.hi)) * inv32;
  const bool small = tmax < 4194304.0f;
  const float cmargin = 0.5f - __fmaf_ru(tmax, 2.384185791015625e-07f, 9.5367431640625e-07f);
  const double inv = fm.inv;

  for (int i = tid; i <= kQWin; i += kQThreads) hw[i] = 0;
  // Codes outside the shared window go to global atomics -- fine while they
  // are rare.  Once a CTA has sent far_budget (kQFarBudget) of them at a rate of
  // at least one code in 16 (large alphabets at tight bounds: L2 atomic
  // throughput then bounds the kernel), the far codes of its remaining tiles
  // are deferred: after its last tile the CTA counts
  // them from the stored u16 codes in a 32768-bin shared histogram (the tile
  // buffers are free by then), one half of the code range at a time.  The
  // switch costs nothing per tile: the warp whose count crosses the budget
  // publishes the next tile as the first deferred one.
  if (tid == 0) s_far = 0, s_budget = a.far_budget, s_dstart = te;
  if (tid == 0) {
    // k carried into the range: k of the last sorted element of tile tb-1
    int64_t kc = 0;
    if (tb > 0) {
      int64_t p = tb * a.tile - 1;
      int64_t src = SORTED ? (tb - 1) * a.tile + a.perm[p] : p;
      bool fast;
      kc = dq_index(x[src], fm, fast);
    }
    s_carry2[0] = kc;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t t, int buf) {
    const int64_t t0 = t * a.tile;
    const int m = (int)min(a.tile, a.n - t0);
    const int mb = m & ~7;  // bulk part (16-byte multiples for both arrays)
    uint32_t bytes = (uint32_t)mb * (SORTED ? 6u : 4u);
    mbar_expect_tx(&bar[buf], bytes);
    if (mb) {
      tma_load(xbuf + buf * kTileMax, x + t0, (uint32_t)mb * 4u, &bar[buf]);
      if (SORTED) tma_load(pbuf + buf * kTileMax, a.perm + t0, (uint32_t)mb * 2u, &bar[buf]);
    }
  };

  if (a.use_tma && tid == 0) {
    issue(tb, 0);
    if (tb + 1 < te) issue(tb + 1, 1);
  }
  uint32_t phases = 0;  // bit b: parity of buffer b's barrier
  for (int64_t t = tb; t < te; t++) {
    const int buf = (int)((t - tb) & 1);
    const int64_t t0 = t * a.tile;
    const int m = (int)min(a.tile, a.n - t0);
    float* xs = xbuf + buf * kTileMax;
    uint16_t* ps = pbuf + buf * kTileMax;
    if (a.use_tma) {
      while (!mbar_try_wait(&bar[buf], (phases >> buf) & 1u)) {
      }
      phases ^= 1u << buf;
      const int mb = m & ~7;
      if (tid < m - mb) {
        xs[mb + tid] = x[t0 + mb + tid];
        if (SORTED) ps[mb + tid] = a.perm[t0 + mb + tid];
      }
    } else {
      for (int i = tid; i < m; i += kQThreads) {
        xs[i] = x[t0 + i];
        if (SORTED) ps[i] = a.perm[t0 + i];
      }
    }
    __syncthreads();

    // ---- warp w owns positions [512 w, 512 w + 512); at step j lane l takes
    // position 512 w + 32 j + l, so shared-memory reads and code stores are
    // consecutive across the warp.  The predecessor's lattice index comes
    // from lane l-1 (one rotate shuffle); lane 0 takes lane 31's from the
    // previous step, and at j = 0 the last index of warp w-1 (recomputed) or
    // of the previous tile (s_carry).
    const int wbase = wid * (kQPer * 32);
    const int cur = (int)((t - tb) & 1);
    int64_t rot_prev = 0;
    if (lane == 0) {
      if (wbase == 0) {
        rot_prev = s_carry2[cur];
      } else if (wbase - 1 < m) {
        const int p = wbase - 1;
        const float xv = SORTED ? xs[min((int)ps[p], m - 1)] : xs[p];
        bool fast;
        rot_prev = dq_index_fast(xv, inv32, fm, fast);
      }
    }
    const int pr = (int)((-t0) & (kChunk - 1));  // position of a chunk start in this tile
    uint16_t* cdst = codes + t0 + wbase + lane;   // advances 32 codes per step
    // 32-bit shared-window addresses, computed once (no per-access
    // generic-to-shared conversion)
    const uint32_t xs_s = smem_u32(xs), ps_s = smem_u32(ps), hw_s = smem_u32(hw);
    uint32_t hwin;  // opaque copy: keeps the compiler from re-deriving the window base per access
    asm volatile("mov.u32 %0, %1;" : "=r"(hwin) : "r"(hw_s));
    int32_t rp32 = (int32_t)max(min(rot_prev, (int64_t)(1 << 30)), -(int64_t)(1 << 30));
    auto step = [&](int j, bool full) {
      const int p = wbase + j * 32 + lane;
      const bool valid = full || p < m;
      float xv = 0.0f;
      if (valid) {
        uint32_t src = (uint32_t)p;
        if (SORTED) src = min(ld_shared_u16(ps_s + 2u * (uint32_t)p), (uint32_t)(m - 1));
        xv = ld_shared_f32(xs_s + 4u * src);
      }
      // FP32 fast lattice index (see dq_index_fast)
      const float tq = xv * inv32;
      const float rq = tq + 12582912.0f;
      const float kf = rq - 12582912.0f;
      const float thr = __fmaf_rn(fabsf(tq), 9.5367431640625e-07f, 9.5367431640625e-07f);
      const bool fast = (0.5f - fabsf(tq - kf)) > thr && fabsf(tq) < 4194304.0f;
      uint32_t code;
      if (__all_sync(0xffffffffu, fast)) {
        // common case: every |k| < 2^22.  32-bit chain: lane 0's predecessor
        // is clamped to +-2^30 (rp32), which keeps any out-of-range q out of
        // range (|q| > half either way), so the escape decision is unchanged
        const int32_t k = __float_as_int(rq) - 0x4B400000;
        const int32_t kr = __shfl_sync(0xffffffffu, k, (lane + 31) & 31);
        int32_t kp = lane == 0 ? rp32 : kr;
        rp32 = kr;
        rot_prev = kr;
        if (p == pr) kp = 0;  // chain restarts every v2 chunk
        const int32_t q = k - kp;
        code = (uint32_t)(q + half) <= (uint32_t)(2 * half - 2) ? (uint32_t)(q + half + 1) : 0u;
        if (valid && p == m - 1) s_carry2[cur ^ 1] = k;  // carry for the next tile
      } else {
        bool fast2;
        const int64_t k = dq_index_fast(xv, inv32, fm, fast2);
        const int64_t kr = __shfl_sync(0xffffffffu, k, (lane + 31) & 31);
        int64_t kp = lane == 0 ? rot_prev : kr;
        rot_prev = kr;
        rp32 = (int32_t)max(min(kr, (int64_t)(1 << 30)), -(int64_t)(1 << 30));
        if (p == pr) kp = 0;
        const int64_t q = k - kp;
        bool ok = (uint64_t)(q + half) <= (uint64_t)(2 * half - 2);
        if (ok && !fast2) {
          float r = (float)__dmul_rn((double)k, twob);
          ok = fabs((double)xv - (double)r) <= b;
        }
        code = ok ? (uint32_t)(q + half + 1) : 0u;
        if (valid && p == m - 1) s_carry2[cur ^ 1] = k;
      }
      if (valid) {
        // histogram: smem window around the centre; escapes (code 0) and
        // far codes go straight to global memory
        const uint32_t wb = code - (uint32_t)wlo;
        if (wb < (uint32_t)kQWin) red_shared_add1(hw_s + 4u * wb);
        else if (code == 0u) atomicAdd(&hist[0], 1u);
        else if (t >= *(volatile long long*)&s_dstart) {
          // deferred
        } else {
          atomicAdd(&hist[code], 1u);
          const uint32_t bud = *(volatile uint32_t*)&s_budget;
          if (atomicAdd(&s_far, 1u) + 1u == bud) {
            if ((uint64_t)(t - tb + 1) * (uint64_t)(a.tile >> 4) <= (uint64_t)bud) s_dstart = t + 1;
            else s_budget = bud < 0x80000000u ? 2u * bud : 0xffffffffu;
          }
        }
        cdst[32 * j] = (uint16_t)code;
      }
    };
    if (m == kQThreads * kQPer && small) {
      // ---- full tile (tile = one 16384-symbol chunk, so the chain restarts at
      // position 0: warp 0 lane 0 starts from k = 0), every |k| < 2^22.  Four
      // consecutive positions per lane per step: at step j lane l takes
      // 512 w + 128 j + 4 l + {0..3}; one 8-byte perm load, one rotate
      // shuffle and one 8-byte code store per four values.  A value is on the
      // FP32 path when its rounding is provably exact against the field-wide
      // error margin (|t - rint(t)| < c); the others take the exact FP64
      // index and reconstruction check (divergent, ~1%).  Escapes count in
      // window bin kQWin; codes outside the window go to global atomics only
      // when some lane holds one.
      uint2* cd = reinterpret_cast<uint2*>(codes + t0 + wbase) + lane;
      int32_t kp0 = wbase == 0 ? 0 : rp32;
      const bool last_lane = (wbase + 4 * lane + 3 == m - 1 - 3 * 128);
#pragma unroll 1
      for (int j = 0; j < kQPer / 4; j++) {
        const uint32_t p0 = (uint32_t)(wbase + j * 128 + 4 * lane);
        float xv[4];
        if (SORTED) {
          uint32_t lo, hi;
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(ps_s + 2u * p0));
          xv[0] = ld_shared_f32(xs_s + ((lo << 2) & 0xfffcu));
          xv[1] = ld_shared_f32(xs_s + ((lo >> 14) & 0xfffcu));
          xv[2] = ld_shared_f32(xs_s + ((hi << 2) & 0xfffcu));
          xv[3] = ld_shared_f32(xs_s + ((hi >> 14) & 0xfffcu));
        } else {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(xs_s + 4u * p0));
          xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
        }
        int32_t k[4];
        bool slow = false;
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float tq = xv[e] * inv32;
          const float rq = tq + 12582912.0f;
          const float dq = tq - (rq - 12582912.0f);
          slow |= !(fabsf(dq) < cmargin);
          k[e] = __float_as_int(rq) - 0x4B400000;
        }
        uint32_t bad = 0;
        if (slow) {
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const float tq = xv[e] * inv32;
            const float dq = tq - ((tq + 12582912.0f) - 12582912.0f);
            if (!(fabsf(dq) < cmargin)) {
              const double kd = rint(__dmul_rn((double)xv[e], inv));
              k[e] = (int32_t)kd;
              const float r = (float)__dmul_rn(kd, twob);
              bad |= (fabs((double)xv[e] - (double)r) <= b ? 0u : 1u) << e;
            }
          }
        }
        const int32_t kr = __shfl_sync(0xffffffffu, k[3], (lane + 31) & 31);
        int32_t kp = lane == 0 ? kp0 : kr;
        kp0 = kr;
        uint32_t code[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const uint32_t u = (uint32_t)(k[e] - kp + half);
          code[e] = u <= (uint32_t)(2 * half - 2) ? u + 1u : 0u;
          kp = k[e];
        }
        if (bad) {
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (bad & (1u << e)) code[e] = 0u;
        }
        if (j == kQPer / 4 - 1 && last_lane) s_carry2[cur ^ 1] = k[3];
        // histogram
        // window bin code - wlo; escapes (code 0) and far codes fall outside
        // the window and take the rare per-element path (escapes to bin kQWin)
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; e++) wv[e] = code[e] - (uint32_t)wlo;
        const uint32_t wmax = max(max(wv[0], wv[1]), max(wv[2], wv[3]));
        if (__any_sync(0xffffffffu, wmax >= (uint32_t)kQWin)) {
          uint32_t far = 0;
#pragma unroll
          for (int e = 0; e < 4; e++) {
            if (code[e] == 0u) red_shared_add1(hwin + 4u * (uint32_t)kQWin);
            else if (wv[e] < (uint32_t)kQWin) red_shared_add1(hwin + 4u * wv[e]);
            else far |= 1u << e;
          }
          if (far) {  // only the lanes that hold far codes pay for the bookkeeping
            // (s_dstart only ever moves to t + 1 during tile t: uniform for the tile)
            if (t < *(volatile long long*)&s_dstart) {
#pragma unroll
              for (int e = 0; e < 4; e++)
                if (far & (1u << e)) atomicAdd(&hist[code[e]], 1u);
              const uint32_t nf = (uint32_t)__popc(far);
              const uint32_t old = atomicAdd(&s_far, nf);
              const uint32_t bud = *(volatile uint32_t*)&s_budget;
              if (old < bud && old + nf >= bud) {
                // the budget is spent: defer from the next tile on if at least
                // 1/16 of the codes so far were far, else examine again at
                // twice the count (a few percent of far codes are cheaper as
                // global atomics than as a second pass over the codes)
                if ((uint64_t)(t - tb + 1) * (uint64_t)(a.tile >> 4) <= (uint64_t)bud) s_dstart = t + 1;
                else s_budget = bud < 0x80000000u ? 2u * bud : 0xffffffffu;
              }
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; e++) red_shared_add1(hwin + 4u * wv[e]);
        }
        cd[32 * j] = make_uint2(code[0] | (code[1] << 16), code[2] | (code[3] << 16));
      }
      rp32 = kp0;
    } else {
#pragma unroll 1
      for (int j = 0; j < kQPer; j++) step(j, false);
    }
    __syncthreads();  // buffer `buf` fully consumed; s_carry visible
    if (a.use_tma && tid == 0 && t + 2 < te) {
      fence_proxy_async();
      issue(t + 2, buf);
    }
  }
  // ---- flush the histogram window (bin kQWin holds escapes, code 0)
  for (int i = tid; i <= kQWin; i += kQThreads) {
    uint32_t c = hw[i];
    int code = i == kQWin ? 0 : wlo + i;
    if (c && code >= 0 && code < (int)a.nbins) atomicAdd(&hist[code], c);
  }
  // ---- far codes of the deferred tiles [s_dstart, te)
  __syncthreads();
  const int64_t td = s_dstart;
  if (td < te) {
    uint32_t* h = reinterpret_cast<uint32_t*>(xbuf);  // [32768]
    for (uint32_t hsel = 0; hsel < 2; hsel++) {
      for (int i = tid; i < 32768; i += kQThreads) h[i] = 0;
      __syncthreads();
      for (int64_t t = td; t < te; t++) {
        const int64_t t0 = t * a.tile;
        const int m = (int)min(a.tile, a.n - t0);
        for (int i = tid; i < m; i += kQThreads) {
          const uint32_t c = codes[t0 + i];
          if (c != 0u && c - (uint32_t)wlo >= (uint32_t)kQWin && (c >> 15) == hsel)
            atomicAdd(&h[c & 32767u], 1u);
        }
      }
      __syncthreads();
      for (int i = tid; i < 32768; i += kQThreads) {
        const uint32_t v = h[i];
        const uint32_t code = (hsel << 15) | (uint32_t)i;
        if (v && (int64_t)code < a.nbins) atomicAdd(&hist[code], v);
      }
      __syncthreads();
    }
  }
}

// ---- sz-lcf (Mode.SZ_LCF, unsorted): LCF predictor on lattice indices,
// pred_0 = 0, pred_1 = k_0, pred_i = 2 k_{i-1} - k_{i-2} (chunk-relative i;
// _kernels.py:162-165 restated for dual quantisation).  Each thread takes
// 16 consecutive positions and recomputes the two lattice indices before
// them, so threads are independent.  (Not on the benchmarked path: kept
// simple, no TMA staging.)
constexpr int kQLThreads = 512;
__global__ void __launch_bounds__(kQLThreads) quantize_lcf_kernel(QArgs a) {
  __shared__ uint32_t hw[kQWin];
  const int field = blockIdx.y;
  const nbzg_field_meta& fm = a.meta->f[field];
  if (fm.is_const || a.n == 0 || a.meta->status) return;
  const float* __restrict__ x = a.f[field];
  uint16_t* __restrict__ codes = a.codes + field * a.code_stride;
  uint32_t* __restrict__ hist = a.hist + field * a.nbins;
  const int half = a.half;
  const int wlo = half + 1 - kQWin / 2;
  const double b = fm.bound, twob = fm.twob;
  const float inv32 = fm.inv32;
  for (int i = threadIdx.x; i < kQWin; i += kQLThreads) hw[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kQLThreads * 16;
  for (int64_t base = ((int64_t)blockIdx.x * kQLThreads + threadIdx.x) * 16; base < a.n;
       base += stride) {
    const int ic0 = (int)(base & (kChunk - 1));
    int64_t k1 = 0, k2 = 0;
    bool f;
    if (ic0 >= 1) k1 = dq_index_fast(x[base - 1], inv32, fm, f);
    if (ic0 >= 2) k2 = dq_index_fast(x[base - 2], inv32, fm, f);
    if (ic0 == 1) k2 = k1;  // pred_1 = k_0 = 2 k_0 - k_0
    const int cnt = (int)min((int64_t)16, a.n - base);
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 16; j++) {
      uint32_t code = 0;
      if (j < cnt) {
        const float xv = x[base + j];
        bool fast;
        const int64_t k = dq_index_fast(xv, inv32, fm, fast);
        const int64_t q = k - (2 * k1 - k2);
        bool ok = (uint64_t)(q + half) <= (uint64_t)(2 * half - 2);
        if (ok && !fast) ok = fabs((double)xv - (double)(float)__dmul_rn((double)k, twob)) <= b;
        code = ok ? (uint32_t)(q + half + 1) : 0u;
        k2 = (ic0 + j == 0) ? k : k1;  // after position 0 both hold k_0
        k1 = k;
        const uint32_t wb = code - (uint32_t)wlo;
        if (wb < (uint32_t)kQWin) atomicAdd(&hw[wb], 1u);
        else atomicAdd(&hist[code], 1u);
      }
      if (j & 1) packed[j >> 1] |= code << 16;
      else packed[j >> 1] = code;
    }
    uint16_t* dst = codes + base;
    if (cnt == 16) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    } else {
      for (int j = 0; j < cnt; j++) dst[j] = (uint16_t)(packed[j >> 1] >> ((j & 1) * 16));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kQWin; i += kQLThreads) {
    const uint32_t c = hw[i];
    const int code = wlo + i;
    if (c && code >= 0 && code < (int)a.nbins) atomicAdd(&hist[code], c);
  }
}

int launch_quantize(const Plan& p, cudaStream_t st, int f0, int nf) {
  if (p.n == 0) return NBZG_OK;
  QArgs a;
  for (int f = 0; f < 6; f++) a.f[f] = p.f[f];
  a.n = p.n;
  a.tile = p.tile;
  a.ntiles = p.ntiles;
  a.perm = p.sorted ? p.perm : nullptr;
  a.meta = p.meta;
  a.half = p.half;
  a.codes = p.codes;
  a.code_stride = (p.n + 7) & ~int64_t(7);
  a.hist = p.hist;
  a.nbins = p.nbins;
  int per_field = max(1, sm_count() / nf);
  if (per_field > p.ntiles) per_field = (int)p.ntiles;
  a.groups = per_field;
  a.f0 = f0;
  a.nf = nf;
  a.far_budget = kQFarBudget;
  if (const char* e = getenv("NBZG_Q_FAR_BUDGET")) a.far_budget = (uint32_t)max(1L, atol(e));
  bool aligned = true;
  for (int f = 0; f < 6; f++) aligned &= (reinterpret_cast<uintptr_t>(p.f[f]) & 15) == 0;
  a.use_tma = aligned && (p.tile % 8 == 0);
  size_t sm = 2 * kTileMax * 4 + 2 * kTileMax * 2 + (kQWin + 4) * 4;
  cudaMemsetAsync(p.hist + (size_t)f0 * p.nbins, 0, sizeof(uint32_t) * nf * p.nbins, st);
  smem_attr((const void*)quantize_kernel<true>, (int)sm);
  smem_attr((const void*)quantize_kernel<false>, (int)sm);
  count_launch();
  if (p.predictor == 1) {
    const int64_t per_cta = (int64_t)kQLThreads * 16;
    int blocks = (int)min((p.n + per_cta - 1) / per_cta, (int64_t)(4 * sm_count() / 6 + 1));
    quantize_lcf_kernel<<<dim3(blocks, 6), kQLThreads, 0, st>>>(a);
  } else if (p.sorted) {
    quantize_kernel<true><<<nf * per_field, kQThreads, sm, st>>>(a);
  } else {
    quantize_kernel<false><<<nf * per_field, kQThreads, sm, st>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
