// nbzg_internal.cuh -- shared device helpers for the B200 (sm_100a) nbz path.
//
// Everything here is HBM-bound integer/byte work plus a little FP64: no
// tensor cores.  Conventions used by every kernel:
//   * 1 GB = 1e9 B; n particles; 6 SoA float32 fields (xx yy zz vx vy vz)
//   * codes are u16: 0 = escape, q + half + 1 otherwise (q in [-half, half-2])
//   * a "tile" is the unit a quantise CTA processes: whole R-index segments,
//     at most 16384 particles (tile == segment at the default segment_size)
//   * a "chunk" is 16384 consecutive codes: the v2 stream's index granularity
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/nbzg.h"

#define NBZG_DEV __device__ __forceinline__

namespace nbzg {

// launch accounting + optional per-kernel CUDA-event tracing (capi.cu)
void count_launch();
void trace_mark(const char* name, cudaStream_t st);

// Bounds checks of the checked build (make variant V=checks
// EXTRA=-DNBZG_CHECKS): a violated index traps the kernel with its location.
// The GPU pool has compute-sanitizer closed, so the test suite runs against
// this build instead (scripts/gpu/checks.sh, profiles/r02_checks.txt).
#ifdef NBZG_CHECKS
#define NBZG_CHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("nbzg check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,          \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                  \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define NBZG_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// NVTX range for the host-side span of one stage (header-only NVTX3: a no-op
// unless a profiler injects its library, e.g. nsys / ncu --nvtx)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

constexpr int kTileMax = 16384;        // particles per tile / codes per chunk
constexpr int kChunk = 16384;          // v2 chunk index granularity (symbols)
constexpr int kEncWin = 16384;         // encoder smem code table: deltas in [-8192, 8191]
constexpr int kMaxCodeLen = 57;        // encode.py:21
constexpr int kHistWindow = 8192;      // smem histogram window (bins) in quantise
constexpr double kIntLimit = 4611686018427387904.0;  // 2^62, quantize.py:29
constexpr double kDqKmax = 4503599627370496.0;       // 2^52 dual-quant clamp

// Per-field resolved parameters + produced sizes (device-resident; copied to
// the host once per call).  Layout mirrored by nbzg_field_meta in nbzg.h.
using FieldMeta = nbzg_field_meta;
using Meta = nbzg_meta;

// ---------------------------------------------------------------- floats
NBZG_DEV uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
NBZG_DEV float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Exact lattice index of x under scale `inv` (= 1/(2b)) or divisor `twob`.
// Fast path in FP32: t32 = x*inv32 is within |t|*2^-22.9 of the exact
// quotient, so rint(t32) is the exact answer whenever t32 is farther than
// |t32|*2^-20 + 2^-20 from a half-integer.  The slow path
// recomputes in FP64 with the reference's exact operation.
//   DIV=true : rint(f64(x) / twob)   (integerize, quantize.py:122-127)
//   DIV=false: rint(f64(x) * inv)    (dual-quant lattice index)
// Returns the double-valued index (no clamping) and whether the fast path
// decided it.
template <bool DIV>
NBZG_DEV double lattice_index(float x, float inv32, double inv, double twob, bool& fast) {
  float t = x * inv32;
  float k = rintf(t);
  float d = fabsf(t - k);
  float thr = fabsf(t) * 9.5367431640625e-07f + 9.5367431640625e-07f;  // 2^-20
  fast = (0.5f - d) > thr && fabsf(t) < 4194304.0f;                       // |t| < 2^22
  if (fast) return (double)k;
  double xd = (double)x;
  return DIV ? rint(__ddiv_rn(xd, twob)) : rint(__dmul_rn(xd, inv));
}

// ---------------------------------------------------------------- bits
NBZG_DEV int bitlen64(uint64_t v) { return v ? 64 - __clzll((long long)v) : 0; }

// spread the low 11 bits of v to every third bit (bit j -> 3j), 32-bit result
NBZG_DEV uint32_t spread3_32(uint32_t v) {
  v &= 0x7ffu;
  v = (v | (v << 16)) & 0x070000ffu;
  v = (v | (v << 8)) & 0x0700f00fu;
  v = (v | (v << 4)) & 0x430c30c3u;
  v = (v | (v << 2)) & 0x49249249u;
  return v;
}
// spread the low 21 bits (bit j -> bit 3j), _kernels.py:757-765 layout
NBZG_DEV uint64_t spread3_64(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// ---------------------------------------------------------------- shared memory
// 32-bit shared-window addresses: computed once per kernel, they spare the
// per-access generic-to-shared conversion the compiler otherwise re-derives
// inside hot loops for pointers into dynamic shared memory.
NBZG_DEV uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
NBZG_DEV uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
// 16-byte read-only load whose L2 miss fills 256 bytes: for per-thread
// sequential streams (a warp touching 32 separate streams would otherwise
// fetch each stream from DRAM one 32-byte sector at a time)
NBZG_DEV uint4 ldg_l2fill(const uint4* p) {
  uint4 r;
  asm("ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
NBZG_DEV uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
NBZG_DEV uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
NBZG_DEV void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
}
NBZG_DEV void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
NBZG_DEV void sts_u64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
template <typename T>
NBZG_DEV T lds_key(uint32_t a);
template <>
NBZG_DEV uint32_t lds_key<uint32_t>(uint32_t a) { return lds_u32(a); }
template <>
NBZG_DEV uint64_t lds_key<uint64_t>(uint32_t a) { return lds_u64(a); }

NBZG_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- scans
// Inclusive warp scan (sum) of a 32-bit value.
template <typename T>
NBZG_DEV T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread. `smem` needs
// blockDim.x/32 + 1 entries.  Returns exclusive prefix; *total = block sum.
template <typename T>
NBZG_DEV T block_excl_scan(T v, T* smem, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? smem[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) smem[lane] = si - s;
    if (lane == nw - 1) smem[32] = si;
  }
  __syncthreads();
  T r = smem[wid] + inc - v;
  *total = smem[32];
  __syncthreads();
  return r;
}

template <typename T>
NBZG_DEV T block_reduce_sum(T v, T* smem) {
  T dummy;
  T ex = block_excl_scan(v, smem, &dummy);
  (void)ex;
  return dummy;
}

// ---------------------------------------------------------------- look-back
// Decoupled look-back over 64-bit status words: top 2 bits = flag
// (0 empty, 1 aggregate, 2 inclusive), low 62 bits = value (sum op).
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

NBZG_DEV void lb_store(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
NBZG_DEV uint64_t lb_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Warp-parallel decoupled look-back, called by ALL 32 lanes of one warp of
// chunk `c` after the chunk knows its local aggregate.  Lane l inspects
// predecessor p - l, so each round covers 32 predecessors with one load per
// lane.  Returns the exclusive prefix (in every lane) and publishes the
// inclusive value.
template <typename T>
NBZG_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

NBZG_DEV uint64_t lookback_sum(uint64_t* status, int64_t c, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (c == 0) {
    if (lane == 0) lb_store(&status[0], kFlagInc | (agg & kValMask));
    return 0;
  }
  if (lane == 0) lb_store(&status[c], kFlagAgg | (agg & kValMask));
  uint64_t excl = 0;
  int64_t p = c - 1;
  while (true) {
    const int64_t idx = p - lane;
    uint64_t s = idx >= 0 ? lb_load(&status[idx]) : kFlagInc;
    uint64_t f = s & ~kValMask;
    if (__any_sync(0xffffffffu, f == 0)) continue;  // predecessors hold lower tickets: running
    uint32_t inc = __ballot_sync(0xffffffffu, f == kFlagInc);
    if (inc) {
      const int first = __ffs(inc) - 1;
      excl += warp_sum<uint64_t>(lane <= first ? (s & kValMask) : 0ull);
      break;
    }
    excl += warp_sum<uint64_t>(s & kValMask);
    p -= 32;
  }
  if (lane == 0) lb_store(&status[c], kFlagInc | ((excl + agg) & kValMask));
  return excl;
}

// Segmented "k-carry" look-back for the decoder: value = (reset:1 | k:61 as
// two's complement).  Composition: a later reset wins, otherwise values add.
NBZG_DEV uint64_t kc_pack(bool reset, int64_t k) {
  return ((uint64_t)reset << 61) | ((uint64_t)k & ((1ull << 61) - 1));
}
NBZG_DEV int64_t kc_val(uint64_t s) {
  return (int64_t)(s << 3) >> 3;  // sign-extend 61 bits
}
NBZG_DEV bool kc_reset(uint64_t s) { return (s >> 61) & 1; }

// Warp-parallel; returns the k carried INTO chunk c (k of the element before
// the chunk; 0 at the stream start) in every lane.
NBZG_DEV int64_t lookback_kcarry(uint64_t* status, int64_t c, bool reset, int64_t kloc) {
  const int lane = threadIdx.x & 31;
  if (c == 0) {
    if (lane == 0) lb_store(&status[0], kFlagInc | kc_pack(true, kloc));
    return 0;
  }
  if (lane == 0) lb_store(&status[c], kFlagAgg | kc_pack(reset, kloc));
  int64_t carry = 0;
  int64_t p = c - 1;
  while (true) {
    const int64_t idx = p - lane;
    uint64_t s = idx >= 0 ? lb_load(&status[idx]) : (kFlagInc | kc_pack(true, 0));
    uint64_t f = s & ~kValMask;
    if (__any_sync(0xffffffffu, f == 0)) continue;
    uint32_t stop = __ballot_sync(0xffffffffu, f == kFlagInc || kc_reset(s));
    if (stop) {
      const int first = __ffs(stop) - 1;
      carry += warp_sum<long long>(lane <= first ? (long long)kc_val(s) : 0ll);
      break;
    }
    carry += warp_sum<long long>((long long)kc_val(s));
    p -= 32;
  }
  int64_t inc = reset ? kloc : carry + kloc;
  if (lane == 0) lb_store(&status[c], kFlagInc | kc_pack(true, inc));
  return carry;
}

}  // namespace nbzg
