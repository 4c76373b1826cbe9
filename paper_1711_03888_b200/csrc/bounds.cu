// bounds.cu -- K1: exact per-field min/max (model.py:104-109) and bound
// resolution (model.py:112-125, pipeline.py:157-181) on device.
//
// One streaming pass over the six SoA fields with 128-bit loads; per-block
// reduction, then one atomicMin/Max per block on an order-preserving u32
// encoding of the floats.  HBM-bound: 24 B/particle read.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

struct Fields6 {
  const float* p[6];
};

__global__ void minmax_init_kernel(uint32_t* mm) {
  int i = threadIdx.x;
  if (i < 12) mm[i] = (i & 1) ? 0u : 0xffffffffu;
}

__global__ void __launch_bounds__(512) minmax6_kernel(Fields6 F, int64_t n, uint32_t* mm) {
  float lo[6], hi[6];
#pragma unroll
  for (int f = 0; f < 6; f++) {
    lo[f] = __int_as_float(0x7f800000);
    hi[f] = -__int_as_float(0x7f800000);
  }
  const int64_t nv = n >> 2;  // float4 count
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
#pragma unroll
    for (int f = 0; f < 6; f++) {
      float4 v = __ldcs(reinterpret_cast<const float4*>(F.p[f]) + i);
      lo[f] = fminf(lo[f], fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
      hi[f] = fmaxf(hi[f], fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
  }
  // tail (n % 4)
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t i = (nv << 2) + threadIdx.x;
#pragma unroll
    for (int f = 0; f < 6; f++) {
      float v = F.p[f][i];
      lo[f] = fminf(lo[f], v);
      hi[f] = fmaxf(hi[f], v);
    }
  }
  __shared__ uint32_t s_lo[6], s_hi[6];
  if (threadIdx.x < 6) {
    s_lo[threadIdx.x] = 0xffffffffu;
    s_hi[threadIdx.x] = 0u;
  }
  __syncthreads();
#pragma unroll
  for (int f = 0; f < 6; f++) {
    float a = lo[f], b = hi[f];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&s_lo[f], f2ord(a));
      atomicMax(&s_hi[f], f2ord(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    atomicMin(&mm[2 * threadIdx.x], s_lo[threadIdx.x]);
    atomicMax(&mm[2 * threadIdx.x + 1], s_hi[threadIdx.x]);
  }
}

int launch_minmax6(const float* const* f, int64_t n, uint32_t* mm, cudaStream_t st) {
  Fields6 F;
  for (int i = 0; i < 6; i++) F.p[i] = f[i];
  count_launch();
  minmax_init_kernel<<<1, 32, 0, st>>>(mm);
  if (n > 0) {
    int64_t nv = (n >> 2);
    int blocks = (int)((nv + 511) / 512);
    int cap = sm_count() * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    count_launch();
    minmax6_kernel<<<blocks, 512, 0, st>>>(F, n, mm);
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// Sorted mode: the same exact min/max of all six fields, one CTA per
// R-index segment at a time, also writing the segment's min/max of the
// three key fields (fields kf0..kf0+2) for K2's per-segment bits/minima.
// One CTA per SM with the whole register file (125 registers: 24 float4 loads
// = 384 bytes in flight per thread) streams at 7.2 TB/s; with the default
// register allocation (97: 12 loads in flight) the kernel ran at 5.7 TB/s, and
// two CTAs of 64 registers per SM are no faster (measured 0.875 / 0.875 /
// 0.92 ms for 1 CTA, 2 CTAs, 2 CTAs without unrolling; 1.10 ms before).
#ifndef NBZG_MM_CTAS
#define NBZG_MM_CTAS 1
#endif
#ifndef NBZG_MM_UNROLL
#define NBZG_MM_UNROLL 2
#endif
constexpr int kMmUnroll = NBZG_MM_UNROLL;
__global__ void __launch_bounds__(512, NBZG_MM_CTAS) minmax_seg_kernel(Fields6 F, int64_t n, int64_t S,
                                                         int64_t nseg, int kf0, uint32_t* mm,
                                                         float* seg_mm) {
  float lo[6], hi[6];
#pragma unroll
  for (int f = 0; f < 6; f++) {
    lo[f] = __int_as_float(0x7f800000);
    hi[f] = -__int_as_float(0x7f800000);
  }
  __shared__ float red[2][3][16];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const int64_t s0 = s * S;
    const int m = (int)min(S, n - s0);
    const int m4 = m >> 2;  // S % 4 == 0: segments start 16-byte aligned
    float sl[6], sh[6];
#pragma unroll
    for (int f = 0; f < 6; f++) {
      sl[f] = __int_as_float(0x7f800000);
      sh[f] = -__int_as_float(0x7f800000);
    }
#pragma unroll kMmUnroll
    for (int v = threadIdx.x; v < m4; v += blockDim.x) {
#pragma unroll
      for (int f = 0; f < 6; f++) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(F.p[f] + s0) + v);
        sl[f] = fminf(sl[f], fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
        sh[f] = fmaxf(sh[f], fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
      }
    }
    for (int i = 4 * m4 + threadIdx.x; i < m; i += blockDim.x)
#pragma unroll
      for (int f = 0; f < 6; f++) {
        const float v = F.p[f][s0 + i];
        sl[f] = fminf(sl[f], v);
        sh[f] = fmaxf(sh[f], v);
      }
#pragma unroll
    for (int f = 0; f < 6; f++) {
      lo[f] = fminf(lo[f], sl[f]);
      hi[f] = fmaxf(hi[f], sh[f]);
    }
    // segment reduction of the key fields
#pragma unroll
    for (int c = 0; c < 3; c++) {
      float a = sl[kf0 + c], b = sh[kf0 + c];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
      }
      if (lane == 0) {
        red[0][c][wid] = a;
        red[1][c][wid] = b;
      }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      const int c = threadIdx.x >> 1, hiw = threadIdx.x & 1;
      float r = red[hiw][c][0];
      for (int q = 1; q < (int)(blockDim.x >> 5); q++)
        r = hiw ? fmaxf(r, red[1][c][q]) : fminf(r, red[0][c][q]);
      seg_mm[6 * s + threadIdx.x] = r;  // [c][min, max]
    }
    __syncthreads();
  }
  __shared__ uint32_t s_lo[6], s_hi[6];
  if (threadIdx.x < 6) {
    s_lo[threadIdx.x] = 0xffffffffu;
    s_hi[threadIdx.x] = 0u;
  }
  __syncthreads();
#pragma unroll
  for (int f = 0; f < 6; f++) {
    float a = lo[f], b = hi[f];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      atomicMin(&s_lo[f], f2ord(a));
      atomicMax(&s_hi[f], f2ord(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    atomicMin(&mm[2 * threadIdx.x], s_lo[threadIdx.x]);
    atomicMax(&mm[2 * threadIdx.x + 1], s_hi[threadIdx.x]);
  }
}

int launch_minmax_seg(const Plan& p, cudaStream_t st) {
  Fields6 F;
  for (int i = 0; i < 6; i++) F.p[i] = p.f[i];
  count_launch();
  minmax_init_kernel<<<1, 32, 0, st>>>(p.minmax);
  int blocks = (int)min(p.nseg, (int64_t)sm_count() * 4);
  if (blocks < 1) blocks = 1;
  count_launch();
  minmax_seg_kernel<<<blocks, 512, 0, st>>>(F, p.n, p.S, p.nseg, p.variant == 1 ? 3 : 0,
                                            p.minmax, p.seg_mm);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// sharded compress, phase 2: the all-gathered global (lo, hi) per field
struct MinMax12 {
  float v[12];
};
__global__ void minmax_set_kernel(MinMax12 h, uint32_t* mm) {
  const int i = threadIdx.x;
  if (i < 12) mm[i] = f2ord(h.v[i]);
}

int launch_minmax_set(const float* h_minmax12, uint32_t* mm, cudaStream_t st) {
  MinMax12 h;
  for (int i = 0; i < 12; i++) h.v[i] = h_minmax12[i];
  count_launch();
  minmax_set_kernel<<<1, 32, 0, st>>>(h, mm);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// resolve_field_bounds (pipeline.py:157-181): constant fields (zero range)
// take the fast path regardless of bound kind; others get
// b = value (absolute) or b = value * (float(hi) - float(lo)) in f64.
struct ResolveArgs {
  const float* f[6];
  int kind[6];
  double value[6];
  int64_t n;
  int64_t nseg;
};

__global__ void resolve_kernel(ResolveArgs a, const uint32_t* mm, nbzg_meta* meta) {
  if (threadIdx.x != 0) return;
  uint32_t mask = 0;
  for (int f = 0; f < 6; f++) {
    nbzg_field_meta& m = meta->f[f];
    float lo = ord2f(mm[2 * f]), hi = ord2f(mm[2 * f + 1]);
    m.lo = lo;
    m.hi = hi;
    m.k = 0;
    m.min_len = m.max_len = 0;
    m.n_esc = m.total_bits = 0;
    m.payload_off = m.payload_len = 0;
    m.index_off = m.bits_off = m.esc_off = 0;
    m.constant = 0.0f;
    m.is_const = 0;
    double b = 0.0;
    if (a.n > 0) {
      double rng = (double)hi - (double)lo;
      if (rng == 0.0) {
        mask |= 1u << f;
        m.is_const = 1;
        m.constant = a.f[f][0];
      } else {
        b = a.kind[f] == 0 ? a.value[f] : a.value[f] * rng;
      }
    }
    m.bound = b;
    m.twob = 2.0 * b;
    m.inv = b > 0.0 ? 1.0 / (2.0 * b) : 0.0;
    m.inv32 = (float)m.inv;
  }
  meta->mask = mask;
  meta->status = 0;
  meta->arena_used = 0;
  meta->nseg = (uint64_t)a.nseg;
}

int launch_resolve(const Plan& p, cudaStream_t st) {
  ResolveArgs a;
  for (int f = 0; f < 6; f++) {
    a.f[f] = p.f[f];
    a.kind[f] = p.bound_kind[f];
    a.value[f] = p.bound_value[f];
  }
  a.n = p.n;
  a.nseg = p.nseg;
  count_launch();
  resolve_kernel<<<1, 32, 0, st>>>(a, p.minmax, p.meta);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

// CPC modes: fields without an SZ stream are marked constant for the SZ
// stages (quantize / codebook / layout / encode skip them); meta->mask keeps
// the true constant mask for the archive and the CPC kernels.
__global__ void sz_skip_kernel(nbzg_meta* meta, uint32_t skip) {
  const int f = threadIdx.x;
  if (f < 6 && ((skip >> f) & 1u)) meta->f[f].is_const = 1;
}

int launch_sz_skip(const Plan& p, cudaStream_t st) {
  count_launch();
  sz_skip_kernel<<<1, 32, 0, st>>>(p.meta, p.sz_skip);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
