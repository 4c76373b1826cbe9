// rlarge.cu -- the R-index sort for segments longer than one 16384-particle
// tile (Settings.segment_size > 16384, sz-lv-prx; rindex.py:155-229 has no
// upper bound on the segment size).
//
// A segment no longer fits a CTA's shared memory, so the segment-local
// stable sort becomes ONE device-wide stable LSD radix sort of composite
// keys (segment << kb) | masked_key -- sorting by segment first keeps every
// particle inside its segment, and LSD passes are stable, so ties keep the
// original order exactly as prx_order's stable sort does (_kernels.py:
// 887-927).  Per 8-bit pass: per-block digit counts (4096 keys per CTA), a
// digit-major exclusive scan over (digit, block), and a stable scatter
// (per-warp MATCH.ANY ranks + the block's per-digit offsets).  The fields
// are then gathered into sorted order and the SZ stages run on them as on
// an unsorted snapshot (the v2 chain restarts every 16384 symbols either
// way).  Output: the u32 global source index per sorted position.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kLBlock = 4096;  // keys per CTA in the radix passes
constexpr int kLThreads = 256;
constexpr int kLWarps = kLThreads / 32;
constexpr int kLPer = kLBlock / kLThreads;  // 16 keys per thread
constexpr int kLScan = 4096;                // entries per CTA of the scan

struct LArgs {
  const float* x[3];
  const nbzg_meta* meta;
  int fbase;  // meta index of x[0] (0, or 3 for the velocity variant)
  const float* seg_mm;  // [nseg][3][2]
  int64_t n, S, nseg;
  int ig, no_clamp;
  uint8_t* seg_bits;
  int64_t* lmn;     // [nseg][3]
  int32_t* lshift;  // [nseg]
  uint32_t* kbits;  // [0]: max masked-key bits over segments
  uint32_t* status;
};

// segment min / max of the key fields when K1 did not produce them
__global__ void __launch_bounds__(256) lseg_minmax_kernel(LArgs a, float* seg_mm) {
  const int64_t s = blockIdx.x;
  const int64_t s0 = s * a.S, s1 = min(a.n, s0 + a.S);
  __shared__ float red[2][3][8];
  float mn[3], mx[3];
  for (int c = 0; c < 3; c++) {
    mn[c] = __int_as_float(0x7f800000);
    mx[c] = -__int_as_float(0x7f800000);
  }
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x)
    for (int c = 0; c < 3; c++) {
      const float v = a.x[c][i];
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
  if (threadIdx.x < 6) {
    const int c = threadIdx.x >> 1, hi = threadIdx.x & 1;
    float r = red[hi][c][0];
    for (int q = 1; q < 8; q++) r = hi ? fmaxf(r, red[1][c][q]) : fminf(r, red[0][c][q]);
    seg_mm[6 * s + threadIdx.x] = r;
  }
}

// per segment (one thread each): minima, need, bits, clamp drop, shift
// (rindex.py:164-198, prx_sort's shift = 3 min(k, bits))
__global__ void lseg_params_kernel(LArgs a) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nseg) return;
  const nbzg_field_meta* fm = a.meta->f + a.fbase;
  int need = 0, bad = 0;
  int64_t rng[3];
  for (int c = 0; c < 3; c++) {
    rng[c] = 0;
    a.lmn[3 * s + c] = 0;
    if (fm[c].is_const) continue;
    const double qa = __ddiv_rn((double)a.seg_mm[6 * s + 2 * c], fm[c].twob);
    const double qb = __ddiv_rn((double)a.seg_mm[6 * s + 2 * c + 1], fm[c].twob);
    if (fabs(qa) > kIntLimit || fabs(qb) > kIntLimit) bad = 1;
    const int64_t ia = (int64_t)rint(qa), ib = (int64_t)rint(qb);
    a.lmn[3 * s + c] = ia;
    rng[c] = ib - ia;
    need = max(need, bitlen64((uint64_t)rng[c]));
  }
  const int bits = min(need, 21);
  const int drop = need > 21 ? need - 21 : 0;
  if (a.no_clamp && need > 21) bad = 1;
  const int eff = min(a.ig, bits);
  a.seg_bits[s] = (uint8_t)bits;
  a.lshift[s] = drop + eff;
  if (bad) atomicCAS(a.status, 0u, (uint32_t)NBZG_BOUND_TOO_SMALL);
  atomicMax(a.kbits, (uint32_t)(3 * (bits - eff)));
}

// composite keys (segment << kb) | masked key, values = source index
__global__ void __launch_bounds__(256) lkeys_kernel(LArgs a, uint64_t* key, uint32_t* val) {
  const nbzg_field_meta* fm = a.meta->f + a.fbase;
  const int kb = (int)*a.kbits;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const int64_t s = i / a.S;
    const int sh = a.lshift[s];
    uint64_t u[3];
    for (int c = 0; c < 3; c++) {
      int64_t iv = 0;
      if (!fm[c].is_const) {
        bool fast;
        iv = (int64_t)lattice_index<true>(a.x[c][i], fm[c].inv32, fm[c].inv, fm[c].twob, fast);
      }
      u[c] = (uint64_t)(iv - a.lmn[3 * s + c]) >> sh;
    }
    // bit j of field t at 3j + 2 - t (_kernels.py:757-786), the shifted-out
    // low groups already gone
    const uint64_t k = (spread3_64(u[0]) << 2) | (spread3_64(u[1]) << 1) | spread3_64(u[2]);
    key[i] = kb < 64 ? (((uint64_t)s << kb) | k) : k;
    val[i] = (uint32_t)i;
  }
}

// ---- one LSD pass: block digit counts, (digit, block) scan, stable scatter
__global__ void __launch_bounds__(kLThreads) lhist_kernel(const uint64_t* key, int64_t n, int sh,
                                                          uint32_t* hist, int64_t nblk) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * kLBlock;
  for (int k = 0; k < kLPer; k++) {
    const int64_t i = b0 + k * kLThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> sh) & 255], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(1024) lscan_sum_kernel(const uint32_t* in, int64_t E,
                                                         uint32_t* part) {
  __shared__ uint32_t tmp[33];
  const int64_t e0 = (int64_t)blockIdx.x * kLScan;
  uint32_t s = 0;
  for (int k = threadIdx.x; k < kLScan; k += blockDim.x)
    if (e0 + k < E) s += in[e0 + k];
  const uint32_t tot = block_reduce_sum<uint32_t>(s, tmp);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) lscan_part_kernel(uint32_t* part, int64_t np) {
  __shared__ uint32_t tmp[33];
  const int R = (int)((np + blockDim.x - 1) / blockDim.x);
  uint32_t s = 0;
  for (int r = 0; r < R; r++) {
    const int64_t i = (int64_t)threadIdx.x * R + r;
    if (i < np) s += part[i];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan<uint32_t>(s, tmp, &tot);
  for (int r = 0; r < R; r++) {
    const int64_t i = (int64_t)threadIdx.x * R + r;
    if (i < np) {
      const uint32_t v = part[i];
      part[i] = ex;
      ex += v;
    }
  }
}

__global__ void __launch_bounds__(1024) lscan_apply_kernel(uint32_t* io, int64_t E,
                                                           const uint32_t* part) {
  __shared__ uint32_t tmp[33];
  const int64_t e0 = (int64_t)blockIdx.x * kLScan;
  constexpr int R = kLScan / 1024;
  uint32_t v[R], s = 0;
  for (int r = 0; r < R; r++) {
    const int64_t i = e0 + (int64_t)threadIdx.x * R + r;
    v[r] = i < E ? io[i] : 0u;
    s += v[r];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan<uint32_t>(s, tmp, &tot) + part[blockIdx.x];
  for (int r = 0; r < R; r++) {
    const int64_t i = e0 + (int64_t)threadIdx.x * R + r;
    if (i < E) io[i] = ex;
    ex += v[r];
  }
}

__global__ void __launch_bounds__(kLThreads) lscatter_kernel(const uint64_t* key, const uint32_t* val,
                                                             int64_t n, int sh, const uint32_t* gscan,
                                                             int64_t nblk, uint64_t* okey,
                                                             uint32_t* oval) {
  __shared__ uint64_t sk[kLBlock];
  __shared__ uint16_t wh[kLWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kLBlock;
  const int m = (int)min((int64_t)kLBlock, n - b0);
  for (int k = threadIdx.x; k < m; k += kLThreads) sk[k] = key[b0 + k];
  for (int k = threadIdx.x; k < kLWarps * 256; k += kLThreads) (&wh[0][0])[k] = 0;
  __syncthreads();
  // warp w ranks its 512 keys in order (stable: warp-major, then step, then lane)
  uint32_t rk[kLPer / 2];
  const int base = w * (kLBlock / kLWarps);
#pragma unroll
  for (int j = 0; j < kLPer; j++) {  // 16 steps of 32 lanes
    const int pos = base + j * 32 + lane;
    const bool valid = pos < m;
    const uint32_t d = valid ? (uint32_t)((sk[pos] >> sh) & 255) : 0x100u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t lt = __popc(peers & lanemask_lt());
    const uint32_t cnt = valid ? wh[w][d] : 0u;
    __syncwarp();
    if (valid && lt == 0) wh[w][d] = (uint16_t)(cnt + __popc(peers));
    __syncwarp();
    const uint32_t r = cnt + lt;
    if (j & 1) rk[j >> 1] |= r << 16;
    else rk[j >> 1] = r;
  }
  __syncthreads();
  // per digit: exclusive offsets of the warps (digit d = thread)
  {
    const int d = threadIdx.x;  // 256 threads = 256 digits
    uint32_t s = 0;
    for (int q = 0; q < kLWarps; q++) {
      const uint32_t c = wh[q][d];
      wh[q][d] = (uint16_t)s;
      s += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kLPer; j++) {
    const int pos = base + j * 32 + lane;
    if (pos < m) {
      const uint32_t d = (uint32_t)((sk[pos] >> sh) & 255);
      const uint32_t r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      const uint64_t g = (uint64_t)gscan[(int64_t)d * nblk + blockIdx.x] + wh[w][d] + r;
      okey[g] = sk[pos];
      oval[g] = val[b0 + pos];
    }
  }
}

// sorted copies of the six fields (the SZ stages then see an unsorted snapshot)
__global__ void __launch_bounds__(256) lgather_kernel(const float* f0, const float* f1,
                                                      const float* f2, const float* f3,
                                                      const float* f4, const float* f5,
                                                      const uint32_t* src, int64_t n, float* out,
                                                      int64_t stride) {
  const float* f[6] = {f0, f1, f2, f3, f4, f5};
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const uint32_t s = src[i];
#pragma unroll
    for (int c = 0; c < 6; c++) out[c * stride + i] = __ldg(f[c] + s);
  }
}

size_t large_ws(int64_t n, int64_t nseg) {
  const int64_t nblk = (n + kLBlock - 1) / kLBlock;
  const int64_t E = 256 * nblk;
  const int64_t np = (E + kLScan - 1) / kLScan;
  return 2 * (8 + 4) * (size_t)(n + 16) + 4 * (size_t)E + 4 * (size_t)(np + 16) +
         6 * 4 * (size_t)((n + 3) & ~int64_t(3)) + 8 * 3 * (size_t)(nseg + 1) +
         4 * (size_t)(nseg + 1) + 4 * 6 * (size_t)(nseg + 1) + 4096;
}

// The sorted field copies head the long-segment workspace; a phase-4 call
// (encode only) points the SZ stages at them again.
void large_fields(Plan& p) {
  const int64_t xs = (p.n + 3) & ~int64_t(3);
  for (int c = 0; c < 6; c++) p.f[c] = reinterpret_cast<float*>(p.large_ws) + c * xs;
}

// K2 for long segments.  On return p.f points at the sorted field copies
// and p.order32 holds the permutation.  One synchronisation: the pass count
// depends on the widest masked key, a device value.
int launch_rindex_large(Plan& p, cudaStream_t st, bool& stop) {
  stop = false;
  if (p.n == 0) return NBZG_OK;
  if (p.variant == 2 || p.cpc) return NBZG_UNSUPPORTED;
  uint8_t* w = p.large_ws;
  auto take = [&](size_t bytes) {
    uint8_t* r = w;
    w += (bytes + 255) & ~size_t(255);
    return r;
  };
  const int64_t n = p.n, nseg = p.nseg;
  const int64_t nblk = (n + kLBlock - 1) / kLBlock;
  const int64_t E = 256 * nblk;
  const int64_t np = (E + kLScan - 1) / kLScan;
  const int64_t xs = (n + 3) & ~int64_t(3);
  float* xsort = reinterpret_cast<float*>(take(6 * 4 * (size_t)xs));  // first: see large_fields
  uint64_t* key[2] = {reinterpret_cast<uint64_t*>(take(8 * (size_t)(n + 16))),
                      reinterpret_cast<uint64_t*>(take(8 * (size_t)(n + 16)))};
  uint32_t* val[2] = {reinterpret_cast<uint32_t*>(take(4 * (size_t)(n + 16))),
                      reinterpret_cast<uint32_t*>(take(4 * (size_t)(n + 16)))};
  uint32_t* hist = reinterpret_cast<uint32_t*>(take(4 * (size_t)E));
  uint32_t* part = reinterpret_cast<uint32_t*>(take(4 * (size_t)(np + 16)));
  LArgs a;
  a.fbase = p.variant == 1 ? 3 : 0;
  for (int c = 0; c < 3; c++) a.x[c] = p.f[a.fbase + c];
  a.meta = p.meta;
  a.n = n;
  a.S = p.S;
  a.nseg = nseg;
  a.ig = p.ig;
  a.no_clamp = p.cpc ? 1 : 0;
  a.seg_bits = p.seg_bits;
  a.lmn = reinterpret_cast<int64_t*>(take(8 * 3 * (size_t)(nseg + 1)));
  a.lshift = reinterpret_cast<int32_t*>(take(4 * (size_t)(nseg + 1)));
  a.kbits = reinterpret_cast<uint32_t*>(take(64));
  a.status = &p.meta->status;
  float* smm = p.seg_mm;
  if (!smm) {
    smm = reinterpret_cast<float*>(take(4 * 6 * (size_t)(nseg + 1)));
    count_launch();
    lseg_minmax_kernel<<<(unsigned)nseg, 256, 0, st>>>(a, smm);
  }
  a.seg_mm = smm;
  cudaMemsetAsync(a.kbits, 0, 4, st);
  count_launch();
  lseg_params_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, st>>>(a);
  uint32_t kb = 0, status = 0;
  cudaMemcpyAsync(&kb, a.kbits, 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&status, a.status, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return NBZG_CUDA_ERROR;
  if (status) {  // BOUND_TOO_SMALL is in meta: no sort, no SZ stages
    stop = true;
    return NBZG_OK;
  }
  int sb = 0;
  while ((int64_t(1) << sb) < nseg) sb++;
  const int total = (int)kb + sb;
  if (total > 64) return NBZG_UNSUPPORTED;
  const int blocks = (int)min((n + 255) / 256, (int64_t)sm_count() * 16);
  count_launch();
  lkeys_kernel<<<blocks, 256, 0, st>>>(a, key[0], val[0]);
  int cur = 0;
  for (int sh = 0; sh < total; sh += 8) {
    count_launch();
    lhist_kernel<<<(unsigned)nblk, kLThreads, 0, st>>>(key[cur], n, sh, hist, nblk);
    count_launch();
    lscan_sum_kernel<<<(unsigned)np, 1024, 0, st>>>(hist, E, part);
    count_launch();
    lscan_part_kernel<<<1, 1024, 0, st>>>(part, np);
    count_launch();
    lscan_apply_kernel<<<(unsigned)np, 1024, 0, st>>>(hist, E, part);
    count_launch();
    lscatter_kernel<<<(unsigned)nblk, kLThreads, 0, st>>>(key[cur], val[cur], n, sh, hist, nblk,
                                                          key[cur ^ 1], val[cur ^ 1]);
    cur ^= 1;
  }
  cudaMemcpyAsync(p.order32, val[cur], 4 * (size_t)n, cudaMemcpyDeviceToDevice, st);
  count_launch();
  lgather_kernel<<<blocks, 256, 0, st>>>(p.f[0], p.f[1], p.f[2], p.f[3], p.f[4], p.f[5], val[cur],
                                         n, xsort, xs);
  for (int c = 0; c < 6; c++) p.f[c] = xsort + c * xs;
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
