// crc.cu -- CRC-64/XZ of device buffers (_kernels.py:954-994: reflected
// ECMA-182 polynomial, init and xorout all ones).
//
// CRC is linear over GF(2):  crc0(A||B) = Z_|B|(crc0(A)) ^ crc0(B), where
// crc0 is the zero-init, no-xorout CRC and Z_L ("feed L zero bytes") is a
// 64x64 bit matrix, applied as 8 byte-sliced lookup tables.  Leading zero
// bytes do not change crc0, so the stream -- minus the < 16 tail bytes past
// the last 16-byte-aligned address, which the fold kernel appends bytewise --
// is front-padded (virtually) to a whole number of 512 KiB CTA spans; every
// 16-byte piece of the padded stream is then aligned in memory:
//   K1 crc_span_kernel: a warp CRCs a 64 KiB block in 128 coalesced 512-byte
//      steps, lane j taking the 16-byte piece j of every step.  A lane's pieces
//      lie 496 bytes apart; "absorb 16 bytes, then 496 zero bytes" is one
//      linear map of (state ^ piece), so its slicing-by-16 tables are
//      Z_496 o T_k -- the same 16 lookups per 16 bytes as contiguous slicing.
//      The tables sit in shared memory entry-major ([byte value][k], 8-byte
//      entries: table k lives in bank pair k) and lane j visits its bytes in
//      the rotated order (s + j) mod 16, so the 16 lanes of a half-warp read
//      16 different tables = 16 different bank pairs: every lookup is
//      conflict-free (2 wavefronts instead of ~6 for random 8-byte reads).
//      The last step uses the plain tables; a shuffle tree folds the lanes
//      (Z_16 ... Z_256), then the CTA's 8 warps -> crc0 of its 512 KiB span;
//   K2 crc_fold_kernel: one CTA folds the span values (sequential runs, then
//      a tree) and applies  crc = Z_n(~0) ^ crc0 ^ ~0.
// The tables (slicing and Z_{2^j}, j = 0..40) are built once on the host and
// uploaded once per device.  HBM-bound: one read of the data.
#include <algorithm>
#include <mutex>

#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kCrcLevels = 41;        // Z_{2^j}, j = 0..40 bytes
constexpr int kCrcBlockLog = 11;      // 2 KiB per thread
constexpr int kCrcThreads = 256;      // threads per span CTA
constexpr int kCrcSpanLog = kCrcBlockLog + 8;  // 512 KiB per CTA
constexpr int kFoldThreads = 1024;
constexpr uint64_t kPoly = 0xC96C5795D7870F42ull;

__device__ uint64_t g_crc_slice[16 * 256];          // T_k[b]: byte b then k zero bytes
__device__ uint64_t g_crc_skip[256 * 16];           // [b][k]: Z_496(T_k[b]) (interleaved pieces)
__device__ uint64_t g_crc_z[kCrcLevels * 8 * 256];  // Z_{2^j} byte-sliced

NBZG_DEV uint64_t zshift(const uint64_t* T, uint64_t v) {  // T: [8][256]
  uint64_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) r ^= __ldg(T + j * 256 + ((v >> (8 * j)) & 0xff));
  return r;
}

// host: build the tables once
namespace {
struct CrcTables {
  uint64_t slice[16 * 256];
  uint64_t skip[256 * 16];
  uint64_t z[kCrcLevels * 8 * 256];
};
const CrcTables& host_tables() {
  static CrcTables* t = [] {
    auto* T = new CrcTables;
    for (int b = 0; b < 256; b++) {
      uint64_t c = (uint64_t)b;
      for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
      T->slice[b] = c;
    }
    for (int k = 1; k < 16; k++)
      for (int b = 0; b < 256; b++) {
        const uint64_t p = T->slice[(k - 1) * 256 + b];
        T->slice[k * 256 + b] = (p >> 8) ^ T->slice[p & 0xff];
      }
    auto apply = [](const uint64_t* Z, uint64_t v) {
      uint64_t r = 0;
      for (int j = 0; j < 8; j++) r ^= Z[j * 256 + ((v >> (8 * j)) & 0xff)];
      return r;
    };
    for (int j = 0; j < 8; j++)  // Z_1: one zero byte
      for (int b = 0; b < 256; b++) {
        const uint64_t v = (uint64_t)b << (8 * j);
        T->z[j * 256 + b] = (v >> 8) ^ T->slice[v & 0xff];
      }
    for (int L = 1; L < kCrcLevels; L++) {  // Z_{2^L} = Z_{2^(L-1)} o Z_{2^(L-1)}
      const uint64_t* P = T->z + (size_t)(L - 1) * 2048;
      for (int j = 0; j < 8; j++)
        for (int b = 0; b < 256; b++)
          T->z[(size_t)L * 2048 + j * 256 + b] = apply(P, apply(P, (uint64_t)b << (8 * j)));
    }
    for (int k = 0; k < 16; k++)  // Z_496 = Z_256 o Z_128 o Z_64 o Z_32 o Z_16
      for (int b = 0; b < 256; b++) {
        uint64_t v = T->slice[k * 256 + b];
        for (int L = 4; L <= 8; L++) v = apply(T->z + (size_t)L * 2048, v);
        T->skip[b * 16 + k] = v;
      }
    return T;
  }();
  return *t;
}

int upload_tables() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return NBZG_CUDA_ERROR;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return NBZG_OK;
  const CrcTables& T = host_tables();
  if (cudaMemcpyToSymbol(g_crc_slice, T.slice, sizeof(T.slice)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_crc_skip, T.skip, sizeof(T.skip)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_crc_z, T.z, sizeof(T.z)) != cudaSuccess)
    return NBZG_CUDA_ERROR;
  done[dev] = true;
  return NBZG_OK;
}
}  // namespace

// Up to kCrcMax buffers per launch (an archive's payloads): one grid over
// all their spans, so small payloads still fill the GPU.
constexpr int kCrcMax = 8;
struct CrcJobs {
  const uint8_t* data[kCrcMax];
  int64_t n[kCrcMax];       // whole length (the init / xorout term)
  int64_t n_main[kCrcMax];  // bytes the span kernel covers: ends 16-byte aligned
  int64_t pad[kCrcMax];     // virtual leading zero bytes of the main part
  int64_t span0[kCrcMax + 1];  // first span of each buffer; span0[count] = total
  uint64_t* out[kCrcMax];
  int run_log[kCrcMax];
  int count;
};

constexpr int kCrcWarpLog = 16;  // 64 KiB per warp: 128 steps of 32 x 16 bytes
constexpr int kCrcSteps = 1 << (kCrcWarpLog - 9);

// crc0 of each 512 KiB span of each front-padded stream (pad zero bytes,
// then data[0, n_main)); persistent CTAs, spans strided by the grid.
__global__ void __launch_bounds__(kCrcThreads) crc_span_kernel(CrcJobs J, uint64_t* span_out) {
  __shared__ __align__(128) uint64_t TS[256 * 16];  // [byte][k]
  __shared__ uint64_t wsum[kCrcThreads / 32];
  for (int i = threadIdx.x; i < 256 * 16; i += kCrcThreads) TS[i] = g_crc_skip[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t jl = (uint32_t)lane & 15u;
  // step s of a piece reads byte (s + jl) & 15 -> table k = 15 - that byte
  uint32_t koff[16];
#pragma unroll
  for (int s = 0; s < 16; s++) koff[s] = ((15u - (uint32_t)s - jl) & 15u) << 3;
  const uint32_t ts_s = (uint32_t)__cvta_generic_to_shared(TS);
  const uint32_t rot8 = 8u * (jl & 3u);
  const bool rw1 = (jl >> 2) & 1u, rw2 = (jl >> 3) & 1u;

  for (int64_t sp = blockIdx.x; sp < J.span0[J.count]; sp += gridDim.x) {
    int b = 0;
    while (b + 1 < J.count && sp >= J.span0[b + 1]) b++;
    const int64_t pad = J.pad[b];
    // padded offset of this warp's block; piece `lane` of step m at p0 + 512 m
    const int64_t p0 = ((sp - J.span0[b]) << kCrcSpanLog) + ((int64_t)warp << kCrcWarpLog) + 16 * lane;
    const uint8_t* base = J.data[b] - pad;  // padded offset 0 (never dereferenced below data)
    auto load = [&](int m) -> uint4 {
      const int64_t p = p0 + 512 * (int64_t)m;
      uint4 d = make_uint4(0, 0, 0, 0);
      if (p + 16 > pad) {
        d = __ldg(reinterpret_cast<const uint4*>(base + p));
        if (p < pad) {  // the piece straddling the start of the data: zero its lead
          const int lead = (int)(pad - p);  // 1 .. 15
          uint32_t w[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int z = lead - 4 * q;  // leading bytes of word q to clear
            w[q] = z >= 4 ? 0u : (z > 0 ? w[q] & (0xffffffffu << (8 * z)) : w[q]);
          }
          d = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      return d;
    };
    uint64_t crc = 0;
    // absorb one piece, then 496 zero bytes (the skip tables)
    auto step = [&](const uint4 d) {
      uint32_t w0 = d.x ^ (uint32_t)crc, w1 = d.y ^ (uint32_t)(crc >> 32), w2 = d.z, w3 = d.w;
      // rotate the 16 bytes right by jl: words, then bytes
      uint32_t t0 = rw1 ? w1 : w0, t1 = rw1 ? w2 : w1, t2 = rw1 ? w3 : w2, t3 = rw1 ? w0 : w3;
      w0 = rw2 ? t2 : t0, w1 = rw2 ? t3 : t1, w2 = rw2 ? t0 : t2, w3 = rw2 ? t1 : t3;
      const uint32_t r[4] = {__funnelshift_r(w0, w1, rot8), __funnelshift_r(w1, w2, rot8),
                             __funnelshift_r(w2, w3, rot8), __funnelshift_r(w3, w0, rot8)};
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int s = 0; s < 16; s++) {
        const uint32_t x = r[s >> 2];
        const uint32_t v7 = (s & 3) == 0 ? (x << 7) : ((s & 3) == 1 ? (x >> 1) : ((s & 3) == 2 ? (x >> 9) : (x >> 17)));
        uint32_t e0, e1;
        asm("ld.shared.v2.u32 {%0, %1}, [%2];"
                     : "=r"(e0), "=r"(e1)
                     : "r"(ts_s + ((v7 & 0x7f80u) | koff[s])));
        lo ^= e0;
        hi ^= e1;
      }
      crc = ((uint64_t)hi << 32) | lo;
    };
    int m = 0;
    for (; m + 4 < kCrcSteps; m += 4) {
      const uint4 d0 = load(m), d1 = load(m + 1), d2 = load(m + 2), d3 = load(m + 3);
      step(d0);
      step(d1);
      step(d2);
      step(d3);
    }
    {
      const uint4 d0 = load(m), d1 = load(m + 1), d2 = load(m + 2), d3 = load(m + 3);
      step(d0);
      step(d1);
      step(d2);
      // the last piece: plain slicing-by-16 (no trailing zeros)
      const uint64_t lo = (((uint64_t)d3.y << 32) | d3.x) ^ crc;
      const uint64_t hi = ((uint64_t)d3.w << 32) | d3.z;
      uint64_t r = 0;
#pragma unroll
      for (int k = 0; k < 8; k++) r ^= __ldg(g_crc_slice + (15 - k) * 256 + ((lo >> (8 * k)) & 0xff));
#pragma unroll
      for (int k = 0; k < 8; k++) r ^= __ldg(g_crc_slice + (7 - k) * 256 + ((hi >> (8 * k)) & 0xff));
      crc = r;
    }
    // fold the warp's 32 lanes (lane j ends 16 (31 - j) bytes before the block
    // end), then the CTA's 8 warps
#pragma unroll
    for (int l = 0; l < 5; l++) {
      const uint64_t right = __shfl_down_sync(0xffffffffu, crc, 1 << l);
      const uint64_t shifted = zshift(g_crc_z + (size_t)(4 + l) * 2048, crc);
      if ((lane & ((2 << l) - 1)) == 0) crc = shifted ^ right;
    }
    if (lane == 0) wsum[warp] = crc;
    __syncthreads();
    if (warp == 0) {
      crc = lane < kCrcThreads / 32 ? wsum[lane] : 0;
#pragma unroll
      for (int l = 0; l < 3; l++) {
        const uint64_t right = __shfl_down_sync(0xffffffffu, crc, 1 << l);
        const uint64_t shifted = zshift(g_crc_z + (size_t)(kCrcWarpLog + l) * 2048, crc);
        if ((lane & ((2 << l) - 1)) == 0) crc = shifted ^ right;
      }
      if (lane == 0) span_out[sp] = crc;
    }
    __syncthreads();  // wsum is reused by the next span
  }
}

// fold C span values (front-padded with zero spans to kFoldThreads runs of
// 2^run_log) and finish; one CTA per buffer
__global__ void __launch_bounds__(kFoldThreads) crc_fold_kernel(CrcJobs J,
                                                               const uint64_t* span_all) {
  const int b = blockIdx.x;
  const uint64_t* span = span_all + J.span0[b];
  const int64_t C = J.span0[b + 1] - J.span0[b];
  const int run_log = J.run_log[b];
  const int64_t n = J.n[b];
  uint64_t* crc_out = J.out[b];
  __shared__ uint64_t v[kFoldThreads];
  const int t = threadIdx.x;
  const int64_t run = int64_t(1) << run_log;
  const int64_t lead = (int64_t(kFoldThreads) << run_log) - C;
  uint64_t c = 0;
  const uint64_t* Zs = g_crc_z + (size_t)kCrcSpanLog * 2048;
  for (int64_t j = 0; j < run; j++) {
    const int64_t e = (int64_t)t * run + j;
    const uint64_t x = e >= lead ? span[e - lead] : 0;
    c = zshift(Zs, c) ^ x;
  }
  v[t] = c;
  __syncthreads();
  for (int l = 0; (1 << l) < kFoldThreads; l++) {
    uint64_t r = 0;
    const bool act = (t & ((2 << l) - 1)) == 0;
    if (act) r = zshift(g_crc_z + (size_t)(kCrcSpanLog + run_log + l) * 2048, v[t]) ^ v[t + (1 << l)];
    __syncthreads();
    if (act) v[t] = r;
    __syncthreads();
  }
  if (t == 0) {
    uint64_t c0 = v[0];  // crc0 of the main part; the < 16 tail bytes follow bytewise
    for (int64_t i = J.n_main[b]; i < n; i++)
      c0 = __ldg(g_crc_slice + ((c0 ^ J.data[b][i]) & 0xff)) ^ (c0 >> 8);
    uint64_t r = ~0ull;
    for (int j = 0; j < kCrcLevels; j++)
      if ((n >> j) & 1) r = zshift(g_crc_z + (size_t)j * 2048, r);
    *crc_out = r ^ c0 ^ ~0ull;
  }
}

static int64_t crc_spans(int64_t n) {
  const int64_t c = (n + (int64_t(1) << kCrcSpanLog) - 1) >> kCrcSpanLog;
  return c ? c : 1;
}

size_t crc_ws(int64_t n) { return sizeof(uint64_t) * (size_t)(crc_spans(n) + 8); }

size_t crc_ws_many(const int64_t* n, int count) {
  size_t s = 8;
  for (int i = 0; i < count; i++) s += (size_t)crc_spans(n[i]);
  return sizeof(uint64_t) * s;
}

// CRC-64/XZ of `count` device buffers in two launches; crc_out[i] (device)
int launch_crc64_many(const uint8_t* const* data, const int64_t* n, int count, uint64_t* crc_out,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
  if (count < 0) return NBZG_BAD_ARG;
  if (count == 0) return NBZG_OK;
  if (int rc = upload_tables()) return rc;
  uint64_t* span = reinterpret_cast<uint64_t*>(ws);
  for (int c0 = 0; c0 < count; c0 += kCrcMax) {
    const int cnt = count - c0 < kCrcMax ? count - c0 : kCrcMax;
    if (ws_bytes < crc_ws_many(n + c0, cnt)) return NBZG_BAD_ARG;
    CrcJobs J;
    J.count = cnt;
    J.span0[0] = 0;
    for (int i = 0; i < cnt; i++) {
      const int64_t ni = n[c0 + i];
      if (ni < 0 || (ni >> kCrcLevels)) return NBZG_BAD_ARG;
      // the main part ends at the last 16-byte-aligned address of the buffer
      int64_t tail = (int64_t)((reinterpret_cast<uintptr_t>(data[c0 + i]) + (uint64_t)ni) & 15);
      if (tail > ni) tail = ni;
      const int64_t nm = ni - tail;
      const int64_t C = crc_spans(nm);
      int run_log = 0;
      while ((int64_t(kFoldThreads) << run_log) < C) run_log++;
      // the fold tree's top level is Z_{2^(span_log + run_log + 9)}
      if (kCrcSpanLog + run_log + 9 >= kCrcLevels) return NBZG_BAD_ARG;
      J.data[i] = data[c0 + i];
      J.n[i] = ni;
      J.n_main[i] = nm;
      J.pad[i] = (C << kCrcSpanLog) - nm;
      J.span0[i + 1] = J.span0[i] + C;
      J.out[i] = crc_out + c0 + i;
      J.run_log[i] = run_log;
    }
    count_launch();
    const int64_t grid = std::min<int64_t>(J.span0[cnt], 4 * (int64_t)sm_count());
    crc_span_kernel<<<(unsigned)grid, kCrcThreads, 0, st>>>(J, span);
    count_launch();
    crc_fold_kernel<<<cnt, kFoldThreads, 0, st>>>(J, span);  // (next batch: stream-ordered)
  }
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

int launch_crc64(const uint8_t* data, int64_t n, uint64_t* crc_out, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  if (ws_bytes < crc_ws(n)) return NBZG_BAD_ARG;
  return launch_crc64_many(&data, &n, 1, crc_out, ws, ws_bytes, st);
}

}  // namespace nbzg
