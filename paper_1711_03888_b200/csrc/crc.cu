// crc.cu -- CRC-64/XZ of device buffers (_kernels.py:954-994: reflected
// ECMA-182 polynomial, init and xorout all ones).
//
// CRC is linear over GF(2):  crc0(A||B) = Z_|B|(crc0(A)) ^ crc0(B), where
// crc0 is the zero-init, no-xorout CRC and Z_L ("feed L zero bytes") is a
// 64x64 bit matrix, applied as 8 byte-sliced lookup tables.  Leading zero
// bytes do not change crc0, so the stream is front-padded (virtually) to a
// whole number of 512 KiB CTA spans:
//   K1 crc_span_kernel: each thread CRCs a 2 KiB block (slicing-by-16 from a
//      32 KiB shared table, 16-byte loads), the CTA folds its 256 blocks in a
//      shuffle / shared-memory tree -> crc0 of its span;
//   K2 crc_fold_kernel: one CTA folds the span values (sequential runs, then
//      a tree) and applies  crc = Z_n(~0) ^ crc0 ^ ~0.
// The tables (slicing and Z_{2^j}, j = 0..40) are built once on the host and
// uploaded once per device.  HBM-bound: one read of the data.
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
  int64_t n[kCrcMax];
  int64_t pad[kCrcMax];
  int64_t span0[kCrcMax + 1];  // first span (CTA) of each buffer; span0[count] = total
  uint64_t* out[kCrcMax];
  int run_log[kCrcMax];
  int count;
};

// crc0 of each 512 KiB span of each front-padded stream (pad zero bytes,
// then data[0, n)).
__global__ void __launch_bounds__(kCrcThreads) crc_span_kernel(CrcJobs J, uint64_t* span_out) {
  __shared__ uint64_t T[16 * 256];
  __shared__ uint64_t wsum[kCrcThreads / 32];
  for (int i = threadIdx.x; i < 16 * 256; i += kCrcThreads) T[i] = g_crc_slice[i];
  int b = 0;
  while (b + 1 < J.count && (int64_t)blockIdx.x >= J.span0[b + 1]) b++;
  const uint8_t* data = J.data[b];
  const int64_t n = J.n[b], pad = J.pad[b];
  __syncthreads();
  const int64_t g = ((int64_t)blockIdx.x - J.span0[b]) * kCrcThreads + threadIdx.x;
  int64_t s = (g << kCrcBlockLog) - pad, e = s + (1 << kCrcBlockLog);
  if (s < 0) s = 0;  // leading virtual zeros leave crc0 at 0
  if (e > n) e = n;
  if (e < s) e = s;  // block entirely inside the padding
  uint64_t crc = 0;
  // unaligned head, 16-byte body, tail
  while (s < e && ((reinterpret_cast<uintptr_t>(data) + s) & 15)) {
    crc = T[(crc ^ data[s]) & 0xff] ^ (crc >> 8);
    s++;
  }
  const uint4* q = reinterpret_cast<const uint4*>(data + s);
  const int64_t nq = (e - s) >> 4;
  auto step = [&](const uint4 d) {
    const uint64_t lo = (((uint64_t)d.y << 32) | d.x) ^ crc;
    const uint64_t hi = ((uint64_t)d.w << 32) | d.z;
    uint64_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) r ^= T[(15 - k) * 256 + ((lo >> (8 * k)) & 0xff)];
#pragma unroll
    for (int k = 0; k < 8; k++) r ^= T[(7 - k) * 256 + ((hi >> (8 * k)) & 0xff)];
    crc = r;
  };
  int64_t i = 0;
  for (; i + 4 <= nq; i += 4) {
    const uint4 d0 = __ldg(q + i), d1 = __ldg(q + i + 1), d2 = __ldg(q + i + 2),
                d3 = __ldg(q + i + 3);
    step(d0);
    step(d1);
    step(d2);
    step(d3);
  }
  for (; i < nq; i++) step(__ldg(q + i));
  for (s += nq << 4; s < e; s++) crc = T[(crc ^ data[s]) & 0xff] ^ (crc >> 8);

  // fold the CTA's 256 blocks: warp tree, then the 8 warp values
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < 5; l++) {
    const uint64_t right = __shfl_down_sync(0xffffffffu, crc, 1 << l);
    const uint64_t shifted = zshift(g_crc_z + (size_t)(kCrcBlockLog + l) * 2048, crc);
    if ((lane & ((2 << l) - 1)) == 0) crc = shifted ^ right;
  }
  if (lane == 0) wsum[warp] = crc;
  __syncthreads();
  if (warp == 0) {
    crc = lane < kCrcThreads / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int l = 0; l < 3; l++) {
      const uint64_t right = __shfl_down_sync(0xffffffffu, crc, 1 << l);
      const uint64_t shifted = zshift(g_crc_z + (size_t)(kCrcBlockLog + 5 + l) * 2048, crc);
      if ((lane & ((2 << l) - 1)) == 0) crc = shifted ^ right;
    }
    if (lane == 0) span_out[blockIdx.x] = crc;
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
    uint64_t r = ~0ull;
    for (int j = 0; j < kCrcLevels; j++)
      if ((n >> j) & 1) r = zshift(g_crc_z + (size_t)j * 2048, r);
    *crc_out = r ^ v[0] ^ ~0ull;
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
      const int64_t C = crc_spans(ni);
      int run_log = 0;
      while ((int64_t(kFoldThreads) << run_log) < C) run_log++;
      // the fold tree's top level is Z_{2^(span_log + run_log + 9)}
      if (kCrcSpanLog + run_log + 9 >= kCrcLevels) return NBZG_BAD_ARG;
      J.data[i] = data[c0 + i];
      J.n[i] = ni;
      J.pad[i] = (C << kCrcSpanLog) - ni;
      J.span0[i + 1] = J.span0[i] + C;
      J.out[i] = crc_out + c0 + i;
      J.run_log[i] = run_log;
    }
    count_launch();
    crc_span_kernel<<<(unsigned)J.span0[cnt], kCrcThreads, 0, st>>>(J, span);
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
