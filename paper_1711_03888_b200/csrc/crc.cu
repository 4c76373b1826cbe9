// crc.cu -- CRC-64/XZ of device buffers (_kernels.py:954-994: reflected
// ECMA-182 polynomial, init and xorout all ones).
//
// CRC is linear over GF(2):  crc(init, A||B) = Z_|B|(crc(init, A)) ^ crc(0, B)
// where Z_L is "feed L zero bytes" -- a 64x64 bit matrix, applied here as 8
// byte-sliced lookup tables.  Tables for Z_{2^j} (j = 0..40) are built on
// device by repeated squaring; 1 KiB blocks are CRC'd in parallel with init
// 0 (leading zero bytes do not change a zero-init CRC, so the stream is
// front-padded to a power-of-two number of blocks) and reduced pairwise in
// log2(blocks) levels; finally crc = Z_n(~0) ^ crc0 ^ ~0.
#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

constexpr int kCrcLevels = 41;           // Z_{2^j}, j = 0..40 bytes
constexpr int kCrcBlockLog = 10;         // 1 KiB blocks
constexpr uint64_t kPoly = 0xC96C5795D7870F42ull;

NBZG_DEV uint64_t zshift(const uint64_t* T, uint64_t v) {  // T: [8][256]
  uint64_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) r ^= T[j * 256 + ((v >> (8 * j)) & 0xff)];
  return r;
}

__global__ void crc_tables_kernel(uint64_t* tabs, uint64_t* base_tab) {
  __shared__ uint64_t tbl[256];
  const int tid = threadIdx.x;
  if (tid < 256) {
    uint64_t c = tid;
    for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
    tbl[tid] = c;
    base_tab[tid] = c;
  }
  __syncthreads();
  // level 0: one zero byte
  for (int e = tid; e < 2048; e += blockDim.x) {
    int j = e >> 8, b = e & 255;
    uint64_t v = (uint64_t)b << (8 * j);
    tabs[e] = (v >> 8) ^ tbl[v & 0xff];
  }
  __syncthreads();
  for (int L = 1; L < kCrcLevels; L++) {
    const uint64_t* P = tabs + (size_t)(L - 1) * 2048;
    uint64_t* Q = tabs + (size_t)L * 2048;
    for (int e = tid; e < 2048; e += blockDim.x) {
      int j = e >> 8, b = e & 255;
      uint64_t v = (uint64_t)b << (8 * j);
      Q[e] = zshift(P, zshift(P, v));
    }
    __syncthreads();
  }
}

// crc0 (init 0, no xorout) of 1 KiB block i of the front-padded stream
__global__ void crc_blocks_kernel(const uint8_t* data, int64_t n, int64_t pad, int64_t nb,
                                  const uint64_t* base_tab, uint64_t* out) {
  __shared__ uint64_t tbl[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tbl[i] = base_tab[i];
  __syncthreads();
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int64_t s = (b << kCrcBlockLog) - pad, e = s + (1 << kCrcBlockLog);
  if (s < 0) s = 0;
  if (e > n) e = n;
  uint64_t crc = 0;
  for (int64_t i = s; i < e; i++) crc = tbl[(crc ^ data[i]) & 0xff] ^ (crc >> 8);
  out[b] = crc;
}

// one tree level: out[i] = Z_{2^(level+10)}(in[2i]) ^ in[2i+1]
__global__ void crc_combine_kernel(const uint64_t* in, uint64_t* outv, int64_t npairs,
                                   const uint64_t* T) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npairs) outv[i] = zshift(T, in[2 * i]) ^ in[2 * i + 1];
}

__global__ void crc_final_kernel(const uint64_t* root, const uint64_t* tabs, int64_t n,
                                 uint64_t* crc_out) {
  if (threadIdx.x != 0) return;
  uint64_t r = ~0ull;
  for (int j = 0; j < kCrcLevels; j++)
    if ((n >> j) & 1) r = zshift(tabs + (size_t)j * 2048, r);
  *crc_out = r ^ *root ^ ~0ull;
}

size_t crc_ws(int64_t n) {
  int64_t nb = (n + (1 << kCrcBlockLog) - 1) >> kCrcBlockLog;
  int64_t np2 = 1;
  while (np2 < nb) np2 <<= 1;
  return sizeof(uint64_t) * ((size_t)kCrcLevels * 2048 + 256 + 2 * (size_t)np2 + 8);
}

int launch_crc64(const uint8_t* data, int64_t n, uint64_t* crc_out, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  if (n < 0 || (n >> kCrcLevels)) return NBZG_BAD_ARG;
  if (ws_bytes < crc_ws(n)) return NBZG_BAD_ARG;
  uint64_t* tabs = reinterpret_cast<uint64_t*>(ws);
  uint64_t* base_tab = tabs + (size_t)kCrcLevels * 2048;
  uint64_t* bufA = base_tab + 256;
  int64_t nb = (n + (1 << kCrcBlockLog) - 1) >> kCrcBlockLog;
  if (nb == 0) nb = 1;
  int64_t np2 = 1;
  while (np2 < nb) np2 <<= 1;
  uint64_t* bufB = bufA + np2;
  count_launch();
  crc_tables_kernel<<<1, 1024, 0, st>>>(tabs, base_tab);
  // front padding: leading (np2 - nb) zero blocks + `pad` zero bytes
  int64_t pad = (np2 << kCrcBlockLog) - n;
  count_launch();
  crc_blocks_kernel<<<(unsigned)((np2 + 255) / 256), 256, 0, st>>>(data, n, pad, np2, base_tab,
                                                                   bufA);
  uint64_t* in = bufA;
  uint64_t* out = bufB;
  int level = kCrcBlockLog;
  for (int64_t cnt = np2; cnt > 1; cnt >>= 1, level++) {
    int64_t npairs = cnt >> 1;
    count_launch();
    crc_combine_kernel<<<(unsigned)((npairs + 255) / 256), 256, 0, st>>>(
        in, out, npairs, tabs + (size_t)level * 2048);
    uint64_t* t = in;
    in = out;
    out = t;
  }
  count_launch();
  crc_final_kernel<<<1, 32, 0, st>>>(in, tabs, n, crc_out);
  return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR;
}

}  // namespace nbzg
