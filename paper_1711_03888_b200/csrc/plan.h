// plan.h -- host-side plan of one compress call: sizes and workspace carving.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nbzg.h"

namespace nbzg {

struct Plan {
  // problem
  int64_t n = 0;
  int sorted = 0;
  int64_t S = 16384;    // segment size
  int64_t tile = 0;     // particles per tile (whole segments, <= 16384)
  int64_t ntiles = 0;
  int64_t nseg = 0;
  int64_t nchunks = 0;  // ceil(n / 16384)
  int64_t nbins = 0;    // interval_count (codes 0 .. 2*half-1)
  int half = 0;
  int ig = 6;
  int variant = 0;      // RIndexVariant: 0 coord, 1 vel, 2 coord+vel
  int predictor = 0;    // 0 last value, 1 LCF (sz-lcf)
  int cpc = 0;          // 0; 1 sz-cpc2000; 2 cpc2000 (full keys, no clamp, minima)
  uint32_t sz_skip = 0; // fields without an SZ stream (CPC modes)
  int fmt = 2;          // 2: v2 SZ_DQ streams; 1: reference-readable SZ_FIELD streams (v1.cu)
  int64_t* minima = nullptr;  // 3 per segment (CPC)
  const float* f[6] = {};
  int bound_kind[6] = {};
  double bound_value[6] = {};
  // workspace
  uint32_t* minmax = nullptr;   // 12 ordered u32
  float* seg_mm = nullptr;      // [nseg][3][2] per-segment min/max of the key fields (from K1)
  uint16_t* keys16 = nullptr;   // [n] compacted R-index keys (split compact sort)
  uint8_t* seg_cw = nullptr;    // [nseg] their width per segment
  nbzg_meta* meta = nullptr;
  uint16_t* perm = nullptr;
  uint8_t* seg_bits = nullptr;
  uint16_t* codes = nullptr;    // 6*n
  uint32_t* hist = nullptr;     // 6*nbins
  uint32_t* cb_sym = nullptr;   // 6*nbins ascending symbols
  uint8_t* cb_len = nullptr;    // 6*nbins lengths by rank
  uint64_t* lut = nullptr;      // 6*nbins
  uint32_t* enc_win = nullptr;  // 6*kEncWin (word << 6 | len) of codes near the centre
  uint8_t* enc_len8 = nullptr;  // 6*nbins code length by symbol (chunk bit counts)
  uint64_t* enc_boff = nullptr; // 6*(32*nchunks+1) block bit offsets, then u32 block bits
  uint32_t* cb_scratch = nullptr;  // 6 * 4*nbins u32 (sort + queues, large-k path)
  uint64_t* lb = nullptr;       // 6*nchunks*2 look-back words
  uint32_t* counters = nullptr; // 64 u32 (tickets, flags)
  uint32_t* tile_flags = nullptr;  // ntiles (u64-key fallback tiles)
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0;
  // fmt 1 (v1.cu) buffers
  int64_t v1_stride = 0;        // per-field stride of the arrays below
  float* v1_xsort = nullptr;    // [6][stride] fields in sorted order (sorted modes)
  uint32_t* v1_codes = nullptr; // [6][stride]
  float* v1_esc = nullptr;      // [6][stride] chunk c's escapes from c * 16384
  uint32_t* v1_esc_cnt = nullptr;  // [6][nchunks]
  uint32_t* v1_cbits = nullptr;    // [6][nchunks]
  uint64_t* v1_boff = nullptr;     // [6][nchunks + 1]
  uint64_t* v1_eoff = nullptr;     // [6][nchunks + 1]
  uint32_t* v1_words = nullptr;    // [6][v1_wstride]
  int64_t v1_wstride = 0;
  // long segments (sorted, S > 16384: rlarge.cu)
  int large = 0;
  uint8_t* large_ws = nullptr;
  uint32_t* order32 = nullptr;  // [n] source index per sorted position
};

// one field of a decompress call (decode.cu)
struct DField {
  const uint8_t* payload;
  int64_t payload_len;
  int32_t kind;  // 3 = SZ_DQ (v2), 0 = SZ_FIELD (v1)
  double bound, twob, inv;
  float inv32;
  float* out;
};

size_t plan_workspace(Plan& p, void* base);  // carve (base may be null: size only)
void plan_shape(Plan& p, int64_t n, int sorted, int64_t interval_count, int64_t segment_size,
                int fmt = 2);

// kernel launchers (each enqueues on `st`)
int launch_minmax6(const float* const* f, int64_t n, uint32_t* minmax12, cudaStream_t st);
int launch_minmax_seg(const Plan& p, cudaStream_t st);
int launch_minmax_set(const float* h_minmax12, uint32_t* minmax12, cudaStream_t st);
int launch_resolve(const Plan& p, cudaStream_t st);
int launch_rindex_sort(const Plan& p, cudaStream_t st);
int launch_rindex_large(Plan& p, cudaStream_t st, bool& stop);
void large_fields(Plan& p);
size_t large_ws(int64_t n, int64_t nseg);
int launch_quantize(const Plan& p, cudaStream_t st, int f0 = 0, int nf = 6);
int launch_codebook(const Plan& p, cudaStream_t st, int f0 = 0, int nf = 6);
int launch_layout(const Plan& p, cudaStream_t st, int f0 = 0, int nf = 6, bool first = true);
int launch_encode(const Plan& p, cudaStream_t st, int f0 = 0, int nf = 6);
bool encode_uses_tpc(const Plan& p);
int launch_sz_skip(const Plan& p, cudaStream_t st);
int launch_v1(const Plan& p, cudaStream_t st);  // fmt 1: all SZ stages (v1.cu)

int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel,
// size): the attribute is per device, so a process-wide flag would leave a
// second GPU at the 48 KB default.  Thread-safe.
void smem_attr(const void* func, int bytes);

}  // namespace nbzg
