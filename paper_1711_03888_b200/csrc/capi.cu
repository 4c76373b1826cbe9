#include <cstdio>
#include <cstdlib>
// capi.cu -- the extern "C" boundary (include/nbzg.h): argument validation,
// workspace carving and kernel sequencing.  Process-wide state is limited to
// mutex-guarded caches (per-device shared-memory attributes and SM counts)
// and the opt-in diagnostics (launch counter, event trace).
#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

#include "nbzg_internal.cuh"
#include "plan.h"

namespace nbzg {

int launch_rindex_keys(const float* x, const float* y, const float* z, int64_t n,
                       const double* bounds3, int64_t S, uint64_t* keys, uint8_t* seg_bits,
                       uint32_t* status, cudaStream_t st);
int launch_prx_order(const uint64_t* keys, int64_t n, int64_t S, const uint8_t* seg_bits, int ig,
                     int64_t* order, cudaStream_t st);
int launch_order_expand(const uint16_t* perm, int64_t n, int64_t tile, int64_t* order,
                        cudaStream_t st);
int launch_codebook_impl(const uint32_t* hist, int64_t nbins, uint32_t* sym, uint8_t* len,
                         uint64_t* lut, uint32_t* scratch, nbzg_meta* meta, int64_t n,
                         int64_t nchunks, int single_field, cudaStream_t st,
                         uint32_t* twin = nullptr, uint8_t* tlen8 = nullptr, int f0 = 0,
                         int nf = 6, int v1 = 0);
int launch_huffman_lengths(const uint32_t* counts, int64_t k, uint8_t* lengths, uint32_t* scr,
                           uint32_t* status, cudaStream_t st);
int launch_huff_encode_raw(const uint16_t* syms, int64_t n, const uint64_t* lut, uint8_t* out,
                           uint32_t* chunk_bits, uint64_t* lb, uint32_t* tickets,
                           cudaStream_t st);
size_t crc_ws(int64_t n);
size_t crc_ws_many(const int64_t* n, int count);
int launch_crc64_many(const uint8_t* const* data, const int64_t* n, int count, uint64_t* crc_out,
                      void* ws, size_t ws_bytes, cudaStream_t st);
int launch_crc64(const uint8_t* data, int64_t n, uint64_t* crc_out, void* ws, size_t ws_bytes,
                 cudaStream_t st);

size_t decompress_ws(int nf, int64_t n, int64_t nbins);
int launch_huff_decode_hook(const uint8_t* bits, uint64_t total, int64_t n, int min_len,
                            int max_len, const uint64_t* first_code, const uint32_t* counts,
                            const uint32_t* first_idx, const uint32_t* ss, uint32_t* out,
                            uint32_t* status, cudaStream_t st);
int launch_deinterleave3(const uint64_t* keys, int64_t n, int64_t* x, int64_t* y, int64_t* z,
                         cudaStream_t st);

// ---- launch counter and event trace (diagnostics for bench.py; the trace is
// off unless nbzg_trace_enable(1) is called)
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct TraceMark {
  const char* name;
  cudaEvent_t ev;
};
static std::mutex g_tmu;
static bool g_trace_on = false;
static std::vector<TraceMark> g_marks;
static std::vector<cudaEvent_t> g_pool;

void trace_mark(const char* name, cudaStream_t st) {
  static const int dbg = getenv("NBZG_DEBUG_SYNC") ? 1 : 0;  // debugging aid
  if (dbg && name) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "nbzg: %s failed: %s\n", name, cudaGetErrorString(e));
  }
  if (!g_trace_on) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  if (g_marks.size() == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  cudaEvent_t e = g_pool[g_marks.size()];
  cudaEventRecord(e, st);
  g_marks.push_back({name, e});
}

// SM count of the current device (cached per device)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  if (dev >= 64) {
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c > 0 ? c : 148;
  }
  int c = cache[dev].load(std::memory_order_relaxed);
  if (c <= 0) {
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    if (c <= 0) c = 148;
    cache[dev].store(c, std::memory_order_relaxed);
  }
  return c;
}

void smem_attr(const void* func, int bytes) {
  struct Done {
    int dev;
    const void* func;
    int bytes;
  };
  static std::mutex mu;
  static std::vector<Done> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const Done& d : done)
    if (d.dev == dev && d.func == func && d.bytes >= bytes) return;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
      cudaSuccess)
    done.push_back({dev, func, bytes});
}

static inline size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

void plan_shape(Plan& p, int64_t n, int sorted, int64_t ic, int64_t S, int fmt) {
  p.n = n;
  p.fmt = fmt;
  p.sorted = sorted;
  p.S = S;
  p.large = sorted && S > kTileMax;
  if (sorted && !p.large) {
    int64_t spt = S >= kTileMax ? 1 : kTileMax / S;
    p.tile = spt * S;
  } else {
    p.tile = kTileMax;
  }
  p.ntiles = (n + p.tile - 1) / p.tile;
  p.nseg = sorted ? (n + S - 1) / S : 0;
  p.nchunks = (n + kChunk - 1) / kChunk;
  p.nbins = fmt == 1 ? ic + 1 : ic;  // v1 codes span [0, 2 half]; v2 [0, 2 half - 1]
  p.half = (int)(ic / 2);
  p.v1_stride = (n + 3) & ~int64_t(3);
  // Huffman's mean length is below log2(k) + 1 <= 18 bits for k <= 2^16 + 1
  p.v1_wstride = fmt == 1 ? (int64_t)((n * 18 + 31) / 32 + 16) : 0;
}

size_t plan_workspace(Plan& p, void* base) {
  uint8_t* b = reinterpret_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) -> uint8_t* {
    uint8_t* r = b ? b + off : nullptr;
    off += al256(bytes);
    return r;
  };
  const int64_t cs = (p.n + 7) & ~int64_t(7);
  p.minmax = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 12));
  p.codes = reinterpret_cast<uint16_t*>(take(sizeof(uint16_t) * 6 * cs));
  p.hist = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * p.nbins));
  p.cb_sym = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * p.nbins));
  p.cb_len = reinterpret_cast<uint8_t*>(take(6 * p.nbins));
  p.lut = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 6 * p.nbins));
  p.enc_win = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * kEncWin));
  p.enc_len8 = reinterpret_cast<uint8_t*>(take(6 * (size_t)p.nbins));
  p.enc_boff = reinterpret_cast<uint64_t*>(
      take(sizeof(uint64_t) * 6 * ((size_t)p.nchunks + 1) +
           sizeof(uint32_t) * 6 * (33 * (size_t)p.nchunks)));
  p.cb_scratch = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * 5 * p.nbins));
  p.lb = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 12 * (p.nchunks + 1)));
  p.counters = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 64));
  p.tile_flags = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * (p.ntiles + 1)));
  p.seg_mm = reinterpret_cast<float*>(take(sizeof(float) * 6 * ((size_t)p.nseg + 1)));
#ifdef NBZG_CS_SPLIT
  if (p.sorted) {
    p.keys16 = reinterpret_cast<uint16_t*>(take(sizeof(uint16_t) * ((size_t)p.n + 8)));
    p.seg_cw = reinterpret_cast<uint8_t*>(take((size_t)p.nseg + 16));
  }
#endif
  if (p.large) p.large_ws = take(large_ws(p.n, p.nseg));
  if (p.fmt == 1) {
    const size_t xs = (size_t)p.v1_stride, nc = (size_t)p.nchunks;
    p.v1_xsort = p.sorted && !p.large ? reinterpret_cast<float*>(take(sizeof(float) * 6 * xs)) : nullptr;
    p.v1_codes = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * xs));
    p.v1_esc = reinterpret_cast<float*>(take(sizeof(float) * 6 * xs));
    p.v1_esc_cnt = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * nc));
    p.v1_cbits = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * nc));
    p.v1_boff = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 6 * (nc + 1)));
    p.v1_eoff = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 6 * (nc + 1)));
    p.v1_words = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 6 * (size_t)p.v1_wstride));
  }
  return off;
}

size_t decompress_ws(int nf, int64_t n, int64_t nbins);  // decode.cu

}  // namespace nbzg

using namespace nbzg;

namespace nbzg {
int launch_decompress(const DField* fields, int nf, int64_t n, int64_t interval_count, void* ws,
                      size_t ws_bytes, uint32_t* status, cudaStream_t st);
__global__ void ord_decode_kernel(uint32_t* m) {
  int i = threadIdx.x;
  if (i < 12) m[i] = __float_as_uint(ord2f(m[i]));
}
}  // namespace nbzg

static int cuda_status() { return cudaGetLastError() == cudaSuccess ? NBZG_OK : NBZG_CUDA_ERROR; }

#ifndef NBZG_SZ_GROUPS
#define NBZG_SZ_GROUPS 2
#endif
// The SZ stages in G field groups so the codebook -- single-CTA Huffman
// builds that leave the rest of the GPU idle -- and the encoding of one
// group overlap the quantisation of the next.  All quantise launches go on
// the caller's stream; group g's codebook, layout and encode follow on its
// own side stream as soon as Q(g) is done (layouts in group order: each
// appends to the arena after the previous group's payloads); the caller's
// stream then waits for every group.  Side streams and events are per call
// (no shared mutable state).
static int sz_stages_split(Plan& p, cudaStream_t st) {
  constexpr int G = NBZG_SZ_GROUPS;
  static_assert(G == 2 || G == 3 || G == 6, "field groups: 2, 3 or 6");
  constexpr int per = 6 / G;
  cudaStream_t sd[G];
  cudaEvent_t eq[G], el[G], ee[G];
  int made = 0;
  int rc = NBZG_OK;
  for (; made < G; made++) {
    if (cudaStreamCreateWithFlags(&sd[made], cudaStreamNonBlocking) != cudaSuccess) break;
    cudaEventCreateWithFlags(&eq[made], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&el[made], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ee[made], cudaEventDisableTiming);
  }
  if (made < G) rc = NBZG_CUDA_ERROR;
#ifndef NBZG_SZ_REVERSE
#define NBZG_SZ_REVERSE 0
#endif
  // group order: REVERSE puts the velocities (large alphabets: the slow
  // codebooks) first, so the last -- exposed -- codebook is a coordinate one
  auto f0_of = [&](int g) { return (NBZG_SZ_REVERSE ? G - 1 - g : g) * per; };
  for (int g = 0; g < G && !rc; g++) {
    if ((rc = launch_quantize(p, st, f0_of(g), per))) break;
    cudaEventRecord(eq[g], st);
  }
  if (!rc) trace_mark("quantize", st);
  for (int g = 0; g < G && !rc; g++) {
    cudaStreamWaitEvent(sd[g], eq[g], 0);
    if ((rc = launch_codebook(p, sd[g], f0_of(g), per))) break;
    if (g > 0) cudaStreamWaitEvent(sd[g], el[g - 1], 0);
    if ((rc = launch_layout(p, sd[g], f0_of(g), per, g == 0))) break;
    cudaEventRecord(el[g], sd[g]);
    if ((rc = launch_encode(p, sd[g], f0_of(g), per))) break;
    cudaEventRecord(ee[g], sd[g]);
  }
  for (int g = 0; g < made; g++) {
    if (!rc) cudaStreamWaitEvent(st, ee[g], 0);
  }
  if (!rc) trace_mark("encode", st);
  for (int g = 0; g < made; g++) {
    cudaEventDestroy(eq[g]);
    cudaEventDestroy(el[g]);
    cudaEventDestroy(ee[g]);
    cudaStreamDestroy(sd[g]);
  }
  return rc ? rc : cuda_status();
}

extern "C" {

const char* nbzg_version(void) { return "nbzg 0.1.0 sm_100a"; }

unsigned long long nbzg_launch_count(void) { return g_launches.load(); }

int nbzg_trace_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_trace_on = on != 0;
  g_marks.clear();
  return NBZG_OK;
}

int nbzg_trace_read(char* names, int name_stride, float* ms, int max) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (g_marks.empty()) return 0;
  cudaEventSynchronize(g_marks.back().ev);
  int cnt = 0;
  for (size_t i = 1; i < g_marks.size() && cnt < max; i++) {
    if (!g_marks[i].name) continue;
    float t = 0.f;
    cudaEventElapsedTime(&t, g_marks[i - 1].ev, g_marks[i].ev);
    std::strncpy(names + (size_t)cnt * name_stride, g_marks[i].name, name_stride - 1);
    names[(size_t)cnt * name_stride + name_stride - 1] = 0;
    ms[cnt] = t;
    cnt++;
  }
  return cnt;
}

int nbzg_device_sm_count(void) { return sm_count(); }

size_t nbzg_compress_workspace_size(int64_t n, int32_t sorted, int64_t interval_count,
                                    int64_t segment_size) {
  return nbzg_compress_workspace_size_fmt(n, sorted, interval_count, segment_size, 2);
}

size_t nbzg_compress_workspace_size_fmt(int64_t n, int32_t sorted, int64_t interval_count,
                                        int64_t segment_size, int32_t fmt) {
  Plan p;
  plan_shape(p, n, sorted, interval_count, segment_size < 1 ? 1 : segment_size,
             fmt == 1 ? 1 : 2);
  return plan_workspace(p, nullptr);
}

size_t nbzg_compress_arena_bound(int64_t n, int64_t interval_count) {
  int lg = 1;
  while ((int64_t(1) << lg) < interval_count) lg++;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t k = interval_count < n ? interval_count : n;
  // Huffman average length < log2(k) + 1, so bits < n * (lg + 1); escapes <= n
  size_t per = 8 + 5 * (size_t)k + 8 + 4 * (size_t)nchunks + 4 +
               4 * (((size_t)n * (lg + 1) + 31) / 32) + 4 * (size_t)n + 16;
  return 6 * per + 256;
}

int nbzg_compress(const nbzg_compress_args* a, void* stream) {
  NvtxScope range_call("nbzg_compress");
  if (!a) return NBZG_BAD_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a->n < 0 || a->n >= (int64_t(1) << 32) - 1) return NBZG_UNSUPPORTED;
  if (a->interval_count < 2 || (a->interval_count & 1) || a->interval_count > 65536)
    return NBZG_UNSUPPORTED;
  if (a->segment_size < 1 || a->ignored_groups < 0) return NBZG_BAD_ARG;
  const bool large = a->sorted && a->segment_size > kTileMax;
  if (large && (a->cpc || a->rindex_variant == 2)) return NBZG_UNSUPPORTED;
  for (int f = 0; f < 6; f++) {
    if (a->n > 0 && (!a->fields[f] || (reinterpret_cast<uintptr_t>(a->fields[f]) & 15)))
      return NBZG_BAD_ARG;
    if (a->bound_kind[f] != 0 && a->bound_kind[f] != 1) return NBZG_BAD_ARG;
    if (!(a->bound_value[f] > 0)) return NBZG_BAD_ARG;
  }
  const int fmt = a->fmt == 0 ? 2 : a->fmt;
  if (fmt != 1 && fmt != 2) return NBZG_BAD_ARG;
  if (fmt == 1 && (a->predictor != 0 || a->cpc != 0)) return NBZG_UNSUPPORTED;
  Plan p;
  plan_shape(p, a->n, a->sorted, a->interval_count, a->segment_size, fmt);
  p.ig = a->ignored_groups;
  if (a->rindex_variant < 0 || a->rindex_variant > 2) return NBZG_BAD_ARG;
  p.variant = a->rindex_variant;
  if (a->predictor < 0 || a->predictor > 1 || (a->predictor == 1 && a->sorted))
    return NBZG_UNSUPPORTED;
  p.predictor = a->predictor;
  if (a->cpc < 0 || a->cpc > 2 || (a->cpc && (!a->sorted || a->rindex_variant != 0)))
    return NBZG_BAD_ARG;
  p.cpc = a->cpc;
  if (p.cpc) {
    p.ig = 0;  // full-key sort (pipeline.py:464: k = 0 when the mode stores minima)
    p.minima = a->seg_minima;
    p.sz_skip = a->sz_skip & 63u;
    if (a->n > 0 && !p.minima) return NBZG_BAD_ARG;
  }
  for (int f = 0; f < 6; f++) {
    p.f[f] = a->fields[f];
    p.bound_kind[f] = a->bound_kind[f];
    p.bound_value[f] = a->bound_value[f];
  }
  if (a->workspace_bytes < plan_workspace(p, nullptr)) return NBZG_BAD_ARG;
  if (a->arena_bytes < nbzg_compress_arena_bound(a->n, a->interval_count)) return NBZG_BAD_ARG;
  if (!a->meta || (a->sorted && a->n > 0 && ((large ? !a->order32 : !a->perm) || !a->seg_bits)))
    return NBZG_BAD_ARG;
  plan_workspace(p, a->workspace);
  p.meta = a->meta;
  p.perm = a->perm;
  p.order32 = a->order32;
  p.seg_bits = a->seg_bits;
  p.arena = a->arena;
  p.arena_bytes = a->arena_bytes;
  int rc;
  if (a->phase < 0 || a->phase > 4) return NBZG_BAD_ARG;
  if (a->phase >= 3 && (p.fmt != 2 || p.cpc || p.predictor)) return NBZG_UNSUPPORTED;
  trace_mark(nullptr, st);
  if (a->phase == 4) {  // resume a phase-3 call: encode only (payload sizes are final)
    NvtxScope r("K5 encode");
    if (p.n == 0) return cuda_status();
    if (p.large) {  // the SZ stages read the sorted copies, as in phase 3
      large_fields(p);
      p.sorted = 0;
    }
    if ((rc = launch_encode(p, st))) return rc;
    trace_mark("encode", st);
    return cuda_status();
  }
  // sorted mode with 3-field keys: K1 walks whole segments and also leaves
  // each segment's key-field min/max, so K2 reads the coordinates once
  const bool segmm = p.sorted && !p.large && p.variant != 2 && p.n > 0 && p.S % 4 == 0;
  {
    NvtxScope range("K1 minmax + resolve");
    if (a->phase == 2) {
      // K1 ran in phase 1 (its segment min/max are still in the workspace);
      // the global min/max replace the shard's
      for (int i = 0; i < 12; i++)
        if (a->h_minmax[i] != a->h_minmax[i]) return NBZG_BAD_ARG;  // NaN
      if ((rc = launch_minmax_set(a->h_minmax, p.minmax, st))) return rc;
    } else {
      if ((rc = segmm ? launch_minmax_seg(p, st) : launch_minmax6(p.f, p.n, p.minmax, st)))
        return rc;
    }
    if (!segmm) p.seg_mm = nullptr;
    trace_mark("minmax6", st);
    if ((rc = launch_resolve(p, st))) return rc;
  }
  trace_mark("resolve", st);
  if (p.n == 0 || a->phase == 1) return cuda_status();
  if (p.large) {
    // one device-wide radix sort, then the SZ stages on sorted copies as on
    // an unsorted snapshot (rlarge.cu)
    NvtxScope r("K2 rindex_sort (long segments)");
    bool stop = false;
    if ((rc = launch_rindex_large(p, st, stop))) return rc;
    trace_mark("rindex_sort", st);
    if (stop) return cuda_status();
    p.sorted = 0;
  } else if (p.sorted) {
    NvtxScope r("K2 rindex_sort");
    if ((rc = launch_rindex_sort(p, st))) return rc;
    trace_mark("rindex_sort", st);
  }
  NvtxScope range_sz("K3-K5 quantize / codebook / encode");
  if (p.sz_skip && (rc = launch_sz_skip(p, st))) return rc;
  if (p.fmt == 1) return launch_v1(p, st);
  if (a->phase != 3 && p.predictor == 0 && encode_uses_tpc(p)) return sz_stages_split(p, st);
  if ((rc = launch_quantize(p, st))) return rc;
  trace_mark("quantize", st);
  if ((rc = launch_codebook(p, st))) return rc;
  trace_mark("codebook", st);
  if ((rc = launch_layout(p, st))) return rc;
  trace_mark("layout", st);
  if (a->phase == 3) return cuda_status();  // sizes only: meta holds every payload length
  if ((rc = launch_encode(p, st))) return rc;
  trace_mark("encode", st);
  return cuda_status();
}

size_t nbzg_decompress_workspace_size(int64_t n, int64_t interval_count, int32_t nfields) {
  return decompress_ws(nfields, n, interval_count + 1);
}

int nbzg_decompress(const nbzg_decompress_args* a, void* stream) {
  NvtxScope range_call("nbzg_decompress");
  if (!a || a->nfields < 0 || a->nfields > 6 || a->n < 0) return NBZG_BAD_ARG;
  if (a->nfields == 0 || a->n == 0) return NBZG_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DField f[6];
  for (int i = 0; i < a->nfields; i++) {
    const int kb = a->kind[i] & ~NBZG_KIND_LCF;
    if ((kb != 0 && kb != 3) || (a->kind[i] & ~(NBZG_KIND_LCF | 15))) return NBZG_BAD_ARG;
    if (!(a->bound[i] > 0)) return NBZG_BAD_ARG;
    f[i].payload = a->payload[i];
    f[i].payload_len = a->payload_len[i];
    f[i].kind = a->kind[i];
    f[i].bound = a->bound[i];
    f[i].twob = 2.0 * a->bound[i];
    f[i].inv = 1.0 / f[i].twob;
    f[i].inv32 = (float)f[i].inv;
    f[i].out = a->out[i];
  }
  // the status word is the caller's (zeroed by it): a preceding decode on
  // the same word (the CPC coordinate stream) keeps its failure
  trace_mark(nullptr, st);
  return launch_decompress(f, a->nfields, a->n, a->interval_count,
                           a->workspace, a->workspace_bytes, a->status, st);
}

int nbzg_minmax6(const float* const* h_fields, int64_t n, float* out12, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int f = 0; f < 6; f++)
    if (n > 0 && (reinterpret_cast<uintptr_t>(h_fields[f]) & 15)) return NBZG_BAD_ARG;
  uint32_t* mm = reinterpret_cast<uint32_t*>(out12);
  int rc = launch_minmax6(h_fields, n, mm, st);
  if (rc) return rc;
  count_launch();
  ord_decode_kernel<<<1, 32, 0, st>>>(mm);  // decode the order-preserving encoding
  return cuda_status();
}

}  // extern "C"

namespace nbzg {
__global__ void integerize_kernel(const float* x, int64_t n, double twob, double inv, float inv32,
                                  int64_t* out, uint32_t* status) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool fast;
  double k = lattice_index<true>(x[i], inv32, inv, twob, fast);
  if (!fast && fabs(__ddiv_rn((double)x[i], twob)) > kIntLimit)
    atomicCAS(status, 0u, (uint32_t)NBZG_BOUND_TOO_SMALL);
  out[i] = (int64_t)k;
}
}  // namespace nbzg

extern "C" {

int nbzg_integerize(const float* x, int64_t n, double bound, int64_t* ints, uint32_t* status_dev,
                    void* stream) {
  if (!(bound > 0)) return NBZG_BAD_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double twob = 2.0 * bound, inv = 1.0 / twob;
  if (n > 0) {
    count_launch();
    integerize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, twob, inv, (float)inv,
                                                                   ints, status_dev);
  }
  return cuda_status();
}

int nbzg_rindex_keys(const float* x, const float* y, const float* z, int64_t n,
                     const double* h_bounds3, int64_t segment_size, uint64_t* keys,
                     uint8_t* seg_bits, uint32_t* status_dev, void* stream) {
  if (segment_size < 1) return NBZG_BAD_ARG;
  return launch_rindex_keys(x, y, z, n, h_bounds3, segment_size, keys, seg_bits, status_dev,
                            reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_prx_order(const uint64_t* keys, int64_t n, int64_t segment_size, const uint8_t* seg_bits,
                   int32_t ignored_groups, int64_t* order, void* stream) {
  if (segment_size < 1 || ignored_groups < 0) return NBZG_BAD_ARG;
  return launch_prx_order(keys, n, segment_size, seg_bits, ignored_groups, order,
                          reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_order_expand(const uint16_t* perm, int64_t n, int64_t segment_size, int64_t* order,
                      void* stream) {
  if (segment_size < 1) return NBZG_BAD_ARG;
  Plan p;
  plan_shape(p, n, 1, 65536, segment_size);
  return launch_order_expand(perm, n, p.tile, order, reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_huffman_lengths(const uint32_t* sorted_counts, int64_t k, uint8_t* lengths,
                         void* workspace, size_t workspace_bytes, uint32_t* status_dev,
                         void* stream) {
  size_t np2 = 1;
  while ((int64_t)np2 < k) np2 <<= 1;
  if (k > 16384 && workspace_bytes < 12 * np2) return NBZG_BAD_ARG;
  return launch_huffman_lengths(sorted_counts, k, lengths, reinterpret_cast<uint32_t*>(workspace),
                                status_dev, reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_huffman_codebook(const uint32_t* hist, int64_t nbins, uint32_t* symbols, uint8_t* lengths,
                          uint64_t* lut, nbzg_meta* meta_out, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (nbins < 1 || nbins > 65536 || workspace_bytes < 20 * (size_t)nbins) return NBZG_BAD_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(meta_out, 0, sizeof(nbzg_meta), st);
  return launch_codebook_impl(hist, nbins, symbols, lengths, lut,
                              reinterpret_cast<uint32_t*>(workspace), meta_out, 1, 1, 0, st);
}

int nbzg_huff_encode(const uint16_t* syms, int64_t n, const uint64_t* lut, uint8_t* out,
                     uint32_t* chunk_bits, void* workspace, size_t workspace_bytes, void* stream) {
  int64_t nchunks = (n + kChunk - 1) / kChunk;
  if (workspace_bytes < 16 * (size_t)nchunks + 64) return NBZG_BAD_ARG;
  if (reinterpret_cast<uintptr_t>(out) & 3) return NBZG_BAD_ARG;
  uint64_t* lb = reinterpret_cast<uint64_t*>(workspace);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(lb + 2 * nchunks);
  return launch_huff_encode_raw(syms, n, lut, out, chunk_bits, lb, tickets,
                                reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_huff_decode(const uint8_t* data, uint64_t total_bits, int64_t n, int32_t min_len,
                     int32_t max_len, const uint64_t* h_first_code, const uint32_t* h_counts,
                     const uint32_t* h_first_idx, const uint32_t* sorted_syms, uint32_t* out,
                     uint32_t* status_dev, void* stream) {
  if (n < 0 || !h_first_code || !h_counts || !h_first_idx) return NBZG_BAD_ARG;
  return launch_huff_decode_hook(data, total_bits, n, min_len, max_len, h_first_code, h_counts,
                                 h_first_idx, sorted_syms, out, status_dev,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_deinterleave3(const uint64_t* keys, int64_t n, int64_t* x, int64_t* y, int64_t* z,
                       void* stream) {
  if (n < 0) return NBZG_BAD_ARG;
  return launch_deinterleave3(keys, n, x, y, z, reinterpret_cast<cudaStream_t>(stream));
}

size_t nbzg_crc64_workspace_size(int64_t n) { return crc_ws(n); }

size_t nbzg_crc64_many_workspace_size(const int64_t* h_n, int32_t count) {
  size_t best = 0;
  for (int c0 = 0; c0 < count; c0 += 8) {
    const size_t s = crc_ws_many(h_n + c0, count - c0 < 8 ? count - c0 : 8);
    best = s > best ? s : best;
  }
  return best ? best : 64;
}

int nbzg_crc64_many(const uint8_t* const* h_data, const int64_t* h_n, int32_t count,
                    uint64_t* crc_dev, void* workspace, size_t workspace_bytes, void* stream) {
  if (count < 0 || (count > 0 && (!h_data || !h_n))) return NBZG_BAD_ARG;
  return launch_crc64_many(h_data, h_n, count, crc_dev, workspace, workspace_bytes,
                           reinterpret_cast<cudaStream_t>(stream));
}

int nbzg_crc64(const uint8_t* data, int64_t n, uint64_t* crc_dev, void* workspace,
               size_t workspace_bytes, void* stream) {
  return launch_crc64(data, n, crc_dev, workspace, workspace_bytes,
                      reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
