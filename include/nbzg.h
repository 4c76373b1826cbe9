/*
 * nbzg.h -- C ABI of the B200 (sm_100a) nbz compression path.
 *
 * Drop-in boundary for the reference package `nbz` (pure Python + numba,
 * /root/reference/pkg/src/nbz).  The reference's operator table is the flat
 * module `nbz._kernels`; its whole-path entry points are
 * `pipeline.compress` / `pipeline.decompress`.  Each function below cites
 * the reference interface it replaces.  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 *
 * Conventions (mirroring _kernels.py's calling convention):
 *   - every pointer argument is a DEVICE pointer unless named h_*;
 *   - the caller owns and pre-allocates every buffer (workspace sizes come
 *     from the *_workspace_size queries);
 *   - `stream` is a cudaStream_t passed as void*; every call is async on it
 *     and reentrant across streams and host threads: all per-call state lives
 *     in the caller's workspace; the only process-wide state is mutex-guarded
 *     (per-device kernel attributes / SM counts, the opt-in launch counter and
 *     event trace);
 *   - the return value is a status (NBZG_OK = 0); device-side failures
 *     (bound too small, invalid code, ...) are reported through the
 *     `status` word of the nbzg_meta block written by the call.
 */
#ifndef NBZG_H_
#define NBZG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NBZG_KIND_LCF = 16 };

enum {
  NBZG_OK = 0,
  NBZG_BOUND_TOO_SMALL = 1, /* quantize.py:123-126 -> BoundTooSmallError */
  NBZG_CODE_TOO_LONG = 2,   /* encode.py:215-216 -> EncodeError */
  NBZG_INVALID_CODE = 3,    /* _kernels.py:348-374 status 1 -> DecodeError */
  NBZG_TRUNCATED = 4,       /* status 2 / pipeline.py:213-214 -> DecodeError */
  NBZG_BAD_ARG = 5,         /* -> ValidationError */
  NBZG_CUDA_ERROR = 6,
  NBZG_UNSUPPORTED = 7,     /* parameter outside the GPU path's range */
  NBZG_BAD_STREAM = 8       /* malformed table / counts -> DecodeError */
};

/* Per-field resolved parameters and produced sizes. */
typedef struct nbzg_field_meta {
  double bound;        /* resolved absolute bound b (model.py:112-125); 0 if constant */
  double twob;         /* 2b   (_kernels.py:154) */
  double inv;          /* 1/(2b) (_kernels.py:155) */
  float inv32;         /* (float)inv, FP32 fast-path scale */
  float constant;      /* value of a constant field (pipeline.py:174-178) */
  float lo, hi;        /* exact f32 min / max (model.py:104-109) */
  uint32_t is_const;
  uint32_t k;          /* Huffman symbols in the table */
  uint32_t min_len, max_len;
  uint64_t n_esc;      /* escapes (code 0) */
  uint64_t total_bits; /* Huffman bitstream length */
  uint64_t payload_off;/* offset of this field's payload in the arena */
  uint64_t payload_len;
  uint64_t index_off;  /* payload-relative offset of u32 chunk_bits[] */
  uint64_t bits_off;   /* payload-relative offset of the bitstream (4-aligned) */
  uint64_t esc_off;    /* payload-relative offset of f32 escapes (4-aligned) */
} nbzg_field_meta;

typedef struct nbzg_meta {
  nbzg_field_meta f[6];
  uint32_t mask;       /* constant-field mask (bit f) */
  uint32_t status;     /* first device-side failure (NBZG_*), 0 if none */
  uint64_t arena_used; /* total payload bytes (sum of payload_len) */
  uint64_t nseg;       /* R-index segments (sorted mode) */
  uint64_t pad;
} nbzg_meta;

/* Whole-snapshot compress of Mode.SZ_LV (sorted=0) / Mode.SZ_LV_PRX (sorted=1).
 * Replaces pipeline.compress (pipeline.py:447-526) for these two modes.
 * Output: payloads of the v2 SZ_DQ streams laid out back to back in `arena`
 * (field order, constant fields skipped), `meta` (device), seg_bits[nseg]
 * (u8, sorted mode) and perm[n] (u16 tile-local source index of every sorted
 * position; the CompressResult.order sidecar, pipeline.py:146-149). */
typedef struct nbzg_compress_args {
  const float *fields[6]; /* device, n floats each */
  int64_t n;
  int32_t sorted;
  int32_t bound_kind[6];  /* 0 = absolute, 1 = value-range relative (model.py:79-101) */
  double bound_value[6];
  int64_t interval_count; /* Settings.interval_count (pipeline.py:79) */
  int64_t segment_size;   /* Settings.segment_size */
  int32_t ignored_groups; /* Settings.ignored_groups */
  int32_t rindex_variant; /* RIndexVariant (rindex.py:24-39): 0 coordinate keys (fields 0-2),
                             1 velocity keys (3-5), 2 coord+velocity keys (all six,
                             group width 6, 10-bit cap) */
  void *workspace;        /* nbzg_compress_workspace_size() bytes */
  size_t workspace_bytes;
  uint8_t *arena;         /* nbzg_compress_arena_bound() bytes */
  size_t arena_bytes;
  nbzg_meta *meta;        /* device */
  uint8_t *seg_bits;      /* device, ceil(n/segment_size) bytes (sorted) */
  uint16_t *perm;         /* device, n entries (sorted, segment_size <= 16384) */
  int32_t predictor;      /* 0 = last value (sz-lv, sz-lv-prx), 1 = LCF 2*prev - prev2
                             (Mode.SZ_LCF, _kernels.py:162-165; unsorted only) */
  int32_t cpc;            /* 0; 1 = sz-cpc2000, 2 = cpc2000 (full keys, no clamp, minima) */
  int64_t *seg_minima;    /* device, 3 x nseg (cpc) */
  uint32_t sz_skip;       /* bit f: no SZ stream for field f (cpc modes) */
  int32_t phase;          /* 0: the whole compress.  Sharded compress in two
                             calls with the same args and workspace: 1 = K1 only, this
                             shard's exact f32 min/max -> meta->f[i].lo / .hi; 2 = resume
                             with the GLOBAL min/max in h_minmax (all-gathered by the
                             caller), so bounds resolve as on the whole snapshot
                             (model.py:104-125) and K1 is not run twice.
                             3 = everything but the encoding: meta holds the exact
                             payload sizes (the `auto` mode compares two modes' sizes);
                             4 = resume a phase-3 call: encode only (same args,
                             workspace and arena).  Phases 3/4: fmt 2, SZ modes */
  float h_minmax[12];     /* phase 2: (lo, hi) of field 0..5, host values */
  int32_t fmt;            /* 0 or 2: v2 SZ_DQ streams (chunk-parallel, container 2);
                             1: reference-readable SZ_FIELD streams (container 1) -- the
                             reference's exact chain restarted by a forced escape every
                             16384 values; sz-lv / sz-lv-prx only.
                             Workspace: nbzg_compress_workspace_size_fmt(..., 1) */
  int32_t pad3;
  uint32_t *order32;      /* device, n entries: sorted mode with segment_size > 16384 (one
                             segment no longer fits a tile; rindex.py:155-229 has no size
                             cap) -- the global source index of every sorted position,
                             replacing perm.  Rindex variants 0/1, no cpc; one host
                             synchronisation (the radix pass count is data-dependent) */
} nbzg_compress_args;

size_t nbzg_compress_workspace_size(int64_t n, int32_t sorted, int64_t interval_count,
                                    int64_t segment_size);
size_t nbzg_compress_workspace_size_fmt(int64_t n, int32_t sorted, int64_t interval_count,
                                        int64_t segment_size, int32_t fmt);
size_t nbzg_compress_arena_bound(int64_t n, int64_t interval_count);
int nbzg_compress(const nbzg_compress_args *args, void *stream);

/* Decompress up to six field payloads (sorted order output, n floats each).
 * Replaces pipeline._parse_sz_stream (pipeline.py:203-223) ->
 * encode.huffman_decode (encode.py:242-261) -> K.huff_decode
 * (_kernels.py:348-374) -> quantize.dequantize_field -> K.sz_dequantize
 * (_kernels.py:126-147).  kind: 3 = SZ_DQ (v2, chunk-parallel), 0 = SZ_FIELD
 * (v1 reference streams, exact sequential chain); + NBZG_KIND_LCF (16) when the
 * archive's mode is sz-lcf (LCF predictor instead of last value).
 * payload: device bytes, any alignment, readable for payload_len + 64 bytes.
 * status: device u32, receives the first failure (NBZG_*); the caller zeroes
 * it (it is never cleared here, so one word can collect the failures of
 * several decodes, e.g. a CPC coordinate stream and the SZ velocities). */
typedef struct nbzg_decompress_args {
  const uint8_t *payload[6];
  int64_t payload_len[6];
  int32_t kind[6];
  double bound[6];        /* resolved bound of the field (archive header) */
  float *out[6];
  int32_t nfields;
  int32_t pad0;
  int64_t n;
  int64_t interval_count;
  void *workspace;        /* nbzg_decompress_workspace_size() bytes */
  size_t workspace_bytes;
  uint32_t *status;
} nbzg_decompress_args;

size_t nbzg_decompress_workspace_size(int64_t n, int64_t interval_count, int32_t nfields);
int nbzg_decompress(const nbzg_decompress_args *args, void *stream);

/* ---- CPC2000 family (Mode.SZ_CPC2000, Mode.CPC2000) ----
 * nbzg_compress with `cpc` = 1 / 2 sorts on full keys (ignored groups 0, no
 * key clamp: NBZG_BOUND_TOO_SMALL past 21 bits, rindex.py:185-190), writes
 * the segment minima (`seg_minima`, 3 x i64 per segment, io.py:115-117) and
 * builds SZ streams only for the fields outside `sz_skip`.  The VLC-family
 * streams then come from two calls on the same stream:
 *   nbzg_cpc_plan  -- per-segment VLC costs under both candidate schemes,
 *                     scheme choice, correction counts, per-stream scans
 *                     (pipeline.py:275-300, 230-237); fills `cmeta`;
 *   nbzg_cpc_pack  -- after the host read `cmeta` and placed each payload at
 *                     cmeta->off[s] of a ZEROED arena (bit region
 *                     off + nseg + 8 16-byte aligned, 64 bytes of slack):
 *                     payload bytes (pipeline.py:316-337 / 378-395 ->
 *                     K.cpc_encode_keys _kernels.py:623-645 /
 *                     K.vlc_encode_segmented _kernels.py:648-660), plus the
 *                     u32 per-segment bit lengths this path appends (v2).
 * Stream s: 0 = coordinates (StreamKind.RINDEX), 1..3 = VLC velocity fields
 * 3..5 (StreamKind.VLC_FIELD, cpc2000 only). */
typedef struct nbzg_cpc_meta {
  uint64_t off[4];        /* payload offset in the arena (host-filled before pack) */
  uint64_t len[4];        /* payload bytes */
  uint64_t total_bits[4]; /* bitstream length */
  uint64_t corr[4][3];    /* correction records per list */
  uint32_t status;        /* NBZG_BOUND_TOO_SMALL / NBZG_CODE_TOO_LONG, 0 if none */
  uint32_t pad;
} nbzg_cpc_meta;

typedef struct nbzg_cpc_args {
  const float *fields[6];    /* device, original (unsorted) order */
  int64_t n;
  int64_t segment_size;
  int32_t mode;              /* 1 sz-cpc2000 (coordinate stream), 2 cpc2000 (+ velocities) */
  int32_t pad0;
  const uint16_t *perm;      /* from nbzg_compress (tile-local sorted -> source) */
  const uint8_t *seg_bits;   /* from nbzg_compress */
  const int64_t *seg_minima; /* from nbzg_compress */
  const nbzg_meta *meta;     /* from nbzg_compress (bounds, ranges, constant mask) */
  void *workspace;           /* nbzg_cpc_workspace_size() bytes */
  size_t workspace_bytes;
  uint8_t *arena;            /* pack only */
  nbzg_cpc_meta *cmeta;      /* device */
} nbzg_cpc_args;

size_t nbzg_cpc_workspace_size(int64_t n, int64_t segment_size);
int nbzg_cpc_plan(const nbzg_cpc_args *args, void *stream);
int nbzg_cpc_pack(const nbzg_cpc_args *args, void *stream);

/* Decode one VLC-family stream (pipeline.py:340-375 / 398-428 ->
 * K.cpc_decode_keys _kernels.py:566-601 + deinterleave3 789-798 /
 * K.vlc_decode_segmented).  indexed = 1: the payload ends with u32
 * per-segment bit lengths (this path's v2 archives: one thread per segment);
 * 0: a reference (v1) stream, segment offsets found by one sequential walk.
 * Coordinates: out[c] = f32((deinterleaved key + minimum) * 2 bound[c]),
 * null for constant coordinates; velocities: out[0]. */
typedef struct nbzg_cpc_decode_args {
  const uint8_t *payload;    /* device, 64 bytes of readable slack */
  int64_t payload_len;
  int32_t kind;              /* 2 = RINDEX (coordinates), 1 = VLC_FIELD */
  int32_t indexed;
  int64_t n;
  int64_t segment_size;
  uint64_t total_bits;       /* from the payload header (host-parsed) */
  const uint8_t *seg_bits;   /* device (coordinates) */
  const int64_t *seg_minima; /* device (coordinates) */
  double bound[3];
  float *out[3];
  void *workspace;           /* nbzg_cpc_decode_workspace_size() bytes */
  size_t workspace_bytes;
  uint32_t *status;          /* device */
} nbzg_cpc_decode_args;

size_t nbzg_cpc_decode_workspace_size(int64_t n, int64_t segment_size);
int nbzg_cpc_decode(const nbzg_cpc_decode_args *args, void *stream);

/* ---- stage-level parity hooks (mirror nbz._kernels, same semantics) ---- */

/* K.huff_decode (_kernels.py:348-374): n symbols from a raw MSB-first
 * bitstream with canonical tables (host arrays of 64: first code, count and
 * first sorted index per length; device sorted symbols).  *status_dev: 0 ok,
 * NBZG_INVALID_CODE, NBZG_TRUNCATED (the reference's 1 / 2).  One thread:
 * a parity hook, not a fast path. */
int nbzg_huff_decode(const uint8_t *data, uint64_t total_bits, int64_t n, int32_t min_len,
                     int32_t max_len, const uint64_t *h_first_code, const uint32_t *h_counts,
                     const uint32_t *h_first_idx, const uint32_t *sorted_syms, uint32_t *out,
                     uint32_t *status_dev, void *stream);

/* K.deinterleave3 (_kernels.py:789-798): the three 21-bit fields of each
 * interleaved key (CPC2000 coordinate decode). */
int nbzg_deinterleave3(const uint64_t *keys, int64_t n, int64_t *x, int64_t *y, int64_t *z,
                       void *stream);

/* model.field_range x6 (model.py:104-109): out[2f] = min, out[2f+1] = max */
int nbzg_minmax6(const float *const *h_fields, int64_t n, float *out12, void *stream);

/* quantize.integerize (quantize.py:117-128): ints = rint(f64(x)/(2b)).
 * *status_dev (u32) receives NBZG_BOUND_TOO_SMALL if max|x/(2b)| > 2^62. */
int nbzg_integerize(const float *x, int64_t n, double bound, int64_t *ints,
                    uint32_t *status_dev, void *stream);

/* rindex.build_r_indices (rindex.py:164-198) + K.interleave3: full u64 keys
 * and per-segment bits from three coordinate fields (bounds[3], 0 = constant
 * coordinate -> zero column). */
int nbzg_rindex_keys(const float *x, const float *y, const float *z, int64_t n,
                     const double *h_bounds3, int64_t segment_size, uint64_t *keys,
                     uint8_t *seg_bits, uint32_t *status_dev, void *stream);

/* rindex.prx_sort (rindex.py:201-229) -> K.prx_order (_kernels.py:887-927):
 * stable per-segment order by key >> 3*min(k, bits), returned as global int64
 * source indices (`order`, the CompressResult sidecar). */
int nbzg_prx_order(const uint64_t *keys, int64_t n, int64_t segment_size,
                   const uint8_t *seg_bits, int32_t ignored_groups, int64_t *order,
                   void *stream);

/* Expand the tile-local u16 permutation written by nbzg_compress into global
 * int64 source indices (the CompressResult.order sidecar). */
int nbzg_order_expand(const uint16_t *perm, int64_t n, int64_t segment_size, int64_t *order,
                      void *stream);

/* K.huffman_lengths (_kernels.py:204-238): two-queue code lengths of k
 * ascending counts (leaf wins ties); single symbol -> length 1.  workspace:
 * 12 * next_pow2(k) bytes (used when k > 16384). */
int nbzg_huffman_lengths(const uint32_t *sorted_counts, int64_t k, uint8_t *lengths,
                         void *workspace, size_t workspace_bytes, uint32_t *status_dev,
                         void *stream);

/* encode.huffman_build (encode.py:199-219) + HuffmanTable._build_tables
 * (encode.py:123-152) from a bincount histogram of nbins u32: ascending
 * symbols (u32), their lengths (u8, by rank), and the encode LUT
 * lut[sym] = (len << 57) | word.  meta_out->f[0] receives k, min/max length,
 * total bits and n_esc (= hist[0]); meta_out->status CODE_TOO_LONG.
 * workspace: 20*nbins bytes. */
int nbzg_huffman_codebook(const uint32_t *hist, int64_t nbins, uint32_t *symbols,
                          uint8_t *lengths, uint64_t *lut, nbzg_meta *meta_out,
                          void *workspace, size_t workspace_bytes, void *stream);

/* K.huff_encode (_kernels.py:304-345): MSB-first concatenation of the code
 * words of u16 symbols into `out` (ceil(total_bits/32)*4 bytes, written as
 * big-endian words, zero padded -- byte-identical to the reference's bytes
 * for the first ceil(total_bits/8)).  chunk_bits[ceil(n/16384)] receives
 * the per-16384-symbol bit counts (the v2 index).  workspace: 16 *
 * ceil(n/16384) + 64 bytes. */
int nbzg_huff_encode(const uint16_t *syms, int64_t n, const uint64_t *lut, uint8_t *out,
                     uint32_t *chunk_bits, void *workspace, size_t workspace_bytes,
                     void *stream);

/* CRC-64/XZ (_kernels.py:954-994) of a device buffer; result to *crc_dev.
 * `data` may have any alignment; the kernel reads whole 16-byte aligned
 * granules, so when `data` is not 16-byte aligned it also touches the (up to
 * 15) bytes before it inside the same granule -- always inside the same device
 * allocation (cudaMalloc aligns to 256 bytes), and masked out of the CRC. */
int nbzg_crc64(const uint8_t *data, int64_t n, uint64_t *crc_dev, void *workspace,
               size_t workspace_bytes, void *stream);
size_t nbzg_crc64_workspace_size(int64_t n);
/* CRC-64/XZ of `count` device buffers (an archive's payloads: io.py:123-124
 * computes one per stream) in one grid; h_data / h_n are host arrays of the
 * device pointers and lengths, crc_dev[count] (device) receives the CRCs. */
int nbzg_crc64_many(const uint8_t *const *h_data, const int64_t *h_n, int32_t count,
                    uint64_t *crc_dev, void *workspace, size_t workspace_bytes, void *stream);
size_t nbzg_crc64_many_workspace_size(const int64_t *h_n, int32_t count);

/* library / device info and diagnostics */
const char *nbzg_version(void);
int nbzg_device_sm_count(void);
/* number of kernels this library has launched (process lifetime) */
unsigned long long nbzg_launch_count(void);
/* per-stage CUDA-event trace of subsequent compress / decompress calls:
 * enable (resets), then read (name, ms) intervals (synchronises). */
int nbzg_trace_enable(int on);
int nbzg_trace_read(char *names, int name_stride, float *ms, int max);

#ifdef __cplusplus
}
#endif
#endif /* NBZG_H_ */
