/*
 * hszg.h — C ABI of libhszg.so, the B200 (sm_100a) implementation of the HSZ
 * decompression / homomorphic-analytics hot path (arXiv 2603.25206).
 *
 * Conventions
 *  - Every data pointer is a DEVICE pointer owned by the caller; the library
 *    never allocates or frees caller memory.  Work that needs scratch space
 *    takes a caller-provided workspace sized by hszg_workspace_bytes().
 *  - Payload buffers must be 16-byte aligned and allocated with at least
 *    HSZG_PAYLOAD_PAD readable bytes past the payload length.
 *  - Calls are asynchronous on the given cudaStream_t (passed as void*),
 *    except the ones documented as synchronous (they read back a small
 *    status word).  Functions are reentrant; there is no global state.
 *  - Status codes map 1:1 onto the reference's exception classes
 *    (hsz/errors.py:4-26); HszgErr carries the reference's message text.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/hsz):
 *  hszg_decode_spans   <- _kernels.decode_stream   (_kernels/__init__.py:22, _bitpack.pyx:90-144)
 *  hszg_encode_spans_xx <- _kernels.encode_stream   (_kernels/__init__.py:21, _bitpack.pyx:14-87)
 *  hszg_validate       <- the per-chunk checks of  _bitpack.pyx:110-140 (run once per upload)
 *  hszg_decode         <- codec.decode_stream      (codec.py:114-121) on a CompressedStream
 *  hszg_reconstruct    <- recorrelate + dequantize (compressors.py:201-226, stages.py:88)
 *  hszg_reduce_xxx     <- stats._exact_sum, _exact_dot, mean_from_xx, std_from_xx (analytics/stats.py:30-173)
 *  hszg_region_reduce  <- (new)
 *  hszg_stencil        <- fields._axis_central_diff, _laplacian_stencil, xx_from_d{p,q,f} (analytics/fields.py:34-168)
 *  hszg_quantize etc.  <- quant.quantize / compressors.decorrelate_* (quant.py:69-82, compressors.py:149-198)
 */
#ifndef HSZG_H
#define HSZG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSZG_PAYLOAD_PAD 16
#define HSZG_END_IN_INDEX (1ull << 63)

/* status codes (hsz/errors.py) */
enum {
    HSZG_OK = 0,
    HSZG_CORRUPT = 1,           /* CorruptStreamError        errors.py:8   */
    HSZG_EPS_TOO_SMALL = 2,     /* EpsTooSmallError          errors.py:20  */
    HSZG_INVALID_ARG = 3,       /* ValueError                              */
    HSZG_UNSUPPORTED_STAGE = 4, /* UnsupportedStageError     errors.py:12  */
    HSZG_CUDA = 5,              /* CUDA runtime failure                     */
    HSZG_ZERO_RANGE = 6,        /* ZeroValueRangeError       errors.py:16  */
    HSZG_VALUE = 7              /* ValueError raised by the data (NaN, -2^31) */
};

/* compressor kinds (compressors.py:29-33) */
enum { HSZG_HSZP = 0, HSZG_HSZP_ND = 1, HSZG_HSZX = 2, HSZG_HSZX_ND = 3 };

/* output element types */
enum { HSZG_I32 = 0, HSZG_F32 = 1, HSZG_F64 = 2 };

/* Stream geometry.  Fill kind/ndims/dims/block_dims/eps and call
 * hszg_geom_init(); it derives the segment ("block") grid of the chunk
 * stream and the chunk count (compressors.py:87-119, codec.py:96-106). */
typedef struct HszgGeom {
    int32_t kind;
    int32_t ndims;
    int64_t dims[3];        /* original dims, row-major (unused trailing = 1) */
    int64_t block_dims[3];  /* resolved block dims as stored in the container */
    double eps;
    /* derived by hszg_geom_init */
    int64_t n;              /* element count */
    int64_t n_chunks;
    int64_t n_blocks;       /* geometry blocks (= metadata entries for HSZX*) */
    int64_t sdims[3];       /* 3-D view of the stream box */
    int64_t sblk[3];        /* segment extents in that view */
    int64_t sgrid[3];       /* segment grid */
} HszgGeom;

/* A device-resident compressed stream (payload + chunk index + metadata). */
typedef struct HszgStream {
    const uint8_t* payload;   /* 16-B aligned, len + HSZG_PAYLOAD_PAD bytes allocated */
    uint64_t payload_len;     /* or HSZG_END_IN_INDEX: the end is offsets[n_chunks] (a view into a longer
                                 resident index whose next entry exists; set only on validated streams) */
    const uint64_t* offsets;  /* n_chunks byte offsets into payload */
    const int32_t* metadata;  /* n_blocks block means (HSZX*), else NULL */
    int32_t canonical;        /* 1 = offsets are the encoder's exclusive scan (set by hszg_validate) */
    int32_t max_bitwidth;     /* set by hszg_validate */
} HszgStream;

typedef struct HszgErr {
    int32_t status;
    int32_t detail;          /* decode check that failed (1 offset, 2 bitwidth, 3 truncated, 4 magnitude, 5 -0) */
    int64_t chunk;           /* first failing chunk (chunk order, as the reference loop) */
    int64_t element;
    int64_t value;
    char message[192];
} HszgErr;

/* Exact integer sums returned by the reduction entry points (device struct). */
typedef struct HszgSums {
    uint64_t s1_lo;  int64_t s1_hi;   /* int128 sum of values            */
    uint64_t s2_lo;  int64_t s2_hi;   /* int128 sum of squares / products */
    int64_t count;
    int32_t vmin, vmax;
    double f1, f2;                    /* float-domain accumulators (stage 4) */
} HszgSums;

/* ---- geometry -------------------------------------------------------- */
int hszg_geom_init(HszgGeom* g);
/* Workspace bytes for an entry point.  s may be NULL (worst case: non-canonical index). */
enum {
    HSZG_WS_VALIDATE = 0,
    HSZG_WS_RECONSTRUCT = 1,   /* out_type selects I32/F32 (in place) or F64 */
    HSZG_WS_REDUCE = 2,
    HSZG_WS_ENCODE = 3,
    HSZG_WS_QUANTIZE = 4,      /* quantize, decorrelate, minmax */
    HSZG_WS_QSUMS = 5          /* hszg_quantized_sums (0: not supported for this stream) */
};
size_t hszg_workspace_bytes(const HszgGeom* g, const HszgStream* s, int op, int out_type);
const char* hszg_version(void);
/* Host-side introspection: stream [start, end) and segment of chunks [first, first+count) from the
 * closed-form geometry (no device needed).  Equals the reference's spans (codec.py:96-106). */
int hszg_locate_chunks(const HszgGeom* g, int64_t first, int64_t count, int64_t* starts, int64_t* ends,
                       int64_t* segs);

/* ---- codec ----------------------------------------------------------- */
/* Validate every chunk once (synchronous).  Sets s->canonical / s->max_bitwidth. */
int hszg_validate(const HszgGeom* g, HszgStream* s, void* ws, size_t ws_bytes, void* stream, HszgErr* err);
/* Stage 2: decode to int32 residuals in stream order (requires a validated stream). */
int hszg_decode(const HszgGeom* g, const HszgStream* s, int32_t* out, void* stream, HszgErr* err);
/* Plugin-level codec over explicit spans (the reference's _kernels interface; synchronous). */
int hszg_decode_spans(const uint8_t* payload, uint64_t len, const int64_t* starts, const int64_t* ends,
                      const uint64_t* offsets, int64_t n_chunks, int32_t* out, void* ws, size_t ws_bytes,
                      void* stream, HszgErr* err);
int hszg_encode_spans_sizes(const int32_t* values, const int64_t* starts, const int64_t* ends,
                            int64_t n_chunks, uint64_t* offsets, uint8_t* bitwidths, uint64_t* total_host,
                            void* ws, size_t ws_bytes, void* stream, HszgErr* err);
int hszg_encode_spans_pack(const int32_t* values, const int64_t* starts, const int64_t* ends,
                           int64_t n_chunks, const uint64_t* offsets, const uint8_t* bitwidths,
                           uint8_t* payload, void* stream, HszgErr* err);
/* Geometry-driven encode of a decorrelated stream (compress, compressors.py:330). */
int hszg_encode_sizes(const HszgGeom* g, const int32_t* p, uint64_t* offsets, uint8_t* bitwidths,
                      uint64_t* total_host, void* ws, size_t ws_bytes, void* stream, HszgErr* err);
int hszg_encode_pack(const HszgGeom* g, const int32_t* p, const uint64_t* offsets, const uint8_t* bitwidths,
                     uint8_t* payload, void* stream, HszgErr* err);

/* ---- stages ---------------------------------------------------------- */
/* Stage 3 (out_type HSZG_I32, q row-major) or stage 4 (HSZG_F32/F64 = q*(2*eps)). */
int hszg_reconstruct(const HszgGeom* g, const HszgStream* s, void* out, int out_type, void* ws,
                     size_t ws_bytes, void* stream, HszgErr* err);
/* hszg_reconstruct of a z-slab sub-stream of a 3-D HSZP_ND field (canonical, n2 % 32 == 0) with the slab's carry
 * q[z0-1] (n1*n2 int32, 16-B aligned) folded into the z prefix: the slab's global q without a separate
 * add pass (stages.py:193-204 slab iteration).  HSZG_UNSUPPORTED_STAGE for other streams. */
int hszg_reconstruct_carry(const HszgGeom* g, const HszgStream* s, void* out, int out_type, const int32_t* carry,
                           void* ws, size_t ws_bytes, void* stream, HszgErr* err);
/* recorrelate (compressors.py:201-226) of a decoded stream-order residual array p (not overwritten). */
int hszg_recorrelate(const HszgGeom* g, const int32_t* p, const int32_t* metadata, void* out, int out_type, void* ws,
                     size_t ws_bytes, void* stream, HszgErr* err);
/* HSZP_ND z-slab carry support (3-D, validated canonical stream): plane_out[y,x] = sum_z p[z,y,x]
 * (int32 wrap-around), straight from the compressed bytes.  Its 2-D prefix is the slab's total
 * contribution to every later plane. */
int hszg_plane_sum(const HszgGeom* g, const HszgStream* s, int32_t* plane_out, void* stream, HszgErr* err);
/* q[i] += carry[i % plane] for i < n (slab carries of slab_iter, stages.py:193-204). */
int hszg_add_plane(int32_t* q, const int32_t* carry, int64_t plane, int64_t n, void* stream);
/* Stage 3 -> 4 on a materialised index array: out = float(q) * two_eps (stages.py:88). */
int hszg_dequantize(const int32_t* q, int64_t n, double two_eps, void* out, int out_type, void* stream);
/* Block-contiguous <-> row-major permutation (canonical_order, grid.py:114-128). */
int hszg_stream_perm(const HszgGeom* g, int64_t* perm, void* stream);
/* Scatter a stream-order int32 array to row-major (as_grid, compressors.py:68-73);
 * add_meta != 0 adds the per-block metadata (stage 3 of HSZX*). */
int hszg_scatter_grid(const HszgGeom* g, const int32_t* src, const int32_t* metadata, int add_meta,
                      int32_t* out, void* stream);
/* Per-point block mean grid (metadata_grid, compressors.py:75-84). */
int hszg_metadata_grid(const HszgGeom* g, const int32_t* metadata, int64_t* out, void* stream);

/* ---- reductions (K-STAT) ---------------------------------------------- */
/* mode: 0 = exact integer sums of q (+min/max) over stream/grid order,
 *       1 = HSZP weighted sum  sum((N-i) p_i)            (stats.py:88)
 *       2 = HSZP_ND weighted   sum(prod(n_k-i_k) p)      (stats.py:95-112)
 *       3 = HSZX* stage-2 sums of q = p + M_b in stream order (no scatter)
 *       4 = stage-1 sum(M_b * S_b)                          (stats.py:69-77)
 * mode 1-4 read the compressed stream; mode 0 reads an int32 array (src).
 * mode | HSZG_REDUCE_NO_EXTREMA: vmin / vmax are not wanted (statistics only; leaner decode). */
#define HSZG_REDUCE_NO_EXTREMA 0x100
int hszg_reduce_stream(const HszgGeom* g, const HszgStream* s, int mode, HszgSums* out_dev, void* ws,
                       size_t ws_bytes, void* stream, HszgErr* err);
/* modes 1-3 over an already-decoded stream-order residual array p (DecorrelatedStream.values) */
int hszg_reduce_array(const HszgGeom* g, const int32_t* p, const int32_t* metadata, int mode, HszgSums* out_dev,
                      void* ws, size_t ws_bytes, void* stream);
int hszg_reduce_i32(const int32_t* src, int64_t n, HszgSums* out_dev, void* ws, size_t ws_bytes, void* stream);
/* float-domain (stage 4): f1 = sum(fl(q*scale)); if mean_ptr != NULL, f2 = sum((fl(q*scale)-mean)^2) */
int hszg_reduce_f64(const int32_t* q, int64_t n, double scale, const double* mean_dev, HszgSums* out_dev,
                    void* ws, size_t ws_bytes, void* stream);
/* int64/int128 sum of a*b over int32 arrays (stats._exact_dot) */
int hszg_reduce_dot(const int32_t* a, const int32_t* b, int64_t n, HszgSums* out_dev, void* ws,
                    size_t ws_bytes, void* stream);

/* ---- regional statistics (K-REG) -------------------- */
/* Per region (origin-aligned R-tiles, edge tiles shrunk, row-major region order):
 * s1[int64], s2 (int128 as lo/hi), qmin, qmax, size. */
int hszg_region_reduce(const int32_t* q, int32_t ndims, const int64_t* dims, const int64_t* region,
                       int64_t* s1, uint64_t* s2_lo, int64_t* s2_hi, int32_t* qmin, int32_t* qmax,
                       int64_t* size, void* stream);

/* Per-region finalisation: mean = S1/size*2eps, var = (size*S2 - S1^2)/(size(size-1))*(2eps)^2 (NaN
 * below 2 points), fmin/fmax = q{min,max}*2eps, *count_dev = #regions with fmin < tau <= fmax. */
/* N2-N4 fused from an HSZX* stream (q = p + M_b, stage 2 / 3 alike; no reconstruction): per-region
 * S1, S2 (lo / hi), qmin, qmax, size as hszg_region_reduce.  Regions (original dims) must be multiples
 * of the block extents (or reach the grid end) and every chunk full; else HSZG_UNSUPPORTED_STAGE and
 * the caller reconstructs q.  ws >= 64 bytes per region.  (new, SURVEY section 8, N2-N4 / K-REG) */
int hszg_region_stream(const HszgGeom* g, const HszgStream* s, const int64_t* region, int64_t* s1, uint64_t* s2_lo,
                       int64_t* s2_hi, int32_t* qmin, int32_t* qmax, int64_t* size, void* ws, size_t ws_bytes,
                       void* stream, HszgErr* err);
int hszg_region_finalize(const int64_t* s1, const uint64_t* s2_lo, const int64_t* s2_hi, const int32_t* qmin,
                         const int32_t* qmax, const int64_t* size, int64_t n_regions, double two_eps, double tau,
                         double* mean, double* var, double* fmin, double* fmax, unsigned long long* count_dev,
                         void* stream);
/* float64 sums of an arbitrary float64 array: f1 = sum(x); f2 = sum((x-mean)^2) if mean_dev. */
int hszg_reduce_flt(const double* x, int64_t n, const double* mean_dev, HszgSums* out_dev, void* ws,
                    size_t ws_bytes, void* stream);

/* ---- stencils (K-STEN) -------------------------------------------------- */
enum {
    HSZG_OP_DERIV = 0,      /* out[k] = D_k(q) * eps (stage 2/3) or (d[i+1]-d[i-1])/2 (stage 4) */
    HSZG_OP_LAPLACIAN = 1,  /* out[0] = L(q) * 2eps (stage 2/3) or float stencil (stage 4)     */
    HSZG_OP_GRADMAG = 2,    /* out[0] = eps * sqrt(sum_k D_k^2)  (N5)                          */
    HSZG_OP_DIVERGENCE = 3, /* out[0] = sum_k D_k(q_k) * eps_k   (fields.py:216-222)           */
    HSZG_OP_CURL = 4,       /* out[...] = curl components        (fields.py:225-236)           */
    HSZG_OP_GRAD_LAP = 5    /* out[0..nd-1] = derivatives, out[nd] = Laplacian, one pass         */
};
/* q[c]: row-major grids (c < ncomp); eps[c] per component.  float_domain 0: int32 indices with
 * integer stencils (stage 2/3); 1: int32 indices read as fl(q*2eps) with the float stencils of
 * fields.py:83-93 (stage 4); 2: float64 input grids, float stencils.  out[k]: HSZG_F32/F64 grids. */
int hszg_stencil(int op, int32_t ndims, const int64_t* dims, int32_t ncomp, const void* const* q,
                 const double* eps, int float_domain, int32_t out_type, void* const* out, void* stream);

/* Windowed 3-D stencil: computes box planes [zlo, zhi) of the (n0,n1,n2) int32 grids q, whose plane 0
 * sits at global axis-0 coordinate gz0 of a field with gN0 planes (boundary layers are global);
 * out[k] receives planes [zlo, zhi) contiguously.  Used by the windowed / sharded pipelines. */
int hszg_stencil_window(int op, const int64_t* dims, int32_t ncomp, const void* const* q, const double* eps,
                        int float_domain, int32_t out_type, void* const* out, int64_t zlo, int64_t zhi,
                        int64_t gz0, int64_t gN0, void* stream);
/* Combine an array of HszgSums (e.g. per-window partials) into one, deterministically. */
int hszg_sums_combine(const HszgSums* parts, int64_t n, HszgSums* out, void* stream);

/* ---- encode side (K-ENC) ------------------------------------------------ */
/* min/max + NaN/Inf count of an fp32 field (resolve_eps, quant.py:56-66): out_dev = {min, max}
 * as doubles, nonfinite_dev = count of NaN/Inf values. */
int hszg_minmax_f32(const float* field, int64_t n, double* out_dev, int64_t* nonfinite_dev, void* ws,
                    size_t ws_bytes, void* stream);
int hszg_minmax_f64(const double* field, int64_t n, double* out_dev, int64_t* nonfinite_dev, void* ws,
                    size_t ws_bytes, void* stream);
/* q = floor(float64(d) * recip + 0.5) with |q| <= QMAX (quant.py:69-82); synchronous status. */
int hszg_quantize_f32(const float* field, int64_t n, double recip, int32_t* q, void* ws, size_t ws_bytes,
                      void* stream, HszgErr* err);
int hszg_quantize_f64(const double* field, int64_t n, double recip, int32_t* q, void* ws, size_t ws_bytes,
                      void* stream, HszgErr* err);
/* p (stream order) + metadata from q (row-major); synchronous status (EpsTooSmallError). */
int hszg_decorrelate(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, void* ws,
                     size_t ws_bytes, void* stream, HszgErr* err);
/* hszg_decorrelate fused with the encoder's per-chunk bit widths and byte sizes (_bitpack.pyx:24-51):
 * when every chunk holds 32 values and the decorrelation kernel sees whole chunks, sizes[c] /
 * bitwidths[c] are written too and *fused = 1 (then hszg_encode_offsets scans them, and p is not
 * re-read); otherwise *fused = 0 and the caller runs hszg_encode_sizes. */
int hszg_decorrelate_sized(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, uint64_t* sizes,
                           uint8_t* bitwidths, int* fused, void* ws, size_t ws_bytes, void* stream, HszgErr* err);
/* Exclusive scan of precomputed chunk sizes (in place: sizes -> offsets) and the payload total. */
int hszg_encode_offsets(const HszgGeom* g, uint64_t* offsets, uint64_t* total_host, void* ws, size_t ws_bytes,
                        void* stream, HszgErr* err);
/* One-pass compress (csrc/compress.cu) of a float32 field: quantize (quant.py:69-82) + decorrelate
 * (compressors.py:149-198) + encode_stream (codec.py:84-106, _bitpack.pyx:24-87) in one kernel, replacing
 * the chain hszg_quantize_f32 -> hszg_decorrelate_sized -> hszg_encode_offsets -> hszg_encode_pack.
 * hszg_compress_plan returns 1 when the geometry has a one-pass front (every chunk 32 values; HSZP,
 * HSZP_ND with n2 % 32 == 0 and n2 <= 8192, HSZX / HSZX_ND with full blocks of 32k <= 8192 values,
 * B2 % 4 == 0) and the workspace / payload capacity it needs (n_chunks * 133 + HSZG_PAYLOAD_PAD: the
 * worst case, the payload length is known only after the pass), else 0.  hszg_compress_fused writes
 * the payload (its length to *total_host, the pad zeroed), the chunk offsets and the block means;
 * synchronous status with the messages of the chain (EpsTooSmallError / ValueError). */
int hszg_compress_plan(const HszgGeom* g, uint64_t* ws_bytes, uint64_t* payload_capacity);
int hszg_compress_fused(const HszgGeom* g, const float* field, double recip, uint8_t* payload, uint64_t capacity,
                        uint64_t* offsets, int32_t* metadata, uint64_t* total_host, void* ws, size_t ws_bytes,
                        void* stream, HszgErr* err);

/* ---- windowed 3-D pipeline (pipeline.py; Algorithm 3 on the device) -------------------------- */
/* fp32 outputs: exact != 0 gives fl32(fl64(D*eps)) (one rounding of the reference float64); exact == 0
 * computes fl32(D * fl32(eps)) in int32/fp32 arithmetic, within 2^-23 relative of it (<< 1e-6). */
/* Exact order-independent statistics: int128 sums split into 32-bit limbs accumulated with
 * 64-bit atomics (limb 3 signed): value = sum_k limb_k * 2^(32k). */
typedef struct HszgAcc {
    uint64_t s1_limb[4];
    uint64_t s2_limb[4];
    int64_t count;
    int32_t vmin, vmax;
} HszgAcc;
int hszg_acc_reset(HszgAcc* acc, void* stream);
/* Gradient (dz, dy, dx) + Laplacian, fp32, of planes [zlo, zhi) of the int32 window q (box planes;
 * plane 0 at global z gz0 of a gN0-plane field; planes zlo-1 / zhi are read where they exist).
 * qprev / qnext (optional) replace the in-window planes zlo-1 / zhi (ring-buffered windows).
 * acc (optional) accumulates sum q, sum q^2, min, max of the output planes. */
int hszg_zgrad_lap(const int32_t* q, int64_t n1, int64_t n2, int64_t zlo, int64_t zhi, int64_t gz0, int64_t gN0,
                   double eps, float* const* out, HszgAcc* acc, const int32_t* qprev, const int32_t* qnext,
                   int exact, void* stream);
/* HSZP_ND z-sweep: from 2-D-prefixed planes P2 (planes a.., plus a lookahead plane when
 * lookahead != NULL: P2 of plane a+nout), the carry q[a-1] (NULL at the global first plane) and optionally the upper
 * neighbour's q plane, emit gradient + Laplacian of nout planes, accumulate stats and write
 * q[a+nout-1] to carry_out — q itself is never stored.  With band_off (hszg_band_scan output) P2 is
 * band-local: row y of plane z adds band_off[z][y / band_rows][:] (look_band_off: the lookahead's);
 * p2_mode: width codes of those band-local prefixes (hszg_band_scan l_mode) — bits 0-3 for P2, bits 4-7
 * for the lookahead plane: 0 int32, 1 int16, 2 int8; pairs equal, or int16 P2 with an int8 lookahead.
 * exact: as hszg_fused_blocks (0 fast, 1 fp64 conversions, 2 table; 2 only on the ring sweep, band_rows % 16
 * == 0, else treated as 1). */
int hszg_zsweep_grad_lap(const int32_t* P2, int64_t n1, int64_t n2, int64_t nout, const int32_t* lookahead,
                         const int32_t* carry, const int32_t* q_upper, int32_t* carry_out, int64_t gz0, int64_t gN0,
                         double eps, float* const* out, HszgAcc* acc, const int32_t* band_off,
                         const int32_t* look_band_off, int64_t band_rows, int p2_mode, int exact, void* stream);
/* Exact sums of the stage-3 indices q (S1, S2, min, max, count) without writing q: HSZP (every chunk
 * full: the look-back scan reduces instead of storing) and 3-D HSZP_ND (n2 % 32 == 0, one band per
 * plane: band scan + a z prefix that reduces).  hszg_workspace_bytes(HSZG_WS_QSUMS) is 0 for other
 * streams (callers then reconstruct and reduce).  Replaces stats.py:115-173's q = recorrelate(...)
 * followed by the sums. */
int hszg_quantized_sums(const HszgGeom* g, const HszgStream* s, HszgSums* out_dev, void* ws, size_t ws_bytes,
                        void* stream, HszgErr* err);
/* HSZX_ND one-pass decode + gradient + Laplacian + stats (8x8x8 blocks dividing the 3-D box, canonical,
 * max bit width <= 16): q never reaches memory.  The stream is a z-slab of a gN0-plane field whose
 * first plane is global plane gz0; halo_lo / halo_hi (optional, n1*n2 int32) are q of the planes just
 * below / above the slab.  zlayers = 8-plane block layers per CTA (z segment of the grid).
 * out[4] = dz, dy, dx, Laplacian (fp32, slab-sized); acc (optional) accumulates the slab's stats.
 * exact: 0 fast fp32 (int32 stencil x fl32(eps), |q| < 2^27), 1 fl32 of the reference float64 by fp64
 * conversions, 2 the same values by a shared-memory table (int32 stencils: the caller guarantees
 * |q| < 2^27).  In the exact modes out may hold only {dz, dy, dx} (Laplacian NULL) or only the
 * Laplacian (the API's derivative / laplacian calls, fields.py:34-93); other subsets: HSZG_INVALID_ARG. */
int hszg_fused_blocks(const HszgGeom* g, const HszgStream* s, int64_t gz0, int64_t gN0, const int32_t* halo_lo,
                      const int32_t* halo_hi, float* const* out, HszgAcc* acc, int64_t zlayers, int exact,
                      void* stream, HszgErr* err);
/* HSZP_ND in one pass over a z-slab (3-D, canonical, n2 % 32 == 0, n2 <= 4096): decode + Lorenzo
 * inversion (x, y, z prefixes) + gradient + Laplacian (+ stats into acc) with q never in memory.
 * band_off / strip_edges: hszg_band_scan of the same stream with band_rows = 16 and L = NULL.
 * carry: q of the plane below the slab (NULL at the field's first plane); q_upper: q of the plane
 * above (NULL at the field's last plane).  out[4] = dz, dy, dx, Laplacian (fp32, slab-sized). */
int hszg_lorenzo_onepass(const HszgGeom* g, const HszgStream* s, const int32_t* band_off,
                         const int32_t* strip_edges, const int32_t* carry, const int32_t* q_upper, int64_t gz0,
                         int64_t gN0, float* const* out, HszgAcc* acc, int exact, void* stream, HszgErr* err);
/* HSZP_ND decode + row prefix + in-band column prefix in one pass (3-D, canonical, n2 % 32 == 0,
 * n2 <= 4096).  L[z][y][x] (optional) = 2-D prefix of plane z restricted to the
 * rows of y's band (bands of band_rows rows); band_off[z][b][x] = sum of the rows of bands < b, i.e.
 * P2 = L + band_off[z][y / band_rows].  strip_edges (optional): for 128-wide x strips s,
 * [z][s][y][0] = row prefix at x = 128s - 1 (0 for s = 0), [z][s][y][1] = at x = 128s + 128 (0 past
 * the row).  L: dims[0]*dims[1]*dims[2] int32; band_off: dims[0]*ceil(dims[1]/band_rows)*dims[2];
 * strip_edges: dims[0]*ceil(dims[2]/128)*E*2 int32 with E = dims[1] rounded up to even (+ 64 spare).
 * l_mode: 0 writes L as int32; 1 as int16 (n2 % 8 == 0), any value that does not fit setting bit 2
 * of *l_overflow; 2 as int8 (n2 % 16 == 0), setting bit 1 (the caller then redoes the pass wider).
 * ctas_per_sm: 0 launches one CTA per (band, plane); k > 0 a persistent grid of k CTAs per SM that
 * leaves room for a concurrent kernel (the z-sweep of an earlier window on another stream). */
int hszg_band_scan(const HszgGeom* g, const HszgStream* s, int64_t band_rows, void* L, int32_t* band_off,
                   int32_t* strip_edges, int l_mode, int32_t* l_overflow, int ctas_per_sm, void* stream,
                   HszgErr* err);
/* HSZP_ND decode fused with the in-row prefix (rows of whole chunks, 256 % (n2/32) == 0). */
int hszg_decode_rowscan(const HszgGeom* g, const HszgStream* s, int32_t* out, void* stream, HszgErr* err);
/* In-place inclusive scan along the middle axis of an int32 [A][M][L] view. */
int hszg_col_scan(int32_t* buf, int64_t A, int64_t M, int64_t L, void* stream);

/* ---- synthetic input (BASELINE config 5, generated on the device; not the hot path) ---- */
int hszg_gen_noise(float* out, int64_t e0, int64_t nz, const int64_t* dims, uint64_t seed, void* stream);
int hszg_gauss_pass(const float* in, float* out, int64_t e0, int64_t nz, const int64_t* dims, int axis,
                    const float* w, int r, void* stream);
int hszg_gauss_pass_z(const float* in, float* out, int64_t e0, int64_t nz, int64_t z0, int64_t nzout,
                      const int64_t* dims, const float* w, int r, void* stream);
int hszg_gen_modes(float* out, int64_t z0, int64_t nz, const int64_t* dims, const double* modes, int nmodes,
                   double scale, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HSZG_H */
