// capi.cu — geometry setup and workspace queries of the C ABI (include/hszg.h).
#include <cstdio>
#include "common.cuh"
#include "lookback.cuh"
#include "tile.cuh"

using namespace hszg;

size_t hszg_reduce_ws_bytes(int64_t tiles);
size_t hszg_quantized_sums_ws(const HszgGeom* g, const HszgStream* s);

// Derive the segment view of a stream (see common.cuh) from the container's
// kind / dims / block dims (compressors.py:87-119, 245-270).
extern "C" int hszg_geom_init(HszgGeom* g) {
    const int nd = g->ndims;
    if (nd < 1 || nd > 3 || g->kind < 0 || g->kind > 3) return HSZG_INVALID_ARG;
    int64_t n = 1;
    for (int k = 0; k < nd; k++) {
        if (g->dims[k] < 1) return HSZG_INVALID_ARG;
        n *= g->dims[k];
    }
    for (int k = nd; k < 3; k++) {
        g->dims[k] = 1;
        g->block_dims[k] = 1;
    }
    g->n = n;
    int64_t box[3] = {1, 1, 1}, seg[3] = {1, 1, 1};
    const bool is_nd = g->kind == HSZG_HSZP_ND || g->kind == HSZG_HSZX_ND;
    if (is_nd && nd < 2) return HSZG_INVALID_ARG;
    for (int k = 0; k < nd; k++) box[3 - nd + k] = g->dims[k];
    if (!is_nd) {
        box[0] = box[1] = 1;
        box[2] = n;
        const int64_t S = g->block_dims[0];
        if (S < 1 || S > n) return HSZG_INVALID_ARG;
        seg[2] = S;
        g->n_blocks = (n + S - 1) / S;
    } else if (g->kind == HSZG_HSZP_ND) {
        seg[0] = 1;
        seg[1] = box[1];
        seg[2] = box[2];
        if (nd == 2) seg[1] = 1;
        int64_t nb = 1;
        for (int k = 0; k < nd; k++) {
            const int64_t b = g->block_dims[k];
            if (b < 1 || b > g->dims[k]) return HSZG_INVALID_ARG;
            nb *= (g->dims[k] + b - 1) / b;
        }
        g->n_blocks = nb;
    } else {
        int64_t nb = 1;
        for (int k = 0; k < nd; k++) {
            const int64_t b = g->block_dims[k];
            if (b < 1 || b > g->dims[k]) return HSZG_INVALID_ARG;
            seg[3 - nd + k] = b;
            nb *= (g->dims[k] + b - 1) / b;
        }
        g->n_blocks = nb;
    }
    for (int a = 0; a < 3; a++) {
        g->sdims[a] = box[a];
        g->sblk[a] = seg[a];
        g->sgrid[a] = (box[a] + seg[a] - 1) / seg[a];
    }
    const SegGeo sg = make_seggeo(*g);
    g->n_chunks = sg.n_chunks;
    return HSZG_OK;
}

extern "C" size_t hszg_workspace_bytes(const HszgGeom* g, const HszgStream* s, int op, int out_type) {
    const bool canonical = s && s->canonical;
    const size_t n4 = (size_t)g->n * 4;
    switch (op) {
        case HSZG_WS_VALIDATE:
            return 256;
        case HSZG_WS_RECONSTRUCT: {
            // fast fused paths (canonical index): only look-back state for HSZP
            const SegGeo sg = make_seggeo(*g);
            const bool fused = canonical && (g->kind == HSZG_HSZX || g->kind == HSZG_HSZP ||
                                             (g->kind == HSZG_HSZX_ND && sg.cpb[0] <= TILE_CHUNKS));
            if (fused) {
                // HSZP: the tile carries of the three-pass scan (recon.cu) or the look-back state
                const int64_t tiles = (g->n_chunks + 31) / 32;
                const size_t a = lookback_ws_bytes(g->n_chunks);
                const size_t b = (((size_t)tiles * 4 + 255) & ~(size_t)255) + 148 * 4 * 4 + 256;
                return (a > b ? a : b) + 256;
            }
            if (canonical && g->kind == HSZG_HSZP_ND && g->ndims == 3)   // band-scan path: band totals
            {
                const int64_t br = recon_band_rows(g->dims[0], g->dims[1], g->dims[2]);
                const int64_t nb = (g->dims[1] + br - 1) / br;
                // + the int16 band-local prefixes of the narrow path (recon.cu band_scan_narrow) and its flag
                const size_t p2b = out_type == HSZG_F64 ? n4 : (((size_t)g->n * 2 + 255) & ~(size_t)255);
                return p2b + (size_t)g->dims[0] * nb * g->dims[2] * 4 + 512;
            }
            // generic: decode buffer (fp64 output only) + per-kind transform scratch
            size_t b = out_type == HSZG_F64 ? n4 : 0;
            if (g->kind == HSZG_HSZP) b += lookback_ws_bytes(g->n);
            if (g->kind == HSZG_HSZX_ND) b += n4;
            return b + 256;
        }
        case HSZG_WS_REDUCE: {
            const int64_t tiles = (g->n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
            size_t b = hszg_reduce_ws_bytes(tiles);
            if (!canonical) b = hszg_reduce_ws_bytes(148 * 16) + n4;
            return b + 256;
        }
        case HSZG_WS_ENCODE:
            return 16 + lookback_ws_bytes(g->n_chunks) + 256;
        case HSZG_WS_QUANTIZE:
            return 148 * 8 * 32 + 256;
        case HSZG_WS_QSUMS:
            return hszg_quantized_sums_ws(g, s);
        default:
            return 0;
    }
}

extern "C" const char* hszg_version(void) { return "hszg 0.1 sm_100a"; }

// Host-side introspection of the closed-form chunk geometry (used by the CPU test-suite to
// check it against the reference's span construction, codec.py:96-106).
extern "C" int hszg_locate_chunks(const HszgGeom* g, int64_t first, int64_t count, int64_t* starts, int64_t* ends,
                                  int64_t* segs) {
    const SegGeo sg = make_seggeo(*g);
    if (first < 0 || first + count > sg.n_chunks) return HSZG_INVALID_ARG;
    for (int64_t i = 0; i < count; i++) {
        const ChunkLoc L = locate_chunk(sg, first + i);
        starts[i] = L.start;
        ends[i] = L.start + L.count;
        if (segs) segs[i] = L.seg;
    }
    return HSZG_OK;
}
