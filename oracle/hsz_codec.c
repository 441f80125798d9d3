/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C restatement of the HSZ fixed-rate chunk codec, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the CPU checker.  Never linked into libhszg.so.
 *
 * Follows /root/reference/pkg/src/hsz/_kernels/_bitpack.pyx:
 *   encode: pass 1 (bitwidth + exclusive scan of chunk sizes)  _bitpack.pyx:24-51
 *           pass 2 (sign bitmap + LSB-first magnitude pack)       _bitpack.pyx:53-86
 *   decode: per-chunk checks and bit loop                         _bitpack.pyx:90-144
 * Byte layout contract: _kernels/_fallback.py:1-8, chunk_byte_size 52-55.
 *
 * Encode-pack and decode are parallelised over chunks with pthreads (chunks
 * are independent); decode reports the first failing chunk in
 * chunk order, exactly like the sequential reference loop.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <pthread.h>
#include <unistd.h>

#define HSZO_INT32_MIN (-2147483647LL - 1)
#define HSZO_MAG_MAX 2147483647ULL

/* error kinds, reported in the same order the reference checks them */
enum {
    HSZO_OK = 0,
    HSZO_OFFSET_PAST_END = 1,   /* _bitpack.pyx:111-112 */
    HSZO_BITWIDTH = 2,          /* _bitpack.pyx:114-115 */
    HSZO_TRUNCATED = 3,         /* _bitpack.pyx:122-123 */
    HSZO_MAG_RANGE = 4,         /* _bitpack.pyx:135-136 */
    HSZO_NEG_ZERO = 5,          /* _bitpack.pyx:138-140 */
    HSZO_INT32_MIN_ENC = 6      /* _bitpack.pyx:35-38 */
};

static int g_threads = 1;

int hszo_num_threads(void) { return g_threads; }

void hszo_set_threads(int n) {
    if (n <= 0) n = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (n < 1) n = 1;
    if (n > 256) n = 256;
    g_threads = n;
}

/* run fn(lo, hi, arg) over [0, n) split across g_threads pthreads */
typedef void (*range_fn)(int64_t lo, int64_t hi, int slot, void* arg);
typedef struct { range_fn fn; int64_t lo, hi; int slot; void* arg; } range_job;
static void* range_entry(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->lo, j->hi, j->slot, j->arg);
    return NULL;
}
static void parallel_range(int64_t n, range_fn fn, void* arg) {
    int t = g_threads;
    if (t <= 1 || n < 4096) { fn(0, n, 0, arg); return; }
    pthread_t th[256];
    range_job jobs[256];
    for (int i = 0; i < t; i++) {
        jobs[i].fn = fn; jobs[i].arg = arg; jobs[i].slot = i;
        jobs[i].lo = n * i / t; jobs[i].hi = n * (i + 1) / t;
        pthread_create(&th[i], NULL, range_entry, &jobs[i]);
    }
    for (int i = 0; i < t; i++) pthread_join(th[i], NULL);
}

static inline int bit_length_u64(uint64_t v) {
    int bw = 0;
    while (v) { bw++; v >>= 1; }
    return bw;
}

/* Pass 1: bitwidths and offsets.  Returns total payload bytes, or -1 on
 * INT32_MIN (reported through *bad_chunk).  _bitpack.pyx:24-51 */
int64_t hszo_encode_sizes(const int32_t* vals, const int64_t* starts, const int64_t* ends,
                          int64_t nchunks, uint8_t* bws, uint64_t* offsets, int64_t* bad_chunk) {
    int64_t total = 0;
    *bad_chunk = -1;
    for (int64_t i = 0; i < nchunks; i++) {
        uint64_t max_mag = 0;
        for (int64_t j = starts[i]; j < ends[i]; j++) {
            int64_t v = vals[j];
            if (v == HSZO_INT32_MIN) { *bad_chunk = i; return -1; }
            uint64_t mag = (uint64_t)(v < 0 ? -v : v);
            if (mag > max_mag) max_mag = mag;
        }
        int bw = bit_length_u64(max_mag);
        bws[i] = (uint8_t)bw;
        offsets[i] = (uint64_t)total;
        int64_t count = ends[i] - starts[i];
        total += 1;
        if (bw > 0) total += (count + 7) / 8 + (count * bw + 7) / 8;
    }
    return total;
}

/* Pass 2: pack into a zero-initialised buffer.  _bitpack.pyx:53-86 */
typedef struct {
    const int32_t* vals; const int64_t* starts; const int64_t* ends;
    const uint8_t* bws; const uint64_t* offsets; uint8_t* out;
} pack_args;

static void pack_range(int64_t lo, int64_t hi, int slot, void* vp) {
    (void)slot;
    pack_args* a = (pack_args*)vp;
    const int32_t* vals = a->vals; const int64_t* starts = a->starts; const int64_t* ends = a->ends;
    const uint8_t* bws = a->bws; const uint64_t* offsets = a->offsets; uint8_t* out = a->out;
    for (int64_t i = lo; i < hi; i++) {
        int64_t s = starts[i], e = ends[i], count = e - s;
        int bw = bws[i];
        uint64_t pos = offsets[i];
        out[pos++] = (uint8_t)bw;
        if (bw == 0) continue;
        for (int64_t j = s; j < e; j++)
            if (vals[j] < 0) out[pos + ((j - s) >> 3)] |= (uint8_t)(1u << ((j - s) & 7));
        pos += (count + 7) / 8;
        uint64_t acc = 0;
        int nbits = 0;
        for (int64_t j = s; j < e; j++) {
            int64_t v = vals[j];
            uint64_t mag = (uint64_t)(v < 0 ? -v : v);
            acc |= mag << nbits;
            nbits += bw;
            while (nbits >= 8) { out[pos++] = (uint8_t)(acc & 0xFF); acc >>= 8; nbits -= 8; }
        }
        if (nbits > 0) out[pos++] = (uint8_t)(acc & 0xFF);
    }
}

void hszo_encode_pack(const int32_t* vals, const int64_t* starts, const int64_t* ends,
                      int64_t nchunks, const uint8_t* bws, const uint64_t* offsets, uint8_t* out) {
    pack_args a = {vals, starts, ends, bws, offsets, out};
    parallel_range(nchunks, pack_range, &a);
}

/* Decode one chunk; returns an error kind (0 ok) and the failing element. */
static inline int decode_chunk(const uint8_t* buf, uint64_t size, int64_t s, int64_t e,
                               uint64_t off, int32_t* vals, int64_t* bad_elem) {
    int64_t count = e - s;
    uint64_t pos = off;
    if (pos >= size) return HSZO_OFFSET_PAST_END;
    int bw = buf[pos];
    if (bw > 32) return HSZO_BITWIDTH;
    pos += 1;
    if (bw == 0) {
        for (int64_t j = 0; j < count; j++) vals[s + j] = 0;
        return HSZO_OK;
    }
    uint64_t sign_pos = pos;
    pos += (uint64_t)((count + 7) / 8);
    uint64_t end = pos + (uint64_t)((count * bw + 7) / 8);
    if (end > size) return HSZO_TRUNCATED;
    uint64_t mask = (bw == 64) ? ~0ULL : ((1ULL << bw) - 1);
    uint64_t acc = 0;
    int nbits = 0;
    for (int64_t j = 0; j < count; j++) {
        while (nbits < bw) { acc |= ((uint64_t)buf[pos]) << nbits; pos++; nbits += 8; }
        uint64_t mag = acc & mask;
        acc >>= bw;
        nbits -= bw;
        if (mag > HSZO_MAG_MAX) { *bad_elem = j; return HSZO_MAG_RANGE; }
        int neg = (buf[sign_pos + (j >> 3)] >> (j & 7)) & 1;
        if (neg) {
            if (mag == 0) { *bad_elem = j; return HSZO_NEG_ZERO; }
            vals[s + j] = (int32_t)(-(int64_t)mag);
        } else {
            vals[s + j] = (int32_t)mag;
        }
    }
    return HSZO_OK;
}

typedef struct {
    const uint8_t* buf; uint64_t size; const int64_t* starts; const int64_t* ends;
    const uint64_t* offsets; int32_t* vals; int64_t first_bad[256];
    int parts;
} dec_args;

static void decode_range(int64_t lo, int64_t hi, int slot, void* vp) {
    dec_args* a = (dec_args*)vp;
    int64_t first = INT64_MAX;
    for (int64_t i = lo; i < hi; i++) {
        int64_t be = 0;
        if (decode_chunk(a->buf, a->size, a->starts[i], a->ends[i], a->offsets[i], a->vals, &be)
            != HSZO_OK) { first = i; break; }
    }
    a->first_bad[slot] = first;
}

/* Decode all chunks; out must hold ends[nchunks-1] int32 values.
 * Returns 0, or an error kind with bad_chunk/bad_elem set to the first
 * failing chunk in chunk order (the reference's sequential semantics). */
int hszo_decode(const uint8_t* buf, uint64_t size, const int64_t* starts, const int64_t* ends,
                const uint64_t* offsets, int64_t nchunks, int32_t* vals,
                int64_t* bad_chunk, int64_t* bad_elem) {
    dec_args* a = (dec_args*)calloc(1, sizeof(dec_args));
    a->buf = buf; a->size = size; a->starts = starts; a->ends = ends; a->offsets = offsets;
    a->vals = vals;
    a->parts = (g_threads <= 1 || nchunks < 4096) ? 1 : g_threads;
    for (int i = 0; i < 256; i++) a->first_bad[i] = INT64_MAX;
    parallel_range(nchunks, decode_range, a);
    int64_t first_bad = INT64_MAX;
    for (int i = 0; i < a->parts; i++) if (a->first_bad[i] < first_bad) first_bad = a->first_bad[i];
    free(a);
    *bad_chunk = -1;
    *bad_elem = -1;
    if (first_bad == INT64_MAX) return HSZO_OK;
    int64_t be = -1;
    int kind = decode_chunk(buf, size, starts[first_bad], ends[first_bad], offsets[first_bad],
                            vals, &be);
    *bad_chunk = first_bad;
    *bad_elem = be;
    return kind;
}
