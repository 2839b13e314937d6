/*
 * ipcomp_oracle.c -- CPU ORACLE (test infrastructure only; see ipcomp_oracle.h).
 *
 * Plain-C restatement of the reference IPComp hot path.  Every function cites
 * the reference file:line it follows (paths relative to /root/reference/proj).
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, like the reference's
 * CMakeLists.txt:25-27, which is what keeps encoder and decoder rounding
 * identical).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load the resulting library.
 */
#include "ipcomp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <zlib.h>

#define KMAXCODE ((int32_t)1 << 30)       /* quantizer.hpp:11 */
#define NBMASK 0xAAAAAAAAu                /* quantizer.hpp:12 */
#define KBUCKETS 1024                     /* planner.cpp:14 */
#define KINFCOST (KBUCKETS + 1)           /* planner.cpp:15 */

enum { E_OK = 0, E_INVALID = 1, E_RUNTIME = 2, E_DOMAIN = 3, E_INFEASIBLE = 4 };

static int fail(char *err, int errlen, int code, const char *msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
    return code;
}

void orc_free(void *p) { free(p); }

/* ------------------------------------------------------------------ bytes */
/* little-endian ByteWriter / ByteReader, common.hpp:56-107 */
typedef struct {
    uint8_t *p;
    uint64_t n, cap;
} wbuf;

static void wb_reserve(wbuf *b, uint64_t extra) {
    if (b->n + extra <= b->cap) return;
    uint64_t c = b->cap ? b->cap : 256;
    while (c < b->n + extra) c *= 2;
    b->p = (uint8_t *)realloc(b->p, c);
    b->cap = c;
}
static void wb_put(wbuf *b, uint64_t v, int nb) {
    wb_reserve(b, (uint64_t)nb);
    for (int i = 0; i < nb; ++i) b->p[b->n++] = (uint8_t)(v >> (8 * i));
}
static void wb_raw(wbuf *b, const void *src, uint64_t n) {
    wb_reserve(b, n);
    if (n) memcpy(b->p + b->n, src, n);
    b->n += n;
}
static uint64_t rd_le(const uint8_t *p, int nb) {
    uint64_t v = 0;
    for (int i = 0; i < nb; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
static double u64_to_f64(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}
static uint64_t f64_to_u64(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}

/* ------------------------------------------------------------------- grid */
/* grid.hpp:14-18 */
static int max_levels_for_cap(uint64_t cap) {
    int l = 1;
    while (l < 63 && ((uint64_t)1 << l) <= cap) ++l;
    return l;
}
/* grid.hpp:21-28 */
static int level_count(const uint64_t *dims, int nd, int max_levels) {
    uint64_t m = 1;
    for (int i = 0; i < nd; ++i)
        if (dims[i] > m) m = dims[i];
    int l = 1;
    while (((uint64_t)1 << l) < m && l < max_levels) ++l;
    return l;
}
static uint64_t lattice_count(uint64_t extent, uint64_t start, uint64_t step) { /* grid.hpp:114-117 */
    if (start >= extent) return 0;
    return (extent - 1 - start) / step + 1;
}

typedef struct {
    int axis;
    uint64_t start[4], step[4], cnt[4];
    uint64_t size;
} pass_t;

typedef struct {
    int nd, levels;
    uint64_t dims[4], strides[4], n;
} grid_t;

static int validate_dims(const uint64_t *dims, int nd, char *err, int errlen) { /* common.hpp:35-42 */
    if (nd < 1 || nd > 4) return fail(err, errlen, E_INVALID, "grid must have between 1 and 4 dimensions");
    for (int i = 0; i < nd; ++i)
        if (dims[i] < 1) return fail(err, errlen, E_INVALID, "grid extents must be positive");
    return E_OK;
}

static void grid_init(grid_t *g, const uint64_t *dims, int nd, int max_levels) {
    g->nd = nd;
    uint64_t acc = 1;
    for (int i = nd - 1; i >= 0; --i) { /* row_strides, common.hpp:45-53 */
        g->dims[i] = dims[i];
        g->strides[i] = acc;
        acc *= dims[i];
    }
    g->n = acc;
    g->levels = level_count(dims, nd, max_levels);
}

/* LevelTraversal::for_each pass boxes, grid.hpp:81-112 */
static int level_passes(const grid_t *g, int level, pass_t *out) {
    const uint64_t s = (uint64_t)1 << (level - 1);
    int np = 0;
    if (level == g->levels) {
        pass_t *p = &out[np];
        p->axis = -1;
        p->size = 1;
        for (int i = 0; i < g->nd; ++i) {
            p->start[i] = 0;
            p->step[i] = s;
            p->cnt[i] = lattice_count(g->dims[i], 0, s);
            p->size *= p->cnt[i];
        }
        if (p->size) ++np;
        return np;
    }
    for (int axis = 0; axis < g->nd; ++axis) {
        if (g->dims[axis] <= s) continue;
        pass_t *p = &out[np];
        p->axis = axis;
        p->size = 1;
        for (int i = 0; i < g->nd; ++i) {
            if (i < axis) {
                p->start[i] = 0;
                p->step[i] = s;
            } else if (i == axis) {
                p->start[i] = s;
                p->step[i] = 2 * s;
            } else {
                p->start[i] = 0;
                p->step[i] = 2 * s;
            }
            p->cnt[i] = lattice_count(g->dims[i], p->start[i], p->step[i]);
            p->size *= p->cnt[i];
        }
        if (p->size) ++np;
    }
    return np;
}

static uint64_t level_size(const grid_t *g, int level) { /* grid.hpp:58-79 */
    pass_t ps[4];
    int np = level_passes(g, level, ps);
    uint64_t t = 0;
    for (int i = 0; i < np; ++i) t += ps[i].size;
    return t;
}

/* row-major walk of one pass box, grid.hpp:124-156 */
typedef struct {
    const pass_t *p;
    int nd;
    uint64_t idx[4], step_flat[4];
    uint64_t flat;
    uint64_t coord_step, coord;
} walk_t;

static void walk_init(walk_t *w, const grid_t *g, const pass_t *p) {
    w->p = p;
    w->nd = g->nd;
    w->flat = 0;
    for (int i = 0; i < g->nd; ++i) {
        w->idx[i] = 0;
        w->step_flat[i] = p->step[i] * g->strides[i];
        w->flat += p->start[i] * g->strides[i];
    }
}
static uint64_t walk_coord(const walk_t *w) { return w->p->axis >= 0 ? w->p->start[w->p->axis] + w->idx[w->p->axis] * w->p->step[w->p->axis] : 0; }
static void walk_next(walk_t *w) {
    for (int d = w->nd - 1; d >= 0; --d) {
        ++w->idx[d];
        w->flat += w->step_flat[d];
        if (w->idx[d] < w->p->cnt[d]) return;
        w->flat -= w->idx[d] * w->step_flat[d];
        w->idx[d] = 0;
    }
}

/* ------------------------------------------------------------- quantizer */
static uint32_t to_negabinary(int32_t q) { /* quantizer.hpp:29-33 */
    return (uint32_t)((int64_t)q + (int64_t)NBMASK) ^ NBMASK;
}
static int32_t from_negabinary(uint32_t w) { return (int32_t)((w ^ NBMASK) - NBMASK); } /* :35-37 */

/* predictor.hpp:14-38 and quantizer.hpp:57-81, instantiated for float and double */
#define DEFINE_NUMERICS(T, SUF)                                                                          \
    static T predict_point_##SUF(const T *st, const grid_t *g, const walk_t *w, uint64_t s, int cubic) { \
        const int axis = w->p->axis;                                                                      \
        if (axis < 0) return (T)0;                                                                        \
        const uint64_t stp = s * g->strides[axis];                                                         \
        const uint64_t coord = walk_coord(w), extent = g->dims[axis], f = w->flat;                        \
        if (cubic && coord >= 3 * s && coord + 3 * s < extent) {                                          \
            const T a = st[f - 3 * stp], b = st[f - stp], c = st[f + stp], d = st[f + 3 * stp];          \
            return (T)(((T)9 * (b + c) - (a + d)) / (T)16);                                               \
        }                                                                                                 \
        if (coord + s < extent) return (T)((st[f - stp] + st[f + stp]) / (T)2);                          \
        return st[f - stp];                                                                               \
    }                                                                                                     \
    static T reconstruct_value_##SUF(T pred, double eb, int64_t code) {                                  \
        return (T)((double)pred + 2.0 * eb * (double)code);                                               \
    }                                                                                                     \
    static int quantize_residual_##SUF(T value, T pred, double eb, int32_t *code, T *recon) {            \
        const double y = (double)value - (double)pred;                                                    \
        if (isfinite(y)) {                                                                                \
            const double q = round(y / (2.0 * eb));                                                       \
            if (fabs(q) <= (double)KMAXCODE) {                                                            \
                const int32_t q0 = (int32_t)q;                                                            \
                const int64_t cands[3] = {(int64_t)q0, (int64_t)q0 - 1, (int64_t)q0 + 1};                 \
                for (int c = 0; c < 3; ++c) {                                                             \
                    if (cands[c] < -KMAXCODE || cands[c] > KMAXCODE) continue;                            \
                    const T r = reconstruct_value_##SUF(pred, eb, cands[c]);                              \
                    const double e = fabs((double)value - (double)r);                                     \
                    if (e <= eb) {                                                                        \
                        *code = (int32_t)cands[c];                                                        \
                        *recon = r;                                                                       \
                        return 0;                                                                         \
                    }                                                                                     \
                }                                                                                         \
            }                                                                                             \
        }                                                                                                 \
        *code = 0;                                                                                        \
        *recon = value;                                                                                   \
        return 1;                                                                                         \
    }

DEFINE_NUMERICS(float, f)
DEFINE_NUMERICS(double, d)

/* -------------------------------------------------------------- backend */
uint32_t orc_crc32(const uint8_t *p, uint64_t n) { /* backend.cpp:9-11 */
    uLong c = crc32(0L, Z_NULL, 0);
    while (n) {
        uInt chunk = n > (1u << 30) ? (1u << 30) : (uInt)n;
        c = crc32(c, p, chunk);
        p += chunk;
        n -= chunk;
    }
    return (uint32_t)c;
}

/* backend.cpp:34-53 (deflate = compress2 level 6, :15-22) */
int orc_backend_encode(const uint8_t *raw, uint64_t n, int preferred, uint8_t **payload, uint64_t *payload_len,
                       int *backend, uint32_t *crc) {
    if (preferred == 1 && n > 0) {
        uLongf cap = compressBound((uLong)n);
        uint8_t *out = (uint8_t *)malloc(cap ? cap : 1);
        int rc = compress2(out, &cap, raw, (uLong)n, 6);
        if (rc != Z_OK) {
            free(out);
            return E_RUNTIME;
        }
        if ((uint64_t)cap < n) {
            *payload = out;
            *payload_len = cap;
            *backend = 1;
            *crc = orc_crc32(out, cap);
            return E_OK;
        }
        free(out);
    }
    uint8_t *cp = (uint8_t *)malloc(n ? n : 1);
    if (n) memcpy(cp, raw, n);
    *payload = cp;
    *payload_len = n;
    *backend = 0;
    *crc = orc_crc32(cp, n);
    return E_OK;
}

/* write_block, backend.cpp:67-73 */
static void write_block(wbuf *w, int backend, uint64_t raw_bits, const uint8_t *payload, uint64_t len, uint32_t crc) {
    wb_put(w, (uint64_t)backend, 1);
    wb_put(w, raw_bits, 8);
    wb_put(w, len, 8);
    wb_put(w, crc, 4);
    wb_raw(w, payload, len);
}

/* ------------------------------------------------------------ loss table */
/* detail::measure_loss_table, pipeline.hpp:85-124 */
static void measure_loss_table(const grid_t *g, int level, int cubic, double eb, const int32_t *codes,
                               const uint32_t *nb, uint64_t count, double *dev, double table[33]) {
    uint32_t low_or = 0;
    for (uint64_t i = 0; i < count; ++i) low_or |= nb[i];
    const int coarsest = level == g->levels;
    const uint64_t s = (uint64_t)1 << (level - 1);
    const double unit = 2.0 * eb;
    double raw[33];
    memset(raw, 0, sizeof raw);
    pass_t ps[4];
    const int np = level_passes(g, level, ps);
    for (int d = 1; d <= 32; ++d) {
        const uint32_t low_mask = d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u);
        if ((low_or & low_mask) == 0) continue;
        double worst = 0.0;
        uint64_t i = 0;
        for (int pi = 0; pi < np; ++pi) {
            walk_t w;
            walk_init(&w, g, &ps[pi]);
            for (uint64_t k = 0; k < ps[pi].size; ++k, ++i) {
                const int64_t truncated = from_negabinary(nb[i] & ~low_mask);
                const double own = unit * (double)(truncated - (int64_t)codes[i]);
                const double v = coarsest ? own : predict_point_d(dev, g, &w, s, cubic) + own;
                dev[w.flat] = v;
                const double a = fabs(v);
                worst = (worst < a) ? a : worst; /* std::max */
                walk_next(&w);
            }
        }
        for (int pi = 0; pi < np; ++pi) { /* reset this level's points */
            walk_t w;
            walk_init(&w, g, &ps[pi]);
            for (uint64_t k = 0; k < ps[pi].size; ++k) {
                dev[w.flat] = 0.0;
                walk_next(&w);
            }
        }
        raw[d] = worst;
    }
    table[0] = 0.0;
    for (int d = 1; d <= 32; ++d) table[d] = (table[d - 1] < raw[d]) ? raw[d] : table[d - 1];
}

/* -------------------------------------------------------------- archive */
typedef struct {
    uint64_t count;
    double delta[33];
    uint64_t outlier_offset, outlier_length, outlier_count;
    uint64_t off[32], len[32];
} record_t;

typedef struct {
    int scalar, interp, levels, lp, anchor_cap, nd;
    uint64_t dims[4];
    double eb, range;
    uint64_t payload_bytes; /* derived */
} header_t;

static int check_header(const header_t *h, char *err, int errlen) { /* archive.cpp:12-21 */
    int rc = validate_dims(h->dims, h->nd, err, errlen);
    if (rc) return rc;
    if (h->levels < 1) return fail(err, errlen, E_RUNTIME, "archive has no levels");
    if (h->lp < 1 || h->lp > h->levels) return fail(err, errlen, E_RUNTIME, "progressive level bound out of range");
    if (!(h->eb > 0.0) || !isfinite(h->eb)) return fail(err, errlen, E_RUNTIME, "archive error bound is not positive");
    return E_OK;
}
static int check_record(const record_t *r, char *err, int errlen) { /* archive.cpp:23-28 */
    if (r->delta[0] != 0.0) return fail(err, errlen, E_RUNTIME, "loss table must start at zero");
    for (int d = 1; d <= 32; ++d)
        if (!(r->delta[d] >= r->delta[d - 1])) return fail(err, errlen, E_RUNTIME, "loss table must be non-decreasing");
    return E_OK;
}

/* serialize_index, archive.cpp:31-65 */
static int serialize_index(const header_t *h, const record_t *recs, wbuf *w, char *err, int errlen) {
    int rc = check_header(h, err, errlen);
    if (rc) return rc;
    wb_raw(w, "IPC1", 4);
    wb_put(w, 1, 2);
    wb_put(w, (uint64_t)h->scalar, 1);
    wb_put(w, (uint64_t)h->interp, 1);
    wb_put(w, (uint64_t)h->nd, 1);
    wb_put(w, 0, 1);
    wb_put(w, 0, 1);
    wb_put(w, 0, 1);
    for (int i = 0; i < h->nd; ++i) wb_put(w, h->dims[i], 8);
    wb_put(w, f64_to_u64(h->eb), 8);
    wb_put(w, (uint64_t)h->levels, 1);
    wb_put(w, (uint64_t)h->lp, 1);
    wb_put(w, (uint64_t)h->anchor_cap, 1);
    wb_put(w, 0, 1);
    wb_put(w, f64_to_u64(h->range), 8);
    for (int level = h->levels; level >= 1; --level) {
        const record_t *r = &recs[level - 1];
        rc = check_record(r, err, errlen);
        if (rc) return rc;
        wb_put(w, r->count, 8);
        for (int d = 0; d < 33; ++d) wb_put(w, f64_to_u64(r->delta[d]), 8);
        wb_put(w, r->outlier_offset, 8);
        wb_put(w, r->outlier_length, 8);
        wb_put(w, r->outlier_count, 8);
        for (int p = 0; p < 32; ++p) {
            wb_put(w, r->off[p], 8);
            wb_put(w, r->len[p], 8);
        }
    }
    return E_OK;
}

/* ------------------------------------------------------------- compress */
/* compress_field<T>, pipeline.hpp:140-223, followed by write_archive, archive.cpp:72-81 */
int orc_compress(int scalar, const void *values, const uint64_t *dims, int nd, double eb, int interp,
                 int progressive_levels, uint64_t anchor_cap, uint8_t **out, uint64_t *out_size, orc_trace *trace,
                 char *err, int errlen) {
    int rc = validate_dims(dims, nd, err, errlen);
    if (rc) return rc;
    if (!(eb > 0.0) || !isfinite(eb)) return fail(err, errlen, E_INVALID, "error bound must be positive and finite");
    grid_t g;
    grid_init(&g, dims, nd, max_levels_for_cap(anchor_cap));
    const int levels = g.levels;
    const int lp = progressive_levels == 0 ? levels : progressive_levels;
    if (lp < 1 || lp > levels) return fail(err, errlen, E_INVALID, "first progressive level out of range");
    const int w = scalar == 0 ? 4 : 8;
    const int cubic = interp == 1;
    const uint64_t n = g.n;

    double lo = INFINITY, hi = -INFINITY; /* pipeline.hpp:151-155, std::min/std::max */
    for (uint64_t i = 0; i < n; ++i) {
        const double v = scalar == 0 ? (double)((const float *)values)[i] : ((const double *)values)[i];
        lo = (v < lo) ? v : lo;
        hi = (hi < v) ? v : hi;
    }

    header_t h;
    memset(&h, 0, sizeof h);
    h.scalar = scalar;
    h.interp = interp;
    h.nd = nd;
    for (int i = 0; i < nd; ++i) h.dims[i] = dims[i];
    h.eb = eb;
    h.range = hi - lo;
    h.levels = levels;
    h.lp = lp;
    h.anchor_cap = (int)(uint8_t)anchor_cap;
    record_t *recs = (record_t *)calloc((size_t)levels, sizeof(record_t));

    void *state = calloc(n, (size_t)w);
    double *dev = (double *)calloc(n, sizeof(double));
    wbuf payload = {0};
    if (trace) {
        memset(trace, 0, sizeof *trace);
        trace->levels = levels;
    }

    for (int level = levels; level >= 1; --level) {
        const uint64_t count = level_size(&g, level);
        const uint64_t s = (uint64_t)1 << (level - 1);
        const int coarsest = level == levels;
        int32_t *codes = (int32_t *)malloc((count ? count : 1) * sizeof(int32_t));
        uint64_t *o_ord = NULL;
        wbuf ob = {0};
        uint64_t n_out = 0;
        pass_t ps[4];
        const int np = level_passes(&g, level, ps);
        uint64_t ordinal = 0;
        for (int pi = 0; pi < np; ++pi) {
            walk_t wk;
            walk_init(&wk, &g, &ps[pi]);
            for (uint64_t k = 0; k < ps[pi].size; ++k, ++ordinal) {
                int32_t code;
                int outl;
                if (scalar == 0) {
                    float *st = (float *)state;
                    const float v = ((const float *)values)[wk.flat];
                    const float pred = coarsest ? 0.0f : predict_point_f(st, &g, &wk, s, cubic);
                    float recon;
                    outl = quantize_residual_f(v, pred, eb, &code, &recon);
                    st[wk.flat] = outl ? v : recon;
                    if (outl) {
                        uint32_t bits;
                        memcpy(&bits, &v, 4);
                        wb_put(&ob, ordinal, 8);
                        wb_put(&ob, bits, 4);
                    }
                } else {
                    double *st = (double *)state;
                    const double v = ((const double *)values)[wk.flat];
                    const double pred = coarsest ? 0.0 : predict_point_d(st, &g, &wk, s, cubic);
                    double recon;
                    outl = quantize_residual_d(v, pred, eb, &code, &recon);
                    st[wk.flat] = outl ? v : recon;
                    if (outl) {
                        wb_put(&ob, ordinal, 8);
                        wb_put(&ob, f64_to_u64(v), 8);
                    }
                }
                if (outl) {
                    o_ord = (uint64_t *)realloc(o_ord, (n_out + 1) * sizeof(uint64_t));
                    o_ord[n_out++] = ordinal;
                }
                codes[ordinal] = code;
                walk_next(&wk);
            }
        }
        uint32_t *nb = (uint32_t *)malloc((count ? count : 1) * sizeof(uint32_t));
        for (uint64_t i = 0; i < count; ++i) nb[i] = to_negabinary(codes[i]); /* :195-196 */

        record_t *rec = &recs[level - 1];
        rec->count = count;
        measure_loss_table(&g, level, cubic, eb, codes, nb, count, dev, rec->delta); /* :200 */

        /* split + xor_encode, bitplane.cpp:7-22,44-49 */
        const uint64_t pb = (count + 7) / 8;
        uint8_t *planes = (uint8_t *)calloc(32 * (pb ? pb : 1), 1);
        for (uint64_t i = 0; i < count; ++i) {
            const uint32_t v = nb[i];
            if (!v) continue;
            for (int p = 0; p < 32; ++p)
                if ((v >> (31 - p)) & 1u) planes[(uint64_t)p * pb + (i >> 3)] |= (uint8_t)(1u << (i & 7));
        }
        for (int p = 31; p >= 1; --p) {
            for (uint64_t b = 0; b < pb; ++b) {
                uint8_t x = planes[(uint64_t)(p - 1) * pb + b];
                if (p >= 2) x ^= planes[(uint64_t)(p - 2) * pb + b];
                planes[(uint64_t)p * pb + b] ^= x;
            }
        }
        rec->outlier_offset = payload.n; /* :209-217 */
        rec->outlier_count = n_out;
        wb_raw(&payload, ob.p, ob.n);
        rec->outlier_length = payload.n - rec->outlier_offset;
        for (int p = 0; p < 32; ++p) {
            uint8_t *pl;
            uint64_t pll;
            int be;
            uint32_t crc;
            if (orc_backend_encode(planes + (uint64_t)p * pb, pb, 1, &pl, &pll, &be, &crc) != E_OK) {
                free(pl);
                return fail(err, errlen, E_RUNTIME, "deflate backend failed to compress");
            }
            rec->off[p] = payload.n;
            write_block(&payload, be, count, pl, pll, crc);
            rec->len[p] = payload.n - rec->off[p];
            free(pl);
        }
        if (trace) {
            const int li = level - 1;
            trace->count[li] = count;
            trace->codes[li] = codes;
            trace->negabinary[li] = nb;
            trace->n_outliers[li] = n_out;
            trace->outlier_ordinal[li] = o_ord;
            trace->outlier_bytes[li] = ob.p;
            trace->xor_planes[li] = planes;
            memcpy(trace->delta[li], rec->delta, sizeof rec->delta);
        } else {
            free(codes);
            free(nb);
            free(o_ord);
            free(ob.p);
            free(planes);
        }
    }
    free(state);
    free(dev);

    wbuf file = {0};
    rc = serialize_index(&h, recs, &file, err, errlen);
    if (rc == E_OK) wb_raw(&file, payload.p, payload.n);
    free(payload.p);
    free(recs);
    if (rc != E_OK) {
        free(file.p);
        return rc;
    }
    *out = file.p;
    *out_size = file.n;
    return E_OK;
}

void orc_trace_free(orc_trace *t) {
    for (int i = 0; i < ORC_MAX_LEVELS; ++i) {
        free(t->codes[i]);
        free(t->negabinary[i]);
        free(t->outlier_ordinal[i]);
        free(t->outlier_bytes[i]);
        free(t->xor_planes[i]);
    }
    memset(t, 0, sizeof *t);
}

/* ---------------------------------------------------------------- reader */
/* ArchiveReader, archive.cpp:117-200 */
typedef struct {
    const uint8_t *data;
    uint64_t size, pos, index_bytes, payload_read;
    header_t h;
    record_t recs[ORC_MAX_LEVELS];
    uint32_t identity;
} reader_t;

static int take(reader_t *r, uint64_t n, char *err, int errlen) {
    if (r->size - r->pos < n) return fail(err, errlen, E_RUNTIME, "truncated archive index");
    return E_OK;
}
#define TAKE(n)                                  \
    do {                                         \
        int _rc = take(r, (n), err, errlen);     \
        if (_rc) return _rc;                     \
    } while (0)

static int reader_open(reader_t *r, const uint8_t *data, uint64_t size, char *err, int errlen) {
    memset(r, 0, sizeof *r);
    r->data = data;
    r->size = size;
    TAKE(4);
    if (memcmp(data, "IPC1", 4) != 0) return fail(err, errlen, E_RUNTIME, "not an archive: bad magic");
    r->pos = 4;
    TAKE(2);
    if (rd_le(data + r->pos, 2) != 1) return fail(err, errlen, E_RUNTIME, "unsupported archive version");
    r->pos += 2;
    TAKE(1);
    const int scalar = data[r->pos++];
    if (scalar > 1) return fail(err, errlen, E_RUNTIME, "unknown scalar kind");
    TAKE(1);
    const int interp = data[r->pos++];
    if (interp > 1) return fail(err, errlen, E_RUNTIME, "unknown interpolation kind");
    TAKE(4);
    const int nd = data[r->pos];
    r->pos += 4;
    if (nd < 1 || nd > 4) return fail(err, errlen, E_RUNTIME, "dimension count out of range");
    header_t *h = &r->h;
    h->scalar = scalar;
    h->interp = interp;
    h->nd = nd;
    for (int i = 0; i < nd; ++i) {
        TAKE(8);
        h->dims[i] = rd_le(data + r->pos, 8);
        r->pos += 8;
    }
    TAKE(8 + 4 + 8);
    h->eb = u64_to_f64(rd_le(data + r->pos, 8));
    r->pos += 8;
    h->levels = data[r->pos];
    h->lp = data[r->pos + 1];
    h->anchor_cap = data[r->pos + 2];
    r->pos += 4;
    h->range = u64_to_f64(rd_le(data + r->pos, 8));
    r->pos += 8;
    int rc = check_header(h, err, errlen);
    if (rc) return rc;
    if (h->levels > ORC_MAX_LEVELS) return fail(err, errlen, E_RUNTIME, "too many levels");
    for (int level = h->levels; level >= 1; --level) {
        record_t *rec = &r->recs[level - 1];
        TAKE(8 * (1 + 33 + 3 + 64));
        const uint8_t *p = data + r->pos;
        rec->count = rd_le(p, 8);
        p += 8;
        for (int d = 0; d < 33; ++d, p += 8) rec->delta[d] = u64_to_f64(rd_le(p, 8));
        rec->outlier_offset = rd_le(p, 8);
        rec->outlier_length = rd_le(p + 8, 8);
        rec->outlier_count = rd_le(p + 16, 8);
        p += 24;
        for (int q = 0; q < 32; ++q, p += 16) {
            rec->off[q] = rd_le(p, 8);
            rec->len[q] = rd_le(p + 8, 8);
        }
        r->pos += 8 * (1 + 33 + 3 + 64);
        rc = check_record(rec, err, errlen);
        if (rc) return rc;
    }
    r->index_bytes = r->pos;
    r->identity = orc_crc32(data, r->pos);
    uint64_t end = 0;
    for (int l = 0; l < h->levels; ++l) {
        const record_t *rec = &r->recs[l];
        if (rec->outlier_offset + rec->outlier_length > end) end = rec->outlier_offset + rec->outlier_length;
        for (int q = 0; q < 32; ++q)
            if (rec->off[q] + rec->len[q] > end) end = rec->off[q] + rec->len[q];
    }
    h->payload_bytes = end;
    return E_OK;
}

/* read_range, archive.cpp:172-181 */
static int read_range(reader_t *r, uint64_t off, uint64_t len, const uint8_t **out, char *err, int errlen) {
    if (off + len > r->h.payload_bytes) return fail(err, errlen, E_RUNTIME, "block offset outside payload");
    if (r->index_bytes + off + len > r->size) return fail(err, errlen, E_RUNTIME, "truncated archive payload");
    *out = r->data + r->index_bytes + off;
    r->payload_read += len;
    return E_OK;
}

/* load_plane + read_block + backend_decode, archive.cpp:183-191, backend.cpp:55-65,75-86 */
static int load_plane_decoded(reader_t *r, int level, int plane, uint64_t count, uint8_t *dst, char *err, int errlen) {
    const record_t *rec = &r->recs[level - 1];
    const uint8_t *b;
    int rc = read_range(r, rec->off[plane], rec->len[plane], &b, err, errlen);
    if (rc) return rc;
    const uint64_t L = rec->len[plane];
    if (L < 1) return fail(err, errlen, E_RUNTIME, "truncated input while parsing");
    const int backend = b[0];
    if (backend > 1) return fail(err, errlen, E_RUNTIME, "unknown backend id");
    if (L < 21) return fail(err, errlen, E_RUNTIME, "truncated input while parsing");
    const uint64_t raw_bits = rd_le(b + 1, 8), plen = rd_le(b + 9, 8);
    const uint32_t crc = (uint32_t)rd_le(b + 17, 4);
    if (L - 21 < plen) return fail(err, errlen, E_RUNTIME, "truncated input while parsing");
    if (L - 21 != plen) return fail(err, errlen, E_RUNTIME, "plane block has trailing bytes");
    if (raw_bits != count) return fail(err, errlen, E_RUNTIME, "plane bit count does not match level");
    const uint8_t *payload = b + 21;
    if (orc_crc32(payload, plen) != crc) return fail(err, errlen, E_RUNTIME, "block checksum mismatch");
    const uint64_t rb = (raw_bits + 7) / 8;
    if (backend == 0) {
        if (plen != rb) return fail(err, errlen, E_RUNTIME, "identity block has wrong length");
        memcpy(dst, payload, rb);
        return E_OK;
    }
    uLongf dl = (uLongf)rb;
    uint8_t dummy;
    const int zrc = uncompress(rb ? dst : &dummy, &dl, payload, (uLong)plen);
    if (zrc != Z_OK || dl != rb) return fail(err, errlen, E_RUNTIME, "deflate backend failed to decompress block");
    return E_OK;
}

static int validate_plan(const header_t *h, const int *k, char *err, int errlen) { /* archive.cpp:202-211 */
    for (int level = 1; level <= h->levels; ++level) {
        const int kk = k[level - 1];
        if (kk < 0 || kk > 32) return fail(err, errlen, E_INVALID, "plan plane count out of range");
        if (level > h->lp && kk != 32) return fail(err, errlen, E_INVALID, "non-progressive levels must load all planes");
    }
    return E_OK;
}

/* decode planes [p0, p1) into merged codewords; xor_decode/merge, bitplane.cpp:24-59 (prefix from
 * merged digits when p0 > 0, as refine_field does, pipeline.hpp:328-339) */
static int decode_planes(reader_t *r, int level, int p0, int p1, uint64_t count, uint32_t *merged, char *err, int errlen) {
    const uint64_t pb = (count + 7) / 8;
    uint8_t *raw = (uint8_t *)malloc(pb ? pb : 1);
    for (int p = p0; p < p1; ++p) {
        int rc = load_plane_decoded(r, level, p, count, raw, err, errlen);
        if (rc) {
            free(raw);
            return rc;
        }
        const uint32_t digit = 1u << (31 - p);
        for (uint64_t i = 0; i < count; ++i) {
            uint32_t bit = (raw[i >> 3] >> (i & 7)) & 1u;
            if (p >= 1) bit ^= (merged[i] >> (32 - p)) & 1u;  /* digit 31-(p-1) */
            if (p >= 2) bit ^= (merged[i] >> (33 - p)) & 1u;  /* digit 31-(p-2) */
            if (bit) merged[i] |= digit;
        }
    }
    free(raw);
    return E_OK;
}

static int load_outliers(reader_t *r, int level, const uint8_t **ob, char *err, int errlen) { /* archive.cpp:193-200 */
    const record_t *rec = &r->recs[level - 1];
    const uint64_t entry = 8 + (r->h.scalar == 0 ? 4 : 8);
    if (rec->outlier_length != rec->outlier_count * entry)
        return fail(err, errlen, E_RUNTIME, "outlier block length does not match its count");
    return read_range(r, rec->outlier_offset, rec->outlier_length, ob, err, errlen);
}

/* detail::apply_level, pipeline.hpp:61-78 */
static void apply_level(void *state, int scalar, const grid_t *g, int level, int cubic, double eb, const uint32_t *merged,
                        const uint8_t *ob, uint64_t n_out) {
    const uint64_t s = (uint64_t)1 << (level - 1);
    const int coarsest = level == g->levels;
    const uint64_t entry = 8 + (scalar == 0 ? 4 : 8);
    uint64_t i = 0, oi = 0;
    pass_t ps[4];
    const int np = level_passes(g, level, ps);
    for (int pi = 0; pi < np; ++pi) {
        walk_t w;
        walk_init(&w, g, &ps[pi]);
        for (uint64_t k = 0; k < ps[pi].size; ++k, ++i) {
            const int64_t code = from_negabinary(merged[i]);
            const int hit = oi < n_out && rd_le(ob + oi * entry, 8) == i;
            if (scalar == 0) {
                float *st = (float *)state;
                const float pred = coarsest ? 0.0f : predict_point_f(st, g, &w, s, cubic);
                float v = reconstruct_value_f(pred, eb, code);
                if (hit) {
                    uint32_t bits = (uint32_t)rd_le(ob + oi * entry + 8, 4);
                    memcpy(&v, &bits, 4);
                }
                st[w.flat] = v;
            } else {
                double *st = (double *)state;
                const double pred = coarsest ? 0.0 : predict_point_d(st, g, &w, s, cubic);
                double v = reconstruct_value_d(pred, eb, code);
                if (hit) v = u64_to_f64(rd_le(ob + oi * entry + 8, 8));
                st[w.flat] = v;
            }
            if (hit) ++oi;
            walk_next(&w);
        }
    }
}

int orc_archive_info(const uint8_t *archive, uint64_t size, orc_info *info, char *err, int errlen) {
    reader_t r;
    int rc = reader_open(&r, archive, size, err, errlen);
    if (rc) return rc;
    memset(info, 0, sizeof *info);
    info->scalar = r.h.scalar;
    info->interp = r.h.interp;
    info->ndims = r.h.nd;
    info->levels = r.h.levels;
    info->progressive_levels = r.h.lp;
    info->anchor_cap = r.h.anchor_cap;
    for (int i = 0; i < r.h.nd; ++i) info->dims[i] = r.h.dims[i];
    info->eb = r.h.eb;
    info->range = r.h.range;
    info->index_bytes = r.index_bytes;
    info->payload_bytes = r.h.payload_bytes;
    info->identity = r.identity;
    for (int l = 0; l < r.h.levels; ++l) {
        info->count[l] = r.recs[l].count;
        memcpy(info->delta[l], r.recs[l].delta, sizeof(double) * 33);
        info->outlier_offset[l] = r.recs[l].outlier_offset;
        info->outlier_length[l] = r.recs[l].outlier_length;
        info->outlier_count[l] = r.recs[l].outlier_count;
        for (int p = 0; p < 32; ++p) {
            info->plane_offset[l][p] = r.recs[l].off[p];
            info->plane_length[l][p] = r.recs[l].len[p];
        }
    }
    return E_OK;
}

/* reconstruct_field<T>, pipeline.hpp:227-287 */
int orc_reconstruct(const uint8_t *archive, uint64_t size, int scalar, const int *k, void *out_values,
                    uint32_t **merged, uint64_t *payload_bytes_loaded, char *err, int errlen) {
    reader_t r;
    int rc = reader_open(&r, archive, size, err, errlen);
    if (rc) return rc;
    const header_t *h = &r.h;
    if (h->scalar != scalar) return fail(err, errlen, E_INVALID, "scalar kind does not match archive");
    rc = validate_plan(h, k, err, errlen);
    if (rc) return rc;
    grid_t g;
    grid_init(&g, h->dims, h->nd, max_levels_for_cap((uint64_t)h->anchor_cap));
    if (g.levels != h->levels) return fail(err, errlen, E_RUNTIME, "archive level count does not match its dimensions");
    memset(out_values, 0, g.n * (scalar == 0 ? 4 : 8));
    for (int l = 0; l < h->levels; ++l)
        if (merged) merged[l] = NULL;
    for (int level = h->levels; level >= 1; --level) {
        const uint64_t count = r.recs[level - 1].count;
        if (count != level_size(&g, level)) return fail(err, errlen, E_RUNTIME, "level point count does not match its dimensions");
        uint32_t *m = (uint32_t *)calloc(count ? count : 1, sizeof(uint32_t));
        rc = decode_planes(&r, level, 0, k[level - 1], count, m, err, errlen);
        const uint8_t *ob = NULL;
        if (!rc) rc = load_outliers(&r, level, &ob, err, errlen);
        if (rc) {
            free(m);
            return rc;
        }
        apply_level(out_values, scalar, &g, level, h->interp == 1, h->eb, m, ob, r.recs[level - 1].outlier_count);
        if (merged && level <= h->lp) merged[level - 1] = m;
        else free(m);
    }
    if (payload_bytes_loaded) *payload_bytes_loaded = r.payload_read;
    return E_OK;
}

/* refine_field<T>, pipeline.hpp:294-352 */
int orc_refine(const uint8_t *archive, uint64_t size, int scalar, const int *session_k,
               uint32_t *const *session_merged, const void *previous, const int *target_k, void *out_values,
               uint32_t **merged_out, uint64_t *payload_bytes_loaded, char *err, int errlen) {
    reader_t r;
    int rc = reader_open(&r, archive, size, err, errlen);
    if (rc) return rc;
    const header_t *h = &r.h;
    if (h->scalar != scalar) return fail(err, errlen, E_INVALID, "scalar kind does not match archive");
    rc = validate_plan(h, target_k, err, errlen);
    if (rc) return rc;
    grid_t g;
    grid_init(&g, h->dims, h->nd, max_levels_for_cap((uint64_t)h->anchor_cap));
    for (int level = 1; level <= h->levels; ++level)
        if (target_k[level - 1] < session_k[level - 1])
            return fail(err, errlen, E_INVALID, "refinement plan must not drop planes the session already loaded");
    const size_t w = scalar == 0 ? 4 : 8;
    memcpy(out_values, previous, g.n * w);
    for (int l = 0; l < h->levels; ++l) merged_out[l] = NULL;
    for (int level = h->levels; level >= 1; --level) {
        if (level > h->lp) continue;
        const uint64_t count = r.recs[level - 1].count;
        uint32_t *m = (uint32_t *)malloc((count ? count : 1) * sizeof(uint32_t));
        if (count) memcpy(m, session_merged[level - 1], count * sizeof(uint32_t));
        rc = decode_planes(&r, level, session_k[level - 1], target_k[level - 1], count, m, err, errlen);
        const uint8_t *ob = NULL;
        if (!rc) rc = load_outliers(&r, level, &ob, err, errlen);
        if (rc) {
            free(m);
            return rc;
        }
        apply_level(out_values, scalar, &g, level, h->interp == 1, h->eb, m, ob, r.recs[level - 1].outlier_count);
        merged_out[level - 1] = m;
    }
    if (payload_bytes_loaded) *payload_bytes_loaded = r.payload_read;
    return E_OK;
}

/* --------------------------------------------------------------- planner */
/* proj/src/planner.cpp */
typedef struct {
    int levels, lp;
    double eb, amp;
    double delta[ORC_MAX_LEVELS][33];
    uint64_t plane_bytes[ORC_MAX_LEVELS][32];
    uint64_t outlier_bytes[ORC_MAX_LEVELS];
} model_t;

static int build_model(const uint8_t *archive, uint64_t size, model_t *m, char *err, int errlen) { /* :30-45 */
    reader_t r;
    int rc = reader_open(&r, archive, size, err, errlen);
    if (rc) return rc;
    m->levels = r.h.levels;
    m->lp = r.h.lp;
    m->eb = r.h.eb;
    m->amp = r.h.interp == 1 ? 1.25 : 1.0; /* predictor.hpp:12 */
    for (int l = 0; l < r.h.levels; ++l) {
        memcpy(m->delta[l], r.recs[l].delta, sizeof(double) * 33);
        for (int p = 0; p < 32; ++p) m->plane_bytes[l][p] = r.recs[l].len[p];
        m->outlier_bytes[l] = r.recs[l].outlier_length;
    }
    return E_OK;
}
static double level_weight(const model_t *m, int level) { return pow(m->amp, level - 1); } /* :17-19 */
static uint64_t optional_bytes(const model_t *m, int level, int dropped) {                 /* :22-26 */
    uint64_t s = 0;
    for (int p = 0; p < 32 - dropped; ++p) s += m->plane_bytes[level - 1][p];
    return s;
}
static double bound_for_plan(const model_t *m, const int *k) { /* :51-58 */
    double sum = 0.0;
    for (int l = 1; l <= m->levels; ++l) sum += level_weight(m, l) * m->delta[l - 1][32 - k[l - 1]];
    return sum + m->eb;
}
static uint64_t mandatory_bytes(const model_t *m) { /* :60-67 */
    uint64_t s = 0;
    for (int l = 1; l <= m->levels; ++l) {
        s += m->outlier_bytes[l - 1];
        if (l > m->lp) s += optional_bytes(m, l, 0);
    }
    return s;
}
static uint64_t plan_bytes(const model_t *m, const int *k) { /* :75-81 */
    uint64_t s = mandatory_bytes(m);
    for (int l = 1; l <= m->lp; ++l) s += optional_bytes(m, l, 32 - k[l - 1]);
    return s;
}

typedef struct {
    int dropped, cost;
    uint64_t bytes;
    double err;
} choice_t;

double orc_bound_for_plan(const uint8_t *archive, uint64_t size, const int *k) {
    model_t m;
    if (build_model(archive, size, &m, NULL, 0)) return NAN;
    return bound_for_plan(&m, k);
}
uint64_t orc_plan_payload_bytes(const uint8_t *archive, uint64_t size, const int *k) {
    model_t m;
    if (build_model(archive, size, &m, NULL, 0)) return 0;
    return plan_bytes(&m, k);
}

/* plan_for_error, planner.cpp:93-200 */
int orc_plan_for_error(const uint8_t *archive, uint64_t size, double max_error, int *k, char *err, int errlen) {
    model_t m;
    int rc = build_model(archive, size, &m, err, errlen);
    if (rc) return rc;
    if (isnan(max_error) || max_error < m.eb)
        return fail(err, errlen, E_INFEASIBLE, "requested error bound is below the archive's compression bound");
    const double slack = max_error - m.eb;
    for (int l = 0; l < m.levels; ++l) k[l] = 32;
    const int lp = m.lp;
    if (lp == 0) return E_OK;
    choice_t cs[ORC_MAX_LEVELS][33];
    int nc[ORC_MAX_LEVELS];
    for (int l = 1; l <= lp; ++l) { /* error_mode_choices, :93-121 */
        const double w = level_weight(&m, l);
        nc[l - 1] = 0;
        for (int d = 0; d <= 32; ++d) {
            const double e = w * m.delta[l - 1][d];
            int cost;
            if (e <= 0.0) cost = 0;
            else if (isinf(slack)) cost = 0;
            else if (slack <= 0.0) cost = KINFCOST;
            else {
                const double units = ceil(e * (double)KBUCKETS / slack);
                cost = units > (double)KINFCOST ? KINFCOST : (int)units;
            }
            if (cost > KBUCKETS) continue;
            const uint64_t b = optional_bytes(&m, l, d);
            choice_t c = {d, cost, b, e};
            if (nc[l - 1] > 0 && cs[l - 1][nc[l - 1] - 1].cost == cost) cs[l - 1][nc[l - 1] - 1] = c;
            else cs[l - 1][nc[l - 1]++] = c;
        }
    }
    uint64_t(*best)[KBUCKETS + 1] = calloc((size_t)lp + 1, sizeof *best);
    for (int i = 1; i <= lp; ++i) {
        const uint64_t base = optional_bytes(&m, i, 0);
        for (int e = 0; e <= KBUCKETS; ++e) {
            uint64_t v = 0;
            int any = 0;
            for (int c = 0; c < nc[i - 1]; ++c) {
                const choice_t *ch = &cs[i - 1][c];
                if (ch->cost > e) continue;
                const uint64_t cand = best[i - 1][e - ch->cost] + (base - ch->bytes);
                if (!any || cand > v) {
                    v = cand;
                    any = 1;
                }
            }
            best[i][e] = v;
        }
    }
    int e = KBUCKETS;
    for (int i = lp; i >= 1; --i) {
        const uint64_t base = optional_bytes(&m, i, 0);
        const uint64_t want = best[i][e];
        int chosen = -1;
        for (int c = nc[i - 1] - 1; c >= 0; --c) {
            const choice_t *ch = &cs[i - 1][c];
            if (ch->cost > e) continue;
            if (best[i - 1][e - ch->cost] + (base - ch->bytes) == want) {
                chosen = c;
                k[i - 1] = 32 - ch->dropped;
                e -= ch->cost;
                break;
            }
        }
        if (chosen < 0) {
            free(best);
            return fail(err, errlen, E_RUNTIME, "plan reconstruction lost the optimum");
        }
    }
    free(best);
    while (bound_for_plan(&m, k) > max_error) {
        int worst = -1;
        double worst_err = 0.0;
        for (int l = 1; l <= lp; ++l) {
            const int d = 32 - k[l - 1];
            const double er = level_weight(&m, l) * m.delta[l - 1][d];
            if (d > 0 && er > worst_err) {
                worst_err = er;
                worst = l;
            }
        }
        if (worst < 0) break;
        k[worst - 1] += 1;
    }
    return E_OK;
}

/* plan_for_size, planner.cpp:202-290 */
typedef struct {
    double err;
    uint64_t bytes;
} value_t;
static int value_lt(value_t a, value_t b) { return a.err < b.err || (a.err == b.err && a.bytes < b.bytes); }

int orc_plan_for_size(const uint8_t *archive, uint64_t size, uint64_t byte_budget, int *k, char *err, int errlen) {
    model_t m;
    int rc = build_model(archive, size, &m, err, errlen);
    if (rc) return rc;
    const uint64_t mandatory = mandatory_bytes(&m);
    if (byte_budget < mandatory)
        return fail(err, errlen, E_INFEASIBLE,
                    "byte budget is below the mandatory payload (outliers and non-progressive levels)");
    const uint64_t budget = byte_budget - mandatory;
    for (int l = 0; l < m.levels; ++l) k[l] = 32;
    const int lp = m.lp;
    if (lp == 0) return E_OK;
    choice_t cs[ORC_MAX_LEVELS][33];
    int nc[ORC_MAX_LEVELS];
    for (int l = 1; l <= lp; ++l) {
        const double w = level_weight(&m, l);
        nc[l - 1] = 0;
        for (int d = 32; d >= 0; --d) {
            const uint64_t b = optional_bytes(&m, l, d);
            int cost;
            if (b == 0) cost = 0;
            else if (budget == 0) cost = KINFCOST;
            else {
                const uint64_t units = (b * KBUCKETS + budget - 1) / budget;
                cost = units > (uint64_t)KBUCKETS ? KINFCOST : (int)units;
            }
            if (cost > KBUCKETS) continue;
            const double e = w * m.delta[l - 1][d];
            choice_t c = {d, cost, b, e};
            if (nc[l - 1] > 0 && cs[l - 1][nc[l - 1] - 1].cost == cost) {
                if (e < cs[l - 1][nc[l - 1] - 1].err) cs[l - 1][nc[l - 1] - 1] = c;
            } else cs[l - 1][nc[l - 1]++] = c;
        }
        if (nc[l - 1] == 0) return fail(err, errlen, E_INFEASIBLE, "no loadable configuration fits the byte budget");
    }
    value_t(*best)[KBUCKETS + 1] = malloc(((size_t)lp + 1) * sizeof *best);
    for (int i = 0; i <= lp; ++i)
        for (int e = 0; e <= KBUCKETS; ++e) best[i][e] = (value_t){i == 0 ? 0.0 : INFINITY, 0};
    for (int i = 1; i <= lp; ++i) {
        for (int e = 0; e <= KBUCKETS; ++e) {
            value_t v = {INFINITY, 0};
            for (int c = 0; c < nc[i - 1]; ++c) {
                const choice_t *ch = &cs[i - 1][c];
                if (ch->cost > e) continue;
                const value_t prev = best[i - 1][e - ch->cost];
                if (isinf(prev.err)) continue;
                const value_t cand = {prev.err + ch->err, prev.bytes + ch->bytes};
                if (value_lt(cand, v)) v = cand;
            }
            best[i][e] = v;
        }
    }
    if (isinf(best[lp][KBUCKETS].err)) {
        free(best);
        return fail(err, errlen, E_INFEASIBLE, "no loadable configuration fits the byte budget");
    }
    int e = KBUCKETS;
    for (int i = lp; i >= 1; --i) {
        const value_t want = best[i][e];
        int found = 0;
        for (int c = 0; c < nc[i - 1]; ++c) {
            const choice_t *ch = &cs[i - 1][c];
            if (ch->cost > e) continue;
            const value_t prev = best[i - 1][e - ch->cost];
            if (isinf(prev.err)) continue;
            const value_t cand = {prev.err + ch->err, prev.bytes + ch->bytes};
            if (cand.err == want.err && cand.bytes == want.bytes) {
                k[i - 1] = 32 - ch->dropped;
                e -= ch->cost;
                found = 1;
                break;
            }
        }
        if (!found) {
            free(best);
            return fail(err, errlen, E_RUNTIME, "plan reconstruction lost the optimum");
        }
    }
    free(best);
    return E_OK;
}

/* ---------------------------------------------------------------- session */
/* write_session, session.cpp:8-23 */
int orc_write_session(uint32_t archive_crc, int levels, const int *k, uint32_t *const *merged, const uint64_t *counts,
                      uint8_t **out, uint64_t *out_size) {
    wbuf w = {0};
    wb_raw(&w, "IPS1", 4);
    wb_put(&w, archive_crc, 4);
    for (int l = levels; l >= 1; --l) {
        wb_put(&w, (uint64_t)k[l - 1], 1);
        const uint64_t cnt = merged[l - 1] ? counts[l - 1] : 0;
        wbuf codes = {0};
        for (uint64_t i = 0; i < cnt; ++i) wb_put(&codes, merged[l - 1][i], 4);
        uint8_t *pl;
        uint64_t pll;
        int be;
        uint32_t crc;
        orc_backend_encode(codes.p, codes.n, 1, &pl, &pll, &be, &crc);
        write_block(&w, be, codes.n * 8, pl, pll, crc);
        free(pl);
        free(codes.p);
    }
    *out = w.p;
    *out_size = w.n;
    return E_OK;
}

/* read_session, session.cpp:26-61 (ByteReader truncation: common.hpp:98; read_block:
 * backend.cpp:75-86; backend_decode: backend.cpp:55-65).  merged_out[l-1] is malloc'd for
 * progressive levels, NULL otherwise. */
int orc_read_session(const uint8_t *archive, uint64_t size, const uint8_t *bytes, uint64_t n, int *k_out,
                     uint32_t **merged_out, char *err, int errlen) {
    reader_t rd;
    int rc = reader_open(&rd, archive, size, err, errlen);
    if (rc) return rc;
    const int L = rd.h.levels, lp = rd.h.lp;
    for (int l = 0; l < ORC_MAX_LEVELS; ++l) merged_out[l] = NULL;
    const char *trunc = "truncated input while parsing";
    uint64_t pos = 0;
#define NEED(k)                                                                         \
    do {                                                                                \
        if (n - pos < (uint64_t)(k)) { rc = fail(err, errlen, E_RUNTIME, trunc); goto bad; } \
    } while (0)
    NEED(4);
    if (memcmp(bytes, "IPS1", 4) != 0) { rc = fail(err, errlen, E_RUNTIME, "not a session file: bad magic"); goto bad; }
    pos = 4;
    NEED(4);
    if ((uint32_t)rd_le(bytes + pos, 4) != rd.identity) {
        rc = fail(err, errlen, E_RUNTIME, "session does not belong to this archive");
        goto bad;
    }
    pos += 4;
    for (int level = L; level >= 1; --level) {
        NEED(1);
        const int k = bytes[pos++];
        k_out[level - 1] = k;
        if (k > 32) { rc = fail(err, errlen, E_RUNTIME, "session plane count out of range"); goto bad; }
        if (level > lp && k != 32) { rc = fail(err, errlen, E_RUNTIME, "session has partial non-progressive level"); goto bad; }
        NEED(1);
        const int backend = bytes[pos];
        pos += 1;
        if (backend > 1) { rc = fail(err, errlen, E_RUNTIME, "unknown backend id"); goto bad; }
        NEED(8);
        const uint64_t raw_bits = rd_le(bytes + pos, 8);
        pos += 8;
        NEED(8);
        const uint64_t plen = rd_le(bytes + pos, 8);
        pos += 8;
        NEED(4);
        const uint32_t crc = (uint32_t)rd_le(bytes + pos, 4);
        pos += 4;
        NEED(plen);
        const uint8_t *payload = bytes + pos;
        pos += plen;
        if (orc_crc32(payload, plen) != crc) { rc = fail(err, errlen, E_RUNTIME, "block checksum mismatch"); goto bad; }
        const uint64_t rb = (raw_bits + 7) / 8;
        uint8_t *raw = (uint8_t *)malloc(rb ? rb : 1);
        if (backend == 0) {
            if (plen != rb) { free(raw); rc = fail(err, errlen, E_RUNTIME, "identity block has wrong length"); goto bad; }
            memcpy(raw, payload, rb);
        } else {
            uLongf dl = (uLongf)rb;
            uint8_t dummy;
            const int zrc = uncompress(rb ? raw : &dummy, &dl, payload, (uLong)plen);
            if (zrc != Z_OK || dl != rb) {
                free(raw);
                rc = fail(err, errlen, E_RUNTIME, "deflate backend failed to decompress block");
                goto bad;
            }
        }
        if (level <= lp) {
            const uint64_t count = rd.recs[level - 1].count;
            if (rb != count * 4) { free(raw); rc = fail(err, errlen, E_RUNTIME, "session codeword array has wrong length"); goto bad; }
            uint32_t *m = (uint32_t *)malloc(count * 4 + 4);
            for (uint64_t i = 0; i < count; ++i) m[i] = (uint32_t)rd_le(raw + 4 * i, 4);
            merged_out[level - 1] = m;
        } else if (rb != 0) {
            free(raw);
            rc = fail(err, errlen, E_RUNTIME, "session stores codewords for a non-progressive level");
            goto bad;
        }
        free(raw);
    }
    if (pos != n) { rc = fail(err, errlen, E_RUNTIME, "session file has trailing bytes"); goto bad; }
    return E_OK;
#undef NEED
bad:
    for (int l = 0; l < ORC_MAX_LEVELS; ++l) {
        free(merged_out[l]);
        merged_out[l] = NULL;
    }
    return rc;
}

/* compute_metrics<T>, pipeline.hpp:354-372 (left-to-right double sum, std::max/std::min
 * semantics: a NaN operand never replaces the running value). out = {max_error, mse, psnr} */
int orc_compute_metrics(int scalar, const void *original, const void *decoded, uint64_t n, double *out) {
    double maxe = 0.0, lo = INFINITY, hi = -INFINITY, sq = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double a = scalar == 0 ? (double)((const float *)original)[i] : ((const double *)original)[i];
        const double b = scalar == 0 ? (double)((const float *)decoded)[i] : ((const double *)decoded)[i];
        const double diff = a - b;
        const double ad = fabs(diff);
        maxe = maxe < ad ? ad : maxe;
        sq += diff * diff;
        lo = a < lo ? a : lo;
        hi = hi < a ? a : hi;
    }
    out[0] = maxe;
    out[1] = n == 0 ? 0.0 : sq / (double)n;
    out[2] = out[1] == 0.0 ? INFINITY : 20.0 * log10((hi - lo) / sqrt(out[1]));
    return E_OK;
}
