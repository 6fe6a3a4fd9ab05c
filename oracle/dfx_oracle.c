/*
 * ORACLE / TEST INFRASTRUCTURE ONLY. See dfx_oracle.h for the contract.
 *
 * A plain-C restatement of the reference engine path. Arithmetic is done in
 * the reference's exact order (fp32, no FMA: built with -ffp-contract=off and
 * no -march, like the reference's x86-64 Release build) so results are
 * bit-identical to /root/reference/proj. Layout is the reference's: CHW
 * tensors and wrapped CHW planar spherical buffers. Every function cites the
 * reference lines (relative to /root/reference/proj) it restates.
 */
#include "dfx_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static _Thread_local char g_err[512];

#define FAIL(code, ...)                                    \
    do {                                                   \
        snprintf(g_err, sizeof g_err, __VA_ARGS__);        \
        return (code);                                     \
    } while (0)
#define CHECK(cond, ...)                                   \
    do {                                                   \
        if (!(cond)) FAIL(DFX_ERR, __VA_ARGS__);           \
    } while (0)
#define TRY(expr)                                          \
    do {                                                   \
        int _rc = (expr);                                  \
        if (_rc) return _rc;                               \
    } while (0)

const char* dfo_last_error(void) { return g_err; }

/* ----------------------------------------------------- integer helpers */
/* common.hpp:37-49 — mathematical floor div / mod for negative coords. */
static int64_t fdiv(int64_t a, int64_t n) {
    int64_t q = a / n;
    if ((a % n != 0) && ((a < 0) != (n < 0))) --q;
    return q;
}
static int64_t fmod64(int64_t a, int64_t n) {
    int64_t r = a % n;
    if (r != 0 && ((r < 0) != (n < 0))) r += n;
    return r;
}
static int64_t cdiv(int64_t a, int64_t n) { return -fdiv(-a, n); }
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static int min_i(int a, int b) { return a < b ? a : b; }
static int max_i(int a, int b) { return a > b ? a : b; }
/* std::max(a, b) == (a < b) ? b : a */
static float fmaxr(float a, float b) { return (a < b) ? b : a; }

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) {
        fprintf(stderr, "dfx_oracle: out of memory\n");
        abort();
    }
    return p;
}

/* ---------------------------------------------------------- tensors (CHW) */
typedef struct {
    int c, h, w;
    float* d;
} tens;

static tens tens_new(int c, int h, int w) {
    tens t = {c, h, w, (float*)xcalloc((size_t)c * h * w, sizeof(float))};
    return t;
}
static void tens_free(tens* t) {
    free(t->d);
    t->d = NULL;
}
#define T_AT(t, cc, yy, xx) ((t).d[((size_t)(cc) * (t).h + (yy)) * (t).w + (xx)])

/* ---------------------------------------------- spherical buffer (wrapped) */
/* tile_grid.hpp:88-128, tile_grid.cpp:5-92: CHW planar, pixel floor_mod wrap. */
typedef struct {
    int tile, rows, cols, c;
    int ph, pw;
    float* d;
} sbuf;

static void sbuf_init(sbuf* b, int tile, int rows, int cols, int c) {
    b->tile = tile;
    b->rows = rows;
    b->cols = cols;
    b->c = c;
    b->ph = rows * tile;
    b->pw = cols * tile;
    b->d = (float*)xcalloc((size_t)c * b->ph * b->pw, sizeof(float));
}
static void sbuf_free(sbuf* b) {
    free(b->d);
    b->d = NULL;
}
static size_t sbuf_idx(const sbuf* b, int c, int64_t gy, int64_t gx) {
    const int py = (int)fmod64(gy, b->ph);
    const int px = (int)fmod64(gx, b->pw);
    return ((size_t)c * b->ph + py) * b->pw + px;
}
static void sbuf_zero_all(sbuf* b) { memset(b->d, 0, sizeof(float) * (size_t)b->c * b->ph * b->pw); }
/* tile_grid.cpp:63-69 */
static void sbuf_zero_tile(sbuf* b, int64_t tx, int64_t ty) {
    for (int c = 0; c < b->c; ++c)
        for (int y = 0; y < b->tile; ++y)
            for (int x = 0; x < b->tile; ++x)
                b->d[sbuf_idx(b, c, ty * b->tile + y, tx * b->tile + x)] = 0.0f;
}
/* tile_grid.cpp:71-79 */
static void sbuf_fill_tile(sbuf* b, int64_t tx, int64_t ty, const float* per_c) {
    for (int c = 0; c < b->c; ++c)
        for (int y = 0; y < b->tile; ++y)
            for (int x = 0; x < b->tile; ++x)
                b->d[sbuf_idx(b, c, ty * b->tile + y, tx * b->tile + x)] = per_c[c];
}

/* --------------------------------------------------------------- geometry */
typedef struct {
    int64_t tx, ty; /* origin */
    int th, tw;
} place_t;

/* Dense grown packet (delta_layers.hpp:18-46): [c][eh+2h][ew+2h], mask th x tw. */
typedef struct {
    place_t pl;
    int tile, halo, c;
    int gh, gw;
    float* d;
    uint8_t* mask;
} pkt;

static pkt pkt_new(place_t pl, int tile, int c, int halo) {
    pkt p;
    p.pl = pl;
    p.tile = tile;
    p.halo = halo;
    p.c = c;
    p.gh = pl.th * tile + 2 * halo;
    p.gw = pl.tw * tile + 2 * halo;
    p.d = (float*)xcalloc((size_t)c * p.gh * p.gw, sizeof(float));
    p.mask = (uint8_t*)xcalloc((size_t)pl.th * pl.tw, 1);
    return p;
}
static void pkt_free(pkt* p) {
    free(p->d);
    free(p->mask);
    p->d = NULL;
    p->mask = NULL;
}
static pkt pkt_clone(const pkt* s) {
    pkt p = *s;
    p.d = (float*)xcalloc((size_t)s->c * s->gh * s->gw, sizeof(float));
    memcpy(p.d, s->d, sizeof(float) * (size_t)s->c * s->gh * s->gw);
    p.mask = (uint8_t*)xcalloc((size_t)s->pl.th * s->pl.tw, 1);
    memcpy(p.mask, s->mask, (size_t)s->pl.th * s->pl.tw);
    return p;
}
#define P_AT(p, cc, yy, xx) ((p).d[((size_t)(cc) * (p).gh + ((yy) + (p).halo)) * (p).gw + ((xx) + (p).halo)])
static int pkt_eh(const pkt* p) { return p->pl.th * p->tile; }
static int pkt_ew(const pkt* p) { return p->pl.tw * p->tile; }
/* delta_layers.hpp:37-41 */
static float pkt_sample(const pkt* p, int c, int y, int x) {
    if (y < -p->halo || y >= pkt_eh(p) + p->halo || x < -p->halo || x >= pkt_ew(p) + p->halo)
        return 0.0f;
    return P_AT(*p, c, y, x);
}

/* Output pixel bitmap over a grown extent (delta_layers.cpp:9-45). */
typedef struct {
    int halo, eh, ew, gh, gw;
    uint8_t* b;
} pixset;

static pixset pix_new(int halo, int eh, int ew) {
    pixset s = {halo, eh, ew, eh + 2 * halo, ew + 2 * halo, NULL};
    s.b = (uint8_t*)xcalloc((size_t)s.gh * s.gw, 1);
    return s;
}
#define PIX(s, yy, xx) ((s).b[(size_t)((yy) + (s).halo) * (s).gw + ((xx) + (s).halo)])

/* delta_layers.cpp:34-45: every output whose window [o*s-back, o*s-back+span)
 * meets the input rect [y0,y1) x [x0,x1). */
static void pix_mark_window(pixset* s, int y0, int y1, int x0, int x1, int span, int back,
                            int stride) {
    const int oy0 = max_i((int)fdiv(y0 + back - span, stride) + 1, -s->halo);
    const int oy1 = min_i((int)fdiv(y1 - 1 + back, stride), s->eh + s->halo - 1);
    const int ox0 = max_i((int)fdiv(x0 + back - span, stride) + 1, -s->halo);
    const int ox1 = min_i((int)fdiv(x1 - 1 + back, stride), s->ew + s->halo - 1);
    for (int y = oy0; y <= oy1; ++y)
        for (int x = ox0; x <= ox1; ++x) PIX(*s, y, x) = 1;
}
/* delta_layers.cpp:52-56 */
static int out_halo_of(int in_halo, int span, int back, int stride) {
    const int64_t lo = cdiv(in_halo + span - back, stride) - 1;
    const int64_t hi = cdiv(in_halo + back, stride);
    return (int)max64(0, max64(lo, hi));
}
/* delta_layers.cpp:60-70 */
static void pix_mark_sources(pixset* s, const pkt* in, int span, int back, int stride) {
    for (int tr = 0; tr < in->pl.th; ++tr)
        for (int tc = 0; tc < in->pl.tw; ++tc) {
            if (!in->mask[tr * in->pl.tw + tc]) continue;
            pix_mark_window(s, tr * in->tile - in->halo, (tr + 1) * in->tile + in->halo,
                            tc * in->tile - in->halo, (tc + 1) * in->tile + in->halo, span, back,
                            stride);
        }
}
/* delta_layers.cpp:72-83 */
static void pix_to_mask(const pixset* s, int th, int tw, int tile, uint8_t* m) {
    for (int tr = 0; tr < th; ++tr)
        for (int tc = 0; tc < tw; ++tc) {
            int any = 0;
            for (int y = tr * tile; y < (tr + 1) * tile && !any; ++y)
                for (int x = tc * tile; x < (tc + 1) * tile && !any; ++x)
                    if (PIX(*s, y, x)) any = 1;
            m[tr * tw + tc] = (uint8_t)any;
        }
}
static int64_t pix_count(const pixset* s) {
    int64_t n = 0;
    for (size_t i = 0; i < (size_t)s->gh * s->gw; ++i) n += s->b[i];
    return n;
}

/* -------------------------------------------------------------- network */
typedef struct {
    char name[64];
    int kind;
    int in0, in1; /* layer index, -1 = network input, -2 = none */
    int cin, cout, k, stride, pad;
    float* w;
    float* bias; /* NULL = none */
    int pool_k, pool_s, factor;
    float* bn_scale;
    float* bn_shift;
    int has_thr;
    float thr;
    int trunc_en;
    /* validate() facts (network.hpp:35-45) */
    int in_channels, channels, in_cum, cum, in_tile, tile, halo_in, halo_out;
    float* beta;
} layer_t;

typedef struct {
    sbuf acc, trunc;
    float thr;
    float* bias_init;
} tstate;
typedef struct {
    sbuf acc, prev;
    int k, s;
} pstate;

typedef struct {
    int used;
    int64_t tx, ty;
    int covered;
} slot_t;

struct dfo_engine {
    int in_channels, nl;
    layer_t* L;
    int* topo;
    int out_layer, ring;
    dfx_engine_config cfg;
    int initialized;
    int64_t frame_index;
    int rows, cols;
    /* ledger (buffer_manager.hpp:13-88) */
    slot_t* slots;
    int has_l, has_r, has_u, has_d;
    int64_t fl, fr, fu, fd;
    tstate in_st;
    tstate** ts; /* per layer or NULL */
    pstate** ps;
    /* last frame */
    pkt in_pkt;
    int have_in_pkt;
    pkt* outs; /* per layer */
    int* have_out;
    uint64_t* lflops;
    uint64_t* ldense;
    uint8_t* in_mask;
    int in_mask_th, in_mask_tw;
    int have_frame;
};

static int name_index(const dfo_engine* e, const char* name) {
    for (int i = 0; i < e->nl; ++i)
        if (strcmp(e->L[i].name, name) == 0) return i;
    return -1;
}

static float* dupf(const float* s, size_t n) {
    if (!s) return NULL;
    float* d = (float*)xcalloc(n, sizeof(float));
    memcpy(d, s, n * sizeof(float));
    return d;
}

/* network.cpp:46-254: topological order, per-layer tile/halo/beta, ring. */
static int validate_net(dfo_engine* e, const dfx_net_desc* nd, int tile_size) {
    CHECK(tile_size >= 1, "validate: tile size must be >= 1");
    CHECK(nd->in_channels >= 1, "validate: input channels must be >= 1");
    CHECK(nd->num_layers >= 1, "validate: network has no layers");
    const int n = nd->num_layers;
    e->nl = n;
    e->in_channels = nd->in_channels;
    e->L = (layer_t*)xcalloc(n, sizeof(layer_t));
    for (int i = 0; i < n; ++i) {
        const dfx_layer_desc* d = &nd->layers[i];
        layer_t* l = &e->L[i];
        CHECK(d->name && d->name[0] && strcmp(d->name, "input") != 0, "validate: bad layer name '%s'",
              d->name ? d->name : "");
        snprintf(l->name, sizeof l->name, "%s", d->name);
        for (int j = 0; j < i; ++j)
            CHECK(strcmp(e->L[j].name, l->name) != 0, "validate: duplicate layer name '%s'", l->name);
        l->kind = d->kind;
        const int want = d->kind == DFX_ADD ? 2 : 1;
        const int have = (d->input0 ? 1 : 0) + (d->input1 ? 1 : 0);
        if (have != want) FAIL(DFX_ERR_VALIDATION, "layer '%s' needs %d input(s)", l->name, want);
        l->cin = d->in_channels;
        l->cout = d->out_channels;
        l->k = d->kernel;
        l->stride = d->stride;
        l->pad = d->padding;
        if (d->kind == DFX_CONV) {
            l->w = dupf(d->weights, (size_t)d->out_channels * d->in_channels * d->kernel * d->kernel);
            l->bias = dupf(d->bias, (size_t)d->out_channels);
        }
        l->pool_k = d->pool_k;
        l->pool_s = d->pool_stride;
        l->factor = d->factor;
        if (d->kind == DFX_BATCHNORM) {
            l->bn_scale = dupf(d->bn_scale, (size_t)d->bn_channels);
            l->bn_shift = dupf(d->bn_shift, (size_t)d->bn_channels);
            l->cin = d->bn_channels;
        }
        l->has_thr = d->has_threshold;
        l->thr = d->threshold;
        l->trunc_en = d->truncate_enabled;
    }
    /* resolve input names */
    for (int i = 0; i < n; ++i) {
        const dfx_layer_desc* d = &nd->layers[i];
        const char* ins[2] = {d->input0, d->input1};
        int* dst[2] = {&e->L[i].in0, &e->L[i].in1};
        for (int j = 0; j < 2; ++j) {
            if (!ins[j]) {
                *dst[j] = -2;
                continue;
            }
            if (strcmp(ins[j], "input") == 0) {
                *dst[j] = -1;
                continue;
            }
            const int k = name_index(e, ins[j]);
            if (k < 0) FAIL(DFX_ERR_VALIDATION, "layer '%s' references unknown '%s'", e->L[i].name, ins[j]);
            *dst[j] = k;
        }
    }
    /* Kahn's algorithm (network.cpp:68-91): FIFO over consumers in index order. */
    int* indeg = (int*)xcalloc(n, sizeof(int));
    int* cons = (int*)xcalloc((size_t)n * 2, sizeof(int));
    int* ncons = (int*)xcalloc(n, sizeof(int));
    int* cons_off = (int*)xcalloc((size_t)n + 1, sizeof(int));
    for (int i = 0; i < n; ++i) {
        const int src[2] = {e->L[i].in0, e->L[i].in1};
        for (int j = 0; j < 2; ++j)
            if (src[j] >= 0) {
                ncons[src[j]]++;
                indeg[i]++;
            }
    }
    for (int i = 0; i < n; ++i) cons_off[i + 1] = cons_off[i] + ncons[i];
    memset(ncons, 0, sizeof(int) * n);
    for (int i = 0; i < n; ++i) {
        const int src[2] = {e->L[i].in0, e->L[i].in1};
        for (int j = 0; j < 2; ++j)
            if (src[j] >= 0) cons[cons_off[src[j]] + ncons[src[j]]++] = i;
    }
    int* queue = (int*)xcalloc(n, sizeof(int));
    int qh = 0, qt = 0;
    e->topo = (int*)xcalloc(n, sizeof(int));
    int nt = 0;
    for (int i = 0; i < n; ++i)
        if (indeg[i] == 0) queue[qt++] = i;
    while (qh < qt) {
        const int i = queue[qh++];
        e->topo[nt++] = i;
        for (int k = 0; k < ncons[i]; ++k) {
            const int c = cons[cons_off[i] + k];
            if (--indeg[c] == 0) queue[qt++] = c;
        }
    }
    free(indeg);
    free(cons);
    free(ncons);
    free(cons_off);
    free(queue);
    if (nt != n) FAIL(DFX_ERR_VALIDATION, "network graph has a cycle");

    /* network.cpp:95-211: per-layer facts. */
    float* in_beta = (float*)xcalloc((size_t)nd->in_channels, sizeof(float));
    int outputs = 0;
    for (int t = 0; t < n; ++t) {
        const int idx = e->topo[t];
        layer_t* o = &e->L[idx];
        int a_ch, a_cum, a_tile, a_halo;
        const float* a_beta;
        if (o->in0 == -1) {
            a_ch = nd->in_channels;
            a_cum = 1;
            a_tile = tile_size;
            a_halo = 0;
            a_beta = in_beta;
        } else {
            const layer_t* a = &e->L[o->in0];
            a_ch = a->channels;
            a_cum = a->cum;
            a_tile = a->tile;
            a_halo = a->halo_out;
            a_beta = a->beta;
        }
        o->in_channels = a_ch;
        o->in_cum = a_cum;
        o->in_tile = a_tile;
        o->halo_in = a_halo;
#define SET_CUM(cumv)                                                                         \
    do {                                                                                      \
        o->cum = (cumv);                                                                      \
        if (tile_size % o->cum != 0)                                                          \
            FAIL(DFX_ERR_VALIDATION,                                                          \
                 "layer '%s': tile size is not a multiple of the cumulative stride", o->name); \
        o->tile = max_i(1, tile_size / o->cum);                                               \
    } while (0)
        switch (o->kind) {
            case DFX_CONV: {
                CHECK(o->cin >= 1 && o->cout >= 1, "conv: channel counts must be >= 1");
                CHECK(o->k >= 1 && o->k % 2 == 1, "conv: kernel dims must be odd");
                CHECK(o->stride >= 1, "conv: stride must be >= 1");
                CHECK(o->pad >= 0, "conv: padding must be >= 0");
                if (o->cin != a_ch)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': expects %d channels, gets %d", o->name, o->cin, a_ch);
                if (o->pad != o->k / 2)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': engine convolutions need same-style padding", o->name);
                if (a_tile % o->stride != 0)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': stride misaligned with tile", o->name);
                o->channels = o->cout;
                SET_CUM(a_cum * o->stride);
                o->halo_out = out_halo_of(a_halo, o->k, o->k / 2, o->stride);
                /* network.cpp:137-150: beta' = bias + (sum_kernel W) * beta */
                o->beta = (float*)xcalloc((size_t)o->channels, sizeof(float));
                for (int oc = 0; oc < o->channels; ++oc) {
                    float v = o->bias ? o->bias[oc] : 0.0f;
                    for (int ic = 0; ic < o->cin; ++ic) {
                        float ws = 0.0f;
                        for (int ky = 0; ky < o->k; ++ky)
                            for (int kx = 0; kx < o->k; ++kx)
                                ws += o->w[(((size_t)oc * o->cin + ic) * o->k + ky) * o->k + kx];
                        v += ws * a_beta[ic];
                    }
                    o->beta[oc] = v;
                }
                break;
            }
            case DFX_RELU:
            case DFX_TRUNCATE:
            case DFX_OUTPUT:
                o->channels = a_ch;
                SET_CUM(a_cum);
                o->halo_out = 0;
                o->beta = (float*)xcalloc((size_t)o->channels, sizeof(float));
                if (o->kind == DFX_OUTPUT && ++outputs > 1)
                    FAIL(DFX_ERR_VALIDATION, "network has more than one output");
                break;
            case DFX_MAXPOOL:
            case DFX_AVGPOOL:
                if (o->pool_k != o->pool_s)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': engine pooling requires k == stride", o->name);
                if (o->pool_s < 1 || a_tile % o->pool_s != 0)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': stride misaligned with tile", o->name);
                o->channels = a_ch;
                SET_CUM(a_cum * o->pool_s);
                o->halo_out = out_halo_of(a_halo, o->pool_k, 0, o->pool_s);
                o->beta = dupf(a_beta, (size_t)a_ch);
                break;
            case DFX_UPSAMPLE:
                if (o->factor < 1 || a_cum % o->factor != 0)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': upsample factor does not divide cumulative stride", o->name);
                o->channels = a_ch;
                SET_CUM(a_cum / o->factor);
                o->halo_out = a_halo * o->factor;
                o->beta = dupf(a_beta, (size_t)a_ch);
                break;
            case DFX_BATCHNORM:
                if (o->cin != a_ch) FAIL(DFX_ERR_VALIDATION, "layer '%s': batchnorm param count", o->name);
                o->channels = a_ch;
                SET_CUM(a_cum);
                o->halo_out = a_halo;
                o->beta = (float*)xcalloc((size_t)a_ch, sizeof(float));
                for (int c = 0; c < a_ch; ++c) o->beta[c] = o->bn_scale[c] * a_beta[c] + o->bn_shift[c];
                break;
            case DFX_ADD: {
                int b_ch, b_cum, b_halo;
                const float* b_beta;
                if (o->in1 == -1) {
                    b_ch = nd->in_channels;
                    b_cum = 1;
                    b_halo = 0;
                    b_beta = in_beta;
                } else {
                    const layer_t* b = &e->L[o->in1];
                    b_ch = b->channels;
                    b_cum = b->cum;
                    b_halo = b->halo_out;
                    b_beta = b->beta;
                }
                if (a_ch != b_ch) FAIL(DFX_ERR_VALIDATION, "layer '%s': add channel mismatch", o->name);
                if (a_cum != b_cum)
                    FAIL(DFX_ERR_VALIDATION, "layer '%s': add joins branches of different cumulative stride", o->name);
                o->channels = a_ch;
                SET_CUM(a_cum);
                o->halo_out = max_i(a_halo, b_halo);
                o->beta = (float*)xcalloc((size_t)a_ch, sizeof(float));
                for (int c = 0; c < a_ch; ++c) o->beta[c] = a_beta[c] + b_beta[c];
                break;
            }
            default:
                FAIL(DFX_ERR_VALIDATION, "layer '%s': unknown kind %d", o->name, o->kind);
        }
#undef SET_CUM
    }
    free(in_beta);
    if (outputs != 1) FAIL(DFX_ERR_VALIDATION, "network needs exactly one output layer");
    /* network.cpp:216-227 */
    for (int i = 0; i < n; ++i) {
        int used = 0;
        for (int j = 0; j < n; ++j)
            if (e->L[j].in0 == i || e->L[j].in1 == i) used = 1;
        if (!used && e->L[i].kind != DFX_OUTPUT) FAIL(DFX_ERR_VALIDATION, "layer '%s' is dangling", e->L[i].name);
    }
    for (int i = 0; i < n; ++i)
        if (e->L[i].kind == DFX_OUTPUT) e->out_layer = i;
    /* network.cpp:229-252: stash ring width */
    int64_t ring = 1;
    for (int t = 0; t < n; ++t) {
        const layer_t* o = &e->L[e->topo[t]];
        if (o->kind == DFX_RELU || o->kind == DFX_TRUNCATE || o->kind == DFX_OUTPUT) {
            ring = max64(ring, cdiv(o->halo_in, o->in_tile));
        } else if (o->kind == DFX_MAXPOOL) {
            const int oh = out_halo_of(o->halo_in, o->pool_k, 0, o->pool_s);
            ring = max64(ring, cdiv(o->halo_in, o->in_tile));
            ring = max64(ring, cdiv(oh, o->tile));
            ring = max64(ring, cdiv((int64_t)oh * o->pool_s + o->pool_k, o->in_tile));
        }
    }
    e->ring = (int)ring;
    return 0;
}

/* ------------------------------------------------------------ homography */
/* alignment.hpp:11-32, alignment.cpp:5-56 */
static double hom_det(const float* m) {
    return (double)m[0] * ((double)m[4] * m[8] - (double)m[5] * m[7]) -
           (double)m[1] * ((double)m[3] * m[8] - (double)m[5] * m[6]) +
           (double)m[2] * ((double)m[3] * m[7] - (double)m[4] * m[6]);
}
static int hom_inverse(const float* a, float* r) {
    const double d = hom_det(a);
    CHECK(fabs(d) > 1e-9, "homography: singular matrix");
    const double inv = 1.0 / d;
    r[0] = (float)(((double)a[4] * a[8] - (double)a[5] * a[7]) * inv);
    r[1] = (float)(((double)a[2] * a[7] - (double)a[1] * a[8]) * inv);
    r[2] = (float)(((double)a[1] * a[5] - (double)a[2] * a[4]) * inv);
    r[3] = (float)(((double)a[5] * a[6] - (double)a[3] * a[8]) * inv);
    r[4] = (float)(((double)a[0] * a[8] - (double)a[2] * a[6]) * inv);
    r[5] = (float)(((double)a[2] * a[3] - (double)a[0] * a[5]) * inv);
    r[6] = (float)(((double)a[3] * a[7] - (double)a[4] * a[6]) * inv);
    r[7] = (float)(((double)a[1] * a[6] - (double)a[0] * a[7]) * inv);
    r[8] = (float)(((double)a[0] * a[4] - (double)a[1] * a[3]) * inv);
    return 0;
}
/* this ∘ inner, renormalised so m[8] == 1 (alignment.cpp:29-42). */
static void hom_compose(const float* m, const float* inner, float* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += (double)m[i * 3 + k] * inner[k * 3 + j];
            r[i * 3 + j] = (float)s;
        }
    if (r[8] != 0.0f && r[8] != 1.0f) {
        const float d = r[8];
        for (int i = 0; i < 8; ++i) r[i] /= d;
        r[8] /= r[8];
    }
}
static int hom_is_int_translation(const float* m, int64_t* dx, int64_t* dy) {
#define IS(v, t) (fabsf((v) - (t)) < 1e-6f)
    if (!IS(m[0], 1) || !IS(m[1], 0) || !IS(m[3], 0) || !IS(m[4], 1) || !IS(m[6], 0) || !IS(m[7], 0) ||
        !IS(m[8], 1))
        return 0;
#undef IS
    const float tx = m[2], ty = m[5];
    if (fabsf(tx - roundf(tx)) > 1e-4f || fabsf(ty - roundf(ty)) > 1e-4f) return 0;
    *dx = (int64_t)llroundf(tx);
    *dy = (int64_t)llroundf(ty);
    return 1;
}

/* alignment.cpp:58-104: inverse-mapping warp, exact integer path. */
static int warp_frame(const tens* f, const float* h, tens* img, tens* fp) {
    float inv[9];
    TRY(hom_inverse(h, inv));
    *img = tens_new(f->c, f->h, f->w);
    *fp = tens_new(1, f->h, f->w);
    int64_t idx, idy;
    if (hom_is_int_translation(h, &idx, &idy)) {
        for (int y = 0; y < f->h; ++y) {
            const int64_t sy = y - idy;
            if (sy < 0 || sy >= f->h) continue;
            for (int x = 0; x < f->w; ++x) {
                const int64_t sx = x - idx;
                if (sx < 0 || sx >= f->w) continue;
                for (int c = 0; c < f->c; ++c) T_AT(*img, c, y, x) = T_AT(*f, c, (int)sy, (int)sx);
                T_AT(*fp, 0, y, x) = 1.0f;
            }
        }
        return 0;
    }
    for (int y = 0; y < f->h; ++y)
        for (int x = 0; x < f->w; ++x) {
            const double xd = x, yd = y;
            const double w = (double)inv[6] * xd + (double)inv[7] * yd + (double)inv[8];
            CHECK(fabs(w) > 1e-12, "homography: point maps to infinity");
            const double sx = ((double)inv[0] * xd + (double)inv[1] * yd + (double)inv[2]) / w;
            const double sy = ((double)inv[3] * xd + (double)inv[4] * yd + (double)inv[5]) / w;
            if (sx < 0.0 || sx > f->w - 1 || sy < 0.0 || sy > f->h - 1) continue;
            const int x0 = (int)floor(sx), y0 = (int)floor(sy);
            const float fx = (float)(sx - x0), fy = (float)(sy - y0);
            const int x1 = min_i(x0 + 1, f->w - 1), y1 = min_i(y0 + 1, f->h - 1);
            for (int c = 0; c < f->c; ++c) {
                const float v00 = T_AT(*f, c, y0, x0), v01 = T_AT(*f, c, y0, x1);
                const float v10 = T_AT(*f, c, y1, x0), v11 = T_AT(*f, c, y1, x1);
                const float top = (1 - fx) * v00 + fx * v01;
                const float bot = (1 - fx) * v10 + fx * v11;
                T_AT(*img, c, y, x) = (1 - fy) * top + fy * bot;
            }
            T_AT(*fp, 0, y, x) = 1.0f;
        }
    return 0;
}

/* alignment.cpp:106-166: embed on the tile grid, crop to the buffer. */
typedef struct {
    tens img, valid;
    place_t pl;
    int64_t dropped;
} aligned_t;

static void snap(const tens* wimg, const tens* wfp, int64_t offx, int64_t offy, int tile,
                 int max_rows, int max_cols, aligned_t* out) {
    const int h = wimg->h, w = wimg->w;
    const int64_t ty0 = fdiv(offy, tile), tx0 = fdiv(offx, tile);
    const int my = (int)(offy - ty0 * tile), mx = (int)(offx - tx0 * tile);
    const int th = (int)cdiv(my + h, tile), tw = (int)cdiv(mx + w, tile);
    int drop_top = 0, drop_left = 0, nth = th, ntw = tw;
    if (max_rows > 0 && th > max_rows) {
        drop_top = (th - max_rows) / 2;
        nth = max_rows;
    }
    if (max_cols > 0 && tw > max_cols) {
        drop_left = (tw - max_cols) / 2;
        ntw = max_cols;
    }
    const int yo = drop_top * tile, xo = drop_left * tile;
    out->img = tens_new(wimg->c, nth * tile, ntw * tile);
    out->valid = tens_new(1, nth * tile, ntw * tile);
    int64_t total = 0, kept = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int cy = my + y - yo, cx = mx + x - xo;
            const int inside = cy >= 0 && cy < nth * tile && cx >= 0 && cx < ntw * tile;
            const float v = T_AT(*wfp, 0, y, x);
            if (v > 0.0f) {
                ++total;
                if (inside) ++kept;
            }
            if (!inside) continue;
            for (int c = 0; c < wimg->c; ++c) T_AT(out->img, c, cy, cx) = T_AT(*wimg, c, y, x);
            T_AT(out->valid, 0, cy, cx) = v;
        }
    out->dropped = (nth != th || ntw != tw) ? total - kept : 0;
    out->pl.tx = tx0 + drop_left;
    out->pl.ty = ty0 + drop_top;
    out->pl.th = nth;
    out->pl.tw = ntw;
}

/* ---------------------------------------------------------------- ledger */
static slot_t* slot_of(dfo_engine* e, int64_t tx, int64_t ty) {
    return &e->slots[fmod64(ty, e->rows) * e->cols + fmod64(tx, e->cols)];
}
/* buffer_manager.hpp:41-44 */
static int holds(dfo_engine* e, int64_t tx, int64_t ty) {
    const slot_t* s = slot_of(e, tx, ty);
    return s->used && s->tx == tx && s->ty == ty;
}
static void ledger_clear(dfo_engine* e) {
    memset(e->slots, 0, sizeof(slot_t) * (size_t)e->rows * e->cols);
    e->has_l = e->has_r = e->has_u = e->has_d = 0;
}

typedef struct {
    int64_t tx, ty;
    int evicts;
    int64_t etx, ety;
} claim_t;
typedef struct {
    int full_reset;
    int nclaims, nfresh, nevicted;
    claim_t* claims;
    int64_t* fresh; /* pairs tx, ty */
} plan_t;

/* buffer_manager.cpp:7-66 */
static void plan_frame(dfo_engine* e, place_t pl, int ring, plan_t* p) {
    memset(p, 0, sizeof *p);
    if ((e->has_l && pl.tx <= e->fl) || (e->has_r && pl.tx + pl.tw - 1 >= e->fr) ||
        (e->has_u && pl.ty <= e->fu) || (e->has_d && pl.ty + pl.th - 1 >= e->fd)) {
        p->full_reset = 1;
        return;
    }
    const int nslot = e->rows * e->cols;
    const int maxc = (pl.th + 2 * ring) * (pl.tw + 2 * ring);
    p->claims = (claim_t*)xcalloc((size_t)maxc, sizeof(claim_t));
    p->fresh = (int64_t*)xcalloc((size_t)pl.th * pl.tw * 2, sizeof(int64_t));
    uint8_t* planned = (uint8_t*)xcalloc((size_t)nslot, 1);
    for (int tr = 0; tr < pl.th; ++tr)
        for (int tc = 0; tc < pl.tw; ++tc) {
            const int64_t tx = pl.tx + tc, ty = pl.ty + tr;
            const slot_t* s = slot_of(e, tx, ty);
            planned[fmod64(ty, e->rows) * e->cols + fmod64(tx, e->cols)] = 1;
            if (!s->used) {
                p->claims[p->nclaims++] = (claim_t){tx, ty, 0, 0, 0};
                p->fresh[2 * p->nfresh] = tx;
                p->fresh[2 * p->nfresh++ + 1] = ty;
            } else if (s->tx == tx && s->ty == ty) {
                if (!s->covered) {
                    p->fresh[2 * p->nfresh] = tx;
                    p->fresh[2 * p->nfresh++ + 1] = ty;
                }
            } else {
                p->claims[p->nclaims++] = (claim_t){tx, ty, 1, s->tx, s->ty};
                p->fresh[2 * p->nfresh] = tx;
                p->fresh[2 * p->nfresh++ + 1] = ty;
                p->nevicted++;
            }
        }
    for (int tr = -ring; tr < pl.th + ring; ++tr)
        for (int tc = -ring; tc < pl.tw + ring; ++tc) {
            if (tr >= 0 && tr < pl.th && tc >= 0 && tc < pl.tw) continue;
            const int64_t tx = pl.tx + tc, ty = pl.ty + tr;
            const int64_t key = fmod64(ty, e->rows) * e->cols + fmod64(tx, e->cols);
            if (planned[key]) continue;
            planned[key] = 1;
            const slot_t* s = slot_of(e, tx, ty);
            if (!s->used) {
                p->claims[p->nclaims++] = (claim_t){tx, ty, 0, 0, 0};
            } else if (!(s->tx == tx && s->ty == ty)) {
                const int live = s->tx >= pl.tx && s->tx < pl.tx + pl.tw && s->ty >= pl.ty &&
                                 s->ty < pl.ty + pl.th;
                if (live) continue;
                p->claims[p->nclaims++] = (claim_t){tx, ty, 1, s->tx, s->ty};
                p->nevicted++;
            }
        }
    free(planned);
}
static void plan_free(plan_t* p) {
    free(p->claims);
    free(p->fresh);
}

static void zero_tile_everywhere(dfo_engine* e, int64_t tx, int64_t ty) {
    sbuf_zero_tile(&e->in_st.acc, tx, ty);
    sbuf_zero_tile(&e->in_st.trunc, tx, ty);
    for (int i = 0; i < e->nl; ++i) {
        if (e->ts[i]) {
            sbuf_zero_tile(&e->ts[i]->acc, tx, ty);
            sbuf_zero_tile(&e->ts[i]->trunc, tx, ty);
        }
        if (e->ps[i]) {
            sbuf_zero_tile(&e->ps[i]->acc, tx, ty);
            sbuf_zero_tile(&e->ps[i]->prev, tx, ty);
        }
    }
}

/* buffer_manager.hpp:61-69 + buffer_manager.cpp:68-81 */
static void apply_plan(dfo_engine* e, const plan_t* p, place_t pl) {
    for (int i = 0; i < p->nclaims; ++i) {
        const claim_t* c = &p->claims[i];
        if (c->evicts) {
            if (c->etx < pl.tx) {
                e->fl = e->has_l ? max64(e->fl, c->etx) : c->etx;
                e->has_l = 1;
            }
            if (c->etx > pl.tx + pl.tw - 1) {
                e->fr = e->has_r ? (e->fr < c->etx ? e->fr : c->etx) : c->etx;
                e->has_r = 1;
            }
            if (c->ety < pl.ty) {
                e->fu = e->has_u ? max64(e->fu, c->ety) : c->ety;
                e->has_u = 1;
            }
            if (c->ety > pl.ty + pl.th - 1) {
                e->fd = e->has_d ? (e->fd < c->ety ? e->fd : c->ety) : c->ety;
                e->has_d = 1;
            }
        }
        slot_t* s = slot_of(e, c->tx, c->ty);
        s->used = 1;
        s->tx = c->tx;
        s->ty = c->ty;
        s->covered = 0;
        zero_tile_everywhere(e, c->tx, c->ty);
    }
    for (int i = 0; i < p->nfresh; ++i) slot_of(e, p->fresh[2 * i], p->fresh[2 * i + 1])->covered = 1;
}

/* ------------------------------------------------------------ delta layers */
/* delta_layers.cpp:100-147 */
static void delta_conv(const layer_t* l, const pkt* in, pkt* out, uint64_t* flops, uint64_t* dense) {
    const int r = l->k / 2, s = l->stride;
    const int ot = in->tile / s;
    const int oh = out_halo_of(in->halo, l->k, r, s);
    *out = pkt_new(in->pl, ot, l->cout, oh);
    pixset tg = pix_new(oh, pkt_eh(out), pkt_ew(out));
    pix_mark_sources(&tg, in, l->k, r, s);
    for (int oy = -oh; oy < pkt_eh(out) + oh; ++oy)
        for (int ox = -oh; ox < pkt_ew(out) + oh; ++ox) {
            if (!PIX(tg, oy, ox)) continue;
            for (int o = 0; o < l->cout; ++o) {
                float acc = 0.0f;
                const float* wo = l->w + (size_t)o * l->cin * l->k * l->k;
                for (int i = 0; i < l->cin; ++i)
                    for (int ky = 0; ky < l->k; ++ky)
                        for (int kx = 0; kx < l->k; ++kx)
                            acc += pkt_sample(in, i, oy * s - r + ky, ox * s - r + kx) *
                                   wo[((size_t)i * l->k + ky) * l->k + kx];
                P_AT(*out, o, oy, ox) = acc;
            }
        }
    pix_to_mask(&tg, in->pl.th, in->pl.tw, ot, out->mask);
    const uint64_t per_px = 2ull * l->k * l->k * l->cin * l->cout;
    *flops = per_px * (uint64_t)pix_count(&tg);
    *dense = per_px * (uint64_t)pkt_eh(out) * (uint64_t)pkt_ew(out);
    free(tg.b);
}

/* delta_layers.cpp:149-232. gate != NULL overrides the threshold rule. */
static void delta_truncate(dfo_engine* e, const pkt* in, tstate* st, int relu, const uint8_t* gate,
                           pkt* out) {
    const int T = in->tile, eh = pkt_eh(in), ew = pkt_ew(in), C = in->c, h = in->halo;
    const int64_t gy0 = in->pl.ty * T, gx0 = in->pl.tx * T;
    *out = pkt_new(in->pl, T, C, 0);
    if (h > 0) {
        for (int y = -h; y < eh + h; ++y)
            for (int x = -h; x < ew + h; ++x) {
                if (y >= 0 && y < eh && x >= 0 && x < ew) {
                    x = ew - 1;
                    continue;
                }
                if (!holds(e, fdiv(gx0 + x, T), fdiv(gy0 + y, T))) continue;
                for (int c = 0; c < C; ++c) st->trunc.d[sbuf_idx(&st->trunc, c, gy0 + y, gx0 + x)] += P_AT(*in, c, y, x);
            }
    }
    for (int tr = 0; tr < in->pl.th; ++tr)
        for (int tc = 0; tc < in->pl.tw; ++tc) {
            if (!in->mask[tr * in->pl.tw + tc]) continue;
            if (!holds(e, in->pl.tx + tc, in->pl.ty + tr)) continue;
            const int y0 = tr * T, x0 = tc * T;
            float tmax = 0.0f;
            for (int c = 0; c < C; ++c)
                for (int y = y0; y < y0 + T; ++y)
                    for (int x = x0; x < x0 + T; ++x) {
                        const float cand = st->trunc.d[sbuf_idx(&st->trunc, c, gy0 + y, gx0 + x)] + P_AT(*in, c, y, x);
                        tmax = fmaxr(tmax, fabsf(cand));
                    }
            const int fire = gate ? gate[tr * in->pl.tw + tc] != 0 : (tmax >= st->thr && tmax > 0.0f);
            if (fire) {
                for (int c = 0; c < C; ++c)
                    for (int y = y0; y < y0 + T; ++y)
                        for (int x = x0; x < x0 + T; ++x) {
                            const size_t ix = sbuf_idx(&st->trunc, c, gy0 + y, gx0 + x);
                            const float cand = st->trunc.d[ix] + P_AT(*in, c, y, x);
                            const float prev = st->acc.d[ix];
                            const float acc = prev + cand;
                            st->acc.d[ix] = acc;
                            st->trunc.d[ix] = 0.0f;
                            P_AT(*out, c, y, x) = relu ? fmaxr(acc, 0.0f) - fmaxr(prev, 0.0f) : cand;
                        }
                out->mask[tr * in->pl.tw + tc] = 1;
            } else {
                for (int c = 0; c < C; ++c)
                    for (int y = y0; y < y0 + T; ++y)
                        for (int x = x0; x < x0 + T; ++x)
                            st->trunc.d[sbuf_idx(&st->trunc, c, gy0 + y, gx0 + x)] += P_AT(*in, c, y, x);
            }
        }
}

/* delta_layers.cpp:234-318 */
static void delta_maxpool(dfo_engine* e, const pkt* in, pstate* st, pkt* out) {
    const int k = st->k, s = st->s, T = in->tile, eh = pkt_eh(in), ew = pkt_ew(in), C = in->c;
    const int64_t gy0 = in->pl.ty * T, gx0 = in->pl.tx * T;
    for (int tr = 0; tr < in->pl.th; ++tr)
        for (int tc = 0; tc < in->pl.tw; ++tc) {
            if (!in->mask[tr * in->pl.tw + tc]) continue;
            if (!holds(e, in->pl.tx + tc, in->pl.ty + tr)) continue;
            for (int c = 0; c < C; ++c)
                for (int y = tr * T; y < (tr + 1) * T; ++y)
                    for (int x = tc * T; x < (tc + 1) * T; ++x)
                        st->acc.d[sbuf_idx(&st->acc, c, gy0 + y, gx0 + x)] += P_AT(*in, c, y, x);
        }
    if (in->halo > 0) {
        const int h = in->halo;
        for (int y = -h; y < eh + h; ++y)
            for (int x = -h; x < ew + h; ++x) {
                if (y >= 0 && y < eh && x >= 0 && x < ew) {
                    x = ew - 1;
                    continue;
                }
                if (!holds(e, fdiv(gx0 + x, T), fdiv(gy0 + y, T))) continue;
                for (int c = 0; c < C; ++c) st->acc.d[sbuf_idx(&st->acc, c, gy0 + y, gx0 + x)] += P_AT(*in, c, y, x);
            }
    }
    const int ot = T / s;
    const int oh = out_halo_of(in->halo, k, 0, s);
    *out = pkt_new(in->pl, ot, C, oh);
    pixset tg = pix_new(oh, pkt_eh(out), pkt_ew(out));
    pix_mark_sources(&tg, in, k, 0, s);
    const int64_t oy0 = in->pl.ty * ot, ox0 = in->pl.tx * ot;
    for (int oy = -oh; oy < pkt_eh(out) + oh; ++oy)
        for (int ox = -oh; ox < pkt_ew(out) + oh; ++ox) {
            if (!PIX(tg, oy, ox)) continue;
            if (!holds(e, fdiv(ox0 + ox, ot), fdiv(oy0 + oy, ot))) continue;
            for (int c = 0; c < C; ++c) {
                float m = 0.0f;
                int first = 1;
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) {
                        const int64_t iy = (oy0 + oy) * s + ky, ix = (ox0 + ox) * s + kx;
                        const float v = holds(e, fdiv(ix, T), fdiv(iy, T)) ? st->acc.d[sbuf_idx(&st->acc, c, iy, ix)] : 0.0f;
                        m = first ? v : fmaxr(m, v);
                        first = 0;
                    }
                float* prev = &st->prev.d[sbuf_idx(&st->prev, c, oy0 + oy, ox0 + ox)];
                P_AT(*out, c, oy, ox) = m - *prev;
                *prev = m;
            }
        }
    pix_to_mask(&tg, in->pl.th, in->pl.tw, ot, out->mask);
    free(tg.b);
}

/* delta_layers.cpp:320-349 */
static void delta_avgpool(const pkt* in, int k, int s, pkt* out) {
    const int ot = in->tile / s, oh = out_halo_of(in->halo, k, 0, s), C = in->c;
    *out = pkt_new(in->pl, ot, C, oh);
    pixset tg = pix_new(oh, pkt_eh(out), pkt_ew(out));
    pix_mark_sources(&tg, in, k, 0, s);
    const float inv = 1.0f / (float)(k * k);
    for (int oy = -oh; oy < pkt_eh(out) + oh; ++oy)
        for (int ox = -oh; ox < pkt_ew(out) + oh; ++ox) {
            if (!PIX(tg, oy, ox)) continue;
            for (int c = 0; c < C; ++c) {
                float sum = 0.0f;
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) sum += pkt_sample(in, c, oy * s + ky, ox * s + kx);
                P_AT(*out, c, oy, ox) = sum * inv;
            }
        }
    pix_to_mask(&tg, in->pl.th, in->pl.tw, ot, out->mask);
    free(tg.b);
}

/* delta_layers.cpp:351-363 */
static void delta_upsample(const pkt* in, int f, pkt* out) {
    *out = pkt_new(in->pl, in->tile * f, in->c, in->halo * f);
    const int oh = out->halo;
    for (int c = 0; c < in->c; ++c)
        for (int y = -oh; y < pkt_eh(out) + oh; ++y)
            for (int x = -oh; x < pkt_ew(out) + oh; ++x)
                P_AT(*out, c, y, x) = P_AT(*in, c, (int)fdiv(y, f), (int)fdiv(x, f));
    memcpy(out->mask, in->mask, (size_t)in->pl.th * in->pl.tw);
}

/* delta_layers.cpp:365-376 */
static void delta_bn(const pkt* in, const float* scale, pkt* out) {
    *out = pkt_clone(in);
    const size_t plane = (size_t)out->gh * out->gw;
    for (int c = 0; c < out->c; ++c)
        for (size_t i = 0; i < plane; ++i) out->d[(size_t)c * plane + i] *= scale[c];
}

/* delta_layers.cpp:378-393 */
static void delta_add(const pkt* a, const pkt* b, pkt* out) {
    const int h = max_i(a->halo, b->halo);
    *out = pkt_new(a->pl, a->tile, a->c, h);
    for (int c = 0; c < a->c; ++c)
        for (int y = -h; y < pkt_eh(out) + h; ++y)
            for (int x = -h; x < pkt_ew(out) + h; ++x)
                P_AT(*out, c, y, x) = pkt_sample(a, c, y, x) + pkt_sample(b, c, y, x);
    for (int i = 0; i < a->pl.th * a->pl.tw; ++i) out->mask[i] = (a->mask[i] || b->mask[i]) ? 1 : 0;
}

/* ------------------------------------------------------------ input stage */
/* alignment.cpp:198-224: separable window max, rows then columns, init 0. */
static void window_max(const float* in, int h, int w, int k, float* out) {
    const int lo = (k - 1) / 2, hi = k - 1 - lo;
    float* mid = (float*)xcalloc((size_t)h * w, sizeof(float));
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float m = 0.0f;
            for (int d = -lo; d <= hi; ++d) {
                const int xx = x + d;
                if (xx < 0 || xx >= w) continue;
                m = fmaxr(m, in[(size_t)y * w + xx]);
            }
            mid[(size_t)y * w + x] = m;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float m = 0.0f;
            for (int d = -lo; d <= hi; ++d) {
                const int yy = y + d;
                if (yy < 0 || yy >= h) continue;
                m = fmaxr(m, mid[(size_t)yy * w + x]);
            }
            out[(size_t)y * w + x] = m;
        }
    free(mid);
}

/* engine.cpp:110-182 (with roi_factor_map alignment.cpp:228-239 and
 * mask_dilate :295-300). raw: the input delta packet (halo 0). */
static void input_gate(dfo_engine* e, const pkt* raw, const plan_t* plan, const tens* roi,
                       uint8_t* gate) {
    const int eh = pkt_eh(raw), ew = pkt_ew(raw), T = raw->tile, C = raw->c;
    const int64_t gy0 = raw->pl.ty * T, gx0 = raw->pl.tx * T;
    const size_t npx = (size_t)eh * ew;
    float* sig = (float*)xcalloc(npx, sizeof(float));
    float* fac = NULL;
    if (roi) {
        float* d0 = (float*)xcalloc(npx, sizeof(float));
        float* d1 = (float*)xcalloc(npx, sizeof(float));
        float* d2 = (float*)xcalloc(npx, sizeof(float));
        window_max(roi->d, eh, ew, 10, d0);
        window_max(roi->d, eh, ew, 20, d1);
        window_max(roi->d, eh, ew, 40, d2);
        fac = (float*)xcalloc(npx, sizeof(float));
        for (size_t i = 0; i < npx; ++i) {
            const float m = (d0[i] + d1[i] + d2[i]) / 3.0f;
            fac[i] = 0.4f + 0.6f * m;
        }
        free(d0);
        free(d1);
        free(d2);
    }
    for (int y = 0; y < eh; ++y)
        for (int x = 0; x < ew; ++x) {
            float m = 0.0f;
            for (int c = 0; c < C; ++c) {
                const float cand = e->in_st.trunc.d[sbuf_idx(&e->in_st.trunc, c, gy0 + y, gx0 + x)] + P_AT(*raw, c, y, x);
                m = fmaxr(m, fabsf(cand));
            }
            if (fac) m *= fac[(size_t)y * ew + x];
            sig[(size_t)y * ew + x] = m > e->cfg.input_threshold ? 1.0f : 0.0f;
        }
    if (e->cfg.noise_suppression) {
        float* kept = (float*)xcalloc(npx, sizeof(float));
        for (int y = 0; y < eh; ++y)
            for (int x = 0; x < ew; ++x) {
                if (sig[(size_t)y * ew + x] == 0.0f) continue;
                int sup = 0;
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int yy = y + dy, xx = x + dx;
                        if (yy < 0 || yy >= eh || xx < 0 || xx >= ew) continue;
                        if (sig[(size_t)yy * ew + xx] > 0.0f) ++sup;
                    }
                if (sup >= 2) kept[(size_t)y * ew + x] = 1.0f;
            }
        free(sig);
        sig = kept;
    }
    if (e->cfg.mask_dilation > 0) {
        float* dil = (float*)xcalloc(npx, sizeof(float));
        window_max(sig, eh, ew, 2 * e->cfg.mask_dilation + 1, dil);
        free(sig);
        sig = dil;
    }
    for (int tr = 0; tr < raw->pl.th; ++tr)
        for (int tc = 0; tc < raw->pl.tw; ++tc) {
            gate[tr * raw->pl.tw + tc] = 0;
            if (!raw->mask[tr * raw->pl.tw + tc]) continue;
            int any = 0;
            for (int y = tr * T; y < (tr + 1) * T && !any; ++y)
                for (int x = tc * T; x < (tc + 1) * T && !any; ++x)
                    if (sig[(size_t)y * ew + x] > 0.0f) any = 1;
            gate[tr * raw->pl.tw + tc] = (uint8_t)any;
        }
    for (int i = 0; i < plan->nfresh; ++i) {
        const int tr = (int)(plan->fresh[2 * i + 1] - raw->pl.ty);
        const int tc = (int)(plan->fresh[2 * i] - raw->pl.tx);
        if (tr >= 0 && tr < raw->pl.th && tc >= 0 && tc < raw->pl.tw && raw->mask[tr * raw->pl.tw + tc])
            gate[tr * raw->pl.tw + tc] = 1;
    }
    free(sig);
    free(fac);
}

/* ---------------------------------------------------------------- engine */
static void tstate_free(tstate* t) {
    if (!t) return;
    sbuf_free(&t->acc);
    sbuf_free(&t->trunc);
    free(t->bias_init);
    free(t);
}

/* engine.cpp:33-76 */
static void allocate(dfo_engine* e, place_t first) {
    const int ring = e->cfg.padded_convolutions ? e->ring : 1;
    e->rows = e->cfg.grid_rows > 0 ? e->cfg.grid_rows : first.th + 2 * ring;
    e->cols = e->cfg.grid_cols > 0 ? e->cfg.grid_cols : first.tw + 2 * ring;
    e->slots = (slot_t*)xcalloc((size_t)e->rows * e->cols, sizeof(slot_t));
    const int T = e->cfg.tile_size;
    sbuf_init(&e->in_st.acc, T, e->rows, e->cols, e->in_channels);
    sbuf_init(&e->in_st.trunc, T, e->rows, e->cols, e->in_channels);
    e->in_st.thr = e->cfg.input_threshold;
    e->in_st.bias_init = (float*)xcalloc((size_t)e->in_channels, sizeof(float));
    for (int i = 0; i < e->nl; ++i) {
        const layer_t* l = &e->L[i];
        if (l->kind == DFX_RELU || l->kind == DFX_TRUNCATE || l->kind == DFX_OUTPUT) {
            float thr = 0.0f;
            if (l->kind != DFX_OUTPUT && l->trunc_en)
                thr = (e->cfg.override_net_thresholds || !l->has_thr) ? e->cfg.default_threshold : l->thr;
            tstate* t = (tstate*)xcalloc(1, sizeof(tstate));
            sbuf_init(&t->acc, l->in_tile, e->rows, e->cols, l->in_channels);
            sbuf_init(&t->trunc, l->in_tile, e->rows, e->cols, l->in_channels);
            t->thr = thr;
            t->bias_init = (float*)xcalloc((size_t)l->in_channels, sizeof(float));
            if (l->in0 >= 0) memcpy(t->bias_init, e->L[l->in0].beta, sizeof(float) * l->in_channels);
            e->ts[i] = t;
        } else if (l->kind == DFX_MAXPOOL) {
            pstate* p = (pstate*)xcalloc(1, sizeof(pstate));
            sbuf_init(&p->acc, l->in_tile, e->rows, e->cols, l->in_channels);
            sbuf_init(&p->prev, l->tile, e->rows, e->cols, l->in_channels);
            p->k = l->pool_k;
            p->s = l->pool_s;
            e->ps[i] = p;
        }
    }
    e->initialized = 1;
}

int dfo_reset(dfo_engine* e) {
    /* engine.cpp:93-108 */
    if (!e->initialized) return 0;
    ledger_clear(e);
    sbuf_zero_all(&e->in_st.acc);
    sbuf_zero_all(&e->in_st.trunc);
    for (int i = 0; i < e->nl; ++i) {
        if (e->ts[i]) {
            sbuf_zero_all(&e->ts[i]->acc);
            sbuf_zero_all(&e->ts[i]->trunc);
        }
        if (e->ps[i]) {
            sbuf_zero_all(&e->ps[i]->acc);
            sbuf_zero_all(&e->ps[i]->prev);
        }
    }
    return 0;
}

int dfo_create(const dfx_net_desc* net, const dfx_engine_config* cfg, dfo_engine** out) {
    dfo_engine* e = (dfo_engine*)xcalloc(1, sizeof(dfo_engine));
    e->cfg = *cfg;
    int rc = validate_net(e, net, cfg->tile_size);
    if (!rc && cfg->tile_size < 1) rc = DFX_ERR, snprintf(g_err, sizeof g_err, "engine: tile size must be >= 1");
    if (!rc && (cfg->input_threshold < 0.0f || cfg->default_threshold < 0.0f))
        rc = DFX_ERR, snprintf(g_err, sizeof g_err, "engine: thresholds must be >= 0");
    if (!rc && cfg->mask_dilation < 0)
        rc = DFX_ERR, snprintf(g_err, sizeof g_err, "engine: mask dilation must be >= 0");
    if (rc) {
        dfo_destroy(e);
        return rc;
    }
    e->ts = (tstate**)xcalloc((size_t)e->nl, sizeof(tstate*));
    e->ps = (pstate**)xcalloc((size_t)e->nl, sizeof(pstate*));
    e->outs = (pkt*)xcalloc((size_t)e->nl, sizeof(pkt));
    e->have_out = (int*)xcalloc((size_t)e->nl, sizeof(int));
    e->lflops = (uint64_t*)xcalloc((size_t)e->nl, sizeof(uint64_t));
    e->ldense = (uint64_t*)xcalloc((size_t)e->nl, sizeof(uint64_t));
    *out = e;
    return 0;
}

static void drop_packets(dfo_engine* e) {
    if (e->have_in_pkt) pkt_free(&e->in_pkt);
    e->have_in_pkt = 0;
    if (e->outs)
        for (int i = 0; i < e->nl; ++i)
            if (e->have_out[i]) {
                pkt_free(&e->outs[i]);
                e->have_out[i] = 0;
            }
}

void dfo_destroy(dfo_engine* e) {
    if (!e) return;
    drop_packets(e);
    if (e->L)
        for (int i = 0; i < e->nl; ++i) {
            layer_t* l = &e->L[i];
            free(l->w);
            free(l->bias);
            free(l->bn_scale);
            free(l->bn_shift);
            free(l->beta);
            if (e->ts) tstate_free(e->ts[i]);
            if (e->ps && e->ps[i]) {
                sbuf_free(&e->ps[i]->acc);
                sbuf_free(&e->ps[i]->prev);
                free(e->ps[i]);
            }
        }
    if (e->initialized) {
        sbuf_free(&e->in_st.acc);
        sbuf_free(&e->in_st.trunc);
        free(e->in_st.bias_init);
    }
    free(e->L);
    free(e->topo);
    free(e->ts);
    free(e->ps);
    free(e->outs);
    free(e->have_out);
    free(e->lflops);
    free(e->ldense);
    free(e->slots);
    free(e->in_mask);
    free(e);
}

/* engine.cpp:184-287 */
int dfo_run_frame(dfo_engine* e, const float* frame, int c, int h, int w, const float* h9,
                  const float* roi, dfx_frame_info* info, float* out, size_t out_cap) {
    CHECK(c == e->in_channels, "run_frame: input channel mismatch");
    const int T = e->cfg.tile_size;
    tens f = {c, h, w, (float*)frame};
    const int64_t offx = (int64_t)llroundf(h9[2]), offy = (int64_t)llroundf(h9[5]);
    const float tr[9] = {1, 0, (float)(-offx), 0, 1, (float)(-offy), 0, 0, 1};
    float res[9];
    hom_compose(tr, h9, res);
    tens wimg, wfp;
    TRY(warp_frame(&f, res, &wimg, &wfp));
    aligned_t al;
    snap(&wimg, &wfp, offx, offy, T, e->initialized ? e->rows : e->cfg.grid_rows,
         e->initialized ? e->cols : e->cfg.grid_cols, &al);
    tens_free(&wimg);
    tens_free(&wfp);
    if (!e->initialized) allocate(e, al.pl);

    drop_packets(e);
    memset(info, 0, sizeof *info);
    info->frame_index = e->frame_index;
    info->origin_tx = al.pl.tx;
    info->origin_ty = al.pl.ty;
    info->tiles_h = al.pl.th;
    info->tiles_w = al.pl.tw;
    info->dropped_pixels = al.dropped;

    const int ring = e->cfg.padded_convolutions ? e->ring : 0;
    plan_t plan;
    plan_frame(e, al.pl, ring, &plan);
    if (plan.full_reset) {
        dfo_reset(e);
        info->reset = 1;
        plan_free(&plan);
        plan_frame(e, al.pl, ring, &plan);
    }
    apply_plan(e, &plan, al.pl);
    for (int i = 0; i < e->nl; ++i) {
        tstate* t = e->ts[i];
        if (!t) continue;
        int any = 0;
        for (int k = 0; k < t->acc.c; ++k)
            if (t->bias_init[k] != 0.0f) any = 1;
        if (!any) continue;
        for (int k = 0; k < plan.nclaims; ++k) sbuf_fill_tile(&t->trunc, plan.claims[k].tx, plan.claims[k].ty, t->bias_init);
    }
    info->fresh = plan.nfresh;
    info->evicted = plan.nevicted;

    tens aroi = {0, 0, 0, NULL};
    if (e->cfg.roi_enabled && roi) {
        tens rf = {1, h, w, (float*)roi};
        tens ri, rfp;
        TRY(warp_frame(&rf, res, &ri, &rfp));
        aligned_t ar;
        snap(&ri, &rfp, offx, offy, T, e->rows, e->cols, &ar);
        tens_free(&ri);
        tens_free(&rfp);
        tens_free(&ar.valid);
        aroi = ar.img;
    }

    /* compute_input_delta, alignment.cpp:168-192 */
    pkt raw = pkt_new(al.pl, T, c, 0);
    {
        const int64_t gy0 = al.pl.ty * T, gx0 = al.pl.tx * T;
        for (int tr_ = 0; tr_ < al.pl.th; ++tr_)
            for (int tc = 0; tc < al.pl.tw; ++tc) {
                int cov = 0;
                for (int y = tr_ * T; y < (tr_ + 1) * T && !cov; ++y)
                    for (int x = tc * T; x < (tc + 1) * T && !cov; ++x)
                        if (T_AT(al.valid, 0, y, x) > 0.0f) cov = 1;
                if (!cov) continue;
                raw.mask[tr_ * al.pl.tw + tc] = 1;
                for (int ch = 0; ch < c; ++ch)
                    for (int y = tr_ * T; y < (tr_ + 1) * T; ++y)
                        for (int x = tc * T; x < (tc + 1) * T; ++x)
                            P_AT(raw, ch, y, x) = T_AT(al.img, ch, y, x) -
                                                  e->in_st.acc.d[sbuf_idx(&e->in_st.acc, ch, gy0 + y, gx0 + x)];
            }
    }
    uint8_t* gate = (uint8_t*)xcalloc((size_t)al.pl.th * al.pl.tw, 1);
    input_gate(e, &raw, &plan, aroi.d ? &aroi : NULL, gate);
    delta_truncate(e, &raw, &e->in_st, 0, gate, &e->in_pkt);
    e->have_in_pkt = 1;
    free(gate);
    pkt_free(&raw);
    tens_free(&aroi);
    plan_free(&plan);
    {
        int cnt = 0;
        for (int i = 0; i < al.pl.th * al.pl.tw; ++i) cnt += e->in_pkt.mask[i];
        info->update_rate = (double)cnt / ((double)al.pl.th * al.pl.tw);
        free(e->in_mask);
        e->in_mask = (uint8_t*)xcalloc((size_t)al.pl.th * al.pl.tw, 1);
        memcpy(e->in_mask, e->in_pkt.mask, (size_t)al.pl.th * al.pl.tw);
        e->in_mask_th = al.pl.th;
        e->in_mask_tw = al.pl.tw;
    }

    for (int i = 0; i < e->nl; ++i) e->lflops[i] = e->ldense[i] = 0;
    for (int t = 0; t < e->nl; ++t) {
        const int idx = e->topo[t];
        const layer_t* l = &e->L[idx];
        const pkt* a = l->in0 == -1 ? &e->in_pkt : &e->outs[l->in0];
        pkt o;
        switch (l->kind) {
            case DFX_CONV:
                delta_conv(l, a, &o, &e->lflops[idx], &e->ldense[idx]);
                info->conv_flops += e->lflops[idx];
                info->dense_flops += e->ldense[idx];
                if (!e->cfg.padded_convolutions && o.halo > 0) {
                    /* engine.cpp:254-264 control crop */
                    pkt cr = pkt_new(o.pl, o.tile, o.c, 0);
                    for (int ch = 0; ch < o.c; ++ch)
                        for (int y = 0; y < pkt_eh(&cr); ++y)
                            for (int x = 0; x < pkt_ew(&cr); ++x) P_AT(cr, ch, y, x) = P_AT(o, ch, y, x);
                    memcpy(cr.mask, o.mask, (size_t)o.pl.th * o.pl.tw);
                    pkt_free(&o);
                    o = cr;
                }
                break;
            case DFX_RELU: delta_truncate(e, a, e->ts[idx], 1, NULL, &o); break;
            case DFX_TRUNCATE:
            case DFX_OUTPUT: delta_truncate(e, a, e->ts[idx], 0, NULL, &o); break;
            case DFX_MAXPOOL: delta_maxpool(e, a, e->ps[idx], &o); break;
            case DFX_AVGPOOL: delta_avgpool(a, l->pool_k, l->pool_s, &o); break;
            case DFX_UPSAMPLE: delta_upsample(a, l->factor, &o); break;
            case DFX_BATCHNORM: delta_bn(a, l->bn_scale, &o); break;
            case DFX_ADD: {
                const pkt* b = l->in1 == -1 ? &e->in_pkt : &e->outs[l->in1];
                delta_add(a, b, &o);
                break;
            }
            default: FAIL(DFX_ERR, "unknown layer kind");
        }
        e->outs[idx] = o;
        e->have_out[idx] = 1;
    }

    /* densify, delta_layers.cpp:395-400, over the placement at output resolution */
    const tstate* os = e->ts[e->out_layer];
    const int ot = os->acc.tile;
    info->out_channels = os->acc.c;
    info->out_height = al.pl.th * ot;
    info->out_width = al.pl.tw * ot;
    const size_t need = (size_t)info->out_channels * info->out_height * info->out_width;
    if (out && out_cap >= need) {
        const int64_t gy0 = al.pl.ty * ot, gx0 = al.pl.tx * ot;
        for (int ch = 0; ch < info->out_channels; ++ch)
            for (int y = 0; y < info->out_height; ++y)
                for (int x = 0; x < info->out_width; ++x) {
                    const size_t ix = sbuf_idx(&os->acc, ch, gy0 + y, gx0 + x);
                    out[((size_t)ch * info->out_height + y) * info->out_width + x] = os->acc.d[ix] + os->trunc.d[ix];
                }
    }
    tens_free(&al.img);
    tens_free(&al.valid);
    e->have_frame = 1;
    e->frame_index++;
    return 0;
}

int dfo_input_mask(dfo_engine* e, uint8_t* out, size_t cap, int* th, int* tw) {
    CHECK(e->have_frame, "no frame");
    *th = e->in_mask_th;
    *tw = e->in_mask_tw;
    CHECK(cap >= (size_t)e->in_mask_th * e->in_mask_tw, "mask buffer too small");
    memcpy(out, e->in_mask, (size_t)e->in_mask_th * e->in_mask_tw);
    return 0;
}

int dfo_layer_flops(dfo_engine* e, const char* name, uint64_t* flops, uint64_t* dense) {
    const int i = name_index(e, name);
    *flops = i >= 0 ? e->lflops[i] : 0;
    *dense = i >= 0 ? e->ldense[i] : 0;
    return 0;
}

int dfo_grid(dfo_engine* e, int* rows, int* cols) {
    *rows = e->rows;
    *cols = e->cols;
    return 0;
}

static const sbuf* pick(dfo_engine* e, const char* layer, int which) {
    if (!e->initialized) return NULL;
    if (strcmp(layer, "input") == 0)
        return which == DFX_STATE_ACC ? &e->in_st.acc : which == DFX_STATE_TRUNC ? &e->in_st.trunc : NULL;
    const int i = name_index(e, layer);
    if (i < 0) return NULL;
    if (e->ts[i]) return which == DFX_STATE_ACC ? &e->ts[i]->acc : which == DFX_STATE_TRUNC ? &e->ts[i]->trunc : NULL;
    if (e->ps[i]) return which == DFX_STATE_ACC ? &e->ps[i]->acc : which == DFX_STATE_PREV ? &e->ps[i]->prev : NULL;
    return NULL;
}

int dfo_read_state(dfo_engine* e, const char* layer, int which, float* out, size_t cap, int* c,
                   int* h, int* w) {
    const sbuf* b = pick(e, layer, which);
    CHECK(b, "no state buffer for layer %s", layer);
    *c = b->c;
    *h = b->ph;
    *w = b->pw;
    const size_t n = (size_t)b->c * b->ph * b->pw;
    if (out) {
        CHECK(cap >= n, "state buffer too small");
        memcpy(out, b->d, n * sizeof(float));
    }
    return 0;
}

int dfo_read_packet(dfo_engine* e, const char* layer, float* out, size_t cap, int* c, int* gh,
                    int* gw, int* halo, uint8_t* mask, size_t mask_cap) {
    const pkt* p = NULL;
    if (strcmp(layer, "input") == 0) {
        if (e->have_in_pkt) p = &e->in_pkt;
    } else {
        const int i = name_index(e, layer);
        if (i >= 0 && e->have_out[i]) p = &e->outs[i];
    }
    CHECK(p, "no packet for layer %s", layer);
    *c = p->c;
    *gh = p->gh;
    *gw = p->gw;
    *halo = p->halo;
    if (out) {
        const size_t n = (size_t)p->c * p->gh * p->gw;
        CHECK(cap >= n && mask_cap >= (size_t)p->pl.th * p->pl.tw, "packet buffer too small");
        memcpy(out, p->d, n * sizeof(float));
        memcpy(mask, p->mask, (size_t)p->pl.th * p->pl.tw);
    }
    return 0;
}

int dfo_read_ledger(dfo_engine* e, int* used, int64_t* ty, int64_t* tx, uint8_t* covered,
                    size_t cap) {
    CHECK(e->initialized, "engine not initialized");
    const size_t n = (size_t)e->rows * e->cols;
    CHECK(cap >= n, "ledger buffer too small");
    for (size_t i = 0; i < n; ++i) {
        used[i] = e->slots[i].used;
        ty[i] = e->slots[i].ty;
        tx[i] = e->slots[i].tx;
        covered[i] = (uint8_t)e->slots[i].covered;
    }
    return 0;
}

int dfo_net_info(dfo_engine* e, int* ring, int* num_layers) {
    *ring = e->ring;
    *num_layers = e->nl;
    return 0;
}

int dfo_layer_info(dfo_engine* e, int layer, int* info7, float* beta, size_t beta_cap) {
    CHECK(layer >= 0 && layer < e->nl, "bad layer index");
    const layer_t* l = &e->L[layer];
    info7[0] = l->kind;
    info7[1] = l->in_channels;
    info7[2] = l->channels;
    info7[3] = l->in_tile;
    info7[4] = l->tile;
    info7[5] = l->halo_in;
    info7[6] = l->halo_out;
    if (beta && beta_cap >= (size_t)l->channels) memcpy(beta, l->beta, sizeof(float) * l->channels);
    return 0;
}
