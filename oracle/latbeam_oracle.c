/*
 * latbeam_oracle.c — serial CPU restatement of the reference decoder.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the CPU
 * baseline that bench.py times beside the GPU); the product path never links,
 * loads or calls it.  Every function names the reference lines it restates.
 *
 * Semantics (all bit-exact with the reference package `latbeam`):
 *   - candidate cost  (tok + w) + acrow[il-1] in f64          kernels.py:97-105, reference.py:110-125
 *   - pack            (enc32(float32(cost)) << 32) | arc       packing.py:37-61
 *   - recombination   strict-less pack wins, per state         decoder.py:189-205
 *   - cutoff          best (over ALL emitting candidates)+beam decoder.py:182-186, 533-539
 *   - epsilon rounds  Jacobi, snapshot frontier costs          reference.py:160-192
 *   - aggregation     state-sorted, eps pred -> index          decoder.py:330-370
 *   - lattice arcs    staged passes resolved at frame end      lattice.py:313-362
 *   - extra costs     backward relaxation, final terminus     lattice.py:365-497
 *   - finalisation    dense renumber + canonical lexsort       lattice.py:537-598
 *   - backtrace       words / alignment (bounded, see A.4)     decoder.py:614-641
 * Extension (not in the reference): max-active histogram cutoff,
 * specified in DESIGN.md §3; max_active = 0 reproduces the reference exactly.
 */
#define _GNU_SOURCE
#include "latbeam_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define SENT 0xFFFFFFFFFFFFFFFFull
#define MAX_ACTIVE_BINS 256
#define CONVERGE_TOL 1e-9
#define MAX_ACTIVE_BEAM_DELTA 0.5   /* Kaldi's beam_delta (adaptive beam after max-active) */

/* ---- packing (packing.py:37-61; kernels.py:51-67) ---- */
static inline uint64_t enc32(double c) {
    float f = (float)c;                     /* round-to-nearest, as np.float32 */
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? (uint64_t)(~u) : (uint64_t)(u | 0x80000000u);
}
static inline uint64_t pack_word(double c, int64_t arc) {
    return (enc32(c) << 32) | (uint64_t)(uint32_t)arc;
}

/* ---- growable vectors ---- */
#define VEC(T, name) T *name; int64_t name##_n, name##_cap
#define VPUSH(name, v)                                                      \
    do {                                                                    \
        if (name##_n == name##_cap) {                                       \
            name##_cap = name##_cap ? 2 * name##_cap : 1024;                \
            name = realloc(name, (size_t)name##_cap * sizeof(*name));       \
        }                                                                   \
        name[name##_n++] = (v);                                             \
    } while (0)

typedef struct {
    int64_t S;
    uint64_t *pack;
    double *cost;
    int64_t *pred;        /* emit: prev token index; eps: source state */
    int32_t *touched;
    int64_t ntouched;
    int64_t *pos;         /* state -> sorted index in the current frame */
    int32_t *pos_stamp;
    int32_t stamp;
    int32_t *tag;         /* per-round improved dedup (decoder.py:214-222 `seen`) */
    int32_t round;
    int32_t *fs, *fs2, *imp;
    double *fc, *fc2;
    double *acrow;
    int32_t D;
} ws_t;

static ws_t *ws_alloc(int64_t S, int32_t D) {
    ws_t *w = calloc(1, sizeof(ws_t));
    w->S = S;
    w->pack = malloc((size_t)S * 8);
    memset(w->pack, 0xFF, (size_t)S * 8);
    w->cost = malloc((size_t)S * 8);
    w->pred = malloc((size_t)S * 8);
    w->touched = malloc((size_t)S * 4);
    w->pos = malloc((size_t)S * 8);
    w->pos_stamp = calloc((size_t)S, 4);
    w->tag = calloc((size_t)S, 4);
    w->fs = malloc((size_t)S * 4);
    w->fs2 = malloc((size_t)S * 4);
    w->imp = malloc((size_t)S * 4);
    w->fc = malloc((size_t)S * 8);
    w->fc2 = malloc((size_t)S * 8);
    w->acrow = malloc((size_t)(D > 0 ? D : 1) * 8);
    w->D = D;
    return w;
}

static void ws_free(ws_t *w) {
    if (!w) return;
    free(w->pack); free(w->cost); free(w->pred); free(w->touched); free(w->pos);
    free(w->pos_stamp); free(w->tag); free(w->fs); free(w->fs2); free(w->imp);
    free(w->fc); free(w->fc2); free(w->acrow); free(w);
}

static void ws_reset_frame(ws_t *w) {   /* decoder.py:123-126, O(touched) */
    for (int64_t k = 0; k < w->ntouched; k++) w->pack[w->touched[k]] = SENT;
    w->ntouched = 0;
}

static inline void offer(ws_t *w, int32_t v, uint64_t word, double cand, int64_t pred, int *improved) {
    /* recombine (decoder.py:189-205): strict-less pack wins */
    if (word < w->pack[v]) {
        if (w->pack[v] == SENT) w->touched[w->ntouched++] = v;
        w->pack[v] = word;
        w->cost[v] = cand;
        w->pred[v] = pred;
        *improved = 1;
    } else {
        *improved = 0;
    }
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

typedef struct {
    int32_t a, u;
    double cand;
} eps_stage_t;

static int cmp_eps_stage(const void *pa, const void *pb) {
    const eps_stage_t *x = pa, *y = pb;
    if (x->a != y->a) return (x->a > y->a) - (x->a < y->a);
    return (x->cand > y->cand) - (x->cand < y->cand);
}

typedef struct {
    int32_t a, from, to;
    double ac;
} lat_arc_t;

static int cmp_lat_arc(const void *pa, const void *pb) {
    const lat_arc_t *x = pa, *y = pb;
    if (x->a != y->a) return (x->a > y->a) - (x->a < y->a);
    if (x->from != y->from) return (x->from > y->from) - (x->from < y->from);
    return (x->to > y->to) - (x->to < y->to);
}

typedef struct {
    /* per-utterance outputs under construction */
    VEC(int32_t, ts); VEC(double, tc); VEC(int64_t, tpa); VEC(int64_t, tpi); VEC(uint64_t, tp);
    VEC(int64_t, toff);
    VEC(double, cut);
    VEC(lat_arc_t, la);
    VEC(int64_t, loff);
    /* staging (per frame) */
    VEC(int32_t, em_a); VEC(int32_t, em_i); VEC(double, em_c); VEC(double, em_ac);
    VEC(eps_stage_t, ep);
    VEC(int32_t, kept);
    int64_t cnt[8];
} run_t;

static void run_free(run_t *r) {
    free(r->ts); free(r->tc); free(r->tpa); free(r->tpi); free(r->tp); free(r->toff);
    free(r->cut); free(r->la); free(r->loff); free(r->em_a); free(r->em_i); free(r->em_c);
    free(r->em_ac); free(r->ep); free(r->kept);
}

static int fail(lbo_result *out, int code, const char *bound, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(out->msg, sizeof(out->msg), fmt, ap);
    va_end(ap);
    out->status = code;
    snprintf(out->bound, sizeof(out->bound), "%s", bound ? bound : "");
    return code;
}

/* ---- epsilon fixpoint: decoder.py:267-311 / reference.py:160-192 ----
 * Frontier (w->fs, w->fc, nf) holds (state, snapshot cost).  Jacobi rounds. */
static int eps_fixpoint(ws_t *w, const lbo_graph *g, double cutoff, int64_t nf, int stage,
                        run_t *r, lbo_result *out) {
    int64_t rounds = 0;
    while (nf > 0) {
        if (++rounds > g->S + 1)
            return fail(out, LBO_INTERNAL, NULL,
                        "epsilon relaxation failed to settle within the state count");
        w->round++;
        int64_t nimp = 0;
        for (int64_t k = 0; k < nf; k++) {
            int32_t u = w->fs[k];
            double cu = w->fc[k];
            r->cnt[3]++;
            for (int64_t a = g->off[u]; a < g->off[u + 1]; a++) {
                if (g->il[a] != 0) continue;
                r->cnt[4]++;
                double cand = cu + g->w[a];
                if (cand > cutoff) continue;
                r->cnt[5]++;
                if (stage) {
                    eps_stage_t s = {(int32_t)a, u, cand};
                    VPUSH(r->ep, s);
                }
                int32_t v = g->dst[a];
                int imp;
                offer(w, v, pack_word(cand, a), cand, u, &imp);
                if (imp && w->tag[v] != w->round) {
                    w->tag[v] = w->round;
                    w->imp[nimp++] = v;
                }
            }
        }
        qsort(w->imp, (size_t)nimp, 4, cmp_i32);    /* reference.py:191 sorted frontier */
        for (int64_t k = 0; k < nimp; k++) {
            w->fs2[k] = w->imp[k];
            w->fc2[k] = w->cost[w->imp[k]];
        }
        int32_t *ts = w->fs; w->fs = w->fs2; w->fs2 = ts;
        double *tc = w->fc; w->fc = w->fc2; w->fc2 = tc;
        nf = nimp;
    }
    return 0;
}

/* max-active cutoff: histogram of the seed costs over
 * [best, best+beam] in MAX_ACTIVE_BINS bins; H = best + max(b*,1)*width where
 * b* is the first bin whose inclusive running count exceeds max_active. */
static double max_active_cutoff(const double *costs, int64_t n, double best, double beam,
                                int64_t max_active, double cutoff) {
    if (max_active <= 0 || n <= max_active) return cutoff;
    int64_t hist[MAX_ACTIVE_BINS];
    memset(hist, 0, sizeof(hist));
    double width = beam / (double)MAX_ACTIVE_BINS;
    for (int64_t k = 0; k < n; k++) {
        double q = (costs[k] - best) / width;
        int b = q >= (double)MAX_ACTIVE_BINS ? MAX_ACTIVE_BINS - 1 : (int)q;
        if (b < 0) b = 0;
        hist[b]++;
    }
    int64_t cum = 0;
    for (int b = 0; b < MAX_ACTIVE_BINS; b++) {
        cum += hist[b];
        if (cum > max_active) {
            volatile double span = (double)(b < 1 ? 1 : b) * width;   /* no FMA contraction */
            double h = best + span;
            return h < cutoff ? h : cutoff;
        }
    }
    return cutoff;
}

/* ---- aggregation: decoder.py:330-370 (with _winners decoder.py:314-327) ---- */
static int aggregate(ws_t *w, const lbo_graph *g, double cutoff, int32_t frame, int init_state,
                     const lbo_config *cfg, run_t *r, lbo_result *out) {
    r->kept_n = 0;
    for (int64_t k = 0; k < w->ntouched; k++) {
        int32_t v = w->touched[k];
        if (v == init_state) continue;
        if (w->cost[v] <= cutoff) VPUSH(r->kept, v);
    }
    if (init_state >= 0) VPUSH(r->kept, init_state);
    qsort(r->kept, (size_t)r->kept_n, 4, cmp_i32);
    int64_t n = r->kept_n;
    if (n == 0)
        return fail(out, LBO_DECODE_FAILURE, NULL, "no tokens survived the beam at frame %d", frame);
    if (n > cfg->max_tokens_per_frame)
        return fail(out, LBO_CAPACITY, "--max-tokens-per-frame",
                    "frame %d kept %lld tokens, over the %lld limit; raise --max-tokens-per-frame",
                    frame, (long long)n, (long long)cfg->max_tokens_per_frame);
    w->stamp++;
    for (int64_t k = 0; k < n; k++) {
        w->pos[r->kept[k]] = k;
        w->pos_stamp[r->kept[k]] = w->stamp;
    }
    for (int64_t k = 0; k < n; k++) {
        int32_t v = r->kept[k];
        int64_t pa, pi;
        double c;
        if (v == init_state) {
            pa = -1; pi = -1; c = 0.0;
        } else {
            pa = (int64_t)(w->pack[v] & 0xFFFFFFFFull);
            c = w->cost[v];
            if (g->il[pa] > 0) {
                pi = w->pred[v];
            } else {
                int32_t u = (int32_t)w->pred[v];
                if (w->pos_stamp[u] != w->stamp)
                    return fail(out, LBO_INTERNAL, NULL, "epsilon winner's source state kept no token");
                pi = w->pos[u];
            }
        }
        VPUSH(r->ts, v); VPUSH(r->tc, c); VPUSH(r->tpa, pa); VPUSH(r->tpi, pi);
        VPUSH(r->tp, w->pack[v]);
    }
    VPUSH(r->toff, r->ts_n);
    return 0;
}

/* ---- lattice resolution of one block: lattice.py:313-362 / reference.py:220-247 ---- */
static int resolve_block(ws_t *w, const lbo_graph *g, double cutoff, const lbo_config *cfg,
                         run_t *r, lbo_result *out) {
    int64_t b0 = r->la_n;
    for (int64_t k = 0; k < r->em_a_n; k++) {
        if (r->em_c[k] > cutoff) continue;
        int32_t v = g->dst[r->em_a[k]];
        if (w->pos_stamp[v] != w->stamp) continue;
        lat_arc_t la = {r->em_a[k], r->em_i[k], (int32_t)w->pos[v], r->em_ac[k]};
        VPUSH(r->la, la);
    }
    if (r->ep_n) {
        qsort(r->ep, (size_t)r->ep_n, sizeof(eps_stage_t), cmp_eps_stage);
        for (int64_t k = 0; k < r->ep_n; k++) {
            if (k > 0 && r->ep[k].a == r->ep[k - 1].a) continue;   /* cheapest per arc id */
            int32_t v = g->dst[r->ep[k].a];
            if (w->pos_stamp[v] != w->stamp) continue;
            int32_t u = r->ep[k].u;
            if (w->pos_stamp[u] != w->stamp)
                return fail(out, LBO_INTERNAL, NULL,
                            "epsilon lattice arc references a source state that kept no token");
            lat_arc_t la = {r->ep[k].a, (int32_t)w->pos[u], (int32_t)w->pos[v], 0.0};
            VPUSH(r->la, la);
        }
    }
    qsort(r->la + b0, (size_t)(r->la_n - b0), sizeof(lat_arc_t), cmp_lat_arc);
    VPUSH(r->loff, r->la_n);
    r->em_a_n = r->em_i_n = r->em_c_n = r->em_ac_n = 0;
    r->ep_n = 0;
    if (r->la_n > cfg->max_lattice_arcs)
        return fail(out, LBO_CAPACITY, "--max-lattice-arcs",
                    "lattice holds %lld arcs, over its %lld capacity; raise --max-lattice-arcs",
                    (long long)r->la_n, (long long)cfg->max_lattice_arcs);
    return 0;
}

/* ---- final extra-cost prune: lattice.py:365-497 (single sweep from the final terminus) ---- */
static int prune_final(const lbo_graph *g, run_t *r, const lbo_config *cfg, const double *terminus,
                       double *ne, uint8_t *pruned, double *extra, lbo_result *out) {
    int32_t T = (int32_t)r->toff_n - 2;
    const double *fwd = r->tc;
    int64_t *toff = r->toff;
    int64_t maxn = 0;
    for (int32_t f = 0; f <= T; f++)
        if (toff[f + 1] - toff[f] > maxn) maxn = toff[f + 1] - toff[f];
    double *cand = NULL, *before = NULL;
    int64_t cap = 0;
    for (int32_t f = T; f >= 0; f--) {
        int64_t n = toff[f + 1] - toff[f];
        double *nf = ne + toff[f];
        for (int64_t i = 0; i < n; i++) nf[i] = (f == T) ? terminus[i] : INFINITY;
        if (f < T) {   /* emitting arcs of block f+1 (lattice.py:444-453) */
            const double *fn = fwd + toff[f + 1];
            const double *nn = ne + toff[f + 1];
            for (int64_t k = r->loff[f + 1]; k < r->loff[f + 2]; k++) {
                lat_arc_t *la = &r->la[k];
                if (g->il[la->a] <= 0) continue;
                double c = (((fwd[toff[f] + la->from] + g->w[la->a]) + la->ac) - fn[la->to]) + nn[la->to];
                if (c < nf[la->from]) nf[la->from] = c;
            }
        }
        /* in-frame epsilon fixpoint (lattice.py:455-469) */
        int64_t ne_cnt = 0;
        for (int64_t k = r->loff[f]; k < r->loff[f + 1]; k++)
            if (g->il[r->la[k].a] == 0) ne_cnt++;
        if (ne_cnt) {
            if (ne_cnt > cap) {
                cap = ne_cnt;
                cand = realloc(cand, (size_t)cap * 8);
                before = realloc(before, (size_t)cap * 8);
            }
            int settled = 0;
            for (int64_t it = 0; it < n + 1; it++) {
                int64_t j = 0;
                for (int64_t k = r->loff[f]; k < r->loff[f + 1]; k++) {
                    lat_arc_t *la = &r->la[k];
                    if (g->il[la->a] != 0) continue;
                    double base = (fwd[toff[f] + la->from] + g->w[la->a]) - fwd[toff[f] + la->to];
                    cand[j] = base + nf[la->to];
                    before[j] = nf[la->from];
                    j++;
                }
                j = 0;
                for (int64_t k = r->loff[f]; k < r->loff[f + 1]; k++) {
                    lat_arc_t *la = &r->la[k];
                    if (g->il[la->a] != 0) continue;
                    if (cand[j] < nf[la->from]) nf[la->from] = cand[j];
                    j++;
                }
                int moved = 0;
                j = 0;
                for (int64_t k = r->loff[f]; k < r->loff[f + 1]; k++) {
                    lat_arc_t *la = &r->la[k];
                    if (g->il[la->a] != 0) continue;
                    if (before[j] - nf[la->from] > CONVERGE_TOL) moved = 1;
                    j++;
                }
                if (!moved) { settled = 1; break; }
            }
            if (!settled) {
                free(cand); free(before);
                return fail(out, LBO_INTERNAL, NULL,
                            "epsilon extra-cost fixpoint did not settle within frame %d", f);
            }
        }
        for (int64_t i = 0; i < n; i++)
            if (!(nf[i] >= 0.0)) nf[i] = (nf[i] != nf[i]) ? nf[i] : 0.0;   /* np.maximum(x, 0) */
    }
    free(cand); free(before);
    /* flag blocks (lattice.py:473-497) */
    for (int32_t b = 0; b <= T; b++) {
        for (int64_t k = r->loff[b]; k < r->loff[b + 1]; k++) {
            lat_arc_t *la = &r->la[k];
            int32_t ff = g->il[la->a] > 0 ? b - 1 : b;
            double x = (((fwd[toff[ff] + la->from] + g->w[la->a]) + la->ac) - fwd[toff[b] + la->to])
                       + ne[toff[b] + la->to];
            if (x < 0.0) x = 0.0;                                    /* np.maximum(x, 0) */
            extra[k] = x;
            pruned[k] = x > cfg->lattice_beam;
        }
    }
    return 0;
}

typedef struct {
    int64_t from, to, il, ol;
    double g, ac;
} fl_row_t;

static int cmp_fl_row(const void *pa, const void *pb) {
    const fl_row_t *x = pa, *y = pb;
#define C(f) if (x->f != y->f) return (x->f > y->f) - (x->f < y->f)
    C(from); C(to); C(il); C(ol); C(g); C(ac);
#undef C
    return 0;
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static int64_t bsearch_i64(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t m = (lo + hi) / 2;
        if (a[m] < key) lo = m + 1; else hi = m;
    }
    return lo;
}

/* ---- finalize: lattice.py:537-598 ---- */
static int finalize(const lbo_graph *g, run_t *r, const uint8_t *pruned, int partial,
                    int64_t start_idx, lbo_result *out) {
    int32_t T = (int32_t)r->toff_n - 2;
    int64_t nlive = 0;
    for (int64_t k = 0; k < r->la_n; k++) nlive += !pruned[k];
    if (nlive == 0) return fail(out, LBO_DECODE_FAILURE, NULL, "no lattice arcs survived pruning");
    int64_t *keys = malloc((size_t)(2 * nlive) * 8);
    fl_row_t *rows = malloc((size_t)nlive * sizeof(fl_row_t));
    int64_t j = 0;
    for (int32_t b = 0; b <= T; b++)
        for (int64_t k = r->loff[b]; k < r->loff[b + 1]; k++) {
            if (pruned[k]) continue;
            lat_arc_t *la = &r->la[k];
            int64_t ff = g->il[la->a] > 0 ? b - 1 : b;
            rows[j].from = (ff << 32) | la->from;
            rows[j].to = ((int64_t)b << 32) | la->to;
            rows[j].il = g->il[la->a];
            rows[j].ol = g->ol[la->a];
            rows[j].g = g->w[la->a];
            rows[j].ac = la->ac;
            keys[2 * j] = rows[j].from;
            keys[2 * j + 1] = rows[j].to;
            j++;
        }
    qsort(keys, (size_t)(2 * nlive), 8, cmp_i64);
    int64_t nn = 0;
    for (int64_t k = 0; k < 2 * nlive; k++)
        if (k == 0 || keys[k] != keys[k - 1]) keys[nn++] = keys[k];
    for (int64_t k = 0; k < nlive; k++) {
        rows[k].from = bsearch_i64(keys, nn, rows[k].from);
        rows[k].to = bsearch_i64(keys, nn, rows[k].to);
    }
    qsort(rows, (size_t)nlive, sizeof(fl_row_t), cmp_fl_row);
    int64_t sp = bsearch_i64(keys, nn, start_idx);
    if (sp >= nn || keys[sp] != start_idx) {
        free(keys); free(rows);
        return fail(out, LBO_DECODE_FAILURE, NULL, "surviving arcs do not connect to the start node");
    }
    out->fl_node_frame = malloc((size_t)nn * 8);
    out->fl_node_idx = malloc((size_t)nn * 8);
    out->fl_final_ids = malloc((size_t)nn * 8);
    out->fl_final_costs = malloc((size_t)nn * 8);
    int64_t nfin = 0;
    for (int64_t k = 0; k < nn; k++) {
        int64_t fr = keys[k] >> 32, idx = keys[k] & 0xFFFFFFFFll;
        out->fl_node_frame[k] = fr;
        out->fl_node_idx[k] = idx;
        if (fr == T) {
            double fc = partial ? 0.0 : g->final_cost[r->ts[r->toff[T] + idx]];
            if (partial || isfinite(fc)) {
                out->fl_final_ids[nfin] = k;
                out->fl_final_costs[nfin] = fc;
                nfin++;
            }
        }
    }
    out->fl_num_nodes = nn;
    out->fl_start = sp;
    out->fl_n_final = nfin;
    out->fl_n_arcs = nlive;
#define AL(name, T_) out->name = malloc((size_t)(nlive ? nlive : 1) * sizeof(T_))
    AL(fl_from, int64_t); AL(fl_to, int64_t); AL(fl_il, int64_t); AL(fl_ol, int64_t);
    AL(fl_g, double); AL(fl_ac, double);
#undef AL
    for (int64_t k = 0; k < nlive; k++) {
        out->fl_from[k] = rows[k].from; out->fl_to[k] = rows[k].to;
        out->fl_il[k] = rows[k].il; out->fl_ol[k] = rows[k].ol;
        out->fl_g[k] = rows[k].g; out->fl_ac[k] = rows[k].ac;
    }
    free(keys); free(rows);
    if (nfin == 0) return fail(out, LBO_DECODE_FAILURE, NULL, "no terminal node survived pruning");
    return 0;
}

#define EXPORT(name, T_, src_, n_)                                     \
    do {                                                               \
        out->name = malloc((size_t)((n_) ? (n_) : 1) * sizeof(T_));    \
        memcpy(out->name, src_, (size_t)(n_) * sizeof(T_));            \
    } while (0)

/* ---- decode_utterance: decoder.py:463-611 ---- */
static int decode_ws(ws_t *w, const lbo_graph *g, const double *costs, int32_t T, int32_t D,
                     const lbo_config *cfg, lbo_result *out) {
    memset(out, 0, sizeof(*out));
    if (!(isfinite(cfg->beam) && cfg->beam > 0))
        return fail(out, LBO_USAGE, NULL, "beam must be a positive finite number");
    if (T < 1 || D < 1) return fail(out, LBO_USAGE, NULL, "cost matrix must be 2-D with T >= 1 and D >= 1");
    run_t r;
    memset(&r, 0, sizeof(r));
    int stage = cfg->want_lattice != 0;
    int rc = 0;
    double *seedc = NULL;
    int64_t seedcap = 0;
    double beam_eff = cfg->beam;   /* adaptive beam; == beam when max_active == 0 */
    VPUSH(r.toff, 0);
    VPUSH(r.loff, 0);

    /* frame 0: decoder.py:510-523 */
    ws_reset_frame(w);
    int32_t s0 = g->start;
    w->pack[s0] = pack_word(0.0, 0);
    w->cost[s0] = 0.0;
    w->pred[s0] = -1;
    w->touched[w->ntouched++] = s0;
    double cutoff = 0.0 + cfg->beam;
    w->fs[0] = s0;
    w->fc[0] = 0.0;
    if ((rc = eps_fixpoint(w, g, cutoff, 1, stage, &r, out))) goto done;
    if ((rc = aggregate(w, g, cutoff, 0, s0, cfg, &r, out))) goto done;
    VPUSH(r.cut, cutoff);
    if (stage && (rc = resolve_block(w, g, cutoff, cfg, &r, out))) goto done;
    int64_t start_idx = 0;
    for (int64_t k = r.toff[0]; k < r.toff[1]; k++)
        if (r.ts[k] == s0) start_idx = k;

    for (int32_t t = 1; t <= T; t++) {
        const double *row = costs + (int64_t)(t - 1) * D;
        for (int32_t d = 0; d < D; d++) w->acrow[d] = row[d] * cfg->acoustic_scale;
        ws_reset_frame(w);
        int64_t p0 = r.toff[t - 1], p1 = r.toff[t];
        double best = INFINITY;
        /* emitting pass (kernels.py:82-122 / emit_pass_numpy kernels.py:312-333) */
        for (int64_t i = 0; i < p1 - p0; i++) {
            int32_t s = r.ts[p0 + i];
            double c = r.tc[p0 + i];
            r.cnt[0]++;
            for (int64_t a = g->off[s]; a < g->off[s + 1]; a++) {
                r.cnt[1]++;
                int32_t l = g->il[a];
                if (l == 0) continue;
                r.cnt[2]++;
                double ac = w->acrow[l - 1];
                double cand = (c + g->w[a]) + ac;
                if (cand < best) best = cand;
                if (stage) {
                    VPUSH(r.em_a, (int32_t)a); VPUSH(r.em_i, (int32_t)i);
                    VPUSH(r.em_c, cand); VPUSH(r.em_ac, ac);
                }
                int imp;
                offer(w, g->dst[a], pack_word(cand, a), cand, i, &imp);
            }
        }
        if (!isfinite(best)) {
            rc = fail(out, LBO_DECODE_FAILURE, NULL, "beam search died at frame %d: no emitting candidates", t);
            goto done;
        }
        cutoff = best + beam_eff;
        /* seeds = winners under the cutoff (decoder.py:540; _winners :314-327) */
        int64_t ns = 0;
        if (w->ntouched > seedcap) { seedcap = w->ntouched; seedc = realloc(seedc, (size_t)seedcap * 8); }
        for (int64_t k = 0; k < w->ntouched; k++) {
            int32_t v = w->touched[k];
            if (w->cost[v] <= cutoff) { w->fs[ns] = v; seedc[ns] = w->cost[v]; ns++; }
        }
        if (ns == 0) {
            rc = fail(out, LBO_DECODE_FAILURE, NULL, "no tokens survived the beam at frame %d", t);
            goto done;
        }
        double c2 = max_active_cutoff(seedc, ns, best, cfg->beam, cfg->max_active, cutoff);
        if (c2 < cutoff) {
            /* max-active bound: next frame's beam adapts (Kaldi GetCutoff's adaptive_beam) */
            double be = (c2 - best) + MAX_ACTIVE_BEAM_DELTA;
            beam_eff = be < cfg->beam ? be : cfg->beam;
            cutoff = c2;
            int64_t m = 0;
            for (int64_t k = 0; k < ns; k++)
                if (seedc[k] <= cutoff) w->fs[m++] = w->fs[k];
            ns = m;
        } else {
            beam_eff = cfg->beam;
        }
        qsort(w->fs, (size_t)ns, 4, cmp_i32);
        for (int64_t k = 0; k < ns; k++) w->fc[k] = w->cost[w->fs[k]];
        if ((rc = eps_fixpoint(w, g, cutoff, ns, stage, &r, out))) goto done;
        if ((rc = aggregate(w, g, cutoff, t, -1, cfg, &r, out))) goto done;
        r.cnt[6] += r.toff[t + 1] - r.toff[t];
        VPUSH(r.cut, cutoff);
        if (stage && (rc = resolve_block(w, g, cutoff, cfg, &r, out))) goto done;
    }
    free(seedc);
    seedc = NULL;

    {
        /* final selection: decoder.py:578-586 */
        int64_t p0 = r.toff[T], n = r.toff[T + 1] - p0;
        double *totals = malloc((size_t)n * 8);
        int partial = 1;
        for (int64_t i = 0; i < n; i++) {
            totals[i] = r.tc[p0 + i] + g->final_cost[r.ts[p0 + i]];
            if (isfinite(totals[i])) partial = 0;
        }
        int64_t bi = 0;
        const double *sel = partial ? r.tc + p0 : totals;
        for (int64_t i = 1; i < n; i++)
            if (sel[i] < sel[bi]) bi = i;
        out->partial = partial;
        out->total_cost = sel[bi];

        if (stage) {
            double *term = malloc((size_t)n * 8);
            for (int64_t i = 0; i < n; i++) term[i] = partial ? 0.0 : totals[i] - totals[bi];
            out->node_extra = malloc((size_t)(r.ts_n ? r.ts_n : 1) * 8);
            out->lat_pruned = malloc((size_t)(r.la_n ? r.la_n : 1));
            out->lat_extra = malloc((size_t)(r.la_n ? r.la_n : 1) * 8);
            rc = prune_final(g, &r, cfg, term, out->node_extra, out->lat_pruned, out->lat_extra, out);
            free(term);
            if (!rc) rc = finalize(g, &r, out->lat_pruned, partial, start_idx, out);
            r.cnt[7] = r.la_n;
        }
        free(totals);
        if (rc) goto done;

        /* backtrace: decoder.py:614-641, bounded */
        VEC(int32_t, wd); VEC(int32_t, ai); VEC(int32_t, af);
        wd = NULL; ai = NULL; af = NULL; wd_n = wd_cap = ai_n = ai_cap = af_n = af_cap = 0;
        int32_t f = T;
        int64_t i = bi, steps = 0, limit = r.ts_n + 1;
        for (;;) {
            int64_t a = r.tpa[r.toff[f] + i];
            if (a < 0) {
                if (f != 0) { rc = fail(out, LBO_INTERNAL, NULL, "initial token found at frame %d", f); break; }
                break;
            }
            if (g->ol[a] > 0) VPUSH(wd, g->ol[a]);
            int64_t pi = r.tpi[r.toff[f] + i];
            if (g->il[a] > 0) { VPUSH(ai, g->il[a]); VPUSH(af, f - 1); f -= 1; }
            i = pi;
            if (++steps > limit) {
                rc = fail(out, LBO_INTERNAL, NULL, "backtrace exceeded %lld steps (epsilon cycle)", (long long)limit);
                break;
            }
        }
        if (!rc) {
            out->n_words = wd_n;
            out->words = malloc((size_t)(wd_n ? wd_n : 1) * 4);
            for (int64_t k = 0; k < wd_n; k++) out->words[k] = wd[wd_n - 1 - k];
            out->n_align = ai_n;
            out->align_il = malloc((size_t)(ai_n ? ai_n : 1) * 4);
            out->align_fr = malloc((size_t)(ai_n ? ai_n : 1) * 4);
            for (int64_t k = 0; k < ai_n; k++) {
                out->align_il[k] = ai[ai_n - 1 - k];
                out->align_fr[k] = af[af_n - 1 - k];
            }
        }
        free(wd); free(ai); free(af);
        if (rc) goto done;
    }

    if (cfg->collect_frames || stage) {
        out->n_frames = T + 1;
        EXPORT(tok_off, int64_t, r.toff, r.toff_n);
        EXPORT(tok_state, int32_t, r.ts, r.ts_n);
        EXPORT(tok_cost, double, r.tc, r.tc_n);
        EXPORT(tok_pred_arc, int64_t, r.tpa, r.tpa_n);
        EXPORT(tok_pred_idx, int64_t, r.tpi, r.tpi_n);
        EXPORT(tok_pack, uint64_t, r.tp, r.tp_n);
        EXPORT(cutoffs, double, r.cut, r.cut_n);
    }
    if (stage) {
        EXPORT(lat_off, int64_t, r.loff, r.loff_n);
        out->lat_arc = malloc((size_t)(r.la_n ? r.la_n : 1) * 4);
        out->lat_from = malloc((size_t)(r.la_n ? r.la_n : 1) * 4);
        out->lat_to = malloc((size_t)(r.la_n ? r.la_n : 1) * 4);
        out->lat_ac = malloc((size_t)(r.la_n ? r.la_n : 1) * 8);
        for (int64_t k = 0; k < r.la_n; k++) {
            out->lat_arc[k] = r.la[k].a; out->lat_from[k] = r.la[k].from;
            out->lat_to[k] = r.la[k].to; out->lat_ac[k] = r.la[k].ac;
        }
    }
done:
    free(seedc);
    memcpy(&out->n_tokens, r.cnt, sizeof(r.cnt));
    ws_reset_frame(w);
    run_free(&r);
    return rc;
}

int lbo_decode(const lbo_graph *g, const double *costs, int32_t T, int32_t D, const lbo_config *cfg,
               lbo_result *out) {
    ws_t *w = ws_alloc(g->S, D);
    int rc = decode_ws(w, g, costs, T, D, cfg, out);
    ws_free(w);
    return rc;
}

void lbo_result_free(lbo_result *r) {
    if (!r) return;
    void *ptrs[] = {r->words, r->align_il, r->align_fr, r->tok_off, r->tok_state, r->tok_cost,
                    r->tok_pred_arc, r->tok_pred_idx, r->tok_pack, r->cutoffs, r->lat_off,
                    r->lat_arc, r->lat_from, r->lat_to, r->lat_ac, r->lat_extra, r->lat_pruned,
                    r->node_extra, r->fl_final_ids, r->fl_final_costs, r->fl_from, r->fl_to,
                    r->fl_il, r->fl_ol, r->fl_g, r->fl_ac, r->fl_node_frame, r->fl_node_idx};
    for (size_t k = 0; k < sizeof(ptrs) / sizeof(ptrs[0]); k++) free(ptrs[k]);
    memset(r, 0, sizeof(*r));
}

/* ---- decode_batch over host threads: decoder.py:644-672 ---- */
typedef struct {
    const lbo_graph *g;
    int32_t n, D;
    const double *const *costs;
    const int32_t *T;
    const lbo_config *cfg;
    double *total_costs;
    int32_t *statuses;
    int64_t *counters;
    int64_t next;
} batch_t;

static void *batch_worker(void *arg) {
    batch_t *b = arg;
    ws_t *w = ws_alloc(b->g->S, b->D);
    for (;;) {
        int64_t u = __atomic_fetch_add(&b->next, 1, __ATOMIC_RELAXED);
        if (u >= b->n) break;
        lbo_result res;
        int rc = decode_ws(w, b->g, b->costs[u], b->T[u], b->D, b->cfg, &res);
        b->statuses[u] = rc;
        b->total_costs[u] = res.total_cost;
        if (b->counters) memcpy(b->counters + 8 * u, &res.n_tokens, 8 * sizeof(int64_t));
        lbo_result_free(&res);
    }
    ws_free(w);
    return NULL;
}

int lbo_decode_batch_mt(const lbo_graph *g, int32_t n, const double *const *costs, const int32_t *T,
                        int32_t D, const lbo_config *cfg, int32_t nthreads, double *total_costs,
                        int32_t *statuses, int64_t *counters) {
    batch_t b = {g, n, D, costs, T, cfg, total_costs, statuses, counters, 0};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n) nthreads = n > 0 ? n : 1;
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; k++) pthread_create(&th[k], NULL, batch_worker, &b);
    for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th);
    return 0;
}

/* ---- single-op surfaces ---- */
int64_t lbo_expand_emitting(const lbo_graph *g, const int32_t *states, const double *costs, int64_t n,
                            const double *acrow, double beam, int32_t *out_states, double *out_costs,
                            double *out_cutoff) {
    /* decoder.py:373-400: emit one frontier, keep winners <= best+beam (no epsilon) */
    ws_t *w = ws_alloc(g->S, 1);
    double best = INFINITY;
    for (int64_t i = 0; i < n; i++) {
        int32_t s = states[i];
        for (int64_t a = g->off[s]; a < g->off[s + 1]; a++) {
            int32_t l = g->il[a];
            if (l == 0) continue;
            double cand = (costs[i] + g->w[a]) + acrow[l - 1];
            if (cand < best) best = cand;
            int imp;
            offer(w, g->dst[a], pack_word(cand, a), cand, i, &imp);
        }
    }
    int64_t m = 0;
    if (!isfinite(best)) {
        *out_cutoff = INFINITY;
    } else {
        double cutoff = best + beam;
        *out_cutoff = cutoff;
        for (int64_t k = 0; k < w->ntouched; k++)
            if (w->cost[w->touched[k]] <= cutoff) out_states[m++] = w->touched[k];
        qsort(out_states, (size_t)m, 4, cmp_i32);
        for (int64_t k = 0; k < m; k++) out_costs[k] = w->cost[out_states[k]];
    }
    ws_free(w);
    return m;
}

int64_t lbo_expand_nonemitting(const lbo_graph *g, const int32_t *states, const double *costs, int64_t n,
                               double cutoff, int32_t *out_states, double *out_costs) {
    /* decoder.py:403-435: seeds behave as won entries pack(cost, 0) */
    ws_t *w = ws_alloc(g->S, 1);
    lbo_result dummy;
    run_t r;
    memset(&r, 0, sizeof(r));
    memset(&dummy, 0, sizeof(dummy));
    for (int64_t i = 0; i < n; i++) {
        int32_t s = states[i];
        w->pack[s] = pack_word(costs[i], 0);
        w->cost[s] = costs[i];
        w->pred[s] = -1;
        w->touched[w->ntouched++] = s;
        w->fs[i] = s;
        w->fc[i] = costs[i];
    }
    int rc = eps_fixpoint(w, g, cutoff, n, 0, &r, &dummy);
    int64_t m = 0;
    if (!rc) {
        for (int64_t k = 0; k < w->ntouched; k++)
            if (w->cost[w->touched[k]] <= cutoff) out_states[m++] = w->touched[k];
        qsort(out_states, (size_t)m, 4, cmp_i32);
        for (int64_t k = 0; k < m; k++) out_costs[k] = w->cost[out_states[k]];
    }
    run_free(&r);
    ws_free(w);
    return rc ? -rc : m;
}
