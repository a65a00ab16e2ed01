/*
 * latbeam_oracle.h — CPU restatement of the reference decoder (TEST INFRASTRUCTURE).
 *
 * This header belongs to the parity oracle, not to the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline / `--impl reference` legs
 * may load the library built from it.  It restates, serially and exactly, the
 * token-passing Viterbi beam search of the reference package `latbeam`
 * (/root/reference/pkg/src/latbeam/decoder.py:463-611, reference.py:69-157),
 * its lattice resolution (lattice.py:313-362, reference.py:220-247), extra-cost
 * pruning (lattice.py:365-497) and finalisation (lattice.py:537-598).  The one
 * addition is the max-active histogram cutoff the reference lacks
 * (SPEC.md:245); it is specified in DESIGN.md §3 and is a no-op at max_active=0.
 */
#ifndef LATBEAM_ORACLE_H
#define LATBEAM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { LBO_OK = 0, LBO_DECODE_FAILURE = 1, LBO_USAGE = 2, LBO_CAPACITY = 3, LBO_INTERNAL = 4 };

typedef struct {
    int64_t S, A;
    int32_t start;
    const int64_t *off;     /* [S+1] CSR offsets (wfst.py:33-90)            */
    const int32_t *src, *dst, *il, *ol;
    const double *w;        /* arc weights                                  */
    const double *final_cost; /* [S], +inf = non-final (wfst.py:56-60)      */
} lbo_graph;

typedef struct {
    double beam, lattice_beam, acoustic_scale;
    int64_t max_active;          /* 0 = off (reference behaviour)             */
    int64_t max_tokens_per_frame;
    int64_t max_lattice_arcs;    /* bound on live lattice arcs                 */
    int32_t want_lattice;
    int32_t collect_frames;      /* keep per-frame token lists / packs         */
} lbo_config;

typedef struct {
    int32_t status;
    char msg[256];
    char bound[64];
    double total_cost;
    int32_t partial;
    int64_t n_words;  int32_t *words;
    int64_t n_align;  int32_t *align_il; int32_t *align_fr;
    /* per-frame token lists, state-sorted (decoder.py:330-370) */
    int32_t n_frames;            /* T+1 */
    int64_t *tok_off;            /* [n_frames+1] */
    int32_t *tok_state; double *tok_cost; int64_t *tok_pred_arc; int64_t *tok_pred_idx;
    uint64_t *tok_pack;
    double *cutoffs;             /* [n_frames] */
    /* work lattice: live arcs by block, sorted by arc id inside a block */
    int64_t *lat_off;            /* [n_frames+1] */
    int32_t *lat_arc, *lat_from, *lat_to;
    double *lat_ac, *lat_extra;
    uint8_t *lat_pruned;
    double *node_extra;          /* parallel to tok_* */
    /* final lattice (lattice.py:500-598) */
    int64_t fl_num_nodes, fl_start, fl_n_final, fl_n_arcs;
    int64_t *fl_final_ids; double *fl_final_costs;
    int64_t *fl_from, *fl_to, *fl_il, *fl_ol; double *fl_g, *fl_ac;
    int64_t *fl_node_frame, *fl_node_idx;
    /* work counters */
    int64_t n_tokens, n_scan, n_cand, eps_front, eps_scan, eps_cand, n_next, n_lat;
} lbo_result;

int  lbo_decode(const lbo_graph *g, const double *costs, int32_t T, int32_t D,
                const lbo_config *cfg, lbo_result *out);
void lbo_result_free(lbo_result *r);

/* Many utterances over nthreads host threads, one utterance per thread at a time
 * (the reference's decode_batch, decoder.py:644-672).  1-best results only. */
int  lbo_decode_batch_mt(const lbo_graph *g, int32_t n, const double *const *costs,
                         const int32_t *T, int32_t D, const lbo_config *cfg, int32_t nthreads,
                         double *total_costs, int32_t *statuses, int64_t *counters /* [n*8] */);

/* Single-op surfaces (decoder.py:373-435). Outputs are state-sorted; caller
 * provides buffers of size >= S.  Return the number of outputs, or -status. */
int64_t lbo_expand_emitting(const lbo_graph *g, const int32_t *states, const double *costs, int64_t n,
                            const double *acrow, double beam, int32_t *out_states,
                            double *out_costs, double *out_cutoff);
int64_t lbo_expand_nonemitting(const lbo_graph *g, const int32_t *states, const double *costs,
                               int64_t n, double cutoff, int32_t *out_states, double *out_costs);

#ifdef __cplusplus
}
#endif
#endif
