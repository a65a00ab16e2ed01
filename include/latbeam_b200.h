/*
 * latbeam_b200.h — C-ABI of the B200-native WFST Viterbi decoder (liblatbeam_b200.so).
 *
 * This is the drop-in boundary for the reference package's decode path
 * (`latbeam`, /root/reference/pkg/src/latbeam).  Every entry point replaces
 * one reference interface, cited beside it; plain pointers and sizes only, no
 * torch types.  All calls return an `lb_status` (0 = OK) mirroring the
 * reference's exception classes (errors.py:8-41) and CLI exit codes
 * (cli.py:470-489); `lb_last_error()` gives the thread-local message.
 *
 * Threading: an lb_graph is immutable after creation and may be shared by
 * host threads; decodes on one graph serialise on the graph's workspace.
 * Ownership: the library owns device replicas and result buffers; callers own
 * their input arrays (copied during the call).
 */
#ifndef LATBEAM_B200_H
#define LATBEAM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LB_OK = 0,
    LB_DECODE_FAILURE = 1, /* errors.py DecodeFailure          */
    LB_USAGE = 2,          /* errors.py UsageError             */
    LB_CAPACITY = 3,       /* errors.py CapacityError(bound)   */
    LB_INTERNAL = 4,       /* errors.py InternalInvariantError */
    LB_CUDA = 5            /* device/runtime failure (no reference counterpart) */
} lb_status;

typedef struct lb_graph lb_graph;
typedef struct lb_result lb_result;

/* DecodeConfig (decoder.py:52-89) + the device knobs.  num_workers,
 * group_size, num_shards, prune_interval and scheduler of the reference only
 * shape CPU threading and have no device meaning. */
typedef struct {
    double beam;                  /* > 0, finite                         */
    double lattice_beam;          /* >= 0                                */
    double acoustic_scale;        /* > 0                                 */
    int64_t max_active;           /* 0 = off (reference), else histogram cutoff */
    int64_t max_tokens_per_frame; /* CapacityError "--max-tokens-per-frame" */
    int64_t max_lattice_arcs;     /* live lattice arcs per utterance; "--max-lattice-arcs" */
    int64_t token_arena;          /* tokens kept per utterance (all frames); 0 = auto; "--token-arena" */
    int32_t want_lattice;         /* decode_utterance(want_lattice=...)  */
    int32_t collect_frame_packs;  /* keep per-frame token lists for readback */
    int32_t lanes;                /* concurrent utterances per launch (CTAs); 0 = auto */
    int32_t threads_per_lane;     /* CTA size: 512, 640 or 768; 0 = auto (640) */
    int32_t ctas_per_lane;        /* thread-block cluster size of a lane (1..16; >8 is a non-portable size); 0 = auto */
    int32_t keep_work_lattice;    /* also keep every live arc + extra (DecodeResult.work_lattice) */
} lb_config;

int32_t lb_version(void);
const char *lb_last_error(void);
int32_t lb_device_count(void);

/* Wfst (wfst.py:33-90): CSR columns, arc id = position.  Uploaded to HBM on
 * `device` as 16 B arc records + side columns.  Limits: fewer
 * than 2^30 states, 2^32 - 1 arcs and input labels below 2^30 (two flag bits
 * ride in the state and label words); LB_USAGE otherwise. */
int lb_graph_create(int32_t device, int64_t num_states, int64_t num_arcs, int32_t start_state,
                    const int64_t *arc_offsets, const int32_t *arc_src, const int32_t *arc_dst,
                    const int32_t *arc_ilabel, const int32_t *arc_olabel, const double *arc_weight,
                    const double *final_cost, lb_graph **out);
int lb_graph_destroy(lb_graph *g);
int64_t lb_graph_device_bytes(const lb_graph *g);

/* decode_batch (decoder.py:644-672) / decode_utterance (decoder.py:463-611):
 * costs[u] is a row-major T[u] x D f64 host matrix (CostMatrix.costs).
 * Blocking; host->device and device->host copies happen inside. */
int lb_decode_batch(const lb_graph *g, int32_t n_utts, const double *const *costs,
                    const int32_t *num_frames, int32_t num_labels, const lb_config *cfg,
                    lb_result **out);

/* Same, with the cost matrices already resident in device memory on the graph's
 * device (e.g. an acoustic model's output tensor).  `stream` is a cudaStream_t
 * (NULL = the library's stream); the call enqueues and waits on it. */
int lb_decode_batch_device(const lb_graph *g, int32_t n_utts, const double *const *dev_costs,
                           const int32_t *num_frames, int32_t num_labels, const lb_config *cfg,
                           void *stream, lb_result **out);

/* Same, with f32 device-resident cost matrices (what an acoustic model emits;
 * PAPER.md:376, 483).  Every value is widened exactly to f64 when its row is
 * loaded (refilling 1-best lanes) or into an HBM scratch first (other modes),
 * so the result equals decoding the widened f64 matrix. */
int lb_decode_batch_device_f32(const lb_graph *g, int32_t n_utts, const float *const *dev_costs,
                               const int32_t *num_frames, int32_t num_labels, const lb_config *cfg,
                               void *stream, lb_result **out);

/* decode_batch across devices: graphs[k] is a replica of the
 * same graph on some device (lb_graph_create per device; the same device may
 * hold several replicas).  Utterances are split longest-first (lb_shard_lpt),
 * each replica decodes its shard on its own host thread, and the result holds
 * every utterance in input order.  No collective: utterances share nothing
 * (decoder.py:644-672, the reference's pool over utterances). */
int lb_decode_batch_multi(const lb_graph *const *graphs, int32_t n_graphs, int32_t n_utts,
                          const double *const *costs, const int32_t *num_frames, int32_t num_labels,
                          const lb_config *cfg, lb_result **out);
/* The LPT assignment lb_decode_batch_multi uses: utterances by descending length
 * (ties: input order), each to the shard with the fewest frames so far (ties:
 * lowest shard).  shard_of[i] in [0, n_shards).  Host-only. */
int lb_shard_lpt(int32_t n_utts, const int32_t *num_frames, int32_t n_shards, int32_t *shard_of);

/* Per-utterance readback.  DecodeResult (decoder.py:92-103). */
int lb_result_count(const lb_result *r, int32_t *n_utts);
int lb_result_status(const lb_result *r, int32_t utt, int32_t *status, char *message,
                     int32_t message_len, char *bound, int32_t bound_len);
int lb_result_best(const lb_result *r, int32_t utt, double *total_cost, int32_t *partial,
                   int64_t *path_len, int64_t *num_tokens, int64_t *num_lattice_arcs);
/* All utterances at once: status[n], total_cost[n], partial[n], path_off[n+1]
 * (prefix offsets of the best paths) and counters[n*8]; any pointer may be NULL.
 * lb_result_paths writes every utterance's best path back to back (path_off). */
int lb_result_bulk(const lb_result *r, int32_t *status, double *total_cost, int32_t *partial,
                   int64_t *path_off, int64_t *counters);
int lb_result_paths(const lb_result *r, int32_t *arcs);
/* Best path as graph arc ids in forward order; words = olabels > 0, alignment
 * = (ilabel, frame) of the emitting hops (decoder.py:614-641). */
int lb_result_path(const lb_result *r, int32_t utt, int32_t *arcs);
/* Token lists per frame (FrameTokens, lattice.py:71-98), in device order
 * (not state-sorted; the host canonicalises).  frame_off has T+2 entries. */
int lb_result_tokens(const lb_result *r, int32_t utt, int64_t *frame_off, int32_t *states,
                     double *costs, int32_t *pred_arc, int32_t *pred_idx, uint64_t *packs);
/* Live lattice arcs per block with their pruning extra cost (lattice.py:473-497);
 * from/to index the device-order token lists of the arc's frames.  Needs
 * keep_work_lattice. */
int lb_result_lattice(const lb_result *r, int32_t utt, int64_t *block_off, int32_t *arc,
                      int32_t *from_idx, int32_t *to_idx, double *extra);
/* Final lattice of a want_lattice decode, finalised on the device
 * (finalize_lattice, lattice.py:537-598): sizes, then the arrays.  node_keys
 * are (frame << 32) | index into the frame's state-sorted token list, ascending
 * (node id = position); arcs are in canonical order (from, to, ilabel,
 * olabel, graph_cost, acoustic_cost). */
int lb_result_final_lattice(const lb_result *r, int32_t utt, int64_t *num_nodes, int64_t *start,
                            int64_t *n_final, int64_t *n_arcs);
int lb_result_final_arrays(const lb_result *r, int32_t utt, uint64_t *node_keys, int64_t *final_ids,
                           double *final_costs, int32_t *from, int32_t *to, int32_t *ilabel,
                           int32_t *olabel, double *graph_cost, double *acoustic_cost);
/* The same arrays in the FinalLattice dtypes (int64 ids/labels, node keys split
 * into node_frame / node_idx), widened on all host threads from the pinned D2H
 * arena.  Any pointer may be NULL to skip that array. */
int lb_result_final_arrays64(const lb_result *r, int32_t utt, int64_t *node_frame, int64_t *node_idx,
                             int64_t *final_ids, double *final_costs, int64_t *from, int64_t *to, int64_t *ilabel,
                             int64_t *olabel, double *graph_cost, double *acoustic_cost);
/* counters[8]: tokens expanded, arcs scanned, emitting candidates, epsilon
 * frontier entries, epsilon arcs scanned, epsilon candidates, tokens kept,
 * lattice arcs. */
int lb_result_counters(const lb_result *r, int32_t utt, int64_t *counters);
/* Device-event timings of the call (ms): decode kernel, prune kernel, H2D, D2H, and the
 * number of kernel launches the call made. */
int lb_result_timing(const lb_result *r, float *decode_ms, float *prune_ms, float *h2d_ms,
                     float *d2h_ms, int32_t *launches);
/* Per-phase device time of the decode kernel summed over lanes (ms): emit, winners,
 * max-active, epsilon, aggregate, lattice, frame turnover, frame0+final.  Zero unless
 * the environment variable LB_PHASE_PROFILE=1 was set for the call (profiling aid). */
int lb_result_phases(const lb_result *r, double *ms8);
/* Same profiling run: per phase, the busy time of every warp up to its arrival at
 * the phase's closing barrier, summed over warps (ms), and the number of
 * warp-phase samples; busy/samples vs the lane phase time separates slow work
 * from waiting on the slowest warp. */
int lb_result_warp_phases(const lb_result *r, double *busy_ms8, double *samples8);
void lb_result_free(lb_result *r);

/* Lattice oracle word error (scoring.py:66-114), many lattices at once, one
 * CTA each.  A lattice view is the FinalLattice columns.  When node_frame is
 * non-decreasing (nodes numbered by (frame, index)) and every arc stays in its
 * frame or advances one frame -- what the decoder produces -- the DP walks the
 * frames in order; otherwise (or node_frame NULL) it relaxes all arcs to a
 * fixpoint, like the reference.  Arcs may come in any order.
 * errors[i] = fewest word errors, -1 = no complete path, -2 = no convergence.
 * Returns LB_USAGE for an empty reference or out-of-range ids. */
typedef struct {
    int64_t num_nodes, start, n_final, n_arcs, n_ref;
    const int64_t *final_ids, *from, *to, *olabel, *node_frame;
    const int32_t *ref;
} lb_lattice_view;
int lb_oracle_wer_batch(int32_t device, int32_t n, const lb_lattice_view *lats, int64_t *errors);

/* write_lattice_text (lattice.py:605-614) in native code, byte-identical to the
 * reference's text (floats as Python repr): returns the text length; the text
 * is written to buf only if cap >= that length.  Host-only, no device needed. */
int64_t lb_lattice_text(int64_t num_nodes, int64_t start, int64_t n_final, const int64_t *final_ids,
                        const double *final_costs, int64_t n_arcs, const int64_t *from, const int64_t *to,
                        const int64_t *ilabel, const int64_t *olabel, const double *graph_cost,
                        const double *acoustic_cost, char *buf, int64_t cap);

/* prune_lattice (lattice.py:365-431) of a work lattice handed in by the caller,
 * on the device.  Frames 0..t: frame_off[t+2] offsets into fwd (each frame's
 * token forward costs); blocks 0..t: block_off[t+2] offsets into the arc
 * columns.  An arc of block b goes from token from_idx of frame b-1 (emitting
 * != 0) or b (epsilon) to token to_idx of frame b.  status: 0 LIVE, 1 PRUNED
 * (pruned arcs stay pruned and do not participate).  terminus = frame t's
 * extra-cost start (zeros, or totals - min(totals) with final costs).  On
 * return every LIVE arc carries its extra (extra[]) and is PRUNED when
 * extra > lattice_beam; node_extra (frame_off[t+1] entries) holds the node
 * extras.  LB_INTERNAL if an in-frame epsilon fixpoint does not settle. */
int lb_prune_lattice(int32_t device, int32_t t, const int64_t *frame_off, const double *fwd,
                     const int64_t *block_off, const int32_t *from_idx, const int32_t *to_idx,
                     const uint8_t *emitting, const double *graph_cost, const double *acoustic_cost,
                     const double *terminus, double lattice_beam, uint8_t *status, double *extra,
                     double *node_extra);

/* finalize_lattice (lattice.py:537-598) of a work lattice handed in by the
 * caller, on the device: its n LIVE arcs with node keys (frame << 32) | token
 * index (from_key / to_key), labels and costs; the start token's index in frame
 * 0; the last frame and, unless partial, its tokens' final costs (+inf = not
 * final).  The FinalLattice comes back as a one-utterance result (status
 * DecodeFailure when nothing survives or the start is cut off), read with
 * lb_result_final_lattice / lb_result_final_arrays64. */
int lb_finalize_lattice(int32_t device, int64_t n, const uint64_t *from_key, const uint64_t *to_key,
                        const int32_t *ilabel, const int32_t *olabel, const double *graph_cost,
                        const double *acoustic_cost, int64_t start_idx, int32_t last_frame, int32_t partial,
                        int64_t n_final_costs, const double *final_costs, lb_result **out);

/* Single-op surfaces (decoder.py:373-435): one frontier on device.
 * out_* need room for num_states entries; *n_out receives the count. */
int lb_expand_emitting(const lb_graph *g, const int32_t *states, const double *costs, int64_t n,
                       const double *acrow, int32_t num_labels, double beam, int32_t *out_states,
                       double *out_costs, int64_t *n_out, double *cutoff);
int lb_expand_nonemitting(const lb_graph *g, const int32_t *states, const double *costs, int64_t n,
                          double cutoff, int32_t *out_states, double *out_costs, int64_t *n_out);

#ifdef __cplusplus
}
#endif
#endif
