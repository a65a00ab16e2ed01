// latbeam_b200.cu — host side of liblatbeam_b200.so: the C-ABI declared in
// include/latbeam_b200.h, graph upload, workspace management, wave scheduling
// of decode lanes, and result readback.  Device code lives in lb_kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <atomic>
#include <thread>
#include <sys/mman.h>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX 3: ranges are free unless a profiler injects itself

#include "../../include/latbeam_b200.h"
#include "lb_kernels.cuh"
#include "lb_lattice.cuh"
#include "lb_batched.cuh"
#include "lb_graph_build.cuh"
#include "lb_scoring.cuh"

using namespace lbk;

// threads of the default lane CTA and its arcs per lane per emit batch
#ifndef LB_LANE_NT
#define LB_LANE_NT 640
#endif
#ifndef LB_UNR640
#define LB_UNR640 2
#endif

namespace {

thread_local std::string g_err;

// NVTX range for the host-side stages of a call (nsys / ncu --nvtx show them):
// staging, the decode launch(es), pruning, finalisation, readback.  The decode
// phases inside the persistent kernel are timed on the device instead
// (LB_PHASE_PROFILE=1, lb_result_phases).
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
};

int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return set_err(LB_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
    } while (0)

template <typename T>
cudaError_t dalloc(T **p, size_t n) {
    return cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T));
}

// Pinned host arena for final lattice arrays: D2H at full link speed into
// page-locked memory that is reused across calls (a result keeps the arena it
// points into alive; the graph reuses it only once no result holds it).
struct HostArena {
    char *p = nullptr;
    size_t cap = 0, used = 0;
    HostArena() = default;
    HostArena(const HostArena &) = delete;
    ~HostArena() {
        if (p) cudaFreeHost(p);
    }
};
template <class T>
struct Span {
    T *p = nullptr;
    size_t n = 0;
    T *data() const { return p; }
    size_t size() const { return n; }
    T *begin() const { return p; }
    T *end() const { return p + n; }
    T &operator[](size_t i) const { return p[i]; }
};

struct UttHost {
    int status = 0;
    std::string msg, bound;
    double total_cost = NAN;
    int partial = 0;
    std::vector<int32_t> path;
    int64_t counters[8] = {0};
    int64_t n_tokens = 0, n_lat = 0;
    std::vector<int64_t> frame_off, block_off;
    std::vector<int32_t> states, pred_arc, pred_idx, larc, lfrom, lto;
    std::vector<double> costs, lextra;
    std::vector<uint64_t> packs;
    // final lattice (device-finalised, lattice.py:500-598)
    bool has_final = false;
    int64_t fl_start = -1;
    std::shared_ptr<HostArena> fl_arena;  // owns the spans below
    Span<uint64_t> fl_nodes;               // (frame << 32) | state-sorted index, ascending
    std::vector<int64_t> fl_final_ids;
    std::vector<double> fl_final_costs;
    Span<int32_t> fl_from, fl_to, fl_il, fl_ol;
    Span<double> fl_g, fl_ac;
};

// Growable device scratch of the lattice finaliser.
struct FlScratch {
    std::vector<void *> bufs;
    size_t tok_cap = 0, arc_cap = 0, temp_cap = 0;
    unsigned long long *keys0 = nullptr, *keys1 = nullptr, *fk = nullptr, *tk = nullptr, *nodes0 = nullptr,
                       *nodes1 = nullptr, *k64a = nullptr, *k64b = nullptr, *count = nullptr;
    int *idx0 = nullptr, *idx1 = nullptr, *rank = nullptr, *perm0 = nullptr, *perm1 = nullptr;
    unsigned *il = nullptr, *ol = nullptr, *fid = nullptr, *tid = nullptr, *k32a = nullptr, *k32b = nullptr;
    double *gc = nullptr, *ac = nullptr, *o_g = nullptr, *o_ac = nullptr, *fcs = nullptr;
    long long *surv = nullptr, *start_rank = nullptr, *fids = nullptr;
    int *o_from = nullptr, *o_to = nullptr, *o_il = nullptr, *o_ol = nullptr, *n_unique = nullptr;
    void *temp = nullptr;
    void release() {
        for (void *p : bufs) cudaFree(p);
        bufs.clear();
        tok_cap = arc_cap = temp_cap = 0;
    }
    ~FlScratch() { release(); }
};

// Per-graph reusable device workspace: lane scratch (O(S) per lane, per-CTA
// lists, candidate buffers) and utterance slots (token / lattice arenas).
struct Workspace {
    int lanes = 0, C = 0;
    int64_t S = 0, tok_cap = 0, lat_cap = 0, ccap = 0;
    int path_cap = 0, tmax = 0;
    bool packs = false, lat = false;
    // lane scratch
    bool batched = false;      // batched-mode layout (StateRec) vs persistent-lane layout
    StateRec *rec = nullptr;
    unsigned long long *pk = nullptr;
    int *tokidx = nullptr, *tpred = nullptr;
    ERec *erec = nullptr;
    double *msnap = nullptr, *tcost = nullptr, *f0cost = nullptr;
    unsigned *tarc = nullptr, *etouched = nullptr;
    EpsWin *rpk = nullptr;
    unsigned *tag = nullptr, *touched = nullptr, *fr = nullptr, *fix = nullptr, *round_ctr = nullptr;
    int4 *cand = nullptr;
    int *candi = nullptr;
    // slots
    unsigned *tok_state = nullptr;
    double *tok_cost = nullptr, *node_extra = nullptr, *lat_extra = nullptr, *tmp = nullptr;
    int *tok_arc = nullptr, *tok_pred = nullptr, *lat_arc = nullptr, *lat_from = nullptr, *lat_to = nullptr;
    unsigned long long *tok_pack = nullptr, *ne_enc = nullptr;
    long long *tok_base = nullptr, *lat_base = nullptr, *out_c = nullptr;
    LaneWs *d_lanes = nullptr;
    LaneWs *d_lanes_mix = nullptr;   // the same lanes with per-lane cluster widths (mixed-width launches)
    std::vector<LaneWs> h_lanes;
    UttDesc *d_desc = nullptr;
    LaneCtl *d_ctl = nullptr;   // batched mode: per-lane control blocks
    std::vector<void *> owned;
    // per-job (utterance) outputs of a call and the job queue (ensure_jobs)
    int jobs_cap = 0, jobs_pstride = 0;
    int *j_path = nullptr, *j_out_i = nullptr, *queue = nullptr;
    double *j_out_d = nullptr;
    long long *j_out_c = nullptr;
    UttJob *d_jobs = nullptr;
    std::vector<void *> jowned;

    void release_jobs() {
        for (void *p : jowned) cudaFree(p);
        jowned.clear();
        jobs_cap = jobs_pstride = 0;
    }
    void release() {
        for (void *p : owned) cudaFree(p);
        owned.clear();
        lanes = 0;
        release_jobs();
    }
};

// Device bytes of one lane's scratch + slot (the lane-count budget).
size_t lane_bytes(int64_t S, int C, int64_t ccap, int64_t tok_cap, int64_t lat_cap, int path_cap, int tmax,
                  bool packs, bool lat, bool batched) {
    // per state: rpk 32 + tag 4 + fr/fix (12 per CTA), then the mode's own layout
    const size_t per_state = batched ? 32 + 32 + 4 + (size_t)C * 16
                                     : 8 + 4 + 16 + 8 + 32 + 4 + (size_t)C * 16;   // pk tokidx erec msnap rpk tag
    const size_t per_cand = batched ? 20 + 4 : 20 + 4 + 8 + 4 + 4 + 8 + 4;       // + winner payload, f0cost
    return (size_t)S * per_state + (size_t)C * ccap * per_cand +
           (size_t)tok_cap * (20 + (packs ? 8 : 0) + (lat ? 16 : 0)) + (size_t)lat_cap * 28 + (size_t)path_cap * 4 +
           (size_t)(tmax + 2) * 16 + 256;
}

}  // namespace

struct lb_graph {
    int device = 0;
    int64_t S = 0, A = 0, E = 0;
    int32_t start = 0, max_ilabel = 0;
    int64_t A_emit = 0;     // emitting arcs
    int64_t max_edeg = 0;   // max emitting out-degree of a state
    int sms = 148;
    int4 *arcs = nullptr;
    unsigned *src = nullptr, *ol = nullptr, *off = nullptr, *eoff = nullptr;
    uint2 *rng = nullptr, *erng = nullptr;
    int4 *eps = nullptr;
    double *fin = nullptr;
    int64_t bytes = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;              // second launch stream (mixed-width lanes)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex mu;
    Workspace ws;    // decode lanes
    Workspace ws1;   // the single-op surfaces (expand_*): one small lane, never evicts ws
    // batched mode: captured CUDA graph of one wave's launch sequence, reused
    // while (workspace, lanes, frames, blocks per lane, Params) stay the same
    cudaGraphExec_t bexec = nullptr;
    std::string bkey;
    int blaunches = 0;
    FlScratch fl;   // lattice finaliser scratch, grown on demand and reused
    double *d_costs = nullptr;
    size_t d_costs_cap = 0;
    double *h_stage = nullptr;
    size_t h_stage_cap = 0;
    std::shared_ptr<HostArena> fl_arena;   // final-lattice D2H arena (see HostArena)
    size_t fl_taken = 0;                   // arena bytes the current / last lattice decode took
    std::map<long long, int> cluster_fit;  // max co-resident lane clusters by (C, threads, smem)
    size_t fl_expect = 0;                  // growth hint: bytes the rest of this decode will likely take
    int *h_ready = nullptr;   // progressive staging counter (mapped pinned)
    int *d_ready = nullptr;
    double *ring = nullptr;   // streamed staging ring of refilling decodes (mapped pinned)
    size_t ring_cap = 0;
    int *ring_ctl = nullptr;  // [0] ready count, [32..] per-slot done marks (mapped pinned)
    int ring_ctl_cap = 0;
    double *dring = nullptr;  // device copy of the ring (DMA staging, decode_ring)
    size_t dring_cap = 0;
    int *dring_ready = nullptr;   // device ready count, written by the copy stream
    int *ring_seq = nullptr;      // pinned sequence values 1..n the copy stream writes into dring_ready
    int ring_seq_cap = 0;
    cudaStream_t copy_stream = nullptr;
    GraphDev dev() const {
        GraphDev g;
        g.arcs = arcs;
        g.src = src;
        g.ol = ol;
        g.off = off;
        g.rng = rng;
        g.erng = erng;
        g.eoff = eoff;
        g.eps = eps;
        g.fin = fin;
        g.S = (int)S;
        g.start = start;
        g.has_eps = E > 0;
        g._pad = 0;
        return g;
    }
};

struct lb_result {
    std::vector<UttHost> utts;
    float t_decode = 0, t_prune = 0, t_h2d = 0, t_d2h = 0;
    int launches = 0;
    double phase_ms[8] = {0};   // lane-summed phase times (LB_PHASE_PROFILE=1 only)
    double warp_ms[8] = {0};    // warp busy time per phase, summed over warps
    double warp_n[8] = {0};     // warp-phase samples
};

namespace {

int ensure_workspace(lb_graph *g, Workspace &w, int lanes, int C, int64_t ccap, int64_t tok_cap, int64_t lat_cap,
                     int path_cap, int tmax, bool packs, bool lat, bool batched) {
    if (w.lanes >= lanes && w.C == C && w.S == g->S && w.ccap >= ccap && w.tok_cap >= tok_cap &&
        w.lat_cap >= lat_cap && w.path_cap >= path_cap && w.tmax >= tmax && (w.packs || !packs) && (w.lat || !lat) &&
        w.batched == batched)
        return LB_OK;
    // Reallocate to exactly this request (never the max of old and new: the
    // lane budget in decode_impl was computed for this request alone).
    w.release();
    ccap = (std::max<int64_t>(ccap, 1) + 31) & ~(int64_t)31;   // 128-byte lines per 32-entry batch (discard)
    const size_t S = (size_t)g->S, nl = (size_t)lanes, nc = (size_t)C;
    auto A = [&](auto **p, size_t n) -> cudaError_t {
        cudaError_t e = dalloc(p, n);
        if (e == cudaSuccess) w.owned.push_back((void *)*p);
        return e;
    };
    const size_t cc = (size_t)ccap;
    if (batched) {
        CK(A(&w.rec, S * nl));
        CK(A(&w.touched, nc * S * nl));
    } else {
        CK(A(&w.pk, S * nl));
        CK(A(&w.tokidx, S * nl));
        CK(A(&w.erec, S * nl));
        CK(A(&w.msnap, S * nl));
        CK(A(&w.touched, nc * cc * nl));
        CK(A(&w.tcost, nc * cc * nl));
        CK(A(&w.tpred, nc * cc * nl));
        CK(A(&w.tarc, nc * cc * nl));
        CK(A(&w.f0cost, nc * cc * nl));
        CK(A(&w.etouched, nc * S * nl));
    }
    CK(A(&w.rpk, 2 * S * nl));
    CK(A(&w.tag, S * nl));
    CK(A(&w.fr, 2 * nc * S * nl));
    CK(A(&w.fix, nc * S * nl));
    CK(A(&w.cand, nc * (size_t)ccap * nl));
    CK(A(&w.candi, nc * (size_t)ccap * nl));
    CK(A(&w.round_ctr, nl));
    const size_t tc = (size_t)tok_cap, lc = (size_t)std::max<int64_t>(lat_cap, 1);
    CK(A(&w.tok_state, tc * nl));
    CK(A(&w.tok_cost, tc * nl));
    CK(A(&w.tok_arc, tc * nl));
    CK(A(&w.tok_pred, tc * nl));
    if (packs) CK(A(&w.tok_pack, tc * nl));
    if (lat) {
        CK(A(&w.node_extra, tc * nl));
        CK(A(&w.ne_enc, tc * nl));
        CK(A(&w.lat_arc, lc * nl));
        CK(A(&w.lat_from, lc * nl));
        CK(A(&w.lat_to, lc * nl));
        CK(A(&w.lat_extra, lc * nl));
        CK(A(&w.tmp, lc * nl));
    }
    CK(A(&w.tok_base, (size_t)(tmax + 2) * nl));
    CK(A(&w.lat_base, (size_t)(tmax + 2) * nl));
    CK(A(&w.d_lanes, nl));
    CK(A(&w.d_lanes_mix, nl));
    CK(A(&w.d_desc, nl));
    CK(A(&w.d_ctl, nl));
    if (batched) {
        init_rec<<<g->sms * 4, 256, 0, g->stream>>>(w.rec, (long long)(S * nl));
    } else {
        CK(cudaMemsetAsync(w.pk, 0xFF, S * nl * 8, g->stream));       // SENT
        CK(cudaMemsetAsync(w.tokidx, 0xFF, S * nl * 4, g->stream));   // -1
        fill_f64<<<g->sms * 4, 256, 0, g->stream>>>(w.msnap, (long long)(S * nl), std::numeric_limits<double>::infinity());
    }
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(w.rpk, 0xFF, 2 * S * nl * sizeof(EpsWin), g->stream));
    CK(cudaMemsetAsync(w.tag, 0, S * nl * 4, g->stream));
    CK(cudaMemsetAsync(w.round_ctr, 0, nl * 4, g->stream));
    std::vector<LaneWs> hl(nl);
    for (size_t l = 0; l < nl; l++) {
        LaneWs &x = hl[l];
        std::memset(&x, 0, sizeof(x));
        if (batched) {
            x.rec = w.rec + l * S;
            x.touched = w.touched + l * nc * S;
        } else {
            x.pk = w.pk + l * S;
            x.tokidx = w.tokidx + l * S;
            x.erec = w.erec + l * S;
            x.msnap = w.msnap + l * S;
            x.touched = w.touched + l * nc * cc;
            x.tcost = w.tcost + l * nc * cc;
            x.tpred = w.tpred + l * nc * cc;
            x.tarc = w.tarc + l * nc * cc;
            x.f0cost = w.f0cost + l * nc * cc;
            x.etouched = w.etouched + l * nc * S;
        }
        x.rpk = w.rpk + l * 2 * S;
        x.tag = w.tag + l * S;
        x.fr = w.fr + l * 2 * nc * S;
        x.fix = w.fix + l * nc * S;
        x.cand = w.cand + l * nc * (size_t)ccap;
        x.candi = w.candi + l * nc * (size_t)ccap;
        x.ccap = ccap;
        x.round_ctr = w.round_ctr + l;
        x.S = (int)S;
        x.C = C;
    }
    CK(cudaMemcpyAsync(w.d_lanes, hl.data(), nl * sizeof(LaneWs), cudaMemcpyHostToDevice, g->stream));
    w.h_lanes = hl;
    CK(cudaStreamSynchronize(g->stream));
    w.lanes = lanes;
    w.C = C;
    w.S = g->S;
    w.ccap = ccap;
    w.tok_cap = tok_cap;
    w.lat_cap = lat ? lat_cap : 0;
    w.path_cap = path_cap;
    w.tmax = tmax;
    w.packs = packs;
    w.lat = lat;
    w.batched = batched;
    return LB_OK;
}

// Epsilon round tags (LaneWs::tag) are compared against a 32-bit per-lane round
// counter that persists across decodes.  Once any lane's counter passes 2^31,
// reset every tag and counter of the workspace, long before a wrap could make a
// stale tag equal the current round (one decode uses far fewer than 2^31 rounds).
int guard_round_tags(Workspace &w, cudaStream_t st) {
    if (w.lanes <= 0) return LB_OK;
    std::vector<unsigned> rc(w.lanes);
    CK(cudaMemcpyAsync(rc.data(), w.round_ctr, 4 * (size_t)w.lanes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    unsigned mx = 0;
    for (unsigned x : rc) mx = std::max(mx, x);
    if (mx < 0x80000000u && !getenv("LB_FORCE_TAG_RESET")) return LB_OK;
    CK(cudaMemsetAsync(w.tag, 0, (size_t)w.S * w.lanes * 4, st));
    CK(cudaMemsetAsync(w.round_ctr, 0, (size_t)w.lanes * 4, st));
    CK(cudaStreamSynchronize(st));
    return LB_OK;
}

// Candidate capacity per CTA: a frame's emitting candidates come from the previous
// frame's tokens (<= max_tok, enforced per frame); warps stride over groups of 32
// tokens, so a CTA of nw warps expands at most nw * ceil(groups / gnw) * 32 tokens.
int64_t cand_capacity(const lb_graph *g, int64_t max_tok, int C, int threads) {
    const int64_t groups = (max_tok + 31) / 32;
    const int64_t nw = threads / 32, gnw = nw * C;
    const int64_t tok_cta = nw * ((groups + gnw - 1) / gnw) * 32;
    // + one partly used chunk per warp (sentinel tails, Lane::emit)
    return std::min<int64_t>(g->A_emit, tok_cta * g->max_edeg) + nw * CAND_CHUNK + CAND_CHUNK;
}

UttDesc slot_desc(const Workspace &w, int l, const double *costs, int T, int64_t tok_cap = -1,
                  int64_t lat_cap = -1) {
    UttDesc d;
    std::memset(&d, 0, sizeof(d));
    const size_t tc = (size_t)w.tok_cap, lc = (size_t)std::max<int64_t>(w.lat_cap, 1);
    d.costs = costs;
    d.T = T;
    d.path_cap = w.path_cap;
    d.tok_cap = tok_cap >= 0 ? std::min<int64_t>(tok_cap, w.tok_cap) : w.tok_cap;
    d.lat_cap = lat_cap >= 0 ? std::min<int64_t>(lat_cap, w.lat_cap) : w.lat_cap;
    d.tok_state = w.tok_state + l * tc;
    d.tok_cost = w.tok_cost + l * tc;
    d.tok_arc = w.tok_arc + l * tc;
    d.tok_pred = w.tok_pred + l * tc;
    d.tok_pack = w.packs ? w.tok_pack + l * tc : nullptr;
    d.tok_base = w.tok_base + (size_t)l * (w.tmax + 2);
    d.lat_base = w.lat_base + (size_t)l * (w.tmax + 2);
    if (w.lat) {
        d.node_extra = w.node_extra + l * tc;
        d.ne_enc = w.ne_enc + l * tc;
        d.lat_arc = w.lat_arc + l * lc;
        d.lat_from = w.lat_from + l * lc;
        d.lat_to = w.lat_to + l * lc;
        d.lat_extra = w.lat_extra + l * lc;
        d.tmp = w.tmp + l * lc;
    }
    return d;   // path / out_* are the job's (ensure_jobs)
}

// Per-job output slots for n utterances with best paths of pstride arcs.
int ensure_jobs(Workspace &w, int n, int pstride) {
    n = std::max(n, 1);
    if (w.jobs_cap >= n && w.jobs_pstride == pstride) return LB_OK;
    w.release_jobs();
    const int cap = std::max(n, w.jobs_cap);
    auto A = [&](auto **p, size_t cnt) -> cudaError_t {
        cudaError_t e = dalloc(p, cnt);
        if (e == cudaSuccess) w.jowned.push_back((void *)*p);
        return e;
    };
    CK(A(&w.j_path, (size_t)cap * pstride));
    CK(A(&w.j_out_i, 8 * (size_t)cap));
    CK(A(&w.j_out_d, 4 * (size_t)cap));
    CK(A(&w.j_out_c, 8 * (size_t)cap));
    CK(A(&w.d_jobs, (size_t)cap));
    CK(A(&w.queue, 1));
    w.jobs_cap = cap;
    w.jobs_pstride = pstride;
    return LB_OK;
}

void fill_message(UttHost &u, int code, int frame, double aux, const lb_config &cfg) {
    char buf[256];
    switch (code) {
        case E_DEAD_NO_CAND:
            u.status = LB_DECODE_FAILURE;
            snprintf(buf, sizeof buf, "beam search died at frame %d: no emitting candidates", frame);
            break;
        case E_DEAD_NO_TOKENS:
            u.status = LB_DECODE_FAILURE;
            snprintf(buf, sizeof buf, "no tokens survived the beam at frame %d", frame);
            break;
        case E_CAP_TOKENS:
            u.status = LB_CAPACITY;
            u.bound = "--max-tokens-per-frame";
            snprintf(buf, sizeof buf, "frame %d kept %lld tokens, over the %lld limit; raise --max-tokens-per-frame",
                     frame, (long long)aux, (long long)cfg.max_tokens_per_frame);
            break;
        case E_CAP_ARENA:
            u.status = LB_CAPACITY;
            u.bound = "--token-arena";
            snprintf(buf, sizeof buf, "token arena overflowed at frame %d (%lld tokens); raise token_arena", frame,
                     (long long)aux);
            break;
        case E_CAP_LATTICE:
            u.status = LB_CAPACITY;
            u.bound = "--max-lattice-arcs";
            snprintf(buf, sizeof buf, "lattice holds %lld arcs at frame %d, over its %lld capacity; raise --max-lattice-arcs",
                     (long long)aux, frame, (long long)cfg.max_lattice_arcs);
            break;
        case E_CAP_PATH:
            u.status = LB_CAPACITY;
            u.bound = "--max-path";
            snprintf(buf, sizeof buf, "best path longer than its buffer");
            break;
        case E_INT_EPS_ROUNDS:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "epsilon relaxation failed to settle within the state count");
            break;
        case E_INT_EPS_PRED:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "epsilon winner's source state kept no token");
            break;
        case E_INT_INIT:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "initial token found at frame %d", frame);
            break;
        case E_INT_BACKTRACE:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "backtrace exceeded its step bound (epsilon cycle at frame %d)", frame);
            break;
        case E_CAP_CAND:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "emitting candidate buffer overflowed at frame %d (sized by construction)", frame);
            break;
        case E_INT_PRUNE_EPS:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "epsilon extra-cost fixpoint did not settle within frame %d", frame);
            break;
        default:
            u.status = LB_INTERNAL;
            snprintf(buf, sizeof buf, "device error code %d at frame %d", code, frame);
    }
    u.msg = buf;
}

int validate_cfg(const lb_config *c) {
    if (!c) return set_err(LB_USAGE, "config is NULL");
    if (!(std::isfinite(c->beam) && c->beam > 0)) return set_err(LB_USAGE, "beam must be a positive finite number");
    if (!(std::isfinite(c->lattice_beam) && c->lattice_beam >= 0)) return set_err(LB_USAGE, "lattice_beam must be >= 0");
    if (!(std::isfinite(c->acoustic_scale) && c->acoustic_scale > 0)) return set_err(LB_USAGE, "acoustic_scale must be > 0");
    if (c->max_active < 0) return set_err(LB_USAGE, "max_active must be >= 0");
    if (c->max_tokens_per_frame < 1) return set_err(LB_USAGE, "max_tokens_per_frame must be >= 1");
    if (c->max_lattice_arcs < 1) return set_err(LB_USAGE, "max_lattice_arcs must be >= 1");
    if (c->threads_per_lane != 0 && c->threads_per_lane != 512 && c->threads_per_lane != LB_LANE_NT &&
        c->threads_per_lane != 768)
        return set_err(LB_USAGE, "threads_per_lane must be 512, 640 or 768");
    if (c->ctas_per_lane < 0 || c->ctas_per_lane > 16) return set_err(LB_USAGE, "ctas_per_lane must be in [0, 16]");
    return LB_OK;
}

// Device lattice finalisation of one utterance (lb_lattice.cuh); fills u.fl_*.
// n elements of T from the graph's pinned arena, kept alive by u.
template <class T>
int arena_take(lb_graph *g, UttHost &u, size_t n, Span<T> &out) {
    const size_t bytes = (n * sizeof(T) + 255) & ~(size_t)255;
    std::shared_ptr<HostArena> &A = g->fl_arena;
    if (!A || A->used + bytes > A->cap) {
        const size_t cap = std::max<size_t>(std::max<size_t>(bytes, g->fl_expect),
                                            A ? 2 * A->cap : ((size_t)64 << 20));
        if (!A || A.use_count() > 1) A = std::make_shared<HostArena>();   // a result still reads the old one
        if (A->p) cudaFreeHost(A->p);
        A->p = nullptr;
        A->cap = A->used = 0;
        const auto ta = std::chrono::steady_clock::now();
        CK(cudaHostAlloc((void **)&A->p, cap, cudaHostAllocDefault));
        if (getenv("LB_FL_DEBUG"))
            fprintf(stderr, "[arena] grow %.0f MB in %.1f ms\n", cap / 1e6,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count());
        A->cap = cap;
    }
    out.p = reinterpret_cast<T *>(A->p + A->used);
    out.n = n;
    A->used += bytes;
    g->fl_taken += bytes;
    if (u.fl_arena != A) u.fl_arena = A;
    return LB_OK;
}

// Returns LB_OK, or an LB_* status for CUDA failures; reference DecodeFailures
// (no surviving arc / start not connected / no terminal node) go to u.status.
int finalize_device(lb_graph *g, const UttDesc &d, int T, int D, double scale, double lattice_beam, int partial,
                    FlScratch &sc, cudaStream_t st, UttHost &u, int remaining = 1) {
    long long tb[2], lbase[2];
    CK(cudaMemcpyAsync(&tb[0], d.tok_base + T + 1, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&lbase[0], d.lat_base + T + 1, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const long long ntok = tb[0], nlat = lbase[0];
    const int nblk = g->sms * 4;
    auto grow = [&](auto **p, size_t n) -> cudaError_t {
        cudaError_t e = dalloc(p, n);
        if (e == cudaSuccess) sc.bufs.push_back((void *)*p);
        return e;
    };
    if ((size_t)ntok > sc.tok_cap || (size_t)nlat > sc.arc_cap || !sc.count) {
        sc.release();
        sc.tok_cap = std::max<size_t>(ntok, 1024);
        sc.arc_cap = std::max<size_t>(nlat, 1024);
        const size_t nt = sc.tok_cap, na = sc.arc_cap;
        CK(grow(&sc.keys0, nt)); CK(grow(&sc.keys1, nt)); CK(grow(&sc.idx0, nt)); CK(grow(&sc.idx1, nt));
        CK(grow(&sc.rank, nt));
        CK(grow(&sc.surv, na)); CK(grow(&sc.fk, na)); CK(grow(&sc.tk, na)); CK(grow(&sc.il, na)); CK(grow(&sc.ol, na));
        CK(grow(&sc.gc, na)); CK(grow(&sc.ac, na)); CK(grow(&sc.nodes0, 2 * na)); CK(grow(&sc.nodes1, 2 * na));
        CK(grow(&sc.fid, na)); CK(grow(&sc.tid, na)); CK(grow(&sc.perm0, na)); CK(grow(&sc.perm1, na));
        CK(grow(&sc.k64a, na)); CK(grow(&sc.k64b, na)); CK(grow(&sc.k32a, na)); CK(grow(&sc.k32b, na));
        CK(grow(&sc.o_from, na)); CK(grow(&sc.o_to, na)); CK(grow(&sc.o_il, na)); CK(grow(&sc.o_ol, na));
        CK(grow(&sc.o_g, na)); CK(grow(&sc.o_ac, na)); CK(grow(&sc.fids, 2 * na)); CK(grow(&sc.fcs, 2 * na));
        CK(grow(&sc.count, 4)); CK(grow(&sc.start_rank, 1)); CK(grow(&sc.n_unique, 1));
        // CUB temp storage for the largest sort / unique of this capacity
        size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, sc.keys0, sc.keys1, sc.idx0, sc.idx1, (int)nt, 0, 64, st));
        CK(cub::DeviceRadixSort::SortKeys(nullptr, t2, sc.nodes0, sc.nodes1, (int)(2 * na), 0, 64, st));
        CK(cub::DeviceSelect::Unique(nullptr, t3, sc.nodes1, sc.nodes0, sc.n_unique, (int)(2 * na), st));
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t4, sc.k64a, sc.k64b, sc.perm0, sc.perm1, (int)na, 0, 64, st));
        sc.temp_cap = std::max(std::max(t1, t2), std::max(t3, t4));
        CK(grow((char **)&sc.temp, sc.temp_cap));
    }
    size_t tcap = sc.temp_cap;
    const int nfr = T + 1;
    // radix sorts run over the key bits actually used
    auto bits = [](unsigned long long x) { int b = 0; while (x) { b++; x >>= 1; } return std::max(b, 1); };
    const int sbits = bits((unsigned long long)std::max<int64_t>(g->S - 1, 1));
    const int fbits = bits((unsigned long long)nfr);
    // 1-2: state-sorted token ranks per frame
    fl_token_keys<<<nblk, 256, 0, st>>>(d.tok_state, d.tok_base, nfr, ntok, sbits, sc.keys0, sc.idx0);
    CK(cub::DeviceRadixSort::SortPairs(sc.temp, tcap, sc.keys0, sc.keys1, sc.idx0, sc.idx1, (int)ntok, 0,
                                       std::min(64, sbits + fbits), st));
    CK(cudaMemsetAsync(sc.start_rank, 0xFF, 8, st));
    fl_token_rank<<<nblk, 256, 0, st>>>(sc.keys1, sc.idx1, d.tok_base, ntok, sbits, g->start, sc.rank, sc.start_rank);
    // 3: survivors
    CK(cudaMemsetAsync(sc.count, 0, 32, st));
    fl_survivors<<<nblk, 256, 0, st>>>(d.lat_extra, nlat, lattice_beam, sc.surv, sc.count);
    unsigned long long m = 0;
    long long start_rank = -1;
    CK(cudaMemcpyAsync(&m, sc.count, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&start_rank, sc.start_rank, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    u.has_final = true;
    if (m == 0) {
        u.status = LB_DECODE_FAILURE;
        u.msg = "no lattice arcs survived pruning";
        return LB_OK;
    }
    // 4: arc fields + node keys, sorted unique nodes, dense ids
    fl_arc_fields<<<nblk, 256, 0, st>>>(g->dev(), sc.surv, (long long)m, d.lat_arc, d.lat_from, d.lat_to, d.lat_base,
                                        d.tok_base, nfr, sc.rank, d.costs, D, scale, sc.fk, sc.tk, sc.il, sc.ol, sc.gc,
                                        sc.ac, sc.nodes0);
    CK(cub::DeviceRadixSort::SortKeys(sc.temp, tcap, sc.nodes0, sc.nodes1, (int)(2 * m), 0, std::min(64, 32 + fbits),
                                      st));
    CK(cub::DeviceSelect::Unique(sc.temp, tcap, sc.nodes1, sc.nodes0, sc.n_unique, (int)(2 * m), st));
    int nn = 0;
    CK(cudaMemcpyAsync(&nn, sc.n_unique, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fl_node_ids<<<nblk, 256, 0, st>>>(sc.fk, sc.tk, (long long)m, sc.nodes0, nn, sc.fid, sc.tid);
    // 5: canonical order = np.lexsort((ac, g, ol, il, to, from)): stable LSD passes, last key primary
    fl_iota<<<nblk, 256, 0, st>>>(sc.perm0, (long long)m);
    int *pa = sc.perm0, *pb = sc.perm1;
    for (int pass = 0; pass < 6; pass++) {
        if (pass < 2) {
            fl_gather_u64<<<nblk, 256, 0, st>>>(pass == 0 ? sc.ac : sc.gc, pa, (long long)m, sc.k64a);
            CK(cub::DeviceRadixSort::SortPairs(sc.temp, tcap, sc.k64a, sc.k64b, pa, pb, (int)m, 0, 64, st));
        } else {
            const unsigned *src = pass == 2 ? sc.ol : pass == 3 ? sc.il : pass == 4 ? sc.tid : sc.fid;
            const int kb = pass == 3 ? bits((unsigned long long)std::max(g->max_ilabel, 1))
                         : pass >= 4 ? bits((unsigned long long)std::max(nn - 1, 1)) : 32;
            fl_gather_u32<<<nblk, 256, 0, st>>>(src, pa, (long long)m, sc.k32a);
            CK(cub::DeviceRadixSort::SortPairs(sc.temp, tcap, sc.k32a, sc.k32b, pa, pb, (int)m, 0, kb, st));
        }
        std::swap(pa, pb);
    }
    fl_emit<<<nblk, 256, 0, st>>>(pa, (long long)m, sc.fid, sc.tid, sc.il, sc.ol, sc.gc, sc.ac, sc.o_from, sc.o_to,
                                  sc.o_il, sc.o_ol, sc.o_g, sc.o_ac);
    // 6: final nodes
    fl_finals<<<nblk, 256, 0, st>>>(sc.nodes0, nn, T, sc.keys1, sbits, d.tok_base, g->fin, partial, sc.fids, sc.fcs,
                                    sc.count + 1);
    CK(cudaGetLastError());
    unsigned long long nf = 0;
    CK(cudaMemcpyAsync(&nf, sc.count + 1, 8, cudaMemcpyDeviceToHost, st));
    // if the arena must grow, size it for this utterance times the ones left
    g->fl_expect = ((size_t)8 * nn + (size_t)32 * m + 7 * 256) * (size_t)std::max(remaining, 1) * 5 / 4;
    if (int rc = arena_take(g, u, nn, u.fl_nodes)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_from)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_to)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_il)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_ol)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_g)) return rc;
    if (int rc = arena_take(g, u, m, u.fl_ac)) return rc;
    CK(cudaMemcpyAsync(u.fl_nodes.data(), sc.nodes0, 8 * (size_t)nn, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_from.data(), sc.o_from, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_to.data(), sc.o_to, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_il.data(), sc.o_il, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_ol.data(), sc.o_ol, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_g.data(), sc.o_g, 8 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_ac.data(), sc.o_ac, 8 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> ids(nf);
    std::vector<double> fcs(nf);
    CK(cudaMemcpy(ids.data(), sc.fids, 8 * nf, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(fcs.data(), sc.fcs, 8 * nf, cudaMemcpyDeviceToHost));
    std::vector<size_t> ord(nf);
    for (size_t i = 0; i < nf; i++) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
    u.fl_final_ids.resize(nf);
    u.fl_final_costs.resize(nf);
    for (size_t i = 0; i < nf; i++) {
        u.fl_final_ids[i] = ids[ord[i]];
        u.fl_final_costs[i] = fcs[ord[i]];
    }
    // start node (frame 0, the start token's rank)
    const uint64_t sk = (uint64_t)(start_rank < 0 ? 0 : start_rank);
    auto it = std::lower_bound(u.fl_nodes.begin(), u.fl_nodes.end(), sk);
    if (start_rank < 0 || it == u.fl_nodes.end() || *it != sk) {
        u.status = LB_DECODE_FAILURE;
        u.msg = "surviving arcs do not connect to the start node";
        return LB_OK;
    }
    u.fl_start = it - u.fl_nodes.begin();
    if (nf == 0) {
        u.status = LB_DECODE_FAILURE;
        u.msg = "no terminal node survived pruning";
    }
    return LB_OK;
}

// One wave in the frame-synchronous batched mode (lb_batched.cuh): 6-7 phase
// kernels per frame over all nw lanes, launched back to back on the stream.
int launch_batched_seq(lb_graph *g, const GraphDev &gd, const Params &p, Workspace &w, int nw, const int32_t *T,
                       int bpl, cudaStream_t st, lb_result *res, int l0 = 0);

// The per-frame launch sequence is captured once into a CUDA graph and replayed:
// ~7 launches per frame would otherwise cost more CPU time than a small batch's
// GPU time, and the graph also shortens the GPU-side gaps between the kernels.
int launch_batched(lb_graph *g, const GraphDev &gd, const Params &p, Workspace &w, int nw, const int32_t *T, int bpl,
                   cudaStream_t st, lb_result *res) {
    if (getenv("LB_BATCH_PROFILE") || getenv("LB_NO_GRAPH")) return launch_batched_seq(g, gd, p, w, nw, T, bpl, st, res);
    int tmax = 0;
    for (int l = 0; l < nw; l++) tmax = std::max(tmax, (int)T[l]);
    std::string key((const char *)&p, sizeof(Params));
    key += std::string(getenv("LB_GROUPS") ? getenv("LB_GROUPS") : "-") + "/";
    key += std::to_string(nw) + "/" + std::to_string(tmax) + "/" + std::to_string(bpl) + "/" +
           std::to_string((unsigned long long)(uintptr_t)w.d_lanes) + "/" +
           std::to_string((unsigned long long)(uintptr_t)w.d_ctl) + "/" +
           std::to_string((unsigned long long)(uintptr_t)w.d_desc);
    if (!g->bexec || g->bkey != key) {
        if (g->bexec) {
            cudaGraphExecDestroy(g->bexec);
            g->bexec = nullptr;
        }
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        lb_result dummy;
        // lane groups on forked streams: independent chains in the graph, so one
        // group's latency-bound epsilon rounds overlap another group's throughput
        // phases (the overlap the persistent-lane kernel gets for free)
        const char *ge = getenv("LB_GROUPS");
        const int groups = std::max(1, std::min(nw, ge ? atoi(ge) : (nw >= 16 ? 4 : nw >= 8 ? 2 : 1)));
        int rc = LB_OK;
        if (groups == 1) {
            rc = launch_batched_seq(g, gd, p, w, nw, T, bpl, cs, &dummy);
        } else {
            cudaEvent_t fork;
            CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
            CK(cudaEventRecord(fork, cs));
            std::vector<cudaStream_t> ss(groups);
            std::vector<cudaEvent_t> joins(groups);
            for (int q = 0; q < groups; q++) {
                const int a = nw * q / groups, b = nw * (q + 1) / groups;
                CK(cudaStreamCreateWithFlags(&ss[q], cudaStreamNonBlocking));
                CK(cudaStreamWaitEvent(ss[q], fork, 0));
                const int bq = std::max(1, (g->sms * 4) / std::max(1, b - a));
                if (!rc) rc = launch_batched_seq(g, gd, p, w, b - a, T + a, bq, ss[q], &dummy, a);
                CK(cudaEventCreateWithFlags(&joins[q], cudaEventDisableTiming));
                CK(cudaEventRecord(joins[q], ss[q]));
                CK(cudaStreamWaitEvent(cs, joins[q], 0));
            }
            for (int q = 0; q < groups; q++) {
                cudaEventDestroy(joins[q]);
                cudaStreamDestroy(ss[q]);
            }
            cudaEventDestroy(fork);
        }
        cudaGraph_t graph;
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        if (ce != cudaSuccess) return set_err(LB_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        CK(cudaGraphInstantiate(&g->bexec, graph, 0));
        cudaGraphDestroy(graph);
        g->bkey = key;
        g->blaunches = dummy.launches;
    }
    CK(cudaGraphLaunch(g->bexec, st));
    res->launches += g->blaunches;
    return LB_OK;
}

int launch_batched_seq(lb_graph *g, const GraphDev &gd, const Params &p, Workspace &w, int nw, const int32_t *T,
                       int bpl, cudaStream_t st, lb_result *res, int l0) {
    int tmax = 0;
    for (int l = 0; l < nw; l++) tmax = std::max(tmax, (int)T[l]);
    const LaneWs *lw = w.d_lanes + l0;     // this lane group's slice (l0 = first lane)
    const UttDesc *ud = w.d_desc + l0;
    LaneCtl *ctl = w.d_ctl + l0;
    const dim3 grid((unsigned)bpl, (unsigned)nw);
    constexpr int ENT = 512, ECL = 2, FNT = 512;
    cudaLaunchConfig_t ec = {};
    ec.gridDim = dim3((unsigned)(nw * ECL));
    ec.blockDim = dim3(ENT);
    ec.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ECL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    ec.attrs = at;
    ec.numAttrs = 1;
    int launches = 0;
    // LB_BATCH_PROFILE=1: CUDA-event time per phase kernel, summed (stderr)
    const bool bprof = getenv("LB_BATCH_PROFILE") != nullptr;
    std::vector<cudaEvent_t> evs;
    std::vector<int> ev_kind;
    auto mark = [&](int kind) {
        if (!bprof) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        evs.push_back(e);
        ev_kind.push_back(kind);
    };
    auto eps = [&]() -> int {
        if (!gd.has_eps) return LB_OK;
        CK(cudaLaunchKernelEx(&ec, b_epsilon<ENT>, gd, p, lw, (LaneCtl *)ctl, nw));
        launches++;
        return LB_OK;
    };
    mark(-1);
    b_init<<<nw, 32, 0, st>>>(gd, p, lw, ud, ctl, nw);
    if (int rc = eps()) return rc;
    b_aggregate<<<grid, BNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
    if (p.want_lattice) b_lattice<<<grid, BNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
    b_turnover<<<nw, 32, 0, st>>>(p, ud, ctl, nw);
    mark(6);
    launches += 3;
    for (int t = 1; t <= tmax; t++) {
        b_emit<<<grid, BNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
        mark(0);
        b_winners<<<grid, BNT, 0, st>>>(gd, p, lw, ctl, nw);
        mark(1);
        b_max_active<<<nw, 32, 0, st>>>(p, ctl, nw);
        mark(2);
        if (int rc = eps()) return rc;
        mark(3);
        b_aggregate<<<grid, BNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
        if (p.want_lattice) b_lattice<<<grid, BNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
        mark(4);
        b_turnover<<<nw, 32, 0, st>>>(p, ud, ctl, nw);
        mark(5);
        launches += 5;
    }
    if (bprof) {
        cudaStreamSynchronize(st);
        double acc[8] = {0};
        for (size_t k = 1; k < evs.size(); k++) {
            float ms = 0;
            cudaEventElapsedTime(&ms, evs[k - 1], evs[k]);
            acc[ev_kind[k]] += ms;
        }
        const char *nm[7] = {"emit", "winners", "max_active", "epsilon", "aggregate", "turnover", "frame0"};
        fprintf(stderr, "[batched profile] frames=%d lanes=%d bpl=%d  ", tmax, nw, bpl);
        for (int k = 0; k < 7; k++) fprintf(stderr, "%s=%.1fus ", nm[k], acc[k] * 1e3 / std::max(tmax, 1));
        fprintf(stderr, "(per frame)\n");
        for (auto e : evs) cudaEventDestroy(e);
    }
    b_final<FNT><<<nw, FNT, 0, st>>>(gd, p, lw, ud, ctl, nw);
    launches++;
    CK(cudaGetLastError());
    res->launches += launches;
    return LB_OK;
}

// How many C-CTA lane clusters of `threads` threads fit on the device at once
// (cudaOccupancyMaxActiveClusters on the 1-best lane kernel), cached per graph.
int max_coresident_clusters(lb_graph *g, int C, int threads, size_t dsm) {
    const long long key = ((long long)C << 40) | ((long long)threads << 24) | (long long)dsm;
    auto it = g->cluster_fit.find(key);
    if (it != g->cluster_fit.end()) return it->second;
    using KernT = void (*)(const GraphDev, const Params, const LaneWs *, const UttDesc *, const UttJob *, int, int *);
    KernT k = threads == 512 ? (KernT)decode_kernel<512, 4, false, false>
            : threads == 768 ? (KernT)decode_kernel<768, 2, false, false>
                             : (KernT)decode_kernel<LB_LANE_NT, LB_UNR640, false, false>;
    int num = 0;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(dsm, 1)) ==
            cudaSuccess &&
        (C <= 8 || cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(C * std::max(1, g->sms / C)));
        lc.blockDim = dim3((unsigned)threads);
        lc.dynamicSmemBytes = dsm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&num, (void *)k, &lc) != cudaSuccess) num = 0;
    }
    cudaGetLastError();
    g->cluster_fit[key] = num;
    return num;
}

// Mode and lane cluster size of a decode call (shared by decode_impl and the
// staging decision of lb_decode_batch).
void choose_mode(lb_graph *g, int n, int D, const lb_config *cfg, bool &batched, int &C) {
    const bool lat = cfg->want_lattice != 0;
    const int threads = cfg->threads_per_lane ? cfg->threads_per_lane : LB_LANE_NT;
    // Mode: the frame-synchronous batched kernels (lb_batched.cuh, replayed as a
    // CUDA graph, lanes in 4 concurrent groups) spread every phase over all SMs
    // and win for small and medium batches (1 utterance: 17.8k vs 8.1k frames/s;
    // 32: 317k vs 259k; 40: 341k vs 316k); the persistent-lane kernel wins from
    // ~44 concurrent utterances up (48: 369k vs 356k; 64: 447k vs 375k frames/s;
    // C2 graph, tools/mode_crossover.sh).  LB_MODE=lane|batched overrides.
    const char *mode_env = getenv("LB_MODE");
    batched = n <= BATCHED_MAX_UTTS;
    if (mode_env && !strcmp(mode_env, "lane")) batched = false;
    if (mode_env && !strcmp(mode_env, "batched")) batched = true;
    int autoC = 2;
    // 1-best batches of 5+ utterances: the widest lane cluster (8, 4 or 3 CTAs)
    // of which n are co-resident beats both the batched mode and 2-CTA lanes
    // (C2 graph, frames/s: 8 utts 124k vs 112k batched at C=8; 32: 373k vs 317k
    // at C=4; 44: 415k vs 349k batched and 350k at C=2 with C=3; measured with
    // tools/mode_auto.sh).
    // 16-CTA lanes (non-portable cluster size; 7 co-resident) took over the
    // smallest batches, single utterances included, on every graph shape
    // (tools/mode_sweep.py, frames/s): C5 1 utt 12.0k vs 8.1k batched, 6 utts
    // 64.5k vs 50.9k at C=8; C1 1 utt 47.0k vs 36.4k batched, 4 utts 183k vs
    // 133k at C=8; C2 1 utt 18.8k vs 17.6k batched, 4 utts 72.9k vs 68.4k.
    // Lattice decodes take 16-CTA lanes only (C3 1 utt 14.5k vs 12.2k batched,
    // 4 utts 56.2k vs 42.5k; C1 4 utts 133.6k vs 90.6k, where 8-CTA lanes lose
    // to the batched mode) and otherwise stay batched / 2-CTA.
    if (!mode_env && cfg->ctas_per_lane == 0 && n >= 1) {
        const bool acs = (size_t)D * 8 <= ACROW_SMEM_MAX;
        const size_t dsm = lane_dyn_smem(threads, D, acs, acs && D % 2 == 0);   // with the row prefetch buffers
        for (int c : {16, 8, 4, 3}) {
            if (c == 16 ? getenv("LB_NO_C16") != nullptr : lat) continue;
            if (n <= max_coresident_clusters(g, c, threads, dsm)) {
                batched = false;
                autoC = c;
                break;
            }
        }
    }
    C = batched ? 1 : (cfg->ctas_per_lane > 0 ? cfg->ctas_per_lane : autoC);
    if (getenv("LB_MODE_DEBUG"))
        fprintf(stderr, "[mode] n=%d %s C=%d (fit C3=%d C4=%d C8=%d C16=%d, smem without row prefetch)\n", n,
                batched ? "batched" : "lane", C,
                max_coresident_clusters(g, 3, threads, lane_dyn_smem(threads, D, (size_t)D * 8 <= ACROW_SMEM_MAX)),
                max_coresident_clusters(g, 4, threads, lane_dyn_smem(threads, D, (size_t)D * 8 <= ACROW_SMEM_MAX)),
                max_coresident_clusters(g, 8, threads, lane_dyn_smem(threads, D, (size_t)D * 8 <= ACROW_SMEM_MAX)),
                max_coresident_clusters(g, 16, threads, lane_dyn_smem(threads, D, (size_t)D * 8 <= ACROW_SMEM_MAX)));
}

// Streaming host ring of a refilling decode (lb_decode_batch, large 1-best batches).
struct RingDev {
    const int *ready;
    int *done;
    const double *base;
    long long slot_doubles;
    int slots;
};

// Queue order of a refilling decode: longest first, ties in input order (LPT).
std::vector<int32_t> lpt_order(int n, const int32_t *T) {
    std::vector<int32_t> ord(n);
    for (int u = 0; u < n; u++) ord[u] = u;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return T[x] > T[y]; });
    return ord;
}

int decode_impl(lb_graph *g, int32_t n, const double *const *dev_costs, const int32_t *T, int32_t D,
                const lb_config *cfg, cudaStream_t st, lb_result *res, float h2d_ms, const int *d_ready = nullptr,
                const RingDev *ring = nullptr, bool costs_f32 = false) {
    Nvtx range_("lb.decode");
    const bool lat = cfg->want_lattice != 0;
    if (lat) {
        // size the arena for what the last lattice decode took, so a steady
        // workload never grows it mid-decode (a growth is a fresh cudaHostAlloc)
        std::shared_ptr<HostArena> &A = g->fl_arena;
        const size_t need = g->fl_taken + g->fl_taken / 4;
        if (g->fl_taken > 0 && (!A || A.use_count() > 1 || A->cap < g->fl_taken)) {
            if (A && A.use_count() == 1 && A->p) {
                cudaFreeHost(A->p);
                A->p = nullptr;
                A->cap = A->used = 0;
            } else {
                A = std::make_shared<HostArena>();
            }
            const auto ta = std::chrono::steady_clock::now();
            CK(cudaHostAlloc((void **)&A->p, need, cudaHostAllocDefault));
            if (getenv("LB_FL_DEBUG"))
                fprintf(stderr, "[arena] presize %.0f MB in %.1f ms\n", need / 1e6,
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count());
            A->cap = need;
        }
        if (A && A.use_count() == 1) A->used = 0;   // no result reads it any more
        g->fl_taken = 0;
    }
    const bool keep_work = lat && cfg->keep_work_lattice != 0;
    const bool packs = cfg->collect_frame_packs != 0 || keep_work;
    int tmax = 1;
    for (int i = 0; i < n; i++) tmax = std::max(tmax, (int)T[i]);
    const int64_t S = g->S;
    int64_t per_frame = std::min<int64_t>(S, cfg->max_tokens_per_frame);
    if (cfg->max_active > 0) per_frame = std::min<int64_t>(per_frame, 4 * cfg->max_active + 1024);
    int64_t tok_cap = cfg->token_arena > 0 ? cfg->token_arena : (int64_t)(tmax + 1) * per_frame;
    tok_cap = std::min<int64_t>(tok_cap, (int64_t)1 << 31);
    const int64_t lat_cap = lat ? std::min<int64_t>(cfg->max_lattice_arcs, (int64_t)1 << 31) : 0;
    const int path_cap = 4 * tmax + 256;
    int threads = cfg->threads_per_lane ? cfg->threads_per_lane : LB_LANE_NT;
    bool batched;
    int C;
    choose_mode(g, n, D, cfg, batched, C);
    const int64_t max_tok = std::min<int64_t>(S, cfg->max_tokens_per_frame);
    int lanes_guess = cfg->lanes > 0 ? cfg->lanes : std::min<int>(n, std::max(1, g->sms / 2));
    lanes_guess = std::max(1, std::min(lanes_guess, n > 0 ? n : 1));
    const int bpl = std::max(1, (g->sms * 4) / lanes_guess);   // batched: blocks per lane per phase kernel
    // batched mode: every warp that gets tokens leaves at most one partly used
    // chunk, and a wave's lane groups may run up to sms*4 blocks per lane (a group
    // of one lane), so the tail is bounded by min(all warps, token groups) chunks
    const int64_t ccap = batched ? std::min<int64_t>(g->A_emit, max_tok * g->max_edeg) +
                                       (std::min<int64_t>((int64_t)g->sms * 4 * BNW, (max_tok + 31) / 32) + 1) * BCCH
                                 : cand_capacity(g, max_tok, C, threads);
    // lanes: requested, else as many as fit a memory budget (<= 1 wave of SMs)

    int lanes = batched ? lanes_guess : (cfg->lanes > 0 ? cfg->lanes : std::min<int>(n, std::max(1, g->sms / C)));
    lanes = std::max(1, std::min(lanes, n > 0 ? n : 1));
    // Refilling 1-best lanes (see below).  When the requested lanes leave SMs
    // idle (64 two-CTA lanes use 128 of 148), the first `n3` lanes run as
    // three-CTA clusters in a concurrent launch on the same job queue, so every
    // SM decodes (still `lanes` lanes; a wider lane just takes more jobs).
    const bool refill_mode = !batched && !lat && !packs && d_ready == nullptr && !getenv("LB_NO_REFILL");
    int n3 = 0;
    if (refill_mode && C == 2 && cfg->ctas_per_lane == 0 && n > lanes && !getenv("LB_NO_MIXED"))
        n3 = std::max(0, std::min(lanes, g->sms - 2 * lanes));
    if (const char *e = getenv("LB_MIXED_N3"))   // test knob: force n3 (2-CTA refilling lanes only)
        if (refill_mode && C == 2 && n > lanes) n3 = std::max(0, std::min(lanes, atoi(e)));
    const int Ca = n3 > 0 ? 3 : C;   // CTA segments allocated per lane
    if (getenv("LB_MODE_DEBUG")) fprintf(stderr, "[lanes] %d lanes, %d of them 3-CTA, C=%d\n", lanes, n3, C);
    const size_t per_lane = lane_bytes(S, Ca, ccap, tok_cap, lat_cap, path_cap, tmax, packs, lat, batched);
    const Workspace &w0 = g->ws;
    const bool fits = w0.batched == batched && w0.lanes >= lanes && w0.C == Ca && w0.S == g->S && w0.ccap >= ccap && w0.tok_cap >= tok_cap &&
                      w0.lat_cap >= lat_cap && w0.path_cap >= path_cap && w0.tmax >= tmax && (w0.packs || !packs) &&
                      (w0.lat || !lat);
    if (!fits) {   // size the lane count to the device memory left (the workspace is reused across calls)
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        // the current workspace is freed before the new one is allocated, whatever its shape
        const size_t reuse = w0.lanes > 0 ? (size_t)w0.lanes * lane_bytes(S, w0.C, w0.ccap, w0.tok_cap, w0.lat_cap,
                                                                           w0.path_cap, w0.tmax, w0.packs, w0.lat,
                                                                           w0.batched)
                                          : 0;
        const size_t budget = (size_t)((double)(free_b + reuse) * 0.85);
        while (lanes > 1 && (size_t)lanes * per_lane > budget) lanes--;
        if ((size_t)lanes * per_lane > budget)
            return set_err(LB_CAPACITY, "not enough device memory for one decode lane; lower token_arena / max_lattice_arcs");
    }
    int rc = ensure_workspace(g, g->ws, lanes, Ca, ccap, tok_cap, lat_cap, path_cap, tmax, packs, lat, batched);
    if (rc) return rc;
    Workspace &w = g->ws;

    Params p;
    std::memset(&p, 0, sizeof(p));   // padding too: the batched-mode graph cache keys on the raw bytes
    p.beam = cfg->beam;
    p.lattice_beam = cfg->lattice_beam;
    p.scale = cfg->acoustic_scale;
    p.max_active = cfg->max_active;
    p.max_tokens = cfg->max_tokens_per_frame;
    p.D = D;
    p.want_lattice = lat;
    p.collect_packs = packs;
    const size_t acrow_bytes = (size_t)D * 8;
    p.acrow_smem = acrow_bytes <= ACROW_SMEM_MAX;
    p.prof = nullptr;
    p.ready = d_ready;
    if (batched && d_ready) return set_err(LB_INTERNAL, "progressive staging needs the lane kernel");
    p.costs_f32 = costs_f32;
    if (ring) {
        p.ring_ready = ring->ready;
        p.ring_done = ring->done;
        p.ring_base = ring->base;
        p.ring_slot_doubles = ring->slot_doubles;
        p.ring_slots = ring->slots;
    }
    const char *pe = getenv("LB_PHASE_PROFILE");
    unsigned long long *d_prof = nullptr;
    if (pe && pe[0] == '1') {
        CK(cudaMalloc((void **)&d_prof, 24 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(d_prof, 0, 24 * sizeof(unsigned long long), st));
        p.prof = d_prof;
    }
    // next-frame row prefetch: f64 rows of even D (16-byte cp.async chunks), not
    // while rows are published progressively, and only if two row buffers fit
    bool aligned = ring == nullptr || (ring->slot_doubles % 2 == 0);   // ring slots start on 128-byte lines
    for (int u = 0; u < n && aligned && !ring; u++) aligned = ((uintptr_t)dev_costs[u] & 15) == 0;
    p.row_pf = !batched && p.acrow_smem && !d_ready && !costs_f32 && (D % 2 == 0) && aligned &&
               !getenv("LB_NO_ROWPF") && lane_dyn_smem(threads, D, true, true) <= 227 * 1024;
    size_t smem = lane_dyn_smem(threads, D, p.acrow_smem != 0, p.row_pf != 0);
    if (const char *e = getenv("LB_SMEM_PAD")) smem += (size_t)atoi(e);   // measurement knob (L1 carveout)
    // decode-lane variants: CTA size x batch width x lattice x phase-profile
    using KernT = void (*)(const GraphDev, const Params, const LaneWs *, const UttDesc *, const UttJob *, int, int *);
    const bool prof = p.prof != nullptr;
#define LB_PICK(NT, U)                                                                     \
    (lat ? (prof ? decode_kernel<NT, U, true, true> : decode_kernel<NT, U, true, false>) \
         : (prof ? decode_kernel<NT, U, false, true> : decode_kernel<NT, U, false, false>))
    KernT kern;
    // 640 threads (96 registers, few spills) measured best on C4: 440k vs 392k
    // frames/s at 768 and 417k at 512 (tools/cta_sweep.sh)
    if (threads == LB_LANE_NT) kern = LB_PICK(LB_LANE_NT, LB_UNR640);
    else if (threads == 768) kern = LB_PICK(768, 2);
    else if (threads == 512) kern = LB_PICK(512, 4);
    else return set_err(LB_USAGE, "threads_per_lane must be 512, 640 or 768");
#undef LB_PICK
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
    if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));   // up to 16 on B200
    const GraphDev gd = g->dev();

    // Per-utterance output slots (status, costs, counters, best path) for the
    // whole call, so lanes that refill from the job queue keep every result.
    const int pstride = path_cap;
    if (int rj = ensure_jobs(w, n, pstride)) return rj;
    std::vector<UttJob> hj(n);
    for (int u = 0; u < n; u++) {
        UttJob &J = hj[u];
        std::memset(&J, 0, sizeof(J));
        J.costs = dev_costs[u];
        J.T = T[u];
        J.path = w.j_path + (size_t)u * pstride;
        J.out_i = w.j_out_i + 8 * (size_t)u;
        J.out_d = w.j_out_d + 4 * (size_t)u;
        J.out_c = w.j_out_c + 8 * (size_t)u;
    }
    // Refilling lanes (1-best in the persistent-lane kernel): ONE launch for the
    // whole call; lanes claim jobs longest first from a device counter, so a
    // ragged batch never waits for a wave's longest utterance.  Lattice and
    // token-list decodes keep their per-utterance arenas until readback, so they
    // run in waves of `lanes` utterances (the wave's lane l decodes job l).
    const bool refill = refill_mode;
    if (ring && !(refill && p.acrow_smem)) return set_err(LB_INTERNAL, "streamed staging needs refilling lanes");
    if (costs_f32 && !(refill && p.acrow_smem)) return set_err(LB_INTERNAL, "f32 rows need refilling lanes");
    std::vector<UttJob> jq(n);
    if (refill) {
        const std::vector<int32_t> ord = lpt_order(n, T);
        for (int k = 0; k < n; k++) jq[k] = hj[ord[k]];
    } else {
        jq = hj;
    }
    CK(cudaMemcpyAsync(w.d_jobs, jq.data(), (size_t)n * sizeof(UttJob), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(w.j_out_i, 0, 8 * sizeof(int) * (size_t)std::max(n, 1), st));

    cudaEvent_t e0, e1, e2, e3;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    CK(cudaEventCreate(&e3));
    res->utts.resize(n);
    res->t_h2d = h2d_ms;
    FlScratch &fl = g->fl;
    std::vector<UttDesc> desc(lanes);
    std::vector<int> hi(8 * (size_t)std::max(n, 1));
    std::vector<double> hd(4 * (size_t)std::max(n, 1));
    std::vector<long long> hc(8 * (size_t)std::max(n, 1));
    std::vector<int> hpath((size_t)pstride * std::max(n, 1));
    const int step = refill ? n : lanes;
    for (int w0 = 0; w0 < n; w0 += step) {
        const int nw = refill ? std::min(lanes, n) : std::min(lanes, n - w0);   // lanes launched
        const int nj = refill ? n : nw;                                          // jobs of the launch
        for (int l = 0; l < nw; l++) {
            desc[l] = slot_desc(w, l, nullptr, 0, tok_cap, lat_cap);
            desc[l].path_cap = pstride;   // the job path slots' stride (ensure_jobs)
            if (!refill) {   // the wave's job l (the prune kernel and finaliser read these)
                desc[l].costs = dev_costs[w0 + l];
                desc[l].T = T[w0 + l];
                desc[l].path = hj[w0 + l].path;
                desc[l].out_i = hj[w0 + l].out_i;
                desc[l].out_d = hj[w0 + l].out_d;
                desc[l].out_c = hj[w0 + l].out_c;
            }
        }
        CK(cudaMemcpyAsync(w.d_desc, desc.data(), nw * sizeof(UttDesc), cudaMemcpyHostToDevice, st));
        if (refill) CK(cudaMemsetAsync(w.queue, 0, sizeof(int), st));
        CK(cudaEventRecord(e0, st));
        if (batched) {
            int rcb = launch_batched(g, gd, p, w, nw, T + w0, bpl, st, res);
            if (rcb) return rcb;
        } else {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)(nw * C));
            lc.blockDim = dim3((unsigned)threads);
            lc.dynamicSmemBytes = smem;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)C;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            if (n3 > 0) {
                // lanes [0, n3) as 3-CTA clusters on a forked stream, the rest as
                // 2-CTA clusters here; both claim from the same queue
                std::vector<LaneWs> hm(w.h_lanes.begin(), w.h_lanes.begin() + nw);
                for (int l = 0; l < nw; l++) hm[l].C = l < n3 ? 3 : 2;
                CK(cudaMemcpyAsync(w.d_lanes_mix, hm.data(), nw * sizeof(LaneWs), cudaMemcpyHostToDevice, st));
                if (!g->stream2) CK(cudaStreamCreateWithFlags(&g->stream2, cudaStreamNonBlocking));
                if (!g->ev_fork) CK(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
                if (!g->ev_join) CK(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
                CK(cudaEventRecord(g->ev_fork, st));
                CK(cudaStreamWaitEvent(g->stream2, g->ev_fork, 0));
                cudaLaunchConfig_t l3 = lc;
                cudaLaunchAttribute a3[1];
                a3[0] = at[0];
                a3[0].val.clusterDim.x = 3;
                l3.attrs = a3;
                l3.gridDim = dim3((unsigned)(n3 * 3));
                l3.stream = g->stream2;
                CK(cudaLaunchKernelEx(&l3, kern, gd, p, (const LaneWs *)w.d_lanes_mix, (const UttDesc *)w.d_desc,
                                      (const UttJob *)w.d_jobs, nj, w.queue));
                lc.gridDim = dim3((unsigned)((nw - n3) * 2));
                if (nw > n3)
                    CK(cudaLaunchKernelEx(&lc, kern, gd, p, (const LaneWs *)(w.d_lanes_mix + n3),
                                          (const UttDesc *)(w.d_desc + n3), (const UttJob *)w.d_jobs, nj, w.queue));
                CK(cudaEventRecord(g->ev_join, g->stream2));
                CK(cudaStreamWaitEvent(st, g->ev_join, 0));
                res->launches += nw > n3 ? 2 : 1;
            } else {
                CK(cudaLaunchKernelEx(&lc, kern, gd, p, (const LaneWs *)w.d_lanes, (const UttDesc *)w.d_desc,
                                      (const UttJob *)(w.d_jobs + (refill ? 0 : w0)), nj, refill ? w.queue : nullptr));
                res->launches++;
            }
        }
        CK(cudaEventRecord(e1, st));
        if (lat) {
            Nvtx rp("lb.prune");
            // one cluster per utterance, as wide as the GPU allows (portable max 8)
            const unsigned pc = (unsigned)std::max(1, std::min(8, g->sms / std::max(nw, 1)));
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)nw * pc);
            lc.blockDim = dim3(1024);
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = pc;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, prune_kernel, gd, p, (const UttDesc *)w.d_desc, nw));
            res->launches++;
        }
        CK(cudaEventRecord(e2, st));
        Nvtx rr("lb.readback+finalize");
        const int u0 = refill ? 0 : w0;
        CK(cudaMemcpyAsync(hi.data() + 8 * (size_t)u0, w.j_out_i + 8 * (size_t)u0, 8 * sizeof(int) * (size_t)nj,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hd.data() + 4 * (size_t)u0, w.j_out_d + 4 * (size_t)u0, 4 * sizeof(double) * (size_t)nj,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hc.data() + 8 * (size_t)u0, w.j_out_c + 8 * (size_t)u0, 8 * sizeof(long long) * (size_t)nj,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hpath.data() + (size_t)pstride * u0, w.j_path + (size_t)pstride * u0,
                           sizeof(int) * (size_t)pstride * nj, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        res->t_decode += ms;
        CK(cudaEventElapsedTime(&ms, e1, e2));
        res->t_prune += ms;
        CK(cudaEventRecord(e2, st));
        for (int k = 0; k < nj; k++) {
            const int uu = u0 + k;
            UttHost &u = res->utts[uu];
            const int code = hi[8 * (size_t)uu + 0];
            std::memcpy(u.counters, &hc[8 * (size_t)uu], sizeof(u.counters));
            if (code != E_OK) {
                fill_message(u, code, hi[8 * (size_t)uu + 1], hd[4 * (size_t)uu + 2], *cfg);
                continue;
            }
            u.status = LB_OK;
            u.partial = hi[8 * (size_t)uu + 2];
            u.total_cost = hd[4 * (size_t)uu + 0];
            const int plen = hi[8 * (size_t)uu + 4];
            if (plen < 0 || plen > pstride) return set_err(LB_INTERNAL, "best path length out of range");
            u.path.assign(hpath.begin() + (size_t)pstride * uu, hpath.begin() + (size_t)pstride * uu + plen);
            if (refill) continue;
            const int l = k;
            if (lat) {
                rc = finalize_device(g, desc[l], T[uu], D, cfg->acoustic_scale, cfg->lattice_beam, u.partial, fl,
                                     st, u, n - uu);
                if (rc) return rc;
            }
            if (packs || keep_work) {
                const int Tu = T[uu];
                const UttDesc &d = desc[l];
                u.frame_off.resize(Tu + 2);
                CK(cudaMemcpy(u.frame_off.data(), d.tok_base, sizeof(long long) * (Tu + 2), cudaMemcpyDeviceToHost));
                const int64_t nt = u.frame_off[Tu + 1];
                u.n_tokens = nt;
                u.states.resize(nt);
                u.costs.resize(nt);
                u.pred_arc.resize(nt);
                u.pred_idx.resize(nt);
                CK(cudaMemcpy(u.states.data(), d.tok_state, 4 * nt, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(u.costs.data(), d.tok_cost, 8 * nt, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(u.pred_arc.data(), d.tok_arc, 4 * nt, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(u.pred_idx.data(), d.tok_pred, 4 * nt, cudaMemcpyDeviceToHost));
                for (auto &x : u.pred_idx) x = x >> 1;
                if (packs) {
                    u.packs.resize(nt);
                    CK(cudaMemcpy(u.packs.data(), d.tok_pack, 8 * nt, cudaMemcpyDeviceToHost));
                }
                if (keep_work) {
                    u.block_off.resize(Tu + 2);
                    CK(cudaMemcpy(u.block_off.data(), d.lat_base, sizeof(long long) * (Tu + 2), cudaMemcpyDeviceToHost));
                    const int64_t na = u.block_off[Tu + 1];
                    u.n_lat = na;
                    u.larc.resize(na);
                    u.lfrom.resize(na);
                    u.lto.resize(na);
                    u.lextra.resize(na);
                    CK(cudaMemcpy(u.larc.data(), d.lat_arc, 4 * na, cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(u.lfrom.data(), d.lat_from, 4 * na, cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(u.lto.data(), d.lat_to, 4 * na, cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(u.lextra.data(), d.lat_extra, 8 * na, cudaMemcpyDeviceToHost));
                }
            }
        }
        CK(cudaEventRecord(e3, st));
        CK(cudaEventSynchronize(e3));
        CK(cudaEventElapsedTime(&ms, e2, e3));
        res->t_d2h += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
    if (d_prof) {
        unsigned long long h[24];
        CK(cudaMemcpy(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost));
        for (int k = 0; k < 8; k++) {
            res->phase_ms[k] = h[k] / 1e6;
            res->warp_ms[k] = h[8 + k] / 1e6;
            res->warp_n[k] = (double)h[16 + k];
        }
        cudaFree(d_prof);
    }
    return guard_round_tags(w, st);
}

// Streamed host input for a refilling decode: job k (LPT queue order) is copied
// into slot k % R of a pinned ring by host threads; a lane that finishes job j
// hands its slot back (ring_done[slot] = j + 1, mapped) and the host reuses it
// for job j + R.  Host memory stays bounded (R slots) and the copy overlaps the
// decode instead of preceding it (pinned buffering of the
// log-likelihood H2D).
//  * DMA ring (default): a publisher thread enqueues, in queue order, the H2D
//    copy of slot k into the same slot of a device ring and then a 4-byte copy
//    of k + 1 into a device ready counter (Params::ring_ready), both on one copy
//    stream, so the counter passes k only after job k's rows are in HBM.  The
//    lanes read their rows from HBM, exactly as an HBM-resident decode does.
//  * Zero-copy ring (LB_RING_ZC=1): the ring is mapped and the lanes read the
//    rows over PCIe; the ready counter is mapped and published by the stagers.
int decode_ring(lb_graph *g, int n, const double *const *costs, const int32_t *T, int D, const lb_config *cfg,
                int lanes, lb_result *res) {
    Nvtx range_("lb.decode_ring");
    int tmax = 1;
    for (int i = 0; i < n; i++) tmax = std::max(tmax, (int)T[i]);
    const long long slot_doubles = ((long long)tmax * D + 15) & ~15ll;   // slots start on 128-byte lines
    int R = std::min(n, std::max(2 * lanes, lanes + 8));
    if (const char *e = getenv("LB_RING_SLOTS")) R = std::max(1, std::min(n, atoi(e)));
    const size_t need = (size_t)R * slot_doubles * 8;
    if (need > g->ring_cap) {
        if (g->ring) cudaFreeHost(g->ring);
        g->ring = nullptr;
        g->ring_cap = 0;
        CK(cudaHostAlloc((void **)&g->ring, need, cudaHostAllocMapped));
        g->ring_cap = need;
    }
    if (R + 1 > g->ring_ctl_cap) {
        if (g->ring_ctl) cudaFreeHost(g->ring_ctl);
        g->ring_ctl = nullptr;
        g->ring_ctl_cap = 0;
        CK(cudaHostAlloc((void **)&g->ring_ctl, sizeof(int) * (size_t)(R + 32), cudaHostAllocMapped));
        g->ring_ctl_cap = R + 32;
    }
    const bool dma = !getenv("LB_RING_ZC");
    if (dma) {
        if (need > g->dring_cap) {
            if (g->dring) cudaFree(g->dring);
            g->dring = nullptr;
            g->dring_cap = 0;
            CK(cudaMalloc((void **)&g->dring, need));
            g->dring_cap = need;
        }
        if (!g->dring_ready) CK(cudaMalloc((void **)&g->dring_ready, 128));
        if (n + 1 > g->ring_seq_cap) {
            if (g->ring_seq) cudaFreeHost(g->ring_seq);
            g->ring_seq = nullptr;
            g->ring_seq_cap = 0;
            CK(cudaHostAlloc((void **)&g->ring_seq, sizeof(int) * (size_t)(n + 1), cudaHostAllocDefault));
            g->ring_seq_cap = n + 1;
            for (int k = 0; k <= n; k++) g->ring_seq[k] = k;
        }
        if (!g->copy_stream) CK(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
        CK(cudaMemsetAsync(g->dring_ready, 0, sizeof(int), g->copy_stream));
        CK(cudaStreamSynchronize(g->copy_stream));   // zero before the kernel can read it
    }
    int *h_ready = g->ring_ctl, *h_done = g->ring_ctl + 32;   // ready on its own line
    __atomic_store_n(h_ready, 0, __ATOMIC_SEQ_CST);
    for (int k = 0; k < R; k++) __atomic_store_n(h_done + k, 0, __ATOMIC_SEQ_CST);
    RingDev rd;
    if (dma) {
        rd.ready = g->dring_ready;
        rd.base = g->dring;
    } else {
        CK(cudaHostGetDevicePointer((void **)&rd.ready, h_ready, 0));
        CK(cudaHostGetDevicePointer((void **)&rd.base, g->ring, 0));
    }
    CK(cudaHostGetDevicePointer((void **)&rd.done, h_done, 0));
    rd.slot_doubles = slot_doubles;
    rd.slots = R;
    const std::vector<int32_t> ord = lpt_order(n, T);
    unsigned nth = std::max(1u, std::min(4u, std::thread::hardware_concurrency()));
    if (const char *se = getenv("LB_STAGE_THREADS")) nth = std::max(1, atoi(se));
    nth = std::min<unsigned>(nth, (unsigned)n);
    std::unique_ptr<std::atomic<int>[]> staged(new std::atomic<int>[n]);
    for (int k = 0; k < n; k++) staged[k].store(0);
    std::atomic<int> pub{0};
    std::atomic<bool> abort_flag{false};
    char *ring = reinterpret_cast<char *>(g->ring);
    auto publish = [&]() {   // advance the in-order published count as far as staged jobs allow
        if (dma) return;         // (the publisher thread below does it)
        int r = pub.load(std::memory_order_acquire);
        while (r < n && staged[r].load(std::memory_order_acquire)) {
            if (pub.compare_exchange_weak(r, r + 1, std::memory_order_acq_rel)) {
                int cur = __atomic_load_n(h_ready, __ATOMIC_ACQUIRE);
                while (cur < r + 1 &&
                       !__atomic_compare_exchange_n(h_ready, &cur, r + 1, false, __ATOMIC_RELEASE, __ATOMIC_ACQUIRE)) {
                }
                r = r + 1;
            }
        }
    };
    auto work = [&](unsigned t) {
        for (int k = (int)t; k < n; k += (int)nth) {
            const int slot = k % R;
            if (k >= R) {   // wait for the slot's previous job (k - R) to hand it back
                int spins = 0;
                while (__atomic_load_n(h_done + slot, __ATOMIC_ACQUIRE) < k - R + 1) {
                    if (abort_flag.load(std::memory_order_relaxed)) return;
                    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
                }
            }
            std::memcpy(ring + (size_t)slot * slot_doubles * 8, costs[ord[k]], (size_t)T[ord[k]] * D * 8);
            staged[k].store(1, std::memory_order_release);
            publish();
        }
    };
    // DMA publisher: job k's slot copy, then the counter, in queue order
    std::atomic<int> dma_err{0};
    auto publisher = [&]() {
        cudaSetDevice(g->device);
        for (int k = 0; k < n; k++) {
            int spins = 0;
            while (!staged[k].load(std::memory_order_acquire)) {
                if (abort_flag.load(std::memory_order_relaxed)) return;
                if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(10));
            }
            const size_t off = (size_t)(k % R) * slot_doubles;
            cudaError_t e = cudaMemcpyAsync(g->dring + off, g->ring + off, (size_t)T[ord[k]] * D * 8,
                                            cudaMemcpyHostToDevice, g->copy_stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(g->dring_ready, g->ring_seq + k + 1, sizeof(int), cudaMemcpyHostToDevice,
                                    g->copy_stream);
            if (e != cudaSuccess) {
                // release the lanes (they would wait for job k forever): publish
                // every job from a fresh stream; the call then fails with LB_CUDA
                dma_err.store((int)e);
                cudaStream_t rs = nullptr;
                if (cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking) == cudaSuccess) {
                    cudaMemcpyAsync(g->dring_ready, g->ring_seq + n, sizeof(int), cudaMemcpyHostToDevice, rs);
                    cudaStreamSynchronize(rs);
                    cudaStreamDestroy(rs);
                }
                return;
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; t++) th.emplace_back(work, t);
    if (dma) th.emplace_back(publisher);
    const int rc = decode_impl(g, n, costs, T, D, cfg, g->stream, res, 0.0f, nullptr, &rd);
    // a kernel that ran to the end consumed every job, so the stagers are done;
    // after a failure they may wait on a slot that is never handed back
    abort_flag.store(true);
    for (auto &x : th) x.join();
    if (dma) CK(cudaStreamSynchronize(g->copy_stream));
    res->t_h2d = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rc == LB_OK && dma_err.load()) return set_err(LB_CUDA, cudaGetErrorString((cudaError_t)dma_err.load()));
    return rc;
}

}  // namespace

extern "C" {

// Python repr() of a float (CPython float_repr_style 'short'): the shortest
// round-trip digits; exponent form iff decpt <= -4 or decpt > 16; ".0" added to
// integral fixed-form values.  Used by the lattice text writer so the native
// output is byte-identical to write_lattice_text (lattice.py:605-614).
static void py_repr(double x, std::string &out) {
    if (std::isnan(x)) { out += "nan"; return; }
    if (std::isinf(x)) { out += x < 0 ? "-inf" : "inf"; return; }
    char b[64];
    auto r = std::to_chars(b, b + sizeof b, x, std::chars_format::scientific);
    std::string t(b, r.ptr);
    size_t i = 0;
    if (t[0] == '-') { out += '-'; i = 1; }
    const size_t epos = t.find('e');
    std::string digits;
    for (size_t k = i; k < epos; k++)
        if (t[k] != '.') digits += t[k];
    const int e10 = std::atoi(t.c_str() + epos + 1);
    const int decpt = e10 + 1;
    const int nd = (int)digits.size();
    if (decpt <= -4 || decpt > 16) {
        out += digits[0];
        if (nd > 1) { out += '.'; out.append(digits, 1, std::string::npos); }
        char eb[16];
        snprintf(eb, sizeof eb, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
        out += eb;
    } else if (decpt <= 0) {
        out += "0.";
        out.append((size_t)(-decpt), '0');
        out += digits;
    } else if (decpt >= nd) {
        out += digits;
        out.append((size_t)(decpt - nd), '0');
        out += ".0";
    } else {
        out.append(digits, 0, (size_t)decpt);
        out += '.';
        out.append(digits, (size_t)decpt, std::string::npos);
    }
}

int32_t lb_version(void) { return 1; }

const char *lb_last_error(void) { return g_err.c_str(); }

int32_t lb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int lb_graph_create(int32_t device, int64_t S, int64_t A, int32_t start, const int64_t *off, const int32_t *src,
                    const int32_t *dst, const int32_t *il, const int32_t *ol, const double *w, const double *fin,
                    lb_graph **out) {
    if (!out) return set_err(LB_USAGE, "out is NULL");
    *out = nullptr;
    if (S < 1 || A < 0 || start < 0 || start >= S) return set_err(LB_USAGE, "bad graph dimensions / start state");
    if (S >= (1ll << 30) || A >= (1ll << 32) - 1)
        return set_err(LB_USAGE, "graph too large: at most 2^30 - 1 states and 2^32 - 2 arcs");
    if (off[0] != 0 || off[S] != A) return set_err(LB_USAGE, "arc offsets must start at 0 and end at num_arcs");
    Nvtx range_("lb_graph_create");
    std::unique_ptr<lb_graph> g(new lb_graph());
    g->device = device;
    g->S = S;
    g->A = A;
    g->start = start;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    // Upload the CSR columns as they are and build the device layout on the GPU
    // (lb_graph_build.cuh); raw columns not kept by the replica are freed after.
    cudaStream_t st = g->stream;
    long long *d_off = nullptr;
    int *d_dst = nullptr, *d_il = nullptr;
    double *d_w = nullptr;
    unsigned *d_ecnt = nullptr, *d_emit = nullptr, *d_err = nullptr;
    int *d_maxil = nullptr;
    unsigned long long *d_sum = nullptr;
    void *d_tmp = nullptr;
    unsigned char *d_epsin = nullptr;
    auto cleanup = [&]() {
        cudaFree(d_off); cudaFree(d_dst); cudaFree(d_il); cudaFree(d_w); cudaFree(d_ecnt); cudaFree(d_emit);
        cudaFree(d_err); cudaFree(d_maxil); cudaFree(d_sum); cudaFree(d_tmp); cudaFree(d_epsin);
    };
    struct Guard { std::function<void()> f; ~Guard() { f(); } } guard{cleanup};
    CK(dalloc(&d_off, S + 1));
    CK(dalloc(&d_dst, A));
    CK(dalloc(&d_il, A));
    CK(dalloc(&d_w, A));
    CK(dalloc(&d_ecnt, S + 1));
    CK(dalloc(&d_emit, S));
    CK(dalloc(&d_err, 1));
    CK(dalloc(&d_maxil, 1));
    CK(dalloc(&d_sum, 2));
    CK(dalloc(&g->arcs, A));
    CK(dalloc(&g->src, A));
    CK(dalloc(&g->ol, A));
    CK(dalloc(&g->off, S + 1));
    CK(dalloc(&g->rng, S));
    CK(dalloc(&g->erng, S));
    CK(dalloc(&g->eoff, S + 1));
    CK(dalloc(&g->fin, S));
    CK(cudaMemcpyAsync(d_off, off, 8 * (S + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_dst, dst, 4 * A, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_il, il, 4 * A, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_w, w, 8 * A, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(g->src, src, 4 * A, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(g->ol, ol, 4 * A, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(g->fin, fin, 8 * S, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_err, 0, 4, st));
    CK(cudaMemsetAsync(d_maxil, 0, 4, st));
    const int nb = g->sms * 8;
    gb_state_pass<<<nb, 256, 0, st>>>(d_off, d_il, S, g->off, g->rng, d_ecnt, d_emit, d_err);
    // epsilon CSR offsets, emitting-arc total and max out-degree
    size_t t1 = 0, t2 = 0, t3 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t1, d_ecnt, g->eoff, (int)(S + 1), st));
    CK(cub::DeviceReduce::Sum(nullptr, t2, d_emit, d_sum, (int)S, st));
    CK(cub::DeviceReduce::Max(nullptr, t3, d_emit, d_sum + 1, (int)S, st));
    CK(dalloc((char **)&d_tmp, std::max(t1, std::max(t2, t3))));
    size_t tt = std::max(t1, std::max(t2, t3));
    CK(cub::DeviceScan::ExclusiveSum(d_tmp, tt, d_ecnt, g->eoff, (int)(S + 1), st));
    tt = std::max(t1, std::max(t2, t3));
    CK(cub::DeviceReduce::Sum(d_tmp, tt, d_emit, d_sum, (int)S, st));
    tt = std::max(t1, std::max(t2, t3));
    CK(cub::DeviceReduce::Max(d_tmp, tt, d_emit, d_sum + 1, (int)S, st));
    unsigned hE = 0, herr = 0;
    unsigned long long hsum[2] = {0, 0};
    CK(cudaMemcpyAsync(&hE, g->eoff + S, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hsum, d_sum, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (herr & GB_BAD_OFFSETS) {
        lb_graph_destroy(g.release());
        return set_err(LB_USAGE, "arc offsets must be non-decreasing");
    }
    g->E = hE;
    g->A_emit = (int64_t)hsum[0];
    g->max_edeg = (int64_t)(unsigned)hsum[1];
    CK(dalloc(&g->eps, g->E));
    gb_state_eps<<<nb, 256, 0, st>>>(d_off, d_il, d_dst, d_w, S, g->eoff, g->eps, g->erng);
    CK(dalloc(&d_epsin, S));
    CK(cudaMemsetAsync(d_epsin, 0, S, st));
    gb_eps_in<<<nb, 256, 0, st>>>(d_dst, d_il, A, S, d_epsin);
    gb_arcs<<<nb, 256, 0, st>>>(d_dst, d_il, (const int *)g->ol, d_w, A, S, g->erng, d_epsin, g->arcs, d_err, d_maxil);
    CK(cudaGetLastError());
    int hmaxil = 0;
    CK(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hmaxil, d_maxil, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (herr & (GB_BAD_FIELD | GB_BAD_WEIGHT)) {
        lb_graph_destroy(g.release());
        return set_err(LB_USAGE, (herr & GB_BAD_FIELD) ? "arc field out of range"
                                                       : "arc weight must be finite and >= 0");
    }
    g->max_ilabel = hmaxil;
    g->bytes = A * 16 + A * 8 + (S + 1) * 8 + 2 * S * 8 + g->E * 16 + S * 8;
    *out = g.release();
    return LB_OK;
}

int lb_graph_destroy(lb_graph *g) {
    if (!g) return LB_OK;
    cudaSetDevice(g->device);
    if (g->bexec) cudaGraphExecDestroy(g->bexec);
    g->ws.release();
    g->ws1.release();
    cudaFree(g->arcs);
    cudaFree(g->src);
    cudaFree(g->ol);
    cudaFree(g->off);
    cudaFree(g->rng);
    cudaFree(g->erng);
    cudaFree(g->eoff);
    cudaFree(g->eps);
    cudaFree(g->fin);
    cudaFree(g->d_costs);
    if (g->h_stage) cudaFreeHost(g->h_stage);
    if (g->h_ready) cudaFreeHost(g->h_ready);
    if (g->ring) cudaFreeHost(g->ring);
    if (g->ring_ctl) cudaFreeHost(g->ring_ctl);
    if (g->dring) cudaFree(g->dring);
    if (g->dring_ready) cudaFree(g->dring_ready);
    if (g->ring_seq) cudaFreeHost(g->ring_seq);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    if (g->stream) cudaStreamDestroy(g->stream);
    if (g->stream2) cudaStreamDestroy(g->stream2);
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_join) cudaEventDestroy(g->ev_join);
    delete g;
    return LB_OK;
}

int64_t lb_graph_device_bytes(const lb_graph *g) { return g ? g->bytes : 0; }

int lb_decode_batch(const lb_graph *gc, int32_t n, const double *const *costs, const int32_t *T, int32_t D,
                    const lb_config *cfg, lb_result **out) {
    Nvtx range_("lb_decode_batch");
    lb_graph *g = const_cast<lb_graph *>(gc);
    if (!g || !out) return set_err(LB_USAGE, "graph/out is NULL");
    *out = nullptr;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (n < 0) return set_err(LB_USAGE, "n_utts must be >= 0");
    if (D < 1) return set_err(LB_USAGE, "num_labels must be >= 1");
    if (g->max_ilabel > D) return set_err(LB_USAGE, "graph uses an input label beyond the cost matrix columns");
    size_t total = 0;
    std::vector<size_t> off(n + 1, 0);
    for (int i = 0; i < n; i++) {   // each matrix starts on a 128-byte line (see CF below)
        if (T[i] < 1) return set_err(LB_USAGE, "every cost matrix needs T >= 1");
        total += ((size_t)T[i] * D + 15) & ~(size_t)15;
        off[i + 1] = total;
    }
    std::lock_guard<std::mutex> lock(g->mu);
    CK(cudaSetDevice(g->device));
    std::unique_ptr<lb_result> res(new lb_result());
    // 1-best decodes in the lane kernel read each frame's row once per lane: the
    // kernel reads the mapped staging buffer directly (zero-copy).  Lattice decodes
    // re-read rows in the prune pass, and the batched mode gathers acoustic costs
    // per candidate: those copy the rows to HBM.
    bool batched_mode = true;
    int lane_c = 1;
    choose_mode(g, n, D, cfg, batched_mode, lane_c);
    const bool lane_mode = !batched_mode;
    // Small batches (a few wide lanes) copy to HBM instead: a lane reading its
    // rows over PCIe without the row prefetch stalls on every frame (one C2
    // utterance on a 16-CTA lane: 19.3 ms zero-copy vs 16.6 ms with the copy;
    // C5 28.3 vs 26.1 ms; tools/c2_timing.py).
    // Batches larger than one set of lanes refill lanes from the job queue; their
    // rows stream through a bounded pinned ring instead of a whole-batch stage.
    const int lanes_est = cfg->lanes > 0 ? cfg->lanes : std::max(1, g->sms / std::max(lane_c, 1));
    const char *zc_min = getenv("LB_ZC_MIN");
    const bool zero_copy = lane_mode && !cfg->want_lattice && (size_t)D * 8 <= ACROW_SMEM_MAX &&
                           (n >= (zc_min ? atoi(zc_min) : 16) || n > lanes_est) && !getenv("LB_E2E_COPY");
    if (zero_copy && n > lanes_est && !cfg->collect_frame_packs && !getenv("LB_NO_RING") &&
        !getenv("LB_NO_REFILL")) {
        rc = decode_ring(g, n, costs, T, D, cfg, lanes_est, res.get());
        if (rc) return rc;
        *out = res.release();
        return LB_OK;
    }
    if (total > g->h_stage_cap) {
        if (g->h_stage) cudaFreeHost(g->h_stage);
        g->h_stage = nullptr;
        CK(cudaHostAlloc((void **)&g->h_stage, std::max<size_t>(total, 1) * 8, cudaHostAllocMapped));
        g->h_stage_cap = total;
    }
    // Stage the caller's matrices into pinned, device-mapped memory with all host
    // threads (one memcpy thread is ~10 GB/s).  Zero-copy decodes stage
    // progressively: frame chunks of every utterance in order, each published
    // through a mapped counter the lanes wait on (Params::ready), so the copy
    // overlaps the decode instead of preceding it.
    const size_t bytes = total * 8;
    const bool progressive = zero_copy && !getenv("LB_NO_PROGRESSIVE") && n > 0;
    // A blocking copy uses every host thread.  A progressive one needs only to
    // stay ahead of the decode (~11 GB/s at C4), and at full width it competes
    // with the lanes' zero-copy reads for host memory: 4 threads measured best
    // (C4 e2e 391k vs 368k frames/s with 16; tools/e2e_time.py).
    unsigned nth = std::max(1u, std::min(progressive ? 4u : 32u, std::thread::hardware_concurrency()));
    if (const char *se = getenv("LB_STAGE_THREADS")) nth = std::max(1, atoi(se));
    if (bytes < ((size_t)8 << 20)) nth = 1;
    int tmax = 1;
    for (int i = 0; i < n; i++) tmax = std::max(tmax, (int)T[i]);
    // Frames per published chunk.  16 rows of D doubles are 128*D bytes, so with
    // line-aligned matrices no 128-byte line spans two chunks: a line the kernel
    // pulls into L2 never holds bytes of a chunk that is not yet published.
    const int CF = 16;
    const int nchunks = progressive ? (tmax + CF - 1) / CF : 1;
    // pieces of chunk c: (destination byte offset, source pointer, bytes)
    struct Piece { size_t dst; const char *src; size_t len; };
    std::vector<std::vector<Piece>> chunks(nchunks);
    std::vector<size_t> chunk_bytes(nchunks, 0);
    for (int c = 0; c < nchunks; c++) {
        for (int i = 0; i < n; i++) {
            const int f0 = progressive ? c * CF : 0, f1 = progressive ? std::min<int>(T[i], (c + 1) * CF) : T[i];
            if (f1 <= f0) continue;
            const size_t len = (size_t)(f1 - f0) * D * 8;
            chunks[c].push_back({(off[i] + (size_t)f0 * D) * 8,
                                 reinterpret_cast<const char *>(costs[i]) + (size_t)f0 * D * 8, len});
            chunk_bytes[c] += len;
        }
    }
    if (progressive && !g->h_ready) {
        CK(cudaHostAlloc((void **)&g->h_ready, 64, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void **)&g->d_ready, g->h_ready, 0));
    }
    if (progressive) __atomic_store_n(g->h_ready, 0, __ATOMIC_SEQ_CST);
    std::vector<std::atomic<int>> done(nth);
    for (auto &d : done) d.store(0);
    char *stage = reinterpret_cast<char *>(g->h_stage);
    int *h_ready = g->h_ready;
    auto work = [&, stage, h_ready](unsigned w) {
        for (int c = 0; c < nchunks; c++) {
            // copy bytes [lo, hi) of chunk c's concatenated pieces
            const size_t lo = chunk_bytes[c] * w / nth, hi = chunk_bytes[c] * (w + 1) / nth;
            size_t base = 0;
            for (const Piece &pc : chunks[c]) {
                const size_t a = std::max(lo, base), b = std::min(hi, base + pc.len);
                if (a < b) std::memcpy(stage + pc.dst + (a - base), pc.src + (a - base), b - a);
                base += pc.len;
                if (base >= hi) break;
            }
            done[w].store(c + 1, std::memory_order_seq_cst);   // seq_cst: two finishers must not both miss each other
            if (progressive) {   // publish the chunks every worker has finished
                int m = c + 1;
                for (unsigned q = 0; q < nth; q++) m = std::min(m, done[q].load(std::memory_order_seq_cst));
                const int frames = m >= nchunks ? tmax : m * CF;
                int cur = __atomic_load_n(h_ready, __ATOMIC_ACQUIRE);
                while (cur < frames &&
                       !__atomic_compare_exchange_n(h_ready, &cur, frames, false, __ATOMIC_RELEASE, __ATOMIC_ACQUIRE)) {
                }
            }
        }
    };
    const auto t_stage = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    std::vector<const double *> dptr(n);
    float h2d = 0.0f;
    // joins the staging threads on every path out of this function (an unjoined
    // std::thread would terminate the process)
    struct Joiner {
        std::vector<std::thread> &v;
        ~Joiner() {
            for (auto &t : v)
                if (t.joinable()) t.join();
        }
    } joiner{th};
    if (progressive) {
        double *dev = nullptr;
        CK(cudaHostGetDevicePointer((void **)&dev, g->h_stage, 0));   // before any thread starts
        for (int i = 0; i < n; i++) dptr[i] = dev + off[i];
        for (unsigned w = 0; w < nth; w++) th.emplace_back(work, w);
        rc = decode_impl(g, n, dptr.data(), T, D, cfg, g->stream, res.get(), 0.0f, g->d_ready);
        for (auto &t : th) t.join();   // the kernel finished, so every chunk was published
        res->t_h2d = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_stage).count();
        if (rc) return rc;
        *out = res.release();
        return LB_OK;
    }
    for (unsigned w = 1; w < nth; w++) th.emplace_back(work, w);
    work(0);
    for (auto &t : th) t.join();
    h2d = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_stage).count();
    if (zero_copy) {
        double *dev = nullptr;
        CK(cudaHostGetDevicePointer((void **)&dev, g->h_stage, 0));
        for (int i = 0; i < n; i++) dptr[i] = dev + off[i];
    } else {
        if (total > g->d_costs_cap) {
            cudaFree(g->d_costs);
            g->d_costs = nullptr;
            CK(dalloc(&g->d_costs, total));
            g->d_costs_cap = total;
        }
        cudaEvent_t h0, h1;
        CK(cudaEventCreate(&h0));
        CK(cudaEventCreate(&h1));
        CK(cudaEventRecord(h0, g->stream));
        CK(cudaMemcpyAsync(g->d_costs, g->h_stage, total * 8, cudaMemcpyHostToDevice, g->stream));
        CK(cudaEventRecord(h1, g->stream));
        CK(cudaEventSynchronize(h1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, h0, h1));
        h2d += ms;
        cudaEventDestroy(h0);
        cudaEventDestroy(h1);
        for (int i = 0; i < n; i++) dptr[i] = g->d_costs + off[i];
    }
    rc = decode_impl(g, n, dptr.data(), T, D, cfg, g->stream, res.get(), h2d);
    if (rc) return rc;
    *out = res.release();
    return LB_OK;
}

// Longest-processing-time-first split of utterances over shards (devices):
// utterances in descending length (ties: input order) each go to the shard with
// the fewest frames so far (ties: lowest shard).  Deterministic.
int lb_shard_lpt(int32_t n, const int32_t *T, int32_t n_shards, int32_t *shard_of) {
    if (n < 0 || n_shards < 1 || (n > 0 && (!T || !shard_of))) return set_err(LB_USAGE, "bad shard arguments");
    std::vector<int32_t> ord(n);
    for (int i = 0; i < n; i++) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return T[a] > T[b]; });
    std::vector<long long> load(n_shards, 0);
    for (int32_t i : ord) {
        int best = 0;
        for (int s = 1; s < n_shards; s++)
            if (load[s] < load[best]) best = s;
        shard_of[i] = best;
        load[best] += std::max(T[i], 0);
    }
    return LB_OK;
}

// decode_batch over several graph replicas (one per device):
// LPT shards, one host thread per replica (each an independent lb_decode_batch on
// its device), results merged back into input order.  No collective: utterances
// share nothing (decoder.py:644-672).
int lb_decode_batch_multi(const lb_graph *const *graphs, int32_t n_graphs, int32_t n, const double *const *costs,
                          const int32_t *T, int32_t D, const lb_config *cfg, lb_result **out) {
    if (!graphs || n_graphs < 1 || !out) return set_err(LB_USAGE, "graphs/out is NULL");
    *out = nullptr;
    for (int k = 0; k < n_graphs; k++)
        if (!graphs[k]) return set_err(LB_USAGE, "graph replica is NULL");
    if (n < 0) return set_err(LB_USAGE, "n_utts must be >= 0");
    if (n_graphs == 1) return lb_decode_batch(graphs[0], n, costs, T, D, cfg, out);
    std::vector<int32_t> shard(n);
    if (int rc = lb_shard_lpt(n, T, n_graphs, shard.data())) return rc;
    std::vector<std::vector<int32_t>> idx(n_graphs);
    for (int i = 0; i < n; i++) idx[shard[i]].push_back(i);
    std::vector<lb_result *> part(n_graphs, nullptr);
    std::vector<int> rcs(n_graphs, LB_OK);
    std::vector<std::string> msgs(n_graphs);
    auto run = [&](int k) {
        Nvtx rs("lb.shard");
        const auto &ix = idx[k];
        std::vector<const double *> c(ix.size());
        std::vector<int32_t> t(ix.size());
        for (size_t j = 0; j < ix.size(); j++) {
            c[j] = costs[ix[j]];
            t[j] = T[ix[j]];
        }
        rcs[k] = lb_decode_batch(graphs[k], (int32_t)ix.size(), c.data(), t.data(), D, cfg, &part[k]);
        if (rcs[k]) msgs[k] = g_err;   // the message is thread-local
    };
    {
        std::vector<std::thread> th;
        for (int k = 1; k < n_graphs; k++) th.emplace_back(run, k);
        run(0);
        for (auto &x : th) x.join();
    }
    std::unique_ptr<lb_result> res(new lb_result());
    res->utts.resize(n);
    int first = LB_OK;
    std::string first_msg;
    for (int k = 0; k < n_graphs; k++) {
        if (rcs[k] && first == LB_OK) {
            first = rcs[k];
            first_msg = msgs[k];
        }
        if (!part[k]) continue;
        lb_result &p = *part[k];
        for (size_t j = 0; j < idx[k].size(); j++) res->utts[idx[k][j]] = std::move(p.utts[j]);
        // the replicas run concurrently: the call's device time is the slowest one's
        res->t_decode = std::max(res->t_decode, p.t_decode);
        res->t_prune = std::max(res->t_prune, p.t_prune);
        res->t_h2d = std::max(res->t_h2d, p.t_h2d);
        res->t_d2h = std::max(res->t_d2h, p.t_d2h);
        res->launches += p.launches;
        delete part[k];
    }
    if (first != LB_OK) return set_err(first, first_msg);
    *out = res.release();
    return LB_OK;
}

int lb_decode_batch_device(const lb_graph *gc, int32_t n, const double *const *dev_costs, const int32_t *T,
                           int32_t D, const lb_config *cfg, void *stream, lb_result **out) {
    lb_graph *g = const_cast<lb_graph *>(gc);
    if (!g || !out) return set_err(LB_USAGE, "graph/out is NULL");
    *out = nullptr;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (n < 0 || D < 1) return set_err(LB_USAGE, "bad batch dimensions");
    if (g->max_ilabel > D) return set_err(LB_USAGE, "graph uses an input label beyond the cost matrix columns");
    for (int i = 0; i < n; i++)
        if (T[i] < 1) return set_err(LB_USAGE, "every cost matrix needs T >= 1");
    std::lock_guard<std::mutex> lock(g->mu);
    CK(cudaSetDevice(g->device));
    std::unique_ptr<lb_result> res(new lb_result());
    cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
    rc = decode_impl(g, n, dev_costs, T, D, cfg, st, res.get(), 0.0f);
    if (rc) return rc;
    *out = res.release();
    return LB_OK;
}

int lb_decode_batch_device_f32(const lb_graph *gc, int32_t n, const float *const *dev_costs, const int32_t *T,
                               int32_t D, const lb_config *cfg, void *stream, lb_result **out) {
    lb_graph *g = const_cast<lb_graph *>(gc);
    if (!g || !out) return set_err(LB_USAGE, "graph/out is NULL");
    *out = nullptr;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (n < 0 || D < 1) return set_err(LB_USAGE, "bad batch dimensions");
    if (g->max_ilabel > D) return set_err(LB_USAGE, "graph uses an input label beyond the cost matrix columns");
    for (int i = 0; i < n; i++)
        if (T[i] < 1) return set_err(LB_USAGE, "every cost matrix needs T >= 1");
    std::lock_guard<std::mutex> lock(g->mu);
    CK(cudaSetDevice(g->device));
    std::unique_ptr<lb_result> res(new lb_result());
    cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
    bool batched = true;
    int C = 1;
    choose_mode(g, n, D, cfg, batched, C);
    // Refilling 1-best lanes widen each row as they load it into shared memory;
    // every other mode reads f64 rows, so the batch is widened into HBM first.
    // Widening f32 -> f64 is exact: the result is the decode of the widened matrix.
    const bool fused = !batched && !cfg->want_lattice && !cfg->collect_frame_packs &&
                       (size_t)D * 8 <= ACROW_SMEM_MAX && !getenv("LB_NO_REFILL") && !getenv("LB_F32_WIDEN");
    if (fused) {
        rc = decode_impl(g, n, reinterpret_cast<const double *const *>(dev_costs), T, D, cfg, st, res.get(), 0.0f,
                         nullptr, nullptr, true);
    } else {
        std::vector<size_t> off(n + 1, 0);
        for (int i = 0; i < n; i++) off[i + 1] = off[i] + (((size_t)T[i] * D + 15) & ~(size_t)15);
        const size_t total = off[n];
        if (total > g->d_costs_cap) {
            cudaFree(g->d_costs);
            g->d_costs = nullptr;
            g->d_costs_cap = 0;
            CK(dalloc(&g->d_costs, total));
            g->d_costs_cap = total;
        }
        std::vector<WidenJob> wj(n);
        std::vector<const double *> dptr(n);
        for (int i = 0; i < n; i++) {
            wj[i].src = dev_costs[i];
            wj[i].dst = g->d_costs + off[i];
            wj[i].n = (long long)T[i] * D;
            dptr[i] = g->d_costs + off[i];
        }
        WidenJob *d_wj = nullptr;
        CK(dalloc(&d_wj, (size_t)std::max(n, 1)));
        struct F { WidenJob *p; ~F() { cudaFree(p); } } fw{d_wj};
        CK(cudaMemcpyAsync(d_wj, wj.data(), sizeof(WidenJob) * (size_t)n, cudaMemcpyHostToDevice, st));
        if (n > 0) {
            widen_f32_kernel<<<dim3(64, (unsigned)n), 256, 0, st>>>(d_wj);
            CK(cudaGetLastError());
        }
        rc = decode_impl(g, n, dptr.data(), T, D, cfg, st, res.get(), 0.0f);
    }
    if (rc) return rc;
    *out = res.release();
    return LB_OK;
}

int lb_result_count(const lb_result *r, int32_t *n) {
    if (!r || !n) return set_err(LB_USAGE, "NULL argument");
    *n = (int32_t)r->utts.size();
    return LB_OK;
}

#define UTT_OR_FAIL                                                                     \
    if (!r || utt < 0 || utt >= (int32_t)r->utts.size()) return set_err(LB_USAGE, "bad result/utterance"); \
    const UttHost &u = r->utts[utt];

// Every utterance's scalar results in one call (the per-utterance getters cost a
// foreign call each, which dominates the host side of a 4096-utterance batch).
int lb_result_bulk(const lb_result *r, int32_t *status, double *total_cost, int32_t *partial, int64_t *path_off,
                   int64_t *counters) {
    if (!r) return set_err(LB_USAGE, "NULL result");
    const size_t n = r->utts.size();
    if (path_off) path_off[0] = 0;
    for (size_t u = 0; u < n; u++) {
        const UttHost &x = r->utts[u];
        if (status) status[u] = x.status;
        if (total_cost) total_cost[u] = x.total_cost;
        if (partial) partial[u] = x.partial;
        if (path_off) path_off[u + 1] = path_off[u] + (int64_t)x.path.size();
        if (counters) std::memcpy(counters + 8 * u, x.counters, sizeof(x.counters));
    }
    return LB_OK;
}

int lb_result_paths(const lb_result *r, int32_t *arcs) {
    if (!r || !arcs) return set_err(LB_USAGE, "NULL argument");
    size_t o = 0;
    for (const UttHost &x : r->utts) {
        if (!x.path.empty()) std::memcpy(arcs + o, x.path.data(), 4 * x.path.size());
        o += x.path.size();
    }
    return LB_OK;
}

int lb_result_status(const lb_result *r, int32_t utt, int32_t *status, char *msg, int32_t msg_len, char *bound,
                     int32_t bound_len) {
    UTT_OR_FAIL
    if (status) *status = u.status;
    if (msg && msg_len > 0) snprintf(msg, msg_len, "%s", u.msg.c_str());
    if (bound && bound_len > 0) snprintf(bound, bound_len, "%s", u.bound.c_str());
    return LB_OK;
}

int lb_result_best(const lb_result *r, int32_t utt, double *total_cost, int32_t *partial, int64_t *path_len,
                   int64_t *num_tokens, int64_t *num_lat) {
    UTT_OR_FAIL
    if (total_cost) *total_cost = u.total_cost;
    if (partial) *partial = u.partial;
    if (path_len) *path_len = (int64_t)u.path.size();
    if (num_tokens) *num_tokens = u.n_tokens;
    if (num_lat) *num_lat = u.n_lat;
    return LB_OK;
}

int lb_result_path(const lb_result *r, int32_t utt, int32_t *arcs) {
    UTT_OR_FAIL
    if (!u.path.empty()) std::memcpy(arcs, u.path.data(), 4 * u.path.size());
    return LB_OK;
}

int lb_result_tokens(const lb_result *r, int32_t utt, int64_t *frame_off, int32_t *states, double *costs,
                     int32_t *pred_arc, int32_t *pred_idx, uint64_t *packs) {
    UTT_OR_FAIL
    if (u.frame_off.empty()) return set_err(LB_USAGE, "token lists were not collected (collect_frame_packs/want_lattice)");
    std::memcpy(frame_off, u.frame_off.data(), 8 * u.frame_off.size());
    const size_t n = (size_t)u.n_tokens;
    if (states) std::memcpy(states, u.states.data(), 4 * n);
    if (costs) std::memcpy(costs, u.costs.data(), 8 * n);
    if (pred_arc) std::memcpy(pred_arc, u.pred_arc.data(), 4 * n);
    if (pred_idx) std::memcpy(pred_idx, u.pred_idx.data(), 4 * n);
    if (packs && !u.packs.empty()) std::memcpy(packs, u.packs.data(), 8 * n);
    return LB_OK;
}

int lb_result_lattice(const lb_result *r, int32_t utt, int64_t *block_off, int32_t *arc, int32_t *from_idx,
                      int32_t *to_idx, double *extra) {
    UTT_OR_FAIL
    if (u.block_off.empty()) return set_err(LB_USAGE, "lattice was not requested");
    std::memcpy(block_off, u.block_off.data(), 8 * u.block_off.size());
    const size_t n = (size_t)u.n_lat;
    std::memcpy(arc, u.larc.data(), 4 * n);
    std::memcpy(from_idx, u.lfrom.data(), 4 * n);
    std::memcpy(to_idx, u.lto.data(), 4 * n);
    std::memcpy(extra, u.lextra.data(), 8 * n);
    return LB_OK;
}

int lb_result_final_lattice(const lb_result *r, int32_t utt, int64_t *num_nodes, int64_t *start, int64_t *n_final,
                            int64_t *n_arcs) {
    UTT_OR_FAIL
    if (!u.has_final) return set_err(LB_USAGE, "lattice was not requested");
    if (num_nodes) *num_nodes = (int64_t)u.fl_nodes.size();
    if (start) *start = u.fl_start;
    if (n_final) *n_final = (int64_t)u.fl_final_ids.size();
    if (n_arcs) *n_arcs = (int64_t)u.fl_from.size();
    return LB_OK;
}

int lb_result_final_arrays(const lb_result *r, int32_t utt, uint64_t *node_keys, int64_t *final_ids,
                           double *final_costs, int32_t *from, int32_t *to, int32_t *ilabel, int32_t *olabel,
                           double *graph_cost, double *acoustic_cost) {
    UTT_OR_FAIL
    if (!u.has_final) return set_err(LB_USAGE, "lattice was not requested");
    const size_t m = u.fl_from.size(), nf = u.fl_final_ids.size();
    if (node_keys) std::memcpy(node_keys, u.fl_nodes.data(), 8 * u.fl_nodes.size());
    if (final_ids) std::memcpy(final_ids, u.fl_final_ids.data(), 8 * nf);
    if (final_costs) std::memcpy(final_costs, u.fl_final_costs.data(), 8 * nf);
    if (from) std::memcpy(from, u.fl_from.data(), 4 * m);
    if (to) std::memcpy(to, u.fl_to.data(), 4 * m);
    if (ilabel) std::memcpy(ilabel, u.fl_il.data(), 4 * m);
    if (olabel) std::memcpy(olabel, u.fl_ol.data(), 4 * m);
    if (graph_cost) std::memcpy(graph_cost, u.fl_g.data(), 8 * m);
    if (acoustic_cost) std::memcpy(acoustic_cost, u.fl_ac.data(), 8 * m);
    return LB_OK;
}

// Ask for transparent huge pages on a fresh destination array before it is
// first touched: the widening below is page-fault bound on new numpy memory
// (4 KB faults), and 2 MB pages cut the fault count 512x.  Only the 2 MB-aligned
// interior is advised; a no-op where THP is off (LB_NO_THP disables it).
static void hugepage_hint(void *p, size_t bytes) {
    static const bool off = getenv("LB_NO_THP") != nullptr;
    if (off || !p || bytes < ((size_t)4 << 20)) return;
    const uintptr_t a = ((uintptr_t)p + ((1u << 21) - 1)) & ~(uintptr_t)((1u << 21) - 1);
    const uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)((1u << 21) - 1);
    if (e > a) madvise((void *)a, e - a, MADV_HUGEPAGE);
}

int lb_result_final_arrays64(const lb_result *r, int32_t utt, int64_t *node_frame, int64_t *node_idx,
                             int64_t *final_ids, double *final_costs, int64_t *from, int64_t *to, int64_t *ilabel,
                             int64_t *olabel, double *graph_cost, double *acoustic_cost) {
    UTT_OR_FAIL
    if (!u.has_final) return set_err(LB_USAGE, "lattice was not requested");
    const size_t m = u.fl_from.size(), nn = u.fl_nodes.size(), nf = u.fl_final_ids.size();
    if (final_ids) std::memcpy(final_ids, u.fl_final_ids.data(), 8 * nf);
    if (final_costs) std::memcpy(final_costs, u.fl_final_costs.data(), 8 * nf);
    // widen from the pinned arena on all host threads (the copies are page-fault
    // bound on fresh numpy pages, which parallelise)
    for (int64_t *q : {from, to, ilabel, olabel}) hugepage_hint(q, 8 * m);
    hugepage_hint(graph_cost, 8 * m);
    hugepage_hint(acoustic_cost, 8 * m);
    hugepage_hint(node_frame, 8 * nn);
    hugepage_hint(node_idx, 8 * nn);
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (m + nn < ((size_t)1 << 18)) nth = 1;
    auto work = [&](unsigned w) {
        const size_t a0 = m * w / nth, a1 = m * (w + 1) / nth;
        for (size_t k = a0; k < a1; k++) {
            if (from) from[k] = u.fl_from[k];
            if (to) to[k] = u.fl_to[k];
            if (ilabel) ilabel[k] = u.fl_il[k];
            if (olabel) olabel[k] = u.fl_ol[k];
        }
        if (graph_cost) std::memcpy(graph_cost + a0, u.fl_g.data() + a0, 8 * (a1 - a0));
        if (acoustic_cost) std::memcpy(acoustic_cost + a0, u.fl_ac.data() + a0, 8 * (a1 - a0));
        const size_t b0 = nn * w / nth, b1 = nn * (w + 1) / nth;
        for (size_t k = b0; k < b1; k++) {
            if (node_frame) node_frame[k] = (int64_t)(u.fl_nodes[k] >> 32);
            if (node_idx) node_idx[k] = (int64_t)(u.fl_nodes[k] & 0xFFFFFFFFull);
        }
    };
    std::vector<std::thread> th;
    for (unsigned w = 1; w < nth; w++) th.emplace_back(work, w);
    work(0);
    for (auto &t : th) t.join();
    return LB_OK;
}

int lb_result_counters(const lb_result *r, int32_t utt, int64_t *c) {
    UTT_OR_FAIL
    std::memcpy(c, u.counters, sizeof(u.counters));
    return LB_OK;
}

int lb_result_timing(const lb_result *r, float *decode_ms, float *prune_ms, float *h2d_ms, float *d2h_ms,
                     int32_t *launches) {
    if (!r) return set_err(LB_USAGE, "NULL result");
    if (decode_ms) *decode_ms = r->t_decode;
    if (prune_ms) *prune_ms = r->t_prune;
    if (h2d_ms) *h2d_ms = r->t_h2d;
    if (d2h_ms) *d2h_ms = r->t_d2h;
    if (launches) *launches = r->launches;
    return LB_OK;
}

int lb_result_phases(const lb_result *r, double *ms8) {
    if (!r || !ms8) return set_err(LB_USAGE, "NULL argument");
    std::memcpy(ms8, r->phase_ms, sizeof(r->phase_ms));
    return LB_OK;
}

int lb_result_warp_phases(const lb_result *r, double *busy_ms8, double *samples8) {
    if (!r || !busy_ms8 || !samples8) return set_err(LB_USAGE, "NULL argument");
    std::memcpy(busy_ms8, r->warp_ms, sizeof(r->warp_ms));
    std::memcpy(samples8, r->warp_n, sizeof(r->warp_n));
    return LB_OK;
}

void lb_result_free(lb_result *r) { delete r; }

int lb_oracle_wer_batch(int32_t device, int32_t n, const lb_lattice_view *lats, int64_t *errors) {
    if (n < 0 || (n > 0 && (!lats || !errors))) return set_err(LB_USAGE, "bad arguments");
    if (n == 0) return LB_OK;
    CK(cudaSetDevice(device));
    // host: frame node ranges and from-frame arc ranges, packed per job
    std::vector<WerJob> jobs(n);
    std::vector<std::vector<int>> packs(n);
    size_t total_best = 0;
    for (int i = 0; i < n; i++) {
        const lb_lattice_view &L = lats[i];
        if (L.n_ref < 1) return set_err(LB_USAGE, "reference word sequence is empty");
        if (L.num_nodes < 1 || L.start < 0 || L.start >= L.num_nodes)
            return set_err(LB_USAGE, "bad lattice dimensions");
        const int64_t N = L.num_nodes, M = L.n_arcs;
        // arcs in from-node order (stable), as scoring.py:80-83 sweeps them
        std::vector<int64_t> ord(M);
        for (int64_t k = 0; k < M; k++) ord[k] = k;
        bool sorted = true;
        for (int64_t k = 1; k < M && sorted; k++) sorted = L.from[k] >= L.from[k - 1];
        if (!sorted) std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return L.from[a] < L.from[b]; });
        for (int64_t k = 0; k < M; k++) {
            if (L.from[k] < 0 || L.from[k] >= N || L.to[k] < 0 || L.to[k] >= N)
                return set_err(LB_USAGE, "lattice arc endpoint out of range");
        }
        for (int64_t q = 0; q < L.n_final; q++)
            if (L.final_ids[q] < 0 || L.final_ids[q] >= N) return set_err(LB_USAGE, "final node id out of range");
        // frame-ordered DP when node ids are in frame order and every arc stays in
        // its frame or steps to the next one (all decoder lattices); otherwise the
        // whole lattice is one "frame" and the in-frame fixpoint is a plain
        // Bellman-Ford over all arcs -- same distances, more rounds.
        bool framed = L.node_frame != nullptr;
        for (int64_t v = 0; framed && v < N; v++)
            framed = L.node_frame[v] >= 0 && (v == 0 || L.node_frame[v] >= L.node_frame[v - 1]);
        for (int64_t k = 0; framed && k < M; k++) {
            const int64_t df = L.node_frame[L.to[k]] - L.node_frame[L.from[k]];
            framed = df == 0 || df == 1;
        }
        int F = 1;
        std::vector<int> nb, ab;
        if (framed) {
            F = (int)L.node_frame[N - 1] + 1;
            nb.assign(F + 1, 0);
            ab.assign(F + 1, 0);
            for (int64_t v = 0, f = 0; f <= F; f++) {
                while (v < N && L.node_frame[v] < f) v++;
                nb[f] = (int)v;
            }
            for (int64_t f = 0, k = 0; f <= F; f++) {
                while (k < M && L.from[ord[k]] < nb[f]) k++;
                ab[f] = (int)k;
            }
        } else {
            nb = {0, (int)N};
            ab = {0, (int)M};
        }
        std::vector<int> afrom(M), ato(M), aol(M);
        for (int64_t k = 0; k < M; k++) {
            afrom[k] = (int)L.from[ord[k]];
            ato[k] = (int)L.to[ord[k]];
            aol[k] = (int)L.olabel[ord[k]];
        }
        std::vector<int> &pk = packs[i];
        auto put = [&](const auto &src, int64_t cnt) {
            size_t o = pk.size();
            for (int64_t k = 0; k < cnt; k++) pk.push_back((int)src[k]);
            return o;
        };
        const size_t o_from = put(afrom.data(), M), o_to = put(ato.data(), M), o_ol = put(aol.data(), M);
        const size_t o_nb = put(nb.data(), F + 1), o_ab = put(ab.data(), F + 1);
        const size_t o_fin = put(L.final_ids, L.n_final), o_ref = put(L.ref, L.n_ref);
        WerJob &J = jobs[i];
        J.num_nodes = (int)N;
        J.start = (int)L.start;
        J.n_final = (int)L.n_final;
        J.F = F;
        J.r = (int)L.n_ref;
        // offsets for now; made device pointers after upload
        J.from = (const int *)o_from; J.to = (const int *)o_to; J.ol = (const int *)o_ol;
        J.nb = (const int *)o_nb; J.ab = (const int *)o_ab; J.finals = (const int *)o_fin; J.ref = (const int *)o_ref;
        J.best = (int *)total_best;
        total_best += (size_t)N * (L.n_ref + 1);
    }
    size_t total_pack = 0;
    for (auto &pk : packs) total_pack += pk.size();
    int *d_pack = nullptr, *d_best = nullptr;
    long long *d_out = nullptr;
    WerJob *d_jobs = nullptr;
    CK(dalloc(&d_pack, total_pack));
    CK(dalloc(&d_best, total_best));
    CK(dalloc(&d_out, n));
    CK(dalloc(&d_jobs, n));
    size_t base = 0;
    for (int i = 0; i < n; i++) {
        CK(cudaMemcpy(d_pack + base, packs[i].data(), 4 * packs[i].size(), cudaMemcpyHostToDevice));
        WerJob &J = jobs[i];
        auto rebase = [&](const int *o) { return (const int *)(d_pack + base + (size_t)o); };
        J.from = rebase(J.from); J.to = rebase(J.to); J.ol = rebase(J.ol); J.nb = rebase(J.nb);
        J.ab = rebase(J.ab); J.finals = rebase(J.finals); J.ref = rebase(J.ref);
        J.best = d_best + (size_t)J.best;
        J.out = d_out + i;
        base += packs[i].size();
    }
    CK(cudaMemcpy(d_jobs, jobs.data(), sizeof(WerJob) * n, cudaMemcpyHostToDevice));
    oracle_wer_kernel<<<n, 1024>>>(d_jobs, n);
    CK(cudaGetLastError());
    std::vector<long long> out(n);
    CK(cudaMemcpy(out.data(), d_out, 8 * n, cudaMemcpyDeviceToHost));
    cudaFree(d_pack);
    cudaFree(d_best);
    cudaFree(d_out);
    cudaFree(d_jobs);
    for (int i = 0; i < n; i++) errors[i] = out[i];
    return LB_OK;
}

int64_t lb_lattice_text(int64_t num_nodes, int64_t start, int64_t n_final, const int64_t *final_ids,
                        const double *final_costs, int64_t n_arcs, const int64_t *from, const int64_t *to,
                        const int64_t *ilabel, const int64_t *olabel, const double *graph_cost,
                        const double *acoustic_cost, char *buf, int64_t cap) {
    std::string head = "NODES " + std::to_string(num_nodes) + " ARCS " + std::to_string(n_arcs) + " START " +
                       std::to_string(start) + "\n";
    for (int64_t i = 0; i < n_final; i++) {
        head += "F " + std::to_string(final_ids[i]) + " ";
        py_repr(final_costs[i], head);
        head += "\n";
    }
    unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n_arcs < 65536) nth = 1;
    std::vector<std::string> part(nth);
    auto work = [&](unsigned w) {
        const int64_t lo = n_arcs * w / nth, hi = n_arcs * (w + 1) / nth;
        std::string &o = part[w];
        o.reserve((size_t)(hi - lo) * 48);
        char ib[96];
        for (int64_t k = lo; k < hi; k++) {
            const int len = snprintf(ib, sizeof ib, "A %lld %lld %lld %lld ", (long long)from[k], (long long)to[k],
                                     (long long)ilabel[k], (long long)olabel[k]);
            o.append(ib, (size_t)len);
            py_repr(graph_cost[k], o);
            o += ' ';
            py_repr(acoustic_cost[k], o);
            o += '\n';
        }
    };
    std::vector<std::thread> th;
    for (unsigned w = 1; w < nth; w++) th.emplace_back(work, w);
    work(0);
    for (auto &t : th) t.join();
    int64_t total = (int64_t)head.size();
    for (auto &p : part) total += (int64_t)p.size();
    if (buf && cap >= total) {
        char *q = buf;
        std::memcpy(q, head.data(), head.size());
        q += head.size();
        for (auto &p : part) {
            std::memcpy(q, p.data(), p.size());
            q += p.size();
        }
    }
    return total;
}

// finalize_lattice (lattice.py:537-598) on the device for a host work lattice:
// the caller passes its LIVE arcs with node keys (frame << 32) | token index;
// nodes are the sorted unique keys (dense ids), arcs come back in the canonical
// np.lexsort((ac, g, ol, il, to, from)) order, final nodes are the last frame's
// nodes with a finite final cost.  The result is read with lb_result_final_*.
int lb_finalize_lattice(int32_t device, int64_t n, const uint64_t *from_key, const uint64_t *to_key,
                        const int32_t *ilabel, const int32_t *olabel, const double *graph_cost,
                        const double *acoustic_cost, int64_t start_idx, int32_t last_frame, int32_t partial,
                        int64_t n_final_costs, const double *final_costs, lb_result **out) {
    if (!out) return set_err(LB_USAGE, "out is NULL");
    *out = nullptr;
    if (n < 0 || last_frame < 0) return set_err(LB_USAGE, "bad lattice dimensions");
    if (n >= (1ll << 31)) return set_err(LB_USAGE, "lattice too large");
    std::unique_ptr<lb_result> res(new lb_result());
    res->utts.resize(1);
    UttHost &u = res->utts[0];
    u.status = LB_OK;
    u.has_final = true;
    if (n == 0) {
        u.status = LB_DECODE_FAILURE;
        u.msg = "no lattice arcs survived pruning";
        *out = res.release();
        return LB_OK;
    }
    CK(cudaSetDevice(device));
    cudaStream_t st = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<void *> bufs;
    struct Free {
        std::vector<void *> &b;
        cudaStream_t s;
        ~Free() {
            for (void *p : b) cudaFree(p);
            cudaStreamDestroy(s);
        }
    } fr{bufs, st};
    auto A = [&](auto **dp, size_t cnt) -> cudaError_t {
        cudaError_t e = dalloc(dp, cnt);
        if (e == cudaSuccess) bufs.push_back((void *)*dp);
        return e;
    };
    const size_t m = (size_t)n;
    unsigned long long *fk, *tk, *nodes0, *nodes1, *k64a, *k64b, *count;
    unsigned *il, *ol, *fid, *tid, *k32a, *k32b;
    double *gc, *ac, *o_g, *o_ac, *fcs, *fc_in;
    int *perm0, *perm1, *o_from, *o_to, *o_il, *o_ol, *n_unique;
    long long *fids;
    CK(A(&fk, m)); CK(A(&tk, m)); CK(A(&nodes0, 2 * m)); CK(A(&nodes1, 2 * m)); CK(A(&k64a, m)); CK(A(&k64b, m));
    CK(A(&count, 1)); CK(A(&il, m)); CK(A(&ol, m)); CK(A(&fid, m)); CK(A(&tid, m)); CK(A(&k32a, m)); CK(A(&k32b, m));
    CK(A(&gc, m)); CK(A(&ac, m)); CK(A(&o_g, m)); CK(A(&o_ac, m)); CK(A(&fcs, 2 * m));
    CK(A(&fc_in, (size_t)std::max<int64_t>(n_final_costs, 1)));
    CK(A(&perm0, m)); CK(A(&perm1, m)); CK(A(&o_from, m)); CK(A(&o_to, m)); CK(A(&o_il, m)); CK(A(&o_ol, m));
    CK(A(&n_unique, 1)); CK(A(&fids, 2 * m));
    CK(cudaMemcpyAsync(fk, from_key, 8 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(tk, to_key, 8 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(nodes0, from_key, 8 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(nodes0 + m, to_key, 8 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(il, ilabel, 4 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ol, olabel, 4 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(gc, graph_cost, 8 * m, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ac, acoustic_cost, 8 * m, cudaMemcpyHostToDevice, st));
    if (n_final_costs > 0 && final_costs)
        CK(cudaMemcpyAsync(fc_in, final_costs, 8 * (size_t)n_final_costs, cudaMemcpyHostToDevice, st));
    // CUB scratch for the largest sort / unique
    size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, nodes0, nodes1, (int)(2 * m), 0, 64, st));
    CK(cub::DeviceSelect::Unique(nullptr, t2, nodes1, nodes0, n_unique, (int)(2 * m), st));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t3, k64a, k64b, perm0, perm1, (int)m, 0, 64, st));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t4, k32a, k32b, perm0, perm1, (int)m, 0, 32, st));
    size_t tcap = std::max(std::max(t1, t2), std::max(t3, t4));
    void *temp = nullptr;
    CK(A((char **)&temp, tcap));
    const int nblk = 148 * 4;
    CK(cub::DeviceRadixSort::SortKeys(temp, tcap, nodes0, nodes1, (int)(2 * m), 0, 64, st));
    tcap = std::max(std::max(t1, t2), std::max(t3, t4));
    CK(cub::DeviceSelect::Unique(temp, tcap, nodes1, nodes0, n_unique, (int)(2 * m), st));
    int nn = 0;
    CK(cudaMemcpyAsync(&nn, n_unique, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fl_node_ids<<<nblk, 256, 0, st>>>(fk, tk, (long long)m, nodes0, nn, fid, tid);
    fl_iota<<<nblk, 256, 0, st>>>(perm0, (long long)m);
    int *pa = perm0, *pb = perm1;
    for (int pass = 0; pass < 6; pass++) {   // np.lexsort((ac, g, ol, il, to, from)): last key primary
        tcap = std::max(std::max(t1, t2), std::max(t3, t4));
        if (pass < 2) {
            fl_gather_u64<<<nblk, 256, 0, st>>>(pass == 0 ? ac : gc, pa, (long long)m, k64a);
            CK(cub::DeviceRadixSort::SortPairs(temp, tcap, k64a, k64b, pa, pb, (int)m, 0, 64, st));
        } else {
            const unsigned *srcp = pass == 2 ? ol : pass == 3 ? il : pass == 4 ? tid : fid;
            fl_gather_u32<<<nblk, 256, 0, st>>>(srcp, pa, (long long)m, k32a);
            CK(cub::DeviceRadixSort::SortPairs(temp, tcap, k32a, k32b, pa, pb, (int)m, 0, 32, st));
        }
        std::swap(pa, pb);
    }
    fl_emit<<<nblk, 256, 0, st>>>(pa, (long long)m, fid, tid, il, ol, gc, ac, o_from, o_to, o_il, o_ol, o_g, o_ac);
    CK(cudaMemsetAsync(count, 0, 8, st));
    fl_finals_given<<<nblk, 256, 0, st>>>(nodes0, nn, last_frame, fc_in, n_final_costs, partial, fids, fcs, count);
    CK(cudaGetLastError());
    unsigned long long nf = 0;
    CK(cudaMemcpyAsync(&nf, count, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // host copies (a private arena owned by the result)
    auto arena = std::make_shared<HostArena>();
    const size_t bytes = 8 * (size_t)nn + 32 * m + 8 * 256;
    CK(cudaHostAlloc((void **)&arena->p, bytes, cudaHostAllocDefault));
    arena->cap = bytes;
    auto take = [&](auto &span, size_t cnt) {
        using T = typename std::remove_reference<decltype(*span.p)>::type;
        span.p = reinterpret_cast<T *>(arena->p + arena->used);
        span.n = cnt;
        arena->used += (cnt * sizeof(T) + 255) & ~(size_t)255;
    };
    take(u.fl_nodes, (size_t)nn);
    take(u.fl_from, m); take(u.fl_to, m); take(u.fl_il, m); take(u.fl_ol, m); take(u.fl_g, m); take(u.fl_ac, m);
    u.fl_arena = arena;
    CK(cudaMemcpyAsync(u.fl_nodes.data(), nodes0, 8 * (size_t)nn, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_from.data(), o_from, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_to.data(), o_to, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_il.data(), o_il, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_ol.data(), o_ol, 4 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_g.data(), o_g, 8 * m, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(u.fl_ac.data(), o_ac, 8 * m, cudaMemcpyDeviceToHost, st));
    std::vector<int64_t> ids(nf);
    std::vector<double> fcv(nf);
    CK(cudaMemcpyAsync(ids.data(), fids, 8 * nf, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fcv.data(), fcs, 8 * nf, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<size_t> ord(nf);
    for (size_t i = 0; i < nf; i++) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
    u.fl_final_ids.resize(nf);
    u.fl_final_costs.resize(nf);
    for (size_t i = 0; i < nf; i++) {
        u.fl_final_ids[i] = ids[ord[i]];
        u.fl_final_costs[i] = fcv[ord[i]];
    }
    const uint64_t sk = (uint64_t)start_idx;
    auto it = std::lower_bound(u.fl_nodes.begin(), u.fl_nodes.end(), sk);
    if (start_idx < 0 || it == u.fl_nodes.end() || *it != sk) {
        u.status = LB_DECODE_FAILURE;
        u.msg = "surviving arcs do not connect to the start node";
    } else {
        u.fl_start = it - u.fl_nodes.begin();
        if (nf == 0) {
            u.status = LB_DECODE_FAILURE;
            u.msg = "no terminal node survived pruning";
        }
    }
    *out = res.release();
    return LB_OK;
}

// prune_lattice (lattice.py:365-431) on the device for a host work lattice.
int lb_prune_lattice(int32_t device, int32_t t, const int64_t *frame_off, const double *fwd, const int64_t *block_off,
                     const int32_t *from_idx, const int32_t *to_idx, const uint8_t *emitting, const double *graph_cost,
                     const double *acoustic_cost, const double *terminus, double lattice_beam, uint8_t *status,
                     double *extra, double *node_extra) {
    if (t < 0 || !frame_off || !block_off) return set_err(LB_USAGE, "bad prune arguments");
    if (!(lattice_beam >= 0)) return set_err(LB_USAGE, "lattice_beam must be >= 0");
    const int64_t ntok = frame_off[t + 1], narc = block_off[t + 1];
    if (ntok < 1 || frame_off[t + 1] - frame_off[t] < 1) return set_err(LB_USAGE, "frontier is empty");
    for (int f = 0; f <= t; f++)
        if (frame_off[f + 1] < frame_off[f] || block_off[f + 1] < block_off[f])
            return set_err(LB_USAGE, "frame / block offsets must be non-decreasing");
    for (int64_t k = 0; k < narc; k++) {   // arc endpoints inside their frames
        int b = (int)(std::upper_bound(block_off, block_off + t + 2, k) - block_off) - 1;
        const int fb = emitting[k] ? b - 1 : b;
        if (fb < 0 || from_idx[k] < 0 || from_idx[k] >= frame_off[fb + 1] - frame_off[fb] || to_idx[k] < 0 ||
            to_idx[k] >= frame_off[b + 1] - frame_off[b])
            return set_err(LB_USAGE, "lattice arc endpoint outside its frame");
    }
    CK(cudaSetDevice(device));
    std::vector<void *> bufs;
    struct Free { std::vector<void *> &b; ~Free() { for (void *p : b) cudaFree(p); } } fr{bufs};
    auto up = [&](auto **dp, const auto *hp, size_t cnt) -> cudaError_t {
        cudaError_t e = dalloc(dp, cnt);
        if (e != cudaSuccess) return e;
        bufs.push_back((void *)*dp);
        return hp ? cudaMemcpy(*dp, hp, sizeof(**dp) * cnt, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    PruneOp op;
    std::memset(&op, 0, sizeof(op));
    long long *d_tb, *d_lb;
    double *d_fwd, *d_g, *d_ac, *d_term, *d_extra, *d_ne_out, *d_tmp;
    int *d_from, *d_to, *d_err;
    unsigned char *d_emit, *d_status;
    unsigned long long *d_ne;
    const size_t nt = (size_t)ntok, na = (size_t)std::max<int64_t>(narc, 1);
    const int64_t nterm = frame_off[t + 1] - frame_off[t];
    CK(up(&d_tb, (const long long *)frame_off, (size_t)t + 2));
    CK(up(&d_lb, (const long long *)block_off, (size_t)t + 2));
    CK(up(&d_fwd, fwd, nt));
    CK(up(&d_from, (const int *)from_idx, (size_t)narc));
    CK(up(&d_to, (const int *)to_idx, (size_t)narc));
    CK(up(&d_emit, (const unsigned char *)emitting, (size_t)narc));
    CK(up(&d_g, graph_cost, (size_t)narc));
    CK(up(&d_ac, acoustic_cost, (size_t)narc));
    CK(up(&d_term, terminus, (size_t)nterm));
    CK(up(&d_status, (const unsigned char *)status, (size_t)narc));
    CK(up(&d_extra, extra, (size_t)narc));
    CK(up(&d_ne_out, (const double *)nullptr, nt));
    CK(up(&d_tmp, (const double *)nullptr, na));
    CK(up(&d_ne, (const unsigned long long *)nullptr, nt));
    CK(up(&d_err, (const int *)nullptr, 1));
    CK(cudaMemset(d_err, 0, 4));
    op.t = t;
    op.tok_base = d_tb;
    op.fwd = d_fwd;
    op.lat_base = d_lb;
    op.from = d_from;
    op.to = d_to;
    op.emit = d_emit;
    op.g = d_g;
    op.ac = d_ac;
    op.terminus = d_term;
    op.status = d_status;
    op.extra = d_extra;
    op.node_extra = d_ne_out;
    op.tmp = d_tmp;
    op.ne = d_ne;
    op.err_out = d_err;
    op.beam = lattice_beam;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaLaunchConfig_t lc = {};
    const unsigned pc = (unsigned)std::max(1, std::min(8, sms));
    lc.gridDim = dim3(pc);
    lc.blockDim = dim3(1024);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, prune_op_kernel, op));
    CK(cudaGetLastError());
    int herr = 0;
    CK(cudaMemcpy(&herr, d_err, 4, cudaMemcpyDeviceToHost));
    if (herr) {
        char buf[128];
        snprintf(buf, sizeof buf, "epsilon extra-cost fixpoint did not settle within frame %d", herr - 1);
        return set_err(LB_INTERNAL, buf);
    }
    CK(cudaMemcpy(status, d_status, (size_t)narc, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(extra, d_extra, 8 * (size_t)narc, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(node_extra, d_ne_out, 8 * nt, cudaMemcpyDeviceToHost));
    return LB_OK;
}

static int expand_common(lb_graph *g, const int32_t *states, const double *costs, int64_t n, const double *acrow,
                         int32_t D, double beam, double cutoff, int mode, int32_t *out_states, double *out_costs,
                         int64_t *n_out, double *cutoff_out) {
    if (!g || !states || !costs || n < 1) return set_err(LB_USAGE, "frontier is empty");
    std::lock_guard<std::mutex> lock(g->mu);
    CK(cudaSetDevice(g->device));
    // the frontier itself sits in the winner / round-0 lists (expand_nonemitting)
    const int64_t ccap = std::max<int64_t>(std::min<int64_t>(g->A_emit, n * g->max_edeg) + 25 * CAND_CHUNK, n);
    int rc = ensure_workspace(g, g->ws1, 1, 1, ccap, n + g->S, 0, 16, 1, false, false, false);
    if (rc) return rc;
    Workspace &w = g->ws1;
    cudaStream_t st = g->stream;
    double *d_row = nullptr;
    if (mode == 0) {
        CK(dalloc(&d_row, D));
        CK(cudaMemcpyAsync(d_row, acrow, 8 * (size_t)D, cudaMemcpyHostToDevice, st));
    }
    if (int rj = ensure_jobs(w, 1, 16)) return rj;
    UttDesc d = slot_desc(w, 0, d_row, 1);
    d.path = w.j_path;
    d.out_i = w.j_out_i;
    d.out_d = w.j_out_d;
    d.out_c = w.j_out_c;
    std::vector<unsigned> hs(states, states + n);
    CK(cudaMemcpyAsync(d.tok_state, hs.data(), 4 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d.tok_cost, costs, 8 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d.out_i, 0, 8 * sizeof(int), st));
    LaneWs L;
    CK(cudaMemcpyAsync(&L, w.d_lanes, sizeof(LaneWs), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.beam = beam;
    p.scale = 1.0;
    p.max_tokens = 1ll << 40;
    p.D = D;
    p.acrow_smem = 0;
    p.ready = nullptr;
    const int esm = (int)lane_dyn_smem(768, 1, false);
    CK(cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, esm));
    expand_kernel<<<1, 768, esm, st>>>(g->dev(), p, L, d, (int)n, mode, cutoff);
    CK(cudaGetLastError());
    int oi[8];
    double od[4];
    CK(cudaMemcpyAsync(oi, d.out_i, sizeof(oi), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(od, d.out_d, sizeof(od), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (d_row) cudaFree(d_row);
    if (oi[0]) return set_err(LB_INTERNAL, "epsilon relaxation failed to settle within the state count");
    const int m = oi[4];
    std::vector<unsigned> os(m);
    CK(cudaMemcpy(os.data(), d.tok_state + n, 4 * (size_t)m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_costs, d.tok_cost + n, 8 * (size_t)m, cudaMemcpyDeviceToHost));
    for (int k = 0; k < m; k++) out_states[k] = (int32_t)os[k];
    *n_out = m;
    if (int rg = guard_round_tags(w, st)) return rg;
    if (cutoff_out) *cutoff_out = od[0];
    return LB_OK;
}

int lb_expand_emitting(const lb_graph *g, const int32_t *states, const double *costs, int64_t n, const double *acrow,
                       int32_t D, double beam, int32_t *out_states, double *out_costs, int64_t *n_out,
                       double *cutoff) {
    if (!(std::isfinite(beam) && beam > 0)) return set_err(LB_USAGE, "beam must be a positive finite number");
    return expand_common(const_cast<lb_graph *>(g), states, costs, n, acrow, D, beam, 0.0, 0, out_states, out_costs,
                         n_out, cutoff);
}

int lb_expand_nonemitting(const lb_graph *g, const int32_t *states, const double *costs, int64_t n, double cutoff,
                          int32_t *out_states, double *out_costs, int64_t *n_out) {
    return expand_common(const_cast<lb_graph *>(g), states, costs, n, nullptr, 1, 1.0, cutoff, 1, out_states,
                         out_costs, n_out, nullptr);
}

}  // extern "C"
