// lb_device.cuh — device-side data structures and primitives of the sm_100a decoder.
//
// Bit-exactness contract with the reference (`latbeam`):
//   * candidate cost   (tok + w) + ac, f64, no FMA (kernels.py:97-105); every f64
//     op below goes through __dadd_rn/__dsub_rn/__dmul_rn and the library is
//     built with -fmad=false, so nvcc cannot contract or reassociate;
//   * pack word        (enc32(float32 cost) << 32) | arc id (packing.py:37-61);
//   * recombination    one 64-bit atomicMin per candidate (decoder.py:189-205).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lbk {

constexpr unsigned long long SENT = 0xFFFFFFFFFFFFFFFFull;
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int NBINS = 256;              // max-active histogram bins
constexpr double CONVERGE_TOL = 1e-9;   // lattice.py:36
constexpr double MAX_ACTIVE_BEAM_DELTA = 0.5;   // Kaldi's beam_delta

// ---- error codes written per utterance (host turns them into messages) ----
enum : int {
    E_OK = 0,
    E_DEAD_NO_CAND = 1,      // DecodeFailure: no emitting candidates
    E_DEAD_NO_TOKENS = 2,    // DecodeFailure: no tokens survived
    E_CAP_TOKENS = 3,        // CapacityError --max-tokens-per-frame
    E_CAP_ARENA = 4,         // CapacityError --token-arena
    E_CAP_LATTICE = 5,       // CapacityError --max-lattice-arcs
    E_CAP_PATH = 6,          // CapacityError (path buffer)
    E_INT_EPS_ROUNDS = 7,    // InternalInvariantError: epsilon rounds > S+1
    E_INT_EPS_PRED = 8,      // InternalInvariantError: eps winner's source kept no token
    E_INT_INIT = 9,          // InternalInvariantError: initial token found at frame f
    E_INT_BACKTRACE = 10,    // InternalInvariantError: backtrace exceeded its step bound
    E_INT_PRUNE_EPS = 11,    // InternalInvariantError: eps extra-cost fixpoint
    E_CAP_CAND = 12,         // CapacityError: candidate buffer (sized by construction; never expected)
};

// Graph replica in HBM.  Arc record = 16 B {dst, ilabel, weight};
// bit 31 of the ilabel word flags "dst owns epsilon out-arcs" (ilabels are
// int32 >= 0, so the bit is free) so the emitting pass knows, for free, which
// winners must enter the epsilon closure.  Epsilon arcs additionally get a
// per-state CSR of 16 B {dst, arc id, weight} records so the closure reads one
// record per epsilon arc.
constexpr unsigned EPS_FLAG = 0x80000000u;
// arc record ilabel word / candidate state word: the destination has no incoming
// epsilon arc, so no epsilon offer can change its word after emit (graphs of
// < 2^30 states; lb_graph_create)
constexpr unsigned NOEPSIN_FLAG = 0x40000000u;
constexpr unsigned STATE_FLAGS = EPS_FLAG | NOEPSIN_FLAG;
struct GraphDev {
    const int4 *arcs;
    const unsigned *src;
    const unsigned *ol;
    const unsigned *off;    // [S+1]
    const uint2 *rng;       // [S] {first arc, end arc}: one 8-byte request per token
    const unsigned *eoff;   // [S+1] epsilon CSR offsets
    const uint2 *erng;      // [S] {first, end} epsilon record of a state (one 8-byte request)
    const int4 *eps;        // epsilon records {dst, arc, w_lo, w_hi}
    const double *fin;      // final cost, +inf = non-final
    int S;
    int start;
    int has_eps;
    int _pad;
};

__device__ __forceinline__ unsigned arc_il(int y) { return (unsigned)y & ~STATE_FLAGS; }

// Per-state record of a lane: everything a touched state needs in ONE 32-byte
// sector, laid out so each phase touches it with as few scattered accesses as
// possible (the decode is bound by scattered L2 accesses per SM):
//   [0,16)  cost, pred, tokidx  -- a winner writes all three in ONE 16 B store
//   [16,24) pack                -- the 64-bit (cost, arc) word, SENT = untouched
//   [24,32) minsnap             -- min epsilon-source snapshot (lattice rule A.5)
// `pred` = (prev token index << 1) | 1 for an emitting winner, source state << 1
// for an epsilon winner; `tokidx` = index in the newest frame's token list.
struct __align__(32) StateRec {
    double cost;
    int pred;
    int tokidx;
    unsigned long long pack;
    double minsnap;
};


// ---- per-state (lane-private, reused frame to frame) accesses: L2 policy ----
// The record/epsilon arrays are accessed with an L2 evict_last cache policy so
// the streamed candidate and token arrays (evict-first) do not push the hot
// state records out of L2 (C4: +3 %; LB_NO_L2HINT builds without it).
#ifndef LB_NO_L2HINT
#define LB_L2HINT 1
#endif
// the secondary per-state arrays (token index, epsilon winners / records, round
// tags) take the same evict-last hint unless LB_SEC_NOHINT (an experiment knob)
#if defined(LB_L2HINT) && !defined(LB_SEC_NOHINT)
#define LB_SECHINT 1
#endif
#ifdef LB_L2HINT
__device__ __forceinline__ unsigned long long l2_pol() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#endif

__device__ __forceinline__ unsigned long long rld_u64(const unsigned long long *a) {
    unsigned long long v;
#ifdef LB_L2HINT
    asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(l2_pol()));
#else
    v = __ldcg(a);
#endif
    return v;
}
__device__ __forceinline__ double rld_f64(const double *a) {
    return __longlong_as_double((long long)rld_u64(reinterpret_cast<const unsigned long long *>(a)));
}
__device__ __forceinline__ int rld_i32(const int *a) {
    int v;
#ifdef LB_SECHINT
    asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(l2_pol()));
#else
    v = __ldcg(a);
#endif
    return v;
}
__device__ __forceinline__ void rst_u64(unsigned long long *a, unsigned long long v) {
#ifdef LB_L2HINT
    asm volatile("st.global.cg.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(l2_pol()) : "memory");
#else
    __stcg(a, v);
#endif
}
__device__ __forceinline__ void rst_f64(double *a, double v) {
    rst_u64(reinterpret_cast<unsigned long long *>(a), (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ ulonglong2 rld_u128(const void *a) {
    ulonglong2 v;
#ifdef LB_SECHINT
    asm volatile("ld.global.cg.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(a), "l"(l2_pol()));
#else
    v = __ldcg(reinterpret_cast<const ulonglong2 *>(a));
#endif
    return v;
}
__device__ __forceinline__ void rst_u128(void *a, ulonglong2 v) {
#ifdef LB_SECHINT
    asm volatile("st.global.cg.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(a), "l"(v.x), "l"(v.y), "l"(l2_pol()) : "memory");
#else
    __stcg(reinterpret_cast<ulonglong2 *>(a), v);
#endif
}

// Read-only graph records (shared by every lane).  LB_GRAPH_HINT: L2 evict_last.
__device__ __forceinline__ int4 gld4(const int4 *a) {
#if defined(LB_GRAPH_HINT) && defined(LB_L2HINT)
    int4 v;
    asm("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(l2_pol()));
    return v;
#else
    return __ldg(a);
#endif
}
__device__ __forceinline__ uint2 gld2(const uint2 *a) {
#if defined(LB_GRAPH_HINT) && defined(LB_L2HINT)
    uint2 v;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(l2_pol()));
    return v;
#else
    return __ldg(a);
#endif
}

// A winner's {cost, pred, tokidx = -1} in one 16-byte store (the stale token
// index of an older frame is dead once the frame's emit barrier has passed).
__device__ __forceinline__ void store_winner(StateRec *r, double cost, int pred) {
    const unsigned long long hi = (unsigned long long)(unsigned)pred | 0xFFFFFFFF00000000ull;
    rst_u128(r, make_ulonglong2((unsigned long long)__double_as_longlong(cost), hi));
}
// The whole record in one 32-byte store.
__device__ __forceinline__ void store_rec32(StateRec *r, double cost, int pred, int tokidx,
                                            unsigned long long pack, double minsnap) {
    const unsigned long long x1 = (unsigned long long)(unsigned)pred | ((unsigned long long)(unsigned)tokidx << 32);
#ifdef LB_L2HINT
    asm volatile("st.global.cg.L2::cache_hint.v4.u64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(r),
                 "l"((unsigned long long)__double_as_longlong(cost)), "l"(x1), "l"(pack),
                 "l"((unsigned long long)__double_as_longlong(minsnap)), "l"(l2_pol())
                 : "memory");
#else
    asm volatile("st.global.cg.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(r),
                 "l"((unsigned long long)__double_as_longlong(cost)), "l"(x1), "l"(pack),
                 "l"((unsigned long long)__double_as_longlong(minsnap))
                 : "memory");
#endif
}

// Round-local epsilon winner of a state: the min improving offer's word and the
// f64 cost of that same offer, updated together by a 128-bit CAS.  Idle value:
// all ones (word SENT).
struct __align__(16) EpsWin {
    unsigned long long word;
    unsigned long long cost_bits;
};

// Per-lane scratch.  O(S) arrays are allocated once and reset
// O(touched) per frame.  Lists marked [C] have one S-sized segment per CTA of
// the lane (CTA-local append counters in shared memory, no DSMEM traffic).
// Candidate buffer cache policy: L2-normal stores and loads.  winners() reads
// each 32-entry batch once and then drops its lines from L2 with
// discard.global.L2 (LB_CAND_DISCARD, the default), so the buffer lives and dies
// in L2 without a DRAM write-back (C4 539k -> 555k frames/s,
// profiles/r02_ab_discard.txt; evict-first stores without the discard were the
// round-1 policy, LB_CAND_CS).
#ifdef LB_CAND_CS
#define CAND_ST __stcs
#define CAND_LD __ldcs
#else
#define CAND_ST __stcg
#define CAND_LD __ldcg
#endif
#if !defined(LB_NO_CAND_DISCARD) && !defined(LB_CAND_CS)
#define LB_CAND_DISCARD 1
#endif

// Epsilon-improved state: its final f64 cost and predecessor (source state << 1).
struct __align__(16) ERec {
    double cost;
    int pred;
    int _pad;
};

// Per-lane scratch.  The batched mode keeps one 32-byte StateRec per state
// (`rec`); the persistent lanes keep only what the hot phases touch per state
// -- the 8-byte recombination word `pk` and the 4-byte token index -- and carry
// every winner's cost / predecessor / arc in compact, coalesced per-frame lists
// (`touched` + `tcost` / `tpred` / `tarc`), so 64 lanes' hot per-state data fit
// in L2.  Epsilon-improved states (few) keep theirs in `erec`.
struct LaneWs {
    StateRec *rec;             // [S] batched mode only
    EpsWin *rpk;               // [2][S] epsilon round winners by round parity
    unsigned *tag;             // [S] epsilon round tag
    unsigned *touched;         // batched: [C][S] states touched; lanes: [C][ccap] emitting winners
    unsigned *fr;              // [2][C][S] epsilon frontier by round parity
    unsigned *fix;             // [C][S] tokens whose predecessor is an epsilon source state
    int4 *cand;                // [C][ccap] emitting candidates {dst|flag, arc, cost_lo, cost_hi}
    int *candi;                // [C][ccap] source token index of each candidate
    long long ccap;            // candidate capacity per CTA
    unsigned *round_ctr;       // persistent per-lane round counter
    int S;
    int C;
    // persistent lanes only
    unsigned long long *pk;    // [S] recombination word (cost key << 32 | arc), SENT = untouched
    int *tokidx;               // [S] index of the state's token in the newest frame's list
    ERec *erec;                // [S] epsilon-improved states' cost / predecessor
    double *msnap;             // [S] min epsilon-source snapshot (lattice rule A.5), +inf idle
    double *tcost;             // [C][ccap] winner cost of touched[k]
    int *tpred;                // [C][ccap] winner predecessor ((token << 1) | 1)
    unsigned *tarc;            // [C][ccap] winner arc
    double *f0cost;            // [C][ccap] round-0 epsilon frontier costs (seeds)
    unsigned *etouched;        // [C][S] states first reached by an epsilon offer this frame
};

// One utterance slot of a wave.
struct UttDesc {
    const double *costs;    // T x D f64 (device)
    int T;
    int path_cap;
    long long tok_cap;
    long long lat_cap;
    unsigned *tok_state;
    double *tok_cost;
    int *tok_arc;           // winning arc (-1 = initial token)
    int *tok_pred;          // (pred index << 1) | emitting
    unsigned long long *tok_pack;
    long long *tok_base;    // [T+2]
    int *lat_arc, *lat_from, *lat_to;
    double *lat_extra;
    long long *lat_base;    // [T+2]
    double *node_extra;     // [tok_cap]
    unsigned long long *ne_enc;
    double *tmp;            // [lat_cap]
    int *path;
    int *out_i;             // status, err_frame, partial, best_idx, path_len, n_frames_done
    double *out_d;          // total_cost, best_total (for prune), err_aux
    long long *out_c;       // counters[8]
};

// One utterance of a decode call: its cost matrix, length and output slots
// (per job, so lanes that refill from the job queue keep every job's result).
struct UttJob {
    const double *costs;    // T x D f64 (device or mapped host)
    int T;
    int _pad;
    int *path;              // [path_cap] best path arcs
    int *out_i;             // [8] status, err_frame, partial, best_idx, path_len, n_frames_done
    double *out_d;          // [4] total_cost, best_total, err_aux
    long long *out_c;       // [8] counters
};

struct Params {
    double beam, lattice_beam, scale;
    long long max_active, max_tokens;
    int D;
    int want_lattice;
    int collect_packs;
    int acrow_smem;
    unsigned long long *prof;   // optional per-phase ns accumulators (LB_PHASE_PROFILE=1)
    int costs_f32;              // job cost matrices are f32 (widened exactly to f64 at the row load)
    int row_pf;                 // two row buffers: the next frame's row is prefetched (Lane::row_async)
    int _pad3;
    const int *ready;           // progressive host staging (mapped): rows of frames < *ready are
                                // in place for every utterance; nullptr = all rows ready
    // Streaming host staging for refilling lanes (mapped pinned ring of
    // ring_slots slots; job j, in queue order, lives in slot j % ring_slots):
    // the host publishes *ring_ready = jobs staged so far, in order; a lane
    // marks ring_done[slot] = j + 1 once job j's rows are no longer needed.
    const int *ring_ready;      // nullptr = no ring (costs per job)
    int *ring_done;
    const double *ring_base;
    long long ring_slot_doubles;
    int ring_slots;
    int _pad2;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- bit helpers ----
__device__ __forceinline__ unsigned long long pack_word(double c, unsigned a) {
    unsigned u = __float_as_uint(__double2float_rn(c));
    unsigned e = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)e << 32) | a;
}
__device__ __forceinline__ unsigned long long enc64(double c) {
    unsigned long long u = (unsigned long long)__double_as_longlong(c);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dec64(unsigned long long e) {
    unsigned long long u = (e >> 63) ? (e ^ 0x8000000000000000ull) : ~e;
    return __longlong_as_double((long long)u);
}
// One 32-byte request for a whole state record (sm_100 256-bit LDG, L2 only).
struct RecView {
    double cost;
    int pred, tokidx;
    unsigned long long pack;
    double minsnap;
};
__device__ __forceinline__ RecView load_rec32(const StateRec *r) {
    unsigned long long x0, x1, x2, x3;
#ifdef LB_L2HINT
    asm volatile("ld.global.cg.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(r), "l"(l2_pol()));
#else
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(r));
#endif
    RecView v;
    v.cost = __longlong_as_double((long long)x0);
    v.pred = (int)(unsigned)(x1 & 0xFFFFFFFFull);
    v.tokidx = (int)(unsigned)(x1 >> 32);
    v.pack = x2;
    v.minsnap = __longlong_as_double((long long)x3);
    return v;
}

// 128-bit compare-and-swap (sm_90+): returns the previous value.
__device__ __forceinline__ ulonglong2 cas128(EpsWin *p, ulonglong2 cmp, ulonglong2 val) {
    ulonglong2 old;
    asm volatile(
        "{\n\t.reg .b128 c, v, d;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
        : "memory");
    return old;
}

// Keep the smaller (word, cost) pair: CAS loop from the idle value.  Words of one
// round are unique (each epsilon arc is offered at most once per round).
__device__ __forceinline__ void epswin_min(EpsWin *p, unsigned long long word, double cost) {
    ulonglong2 cur = make_ulonglong2(~0ull, ~0ull);
    const ulonglong2 val = make_ulonglong2(word, (unsigned long long)__double_as_longlong(cost));
    for (;;) {
        const ulonglong2 prev = cas128(p, cur, val);
        if (prev.x == cur.x && prev.y == cur.y) return;
        if (prev.x <= word) return;
        cur = prev;
    }
}

// The same, also telling whether this offer was the round's FIRST improving one
// for the state (its CAS replaced the idle value): the caller then lists the
// state in the next frontier, exactly once per round.
__device__ __forceinline__ bool epswin_min_first(EpsWin *p, unsigned long long word, double cost) {
    ulonglong2 cur = make_ulonglong2(~0ull, ~0ull);
    const ulonglong2 val = make_ulonglong2(word, (unsigned long long)__double_as_longlong(cost));
    bool first = true;
    for (;;) {
        const ulonglong2 prev = cas128(p, cur, val);
        if (prev.x == cur.x && prev.y == cur.y) return first;
        if (prev.x <= word) return false;
        cur = prev;
        first = false;
    }
}

// Global-space atomics with their results (explicit .global: a generic 64-bit
// atomicMin would carry a shared-memory CAS fallback path).
__device__ __forceinline__ unsigned long long atom_min_u64(unsigned long long *a, unsigned long long v) {
    unsigned long long o;
#ifdef LB_L2HINT
    asm volatile("atom.relaxed.gpu.global.min.L2::cache_hint.u64 %0, [%1], %2, %3;" : "=l"(o) : "l"(a), "l"(v), "l"(l2_pol()) : "memory");
#else
    asm volatile("atom.relaxed.gpu.global.min.u64 %0, [%1], %2;" : "=l"(o) : "l"(a), "l"(v) : "memory");
#endif
    return o;
}
__device__ __forceinline__ unsigned atom_exch_u32(unsigned *a, unsigned v) {
    unsigned o;
#ifdef LB_SECHINT
    asm volatile("atom.relaxed.gpu.global.exch.L2::cache_hint.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(a), "r"(v), "l"(l2_pol()) : "memory");
#else
    asm volatile("atom.relaxed.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(o) : "l"(a), "r"(v) : "memory");
#endif
    return o;
}

__device__ __forceinline__ unsigned long long atom_exch_u64(unsigned long long *a, unsigned long long v) {
    unsigned long long o;
#if defined(LB_L2HINT) && defined(LB_EXCH_HINT)
    asm volatile("atom.relaxed.gpu.global.exch.L2::cache_hint.b64 %0, [%1], %2, %3;" : "=l"(o) : "l"(a), "l"(v), "l"(l2_pol()) : "memory");
#else
    asm volatile("atom.relaxed.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(a), "l"(v) : "memory");
#endif
    return o;
}
__device__ __forceinline__ void rst_i32(int *a, int v) {
#ifdef LB_SECHINT
    asm volatile("st.global.cg.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(l2_pol()) : "memory");
#else
    __stcg(a, v);
#endif
}

// Fire-and-forget 64-bit min at L2 (REDG): the issuing thread never waits.
__device__ __forceinline__ void red_min_u64(unsigned long long *a, unsigned long long v) {
#ifdef LB_L2HINT
    asm volatile("red.relaxed.gpu.global.min.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(l2_pol()) : "memory");
#else
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
#endif
}

__device__ __forceinline__ void load_arc(const int4 *arcs, unsigned a, unsigned &dst, unsigned &il,
                                         double &w) {
    int4 r = __ldg(arcs + a);
    dst = (unsigned)r.x;
    il = arc_il(r.y);
    w = __hiloint2double(r.w, r.z);
}

// Warp-aggregated append: one shared-memory atomic per converged group.
__device__ __forceinline__ int agg_append(int *counter) {
    unsigned mask = __activemask();
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    int rank = __popc(mask & ((1u << lane) - 1u));
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + rank;
}

// Warp-staged list append (warp-collective: all 32 lanes call push/flush
// together).  Items collect in a per-warp shared-memory stage and reach the
// global list in bulk: ONE counter atomic per flush instead of one per warp
// batch, so the warps of a CTA never serialize on a shared counter.
constexpr int SW = 128;
struct WStage {
    unsigned *buf;   // SW entries of this warp's stage
    int n;           // staged count (warp-uniform)
    __device__ __forceinline__ void flush(int *counter, unsigned *out) {
        __syncwarp();
        if (n == 0) return;
        int base = 0;
        if ((threadIdx.x & 31) == 0) base = atomicAdd(counter, n);
        base = __shfl_sync(FULL, base, 0);
        for (int i = threadIdx.x & 31; i < n; i += 32) __stcg(out + base + i, buf[i]);
        __syncwarp();
        n = 0;
    }
    __device__ __forceinline__ void push(bool pred, unsigned val, int *counter, unsigned *out) {
        const int lane = threadIdx.x & 31;
        const unsigned m = __ballot_sync(FULL, pred);
        if (pred) buf[n + __popc(m & ((1u << lane) - 1u))] = val;
        n += __popc(m);
        if (n > SW - 32) flush(counter, out);
    }
};

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

}  // namespace lbk
