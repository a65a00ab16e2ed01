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
};

// Graph replica in HBM.  Arc record = 16 B {dst, ilabel, weight};
// epsilon arcs additionally get a per-state CSR of 16 B {dst, arc id, weight}
// records so the closure reads one record per epsilon arc.
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

// Per-state record of a lane: everything a touched state needs in ONE 32-byte
// sector.  cost[] is double-buffered by frame parity so the previous frame's
// token cost of a source state stays readable while the current frame writes.
struct __align__(32) StateRec {
    unsigned long long pack;   // packed (cost, arc) word, SENT = untouched
    double cost[2];            // f64 winner cost of frame t in cost[t & 1]
    int pred;                  // (prev token index << 1) | 1  or  (source state << 1)
    int tokidx;                // token index in the newest frame (sparse-set check)
};

// Per-lane scratch, all indexed by state (O(S) once, reset O(touched) per frame).
struct LaneWs {
    StateRec *rec;
    double *minsnap;        // min frontier snapshot cost this frame (lattice eps rule)
    unsigned *tag;          // epsilon round tag
    unsigned *touched;
    unsigned *fs0, *fs1;    // epsilon frontier: state,
    double *fc0, *fc1;      //   snapshot cost,
    uint2 *fe0, *fe1;       //   epsilon record range
    unsigned *round_ctr;    // persistent per-lane round counter
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

struct Params {
    double beam, lattice_beam, scale;
    long long max_active, max_tokens;
    int D;
    int want_lattice;
    int collect_packs;
    int acrow_smem;
    unsigned long long *prof;   // optional per-phase ns accumulators (LB_PHASE_PROFILE=1)
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
struct RecView {
    unsigned long long pack;
    double cost0, cost1;
    int pred, tokidx;
    __device__ __forceinline__ double cost(int parity) const { return parity ? cost1 : cost0; }
};

__device__ __forceinline__ RecView load_rec(const StateRec *r) {
    const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2 *>(r));
    const ulonglong2 b = __ldcg(reinterpret_cast<const ulonglong2 *>(r) + 1);
    RecView v;
    v.pack = a.x;
    v.cost0 = __longlong_as_double((long long)a.y);
    v.cost1 = __longlong_as_double((long long)b.x);
    v.pred = (int)(unsigned)(b.y & 0xFFFFFFFFull);
    v.tokidx = (int)(unsigned)(b.y >> 32);
    return v;
}

// One 32-byte request for a whole state record (sm_100 256-bit LDG/STG, L2 only).
__device__ __forceinline__ RecView load_rec32(const StateRec *r) {
    unsigned long long x0, x1, x2, x3;
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(r) : "memory");
    RecView v;
    v.pack = x0;
    v.cost0 = __longlong_as_double((long long)x1);
    v.cost1 = __longlong_as_double((long long)x2);
    v.pred = (int)(unsigned)(x3 & 0xFFFFFFFFull);
    v.tokidx = (int)(unsigned)(x3 >> 32);
    return v;
}
__device__ __forceinline__ void store_rec32(StateRec *r, unsigned long long pack, double c0, double c1,
                                            int pred, int tokidx) {
    const unsigned long long x3 = (unsigned long long)(unsigned)pred | ((unsigned long long)(unsigned)tokidx << 32);
    asm volatile("st.global.cg.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(r), "l"(pack),
                 "l"((unsigned long long)__double_as_longlong(c0)), "l"((unsigned long long)__double_as_longlong(c1)),
                 "l"(x3)
                 : "memory");
}

__device__ __forceinline__ void load_arc(const int4 *arcs, unsigned a, unsigned &dst, unsigned &il,
                                         double &w) {
    int4 r = __ldg(arcs + a);
    dst = (unsigned)r.x;
    il = (unsigned)r.y;
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
