// lb_kernels.cuh — the sm_100a decode-lane kernels.
//
// A decode lane is one thread-block CLUSTER (C CTAs, C = 1..4) that owns one
// utterance of a wave (the paper's sequence parallelism, as
// lanes instead of MPS processes).  The lane walks the utterance's frames in
// order; inside a frame its C CTAs split every phase below and meet at cluster
// barriers.  Lane-wide counters (token / lattice list lengths, error flag) live
// in the rank-0 CTA's shared memory and are reached through DSMEM; every other
// list (candidates, touched states, epsilon frontiers, fixes) is CTA-local with
// a shared-memory append counter, so the hot loops never wait on a remote
// atomic.  No frame ever leaves the GPU.
//
//   emit      warp-cooperative expansion of the previous frame's tokens: the warp
//             takes 32 tokens, prefix-scans their out-degrees with shuffles
//             (Alg. 2 / static partition, scheduler.py:60-78) and walks the
//             flattened arc range 32*UNR arcs at a time, each lane binary-
//             searching its owner token with shuffles; 16 B arc loads; one
//             fire-and-forget 64-bit RED.MIN per candidate on the packed
//             (cost, arc) word (Alg. 1, decoder.py:189-205) and a coalesced
//             append of the candidate {dst, arc, cost, token} to the CTA's
//             candidate buffer.  The frame best is a cluster min over ALL
//             candidates (decoder.py:533-539).
//   winners   per candidate: it owns its state iff the state's final word is its
//             own word (arc ids make words unique); the owner records the
//             state's f64 cost / predecessor (decoder.py:314-327), lists the state
//             as touched, seeds the epsilon frontier and the max-active histogram.
//   epsilon   Jacobi rounds (reference.py:160-192) with ONE cluster barrier per
//             round: a frontier state first recovers its cost from the previous
//             round's round-local winning word (rpk, a second 64-bit min that only
//             improving offers reach) and its source's parked snapshot, then
//             offers from that snapshot.  Round barriers keep the reference's
//             snapshot semantics bit-exact.
//   aggregate touched states under the cutoff become the frame's token list
//             (device order; the host sorts by state when lists are read back);
//             the same pass resets the state word (O(touched), not O(S)).
//   lattice   live arcs by rule A.5: emitting arc live iff its
//             candidate <= cutoff and its destination was kept; epsilon arc live
//             iff both ends kept and min-snapshot(src) + w <= cutoff.
#pragma once
#include <cooperative_groups.h>

#include "lb_device.cuh"

namespace lbk {

namespace cgx = cooperative_groups;

// Shared state of a lane CTA.  Lane-wide fields are authoritative in the rank-0
// CTA; per-CTA fields are this CTA's append counters.  Counters are
// double-buffered by frame parity (epsilon frontier lengths by round mod 3) so
// the set for frame t+1 is cleared while frame t runs, without a barrier.
struct Smem {
    // lane-wide (rank 0)
    int ntok[2], nlat[2];
    int err, err_frame;
    long long err_aux;
    // per CTA
    int ntouched[2], ncand[2], nseed[2], nfix[2], netouched[2];
    int nfinal[2];                 // seeds final after winners (list B, top of the touched segment)
    int nfr[3];
    unsigned long long best[2];    // order-preserving f64 running best (frame parity)
    unsigned long long c_tok, c_scan, c_cand, c_front, c_escan, c_ecand, c_next;
    unsigned round_id;             // epsilon round tag (identical in every CTA of the lane)
    double red0;
    int ired0;
    double red[32];
    int ired[32];
    int hist[2][NBINS];            // max-active histogram (frame parity)
    int ready_seen;                // last value of *Params::ready this CTA observed
};

// The lane CTA's shared state and dynamic shared memory, declared at namespace
// scope so every phase addresses them as shared::cta directly (a generic
// pointer into a cluster's shared window costs an address conversion per use).
__shared__ Smem lane_sm;
extern __shared__ double lane_dyn[];

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7FF0000000000000ll); }

// The cluster that runs one lane.
struct Grp {
    Smem *M;        // rank-0 CTA's shared state (DSMEM)
    int rank, C;
    __device__ __forceinline__ void sync() const { cgx::this_cluster().sync(); }
    __device__ __forceinline__ Smem *at(int q) const { return cgx::this_cluster().map_shared_rank(&lane_sm, q); }
    __device__ __forceinline__ int gtid() const { return rank * blockDim.x + threadIdx.x; }
    __device__ __forceinline__ int gstride() const { return C * blockDim.x; }
    __device__ __forceinline__ int gwarp() const { return rank * (blockDim.x >> 5) + (threadIdx.x >> 5); }
    __device__ __forceinline__ int gnw() const { return C * (blockDim.x >> 5); }
    __device__ __forceinline__ bool leader() const { return rank == 0 && threadIdx.x == 0; }
};

// Cluster-wide (value, state) lexicographic min; result on every thread.
__device__ __forceinline__ void cl_argmin(double &v, int &s, const Grp &G) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(FULL, v, o);
        int os = __shfl_xor_sync(FULL, s, o);
        if (ov < v || (ov == v && os < s)) { v = ov; s = os; }
    }
    if (lane == 0) { lane_sm.red[warp] = v; lane_sm.ired[warp] = s; }
    __syncthreads();
    if (warp == 0) {
        double x = lane < nw ? lane_sm.red[lane] : inf_d();
        int y = lane < nw ? lane_sm.ired[lane] : 0x7FFFFFFF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(FULL, x, o);
            int os = __shfl_xor_sync(FULL, y, o);
            if (ov < x || (ov == x && os < y)) { x = ov; y = os; }
        }
        if (lane == 0) { lane_sm.red0 = x; lane_sm.ired0 = y; }
    }
    G.sync();
    v = inf_d();
    s = 0x7FFFFFFF;
    for (int q = 0; q < G.C; q++) {
        const Smem *R = G.at(q);
        const double x = R->red0;
        const int y = R->ired0;
        if (x < v || (x == v && y < s)) { v = x; s = y; }
    }
    G.sync();
}

// Warp-cooperative load-balanced walk over every (token, out-arc) pair of a
// token list, UNR arcs per lane per batch; warps of all CTAs of the lane share
// the list.  Per group of 32 tokens the warp prefix-scans the out-degrees with
// shuffles (the static partition of scheduler.py:60-78 at warp granularity);
// each token then writes its lane id over its arc slots in a per-warp shared
// memory map (`own`, WMAP slots), so an arc slot finds its owner token with ONE
// shared load instead of a 5-step shuffle binary search (the search remains as
// the fallback for groups wider than the map).  The next group's tokens are
// fetched while the current group's arcs are walked.  f(valid[], i[], arc[],
// cost[]) receives one batch; the batch loop is warp-uniform, so f may use
// full-mask warp collectives.
constexpr int WMAP = 512;
// winner payload lists (written by winners, read once by aggregate): streamed
// with evict-first under LB_PAY_EF (an experiment knob), L2-normal otherwise
#ifdef LB_PAY_EF
#define PAY_ST __stcs
#define PAY_LD __ldcs
#else
#define PAY_ST __stcg
#define PAY_LD __ldcg
#endif
template <int UNR, class OwnT, class F>
__device__ __forceinline__ void for_each_token_arc_batched(const GraphDev &g, int gwarp, int gnw,
                                                           const unsigned *ts, const double *tc, int n,
                                                           unsigned &c_scan, OwnT *own, F &&f) {
    const int lane = threadIdx.x & 31;
    const int step = gnw * 32;
    int base = gwarp * 32;
    unsigned s = 0u;
    double c = 0.0;
    if (base + lane < n) {
        s = __ldcg(ts + base + lane);
        c = __ldcg(tc + base + lane);
    }
    for (; base < n; base += step) {
        const bool valid = base + lane < n;
        const uint2 rg = valid ? gld2(g.rng + s) : make_uint2(0u, 0u);
        // prefetch the next group's tokens
        const int nb = base + step;
        unsigned s_n = 0u;
        double c_n = 0.0;
        if (nb + lane < n) {
            s_n = __ldcg(ts + nb + lane);
            c_n = __ldcg(tc + nb + lane);
        }
        const unsigned lo = rg.x;
        const int deg = (int)(rg.y - rg.x);
        int incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const int excl = incl - deg;
        const int total = __shfl_sync(FULL, incl, 31);
        if (lane == 0) c_scan += (unsigned)total;
        const bool mapped = total <= WMAP;
        if (mapped) {
            for (int j = excl; j < incl; j++) own[j] = (OwnT)lane;
            __syncwarp();
        }
        for (int j0 = 0; j0 < total; j0 += 32 * UNR) {
            bool vv[UNR];
            int ii[UNR];
            unsigned aa[UNR];
            double cc[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const int j = j0 + u * 32 + lane;
                int k = 0;
                if (mapped) {
                    k = j < total ? own[j] : 0;
                } else {
#pragma unroll
                    for (int b = 16; b > 0; b >>= 1) {
                        int t = __shfl_sync(FULL, incl, k + b - 1);
                        if (t <= j) k += b;
                    }
                }
                const int ek = __shfl_sync(FULL, excl, k);
                const unsigned lk = __shfl_sync(FULL, lo, k);
                cc[u] = __shfl_sync(FULL, c, k);
                vv[u] = j < total;
                ii[u] = base + k;
                aa[u] = lk + (unsigned)(j - ek);
            }
            f(vv, ii, aa, cc);
        }
        if (mapped) __syncwarp();
        s = s_n;
        c = c_n;
    }
}

// Dynamic shared memory of a lane CTA of `threads` threads (see Lane::Lane).
// Per-warp phase scratch (bytes), aliased between phases: winners uses two u32
// stages of SW entries; aggregate a token stage of SWT entries {cost, minsnap,
// state, arc, key, pred} and a u32 fix stage.
constexpr int SWT = 64;
constexpr size_t ACROW_SMEM_MAX = 48 * 1024;   // acoustic rows up to 6144 pdfs live in shared memory
constexpr int SWW = 96;   // winners stages: touched {v, arc, pred, cost} and round-0 frontier {v, cost}
constexpr int WSCR = (SWT * 32 + SW * 4) > SWW * 32 ? (SWT * 32 + SW * 4) : SWW * 32;
static_assert(SWW * 20 + SWW * 12 <= WSCR, "winners stages fit the warp scratch");
// `row_pf`: two row buffers (the next frame's row is prefetched, Lane::row_async).
inline size_t lane_dyn_smem(int threads, int D, bool acrow_smem, bool row_pf = false) {
    const size_t nw = (size_t)threads / 32;
    return (acrow_smem ? (size_t)D * 8 * (row_pf ? 2 : 1) : 0) + nw * WMAP + nw * WSCR + nw * NBINS * 4;
}
constexpr int CAND_CHUNK = 256;   // Lane::CCH

// Max-active histogram bin of a seed:
// min(NBINS-1, max(0, trunc(RN((c - best) / width)))) exactly.  The quotient is
// taken as a product with the rounded reciprocal, and recomputed with a true
// division only when that product lies within 1e-9 of an integer (the only
// place the two can truncate differently), so the bin is bit-exact with the
// oracle's division at a fraction of its cost.
__device__ __forceinline__ int hist_bin(double c, double best, double width, double inv_w) {
    const double d = __dsub_rn(c, best);
    double q = __dmul_rn(d, inv_w);
    const double fr = q - floor(q);
    if (fr < 1e-9 || fr > 1.0 - 1e-9) q = __ddiv_rn(d, width);
    return q >= (double)NBINS ? NBINS - 1 : (q < 0.0 ? 0 : (int)q);
}

// Per-lane decode phases.  UNR = independent arcs per thread per emit batch.
template <int UNR>
struct Lane {
#ifdef LB_WUNR
    static constexpr int WUNR = LB_WUNR;
#else
    static constexpr int WUNR = 1;   // candidates per thread per winners batch (next batch prefetched)
#endif
#ifdef LB_EUNR
    static constexpr int EUNR = LB_EUNR;
#else
    static constexpr int EUNR = 1;   // frontier entries per thread per epsilon batch (2: spills, -4 %)
#endif
    const GraphDev &g;      // __grid_constant__ kernel parameters: referenced in place,
    const Params &p;        // never copied to local memory
    const LaneWs &L;
    const UttDesc &io;
    const Grp G;
    unsigned long long *wprof = nullptr;   // per-warp busy-time accumulators (profiling only)
    const double *row;      // global row of the current frame
    int par;                // parity of the current frame (counter set)

    // Dynamic shared memory (lane_dyn): [acrow: D f64 when p.acrow_smem][per-warp
    // scratch][per-warp histograms][byte owner maps].  Addresses are derived from the
    // namespace-scope shared array at each use so they stay shared::cta.
    __device__ Lane(const GraphDev &g_, const Params &p_, const LaneWs &L_, const UttDesc &io_,
                    const Grp &G_, double *)
        : g(g_), p(p_), L(L_), io(io_), G(G_), row(nullptr), par(0) {}
    __device__ __forceinline__ int acrow_doubles() const { return p.acrow_smem ? p.D * (p.row_pf ? 2 : 1) : 0; }
    // [acrow][per-warp scratch][per-warp histograms][byte owner maps]: a lane id
    // fits a byte, and every byte of shared memory saved is L1 capacity
    __device__ __forceinline__ char *scratch_all() const { return reinterpret_cast<char *>(lane_dyn + acrow_doubles()); }
    __device__ __forceinline__ unsigned char *own_all() const {
        return reinterpret_cast<unsigned char *>(scratch_all() + (blockDim.x >> 5) * (WSCR + NBINS * 4));
    }
    __device__ __forceinline__ int *whist_all() const {
        return reinterpret_cast<int *>(scratch_all() + (blockDim.x >> 5) * WSCR);
    }
    __device__ __forceinline__ char *scratch() const { return scratch_all() + (threadIdx.x >> 5) * WSCR; }
    // u32 stage q (0, 1) of this warp's scratch (winners)
    __device__ __forceinline__ WStage stage(int q) const {
        WStage st;
        st.buf = reinterpret_cast<unsigned *>(scratch()) + q * SW;
        st.n = 0;
        return st;
    }

    // Profiling aid: a warp's busy time inside a phase (up to its arrival at the
    // phase's closing barrier), summed over warps; [ph] = ns, [8 + ph] = samples.
    __device__ __forceinline__ unsigned long long wbegin() const { return wprof ? gtimer() : 0ull; }
    __device__ __forceinline__ void wend(int ph, unsigned long long t0) const {
        if (wprof) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                atomicAdd(wprof + ph, gtimer() - t0);
                atomicAdd(wprof + 8 + ph, 1ull);
            }
        }
    }

    // this CTA's segments of the per-CTA lists
    // emitting winners of this CTA (with their payload) and epsilon-reached states
    __device__ __forceinline__ size_t cseg() const { return (size_t)G.rank * L.ccap; }
    __device__ __forceinline__ unsigned *touched() const { return L.touched + cseg(); }
    __device__ __forceinline__ unsigned *etouched() const { return L.etouched + (size_t)G.rank * L.S; }
    __device__ __forceinline__ unsigned *front(int r) const {
        return L.fr + ((size_t)(r & 1) * L.C + G.rank) * L.S;
    }
    __device__ __forceinline__ EpsWin *rpk(int r) const { return L.rpk + (size_t)(r & 1) * L.S; }

    __device__ __forceinline__ unsigned *fixes() const { return L.fix + (size_t)G.rank * L.S; }
    __device__ __forceinline__ unsigned char *wmap() const { return own_all() + (threadIdx.x >> 5) * WMAP; }

    __device__ __forceinline__ double ac(unsigned il) const {
        // with the row prefetch, frame t's row (t-1) sits in buffer (t-1)&1 = par^1
        return p.acrow_smem ? lane_dyn[(p.row_pf ? (par ^ 1) * p.D : 0) + il - 1]
                            : __dmul_rn(__ldg(row + il - 1), p.scale);
    }

    // Next-frame row prefetch (p.row_pf; f64 rows of even D, 16-byte aligned,
    // device-resident or streamed ring): frame t's emit reads row t-1 from buffer
    // (t-1)&1 while row t is already in flight into the other buffer with
    // cp.async (L2 only, .cg, so a ring slot's stale line can never come from L1).
    // Each thread scales exactly the doubles it copied, after its own wait; the
    // barrier before emit publishes them.
    __device__ __forceinline__ void row_async(const double *r, int buf) {
        const unsigned base = (unsigned)__cvta_generic_to_shared(lane_dyn + buf * p.D);
        const int chunks = p.D >> 1;
        for (int q = threadIdx.x; q < chunks; q += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + 16u * q), "l"(r + 2 * q) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __device__ __forceinline__ void row_finish(int buf) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        double *d = lane_dyn + buf * p.D;
        const int chunks = p.D >> 1;
        for (int q = threadIdx.x; q < chunks; q += blockDim.x) {
            d[2 * q] = __dmul_rn(d[2 * q], p.scale);
            d[2 * q + 1] = __dmul_rn(d[2 * q + 1], p.scale);
        }
    }

    __device__ __forceinline__ void set_error(int code, int frame, long long aux) const {
        if (atomicCAS(&G.M->err, 0, code) == 0) {
            G.M->err_frame = frame;
            G.M->err_aux = aux;
        }
    }

    // Frame rows staged progressively by the host (lb_decode_batch, zero-copy):
    // wait until the rows of frames < need are published.  The smem copy of the
    // flag is written only between two barriers (every thread has tested it
    // before thread 0 updates it), so the test is CTA-uniform; the barriers are
    // spent only when the copy is behind (about once per chunk).
    __device__ void wait_rows(int need) {
        if (lane_sm.ready_seen >= need) return;
        __syncthreads();
        if (threadIdx.x == 0) {
            int r;
            for (;;) {
                asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(r) : "l"(p.ready) : "memory");
                if (r >= need) break;
                __nanosleep(1000);
            }
            lane_sm.ready_seen = r;
        }
        __syncthreads();
    }

    __device__ void load_row(const double *r, int frame) {
        row = r;
        if (p.costs_f32) {   // f32 log-likelihoods (an acoustic model's output): widened exactly
            const float *rf = reinterpret_cast<const float *>(r);
            for (int d = threadIdx.x; d < p.D; d += blockDim.x)
                lane_dyn[d] = __dmul_rn((double)__ldg(rf + d), p.scale);
        } else if (p.ready || p.ring_ready) {
            if (p.ready) wait_rows(frame + 1);
            // L2-only loads (ld.cg): a published row was never cached before it was
            // written (the host aligns chunks to 128-byte lines); ld.cv would be
            // safe without that but costs ~130 us per frame on mapped memory.
            for (int d = threadIdx.x; d < p.D; d += blockDim.x) lane_dyn[d] = __dmul_rn(__ldcg(r + d), p.scale);
        } else if (p.acrow_smem) {
            for (int d = threadIdx.x; d < p.D; d += blockDim.x) lane_dyn[d] = __dmul_rn(__ldg(r + d), p.scale);
        }
    }

    // Clear the counter set of the NEXT frame (its previous readers are done).
    __device__ __forceinline__ void clear_next_counters() const {
        const int q = par ^ 1;
        if (G.leader()) G.M->ntok[q] = G.M->nlat[q] = 0;
        if (threadIdx.x == 0) {
            lane_sm.ntouched[q] = lane_sm.ncand[q] = lane_sm.nseed[q] = lane_sm.nfix[q] = lane_sm.netouched[q] = 0;
            lane_sm.nfinal[q] = 0;
            lane_sm.best[q] = SENT;
        }
    }

    // ---- emit: returns the lane-wide best candidate (one cluster barrier) ----
    // Every candidate feeds the frame best, but a candidate whose float32 key is
    // above the float32 key of a running upper bound of this frame's cutoff
    // (running best + beam_eff) is dropped: it can neither be the best nor the
    // winner of a state that survives the cutoff, and no epsilon offer (cost
    // <= cutoff) can tie with it, so every kept state's winner is unchanged.
    // The running best is one shared word per CTA, read every batch and pushed
    // (one warp-aggregated atomic) only by a batch that improves it.  Surviving
    // candidates go to the CTA's candidate buffer in per-warp chunks of CCH
    // slots (one counter atomic per chunk); a chunk's unused tail is filled
    // with sentinels (x = -1) that winners() skips.
    static constexpr int CCH = CAND_CHUNK;
    __device__ double emit(const unsigned *pts, const double *ptc, int np, double beam_eff, int frame) {
        unsigned long long *pk = L.pk;
        unsigned c_scan = 0, c_cand = 0;
        int *ncand = &lane_sm.ncand[par];
        int4 *cb = L.cand + (size_t)G.rank * L.ccap;
        int *cbi = L.candi + (size_t)G.rank * L.ccap;
        const long long ccap = L.ccap;
        unsigned long long *run = &lane_sm.best[par];
        const int lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1u;
        int cstart = 0, cused = CCH;          // current chunk (warp-uniform); none yet
        bool overflow = false;
        if (threadIdx.x == 0) lane_sm.nfr[0] = lane_sm.nfr[1] = lane_sm.nfr[2] = 0;
        const unsigned long long t0 = wbegin();
        auto fill_tail = [&]() {
            for (int i = cused + lane; i < CCH; i += 32) CAND_ST(cb + cstart + i, make_int4(-1, 0, 0, 0));
        };
        for_each_token_arc_batched<UNR>(g, G.gwarp(), G.gnw(), pts, ptc, np, c_scan, wmap(),
                                        [&](const bool *vv, const int *ii, const unsigned *aa, const double *cc) {
            int4 r[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (vv[u]) r[u] = gld4(g.arcs + aa[u]);
            unsigned long long known = *(volatile unsigned long long *)run;
            double cand[UNR];
            double bmin = inf_d();
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                cand[u] = inf_d();
                const unsigned il = vv[u] ? arc_il(r[u].y) : 0u;
                if (il != 0) {
                    const double w = __hiloint2double(r[u].w, r[u].z);
                    cand[u] = __dadd_rn(__dadd_rn(cc[u], w), ac(il));
                    bmin = fmin(bmin, cand[u]);
                }
            }
            unsigned long long eb = enc64(bmin);
            if (__any_sync(FULL, eb < known)) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long x = __shfl_xor_sync(FULL, eb, o);
                    eb = x < eb ? x : eb;
                }
                if (lane == 0) atomicMin(run, eb);
                known = eb < known ? eb : known;
            }
            unsigned bound_key = 0xFFFFFFFFu;     // enc32 of the running cutoff bound
            if (known != SENT) bound_key = (unsigned)(pack_word(__dadd_rn(dec64(known), beam_eff), 0u) >> 32);
            bool em[UNR];
            int off[UNR];
            int tot = 0;
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                em[u] = false;
                if (cand[u] < inf_d()) {
                    const unsigned long long word = pack_word(cand[u], aa[u]);
                    em[u] = (unsigned)(word >> 32) <= bound_key;
                    if (em[u]) red_min_u64(pk + r[u].x, word);
                }
                const unsigned bb = __ballot_sync(FULL, em[u]);
                off[u] = tot + __popc(bb & lt);
                tot += __popc(bb);
            }
            if (tot == 0) return;
            c_cand += (lane == 0) ? (unsigned)tot : 0u;
            if (cused + tot > CCH) {
                if (cused < CCH) fill_tail();
                int nb = 0;
                if (lane == 0) nb = atomicAdd(ncand, CCH);
                cstart = __shfl_sync(FULL, nb, 0);
                cused = 0;
                if ((long long)cstart + CCH > ccap) {
                    overflow = true;
                    if (lane == 0) set_error(E_CAP_CAND, frame, (long long)cstart + CCH);
                }
            }
            if (!overflow) {
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    if (em[u]) {
                        const long long bits = __double_as_longlong(cand[u]);
                        const unsigned flag = (unsigned)r[u].y & STATE_FLAGS;
                        const int k = cstart + cused + off[u];
                        CAND_ST(cb + k, make_int4((int)((unsigned)r[u].x | flag), (int)aa[u],
                                                 (int)(bits & 0xFFFFFFFFll), (int)(bits >> 32)));
                        CAND_ST(cbi + k, ii[u]);
                    }
                }
            }
            cused += tot;
        });
        if (cused < CCH && !overflow) fill_tail();
        c_cand = warp_sum(c_cand);
        c_scan = warp_sum(c_scan);
        if (lane == 0) {
            atomicAdd(&lane_sm.c_cand, (unsigned long long)c_cand);
            atomicAdd(&lane_sm.c_scan, (unsigned long long)c_scan);
        }
        wend(0, t0);
        G.sync();
        unsigned long long b = SENT;
        for (int q = 0; q < G.C; q++) {
            const unsigned long long x = G.at(q)->best[par];
            b = x < b ? x : b;
        }
        return dec64(b);
    }

    // Epsilon predecessors of the PREVIOUS frame's tokens (source state -> token
    // index), run inside the next frame's emit phase so it needs no barrier of its
    // own: the indices it reads were final at the previous aggregate barrier and
    // are not rewritten before this frame's aggregate.  `fpar` = previous frame's
    // parity (its fix count), `tbf`/`nf` = its token list.
    __device__ void fix_preds(int fpar, int frame, long long tbf, int nf) {
        const int mine = lane_sm.nfix[fpar];
        const unsigned *fx = fixes();
        for (int q = threadIdx.x; q < mine; q += blockDim.x) {
            const long long o = tbf + (long long)__ldcg(fx + q);
            const int u = __ldcg(io.tok_pred + o) >> 1;
            const int pi = rld_i32(L.tokidx + u);
            if (pi < 0 || pi >= nf || __ldcg(io.tok_state + tbf + pi) != (unsigned)u)
                set_error(E_INT_EPS_PRED, frame, u);
            __stcg(io.tok_pred + o, pi << 1);
        }
    }

    // ---- winners: owners of the state words; seeds; epsilon frontier (round 0); histogram ----
    // Warp-uniform loop over the CTA's candidate buffer (32*WUNR entries per warp
    // step).  A candidate owns its state iff the state's final word is its own
    // word (arc ids make words unique).  The owner's payload {state, arc,
    // predecessor, f64 cost} goes to this CTA's touched list and, for a seed
    // with epsilon arcs, {state, cost} to the round-0 frontier -- both through
    // per-warp shared-memory stages flushed in bulk (one counter atomic per
    // flush, coalesced writes), so no per-state record is written here.  The
    // max-active histogram is per warp and summed into the CTA histogram at the
    // end, so no shared-memory atomic is ever contended.
    struct WinStage {   // per-warp stage of owner payloads (SWW entries)
        unsigned *v, *a;
        int *p;
        double *c;
        int n;
    };
    struct FrStage {    // per-warp stage of round-0 frontier entries (SWW entries)
        unsigned *v;
        double *c;
        int n;
    };
    // Flush a winner stage: entries marked final (bit 31 of the state) go to list
    // B, filled downward from the top of this CTA's touched segment (counter
    // `nfin`); the others to list A from the bottom (counter `counter`).  The two
    // never meet: together they hold at most one entry per candidate.
    __device__ __forceinline__ void win_flush(WinStage &st, int *counter, int *nfin) const {
        __syncwarp();
        if (st.n == 0) return;
        const int lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1u;
        int nb = 0;
        for (int i0 = 0; i0 < st.n; i0 += 32) {
            const int i = i0 + lane;
            nb += __popc(__ballot_sync(FULL, i < st.n && (st.v[i] >> 31)));
        }
        int ba = 0, bb = 0;
        if (lane == 0) {
            if (st.n > nb) ba = atomicAdd(counter, st.n - nb);
            if (nb) bb = atomicAdd(nfin, nb);
        }
        ba = __shfl_sync(FULL, ba, 0);
        bb = __shfl_sync(FULL, bb, 0);
        const size_t cs = cseg(), top = cs + (size_t)L.ccap - 1;
        for (int i0 = 0; i0 < st.n; i0 += 32) {
            const int i = i0 + lane;
            const bool in = i < st.n;
            const unsigned v = in ? st.v[i] : 0u;
            const bool fb = in && (v >> 31);
            const unsigned mb = __ballot_sync(FULL, fb), ma = __ballot_sync(FULL, in && !fb);
            if (in) {
                const size_t o = fb ? top - (size_t)(bb + __popc(mb & lt)) : cs + (size_t)(ba + __popc(ma & lt));
                PAY_ST(L.touched + o, v & 0x7FFFFFFFu);
                PAY_ST(L.tarc + o, st.a[i]);
                PAY_ST(L.tpred + o, st.p[i]);
                PAY_ST(L.tcost + o, st.c[i]);
            }
            ba += __popc(ma);
            bb += __popc(mb);
        }
        __syncwarp();
        st.n = 0;
    }
    __device__ __forceinline__ void fr_flush(FrStage &st, int *counter, unsigned *out) const {
        __syncwarp();
        if (st.n == 0) return;
        int base = 0;
        if ((threadIdx.x & 31) == 0) base = atomicAdd(counter, st.n);
        base = __shfl_sync(FULL, base, 0);
        double *oc = L.f0cost + cseg() + base;
        for (int i = threadIdx.x & 31; i < st.n; i += 32) {
            __stcg(out + base + i, st.v[i]);
            __stcg(oc + i, st.c[i]);
        }
        __syncwarp();
        st.n = 0;
    }

    __device__ void winners(double cutoff, double best) {
        const int nc = lane_sm.ncand[par];
        const bool hist = p.max_active > 0;
        const double width = __ddiv_rn(p.beam, (double)NBINS);
        const double inv_w = __drcp_rn(width);
        const int4 *cb = L.cand + (size_t)G.rank * L.ccap;
        const int *cbi = L.candi + (size_t)G.rank * L.ccap;
        unsigned long long *pk = L.pk;
        unsigned *f0 = front(0);
        int *ntouched = &lane_sm.ntouched[par], *nf0 = &lane_sm.nfr[0];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        const unsigned lt = (1u << lane) - 1u;
        int *wh = whist_all() + warp * NBINS;
        if (hist)
            for (int b = lane; b < NBINS; b += 32) wh[b] = 0;
        __syncwarp();
        char *scr = scratch();
        WinStage sw;
        sw.c = reinterpret_cast<double *>(scr);
        sw.v = reinterpret_cast<unsigned *>(sw.c + SWW);
        sw.a = sw.v + SWW;
        sw.p = reinterpret_cast<int *>(sw.a + SWW);
        sw.n = 0;
        FrStage sf;
        sf.c = reinterpret_cast<double *>(sw.p + SWW);
        sf.v = reinterpret_cast<unsigned *>(sf.c + SWW);
        sf.n = 0;
        unsigned nseed = 0;
        const unsigned long long t0 = wbegin();
#ifndef LB_WIN_NOPIPE
        // two-stage pipeline: batch b's state words were requested during batch
        // b-1, and batch b+2's candidate records are requested during batch b
        // (winners 32.4 -> 28.8 us per lane-frame at 64 lanes)
        const int stride = nw * 32 * WUNR;
        auto cand_at = [&](int k, int4 &e, int &t) {
            e.x = -1;
            t = 0;
            if (k < nc) {
                e = CAND_LD(cb + k);
                t = CAND_LD(cbi + k);
            }
        };
        int4 ec[WUNR], en[WUNR];
        int tc[WUNR], tn[WUNR];
        unsigned long long pc[WUNR];
#pragma unroll
        for (int u = 0; u < WUNR; u++) {
            cand_at(warp * 32 * WUNR + u * 32 + lane, ec[u], tc[u]);
            cand_at(warp * 32 * WUNR + stride + u * 32 + lane, en[u], tn[u]);
        }
#pragma unroll
        for (int u = 0; u < WUNR; u++) pc[u] = ec[u].x != -1 ? rld_u64(pk + ((unsigned)ec[u].x & ~STATE_FLAGS)) : 0ull;
        for (int kb = warp * 32 * WUNR; kb < nc; kb += stride) {
            int4 e[WUNR];
            int ti[WUNR];
            unsigned long long pw[WUNR];
#pragma unroll
            for (int u = 0; u < WUNR; u++) {
                e[u] = ec[u];
                ti[u] = tc[u];
                pw[u] = pc[u];
                ec[u] = en[u];
                tc[u] = tn[u];
                pc[u] = ec[u].x != -1 ? rld_u64(pk + ((unsigned)ec[u].x & ~STATE_FLAGS)) : 0ull;
                cand_at(kb + 2 * stride + u * 32 + lane, en[u], tn[u]);
            }
#else
        // candidate records of the next batch are fetched one batch ahead
        int4 en[WUNR];
        int tn[WUNR];
#pragma unroll
        for (int u = 0; u < WUNR; u++) {
            const int k = warp * 32 * WUNR + u * 32 + lane;
            en[u].x = -1;
            tn[u] = 0;
            if (k < nc) {
                en[u] = CAND_LD(cb + k);
                tn[u] = CAND_LD(cbi + k);
            }
        }
        for (int kb = warp * 32 * WUNR; kb < nc; kb += nw * 32 * WUNR) {
            int4 e[WUNR];
            int ti[WUNR];
#pragma unroll
            for (int u = 0; u < WUNR; u++) {
                e[u] = en[u];
                ti[u] = tn[u];
                const int k = kb + nw * 32 * WUNR + u * 32 + lane;
                en[u].x = -1;
                if (k < nc) {
                    en[u] = CAND_LD(cb + k);
                    tn[u] = CAND_LD(cbi + k);
                }
            }
            unsigned long long pw[WUNR];
#pragma unroll
            for (int u = 0; u < WUNR; u++)
                pw[u] = e[u].x != -1 ? rld_u64(pk + ((unsigned)e[u].x & ~STATE_FLAGS)) : 0ull;
#endif
#pragma unroll
            for (int u = 0; u < WUNR; u++) {
                const unsigned v = (unsigned)e[u].x & ~STATE_FLAGS;
                const double cand = __hiloint2double(e[u].w, e[u].z);
                const bool own = e[u].x != -1 && pw[u] == pack_word(cand, (unsigned)e[u].y);
                const bool seed = own && cand <= cutoff;
#ifndef LB_WIN_KEEP_ALL
                // An owner above the cutoff can only be kept if an epsilon offer
                // (<= cutoff) improves it later, and such an offer finds the word
                // reset and lists the state as epsilon-reached (erec).  So it is
                // reset here and never enters the winner list: aggregate touches
                // only the seeds (about half the owners at max-active; 140 -> 132
                // us per lane-frame).  (Resetting with a compare-and-swap instead
                // of reading the words above the cutoff measured slower.)
                if (own && !seed) rst_u64(pk + v, SENT);
                const bool listed = seed;
#else
                const bool listed = own;
#endif
#ifndef LB_NO_FINAL_SEEDS
                // A seed whose state has no incoming epsilon arc is final now: no
                // epsilon offer can reach its word.  Reset the word here and list
                // the seed in list B, which aggregate consumes without the atomic
                // exchange (list A keeps the seeds epsilon offers may improve).
                const bool fin = seed && ((unsigned)e[u].x & NOEPSIN_FLAG);
                if (fin) rst_u64(pk + v, SENT);
#else
                const bool fin = false;
#endif
                const unsigned mo = __ballot_sync(FULL, listed);
                if (listed) {
                    const int j = sw.n + __popc(mo & lt);
                    sw.v[j] = v | (fin ? 0x80000000u : 0u);
                    sw.a[j] = (unsigned)e[u].y;
                    sw.p[j] = (ti[u] << 1) | 1;
                    sw.c[j] = cand;
                }
                sw.n += __popc(mo);
                nseed += seed;
                // only states with epsilon arcs enter the closure
                const bool fz = seed && ((unsigned)e[u].x & EPS_FLAG);
                const unsigned mf = __ballot_sync(FULL, fz);
                if (fz) {
                    const int j = sf.n + __popc(mf & lt);
                    sf.v[j] = v;
                    sf.c[j] = cand;
                }
                sf.n += __popc(mf);
                if (hist && seed) atomicAdd(wh + hist_bin(cand, best, width, inv_w), 1);
                if (sw.n > SWW - 32) win_flush(sw, ntouched, &lane_sm.nfinal[par]);
                if (sf.n > SWW - 32) fr_flush(sf, nf0, f0);
            }
#ifdef LB_CAND_DISCARD
            // this batch's candidate lines are dead (read once, their values are in
            // registers and used above): drop them from L2 without a write-back
            if (lane < 5 * WUNR) {
                const int q = lane % 5, uu = lane / 5;
                const void *a = q < 4 ? (const void *)(cb + kb + uu * 32 + q * 8) : (const void *)(cbi + kb + uu * 32);
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
            }
#endif
        }
        win_flush(sw, ntouched, &lane_sm.nfinal[par]);
        fr_flush(sf, nf0, f0);
        nseed = warp_sum(nseed);
        if (lane == 0 && nseed) atomicAdd(&lane_sm.nseed[par], (int)nseed);
        wend(1, t0);
        if (hist) {
            __syncthreads();
            for (int b = threadIdx.x; b < NBINS; b += blockDim.x) {
                int sum = 0;
                for (int w = 0; w < nw; w++) sum += whist_all()[w * NBINS + b];
                lane_sm.hist[par][b] = sum;
            }
        }
    }

    // Lane-wide seed count (after the barrier that follows winners()).
    __device__ __forceinline__ int lane_seeds() const {
        int s = 0;
        for (int q = 0; q < G.C; q++) s += G.at(q)->nseed[par];
        return s;
    }

    // max-active cutoff: H = best + max(b*,1)*width, b* = first
    // bin whose inclusive running count exceeds max_active.  Warp 0 of every CTA
    // merges the lane's per-CTA histograms through DSMEM (8 bins per lane) and
    // computes the same value, so no cluster barrier is needed.  Called after a
    // cluster barrier that follows winners().
    __device__ double max_active_cutoff(double cutoff, double best) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        constexpr int PER = NBINS / 32;
        if (warp == 0) {
            int loc[PER];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < PER; q++) loc[q] = 0;
            for (int r = 0; r < G.C; r++) {
                const Smem *R = G.at(r);
#pragma unroll
                for (int q = 0; q < PER; q++) loc[q] += R->hist[par][lane * PER + q];
            }
#pragma unroll
            for (int q = 0; q < PER; q++) sum += loc[q];
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            long long cum = incl - sum;
            int found = -1;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                cum += loc[q];
                if (found < 0 && cum > p.max_active) found = lane * PER + q;
            }
            const unsigned m = __ballot_sync(FULL, found >= 0);
            double c2 = cutoff;
            if (m) {
                const int bstar = __shfl_sync(FULL, found, __ffs(m) - 1);
                const double width = __ddiv_rn(p.beam, (double)NBINS);
                const double h = __dadd_rn(best, __dmul_rn((double)(bstar < 1 ? 1 : bstar), width));
                c2 = h < cutoff ? h : cutoff;
            }
            if (lane == 0) lane_sm.red0 = c2;
        }
        __syncthreads();
        const double r = lane_sm.red0;
        __syncthreads();
        return r;
    }

    // ---- epsilon closure under a fixed cutoff: Jacobi rounds, ONE barrier each ----
    // Round r processes this CTA's frontier F_r (states improved in round r-1;
    // round 0 = seeds).  Every improving offer of round r-1 to v also entered the
    // pair (word, f64 cost) into rpk[(r-1)&1][v] with a 128-bit CAS-min, so the
    // round winner's word AND its exact f64 cost are one 16-byte load away
    // (offers of round r go to the other buffer and cannot disturb it).  v
    // adopts that cost, then offers from it: exactly the reference's snapshot
    // semantics (reference.py:160-192).
    __device__ bool epsilon(double cutoff, int frame) {
        const bool LAT = p.want_lattice;
        unsigned long long *pk = L.pk;
        const unsigned round_id0 = lane_sm.round_id;
        unsigned round_id = round_id0;
        unsigned c_escan = 0, c_ecand = 0, c_front = 0;
        unsigned *etl = etouched();
        int *netouched = &lane_sm.netouched[par];
        const int bd = blockDim.x;
        bool ok = true;
        for (int r = 0;; r++) {
            int total = 0;
            for (int q = 0; q < G.C; q++) total += G.at(q)->nfr[r % 3];
            if (total == 0) break;
            if (r > g.S + 1) {
                if (G.leader()) set_error(E_INT_EPS_ROUNDS, frame, 0);
                ok = false;
                break;
            }
            ++round_id;
            const int nf = lane_sm.nfr[r % 3];
            const unsigned *fs = front(r);
            unsigned *fsn = front(r + 1);

            int *nnext = &lane_sm.nfr[(r + 1) % 3];
            if (threadIdx.x == 0) lane_sm.nfr[(r + 2) % 3] = 0;   // read at round r-1's start, one barrier ago
            EpsWin *rprev = rpk(r + 1);                         // == rpk(r - 1)
            EpsWin *rcur = rpk(r);
            const unsigned long long t0 = wbegin();
            for (int k0 = threadIdx.x; k0 < nf; k0 += EUNR * bd) {
                unsigned v[EUNR];
                uint2 er[EUNR];
                double c[EUNR];
                unsigned src[EUNR];
#pragma unroll
                for (int u = 0; u < EUNR; u++) {
                    const int k = k0 + u * bd;
                    v[u] = k < nf ? __ldcg(fs + k) : 0xFFFFFFFFu;
                    c[u] = (r == 0 && k < nf) ? __ldcg(L.f0cost + cseg() + k) : 0.0;   // seeds carry their cost
                }
#pragma unroll
                for (int u = 0; u < EUNR; u++) {
                    if (v[u] == 0xFFFFFFFFu) continue;
                    er[u] = gld2(g.erng + v[u]);
                    if (r > 0) {
                        const ulonglong2 w2 = rld_u128(rprev + v[u]);
                        rst_u128(rprev + v[u], make_ulonglong2(~0ull, ~0ull));
                        c[u] = __longlong_as_double((long long)w2.y);
                        // the winner's source state: loaded now, stored after the
                        // offers below (a store waiting on this load would stall them)
                        src[u] = __ldg(g.src + (unsigned)w2.x);
                    }
                }
#pragma unroll
                for (int u = 0; u < EUNR; u++) {
                    if (v[u] == 0xFFFFFFFFu) continue;
                    if (!(c[u] <= cutoff)) continue;      // round-0 seeds above a max-active cutoff
                    c_front++;
                    if (LAT) {
                        const double m = rld_f64(L.msnap + v[u]);
                        if (c[u] < m) rst_f64(L.msnap + v[u], c[u]);
                    }
                    c_escan += er[u].y - er[u].x;
                    for (unsigned e = er[u].x; e < er[u].y; ++e) {
                        const int4 rr = gld4(g.eps + e);
                        const double cand = __dadd_rn(c[u], __hiloint2double(rr.w, rr.z));
                        if (!(cand <= cutoff)) continue;
                        c_ecand++;
                        const unsigned x = (unsigned)rr.x;
                        const unsigned long long word = pack_word(cand, (unsigned)rr.y);
                        const unsigned long long old = atom_min_u64(pk + x, word);
                        if (old == SENT) {   // first reached by epsilon this frame
                            const int sl = agg_append(netouched);
                            __stcg(etl + sl, x);
                        }
                        if (old > word) {
#ifdef LB_EPS_TAG
                            // tag exchange issued before the winner CAS: both in flight together
                            const unsigned tg = atom_exch_u32(L.tag + x, round_id);
                            epswin_min(rcur + x, word, cand);
                            const bool first = tg != round_id;
#else
                            // the round's first improving offer to x (its CAS replaced
                            // the idle round winner) lists x in the next frontier
                            const bool first = epswin_min_first(rcur + x, word, cand);
#endif
                            if (first) {
                                const int sl = agg_append(nnext);
                                __stcg(fsn + sl, x);
                            }
                        }
                    }
                }
                if (r > 0) {
#pragma unroll
                    for (int u = 0; u < EUNR; u++)
                        if (v[u] != 0xFFFFFFFFu)
                            rst_u128(L.erec + v[u], make_ulonglong2((unsigned long long)__double_as_longlong(c[u]),
                                                                    (unsigned long long)(unsigned)(src[u] << 1)));
                }
            }
            wend(3, t0);
            G.sync();
        }
        c_escan = warp_sum(c_escan);
        c_ecand = warp_sum(c_ecand);
        c_front = warp_sum(c_front);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&lane_sm.c_escan, (unsigned long long)c_escan);
            atomicAdd(&lane_sm.c_ecand, (unsigned long long)c_ecand);
            atomicAdd(&lane_sm.c_front, (unsigned long long)c_front);
        }
        // (unchanged when no round ran: then no barrier separates this from the
        // read at the top, so only a changed value is written)
        if (threadIdx.x == 0 && round_id != round_id0) lane_sm.round_id = round_id;
        if (!ok) G.sync();
        return ok;
    }

    // ---- aggregate + reset: frame token list at io.tok_*[tb ...]; returns count or -1 ----
    // Warp-uniform loop over this CTA's emitting winners (payload read
    // coalesced) and then its epsilon-reached states.  ONE scattered access per
    // state does both the read of the final word and its reset (atom.exch to
    // SENT).  A winner whose word survived keeps its payload; a state whose
    // word an epsilon offer improved takes its cost / predecessor from `erec`.
    // Kept states are staged per warp; a stage flush takes lane-wide token
    // indices in bulk (one DSMEM counter atomic per flush), writes the token
    // records coalesced and the states' token indices.  Tokens whose
    // predecessor is an epsilon source STATE go to this CTA's fix list;
    // fix_preds() maps them to token indices during the next frame's emit.
    struct TokStage {
        double *cost;
        unsigned *v, *arc, *key;
        int *pred;
        int n;
    };
    __device__ __forceinline__ TokStage tok_stage() const {
        char *b = scratch();
        TokStage t;
        t.cost = reinterpret_cast<double *>(b);
        t.v = reinterpret_cast<unsigned *>(t.cost + SWT);
        t.arc = t.v + SWT;
        t.key = t.arc + SWT;
        t.pred = reinterpret_cast<int *>(t.key + SWT);
        t.n = 0;
        return t;
    }
    __device__ __forceinline__ WStage fix_stage() const {
        WStage st;
        st.buf = reinterpret_cast<unsigned *>(scratch() + SWT * 32);
        st.n = 0;
        return st;
    }

    __device__ void flush_tokens(TokStage &st, WStage &sf, int frame, long long tb, long long room) {
        __syncwarp();
        if (st.n == 0) return;
        const int lane = threadIdx.x & 31;
        int base = 0;
        if (lane == 0) base = atomicAdd(&G.M->ntok[par], st.n);
        base = __shfl_sync(FULL, base, 0);
        for (int i0 = 0; i0 < st.n; i0 += 32) {
            const int i = i0 + lane;
            bool fx = false;
            const int idx = base + i;
            if (i < st.n && idx < room) {
                const unsigned v = st.v[i];
                const bool init = frame == 0 && (int)v == g.start;
                const double c = st.cost[i];
                const int pr = st.pred[i];
                const long long o = tb + idx;
                __stcg(io.tok_state + o, v);
                __stcg(io.tok_cost + o, init ? 0.0 : c);
                __stcs(io.tok_arc + o, init ? -1 : (int)st.arc[i]);
                __stcs(io.tok_pred + o, init ? -1 : pr);
                if (p.collect_packs)
                    __stcs(io.tok_pack + o, ((unsigned long long)st.key[i] << 32) | st.arc[i]);
                rst_i32(L.tokidx + v, idx);
                fx = !init && (pr & 1) == 0;
            }   // over the arena: the error is raised after the barrier (the word is already reset)
            sf.push(fx, (unsigned)idx, &lane_sm.nfix[par], fixes());
        }
        __syncwarp();
        st.n = 0;
    }

    __device__ int aggregate(double cutoff, int frame, long long tb) {
        // k in [0, nb): list B (final seeds, no exchange), [nb, nb + nt): list A,
        // then the epsilon-reached states
        const int nb = lane_sm.nfinal[par], nt = nb + lane_sm.ntouched[par];
        const int ne = lane_sm.netouched[par], ntot = nt + ne;
        const long long room = io.tok_cap - tb;
        unsigned long long *pk = L.pk;
        const unsigned *tl = touched(), *etl = etouched();
        const size_t cs = cseg();
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        const unsigned lt = (1u << lane) - 1u;
        TokStage st = tok_stage();
        WStage sf = fix_stage();
        const unsigned long long t0 = wbegin();
        // the next batch's list entries (and winner payloads) are fetched one batch ahead
        auto fetch = [&](int k, unsigned &v, unsigned &a, int &pr, double &c) {
            v = 0;
            a = 0;
            pr = 0;
            c = 0.0;
            if (k < nt) {
                const size_t o = k < nb ? (size_t)L.ccap - 1 - (size_t)k : (size_t)(k - nb);
                v = PAY_LD(tl + o);
                a = PAY_LD(L.tarc + cs + o);
                pr = PAY_LD(L.tpred + cs + o);
                c = PAY_LD(L.tcost + cs + o);
            } else if (k < ntot) {
                v = __ldcg(etl + (k - nt));
            }
        };
        unsigned vn, an;
        int prn;
        double cn;
        fetch(warp * 32 + lane, vn, an, prn, cn);
        for (int kb = warp * 32; kb < ntot; kb += nw * 32) {
            const int k = kb + lane;
            const bool valid = k < ntot, win = k < nt, fin = k < nb;
            unsigned v = vn, a = an;
            int pr = prn;
            double c = cn;
            fetch(k + nw * 32, vn, an, prn, cn);
            // read the final word and reset it in one atomic (issuing the next
            // batch's exchanges a batch ahead measured no faster); a final seed's
            // word is its own and was reset in winners
            const unsigned long long x = fin ? pack_word(c, a) : valid ? atom_exch_u64(pk + v, SENT) : SENT;
            if (valid && (!win || x != pack_word(c, a))) {   // improved by an epsilon offer
                const ulonglong2 er = rld_u128(L.erec + v);
                c = __longlong_as_double((long long)er.x);
                pr = (int)(unsigned)er.y;
                a = (unsigned)x;
            }
            const bool init = valid && frame == 0 && (int)v == g.start;
            const bool keep = valid && (init || c <= cutoff);
            const unsigned m = __ballot_sync(FULL, keep);
            if (keep) {
                const int j = st.n + __popc(m & lt);
                st.v[j] = v;
                st.cost[j] = c;
                st.arc[j] = a;
                st.key[j] = (unsigned)(x >> 32);
                st.pred[j] = pr;
            }
            st.n += __popc(m);
            if (st.n > SWT - 32) flush_tokens(st, sf, frame, tb, room);
        }
        flush_tokens(st, sf, frame, tb, room);
        sf.flush(&lane_sm.nfix[par], fixes());
        wend(4, t0);
        G.sync();
        const int n = G.M->ntok[par];
        if (n == 0 || (long long)n > p.max_tokens || (long long)n > room) {
            if (G.leader()) {
                if (n == 0) set_error(E_DEAD_NO_TOKENS, frame, 0);
                else if ((long long)n > p.max_tokens) set_error(E_CAP_TOKENS, frame, n);
                else set_error(E_CAP_ARENA, frame, tb + n);
            }
            G.sync();
            return -1;
        }
        return n;
    }

    __device__ __forceinline__ void lat_push(int arc, int from, int to, long long lb) {
        const int sl = agg_append(&G.M->nlat[par]);
        const long long gs = lb + sl;
        if (gs < io.lat_cap) {
            __stcg(io.lat_arc + gs, arc);
            __stcg(io.lat_from + gs, from);
            __stcg(io.lat_to + gs, to);
        }
    }

    __device__ __forceinline__ bool kept(unsigned v, long long tb, int n, int &j) const {
        j = rld_i32(L.tokidx + v);
        return j >= 0 && j < n && __ldcg(io.tok_state + tb + j) == v;
    }

    // ---- lattice arcs of block `frame` (rule A.5); resets minsnap; returns arc count or -1 ----
    __device__ int lattice(double cutoff, int frame, long long tbp, int np, long long tb, int n,
                           long long lb) {
        if (frame > 0) {
            unsigned dummy = 0;
            for_each_token_arc_batched<UNR>(g, G.gwarp(), G.gnw(), io.tok_state + tbp, io.tok_cost + tbp, np, dummy, wmap(),
                                            [&](const bool *vv, const int *ii, const unsigned *aa, const double *cc) {
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    if (!vv[u]) continue;
                    const int4 r = __ldg(g.arcs + aa[u]);
                    const unsigned il = arc_il(r.y);
                    if (il == 0) continue;
                    const double w = __hiloint2double(r.w, r.z);
                    const double cand = __dadd_rn(__dadd_rn(cc[u], w), ac(il));
                    int j;
                    if (cand <= cutoff && kept((unsigned)r.x, tb, n, j)) lat_push((int)aa[u], ii[u], j, lb);
                }
            });
        }
        if (g.has_eps) {
            const double inf = inf_d();
            for (int j = G.gtid(); j < n; j += G.gstride()) {
                const unsigned u = __ldcg(io.tok_state + tb + j);
                const unsigned e0 = __ldg(g.eoff + u), e1 = __ldg(g.eoff + u + 1);
                const double ms = rld_f64(L.msnap + u);
                if (ms < inf) rst_f64(L.msnap + u, inf);
                for (unsigned e = e0; e < e1; ++e) {
                    const int4 r = __ldg(g.eps + e);
                    int jv;
                    if (__dadd_rn(ms, __hiloint2double(r.w, r.z)) <= cutoff && kept((unsigned)r.x, tb, n, jv))
                        lat_push(r.y, j, jv, lb);
                }
            }
        }
        G.sync();
        const int nl = G.M->nlat[par];
        if (lb + nl > io.lat_cap) {
            if (G.leader()) set_error(E_CAP_LATTICE, frame, lb + nl);
            G.sync();
            return -1;
        }
        return nl;
    }

    // ---- error path: O(touched) reset of every per-state word this frame touched ----
    __device__ void reset_touched() {
        G.sync();
        const int nb = lane_sm.nfinal[par], nt = lane_sm.ntouched[par], ne = lane_sm.netouched[par];
        const unsigned *tl = touched(), *etl = etouched();
        const double inf = inf_d();
        for (int k = threadIdx.x; k < nb + nt + ne; k += blockDim.x) {
            const unsigned v = k < nb ? __ldcg(tl + L.ccap - 1 - k)
                             : k < nb + nt ? __ldcg(tl + (k - nb)) : __ldcg(etl + (k - nb - nt));
            rst_u64(L.pk + v, SENT);
            rst_f64(L.msnap + v, inf);
            rst_u128(rpk(0) + v, make_ulonglong2(~0ull, ~0ull));
            rst_u128(rpk(1) + v, make_ulonglong2(~0ull, ~0ull));
        }
        G.sync();
    }
};

__device__ __forceinline__ void init_smem(unsigned round_ctr) {
    Smem &sm = lane_sm;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; q++) {
            sm.ntok[q] = sm.nlat[q] = 0;
            sm.ntouched[q] = sm.ncand[q] = sm.nseed[q] = sm.nfix[q] = sm.netouched[q] = 0;
            sm.nfinal[q] = 0;
            sm.best[q] = SENT;
        }
        sm.nfr[0] = sm.nfr[1] = sm.nfr[2] = 0;
        sm.err = sm.err_frame = 0;
        sm.err_aux = 0;
        sm.round_id = round_ctr;
        sm.ready_seen = 0;
        sm.c_tok = sm.c_scan = sm.c_cand = sm.c_front = sm.c_escan = sm.c_ecand = sm.c_next = 0;
    }
}

// Seed the start state (frame 0, decoder.py:510-513) into the rank-0 CTA's lists.
template <int UNR>
__device__ __forceinline__ void seed_start(Lane<UNR> &ln, const GraphDev &g, const LaneWs &L) {
    if (ln.G.leader()) {
        __stcg(L.pk + g.start, pack_word(0.0, 0u));
        const size_t k = 0;   // the rank-0 CTA's first emitting-winner slot
        __stcg(L.touched + k, (unsigned)g.start);
        __stcg(L.tcost + k, 0.0);
        __stcg(L.tpred + k, -1);
        __stcg(L.tarc + k, 0u);
        lane_sm.ntouched[0] = 1;
        if (g.has_eps) {
            __stcg(ln.front(0), (unsigned)g.start);
            __stcg(L.f0cost + k, 0.0);
            lane_sm.nfr[0] = 1;
        }
    }
}

// ===========================================================================
// Full-utterance decode of one job on one lane (a cluster).  Cluster barriers
// per frame: emit 1, winners 1, epsilon 1 per round, aggregate 1-2, lattice 1.
// `io` is the CTA's shared-memory descriptor of the job: the lane's arenas plus
// the job's costs, length and output slots.
// ===========================================================================
template <int UNR, bool LAT, bool PROF>
__device__ __forceinline__ void decode_one(const GraphDev &g, const Params &p, const LaneWs &L,
                                           const UttDesc &io, const Grp &G) {
    Smem &sm = lane_sm;
    Lane<UNR> ln(g, p, L, io, G, lane_dyn);
    if (PROF) ln.wprof = p.prof + 8;
    const int T = io.T;
    const double inf = inf_d();
    long long tb = 0, lb = 0;
    int ntok = 0, tdone = 0;

    // optional phase profile: leader accumulates globaltimer deltas per phase
    unsigned long long t_last = 0;
    auto mark = [&](int ph) {
        if (PROF && G.leader()) {
            const unsigned long long t = gtimer();
            if (ph >= 0) atomicAdd(p.prof + ph, t - t_last);
            t_last = t;
        }
    };
    mark(-1);
    double beam_eff = p.beam;   // adaptive beam; == beam without max-active

    // ---- frame 0 (decoder.py:510-523): start token, epsilon closure ----
    ln.par = 0;
    seed_start(ln, g, L);
    if (G.leader()) {
        io.tok_base[0] = 0;
        if (LAT) io.lat_base[0] = 0;
    }
    G.sync();
    double cutoff = __dadd_rn(0.0, p.beam);
    bool ok = ln.epsilon(cutoff, 0);
    bool reset_done = false;
    if (ok) {
        ntok = ln.aggregate(cutoff, 0, tb);
        reset_done = true;
        ok = ntok > 0;
    }
    if (LAT && ok) {
        const int nl = ln.lattice(cutoff, 0, 0, 0, tb, ntok, lb);
        ok = nl >= 0;
        if (ok) lb += nl;
    }
    if (G.leader()) {
        io.tok_base[1] = tb + (ok ? ntok : 0);
        if (LAT) io.lat_base[1] = lb;
    }
    if (!reset_done) ln.reset_touched();
    mark(7);

    for (int t = 1; ok && t <= T; t++) {
        const long long tbp = tb;
        const int np = ntok;
        tb += ntok;
        if (G.leader()) sm.c_tok += np;
        ln.par = t & 1;
        reset_done = false;
        if (p.row_pf) {   // row t-1 was requested during frame t-1 (or now, at t = 1)
            if (t == 1) ln.row_async(io.costs, 0);
            ln.row_finish((t - 1) & 1);
            if (t < T) ln.row_async(io.costs + (long long)t * p.D, t & 1);
        } else {
            ln.load_row(p.costs_f32 ? reinterpret_cast<const double *>(reinterpret_cast<const float *>(io.costs) +
                                                                       (long long)(t - 1) * p.D)
                                    : io.costs + (long long)(t - 1) * p.D,
                        t - 1);
        }
        if (g.has_eps) ln.fix_preds((t - 1) & 1, t - 1, tbp, np);
        __syncthreads();
        const double best = ln.emit(io.tok_state + tbp, io.tok_cost + tbp, np, beam_eff, t);
        ln.clear_next_counters();   // frame t-1's readers are past the emit barrier
        mark(0);
        if (!(best < inf)) {
            if (G.leader()) ln.set_error(E_DEAD_NO_CAND, t, 0);
            ok = false;
            break;
        }
        if (G.M->err) { ok = false; break; }   // candidate buffer overflow (never by construction)
        cutoff = __dadd_rn(best, beam_eff);
        ln.winners(cutoff, best);
        G.sync();
        mark(1);
        const int nf = ln.lane_seeds();
        if (nf == 0) {
            if (G.leader()) ln.set_error(E_DEAD_NO_TOKENS, t, 0);
            ok = false;
            break;
        }
        bool tightened = false;
        if (p.max_active > 0 && nf > p.max_active) {
            const double c2 = ln.max_active_cutoff(cutoff, best);
            if (c2 < cutoff) {
                tightened = true;
                cutoff = c2;
            }
        }
        // Kaldi's adaptive beam: after a max-active tightening the next frame's beam
        // is (cutoff - best) + beam_delta, capped at beam; otherwise the full beam.
        if (tightened) {
            const double be = __dadd_rn(__dsub_rn(cutoff, best), MAX_ACTIVE_BEAM_DELTA);
            beam_eff = be < p.beam ? be : p.beam;
        } else {
            beam_eff = p.beam;
        }
        mark(2);
        if (g.has_eps) {
            ok = ln.epsilon(cutoff, t);
            if (!ok) break;
        }
        mark(3);
        ntok = ln.aggregate(cutoff, t, tb);
        reset_done = true;
        mark(4);
        if (ntok < 0) { ok = false; break; }
        if (G.leader()) sm.c_next += ntok;
        if (LAT) {
            const int nl = ln.lattice(cutoff, t, tbp, np, tb, ntok, lb);
            if (nl < 0) { ok = false; break; }
            lb += nl;
        }
        mark(5);
        if (G.leader()) {
            io.tok_base[t + 1] = tb + ntok;
            if (LAT) io.lat_base[t + 1] = lb;
        }
        mark(6);
        tdone = t;
    }
    if (!ok && !reset_done) ln.reset_touched();
    if (ok && g.has_eps) ln.fix_preds(T & 1, T, tb, ntok);   // the last frame's epsilon predecessors
    G.sync();

    // ---- counters: per-CTA partials merged through DSMEM ----
    if (G.leader()) {
        unsigned long long cs = 0, cc = 0, cf = 0, ces = 0, cec = 0;
        for (int q = 0; q < G.C; q++) {
            const Smem *R = G.at(q);
            cs += R->c_scan;
            cc += R->c_cand;
            cf += R->c_front;
            ces += R->c_escan;
            cec += R->c_ecand;
        }
        io.out_c[0] = (long long)sm.c_tok;
        io.out_c[1] = (long long)cs;
        io.out_c[2] = (long long)cc;
        io.out_c[3] = (long long)cf;
        io.out_c[4] = (long long)ces;
        io.out_c[5] = (long long)cec;
        io.out_c[6] = (long long)sm.c_next;
        io.out_c[7] = lb;
        io.out_i[5] = tdone;
    }
    const int err = G.M->err;
    if (!ok || err) {
        if (G.leader()) {
            io.out_i[0] = err ? err : E_INT_INIT;
            io.out_i[1] = sm.err_frame;
            io.out_d[2] = (double)sm.err_aux;
        }
        G.sync();
        return;
    }

    // ---- final selection (decoder.py:578-586): argmin, ties -> smallest state ----
    double bt = inf, bc = inf;
    int st = 0x7FFFFFFF, sc = 0x7FFFFFFF;
    for (int j = G.gtid(); j < ntok; j += G.gstride()) {
        const unsigned s = __ldcg(io.tok_state + tb + j);
        const double c = __ldcg(io.tok_cost + tb + j);
        const double tot = __dadd_rn(c, __ldg(g.fin + s));
        if (tot < bt || (tot == bt && (int)s < st)) { bt = tot; st = (int)s; }
        if (c < bc || (c == bc && (int)s < sc)) { bc = c; sc = (int)s; }
    }
    cl_argmin(bt, st, G);
    cl_argmin(bc, sc, G);
    const bool partial = !(bt < inf);
    const int bstate = partial ? sc : st;
    if (G.leader()) {
        const double total = partial ? bc : bt;
        const int bidx = __ldcg(L.tokidx + bstate);
        io.out_i[2] = partial;
        io.out_i[3] = bidx;
        io.out_d[0] = total;
        io.out_d[1] = total;
        // ---- backtrace (decoder.py:614-641), bounded ----
        int f = T, i = bidx, hops = 0, e = 0;
        long long steps = 0;
        const long long limit = tb + ntok + 1;
        for (;;) {
            const long long base = io.tok_base[f];
            const int a = __ldcg(io.tok_arc + base + i);
            const int pr = __ldcg(io.tok_pred + base + i);
            if (a < 0) {
                if (f != 0) e = E_INT_INIT;
                break;
            }
            if (hops >= io.path_cap) { e = E_CAP_PATH; break; }
            io.path[hops++] = a;
            i = pr >> 1;
            if (pr & 1) f--;
            if (++steps > limit) { e = E_INT_BACKTRACE; break; }
        }
        for (int k = 0; k < hops / 2; k++) {
            const int x = io.path[k];
            io.path[k] = io.path[hops - 1 - k];
            io.path[hops - 1 - k] = x;
        }
        io.out_i[4] = hops;
        io.out_i[0] = e;
        io.out_i[1] = e ? f : 0;
    }
    mark(7);
    G.sync();
}

// Per-CTA shared copy of the current job's descriptor (lane arenas + job fields).
__shared__ UttDesc lane_io;
__shared__ int lane_job;

// ===========================================================================
// Persistent decode lanes: one cluster per lane.  With a queue, a lane claims
// jobs from the device counter (jobs are in longest-first order, the host's
// LPT sort) and refills itself the moment it finishes one, as the reference's
// decode_batch pool starts the next utterance when a worker frees up
// (decoder.py:666-672); without one, lane l decodes job l (lattice waves).
// ===========================================================================
template <int NT, int UNR, bool LAT, bool PROF>
__global__ void __launch_bounds__(NT, 1)
decode_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
              const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ slots,
              const UttJob *__restrict__ jobs, int n_jobs, int *queue) {
    Smem &sm = lane_sm;
    cgx::cluster_group cl = cgx::this_cluster();
    Grp G;
    G.C = (int)cl.num_blocks();
    G.rank = (int)cl.block_rank();
    G.M = cl.map_shared_rank(&sm, 0);
    const int lane = blockIdx.x / G.C;      // uniform across the cluster
    const LaneWs &L = lanes[lane];
    unsigned round_id = __ldcg(L.round_ctr);
    int ready_seen = 0;
    for (int it = 0;; it++) {
        if (queue) {
            if (G.leader()) lane_job = atomicAdd(queue, 1);
            G.sync();
            const int j = *cl.map_shared_rank(&lane_job, 0);
            G.sync();   // every CTA has read the claim before the next one
            if (threadIdx.x == 0) lane_job = j;
        } else if (threadIdx.x == 0) {
            lane_job = it == 0 ? lane : n_jobs;
        }
        __syncthreads();
        const int j = lane_job;
        if (j >= n_jobs) break;
        if (p.ring_ready) {   // streamed host rows: wait until job j is staged
            if (threadIdx.x == 0) {
                int r;
                for (;;) {
                    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(r) : "l"(p.ring_ready) : "memory");
                    if (r > j) break;
                    __nanosleep(2000);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            UttDesc d = slots[lane];
            const UttJob &J = jobs[j];
            d.costs = p.ring_ready ? p.ring_base + (long long)(j % p.ring_slots) * p.ring_slot_doubles : J.costs;
            d.T = J.T;
            d.path = J.path;
            d.out_i = J.out_i;
            d.out_d = J.out_d;
            d.out_c = J.out_c;
            lane_io = d;
            init_smem(round_id);
            sm.ready_seen = ready_seen;
        }
        G.sync();
        decode_one<UNR, LAT, PROF>(g, p, L, lane_io, G);
        round_id = sm.round_id;
        ready_seen = sm.ready_seen;
        if (p.ring_ready) {
            // Hand the slot back: drop its lines from L2 (the host rewrites the
            // slot for job j + ring_slots, and a stale line must not survive),
            // then publish with a system-scope release.
            const char *base = reinterpret_cast<const char *>(lane_io.costs);
            const long long lines = ((long long)lane_io.T * p.D * 8 + 127) / 128;
            for (long long q = G.gtid(); q < lines; q += G.gstride())
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + q * 128) : "memory");
            G.sync();
            if (G.leader()) {
                asm volatile("fence.sc.sys;" ::: "memory");
                asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p.ring_done + (j % p.ring_slots)), "r"(j + 1)
                             : "memory");
            }
        }
    }
    if (G.leader()) __stcg(L.round_ctr, round_id);
    G.sync();   // keep rank 0's shared memory alive until every CTA is done with it
}

// largest b with base[b] <= k (base has nb non-decreasing entries)
__device__ __forceinline__ int upper_block(const long long *base, int nb, long long k) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= k) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ===========================================================================
// Lattice extra-cost pruning (lattice.py:365-497) from the final terminus, one
// thread-block cluster per utterance (cluster size chosen by the host so the
// whole GPU works even for one utterance): backward over frames, emitting arcs
// relax node extras with a 64-bit atomicMin on the order-preserving f64
// encoding, the in-frame epsilon fixpoint runs Jacobi iterations, then every
// arc is flagged.  Phases of a frame meet at cluster barriers.
// ===========================================================================
__global__ void __launch_bounds__(1024, 1)
prune_kernel(GraphDev g, Params p, const UttDesc *__restrict__ utts, int n_utts) {
    __shared__ int s_moved;
    cgx::cluster_group cl = cgx::this_cluster();
    const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int u = blockIdx.x / C;
    if (u >= n_utts) return;
    const UttDesc io = utts[u];
    if (io.out_i[0] != E_OK) return;   // uniform across the cluster
    int *m0 = cl.map_shared_rank(&s_moved, 0);
    const int tid = rank * blockDim.x + threadIdx.x, bd = C * blockDim.x;
    const int T = io.T;
    const bool partial = io.out_i[2] != 0;
    const double best_total = io.out_d[1];
    const double inf = inf_d();
    const int D = p.D;
    for (int f = T; f >= 0; f--) {
        const long long b0 = io.tok_base[f];
        const int nfr = (int)(io.tok_base[f + 1] - b0);
        unsigned long long *ne = io.ne_enc + b0;
        const double *fwd = io.tok_cost + b0;
        if (f == T) {
            for (int i = tid; i < nfr; i += bd) {
                const unsigned s = __ldcg(io.tok_state + b0 + i);
                const double x = partial ? 0.0 : __dsub_rn(__dadd_rn(__ldcg(fwd + i), __ldg(g.fin + s)), best_total);
                __stcg(ne + i, enc64(x));
            }
            cl.sync();
        } else {
            for (int i = tid; i < nfr; i += bd) __stcg(ne + i, enc64(inf));
            cl.sync();
            const long long b1 = io.tok_base[f + 1];
            const double *fwdn = io.tok_cost + b1;
            const double *nen = io.node_extra + b1;
            const double *row = io.costs + (long long)f * D;
            for (long long k = io.lat_base[f + 1] + tid; k < io.lat_base[f + 2]; k += bd) {
                const unsigned a = (unsigned)__ldcg(io.lat_arc + k);
                unsigned dst, il;
                double w;
                load_arc(g.arcs, a, dst, il, w);
                if (il == 0) continue;
                const int from = __ldcg(io.lat_from + k), to = __ldcg(io.lat_to + k);
                const double acv = __dmul_rn(__ldg(row + il - 1), p.scale);
                const double c = __dadd_rn(__dsub_rn(__dadd_rn(__dadd_rn(__ldcg(fwd + from), w), acv), __ldcg(fwdn + to)),
                                           __ldcg(nen + to));
                atom_min_u64(ne + from, enc64(c));
            }
            cl.sync();
        }
        // in-frame epsilon fixpoint (lattice.py:455-469)
        if (g.has_eps) {
            const long long k0 = io.lat_base[f], k1 = io.lat_base[f + 1];
            for (int it = 0;; it++) {
                if (rank == 0 && threadIdx.x == 0) s_moved = 0;
                cl.sync();
                for (long long k = k0 + tid; k < k1; k += bd) {
                    const unsigned a = (unsigned)__ldcg(io.lat_arc + k);
                    unsigned dst, il;
                    double w;
                    load_arc(g.arcs, a, dst, il, w);
                    if (il != 0) continue;
                    const int from = __ldcg(io.lat_from + k), to = __ldcg(io.lat_to + k);
                    const double base = __dsub_rn(__dadd_rn(__ldcg(fwd + from), w), __ldcg(fwd + to));
                    const double c = __dadd_rn(base, dec64(__ldcg(ne + to)));
                    const double before = dec64(__ldcg(ne + from));
                    __stcg(io.tmp + k, c);
                    if (__dsub_rn(before, c) > CONVERGE_TOL) *m0 = 1;
                }
                cl.sync();
                for (long long k = k0 + tid; k < k1; k += bd) {
                    const unsigned a = (unsigned)__ldcg(io.lat_arc + k);
                    if (arc_il(__ldg(g.arcs + a).y) != 0) continue;
                    atom_min_u64(ne + __ldcg(io.lat_from + k), enc64(__ldcg(io.tmp + k)));
                }
                cl.sync();
                const int moved = *m0;
                cl.sync();
                if (!moved) break;
                if (it >= nfr) {
                    if (tid == 0) io.out_i[0] = E_INT_PRUNE_EPS, io.out_i[1] = f;
                    return;
                }
            }
        }
        for (int i = tid; i < nfr; i += bd) {
            const double x = dec64(__ldcg(ne + i));
            __stcg(io.node_extra + b0 + i, x < 0.0 ? 0.0 : x);
        }
        cl.sync();
    }
    // flag pass (lattice.py:473-497): every arc's extra, all blocks at once
    const long long nl = io.lat_base[T + 1];
    for (long long k = tid; k < nl; k += bd) {
        const int b = upper_block(io.lat_base, T + 2, k);
        const long long tbb = io.tok_base[b];
        const unsigned a = (unsigned)__ldcg(io.lat_arc + k);
        unsigned dst, il;
        double w;
        load_arc(g.arcs, a, dst, il, w);
        const int from = __ldcg(io.lat_from + k), to = __ldcg(io.lat_to + k);
        const long long fb = il > 0 ? io.tok_base[b - 1] : tbb;
        const double acv = il > 0 ? __dmul_rn(__ldg(io.costs + (long long)(b - 1) * D + il - 1), p.scale) : 0.0;
        const double x = __dadd_rn(__dsub_rn(__dadd_rn(__dadd_rn(__ldcg(io.tok_cost + fb + from), w), acv),
                                             __ldcg(io.tok_cost + tbb + to)),
                                   __ldcg(io.node_extra + tbb + to));
        __stcg(io.lat_extra + k, x < 0.0 ? 0.0 : x);
    }
}

// ===========================================================================
// prune_lattice single-op surface (lattice.py:365-497) over an arbitrary work
// lattice handed in by the host: frames 0..t of token costs, blocks 0..t of
// arcs with their status (LIVE 0 / PRUNED 1; pruned arcs stay pruned and do
// not participate), graph / acoustic costs and an emitting flag.  Same
// relaxation as prune_kernel (one cluster, backward over frames, 64-bit
// atomicMin on the order-preserving f64 key, Jacobi in-frame epsilon
// fixpoint, clamp at 0), from the given terminus; then every LIVE arc of
// blocks 0..t gets its extra and is flagged PRUNED when extra > lattice_beam.
// ===========================================================================
struct PruneOp {
    int t;
    int err;                          // out: E_INT_PRUNE_EPS frame + 1, or 0
    const long long *tok_base;        // [t+2]
    const double *fwd;                // token forward costs, frames 0..t
    const long long *lat_base;        // [t+2]
    const int *from, *to;
    const unsigned char *emit;
    const double *g, *ac, *terminus;
    unsigned char *status;
    double *extra, *node_extra, *tmp;
    unsigned long long *ne;
    int *err_out;
    double beam;
};

__global__ void __launch_bounds__(1024, 1) prune_op_kernel(const __grid_constant__ PruneOp op) {
    __shared__ int s_moved;
    cgx::cluster_group cl = cgx::this_cluster();
    const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    int *m0 = cl.map_shared_rank(&s_moved, 0);
    const int tid = rank * blockDim.x + threadIdx.x, bd = C * blockDim.x;
    const double inf = inf_d();
    for (int f = op.t; f >= 0; f--) {
        const long long b0 = op.tok_base[f];
        const int nfr = (int)(op.tok_base[f + 1] - b0);
        unsigned long long *ne = op.ne + b0;
        const double *fwd = op.fwd + b0;
        for (int i = tid; i < nfr; i += bd) __stcg(ne + i, enc64(f == op.t ? op.terminus[i] : inf));
        cl.sync();
        if (f < op.t) {
            const long long b1 = op.tok_base[f + 1];
            for (long long k = op.lat_base[f + 1] + tid; k < op.lat_base[f + 2]; k += bd) {
                if (op.status[k] != 0 || !op.emit[k]) continue;
                const int from = op.from[k], to = op.to[k];
                const double c = __dadd_rn(__dsub_rn(__dadd_rn(__dadd_rn(fwd[from], op.g[k]), op.ac[k]),
                                                     op.fwd[b1 + to]),
                                           op.node_extra[b1 + to]);
                atom_min_u64(ne + from, enc64(c));
            }
            cl.sync();
        }
        const long long k0 = op.lat_base[f], k1 = op.lat_base[f + 1];
        for (int it = 0;; it++) {
            if (rank == 0 && threadIdx.x == 0) s_moved = 0;
            cl.sync();
            for (long long k = k0 + tid; k < k1; k += bd) {
                if (op.status[k] != 0 || op.emit[k]) continue;
                const int from = op.from[k], to = op.to[k];
                const double base = __dsub_rn(__dadd_rn(fwd[from], op.g[k]), fwd[to]);
                const double c = __dadd_rn(base, dec64(__ldcg(ne + to)));
                const double before = dec64(__ldcg(ne + from));
                __stcg(op.tmp + k, c);
                if (__dsub_rn(before, c) > CONVERGE_TOL) *m0 = 1;
            }
            cl.sync();
            for (long long k = k0 + tid; k < k1; k += bd) {
                if (op.status[k] != 0 || op.emit[k]) continue;
                atom_min_u64(ne + op.from[k], enc64(__ldcg(op.tmp + k)));
            }
            cl.sync();
            const int moved = *m0;
            cl.sync();
            if (!moved) break;
            if (it >= nfr) {
                if (tid == 0) *op.err_out = f + 1;
                return;
            }
        }
        for (int i = tid; i < nfr; i += bd) {
            const double x = dec64(__ldcg(ne + i));
            __stcg(op.node_extra + b0 + i, x < 0.0 ? 0.0 : x);
        }
        cl.sync();
    }
    const long long nl = op.lat_base[op.t + 1];
    for (long long k = tid; k < nl; k += bd) {
        if (op.status[k] != 0) continue;
        const int b = upper_block(op.lat_base, op.t + 2, k);
        const long long tbb = op.tok_base[b];
        const long long fb = op.emit[k] ? op.tok_base[b - 1] : tbb;
        const double x = __dadd_rn(__dsub_rn(__dadd_rn(__dadd_rn(op.fwd[fb + op.from[k]], op.g[k]), op.ac[k]),
                                             op.fwd[tbb + op.to[k]]),
                                   op.node_extra[tbb + op.to[k]]);
        const double e = x < 0.0 ? 0.0 : x;
        op.extra[k] = e;
        if (e > op.beam) op.status[k] = 1;
    }
}

// ===========================================================================
// Single-op surfaces (decoder.py:373-435), one CTA (a cluster of one).
//   mode 0 = expand_emitting: tokens at io.tok_*[0..n); acrow (scaled) at
//            io.costs; writes winners <= cutoff to io.tok_state/tok_cost[n ...].
//   mode 1 = expand_nonemitting: seeds at io.tok_*[0..n) act as won entries
//            pack(cost, 0); closes under `cutoff`; writes the merged frontier.
// ===========================================================================
__global__ void __launch_bounds__(768, 1)
expand_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
              const __grid_constant__ LaneWs L, const __grid_constant__ UttDesc io, int n, int mode,
              double cutoff_in) {
    Smem &sm = lane_sm;
    Grp G;
    G.C = 1;
    G.rank = 0;
    G.M = cgx::this_cluster().map_shared_rank(&sm, 0);
    const int tid = threadIdx.x;
    init_smem(__ldcg(L.round_ctr));
    __syncthreads();
    Lane<2> ln(g, p, L, io, G, lane_dyn);
    double cutoff = cutoff_in;
    ln.par = 1;
    if (mode == 0) {
        ln.load_row(io.costs, 0);
        __syncthreads();
        const double best = ln.emit(io.tok_state, io.tok_cost, n, p.beam, 1);
        if (!(best < inf_d())) {
            cutoff = inf_d();
        } else {
            cutoff = __dadd_rn(best, p.beam);
            ln.winners(cutoff, best);
        }
    } else {
        for (int i = tid; i < n; i += blockDim.x) {
            const unsigned s = __ldcg(io.tok_state + i);
            const double c = __ldcg(io.tok_cost + i);
            __stcg(L.pk + s, pack_word(c, 0u));
            __stcg(L.touched + i, s);
            __stcg(L.tcost + i, c);
            __stcg(L.tarc + i, 0u);
            __stcg(L.tpred + i, -1);
            __stcg(ln.front(0) + i, s);
            __stcg(L.f0cost + i, c);
        }
        __syncthreads();
        if (tid == 0) { sm.ntouched[1] = n; sm.nfr[0] = n; }
        __syncthreads();
        if (!ln.epsilon(cutoff, 0)) {
            if (tid == 0) io.out_i[0] = sm.err;
        }
    }
    __syncthreads();
    // the closure's states: emitting winners / seeds with their payload, then the
    // epsilon-reached ones; the final word says whether epsilon improved a state
    // (list B first: final seeds whose words winners already reset)
    const int nb = sm.nfinal[1], nt = nb + sm.ntouched[1], ne = sm.netouched[1];
    const unsigned *tl = ln.touched(), *etl = ln.etouched();
    for (int k = tid; k < nt + ne; k += blockDim.x) {
        const bool win = k < nt, fin = k < nb;
        const size_t o = fin ? (size_t)L.ccap - 1 - (size_t)k : (size_t)(k - nb);
        const unsigned v = win ? __ldcg(tl + o) : __ldcg(etl + (k - nt));
        double c = win ? __ldcg(L.tcost + o) : 0.0;
        const unsigned a = win ? __ldcg(L.tarc + o) : 0u;
        const unsigned long long x = fin ? pack_word(c, a) : atom_exch_u64(L.pk + v, SENT);
        if (!win || x != pack_word(c, a)) c = __ldcg(&L.erec[v].cost);
        if (c <= cutoff) {
            const int idx = agg_append(&sm.ntok[1]);
            __stcg(io.tok_state + n + idx, v);
            __stcg(io.tok_cost + n + idx, c);
        }
    }
    __syncthreads();
    if (tid == 0) {
        io.out_i[4] = sm.ntok[1];
        io.out_d[0] = cutoff;
        if (sm.err && !io.out_i[0]) io.out_i[0] = sm.err;
        __stcg(L.round_ctr, sm.round_id);
    }
}

// f32 -> f64 widening of device-resident cost matrices (exact), one matrix per grid row.
struct WidenJob {
    const float *src;
    double *dst;
    long long n;
};
__global__ void widen_f32_kernel(const WidenJob *__restrict__ jobs) {
    const WidenJob J = jobs[blockIdx.y];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < J.n; i += (long long)gridDim.x * blockDim.x)
        J.dst[i] = (double)__ldg(J.src + i);
}

__global__ void fill_f64(double *a, long long n, double v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] = v;
}

// Workspace initialisation: every state record idle (pack SENT, no token, minsnap +inf).
__global__ void init_rec(StateRec *r, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        StateRec x;
        x.pack = SENT;
        x.cost = 0.0;
        x.pred = -1;
        x.tokidx = -1;
        x.minsnap = inf_d();
        r[i] = x;
    }
}

}  // namespace lbk
