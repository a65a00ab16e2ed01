// lb_kernels.cuh — the sm_100a decode-lane kernels.
//
// A decode lane is one thread-block CLUSTER (C CTAs, C = 1..4) that owns one
// utterance of a wave (the paper's sequence parallelism, as
// lanes instead of MPS processes).  The lane walks the utterance's frames in
// order; inside a frame its C CTAs split every phase below and meet at cluster
// barriers.  The lane's counters (touched / frontier / token / lattice list
// lengths, error flag) live in the shared memory of the cluster's rank-0 CTA and
// are updated through distributed shared memory, so no frame ever leaves the
// GPU.  Fewer, wider lanes keep every lane's hot per-state records L2-resident
// (SURVEY.md §7 step 7).  Hot loops are batched UNR-wide so every thread keeps
// UNR independent gathers / atomics in flight.
//
//   emit      warp-cooperative expansion of the previous frame's tokens: the warp
//             takes 32 tokens, prefix-scans their out-degrees with shuffles
//             (Alg. 2 / static partition, scheduler.py:60-78) and walks the
//             flattened arc range 32*UNR arcs at a time, each lane binary-
//             searching its owner token with shuffles; 16 B arc loads; one 64-bit
//             atomicMin per candidate on the packed (cost, arc) word (Alg. 1,
//             decoder.py:189-205); states seen for the first time (old ==
//             sentinel) go to the touched list (one DSMEM atomic per warp).  The
//             frame best is a cluster min over ALL candidates.
//   winners   per touched state: the winner's f64 cost is recomputed from its
//             arc and its source token's cost (same operands, same order =>
//             bit-identical to the offer); seed if cost <= cutoff; max-active
//             histogram (per CTA, merged through DSMEM).
//   epsilon   Jacobi rounds (reference.py:160-192): phase A offers pack words
//             from snapshot costs, phase B lets the round's unique winning offer
//             write the state's f64 cost / source.
//   aggregate touched states under the cutoff become the frame's token list
//             (device order; the host sorts by state when lists are read back);
//             the same pass resets the state's pack word (O(touched), not O(S)).
//   lattice   live arcs by rule A.5: emitting arc live iff its
//             candidate <= cutoff and its destination was kept; epsilon arc live
//             iff both ends kept and min-snapshot(src) + w <= cutoff.
#pragma once
#include <cooperative_groups.h>

#include "lb_device.cuh"

namespace lbk {

namespace cgx = cooperative_groups;

// Shared state of a lane.  Lane-wide fields are authoritative in the rank-0 CTA
// (reached through DSMEM); they are double-buffered by frame parity (and the
// epsilon frontier length by round parity) so a frame needs no barrier just to
// reset counters: the set for frame t+1 is cleared while frame t runs.
struct Smem {
    int ntouched[2], ntok[2], nfix[2], nlat[2];
    int nfr[3];                    // epsilon frontier lengths (round mod 3)
    int nseed[2];                  // seeds (winners <= cutoff) per frame parity
    unsigned long long best[2];    // order-preserving f64 frame best (frame parity)
    int err, err_frame;
    long long err_aux;
    unsigned long long c_tok, c_scan, c_cand, c_front, c_escan, c_ecand, c_next;
    // per CTA
    unsigned round_id;             // epsilon round tag (identical in every CTA of the lane)
    double red0;
    int ired0;
    double red[32];
    int ired[32];
    int hist[2][NBINS];            // max-active histogram (frame parity)
};

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7FF0000000000000ll); }

// The cluster that runs one lane.
struct Grp {
    Smem *S;        // this CTA's shared state
    Smem *M;        // rank-0 CTA's shared state (DSMEM)
    int rank, C;
    __device__ __forceinline__ void sync() const { cgx::this_cluster().sync(); }
    __device__ __forceinline__ Smem *at(int q) const { return cgx::this_cluster().map_shared_rank(S, q); }
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
    if (lane == 0) { G.S->red[warp] = v; G.S->ired[warp] = s; }
    __syncthreads();
    if (warp == 0) {
        double x = lane < nw ? G.S->red[lane] : inf_d();
        int y = lane < nw ? G.S->ired[lane] : 0x7FFFFFFF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(FULL, x, o);
            int os = __shfl_xor_sync(FULL, y, o);
            if (ov < x || (ov == x && os < y)) { x = ov; y = os; }
        }
        if (lane == 0) { G.S->red0 = x; G.S->ired0 = y; }
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
// the list.  f(valid[], i[], arc[], cost[]) receives one batch.
template <int UNR, class F>
__device__ __forceinline__ void for_each_token_arc_batched(const GraphDev &g, const Grp &G,
                                                           const unsigned *ts, const double *tc, int n,
                                                           unsigned &c_scan, F &&f) {
    const int lane = threadIdx.x & 31;
    for (int base = G.gwarp() * 32; base < n; base += G.gnw() * 32) {
        const int i = base + lane;
        const bool valid = i < n;
        const unsigned s = valid ? __ldcg(ts + i) : 0u;
        const double c = valid ? __ldcg(tc + i) : 0.0;
        const uint2 rg = valid ? __ldg(g.rng + s) : make_uint2(0u, 0u);
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
        for (int j0 = 0; j0 < total; j0 += 32 * UNR) {
            bool vv[UNR];
            int ii[UNR];
            unsigned aa[UNR];
            double cc[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const int j = j0 + u * 32 + lane;
                int k = 0;
#pragma unroll
                for (int b = 16; b > 0; b >>= 1) {
                    int t = __shfl_sync(FULL, incl, k + b - 1);
                    if (t <= j) k += b;
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
    }
}

// Per-lane decode phases.  UNR = independent items per thread per batch.
template <int UNR>
struct Lane {
    const GraphDev &g;      // __grid_constant__ kernel parameters: referenced in place,
    const Params &p;        // never copied to local memory
    const LaneWs &L;
    const UttDesc &io;
    const Grp G;
    double *acrow;          // shared-memory row (when p.acrow_smem)
    const double *row;      // global row of the current frame
    int par;                // parity of the current frame (cost slot, counter set)

    __device__ Lane(const GraphDev &g_, const Params &p_, const LaneWs &L_, const UttDesc &io_,
                    const Grp &G_, double *acrow_)
        : g(g_), p(p_), L(L_), io(io_), G(G_), acrow(acrow_), row(nullptr), par(0) {}

    __device__ __forceinline__ unsigned *fsb(int r) const { return (r & 1) ? L.fs1 : L.fs0; }
    __device__ __forceinline__ double *fcb(int r) const { return (r & 1) ? L.fc1 : L.fc0; }
    __device__ __forceinline__ uint2 *feb(int r) const { return (r & 1) ? L.fe1 : L.fe0; }

    __device__ __forceinline__ double ac(unsigned il) const {
        return p.acrow_smem ? acrow[il - 1] : __dmul_rn(__ldg(row + il - 1), p.scale);
    }

    __device__ __forceinline__ void set_error(int code, int frame, long long aux) const {
        if (atomicCAS(&G.M->err, 0, code) == 0) {
            G.M->err_frame = frame;
            G.M->err_aux = aux;
        }
    }

    __device__ void load_row(const double *r) {
        row = r;
        if (p.acrow_smem)
            for (int d = threadIdx.x; d < p.D; d += blockDim.x) acrow[d] = __dmul_rn(__ldg(r + d), p.scale);
    }

    // Clear the counter set of the NEXT frame (leader only; its last readers are done).
    __device__ __forceinline__ void clear_next_counters() const {
        if (G.leader()) {
            Smem *M = G.M;
            const int q = par ^ 1;
            M->ntouched[q] = M->ntok[q] = M->nfix[q] = M->nlat[q] = M->nseed[q] = 0;
        }
        if (threadIdx.x == 0) G.S->best[par ^ 1] = SENT;   // per-CTA partial of the next frame
        for (int b = threadIdx.x; b < NBINS; b += blockDim.x) G.S->hist[par ^ 1][b] = 0;
    }

    // ---- emit: returns the lane-wide best candidate (one cluster barrier) ----
    // Every candidate feeds the frame best, but a candidate whose float32 key is
    // above the float32 key of a running upper bound of this frame's cutoff
    // (running best + beam_eff) skips its atomic: it can neither be the best nor
    // the winner of a state that survives the cutoff, and no epsilon offer (cost
    // <= cutoff) can tie with it, so every kept state's winner is unchanged.
    __device__ double emit(const unsigned *pts, const double *ptc, int np, double beam_eff) {
        double lbest = inf_d();
        StateRec *rec = L.rec;
        unsigned c_scan = 0, c_cand = 0;
        int *ntouched = &G.M->ntouched[par];
        unsigned long long *run = &G.S->best[par];
        unsigned bound_key = 0xFFFFFFFFu;     // enc32 of the running cutoff bound
        if (G.leader()) G.M->nfr[0] = G.M->nfr[1] = G.M->nfr[2] = 0;
        for_each_token_arc_batched<UNR>(g, G, pts, ptc, np, c_scan,
                                        [&](const bool *vv, const int *, const unsigned *aa, const double *cc) {
            int4 r[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (vv[u]) r[u] = __ldg(g.arcs + aa[u]);
            double cand[UNR];
            double bmin = inf_d();
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                cand[u] = inf_d();
                if (vv[u] && r[u].y != 0) {
                    const double w = __hiloint2double(r[u].w, r[u].z);
                    cand[u] = __dadd_rn(__dadd_rn(cc[u], w), ac((unsigned)r[u].y));
                    bmin = fmin(bmin, cand[u]);
                }
            }
            lbest = fmin(lbest, bmin);
            // share the running best through the CTA (one shared atomic per warp batch)
            bmin = warp_min(bmin);
            unsigned long long rb = 0;
            if ((threadIdx.x & 31) == 0) {
                const unsigned long long e = enc64(bmin);
                const unsigned long long o = atomicMin(run, e);
                rb = o < e ? o : e;
            }
            rb = __shfl_sync(FULL, rb, 0);
            const double rbest = dec64(rb);
            if (rbest < inf_d()) {
                const unsigned k = (unsigned)(pack_word(__dadd_rn(rbest, beam_eff), 0u) >> 32);
                bound_key = k < bound_key ? k : bound_key;
            }
            unsigned long long old[UNR];
            bool em[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                em[u] = cand[u] < inf_d();
                if (em[u]) {
                    const unsigned long long word = pack_word(cand[u], aa[u]);
                    em[u] = (unsigned)(word >> 32) <= bound_key;
                    if (em[u]) {
                        old[u] = atomicMin(&rec[r[u].x].pack, word);
                        c_cand++;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                if (em[u] && old[u] == SENT) {
                    const int sl = agg_append(ntouched);
                    __stcg(L.touched + sl, (unsigned)r[u].x);
                }
            }
        });
        lbest = warp_min(lbest);
        c_cand = warp_sum(c_cand);
        c_scan = warp_sum(c_scan);
        if ((threadIdx.x & 31) == 0) {
            // CTA-local shared atomics; the lane-wide min is merged after the barrier
            atomicMin(run, enc64(lbest));
            atomicAdd(&G.S->c_cand, (unsigned long long)c_cand);
            atomicAdd(&G.S->c_scan, (unsigned long long)c_scan);
        }
        G.sync();
        unsigned long long b = SENT;
        for (int q = 0; q < G.C; q++) {
            const unsigned long long x = G.at(q)->best[par];
            b = x < b ? x : b;
        }
        return dec64(b);
    }

    // ---- winners: f64 cost of every touched state; seeds; epsilon frontier (round 0); histogram ----
    __device__ void winners(double cutoff, double best) {
        const int nt = G.M->ntouched[par];
        const bool hist = p.max_active > 0;
        const bool eps = g.has_eps;
        const double width = __ddiv_rn(p.beam, (double)NBINS);
        const int pp = par ^ 1;
        StateRec *rec = L.rec;
        int *nfront = &G.M->nfr[0], *nseed = &G.M->nseed[par];
        int *hst = G.S->hist[par];
        const int stride = G.gstride();
        for (int k0 = G.gtid(); k0 < nt; k0 += UNR * stride) {
            unsigned v[UNR];
            bool ok[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const int k = k0 + u * stride;
                ok[u] = k < nt;
                v[u] = ok[u] ? __ldcg(L.touched + k) : 0u;
            }
            unsigned a[UNR];
            uint2 er[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                a[u] = ok[u] ? (unsigned)__ldcg(&rec[v[u]].pack) : 0u;
                er[u] = (ok[u] && eps) ? __ldg(g.erng + v[u]) : make_uint2(0u, 0u);
            }
            int4 ar[UNR];
            unsigned src[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                if (ok[u]) {
                    ar[u] = __ldg(g.arcs + a[u]);
                    src[u] = __ldg(g.src + a[u]);
                }
            }
            double pc[UNR];
            int pi[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                if (ok[u]) {
                    const RecView sr = load_rec32(&rec[src[u]]);
                    pc[u] = sr.cost(pp);
                    pi[u] = sr.tokidx;
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                if (!ok[u]) continue;
                const double w = __hiloint2double(ar[u].w, ar[u].z);
                const double cand = __dadd_rn(__dadd_rn(pc[u], w), ac((unsigned)ar[u].y));
                __stcg(&rec[v[u]].cost[par], cand);
                __stcg(&rec[v[u]].pred, (pi[u] << 1) | 1);
                if (cand <= cutoff) {
                    agg_append(nseed);
                    if (er[u].x < er[u].y) {      // only states with epsilon arcs enter the closure
                        const int sl = agg_append(nfront);
                        __stcg(L.fs0 + sl, v[u]);
                        __stcg(L.fc0 + sl, cand);
                        __stcg(L.fe0 + sl, er[u]);
                    }
                    if (hist) {
                        const double q = __ddiv_rn(__dsub_rn(cand, best), width);
                        const int bin = q >= (double)NBINS ? NBINS - 1 : (q < 0.0 ? 0 : (int)q);
                        atomicAdd(&hst[bin], 1);
                    }
                }
            }
        }
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
            if (lane == 0) G.S->red0 = c2;
        }
        __syncthreads();
        const double r = G.S->red0;
        __syncthreads();
        return r;
    }

    // Keep the round-0 epsilon frontier entries with cost <= cutoff (after a
    // max-active tightening): buffer 0 -> buffer 1 (count nfr[1]), one batched
    // pass and one barrier; the epsilon closure then starts at round 1.
    __device__ void filter_seeds(double cutoff) {
        const int nf = G.M->nfr[0];
        int *nout = &G.M->nfr[1];
        const int stride = G.gstride();
        for (int k0 = G.gtid(); k0 < nf; k0 += 4 * stride) {
            double c[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = k0 + u * stride;
                c[u] = k < nf ? __ldcg(L.fc0 + k) : inf_d();
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (c[u] <= cutoff) {
                    const int k = k0 + u * stride;
                    const int sl = agg_append(nout);
                    __stcg(L.fs1 + sl, __ldcg(L.fs0 + k));
                    __stcg(L.fc1 + sl, c[u]);
                    __stcg(L.fe1 + sl, __ldcg(L.fe0 + k));
                }
            }
        }
        G.sync();
    }

    // ---- epsilon closure under a fixed cutoff: Jacobi rounds, two barriers each ----
    // Round r reads frontier buffer (r&1) = (state, snapshot cost, epsilon range),
    // count nfr[r%3].  Phase A: each entry parks its snapshot in its record's
    // cost[par^1] slot (dead after winners), offers pack words, and tags improved
    // states (the first tagger appends the state to the next frontier).  Phase B:
    // for each improved state the winning arc is read from the pack; its f64 cost
    // is recomputed from the source's parked snapshot (same operands => the
    // winning offer's exact value) and written with the source as predecessor.
    __device__ bool epsilon(double cutoff, int frame, int r0 = 0) {
        const bool LAT = p.want_lattice;
        StateRec *rec = L.rec;
        const int stride = G.gstride();
        const int pp = par ^ 1;
        unsigned round_id = G.S->round_id;
        unsigned c_escan = 0, c_ecand = 0, c_front = 0;
        bool ok = true;
        for (int r = r0;; r++) {
            const int nf = G.M->nfr[r % 3];
            if (nf == 0) break;
            if (r > g.S + 1) {
                if (G.leader()) set_error(E_INT_EPS_ROUNDS, frame, 0);
                ok = false;
                break;
            }
            ++round_id;
            const unsigned *fs = fsb(r);
            const double *fc = fcb(r);
            const uint2 *fe = feb(r);
            unsigned *fsn = fsb(r + 1);
            double *fcn = fcb(r + 1);
            uint2 *fen = feb(r + 1);
            int *nnext = &G.M->nfr[(r + 1) % 3];
            if (G.leader()) G.M->nfr[(r + 2) % 3] = 0;   // read at round r-1's start, two barriers ago
            // phase A: offers from snapshot costs
            for (int k = G.gtid(); k < nf; k += stride) {
                const double cu = __ldcg(fc + k);
                if (!(cu <= cutoff)) continue;
                const unsigned u = __ldcg(fs + k);
                const uint2 er = __ldcg(fe + k);
                c_front++;
                if (LAT) {
                    const double m = __ldcg(L.minsnap + u);
                    if (cu < m) __stcg(L.minsnap + u, cu);
                }
                __stcg(&rec[u].cost[pp], cu);
                c_escan += er.y - er.x;
                for (unsigned e = er.x; e < er.y; ++e) {
                    const int4 rr = __ldg(g.eps + e);
                    const double cand = __dadd_rn(cu, __hiloint2double(rr.w, rr.z));
                    if (!(cand <= cutoff)) continue;
                    c_ecand++;
                    const unsigned v = (unsigned)rr.x;
                    const unsigned long long word = pack_word(cand, (unsigned)rr.y);
                    const unsigned long long old = atomicMin(&rec[v].pack, word);
                    if (old == SENT) {
                        const int sl = agg_append(&G.M->ntouched[par]);
                        __stcg(L.touched + sl, v);
                    }
                    if (old > word && atomicExch(L.tag + v, round_id) != round_id) {
                        const int sl = agg_append(nnext);
                        __stcg(fsn + sl, v);
                    }
                }
            }
            G.sync();
            // phase B: improved states recover their round winner from the pack
            const int nn = *nnext;
            for (int k = G.gtid(); k < nn; k += stride) {
                const unsigned v = __ldcg(fsn + k);
                const unsigned a = (unsigned)__ldcg(&rec[v].pack);
                const double w = __ldg(reinterpret_cast<const double *>(g.arcs + a) + 1);
                const unsigned u = __ldg(g.src + a);
                const uint2 er = __ldg(g.erng + v);
                const double cand = __dadd_rn(__ldcg(&rec[u].cost[pp]), w);
                __stcg(&rec[v].cost[par], cand);
                __stcg(&rec[v].pred, (int)(u << 1));
                __stcg(fcn + k, cand);
                __stcg(fen + k, er);
            }
            G.sync();
        }
        c_escan = warp_sum(c_escan);
        c_ecand = warp_sum(c_ecand);
        c_front = warp_sum(c_front);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&G.S->c_escan, (unsigned long long)c_escan);
            atomicAdd(&G.S->c_ecand, (unsigned long long)c_ecand);
            atomicAdd(&G.S->c_front, (unsigned long long)c_front);
        }
        if (threadIdx.x == 0) G.S->round_id = round_id;
        if (!ok) G.sync();
        return ok;
    }

    // ---- aggregate + reset: frame token list at io.tok_*[tb ...]; returns count or -1 ----
    __device__ int aggregate(double cutoff, int frame, long long tb) {
        const int nt = G.M->ntouched[par];
        const long long room = io.tok_cap - tb;
        StateRec *rec = L.rec;
        unsigned *fix = L.fs1;  // scratch: tokens whose predecessor is an epsilon source state
        int *ntok = &G.M->ntok[par], *nfix = &G.M->nfix[par];
        const int stride = G.gstride();
        for (int k0 = G.gtid(); k0 < nt; k0 += UNR * stride) {
            unsigned v[UNR];
            bool ok[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const int k = k0 + u * stride;
                ok[u] = k < nt;
                v[u] = ok[u] ? __ldcg(L.touched + k) : 0u;
            }
            RecView r[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (ok[u]) r[u] = load_rec32(&rec[v[u]]);
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                if (!ok[u]) continue;
                const bool init = frame == 0 && (int)v[u] == g.start;
                const double c = init ? 0.0 : r[u].cost(par);
                int tidx = r[u].tokidx;
                if (init || c <= cutoff) {
                    const int idx = agg_append(ntok);
                    if (idx < room) {
                        const long long o = tb + idx;
                        __stcg(io.tok_state + o, v[u]);
                        __stcg(io.tok_cost + o, c);
                        __stcg(io.tok_arc + o, init ? -1 : (int)(unsigned)r[u].pack);
                        __stcg(io.tok_pred + o, init ? -1 : r[u].pred);
                        if (p.collect_packs) __stcg(io.tok_pack + o, r[u].pack);
                        tidx = idx;
                        if (!init && (r[u].pred & 1) == 0) {
                            const int f = agg_append(nfix);
                            __stcg(fix + f, (unsigned)idx);
                        }
                    }
                }
                __stcg(&rec[v[u]].pack, SENT);
                if (tidx != r[u].tokidx) __stcg(&rec[v[u]].tokidx, tidx);
            }
        }
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
        // epsilon predecessors: source state -> token index of this frame
        const int nfx = G.M->nfix[par];
        if (nfx > 0) {
            for (int q = G.gtid(); q < nfx; q += stride) {
                const long long o = tb + (long long)__ldcg(fix + q);
                const int u = __ldcg(io.tok_pred + o) >> 1;
                const int pi = __ldcg(&rec[u].tokidx);
                if (pi < 0 || pi >= n || __ldcg(io.tok_state + tb + pi) != (unsigned)u)
                    set_error(E_INT_EPS_PRED, frame, u);
                __stcg(io.tok_pred + o, pi << 1);
            }
            G.sync();
            if (G.M->err) return -1;
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
        j = __ldcg(&L.rec[v].tokidx);
        return j >= 0 && j < n && __ldcg(io.tok_state + tb + j) == v;
    }

    // ---- lattice arcs of block `frame` (rule A.5); resets minsnap; returns arc count or -1 ----
    __device__ int lattice(double cutoff, int frame, long long tbp, int np, long long tb, int n,
                           long long lb) {
        if (frame > 0) {
            unsigned dummy = 0;
            for_each_token_arc_batched<UNR>(g, G, io.tok_state + tbp, io.tok_cost + tbp, np, dummy,
                                            [&](const bool *vv, const int *ii, const unsigned *aa, const double *cc) {
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    if (!vv[u]) continue;
                    const int4 r = __ldg(g.arcs + aa[u]);
                    if (r.y == 0) continue;
                    const double w = __hiloint2double(r.w, r.z);
                    const double cand = __dadd_rn(__dadd_rn(cc[u], w), ac((unsigned)r.y));
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
                const double ms = __ldcg(L.minsnap + u);
                __stcg(L.minsnap + u, inf);
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

    // ---- error path: O(touched) reset of every state word this frame touched ----
    __device__ void reset_touched() {
        G.sync();
        const int nt = G.M->ntouched[par];
        const double inf = inf_d();
        for (int k = G.gtid(); k < nt; k += G.gstride()) {
            const unsigned v = __ldcg(L.touched + k);
            __stcg(&L.rec[v].pack, SENT);
            if (p.want_lattice) __stcg(L.minsnap + v, inf);
        }
        G.sync();
    }
};

__device__ __forceinline__ void init_smem(Smem &sm, unsigned round_ctr) {
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; q++) {
            sm.ntouched[q] = sm.ntok[q] = sm.nfix[q] = sm.nlat[q] = sm.nseed[q] = 0;
            sm.best[q] = SENT;
        }
        sm.nfr[0] = sm.nfr[1] = sm.nfr[2] = 0;
        sm.err = sm.err_frame = 0;
        sm.err_aux = 0;
        sm.round_id = round_ctr;
        sm.c_tok = sm.c_scan = sm.c_cand = sm.c_front = sm.c_escan = sm.c_ecand = sm.c_next = 0;
    }
    for (int b = threadIdx.x; b < 2 * NBINS; b += blockDim.x) sm.hist[b / NBINS][b % NBINS] = 0;
}

// ===========================================================================
// Full-utterance decode: one cluster (lane) per utterance of the wave.
// Cluster barriers per frame: emit 1, winners 1, epsilon 2 per round,
// aggregate 1-2, lattice 1.
// ===========================================================================
template <int NT, int UNR, bool LAT, bool PROF>
__global__ void __launch_bounds__(NT, 1)
decode_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
              const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ utts, int n_utts) {
    __shared__ Smem sm;
    extern __shared__ double s_acrow[];
    cgx::cluster_group cl = cgx::this_cluster();
    Grp G;
    G.C = (int)cl.num_blocks();
    G.rank = (int)cl.block_rank();
    G.S = &sm;
    G.M = cl.map_shared_rank(&sm, 0);
    const int u_idx = blockIdx.x / G.C;      // uniform across the cluster
    if (u_idx >= n_utts) return;
    const LaneWs &L = lanes[u_idx];
    const UttDesc &io = utts[u_idx];
    init_smem(sm, __ldcg(L.round_ctr));
    G.sync();

    Lane<UNR> ln(g, p, L, io, G, s_acrow);
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
    if (G.leader()) {
        __stcg(&L.rec[g.start].pack, pack_word(0.0, 0u));
        __stcg(&L.rec[g.start].cost[0], 0.0);
        __stcg(&L.rec[g.start].pred, -1);
        __stcg(L.touched, (unsigned)g.start);
        __stcg(L.fs0, (unsigned)g.start);
        __stcg(L.fc0, 0.0);
        __stcg(L.fe0, g.has_eps ? __ldg(g.erng + g.start) : make_uint2(0u, 0u));
        sm.ntouched[0] = 1;
        sm.nfr[0] = 1;
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
        ln.load_row(io.costs + (long long)(t - 1) * p.D);
        __syncthreads();
        const double best = ln.emit(io.tok_state + tbp, io.tok_cost + tbp, np, beam_eff);
        ln.clear_next_counters();   // frame t-1's readers are past the emit barrier
        mark(0);
        if (!(best < inf)) {
            if (G.leader()) ln.set_error(E_DEAD_NO_CAND, t, 0);
            ok = false;
            break;
        }
        cutoff = __dadd_rn(best, beam_eff);
        ln.winners(cutoff, best);
        G.sync();
        mark(1);
        const int nf = G.M->nseed[ln.par];
        if (nf == 0) {
            if (G.leader()) ln.set_error(E_DEAD_NO_TOKENS, t, 0);
            ok = false;
            break;
        }
        int r0 = 0;
        bool tightened = false;
        if (p.max_active > 0 && nf > p.max_active) {
            const double c2 = ln.max_active_cutoff(cutoff, best);
            if (c2 < cutoff) {
                tightened = true;
                cutoff = c2;
                if (g.has_eps) {   // without epsilon arcs the seeds are never read again
                    ln.filter_seeds(cutoff);
                    r0 = 1;
                }
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
            ok = ln.epsilon(cutoff, t, r0);
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
        __stcg(L.round_ctr, sm.round_id);
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
        const int bidx = __ldcg(&L.rec[bstate].tokidx);
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
    G.sync();   // keep rank 0's shared memory alive until every CTA is done with it
}

// ===========================================================================
// Lattice extra-cost pruning (lattice.py:365-497) from the final terminus,
// one CTA per utterance: backward over frames, emitting arcs relax node
// extras with a 64-bit atomicMin on the order-preserving f64 encoding, the
// in-frame epsilon fixpoint runs Jacobi iterations, then every arc is flagged.
// ===========================================================================
__global__ void __launch_bounds__(1024, 1)
prune_kernel(GraphDev g, Params p, const UttDesc *__restrict__ utts, int n_utts) {
    __shared__ int s_moved;
    if ((int)blockIdx.x >= n_utts) return;
    const UttDesc io = utts[blockIdx.x];
    if (io.out_i[0] != E_OK) return;
    const int tid = threadIdx.x, bd = blockDim.x;
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
            __syncthreads();
        } else {
            for (int i = tid; i < nfr; i += bd) __stcg(ne + i, enc64(inf));
            __syncthreads();
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
                atomicMin(ne + from, enc64(c));
            }
            __syncthreads();
        }
        // in-frame epsilon fixpoint (lattice.py:455-469)
        if (g.has_eps) {
            const long long k0 = io.lat_base[f], k1 = io.lat_base[f + 1];
            for (int it = 0;; it++) {
                if (tid == 0) s_moved = 0;
                __syncthreads();
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
                    io.tmp[k] = c;
                    if (__dsub_rn(before, c) > CONVERGE_TOL) s_moved = 1;
                }
                __syncthreads();
                for (long long k = k0 + tid; k < k1; k += bd) {
                    const unsigned a = (unsigned)__ldcg(io.lat_arc + k);
                    if ((unsigned)__ldg(g.arcs + a).y != 0) continue;
                    atomicMin(ne + __ldcg(io.lat_from + k), enc64(io.tmp[k]));
                }
                __syncthreads();
                const int moved = s_moved;
                __syncthreads();
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
        __syncthreads();
    }
    // flag pass (lattice.py:473-497)
    for (int b = 0; b <= T; b++) {
        const long long tbb = io.tok_base[b];
        for (long long k = io.lat_base[b] + tid; k < io.lat_base[b + 1]; k += bd) {
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
            io.lat_extra[k] = x < 0.0 ? 0.0 : x;
        }
    }
}

// ===========================================================================
// Single-op surfaces (decoder.py:373-435), one CTA (a cluster of one).
//   mode 0 = expand_emitting: tokens at io.tok_*[0..n), whose states carry
//            (cost[0], tokidx) from setup_tokens; acrow (scaled) at io.costs;
//            writes winners <= cutoff to io.tok_state/tok_cost[n ...].
//   mode 1 = expand_nonemitting: seeds at io.tok_*[0..n) act as won entries
//            pack(cost, 0); closes under `cutoff`; writes the merged frontier.
// ===========================================================================
__global__ void __launch_bounds__(1024, 1)
expand_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
              const __grid_constant__ LaneWs L, const __grid_constant__ UttDesc io, int n, int mode,
              double cutoff_in) {
    __shared__ Smem sm;
    extern __shared__ double s_acrow[];
    Grp G;
    G.C = 1;
    G.rank = 0;
    G.S = &sm;
    G.M = cgx::this_cluster().map_shared_rank(&sm, 0);
    const int tid = threadIdx.x;
    init_smem(sm, __ldcg(L.round_ctr));
    __syncthreads();
    Lane<2> ln(g, p, L, io, G, s_acrow);
    double cutoff = cutoff_in;
    ln.par = 1;
    if (mode == 0) {
        ln.load_row(io.costs);
        __syncthreads();
        const double best = ln.emit(io.tok_state, io.tok_cost, n, p.beam);
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
            __stcg(&L.rec[s].pack, pack_word(c, 0u));
            __stcg(&L.rec[s].cost[1], c);
            __stcg(&L.rec[s].pred, -1);
            __stcg(L.touched + i, s);
            __stcg(L.fs0 + i, s);
            __stcg(L.fc0 + i, c);
            __stcg(L.fe0 + i, g.has_eps ? __ldg(g.erng + s) : make_uint2(0u, 0u));
        }
        __syncthreads();
        if (tid == 0) { sm.ntouched[1] = n; sm.nfr[0] = n; }
        __syncthreads();
        if (!ln.epsilon(cutoff, 0)) {
            if (tid == 0) io.out_i[0] = sm.err;
        }
    }
    __syncthreads();
    const int nt = sm.ntouched[1];
    for (int k = tid; k < nt; k += blockDim.x) {
        const unsigned v = __ldcg(L.touched + k);
        const double c = __ldcg(&L.rec[v].cost[1]);
        if (c <= cutoff) {
            const int idx = agg_append(&sm.ntok[1]);
            __stcg(io.tok_state + n + idx, v);
            __stcg(io.tok_cost + n + idx, c);
        }
        __stcg(&L.rec[v].pack, SENT);
    }
    __syncthreads();
    if (tid == 0) {
        io.out_i[4] = sm.ntok[1];
        io.out_d[0] = cutoff;
        __stcg(L.round_ctr, sm.round_id);
    }
}

// Fill helpers.
__global__ void fill_f64(double *p, double v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}
// expand_emitting setup: the frontier's states carry (cost[0], tokidx) like a previous frame.
__global__ void setup_tokens(StateRec *rec, const unsigned *states, const double *costs, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        rec[states[i]].cost[0] = costs[i];
        rec[states[i]].tokidx = i;
    }
}

}  // namespace lbk
