// lb_kernels.cuh — the sm_100a decode-lane kernels.
//
// One CTA is one decode lane and owns one utterance of a wave (the paper's
// sequence parallelism, as lanes instead of MPS processes).
// A lane walks the utterance's frames in order; inside a frame the CTA runs the
// phases below, separated by __syncthreads (no grid-wide sync, no host round
// trip per frame):
//
//   emit      warp-cooperative expansion of the previous frame's tokens: the warp
//             takes 32 tokens, prefix-scans their out-degrees with shuffles
//             (Alg. 2 / static partition, scheduler.py:60-78) and walks the
//             flattened arc range 32 arcs at a time, each lane binary-searching
//             its owner token with shuffles; 16 B arc loads; one 64-bit atomicMin
//             per candidate on the packed (cost, arc) word (Alg. 1,
//             decoder.py:189-205); states seen for the first time (old ==
//             sentinel) are appended to the touched list with one shared atomic
//             per warp.  The frame best is a block min over ALL candidates.
//   winners   per touched state: the winner's f64 cost is recomputed from its
//             arc (same operands, same order => bit-identical to the offer) and
//             the state is seeded if cost <= cutoff; max-active histogram.
//   epsilon   Jacobi rounds (reference.py:160-192): phase A offers pack words
//             from snapshot costs, phase B lets the unique winning offer of the
//             round write the state's f64 cost / source.
//   aggregate touched states under the cutoff become the frame's token list
//             (device order; the host sorts by state when lists are read back).
//   lattice   live arcs by rule A.5: emitting arc live iff its
//             candidate <= cutoff and its destination was kept; epsilon arc live
//             iff both ends kept and min-snapshot(src) + w <= cutoff.
//   reset     O(touched) reset of the per-state words (not O(S), decoder.py:123).
#pragma once
#include "lb_device.cuh"

namespace lbk {

struct Smem {
    int ntouched, nfront, nnext, ntok, nlat, err, err_frame, moved;
    long long err_aux;
    double cutoff;
    double red[32];
    long long lred[32];
    int ired[32];
    int hist[NBINS];
};

__device__ __forceinline__ double block_min(double v, Smem &sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_min(v);
    if (lane == 0) sm.red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double x = lane < nw ? sm.red[lane] : __longlong_as_double(0x7FF0000000000000ll);
        x = warp_min(x);
        if (lane == 0) sm.red[0] = x;
    }
    __syncthreads();
    double r = sm.red[0];
    __syncthreads();
    return r;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, Smem &sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sm.lred[warp] = (long long)v;
    __syncthreads();
    T r = 0;
    if (threadIdx.x == 0)
        for (int k = 0; k < nw; k++) r += (T)sm.lred[k];
    __syncthreads();
    return r;   // valid on thread 0
}

// (value, state) lexicographic min; returns on all threads.
__device__ __forceinline__ void block_argmin(double &v, int &s, Smem &sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(FULL, v, o);
        int os = __shfl_xor_sync(FULL, s, o);
        if (ov < v || (ov == v && os < s)) { v = ov; s = os; }
    }
    if (lane == 0) { sm.red[warp] = v; sm.ired[warp] = s; }
    __syncthreads();
    if (warp == 0) {
        double x = lane < nw ? sm.red[lane] : __longlong_as_double(0x7FF0000000000000ll);
        int y = lane < nw ? sm.ired[lane] : 0x7FFFFFFF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(FULL, x, o);
            int os = __shfl_xor_sync(FULL, y, o);
            if (ov < x || (ov == x && os < y)) { x = ov; y = os; }
        }
        if (lane == 0) { sm.red[0] = x; sm.ired[0] = y; }
    }
    __syncthreads();
    v = sm.red[0];
    s = sm.ired[0];
    __syncthreads();
}

// Warp-cooperative load-balanced walk over every (token, out-arc) pair of a
// token list.  f(i, arc, token_cost) runs once per pair (possibly divergent).
template <class F>
__device__ __forceinline__ void for_each_token_arc(const GraphDev &g, const unsigned *ts,
                                                   const double *tc, int n, unsigned &c_scan, F &&f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = warp * 32; base < n; base += nw * 32) {
        const int i = base + lane;
        const bool valid = i < n;
        const unsigned s = valid ? __ldcg(ts + i) : 0u;
        const double c = valid ? __ldcg(tc + i) : 0.0;
        const unsigned lo = valid ? __ldg(g.off + s) : 0u;
        const unsigned hi = valid ? __ldg(g.off + s + 1) : 0u;
        const int deg = (int)(hi - lo);
        int incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const int excl = incl - deg;
        const int total = __shfl_sync(FULL, incl, 31);
        if (lane == 0) c_scan += (unsigned)total;
        for (int j0 = 0; j0 < total; j0 += 32) {
            const int j = j0 + lane;
            int k = 0;
#pragma unroll
            for (int b = 16; b > 0; b >>= 1) {
                int t = __shfl_sync(FULL, incl, k + b - 1);
                if (t <= j) k += b;
            }
            const int ek = __shfl_sync(FULL, excl, k);
            const unsigned lk = __shfl_sync(FULL, lo, k);
            const double ck = __shfl_sync(FULL, c, k);
            if (j < total) f(base + k, lk + (unsigned)(j - ek), ck);
        }
    }
}

// Per-CTA decode state.  All members are block-uniform except the counters.
struct Lane {
    const GraphDev &g;
    const Params &p;
    const LaneWs &L;
    const UttDesc &io;
    Smem &sm;
    double *acrow;          // shared-memory row (when p.acrow_smem)
    const double *row;      // global row of the current frame
    unsigned *fs, *fsn;
    double *fc, *fcn;
    unsigned round_id;
    unsigned c_scan = 0, c_cand = 0, c_escan = 0, c_ecand = 0;
    long long c_tok = 0, c_front = 0, c_next = 0;

    __device__ Lane(const GraphDev &g_, const Params &p_, const LaneWs &L_, const UttDesc &io_,
                    Smem &sm_, double *acrow_)
        : g(g_), p(p_), L(L_), io(io_), sm(sm_), acrow(acrow_), row(nullptr), fs(L_.fs0),
          fsn(L_.fs1), fc(L_.fc0), fcn(L_.fc1), round_id(0) {}

    __device__ __forceinline__ double ac(unsigned il) const {
        return p.acrow_smem ? acrow[il - 1] : __dmul_rn(__ldg(row + il - 1), p.scale);
    }

    __device__ __forceinline__ void set_error(int code, int frame, long long aux) {
        if (atomicCAS(&sm.err, 0, code) == 0) {
            sm.err_frame = frame;
            sm.err_aux = aux;
        }
    }

    __device__ void load_row(const double *r) {
        row = r;
        if (p.acrow_smem)
            for (int d = threadIdx.x; d < p.D; d += blockDim.x) acrow[d] = __dmul_rn(__ldg(r + d), p.scale);
    }

    // ---- emit: returns the block-wide best candidate ----
    __device__ double emit(const unsigned *pts, const double *ptc, int np) {
        double lbest = __longlong_as_double(0x7FF0000000000000ll);
        for_each_token_arc(g, pts, ptc, np, c_scan, [&](int, unsigned a, double ck) {
            unsigned dst, il;
            double w;
            load_arc(g.arcs, a, dst, il, w);
            if (il == 0) return;
            c_cand++;
            const double cand = __dadd_rn(__dadd_rn(ck, w), ac(il));
            lbest = fmin(lbest, cand);
            const unsigned long long word = pack_word(cand, a);
            const unsigned long long old = atomicMin(L.pack + dst, word);
            if (old == SENT) {
                const int sl = agg_append(&sm.ntouched);
                __stcg(L.touched + sl, dst);
            }
        });
        return block_min(lbest, sm);
    }

    // ---- winners: f64 cost of every touched state; seed frontier; histogram ----
    __device__ void winners(const double *ptc, double cutoff, double best) {
        const int nt = sm.ntouched;
        const bool hist = p.max_active > 0;
        const double width = __ddiv_rn(p.beam, (double)NBINS);
        for (int k = threadIdx.x; k < nt; k += blockDim.x) {
            const unsigned v = __ldcg(L.touched + k);
            const unsigned a = (unsigned)__ldcg(L.pack + v);
            unsigned dst, il;
            double w;
            load_arc(g.arcs, a, dst, il, w);
            const unsigned src = __ldg(g.src + a);
            const int i = __ldcg(L.tokidx + src);
            const double cand = __dadd_rn(__dadd_rn(__ldcg(ptc + i), w), ac(il));
            __stcg(L.cost + v, cand);
            __stcg(L.pred + v, i);
            if (cand <= cutoff) {
                const int sl = agg_append(&sm.nfront);
                __stcg(fs + sl, v);
                __stcg(fc + sl, cand);
                if (hist) {
                    const double q = __ddiv_rn(__dsub_rn(cand, best), width);
                    const int bin = q >= (double)NBINS ? NBINS - 1 : (q < 0.0 ? 0 : (int)q);
                    atomicAdd(&sm.hist[bin], 1);
                }
            }
        }
    }

    // max-active cutoff: H = best + max(b*,1)*width, b* = first
    // bin whose inclusive running count exceeds max_active.  Warp 0 scans the
    // 256-bin histogram (8 bins per lane); result is uniform.
    __device__ double max_active_cutoff(double cutoff, double best) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        constexpr int PER = NBINS / 32;
        if (warp == 0) {
            int loc[PER];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                loc[q] = sm.hist[lane * PER + q];
                sum += loc[q];
            }
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
            if (lane == 0) sm.cutoff = c2;
        }
        __syncthreads();
        const double r = sm.cutoff;
        __syncthreads();
        return r;
    }

    // Keep frontier entries with cost <= cutoff (after a max-active tightening).
    __device__ void filter_frontier(double cutoff) {
        const int nf = sm.nfront;
        for (int k = threadIdx.x; k < nf; k += blockDim.x) {
            const double c = __ldcg(fc + k);
            if (c <= cutoff) {
                const int sl = agg_append(&sm.nnext);
                __stcg(fsn + sl, __ldcg(fs + k));
                __stcg(fcn + sl, c);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            sm.nfront = sm.nnext;
            sm.nnext = 0;
        }
        swap_frontier();
        __syncthreads();
    }

    __device__ __forceinline__ void swap_frontier() {
        unsigned *t = fs; fs = fsn; fsn = t;
        double *u = fc; fc = fcn; fcn = u;
    }

    // ---- epsilon closure under a fixed cutoff (Jacobi rounds) ----
    __device__ bool epsilon(double cutoff, int frame) {
        const bool LAT = p.want_lattice;
        long long rounds = 0;
        for (;;) {
            const int nf = sm.nfront;
            if (nf == 0) return true;
            if (++rounds > (long long)g.S + 1) {
                if (threadIdx.x == 0) set_error(E_INT_EPS_ROUNDS, frame, 0);
                __syncthreads();
                return false;
            }
            ++round_id;
            c_front += nf;
            // phase A: offers from snapshot costs
            for (int k = threadIdx.x; k < nf; k += blockDim.x) {
                const unsigned u = __ldcg(fs + k);
                const double cu = __ldcg(fc + k);
                if (LAT) {
                    const double m = __ldcg(L.minsnap + u);
                    if (cu < m) __stcg(L.minsnap + u, cu);
                }
                const unsigned e0 = __ldg(g.eoff + u), e1 = __ldg(g.eoff + u + 1);
                c_escan += e1 - e0;
                for (unsigned e = e0; e < e1; ++e) {
                    const unsigned a = __ldg(g.eids + e);
                    unsigned v, il;
                    double w;
                    load_arc(g.arcs, a, v, il, w);
                    const double cand = __dadd_rn(cu, w);
                    if (!(cand <= cutoff)) continue;
                    c_ecand++;
                    const unsigned long long word = pack_word(cand, a);
                    const unsigned long long old = atomicMin(L.pack + v, word);
                    if (old == SENT) {
                        const int sl = agg_append(&sm.ntouched);
                        __stcg(L.touched + sl, v);
                    }
                    if (old > word && atomicExch(L.tag + v, round_id) != round_id) {
                        const int sl = agg_append(&sm.nnext);
                        __stcg(fsn + sl, v);
                    }
                }
            }
            __syncthreads();
            // phase B: the round's unique winning offer writes cost / source
            for (int k = threadIdx.x; k < nf; k += blockDim.x) {
                const unsigned u = __ldcg(fs + k);
                const double cu = __ldcg(fc + k);
                const unsigned e0 = __ldg(g.eoff + u), e1 = __ldg(g.eoff + u + 1);
                for (unsigned e = e0; e < e1; ++e) {
                    const unsigned a = __ldg(g.eids + e);
                    unsigned v, il;
                    double w;
                    load_arc(g.arcs, a, v, il, w);
                    const double cand = __dadd_rn(cu, w);
                    if (!(cand <= cutoff)) continue;
                    if (__ldcg(L.pack + v) == pack_word(cand, a) && __ldcg(L.tag + v) == round_id) {
                        __stcg(L.cost + v, cand);
                        __stcg(L.pred + v, (int)u);
                    }
                }
            }
            __syncthreads();
            const int nn = sm.nnext;
            for (int k = threadIdx.x; k < nn; k += blockDim.x)
                __stcg(fcn + k, __ldcg(L.cost + __ldcg(fsn + k)));
            __syncthreads();
            if (threadIdx.x == 0) {
                sm.nfront = nn;
                sm.nnext = 0;
            }
            swap_frontier();
            __syncthreads();
        }
    }

    // ---- aggregate: frame token list at io.tok_*[tb ...]; returns token count or -1 ----
    __device__ int aggregate(double cutoff, int frame, long long tb) {
        const int nt = sm.ntouched;
        const long long room = io.tok_cap - tb;
        for (int k = threadIdx.x; k < nt; k += blockDim.x) {
            const unsigned v = __ldcg(L.touched + k);
            const bool init = frame == 0 && (int)v == g.start;
            const double c = init ? 0.0 : __ldcg(L.cost + v);
            if (init || c <= cutoff) {
                const int idx = agg_append(&sm.ntok);
                if (idx < room) {
                    __stcg(io.tok_state + tb + idx, v);
                    __stcg(io.tok_cost + tb + idx, c);
                    __stcg(L.tokidx + v, idx);
                }
            }
        }
        __syncthreads();
        const int n = sm.ntok;
        if (n == 0) {
            if (threadIdx.x == 0) set_error(E_DEAD_NO_TOKENS, frame, 0);
        } else if ((long long)n > p.max_tokens) {
            if (threadIdx.x == 0) set_error(E_CAP_TOKENS, frame, n);
        } else if ((long long)n > room) {
            if (threadIdx.x == 0) set_error(E_CAP_ARENA, frame, tb + n);
        }
        __syncthreads();
        if (sm.err) return -1;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const unsigned v = __ldcg(io.tok_state + tb + j);
            const unsigned long long pw = __ldcg(L.pack + v);
            int arc = -1, pred = -1;
            if (!(frame == 0 && (int)v == g.start)) {
                arc = (int)(unsigned)pw;
                const unsigned il = (unsigned)__ldg(g.arcs + arc).y;
                const int pr = __ldcg(L.pred + v);
                if (il > 0) {
                    pred = (pr << 1) | 1;
                } else {
                    const int pi = __ldcg(L.tokidx + pr);
                    if (pi < 0 || pi >= n || __ldcg(io.tok_state + tb + pi) != (unsigned)pr)
                        set_error(E_INT_EPS_PRED, frame, v);
                    pred = pi << 1;
                }
            }
            __stcg(io.tok_arc + tb + j, arc);
            __stcg(io.tok_pred + tb + j, pred);
            if (p.collect_packs) __stcg(io.tok_pack + tb + j, pw);
        }
        __syncthreads();
        return sm.err ? -1 : n;
    }

    __device__ __forceinline__ void lat_push(int arc, int from, int to, long long lb) {
        const int sl = agg_append(&sm.nlat);
        const long long gs = lb + sl;
        if (gs < io.lat_cap) {
            __stcg(io.lat_arc + gs, arc);
            __stcg(io.lat_from + gs, from);
            __stcg(io.lat_to + gs, to);
        }
    }

    __device__ __forceinline__ bool kept(unsigned v, long long tb, int n, int &j) const {
        j = __ldcg(L.tokidx + v);
        return j >= 0 && j < n && __ldcg(io.tok_state + tb + j) == v;
    }

    // ---- lattice arcs of block `frame` (rule A.5) ----
    __device__ bool lattice(double cutoff, int frame, long long tbp, int np, long long tb, int n,
                            long long lb) {
        if (frame > 0) {
            unsigned dummy = 0;
            for_each_token_arc(g, io.tok_state + tbp, io.tok_cost + tbp, np, dummy,
                               [&](int i, unsigned a, double ck) {
                                   unsigned dst, il;
                                   double w;
                                   load_arc(g.arcs, a, dst, il, w);
                                   if (il == 0) return;
                                   const double cand = __dadd_rn(__dadd_rn(ck, w), ac(il));
                                   int j;
                                   if (cand <= cutoff && kept(dst, tb, n, j)) lat_push((int)a, i, j, lb);
                               });
        }
        if (g.has_eps) {
            for (int j = threadIdx.x; j < n; j += blockDim.x) {
                const unsigned u = __ldcg(io.tok_state + tb + j);
                const unsigned e0 = __ldg(g.eoff + u), e1 = __ldg(g.eoff + u + 1);
                if (e0 == e1) continue;
                const double ms = __ldcg(L.minsnap + u);
                for (unsigned e = e0; e < e1; ++e) {
                    const unsigned a = __ldg(g.eids + e);
                    unsigned v, il;
                    double w;
                    load_arc(g.arcs, a, v, il, w);
                    int jv;
                    if (__dadd_rn(ms, w) <= cutoff && kept(v, tb, n, jv)) lat_push((int)a, j, jv, lb);
                }
            }
        }
        __syncthreads();
        const int nl = sm.nlat;
        if (lb + nl > io.lat_cap) {
            if (threadIdx.x == 0) set_error(E_CAP_LATTICE, frame, lb + nl);
        }
        __syncthreads();
        return sm.err == 0;
    }

    // ---- O(touched) reset ----
    __device__ void reset() {
        const int nt = sm.ntouched;
        const bool LAT = p.want_lattice;
        const double inf = __longlong_as_double(0x7FF0000000000000ll);
        for (int k = threadIdx.x; k < nt; k += blockDim.x) {
            const unsigned v = __ldcg(L.touched + k);
            __stcg(L.pack + v, SENT);
            if (LAT) __stcg(L.minsnap + v, inf);
        }
        for (int b = threadIdx.x; b < NBINS; b += blockDim.x) sm.hist[b] = 0;
        __syncthreads();
        if (threadIdx.x == 0) {
            sm.ntouched = 0;
            sm.nfront = 0;
            sm.nnext = 0;
            sm.ntok = 0;
            sm.nlat = 0;
        }
        __syncthreads();
    }
};

// ===========================================================================
// Full-utterance decode: one CTA per utterance of the wave.
// ===========================================================================
__global__ void __launch_bounds__(1024, 1)
decode_kernel(GraphDev g, Params p, const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ utts,
              int n_utts) {
    __shared__ Smem sm;
    extern __shared__ double s_acrow[];
    if ((int)blockIdx.x >= n_utts) return;
    const LaneWs L = lanes[blockIdx.x];
    const UttDesc io = utts[blockIdx.x];
    const int tid = threadIdx.x;
    if (tid == 0) {
        sm.ntouched = sm.nfront = sm.nnext = sm.ntok = sm.nlat = sm.err = sm.err_frame = 0;
        sm.err_aux = 0;
    }
    for (int b = tid; b < NBINS; b += blockDim.x) sm.hist[b] = 0;
    __syncthreads();

    Lane ln(g, p, L, io, sm, s_acrow);
    ln.round_id = __ldcg(L.round_ctr);
    const int T = io.T;
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    long long tb = 0, lb = 0;
    int ntok = 0, tdone = 0;

    // ---- frame 0 (decoder.py:510-523): start token, epsilon closure ----
    if (tid == 0) {
        __stcg(L.pack + g.start, pack_word(0.0, 0u));
        __stcg(L.cost + g.start, 0.0);
        __stcg(L.pred + g.start, -1);
        __stcg(L.touched, (unsigned)g.start);
        __stcg(ln.fs, (unsigned)g.start);
        __stcg(ln.fc, 0.0);
        sm.ntouched = 1;
        sm.nfront = 1;
        io.tok_base[0] = 0;
        if (p.want_lattice) io.lat_base[0] = 0;
    }
    __syncthreads();
    double cutoff = __dadd_rn(0.0, p.beam);
    bool ok = ln.epsilon(cutoff, 0);
    if (ok) {
        ntok = ln.aggregate(cutoff, 0, tb);
        ok = ntok > 0;
    }
    if (ok && p.want_lattice) {
        ok = ln.lattice(cutoff, 0, 0, 0, tb, ntok, lb);
        lb += sm.nlat;
    }
    if (tid == 0) {
        io.tok_base[1] = tb + (ok ? ntok : 0);
        if (p.want_lattice) io.lat_base[1] = lb;
    }
    ln.reset();

    for (int t = 1; ok && t <= T; t++) {
        const long long tbp = tb;
        const int np = ntok;
        tb += ntok;
        ln.c_tok += np;
        ln.load_row(io.costs + (long long)(t - 1) * p.D);
        __syncthreads();
        const double best = ln.emit(io.tok_state + tbp, io.tok_cost + tbp, np);
        if (!(best < inf)) {
            if (tid == 0) ln.set_error(E_DEAD_NO_CAND, t, 0);
            ok = false;
            break;
        }
        cutoff = __dadd_rn(best, p.beam);
        ln.winners(io.tok_cost + tbp, cutoff, best);
        __syncthreads();
        if (sm.nfront == 0) {
            if (tid == 0) ln.set_error(E_DEAD_NO_TOKENS, t, 0);
            ok = false;
            break;
        }
        if (p.max_active > 0 && sm.nfront > p.max_active) {
            const double c2 = ln.max_active_cutoff(cutoff, best);
            if (c2 < cutoff) {
                cutoff = c2;
                ln.filter_frontier(cutoff);
            }
        }
        if (g.has_eps) {
            ok = ln.epsilon(cutoff, t);
            if (!ok) break;
        } else {
            __syncthreads();
            if (tid == 0) sm.nfront = 0;
        }
        ntok = ln.aggregate(cutoff, t, tb);
        if (ntok < 0) { ok = false; break; }
        ln.c_next += ntok;
        if (p.want_lattice) {
            ok = ln.lattice(cutoff, t, tbp, np, tb, ntok, lb);
            lb += sm.nlat;
        }
        if (tid == 0) {
            io.tok_base[t + 1] = tb + ntok;
            if (p.want_lattice) io.lat_base[t + 1] = lb;
        }
        ln.reset();
        tdone = t;
    }
    if (!ok) ln.reset();
    __syncthreads();

    // ---- counters ----
    const unsigned long long s_scan = block_sum<unsigned long long>(ln.c_scan, sm);
    const unsigned long long s_cand = block_sum<unsigned long long>(ln.c_cand, sm);
    const unsigned long long s_escan = block_sum<unsigned long long>(ln.c_escan, sm);
    const unsigned long long s_ecand = block_sum<unsigned long long>(ln.c_ecand, sm);
    if (tid == 0) {
        io.out_c[0] = ln.c_tok;
        io.out_c[1] = (long long)s_scan;
        io.out_c[2] = (long long)s_cand;
        io.out_c[3] = ln.c_front;
        io.out_c[4] = (long long)s_escan;
        io.out_c[5] = (long long)s_ecand;
        io.out_c[6] = ln.c_next;
        io.out_c[7] = lb;
        __stcg(L.round_ctr, ln.round_id);
        io.out_i[5] = tdone;
    }
    if (!ok || sm.err) {
        if (tid == 0) {
            io.out_i[0] = sm.err ? sm.err : E_INT_INIT;
            io.out_i[1] = sm.err_frame;
            io.out_d[2] = (double)sm.err_aux;
        }
        return;
    }

    // ---- final selection (decoder.py:578-586): argmin, ties -> smallest state ----
    double bt = inf, bc = inf;
    int st = 0x7FFFFFFF, sc = 0x7FFFFFFF;
    for (int j = tid; j < ntok; j += blockDim.x) {
        const unsigned s = __ldcg(io.tok_state + tb + j);
        const double c = __ldcg(io.tok_cost + tb + j);
        const double tot = __dadd_rn(c, __ldg(g.fin + s));
        if (tot < bt || (tot == bt && (int)s < st)) { bt = tot; st = (int)s; }
        if (c < bc || (c == bc && (int)s < sc)) { bc = c; sc = (int)s; }
    }
    block_argmin(bt, st, sm);
    block_argmin(bc, sc, sm);
    const bool partial = !(bt < inf);
    const int bstate = partial ? sc : st;
    if (tid == 0) {
        const double total = partial ? bc : bt;
        const int bidx = __ldcg(L.tokidx + bstate);
        io.out_i[2] = partial;
        io.out_i[3] = bidx;
        io.out_d[0] = total;
        io.out_d[1] = total;
        // ---- backtrace (decoder.py:614-641), bounded ----
        int f = T, i = bidx, hops = 0, err = 0;
        long long steps = 0;
        const long long limit = tb + ntok + 1;
        for (;;) {
            const long long base = io.tok_base[f];
            const int a = __ldcg(io.tok_arc + base + i);
            const int pr = __ldcg(io.tok_pred + base + i);
            if (a < 0) {
                if (f != 0) err = E_INT_INIT;
                break;
            }
            if (hops >= io.path_cap) { err = E_CAP_PATH; break; }
            io.path[hops++] = a;
            i = pr >> 1;
            if (pr & 1) f--;
            if (++steps > limit) { err = E_INT_BACKTRACE; break; }
        }
        for (int k = 0; k < hops / 2; k++) {
            const int x = io.path[k];
            io.path[k] = io.path[hops - 1 - k];
            io.path[hops - 1 - k] = x;
        }
        io.out_i[4] = hops;
        io.out_i[0] = err;
        io.out_i[1] = err ? f : 0;
    }
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
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
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
// Single-op surfaces (decoder.py:373-435), one CTA.
//   mode 0 = expand_emitting: tokens at io.tok_*[0..n) with tokidx set; acrow
//            (scaled) at io.costs; writes (state, cost) winners <= cutoff to
//            io.tok_state/tok_cost[n ...] and cutoff to io.out_d[0].
//   mode 1 = expand_nonemitting: seeds at io.tok_*[0..n) act as won entries
//            pack(cost, 0); closes under `cutoff`; writes the merged frontier.
// ===========================================================================
__global__ void __launch_bounds__(1024, 1)
expand_kernel(GraphDev g, Params p, LaneWs L, UttDesc io, int n, int mode, double cutoff_in) {
    __shared__ Smem sm;
    extern __shared__ double s_acrow[];
    const int tid = threadIdx.x;
    if (tid == 0) {
        sm.ntouched = sm.nfront = sm.nnext = sm.ntok = sm.nlat = sm.err = sm.err_frame = 0;
        sm.err_aux = 0;
    }
    for (int b = tid; b < NBINS; b += blockDim.x) sm.hist[b] = 0;
    __syncthreads();
    Lane ln(g, p, L, io, sm, s_acrow);
    ln.round_id = __ldcg(L.round_ctr);
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    double cutoff = cutoff_in;
    if (mode == 0) {
        ln.load_row(io.costs);
        __syncthreads();
        const double best = ln.emit(io.tok_state, io.tok_cost, n);
        if (!(best < inf)) {
            cutoff = inf;
        } else {
            cutoff = __dadd_rn(best, p.beam);
            ln.winners(io.tok_cost, cutoff, best);
        }
    } else {
        for (int i = tid; i < n; i += blockDim.x) {
            const unsigned s = __ldcg(io.tok_state + i);
            const double c = __ldcg(io.tok_cost + i);
            __stcg(L.pack + s, pack_word(c, 0u));
            __stcg(L.cost + s, c);
            __stcg(L.pred + s, -1);
            __stcg(L.touched + i, s);
            __stcg(ln.fs + i, s);
            __stcg(ln.fc + i, c);
        }
        __syncthreads();
        if (tid == 0) { sm.ntouched = n; sm.nfront = n; }
        __syncthreads();
        if (!ln.epsilon(cutoff, 0)) {
            if (tid == 0) io.out_i[0] = sm.err;
        }
    }
    __syncthreads();
    const int nt = sm.ntouched;
    for (int k = tid; k < nt; k += blockDim.x) {
        const unsigned v = __ldcg(L.touched + k);
        const double c = __ldcg(L.cost + v);
        if (c <= cutoff) {
            const int idx = agg_append(&sm.ntok);
            __stcg(io.tok_state + n + idx, v);
            __stcg(io.tok_cost + n + idx, c);
        }
    }
    __syncthreads();
    if (tid == 0) {
        io.out_i[4] = sm.ntok;
        io.out_d[0] = cutoff;
        __stcg(L.round_ctr, ln.round_id);
    }
    ln.reset();
}

// Fill helpers.
__global__ void fill_f64(double *p, double v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}
__global__ void set_tokidx(int *tokidx, const unsigned *states, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) tokidx[states[i]] = i;
}

}  // namespace lbk
