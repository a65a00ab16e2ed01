// lb_batched.cuh — frame-synchronous batched decode (the default throughput mode).
//
// The persistent-lane kernel (lb_kernels.cuh decode_kernel) gives each utterance
// a 2-CTA cluster and walks all of its frames inside one launch; every phase of
// a frame is then a short dependent chain on 2 SMs, and the lane is latency
// bound.  This mode turns each phase of a frame into ONE
// GPU-wide kernel over all lanes of the wave (Kaldi's batched CUDA decoder
// organises its channels the same way): blockIdx.y is the lane, blockIdx.x
// splits the lane's work, every block runs at full occupancy, and kernel
// boundaries are the phase barriers.  Per-lane control state lives in global
// memory (LaneCtl).  The epsilon closure, whose rounds are inherently
// sequential and small, stays a per-lane cluster kernel.
//
// Per frame t >= 1:  emit -> winners -> max_active -> [epsilon] -> aggregate -> turnover
// (frame 0:          init -> [epsilon] -> aggregate -> turnover; after the last frame: final).
// Semantics are exactly those of the lane kernel (same device functions for the
// arithmetic, the packed word, the tie-break, the Jacobi rounds and max-active).
#pragma once
#include "lb_kernels.cuh"

namespace lbk {

struct LaneCtl {
    int active;              // still decoding
    int err, err_frame;      // first error (E_*), frame
    int dirty;               // per-state records touched and not yet reset
    long long err_aux;
    int t, T;                // current frame, utterance length
    int ntok;                // tokens of frame t-1 (input of emit)
    int ntok_new;            // tokens appended by this frame's aggregate
    long long tbp, tb;       // arena offsets of frame t-1 / frame t
    unsigned long long best; // enc64 frame best (SENT = none)
    double cutoff, beam_eff;
    int ncand, ntouched, nseed, nfix_prev, nfix;
    int nfr[3];
    unsigned round_id;
    int nlat;
    long long lb;            // lattice arena offset of this frame
    unsigned long long c[8]; // work counters
    int hist[NBINS];         // max-active histogram of this frame
};

__device__ __forceinline__ void ctl_error(LaneCtl &c, int code, int frame, long long aux) {
    if (atomicCAS(&c.err, 0, code) == 0) {
        c.err_frame = frame;
        c.err_aux = aux;
    }
    c.active = 0;
}

__device__ __forceinline__ double b_ac(const double *row, unsigned il, double scale) {
    return __dmul_rn(__ldg(row + il - 1), scale);
}

constexpr int BNT = 256;           // threads per block of the phase kernels
constexpr int BNW = BNT / 32;
constexpr int BUNR = 2;            // arcs per thread per emit batch
constexpr int BWUNR = 4;           // candidates per thread per winners batch
constexpr int BAUNR = 2;           // touched states per thread per aggregate batch
constexpr int BCCH = 256;          // candidate chunk per warp
constexpr int BATCHED_MAX_UTTS = 44;   // host: batched mode up to this many utterances per call

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) b_init(const GraphDev g, const Params p, const LaneWs *lanes,
                                             const UttDesc *utts, LaneCtl *ctl, int n) {
    const int l = blockIdx.x;
    if (l >= n || threadIdx.x != 0) return;
    LaneCtl &c = ctl[l];
    const LaneWs &L = lanes[l];
    const UttDesc &io = utts[l];
    c.active = 1;
    c.err = c.err_frame = 0;
    c.dirty = 1;
    c.err_aux = 0;
    c.t = 0;
    c.T = io.T;
    c.ntok = 0;
    c.ntok_new = 0;
    c.tbp = c.tb = 0;
    c.best = SENT;
    c.cutoff = __dadd_rn(0.0, p.beam);
    c.beam_eff = p.beam;
    c.ncand = c.nseed = c.nfix_prev = c.nfix = 0;
    c.ntouched = 1;
    c.nfr[0] = g.has_eps ? 1 : 0;
    c.nfr[1] = c.nfr[2] = 0;
    c.round_id = __ldcg(L.round_ctr);
    c.nlat = 0;
    c.lb = 0;
    for (int k = 0; k < 8; k++) c.c[k] = 0;
    for (int b = 0; b < NBINS; b++) c.hist[b] = 0;
    StateRec *r = &L.rec[g.start];
    __stcg(&r->pack, pack_word(0.0, 0u));
    __stcg(&r->cost, 0.0);
    __stcg(&r->pred, -1);
    __stcg(L.touched, (unsigned)g.start);
    if (g.has_eps) __stcg(L.fr, (unsigned)g.start);
    io.tok_base[0] = 0;
    if (p.want_lattice) io.lat_base[0] = 0;
}

// ---------------------------------------------------------------------------
// emit: walk frame t-1's tokens; RED.MIN recombination; candidates -> lane buffer.
// Also maps frame t-1's epsilon predecessors to token indices (fix list).
__global__ void __launch_bounds__(BNT, 4) b_emit(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
                                                 const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ utts,
                                                 LaneCtl *__restrict__ ctl, int n) {
    __shared__ int own_s[BNW][WMAP];
    const int l = blockIdx.y;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const LaneWs &L = lanes[l];
    const UttDesc &io = utts[l];
    const int t = c.t;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const long long tbp = c.tbp;
    const int np = c.ntok;
    // epsilon predecessors of frame t-1 (source state -> token index)
    if (g.has_eps) {
        const int nfx = c.nfix_prev;
        for (int q = blockIdx.x * BNT + threadIdx.x; q < nfx; q += gridDim.x * BNT) {
            const long long o = tbp + (long long)__ldcg(L.fix + q);
            const int u = __ldcg(io.tok_pred + o) >> 1;
            const int pi = __ldcg(&L.rec[u].tokidx);
            if (pi < 0 || pi >= np || __ldcg(io.tok_state + tbp + pi) != (unsigned)u)
                ctl_error(c, E_INT_EPS_PRED, t - 1, u);
            __stcg(io.tok_pred + o, pi << 1);
        }
    }
    const double *row = io.costs + (long long)(t - 1) * p.D;
    const double beam_eff = c.beam_eff;
    StateRec *rec = L.rec;
    int4 *cb = L.cand;
    int *cbi = L.candi;
    const long long ccap = L.ccap;
    unsigned long long *run = &c.best;
    unsigned c_scan = 0, c_cand = 0;
    int cstart = 0, cused = BCCH;
    bool overflow = false;
    auto fill_tail = [&]() {
        for (int i = cused + lane; i < BCCH; i += 32) __stcs(cb + cstart + i, make_int4(-1, 0, 0, 0));
    };
    for_each_token_arc_batched<BUNR>(g, blockIdx.x * BNW + warp, gridDim.x * BNW, io.tok_state + tbp,
                                     io.tok_cost + tbp, np, c_scan, own_s[warp],
                                     [&](const bool *vv, const int *ii, const unsigned *aa, const double *cc) {
        int4 r[BUNR];
#pragma unroll
        for (int u = 0; u < BUNR; u++)
            if (vv[u]) r[u] = __ldg(g.arcs + aa[u]);
        unsigned long long known = __ldcg(run);
        double cand[BUNR];
        double bmin = inf_d();
#pragma unroll
        for (int u = 0; u < BUNR; u++) {
            cand[u] = inf_d();
            const unsigned il = vv[u] ? arc_il(r[u].y) : 0u;
            if (il != 0) {
                const double w = __hiloint2double(r[u].w, r[u].z);
                cand[u] = __dadd_rn(__dadd_rn(cc[u], w), b_ac(row, il, p.scale));
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
            if (lane == 0) red_min_u64(run, eb);
            known = eb < known ? eb : known;
        }
        unsigned bound_key = 0xFFFFFFFFu;
        if (known != SENT) bound_key = (unsigned)(pack_word(__dadd_rn(dec64(known), beam_eff), 0u) >> 32);
        bool em[BUNR];
        int off[BUNR];
        int tot = 0;
#pragma unroll
        for (int u = 0; u < BUNR; u++) {
            em[u] = false;
            if (cand[u] < inf_d()) {
                const unsigned long long word = pack_word(cand[u], aa[u]);
                em[u] = (unsigned)(word >> 32) <= bound_key;
                if (em[u]) red_min_u64(&rec[r[u].x].pack, word);
            }
            const unsigned bb = __ballot_sync(FULL, em[u]);
            off[u] = tot + __popc(bb & lt);
            tot += __popc(bb);
        }
        if (tot == 0) return;
        c_cand += (lane == 0) ? (unsigned)tot : 0u;
        if (cused + tot > BCCH) {
            if (cused < BCCH && !overflow) fill_tail();
            int nb = 0;
            if (lane == 0) nb = atomicAdd(&c.ncand, BCCH);
            cstart = __shfl_sync(FULL, nb, 0);
            cused = 0;
            if ((long long)cstart + BCCH > ccap) {
                overflow = true;
                if (lane == 0) ctl_error(c, E_CAP_CAND, t, (long long)cstart + BCCH);
            }
        }
        if (!overflow) {
#pragma unroll
            for (int u = 0; u < BUNR; u++) {
                if (em[u]) {
                    const long long bits = __double_as_longlong(cand[u]);
                    const unsigned flag = (unsigned)r[u].y & EPS_FLAG;
                    const int k = cstart + cused + off[u];
                    __stcs(cb + k, make_int4((int)((unsigned)r[u].x | flag), (int)aa[u], (int)(bits & 0xFFFFFFFFll),
                                             (int)(bits >> 32)));
                    __stcs(cbi + k, ii[u]);
                }
            }
        }
        cused += tot;
    });
    if (cused < BCCH && !overflow) fill_tail();
    c_cand = warp_sum(c_cand);
    c_scan = warp_sum(c_scan);
    if (lane == 0) {
        atomicAdd(&c.c[1], (unsigned long long)c_scan);
        atomicAdd(&c.c[2], (unsigned long long)c_cand);
    }
}

// ---------------------------------------------------------------------------
// winners: owner test per candidate; touched list; seeds -> round-0 frontier and histogram.
__global__ void __launch_bounds__(BNT, 4) b_winners(const __grid_constant__ GraphDev g,
                                                    const __grid_constant__ Params p,
                                                    const LaneWs *__restrict__ lanes, LaneCtl *__restrict__ ctl,
                                                    int n) {
    __shared__ unsigned stage_s[BNW][2][SW];
    __shared__ int hist_s[NBINS];
    const int l = blockIdx.y;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const unsigned long long bk = c.best;
    if (bk == SENT) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl_error(c, E_DEAD_NO_CAND, c.t, 0);
        return;
    }
    const LaneWs &L = lanes[l];
    const double best = dec64(bk);
    const double cutoff = __dadd_rn(best, c.beam_eff);
    const bool hist = p.max_active > 0;
    const double width = __ddiv_rn(p.beam, (double)NBINS);
    const double inv_w = __drcp_rn(width);
    const int nc = c.ncand;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (hist)
        for (int b = threadIdx.x; b < NBINS; b += BNT) hist_s[b] = 0;
    __syncthreads();
    StateRec *rec = L.rec;
    const int4 *cb = L.cand;
    const int *cbi = L.candi;
    WStage st_t, st_f;
    st_t.buf = stage_s[warp][0];
    st_t.n = 0;
    st_f.buf = stage_s[warp][1];
    st_f.n = 0;
    unsigned nseed = 0;
    const int gw = blockIdx.x * BNW + warp, gnw = gridDim.x * BNW;
    for (int kb = gw * 32 * BWUNR; kb < nc; kb += gnw * 32 * BWUNR) {
        int4 e[BWUNR];
        int ti[BWUNR];
#pragma unroll
        for (int u = 0; u < BWUNR; u++) {
            const int k = kb + u * 32 + lane;
            e[u].x = -1;
            if (k < nc) {
                e[u] = __ldcs(cb + k);
                if (e[u].x != -1) ti[u] = __ldcs(cbi + k);
            }
        }
        unsigned long long pk[BWUNR];
#pragma unroll
        for (int u = 0; u < BWUNR; u++)
            pk[u] = e[u].x != -1 ? __ldcg(&rec[(unsigned)e[u].x & ~EPS_FLAG].pack) : 0ull;
#pragma unroll
        for (int u = 0; u < BWUNR; u++) {
            const unsigned v = (unsigned)e[u].x & ~EPS_FLAG;
            const double cand = __hiloint2double(e[u].w, e[u].z);
            const bool own = e[u].x != -1 && pk[u] == pack_word(cand, (unsigned)e[u].y);
            if (own) store_winner(&rec[v], cand, (ti[u] << 1) | 1);
            st_t.push(own, v, &c.ntouched, L.touched);
            const bool seed = own && cand <= cutoff;
            nseed += seed;
            st_f.push(seed && ((unsigned)e[u].x & EPS_FLAG), v, &c.nfr[0], L.fr);
            if (hist && seed) atomicAdd(hist_s + hist_bin(cand, best, width, inv_w), 1);
        }
    }
    st_t.flush(&c.ntouched, L.touched);
    st_f.flush(&c.nfr[0], L.fr);
    nseed = warp_sum(nseed);
    if (lane == 0 && nseed) atomicAdd(&c.nseed, (int)nseed);
    if (hist) {
        __syncthreads();
        for (int b = threadIdx.x; b < NBINS; b += BNT)
            if (hist_s[b]) atomicAdd(&c.hist[b], hist_s[b]);
    }
}

// ---------------------------------------------------------------------------
// max-active cutoff and adaptive beam; one warp per lane.
__global__ void __launch_bounds__(32) b_max_active(const Params p, LaneCtl *ctl, int n) {
    const int l = blockIdx.x;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const int lane = threadIdx.x;
    const double best = dec64(c.best);
    double cutoff = __dadd_rn(best, c.beam_eff);
    const int ns = c.nseed;
    if (ns == 0) {
        if (lane == 0) ctl_error(c, E_DEAD_NO_TOKENS, c.t, 0);
        return;
    }
    bool tightened = false;
    constexpr int PER = NBINS / 32;
    if (p.max_active > 0 && ns > p.max_active) {
        int loc[PER];
        int sum = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            loc[q] = c.hist[lane * PER + q];
            sum += loc[q];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int x = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += x;
        }
        long long cum = incl - sum;
        int found = -1;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            cum += loc[q];
            if (found < 0 && cum > p.max_active) found = lane * PER + q;
        }
        const unsigned m = __ballot_sync(FULL, found >= 0);
        if (m) {
            const int bstar = __shfl_sync(FULL, found, __ffs(m) - 1);
            const double width = __ddiv_rn(p.beam, (double)NBINS);
            const double h = __dadd_rn(best, __dmul_rn((double)(bstar < 1 ? 1 : bstar), width));
            if (h < cutoff) {
                cutoff = h;
                tightened = true;
            }
        }
    }
    if (p.max_active > 0)
        for (int b = lane; b < NBINS; b += 32) c.hist[b] = 0;
    if (lane == 0) {
        c.cutoff = cutoff;
        if (tightened) {
            const double be = __dadd_rn(__dsub_rn(cutoff, best), MAX_ACTIVE_BEAM_DELTA);
            c.beam_eff = be < p.beam ? be : p.beam;
        } else {
            c.beam_eff = p.beam;
        }
    }
}

// ---------------------------------------------------------------------------
// epsilon closure: one cluster per lane, Jacobi rounds with one cluster barrier
// each (same round-winner scheme as Lane::epsilon); lane lists in global memory.
template <int NT>
__global__ void __launch_bounds__(NT, 1) b_epsilon(const __grid_constant__ GraphDev g,
                                                   const __grid_constant__ Params p,
                                                   const LaneWs *__restrict__ lanes, LaneCtl *__restrict__ ctl,
                                                   int n) {
    cgx::cluster_group cl = cgx::this_cluster();
    const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int l = blockIdx.x / C;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    if (!__ldcg(&c.active)) return;   // uniform across the cluster (read before any write this launch)
    const LaneWs &L = lanes[l];
    const double cutoff = c.cutoff;
    const int frame = c.t;
    const bool LAT = p.want_lattice;
    StateRec *rec = L.rec;
    const int gtid = rank * NT + threadIdx.x, gstride = C * NT;
    unsigned round_id = c.round_id;
    unsigned c_escan = 0, c_ecand = 0, c_front = 0;
    bool ok = true;
    for (int r = 0;; r++) {
        const int nf = __ldcg(&c.nfr[r % 3]);
        if (nf == 0) break;
        if (r > g.S + 1) {
            if (gtid == 0) ctl_error(c, E_INT_EPS_ROUNDS, frame, 0);
            ok = false;
            break;
        }
        ++round_id;
        const unsigned *fs = L.fr + (size_t)(r & 1) * L.S;
        unsigned *fsn = L.fr + (size_t)((r + 1) & 1) * L.S;
        int *nnext = &c.nfr[(r + 1) % 3];
        if (gtid == 0) c.nfr[(r + 2) % 3] = 0;
        EpsWin *rprev = L.rpk + (size_t)((r + 1) & 1) * L.S;
        EpsWin *rcur = L.rpk + (size_t)(r & 1) * L.S;
        for (int k = gtid; k < nf; k += gstride) {
            const unsigned v = __ldcg(fs + k);
            const uint2 er = __ldg(g.erng + v);
            double cu;
            unsigned src = 0;
            if (r == 0) {
                cu = rld_f64(&rec[v].cost);
            } else {
                const ulonglong2 w2 = rld_u128(rprev + v);
                rst_u128(rprev + v, make_ulonglong2(~0ull, ~0ull));
                cu = __longlong_as_double((long long)w2.y);
                src = __ldg(g.src + (unsigned)w2.x);   // stored after the offers (see the lane kernel)
            }
            if (cu <= cutoff) {
                c_front++;
                if (LAT) {
                    const double m = rld_f64(&rec[v].minsnap);
                    if (cu < m) rst_f64(&rec[v].minsnap, cu);
                }
                c_escan += er.y - er.x;
                for (unsigned e = er.x; e < er.y; ++e) {
                    const int4 rr = __ldg(g.eps + e);
                    const double cand = __dadd_rn(cu, __hiloint2double(rr.w, rr.z));
                    if (!(cand <= cutoff)) continue;
                    c_ecand++;
                    const unsigned x = (unsigned)rr.x;
                    const unsigned long long word = pack_word(cand, (unsigned)rr.y);
                    const unsigned long long old = atom_min_u64(&rec[x].pack, word);
                    if (old == SENT) {
                        const int sl = agg_append(&c.ntouched);
                        __stcg(L.touched + sl, x);
                    }
                    if (old > word) {
                        const unsigned tg = atom_exch_u32(L.tag + x, round_id);
                        epswin_min(rcur + x, word, cand);
                        if (tg != round_id) {
                            const int sl = agg_append(nnext);
                            __stcg(fsn + sl, x);
                        }
                    }
                }
            }
            if (r > 0) store_winner(&rec[v], cu, (int)(src << 1));
        }
        cl.sync();
    }
    c_escan = warp_sum(c_escan);
    c_ecand = warp_sum(c_ecand);
    c_front = warp_sum(c_front);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&c.c[3], (unsigned long long)c_front);
        atomicAdd(&c.c[4], (unsigned long long)c_escan);
        atomicAdd(&c.c[5], (unsigned long long)c_ecand);
    }
    if (ok) {
        cl.sync();   // every CTA has read c.round_id before it moves on
        if (gtid == 0) c.round_id = round_id;
    }
}

// ---------------------------------------------------------------------------
// aggregate: touched states under the cutoff become frame t's tokens (staged per
// warp, lane-wide indices in bulk), words reset, epsilon-pred fixes listed.
__global__ void __launch_bounds__(BNT, 4) b_aggregate(const __grid_constant__ GraphDev g,
                                                      const __grid_constant__ Params p,
                                                      const LaneWs *__restrict__ lanes,
                                                      const UttDesc *__restrict__ utts, LaneCtl *__restrict__ ctl,
                                                      int n) {
    __shared__ double s_cost[BNW][SWT], s_ms[BNW][SWT];
    __shared__ unsigned s_v[BNW][SWT], s_arc[BNW][SWT], s_key[BNW][SWT];
    __shared__ int s_pred[BNW][SWT];
    __shared__ unsigned s_fix[BNW][SW];
    const int l = blockIdx.y;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const LaneWs &L = lanes[l];
    const UttDesc &io = utts[l];
    const int frame = c.t;
    const double cutoff = c.cutoff;
    const long long tb = c.tb;
    const long long room = io.tok_cap - tb;
    const int nt = c.ntouched;
    StateRec *rec = L.rec;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int sn = 0;
    WStage sf;
    sf.buf = s_fix[warp];
    sf.n = 0;
    auto flush = [&]() {
        __syncwarp();
        if (sn == 0) return;
        int base = 0;
        if (lane == 0) base = atomicAdd(&c.ntok_new, sn);
        base = __shfl_sync(FULL, base, 0);
        for (int i0 = 0; i0 < sn; i0 += 32) {
            const int i = i0 + lane;
            bool fx = false;
            const int idx = base + i;
            if (i < sn && idx < room) {
                const unsigned v = s_v[warp][i];
                const bool init = frame == 0 && (int)v == g.start;
                const double cst = s_cost[warp][i];
                const int pr = s_pred[warp][i];
                const long long o = tb + idx;
                __stcg(io.tok_state + o, v);
                __stcg(io.tok_cost + o, init ? 0.0 : cst);
                __stcs(io.tok_arc + o, init ? -1 : (int)s_arc[warp][i]);
                __stcs(io.tok_pred + o, init ? -1 : pr);
                if (p.collect_packs)
                    __stcs(io.tok_pack + o, ((unsigned long long)s_key[warp][i] << 32) | s_arc[warp][i]);
                store_rec32(&rec[v], cst, pr, idx, SENT, s_ms[warp][i]);
                fx = !init && (pr & 1) == 0;
            } else if (i < sn) {
                __stcg(&rec[s_v[warp][i]].pack, SENT);
            }
            sf.push(fx, (unsigned)idx, &c.nfix, L.fix);
        }
        __syncwarp();
        sn = 0;
    };
    const int gw = blockIdx.x * BNW + warp, gnw = gridDim.x * BNW;
    for (int kb = gw * 32 * BAUNR; kb < nt; kb += gnw * 32 * BAUNR) {
        unsigned v[BAUNR];
#pragma unroll
        for (int u = 0; u < BAUNR; u++) {
            const int k = kb + u * 32 + lane;
            v[u] = k < nt ? __ldcg(L.touched + k) : 0xFFFFFFFFu;
        }
        RecView rv[BAUNR];
#pragma unroll
        for (int u = 0; u < BAUNR; u++)
            if (v[u] != 0xFFFFFFFFu) rv[u] = load_rec32(&rec[v[u]]);
#pragma unroll
        for (int u = 0; u < BAUNR; u++) {
            const bool valid = v[u] != 0xFFFFFFFFu;
            const bool init = valid && frame == 0 && (int)v[u] == g.start;
            const bool keep = valid && (init || rv[u].cost <= cutoff);
            if (valid && !keep) __stcg(&rec[v[u]].pack, SENT);
            const unsigned m = __ballot_sync(FULL, keep);
            if (keep) {
                const int j = sn + __popc(m & lt);
                s_v[warp][j] = v[u];
                s_cost[warp][j] = rv[u].cost;
                s_ms[warp][j] = rv[u].minsnap;
                s_arc[warp][j] = (unsigned)rv[u].pack;
                s_key[warp][j] = (unsigned)(rv[u].pack >> 32);
                s_pred[warp][j] = rv[u].pred;
            }
            sn += __popc(m);
            if (sn > SWT - 32) flush();
        }
    }
    flush();
    sf.flush(&c.nfix, L.fix);
}

// ---------------------------------------------------------------------------
// lattice arcs of block t (rule A.5, lattice.py:313-362): emitting arc live iff
// its candidate <= cutoff and its destination was kept; epsilon arc live iff both
// ends kept and min-snapshot(src) + w <= cutoff.  Resets minsnap.
__device__ __forceinline__ bool b_kept(const LaneWs &L, const UttDesc &io, unsigned v, long long tb, int n, int &j) {
    j = __ldcg(&L.rec[v].tokidx);
    return j >= 0 && j < n && __ldcg(io.tok_state + tb + j) == v;
}

__global__ void __launch_bounds__(BNT, 4) b_lattice(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
                                                    const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ utts,
                                                    LaneCtl *__restrict__ ctl, int n_lanes) {
    __shared__ int own_s[BNW][WMAP];
    const int l = blockIdx.y;
    if (l >= n_lanes) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const LaneWs &L = lanes[l];
    const UttDesc &io = utts[l];
    const int t = c.t;
    const int warp = threadIdx.x >> 5;
    const double cutoff = c.cutoff;
    const long long tb = c.tb, lb = c.lb;
    const int n = c.ntok_new;
    auto push = [&](int arc, int from, int to) {
        const int sl = agg_append(&c.nlat);
        const long long gs = lb + sl;
        if (gs < io.lat_cap) {
            __stcg(io.lat_arc + gs, arc);
            __stcg(io.lat_from + gs, from);
            __stcg(io.lat_to + gs, to);
        }
    };
    if (t > 0) {
        const double *row = io.costs + (long long)(t - 1) * p.D;
        unsigned dummy = 0;
        for_each_token_arc_batched<BUNR>(g, blockIdx.x * BNW + warp, gridDim.x * BNW, io.tok_state + c.tbp,
                                         io.tok_cost + c.tbp, c.ntok, dummy, own_s[warp],
                                         [&](const bool *vv, const int *ii, const unsigned *aa, const double *cc) {
#pragma unroll
            for (int u = 0; u < BUNR; u++) {
                if (!vv[u]) continue;
                const int4 r = __ldg(g.arcs + aa[u]);
                const unsigned il = arc_il(r.y);
                if (il == 0) continue;
                const double cand = __dadd_rn(__dadd_rn(cc[u], __hiloint2double(r.w, r.z)), b_ac(row, il, p.scale));
                int j;
                if (cand <= cutoff && b_kept(L, io, (unsigned)r.x, tb, n, j)) push((int)aa[u], ii[u], j);
            }
        });
    }
    if (g.has_eps) {
        const double inf = inf_d();
        for (int j = blockIdx.x * BNT + threadIdx.x; j < n; j += gridDim.x * BNT) {
            const unsigned u = __ldcg(io.tok_state + tb + j);
            const unsigned e0 = __ldg(g.eoff + u), e1 = __ldg(g.eoff + u + 1);
            const double ms = __ldcg(&L.rec[u].minsnap);
            __stcg(&L.rec[u].minsnap, inf);
            for (unsigned e = e0; e < e1; ++e) {
                const int4 r = __ldg(g.eps + e);
                int jv;
                if (__dadd_rn(ms, __hiloint2double(r.w, r.z)) <= cutoff && b_kept(L, io, (unsigned)r.x, tb, n, jv))
                    push(r.y, j, jv);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// turnover: close frame t (checks, offsets, counters), open frame t+1.
__global__ void __launch_bounds__(32) b_turnover(const Params p, const UttDesc *utts, LaneCtl *ctl, int n) {
    const int l = blockIdx.x;
    if (l >= n || threadIdx.x != 0) return;
    LaneCtl &c = ctl[l];
    if (!c.active) return;
    const UttDesc &io = utts[l];
    const int t = c.t;
    const int k = c.ntok_new;
    const long long room = io.tok_cap - c.tb;
    if (k == 0 || (long long)k > p.max_tokens || (long long)k > room) {
        if (k == 0) ctl_error(c, E_DEAD_NO_TOKENS, t, 0);
        else if ((long long)k > p.max_tokens) ctl_error(c, E_CAP_TOKENS, t, k);
        else ctl_error(c, E_CAP_ARENA, t, c.tb + k);
        c.dirty = 0;   // aggregate has reset every word it touched
        return;
    }
    io.tok_base[t + 1] = c.tb + k;
    if (p.want_lattice) {
        const long long lb = c.lb + c.nlat;
        if (lb > io.lat_cap) {
            ctl_error(c, E_CAP_LATTICE, t, lb);
            c.dirty = 0;
            return;
        }
        c.lb = lb;
        c.nlat = 0;
        io.lat_base[t + 1] = lb;
    }
    if (t > 0) c.c[6] += (unsigned long long)k;
    c.tbp = c.tb;
    c.tb += k;
    c.ntok = k;
    c.nfix_prev = c.nfix;
    c.nfix = 0;
    c.ncand = c.ntouched = c.nseed = c.ntok_new = 0;
    c.nfr[0] = c.nfr[1] = c.nfr[2] = 0;
    c.best = SENT;
    c.dirty = 0;
    if (t >= c.T) {
        c.active = 0;    // decoded to the end; b_final takes over
    } else {
        c.t = t + 1;
        c.c[0] += (unsigned long long)k;   // tokens the next emit expands
        c.dirty = 1;
    }
}

// ---------------------------------------------------------------------------
// final: last frame's epsilon predecessors, final selection (decoder.py:578-586),
// bounded backtrace (decoder.py:614-641), error reporting and cleanup.
template <int NT>
__global__ void __launch_bounds__(NT, 1) b_final(const __grid_constant__ GraphDev g, const __grid_constant__ Params p,
                                                 const LaneWs *__restrict__ lanes, const UttDesc *__restrict__ utts,
                                                 LaneCtl *__restrict__ ctl, int n) {
    __shared__ double red_v[32];
    __shared__ int red_s[32];
    __shared__ double bc_v;
    __shared__ int bc_s;
    const int l = blockIdx.x;
    if (l >= n) return;
    LaneCtl &c = ctl[l];
    const LaneWs &L = lanes[l];
    const UttDesc &io = utts[l];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
    if (tid == 0) {
        for (int k = 0; k < 8; k++) io.out_c[k] = (long long)c.c[k];
        io.out_c[7] = c.lb;
        __stcg(L.round_ctr, c.round_id);
        io.out_i[5] = c.err ? c.err_frame : c.T;
    }
    if (c.err) {
        if (c.dirty) {   // the failing frame's words were never reset
            const int nc = c.ncand;
            for (int k = tid; k < nc; k += NT) {   // emitted but maybe not yet listed as touched
                const int x = __ldcg(&L.cand[k].x);
                if (x != -1) __stcg(&L.rec[(unsigned)x & ~EPS_FLAG].pack, SENT);
            }
            const int nt = c.ntouched;
            for (int k = tid; k < nt; k += NT) {
                const unsigned v = __ldcg(L.touched + k);
                __stcg(&L.rec[v].pack, SENT);
                __stcg(&L.rec[v].minsnap, inf_d());
                __stcg(reinterpret_cast<ulonglong2 *>(L.rpk + v), make_ulonglong2(~0ull, ~0ull));
                __stcg(reinterpret_cast<ulonglong2 *>(L.rpk + L.S + v), make_ulonglong2(~0ull, ~0ull));
            }
        }
        if (tid == 0) {
            io.out_i[0] = c.err;
            io.out_i[1] = c.err_frame;
            io.out_d[2] = (double)c.err_aux;
        }
        return;
    }
    const int T = c.T;
    const long long tb = c.tbp;   // frame T's tokens
    const int ntok = c.ntok;
    // epsilon predecessors of the last frame
    if (g.has_eps) {
        for (int q = tid; q < c.nfix_prev; q += NT) {
            const long long o = tb + (long long)__ldcg(L.fix + q);
            const int u = __ldcg(io.tok_pred + o) >> 1;
            const int pi = __ldcg(&L.rec[u].tokidx);
            if (pi < 0 || pi >= ntok || __ldcg(io.tok_state + tb + pi) != (unsigned)u) {
                if (atomicCAS(&c.err, 0, E_INT_EPS_PRED) == 0) c.err_frame = T;
            }
            __stcg(io.tok_pred + o, pi << 1);
        }
        __syncthreads();
        if (c.err) {
            if (tid == 0) { io.out_i[0] = c.err; io.out_i[1] = c.err_frame; }
            return;
        }
    }
    const double inf = inf_d();
    double bt = inf, bc = inf;
    int st = 0x7FFFFFFF, sc = 0x7FFFFFFF;
    for (int j = tid; j < ntok; j += NT) {
        const unsigned s = __ldcg(io.tok_state + tb + j);
        const double cst = __ldcg(io.tok_cost + tb + j);
        const double tot = __dadd_rn(cst, __ldg(g.fin + s));
        if (tot < bt || (tot == bt && (int)s < st)) { bt = tot; st = (int)s; }
        if (cst < bc || (cst == bc && (int)s < sc)) { bc = cst; sc = (int)s; }
    }
    auto block_argmin = [&](double &v, int &s) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, v, o);
            const int os = __shfl_xor_sync(FULL, s, o);
            if (ov < v || (ov == v && os < s)) { v = ov; s = os; }
        }
        if (lane == 0) { red_v[warp] = v; red_s[warp] = s; }
        __syncthreads();
        if (warp == 0) {
            double x = lane < nw ? red_v[lane] : inf;
            int y = lane < nw ? red_s[lane] : 0x7FFFFFFF;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(FULL, x, o);
                const int os = __shfl_xor_sync(FULL, y, o);
                if (ov < x || (ov == x && os < y)) { x = ov; y = os; }
            }
            if (lane == 0) { bc_v = x; bc_s = y; }
        }
        __syncthreads();
        v = bc_v;
        s = bc_s;
        __syncthreads();
    };
    block_argmin(bt, st);
    block_argmin(bc, sc);
    if (tid != 0) return;
    const bool partial = !(bt < inf);
    const int bstate = partial ? sc : st;
    const double total = partial ? bc : bt;
    const int bidx = __ldcg(&L.rec[bstate].tokidx);
    io.out_i[2] = partial;
    io.out_i[3] = bidx;
    io.out_d[0] = total;
    io.out_d[1] = total;
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

}  // namespace lbk
