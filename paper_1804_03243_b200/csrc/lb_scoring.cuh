// lb_scoring.cuh — batch lattice oracle word error on the GPU.
//
// oracle_wer (scoring.py:66-114 of `latbeam`) is the fewest word errors over
// all complete lattice paths: a shortest path in the product graph
// (node, ref position j) with
//   (u, j) -> (u, j+1)  cost 1                    deletion
//   arc u->v, olabel 0:  (u, j) -> (v, j)   cost 0 epsilon output
//   arc u->v, olabel w:  (u, j) -> (v, j)   cost 1 insertion
//                        (u, j) -> (v, j+1) cost [w != ref[j]]  match / substitution
// The reference sweeps all arcs to a fixpoint; the distances are unique, so
// any exact shortest-path order gives the same integers.  Here one CTA scores
// one lattice: node ids are sorted by (frame, index), emitting arcs go from
// frame f-1 to f and epsilon arcs stay inside a frame, so frames are processed
// in order -- incoming emitting arcs, deletion closure, then the in-frame
// epsilon arcs to a fixpoint -- and every arc is relaxed about once.
#pragma once
#include "lb_device.cuh"

namespace lbk {

constexpr int WER_INF = 0x3FFFFFFF;

struct WerJob {
    const int *from, *to, *ol;   // arcs, sorted by from (FinalLattice canonical order)
    const int *nb;               // [F+1] first node of each frame
    const int *ab;               // [F+1] first arc whose from-node is in each frame
    const int *finals;           // final node ids
    const int *ref;              // reference words
    int *best;                   // [num_nodes][r+1] DP table (scratch)
    int num_nodes, start, n_final, F, r;
    long long *out;              // errors, or -1 (no complete path) / -2 (no convergence)
};

__device__ __forceinline__ bool wer_relax(const WerJob &J, int u, int v, int w, int j) {
    const int r1 = J.r + 1;
    const int b = __ldcg(J.best + (long long)u * r1 + j);
    if (b >= WER_INF) return false;
    bool ch = false;
    int *bv = J.best + (long long)v * r1;
    if (w == 0) {
        ch |= atomicMin(bv + j, b) > b;
    } else {
        ch |= atomicMin(bv + j, b + 1) > b + 1;
        if (j < J.r) {
            const int c = b + (w != J.ref[j] ? 1 : 0);
            ch |= atomicMin(bv + j + 1, c) > c;
        }
    }
    return ch;
}

// deletion closure of one node: best[v][j] = min(best[v][j], best[v][j-1] + 1)
__device__ __forceinline__ void wer_close(const WerJob &J, int v) {
    int *bv = J.best + (long long)v * (J.r + 1);
    int prev = __ldcg(bv);
    for (int j = 1; j <= J.r; j++) {
        const int x = __ldcg(bv + j);
        const int y = prev + 1 < x ? prev + 1 : x;
        if (y != x) __stcg(bv + j, y);
        prev = y;
    }
}

__global__ void __launch_bounds__(1024) oracle_wer_kernel(const WerJob *jobs, int n_jobs) {
    __shared__ int s_changed;
    if ((int)blockIdx.x >= n_jobs) return;
    const WerJob J = jobs[blockIdx.x];
    const int tid = threadIdx.x, bd = blockDim.x, r1 = J.r + 1;
    for (long long i = tid; i < (long long)J.num_nodes * r1; i += bd) J.best[i] = WER_INF;
    __syncthreads();
    if (tid == 0) J.best[(long long)J.start * r1] = 0;
    __syncthreads();
    for (int f = 0; f < J.F; f++) {
        const int n0 = J.nb[f], n1 = J.nb[f + 1];
        if (f > 0) {   // emitting arcs from frame f-1 into frame f
            const int a0 = J.ab[f - 1], a1 = J.ab[f];
            for (long long q = tid; q < (long long)(a1 - a0) * r1; q += bd) {
                const int k = a0 + (int)(q / r1), j = (int)(q % r1);
                const int v = J.to[k];
                if (v >= n0) wer_relax(J, J.from[k], v, J.ol[k], j);
            }
            __syncthreads();
        }
        for (int v = n0 + tid; v < n1; v += bd) wer_close(J, v);
        __syncthreads();
        // in-frame epsilon arcs to a fixpoint
        const int a0 = J.ab[f], a1 = J.ab[f + 1];
        for (int it = 0;; it++) {
            if (tid == 0) s_changed = 0;
            __syncthreads();
            bool ch = false;
            for (long long q = tid; q < (long long)(a1 - a0) * r1; q += bd) {
                const int k = a0 + (int)(q / r1), j = (int)(q % r1);
                const int v = J.to[k];
                if (v < n1) ch |= wer_relax(J, J.from[k], v, J.ol[k], j);
            }
            if (ch) s_changed = 1;
            __syncthreads();
            const int changed = s_changed;
            if (!changed) break;
            for (int v = n0 + tid; v < n1; v += bd) wer_close(J, v);
            __syncthreads();
            if (it > (n1 - n0) * r1 + 2) {
                if (tid == 0) *J.out = -2;
                return;
            }
        }
    }
    // best complete path: min over final nodes of best[f][r]
    __syncthreads();
    if (tid == 0) {
        int m = WER_INF;
        for (int i = 0; i < J.n_final; i++) {
            const int x = __ldcg(J.best + (long long)J.finals[i] * r1 + J.r);
            m = x < m ? x : m;
        }
        *J.out = m >= WER_INF ? -1 : m;
    }
}

}  // namespace lbk
