// lb_lattice.cuh — device-side lattice finalisation.
//
// After prune_kernel has flagged every live lattice arc with its extra cost,
// the final lattice of an utterance (lattice.py:537-598, `finalize_lattice`) is
// built on the device and only the surviving arcs leave the GPU:
//   1. token ranks: each frame's tokens sorted by state (the reference's
//      state-sorted FrameTokens order, decoder.py:330-370) -> rank per token;
//   2. survivors: arcs with extra <= lattice_beam (lattice.py:473-497);
//   3. per survivor: node keys (frame << 32 | rank) of both ends, labels,
//      graph cost and acoustic cost;
//   4. nodes: the sorted unique endpoint keys, dense ids by binary search;
//   5. canonical arc order: np.lexsort((ac, g, ol, il, to, from)) as six
//      stable LSD radix-sort passes (CUB), last key primary;
//   6. final nodes: last-frame nodes with a finite graph final cost (all of
//      them, cost 0, for a partial result).
#pragma once
#include <cub/cub.cuh>

#include "lb_device.cuh"

namespace lbk {

__device__ __forceinline__ int upper_frame(const long long *base, int nb, long long i) {
    // largest f with base[f] <= i, base has nb entries (non-decreasing)
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// token key = (frame << sbits) | state, sbits = bits of the largest state id, so
// the radix sort runs over sbits + frame bits only
__global__ void fl_token_keys(const unsigned *tok_state, const long long *tok_base, int nframes, long long ntok,
                              int sbits, unsigned long long *keys, int *idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ntok; i += (long long)gridDim.x * blockDim.x) {
        const int f = upper_frame(tok_base, nframes + 1, i);
        keys[i] = ((unsigned long long)f << sbits) | tok_state[i];
        idx[i] = (int)i;
    }
}

__global__ void fl_token_rank(const unsigned long long *skeys, const int *sidx, const long long *tok_base, long long ntok,
                              int sbits, int start_state, int *rank, long long *start_rank) {
    const unsigned long long smask = (1ull << sbits) - 1ull;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ntok; j += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(skeys[j] >> sbits);
        const int r = (int)(j - tok_base[f]);
        rank[sidx[j]] = r;
        if (f == 0 && (int)(skeys[j] & smask) == start_state) *start_rank = r;
    }
}

__global__ void fl_survivors(const double *extra, long long n, double beam, long long *out, unsigned long long *count) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        if (extra[k] <= beam) out[atomicAdd(count, 1ull)] = k;
    }
}

// -0.0 -> +0.0 then the order-preserving u64 (numpy sorts -0.0 == 0.0)
__device__ __forceinline__ unsigned long long fkey(double x) { return enc64(__dadd_rn(x, 0.0)); }

__global__ void fl_arc_fields(GraphDev g, const long long *surv, long long m, const int *lat_arc, const int *lat_from,
                              const int *lat_to, const long long *lat_base, const long long *tok_base, int nframes,
                              const int *rank, const double *costs, int D, double scale, unsigned long long *fk,
                              unsigned long long *tk, unsigned *il_out, unsigned *ol_out, double *g_out,
                              double *ac_out, unsigned long long *nodes) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < m; s += (long long)gridDim.x * blockDim.x) {
        const long long k = surv[s];
        const int b = upper_frame(lat_base, nframes + 1, k);
        const unsigned a = (unsigned)lat_arc[k];
        const int4 r = __ldg(g.arcs + a);
        const unsigned il = arc_il(r.y);
        const int ff = il > 0 ? b - 1 : b;
        const unsigned long long f = ((unsigned long long)ff << 32) | (unsigned)rank[tok_base[ff] + lat_from[k]];
        const unsigned long long t = ((unsigned long long)b << 32) | (unsigned)rank[tok_base[b] + lat_to[k]];
        fk[s] = f;
        tk[s] = t;
        il_out[s] = il;
        ol_out[s] = g.ol[a];
        g_out[s] = __hiloint2double(r.w, r.z);
        ac_out[s] = il > 0 ? __dmul_rn(costs[(long long)(b - 1) * D + il - 1], scale) : 0.0;
        nodes[2 * s] = f;
        nodes[2 * s + 1] = t;
    }
}

__device__ __forceinline__ int find_node(const unsigned long long *nodes, int n, unsigned long long key) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nodes[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void fl_node_ids(const unsigned long long *fk, const unsigned long long *tk, long long m,
                            const unsigned long long *nodes, int nn, unsigned *fid, unsigned *tid) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < m; s += (long long)gridDim.x * blockDim.x) {
        fid[s] = (unsigned)find_node(nodes, nn, fk[s]);
        tid[s] = (unsigned)find_node(nodes, nn, tk[s]);
    }
}

// key_out[i] = key(perm[i]) for one LSD pass
__global__ void fl_gather_u64(const double *x, const int *perm, long long m, unsigned long long *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        out[i] = fkey(x[perm[i]]);
}
__global__ void fl_gather_u32(const unsigned *x, const int *perm, long long m, unsigned *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        out[i] = x[perm[i]];
}
__global__ void fl_iota(int *p, long long m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

// final arrays in canonical order
__global__ void fl_emit(const int *perm, long long m, const unsigned *fid, const unsigned *tid, const unsigned *il,
                        const unsigned *ol, const double *gc, const double *ac, int *o_from, int *o_to, int *o_il,
                        int *o_ol, double *o_g, double *o_ac) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const int j = perm[i];
        o_from[i] = (int)fid[j];
        o_to[i] = (int)tid[j];
        o_il[i] = (int)il[j];
        o_ol[i] = (int)ol[j];
        o_g[i] = gc[j];
        o_ac[i] = ac[j];
    }
}

// final nodes: last-frame nodes (frame == T) with finite graph final cost of their state
__global__ void fl_finals(const unsigned long long *nodes, int nn, int T, const unsigned long long *skeys, int sbits,
                          const long long *tok_base, const double *fin, int partial, long long *ids, double *fcs,
                          unsigned long long *count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
        if ((int)(nodes[i] >> 32) != T) continue;
        const unsigned idx = (unsigned)nodes[i];
        const unsigned state = (unsigned)(skeys[tok_base[T] + idx] & ((1ull << sbits) - 1ull));
        const double fc = partial ? 0.0 : fin[state];
        if (partial || fc < __longlong_as_double(0x7FF0000000000000ll)) {
            const unsigned long long k = atomicAdd(count, 1ull);
            ids[k] = i;
            fcs[k] = fc;
        }
    }
}

// final nodes for a host-given work lattice: last-frame nodes whose token has a
// finite final cost (fc[idx], the reference's final_token_costs), or all of them
// with cost 0 for a partial result (lattice.py:576-580)
__global__ void fl_finals_given(const unsigned long long *nodes, int nn, int T, const double *fc, long long nfc,
                                int partial, long long *ids, double *fcs, unsigned long long *count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
        if ((int)(nodes[i] >> 32) != T) continue;
        const long long idx = (long long)(unsigned)nodes[i];
        const double c = partial ? 0.0 : (idx < nfc ? fc[idx] : __longlong_as_double(0x7FF0000000000000ll));
        if (partial || c < __longlong_as_double(0x7FF0000000000000ll)) {
            const unsigned long long k = atomicAdd(count, 1ull);
            ids[k] = i;
            fcs[k] = c;
        }
    }
}

}  // namespace lbk
