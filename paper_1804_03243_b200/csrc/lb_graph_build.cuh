// lb_graph_build.cuh — device-side build of the graph replica.
//
// lb_graph_create uploads the reference's CSR columns (wfst.py:33-90) as they are
// and builds the device layout on the GPU: the 16 B arc records with the
// EPS_FLAG bit, the per-state {first, end} ranges, the per-state epsilon CSR
// (records {dst, arc id, weight} in arc order) and the statistics the host
// needs.  Validation (wfst.py:128-176 rules: offsets non-decreasing, fields in
// range, weights finite and >= 0) runs in the same passes.  A 50M-arc graph
// builds in tens of milliseconds instead of seconds of host loops.
#pragma once
#include <cub/cub.cuh>

#include "lb_device.cuh"

namespace lbk {

enum : unsigned { GB_BAD_OFFSETS = 1u, GB_BAD_FIELD = 2u, GB_BAD_WEIGHT = 4u };

// per state: offsets as u32, arc range, epsilon / emitting out-degrees
__global__ void gb_state_pass(const long long *off, const int *il, long long S, unsigned *off32, uint2 *rng,
                              unsigned *ecnt, unsigned *emit, unsigned *err) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < S; s += (long long)gridDim.x * blockDim.x) {
        const long long lo = off[s], hi = off[s + 1];
        if (hi < lo) {
            atomicOr(err, GB_BAD_OFFSETS);
            ecnt[s] = emit[s] = 0;
            continue;
        }
        unsigned ne = 0, nm = 0;
        for (long long a = lo; a < hi; a++) {
            if (il[a] == 0) ne++;
            else nm++;
        }
        ecnt[s] = ne;
        emit[s] = nm;
        off32[s] = (unsigned)lo;
        rng[s] = make_uint2((unsigned)lo, (unsigned)hi);
        if (s == S - 1) {
            off32[S] = (unsigned)hi;
            ecnt[S] = 0;
        }
    }
}

// per state: its epsilon records, in arc order, and its epsilon range
__global__ void gb_state_eps(const long long *off, const int *il, const int *dst, const double *w, long long S,
                             const unsigned *eoff, int4 *eps, uint2 *erng) {
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < S; s += (long long)gridDim.x * blockDim.x) {
        unsigned k = eoff[s];
        erng[s] = make_uint2(eoff[s], eoff[s + 1]);
        const long long lo = off[s], hi = off[s + 1];
        for (long long a = lo; a < hi; a++) {
            if (il[a] != 0) continue;
            const long long bits = __double_as_longlong(w[a]);
            eps[k++] = make_int4(dst[a], (int)a, (int)(bits & 0xFFFFFFFFll), (int)(bits >> 32));
        }
    }
}

// states entered by an epsilon arc (ilabel 0)
__global__ void gb_eps_in(const int *dst, const int *il, long long A, long long S, unsigned char *eps_in) {
    for (long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x; a < A; a += (long long)gridDim.x * blockDim.x) {
        const int d = dst[a];
        if (il[a] == 0 && d >= 0 && d < S) eps_in[d] = 1;
    }
}

// per arc: validation, the 16 B record with the "dst owns epsilon arcs" and
// "dst has no incoming epsilon arc" flags
__global__ void gb_arcs(const int *dst, const int *il, const int *ol, const double *w, long long A, long long S,
                        const uint2 *erng, const unsigned char *eps_in, int4 *arcs, unsigned *err, int *max_il) {
    int mx = 0;
    for (long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x; a < A; a += (long long)gridDim.x * blockDim.x) {
        const int d = dst[a], l = il[a];
        if (d < 0 || d >= S || l < 0 || l >= (int)NOEPSIN_FLAG || ol[a] < 0) {
            atomicOr(err, GB_BAD_FIELD);
            continue;
        }
        const double x = w[a];
        if (!(x >= 0.0 && x <= 1.7976931348623157e308)) atomicOr(err, GB_BAD_WEIGHT);
        const uint2 er = erng[d];
        const unsigned y = (unsigned)l | (er.y > er.x ? EPS_FLAG : 0u) | (eps_in[d] ? 0u : NOEPSIN_FLAG);
        const long long bits = __double_as_longlong(x);
        arcs[a] = make_int4(d, (int)y, (int)(bits & 0xFFFFFFFFll), (int)(bits >> 32));
        mx = l > mx ? l : mx;
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_il, mx);
}

}  // namespace lbk
