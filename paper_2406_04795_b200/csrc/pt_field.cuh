// Device-side description and evaluation of implicit manifolds.
//   F(q) = sum_j w_j exp(-gamma |q - s_j|^2) + bias - barrier(q)    manifold.py:177-208, _kernels.pyx:18-40
//   barrier(q) = gain*scale*sum_d [softplus((lo_d-q_d)/scale) + softplus((q_d-hi_d)/scale)]   manifold.py:165-169
//   sphere / ellipsoid / plane test fields                           manifold.py:75-140
#pragma once
#include "pt_common.cuh"

struct PtFieldDev {
    int kind;              // PT_FIELD_*
    int n;
    long long S;           // support vectors
    int row;               // doubles per packed support row (odd, >= n+1): coords, weight, pad
    const double* sv;      // [S][row]
    const float* sv32;     // [S][row32] fp32 screening copy (row32 = n+2: coords*c, |s|^2 term, w)
    double gamma, bias;
    int has_barrier;
    double b_scale, b_gain;
    double b_lo[PT_NMAX], b_hi[PT_NMAX];
    double p0[PT_NMAX];    // sphere/ellipsoid centre, plane normal
    double p1[PT_NMAX];    // ellipsoid semi-axes
    double c0;             // sphere radius^2, plane offset
    double err32;          // rigorous bound on |F32 - F64| excluding the barrier (screening mode)
};

static inline int pt_sv_row(int n) { int r = n + 1; return (r & 1) ? r : r + 1; }

#ifdef __CUDACC__
// numpy.logaddexp(0, v) branch structure (npy_logaddexp): max + log1p(exp(-|diff|))
__device__ __forceinline__ double pt_softplus(double v) {
    double tmp = 0.0 - v;
    if (tmp > 0.0) return log1p(exp(-tmp));
    else if (tmp <= 0.0) return v + log1p(exp(tmp));
    return v;  // NaN
}

template <int N>
__device__ __forceinline__ double pt_barrier_value(const PtFieldDev& f, const double* p) {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) {
        double lo = pt_softplus(__ddiv_rn(__dsub_rn(f.b_lo[d], p[d]), f.b_scale));
        double hi = pt_softplus(__ddiv_rn(__dsub_rn(p[d], f.b_hi[d]), f.b_scale));
        acc = __dadd_rn(acc, __dadd_rn(lo, hi));
    }
    return __dmul_rn(__dmul_rn(f.b_gain, f.b_scale), acc);
}

// numpy einsum("ij,ij->i", d, d) for contiguous rows on this image's numpy build: two SIMD lanes
// accumulate even / odd columns, an odd tail goes to lane 0, then lane0 + lane1; no FMA.
template <int N>
__device__ __forceinline__ double pt_einsum_sq(const double* d) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j + 1 < N; j += 2) {
        a0 = __dadd_rn(a0, __dmul_rn(d[j], d[j]));
        a1 = __dadd_rn(a1, __dmul_rn(d[j + 1], d[j + 1]));
    }
    if (N & 1) a0 = __dadd_rn(a0, __dmul_rn(d[N - 1], d[N - 1]));
    return __dadd_rn(a0, a1);
}

template <int N>
__device__ __forceinline__ double pt_analytic_value(const PtFieldDev& f, const double* p) {
    double d[N];
    if (f.kind == PT_FIELD_SPHERE) {
#pragma unroll
        for (int j = 0; j < N; ++j) d[j] = __dsub_rn(p[j], f.p0[j]);
        return __dsub_rn(pt_einsum_sq<N>(d), f.c0);
    } else if (f.kind == PT_FIELD_ELLIPSOID) {
#pragma unroll
        for (int j = 0; j < N; ++j) d[j] = __ddiv_rn(__dsub_rn(p[j], f.p0[j]), f.p1[j]);
        return __dsub_rn(pt_einsum_sq<N>(d), 1.0);
    } else {  // plane: points @ normal - offset
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) acc = __dadd_rn(acc, __dmul_rn(p[j], f.p0[j]));
        return __dsub_rn(acc, f.c0);
    }
}
#endif
