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
    int row;               // doubles per packed support row (odd, >= n+2): coords, weight, -gamma*log2(e)*|s|^2, pad
    const double* sv;      // [S][row]
    const float* sv32;     // [S][row32] fp32 screening copy: coords, -gamma*log2(e)*|s|^2, weight, pad
    int row32;             // floats per fp32 row (multiple of 4)
    double smax;           // max_j |s_j| (enters the fp32 error bound)
    double gamma, bias;
    double amb_tol;        // 1e-12*(sum|w| + |bias|): below it a sign is "ambiguous" (the reference's own cross-backend
                           // tolerance on the kernel sum, pkg/tests/test_backends.py:81-93); such vertices are counted
    int has_barrier;
    double b_scale, b_gain;
    double b_lo[PT_NMAX], b_hi[PT_NMAX];
    double p0[PT_NMAX];    // sphere/ellipsoid centre, plane normal
    double p1[PT_NMAX];    // ellipsoid semi-axes
    double c0;             // sphere radius^2, plane offset
};

static inline int pt_sv_row(int n) { return (n + 2) | 1; }
static inline int pt_sv_row32(int n) { return (n + 2 + 3) & ~3; }

#define PT_L2E 1.4426950408889634
#define PT_LN2 0.6931471805599453
#define PT_U32 5.9604644775390625e-08   /* 2^-24, unit roundoff of binary32 */

// ---- tensor-core screen (kernels in pt_field_tc.cuh) ----------------------------------------------------
#define PT_TC_M 128                 /* points per CTA chunk = UMMA M = TMEM lanes */
#define PT_TC_N 128                 /* support vectors per UMMA = accumulator columns */
#define PT_TC_THREADS 256           /* two row groups of 4 warps; warp w and w+4 both sit on TMEM lanes 32(w%4).. */
#define PT_TC_SMEM_LIMIT 232448     /* 227 KB */
/* bound, in units of u32*T (T = gamma*log2e*(|p|+max|s|)^2), on |arg_tc - arg|: 1.5 from the tf32 splits plus the
 * tensor-core accumulation (each addend of a k-step is truncated at about 2^-23 of the largest one).  PTX does not
 * specify the latter, so it is CALIBRATED: worst case measured over 4e8 pairs is 7.4 (benchmarks/tc_calibrate.py), and
 * tests/test_gpu_parity.py::test_tc_screen_exponent_error asserts the measured maximum stays below half of this */
#define PT_TC_ARG_ULPS 16.0

static inline int pt_tc_kt(int n) { return ((3 * n + 6) + 7) & ~7; }
static inline long long pt_tc_spad(long long S) { return ((S + PT_TC_N - 1) / PT_TC_N) * PT_TC_N; }
static inline size_t pt_tc_smem_bytes(int n, long long S) {
    const size_t kc = (size_t)pt_tc_kt(n) / 4;
    return kc * (size_t)pt_tc_spad(S) * 16 + 2 * kc * PT_TC_M * 16 + (size_t)pt_tc_spad(S) * 4 + 64;
}
// largest support chunk (multiple of PT_TC_N rows) that fits one CTA's shared memory next to the A operands
static inline int pt_tc_chunk_rows(int n) {
    const size_t kc = (size_t)pt_tc_kt(n) / 4;
    const size_t fixed = 2 * kc * PT_TC_M * 16 + 64;
    const size_t per_row = kc * 16 + 4;
    return (int)(((PT_TC_SMEM_LIMIT - fixed) / per_row) / PT_TC_N) * PT_TC_N;
}

struct PtTcDev {
    const float* bt;   // [KT/4][Spad][4] tf32 pieces of the support side, UMMA K-major core-matrix order
    const float* wt;   // [Spad] fp32 weights (0 for the pad rows)
    int spad;
    int kt;
};

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

// Same value as pt_barrier_value, with the 2N softplus terms spread over the G lanes that share a
// point (lane g of the group computes terms g, g+G, ...); the sum is formed in the reference order on
// every lane.  All G lanes of the group must call it.
template <int N, int G>
__device__ __forceinline__ double pt_barrier_group(const PtFieldDev& f, const double* p, int g) {
    if (G == 1) return pt_barrier_value<N>(f, p);
    double mine[(2 * N + G - 1) / G];
#pragma unroll
    for (int k = 0; k < (2 * N + G - 1) / G; ++k) {
        const int i = g + k * G;
        double v = 0.0;
        if (i < 2 * N) {
            const int d = i >> 1;
            v = (i & 1) ? pt_softplus(__ddiv_rn(__dsub_rn(p[d], f.b_hi[d]), f.b_scale))
                        : pt_softplus(__ddiv_rn(__dsub_rn(f.b_lo[d], p[d]), f.b_scale));
        }
        mine[k] = v;
    }
    const int lane0 = (threadIdx.x & 31) & ~(G - 1);
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) {
        const int il = 2 * d, ih = 2 * d + 1;
        const double lo = __shfl_sync(0xffffffffu, mine[il / G], lane0 + (il % G));
        const double hi = __shfl_sync(0xffffffffu, mine[ih / G], lane0 + (ih % G));
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
