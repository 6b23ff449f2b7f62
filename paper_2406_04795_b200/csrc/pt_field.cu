// Field evaluation and per-edge root solve (bisection) kernels + their C ABI.
//
//   pt_eval_rbf_kernel<N,G>    values/signs of the kernel-SVM field at m points; G lanes share a
//                              point and split the support set, support rows staged in shared memory
//   pt_bisect_rbf_kernel<N,G>  intersection_points_batch: every segment halves its own bracket
//                              until seg*(hi-lo) <= eps  (manifold.py:368-383)
//   *_analytic_*               same for sphere/ellipsoid/plane fields, arithmetic ordered like numpy
#include <stdlib.h>
#include <cub/cub.cuh>
#include "pt_internal.cuh"
#include "pt_field.cuh"

struct pt_field {
    pt_ctx* ctx = nullptr;
    PtFieldDev d;
    PtBuf<double> sv;
    PtBuf<float> sv32;
    int precision = 0;
    double sum_abs_w = 0.0;
    // tensor-core screen (pt_field_tc.cuh): packed tf32 support operand; tc_ok = it fits one CTA's shared memory
    PtBuf<float> tc_bt, tc_wt;
    PtTcDev tc;
    bool tc_ok = false;          // the tf32 operand exists (n <= 6)
    bool tc_resident = false;    // ... and the whole support set fits one CTA's shared memory (persistent kernel)
    bool tc_levels = false;      // force the level-synchronous driver (PERMATRACE_B200_TC_LEVELS=1)
    bool tc4 = false;            // n = 6 and the 5-chunk operand + four A buffers fit: four row groups per CTA
    // one-pass Taylor-model root solve (pt_field_taylor.cuh): sign-sorted rows with log2|w| folded into the exponent
    PtBuf<double> svt;
    long long t_pos = 0, t_tot = 0;
    bool taylor = false;
    PtBuf<double> dirtab;        // direction sums of the sorted rows (rows grouped by direction take one FMA for u_j)
    bool taylor_dir = false;
};

int pt_field_dim(const pt_field* f) { return f->d.n; }

#define PT_EVAL_THREADS 256
#define PT_EVAL_TILE 256

#define PT_ROW64(N) (((N) + 2) | 1)

// optional row indirection of the evaluation kernel: a compacted list whose length lives on the device
struct PtRowList { const uint32_t* list; const unsigned long long* count; };
#define PT_EXP_TAB 256   /* entries of the 2^(i/256) table behind every tile */
#define PT_SMEM64(N) ((size_t)(PT_EVAL_TILE * PT_ROW64(N) + PT_EXP_TAB) * sizeof(double))

// 2^x for x <= ~0 in fp64: x = (256k + i)/256 + r, |r| <= 1/512; 2^r by a degree-4 Taylor polynomial
// (truncation 3.8e-17), 2^(i/256) from a 256-entry shared-memory table, 2^k by an exponent-field add.
// Arguments below -1000 are clamped (the term is < 1e-300 of its weight).  Branch-free on purpose so
// independent rows interleave; non-finite points are handled once per point (PtPoint64::poison).
__device__ __forceinline__ double pt_exp2_neg(double x, const double* __restrict__ tab) {
    if ((unsigned)__double2hiint(x) > 0xC08F4000u) x = -1000.0;   // x < -1000 (integer compare: keeps the FP64 pipe free)
    const double MAGIC = 6755399441055744.0;   // 1.5 * 2^52: the low word of x*256 + MAGIC is round(256 x)
    const double t = fma(x, 256.0, MAGIC);
    const int mi = __double2loint(t);
    const double r = fma(t - MAGIC, -0.00390625, x);
    double p = 0.009618129107628477;
    p = fma(p, r, 0.055504108664821576);
    p = fma(p, r, 0.2402265069591007);
    p = fma(p, r, 0.6931471805599453);
    p = fma(p, r, 1.0);
    const double v = tab[mi & (PT_EXP_TAB - 1)] * p;
    return __hiloint2double(__double2hiint(v) + ((mi >> 8) << 20), __double2loint(v));
}

// per-point constants of the expanded exponent: -gamma*log2(e)*|p - s|^2 = c_s + c_p + sum_d p_d s'_d with
// s'_d = 2*gamma*log2(e)*s_d stored in the packed support rows (so the point itself is the only per-point vector)
template <int N>
struct PtPoint64 {
    double q[N];
    double cp;
    double poison;   // 0 for a finite point, NaN otherwise (added to every sum so F is NaN like the reference's)
    __device__ __forceinline__ void set(const double* p, double gl) {
        double p2 = 0.0;
#pragma unroll
        for (int d = 0; d < N; ++d) { q[d] = p[d]; p2 = fma(p[d], p[d], p2); }
        cp = -gl * p2;
        poison = p2 - p2;
    }
};

template <int N>
__device__ __forceinline__ double pt_rbf_term(const double* __restrict__ row, const PtPoint64<N>& pp,
                                              const double* __restrict__ tab) {
    double arg = row[N + 1] + pp.cp;
#pragma unroll
    for (int d = 0; d < N; ++d) arg = fma(pp.q[d], row[d], arg);
    return row[N] * pt_exp2_neg(arg, tab);
}

__device__ __forceinline__ void pt_exp_table_init(double* tab) {
    for (int i = threadIdx.x; i < PT_EXP_TAB; i += blockDim.x) tab[i] = exp2((double)i * (1.0 / PT_EXP_TAB));
}

// accumulate this lane's share of sum_j w_j k(p, s_j); all threads of the block must call it
// (tile holds PT_EVAL_TILE rows followed by the 32-entry 2^(i/32) table, see pt_exp_table_init)
template <int N, int G>
__device__ __forceinline__ double pt_rbf_block_sum(const PtFieldDev& f, const double* p, int g, double* tile) {
    const int ROW = PT_ROW64(N);
    const double* tab = tile + PT_EVAL_TILE * ROW;
    PtPoint64<N> pp;
    pp.set(p, f.gamma * PT_L2E);
    double acc = 0.0;
    for (long long t0 = 0; t0 < f.S; t0 += PT_EVAL_TILE) {
        long long rem = f.S - t0;
        int cnt = rem < PT_EVAL_TILE ? (int)rem : PT_EVAL_TILE;
        __syncthreads();
        const double* src = f.sv + t0 * ROW;
        for (int i = threadIdx.x; i < cnt * ROW; i += PT_EVAL_THREADS) tile[i] = src[i];
        __syncthreads();
        // four independent accumulators: the serial exponent/polynomial chains of neighbouring rows overlap
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = g;
        for (; j + 3 * G < cnt; j += 4 * G) {
            s0 += pt_rbf_term<N>(tile + j * ROW, pp, tab);
            s1 += pt_rbf_term<N>(tile + (j + G) * ROW, pp, tab);
            s2 += pt_rbf_term<N>(tile + (j + 2 * G) * ROW, pp, tab);
            s3 += pt_rbf_term<N>(tile + (j + 3 * G) * ROW, pp, tab);
        }
        for (; j < cnt; j += G) s0 += pt_rbf_term<N>(tile + j * ROW, pp, tab);
        acc += (s0 + s1) + (s2 + s3);
    }
    acc += pp.poison;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    return acc;
}

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_eval_rbf_kernel(PtFieldDev f, PtRowList rows, const double* __restrict__ pts, size_t m_all, double* __restrict__ vals,
                   int8_t* __restrict__ signs, unsigned long long* work, unsigned long long* amb, float* __restrict__ vals32 = nullptr) {
    extern __shared__ double tile[];
    const int PB = PT_EVAL_THREADS / G;
    const size_t m = rows.list ? (size_t)*rows.count : m_all;      // optional compacted row list (device-side count)
    if ((size_t)blockIdx.x * PB >= m) return;
    pt_exp_table_init(tile + PT_EVAL_TILE * PT_ROW64(N));
    const size_t idx = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = idx < m;
    const size_t pi = valid ? (rows.list ? (size_t)rows.list[idx] : idx) : 0;
    double p[N];
#pragma unroll
    for (int d = 0; d < N; ++d) p[d] = valid ? pts[pi * N + d] : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&work[1], (unsigned long long)m);
    double acc = pt_rbf_block_sum<N, G>(f, p, g, tile);
    if (valid && g == 0) {
        double F = f.bias + acc;
        if (f.has_barrier) F -= pt_barrier_value<N>(f, p);
        if (vals) vals[pi] = F;
        if (vals32) vals32[pi] = (float)F;
        if (signs) {
            signs[pi] = F > 0.0 ? (int8_t)1 : (int8_t)-1;
            if (fabs(F) < f.amb_tol) atomicAdd(amb, 1ull);     // rare by construction: no contention
        }
    }
}

template <int N>
__global__ void pt_eval_analytic_kernel(PtFieldDev f, const double* __restrict__ pts, size_t m,
                                        double* __restrict__ vals, int8_t* __restrict__ signs) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double p[N];
#pragma unroll
    for (int d = 0; d < N; ++d) p[d] = pts[i * N + d];
    double F = pt_analytic_value<N>(f, p);
    if (vals) vals[i] = F;
    if (signs) signs[i] = F > 0.0 ? (int8_t)1 : (int8_t)-1;
}

// gradient of the kernel-SVM field (manifold.py:210-217): grad F = -2 gamma sum_j w_j k_j (p - s_j) - grad barrier.
// With the rows holding s' = 2 gl s:  sum_j w_j k_j (p - s_j) = p A - V / (2 gl),  A = sum w k,  V = sum w k s'.
template <int N>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_gradient_rbf_kernel(PtFieldDev f, const double* __restrict__ pts, size_t m, double* __restrict__ out) {
    extern __shared__ double tile[];
    const int ROW = PT_ROW64(N);
    pt_exp_table_init(tile + PT_EVAL_TILE * ROW);
    const double* tab = tile + PT_EVAL_TILE * ROW;
    const size_t pi = (size_t)blockIdx.x * PT_EVAL_THREADS + threadIdx.x;
    const bool valid = pi < m;
    double p[N];
#pragma unroll
    for (int d = 0; d < N; ++d) p[d] = valid ? pts[pi * N + d] : 0.0;
    PtPoint64<N> pp;
    pp.set(p, f.gamma * PT_L2E);
    double A = 0.0, V[N];
#pragma unroll
    for (int d = 0; d < N; ++d) V[d] = 0.0;
    for (long long t0 = 0; t0 < f.S; t0 += PT_EVAL_TILE) {
        long long rem = f.S - t0;
        const int cnt = rem < PT_EVAL_TILE ? (int)rem : PT_EVAL_TILE;
        __syncthreads();
        const double* src = f.sv + t0 * ROW;
        for (int i = threadIdx.x; i < cnt * ROW; i += PT_EVAL_THREADS) tile[i] = src[i];
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
            const double* row = tile + j * ROW;
            const double e = pt_rbf_term<N>(row, pp, tab);
            A += e;
#pragma unroll
            for (int d = 0; d < N; ++d) V[d] = fma(e, row[d], V[d]);
        }
    }
    if (!valid) return;
    const double inv2gl = 1.0 / (2.0 * f.gamma * PT_L2E);
#pragma unroll
    for (int d = 0; d < N; ++d) {
        double g = -2.0 * f.gamma * (p[d] * A - V[d] * inv2gl) + pp.poison;
        if (f.has_barrier) {
            const double sh = 1.0 / (1.0 + exp(-(p[d] - f.b_hi[d]) / f.b_scale));
            const double sl = 1.0 / (1.0 + exp(-(f.b_lo[d] - p[d]) / f.b_scale));
            g -= f.b_gain * (sh - sl);
        }
        out[pi * N + d] = g;
    }
}

// segment setup shared by both bisection kernels: diff, seg = ||b-a||_2 (numpy: sequential sum of
// squares, sqrt), all separately rounded
template <int N>
__device__ __forceinline__ double pt_segment(const double* a, const double* b, double* diff) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) { diff[d] = __dsub_rn(b[d], a[d]); s = __dadd_rn(s, __dmul_rn(diff[d], diff[d])); }
    return sqrt(s);
}

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_bisect_rbf_kernel(PtFieldDev f, const double* __restrict__ a_, const double* __restrict__ b_,
                     const int8_t* __restrict__ signs_a, size_t m, double eps, double* __restrict__ out,
                     unsigned long long* work) {
    extern __shared__ double tile[];
    pt_exp_table_init(tile + PT_EVAL_TILE * PT_ROW64(N));
    const int PB = PT_EVAL_THREADS / G;
    const size_t ei = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = ei < m;
    double a[N], diff[N], p[N];
    double seg = 0.0;
    int sa = 1;
    if (valid) {
        double b[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
        seg = pt_segment<N>(a, b, diff);
        sa = signs_a[ei];
    } else {
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; }
    }
    double lo = 0.0, hi = 1.0;
    bool active = valid && seg > eps;
    unsigned iters = 0;
    while (__syncthreads_or(active ? 1 : 0)) {
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
        for (int d = 0; d < N; ++d) p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d]));
        double acc = pt_rbf_block_sum<N, G>(f, p, g, tile);
        double F = f.bias + acc;
        if (f.has_barrier) F -= pt_barrier_group<N, G>(f, p, g);
        const int s = F > 0.0 ? 1 : -1;
        if (active) {
            if (s == sa) lo = mid; else hi = mid;
            active = __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
            ++iters;
        }
    }
    {
        // rows x iterations actually needed (idle lanes of finished rows are not counted)
        unsigned mine = (g == 0) ? iters : 0u;
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&work[0], (unsigned long long)mine);
    }
    if (valid && g == 0) {
        const double t = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
        for (int d = 0; d < N; ++d) out[ei * N + d] = __dadd_rn(a[d], __dmul_rn(t, diff[d]));
    }
}

template <int N>
__global__ void pt_bisect_analytic_kernel(PtFieldDev f, const double* __restrict__ a_, const double* __restrict__ b_,
                                          const int8_t* __restrict__ signs_a, size_t m, double eps,
                                          double* __restrict__ out) {
    size_t ei = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ei >= m) return;
    double a[N], b[N], diff[N], p[N];
#pragma unroll
    for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
    const double seg = pt_segment<N>(a, b, diff);
    const int sa = signs_a[ei];
    double lo = 0.0, hi = 1.0;
    bool active = seg > eps;
    while (active) {
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
        for (int d = 0; d < N; ++d) p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d]));
        const double F = pt_analytic_value<N>(f, p);
        const int s = F > 0.0 ? 1 : -1;
        if (s == sa) lo = mid; else hi = mid;
        active = __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
    }
    const double t = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
    for (int d = 0; d < N; ++d) out[ei * N + d] = __dadd_rn(a[d], __dmul_rn(t, diff[d]));
}


// ==== evaluation-based root solve =======================================================================
// Batches of 9.5 k rows and more are solved by ONE pass of the Taylor-model kernel (pt_field_taylor.cuh, included below);
// what follows serves smaller batches and the rows that kernel leaves open (none on the benchmark workloads).
// The reference bisects every crossing edge ~30 times in fp64.  This path returns the SAME dyadic
// bracket midpoint with ~6 fp64 evaluations per edge:
//   K1 pt_bisect32_kernel     replays the bisection with the field evaluated in fp32; a step is taken only
//                             when |F32| exceeds a rigorous bound on |F32 - F| (the decision then equals the
//                             fp64 one); otherwise the row stops with its current dyadic bracket.
//   K2 pt_bisect_resolve      rows that stopped while the bracket is still wide take ONE true fp64 bisection
//                             step and go back to K1 (compacted row lists, so nobody waits for them).
//   K3 pt_bisect_newton       for a bracket [lo,hi] of width w: evaluates F, F', F'' at the next midpoint
//                             (a true bisection step), then proves F monotone on the bracket from
//                             |F'(m)| > w|F''(m)| + w^2 M3/2 (M3 = global bound on the third derivative along
//                             the edge).  A monotone bracket holds exactly one root, so the reference's final
//                             depth-I cell is the one containing it: Newton + secant steps locate the root, and
//                             the cell is VERIFIED by evaluating F at its two ends with the midpoints' own
//                             arithmetic (a side has signs_a, the other does not).
//   K4 pt_bisect_rbf_kernel   rows whose proof or verification failed finish by plain fp64 bisection from
//                             their (always true) bisection bracket.
#define PT_TILE32 512
#ifndef PT_RETRY_ERR_RATIO
#define PT_RETRY_ERR_RATIO 8.0
#endif
#define PT_NEWTON_RETRIES 24          /* proof attempts (each one true step) a row may take before plain bisection */
#define PT_RESOLVE_ROUNDS 9           /* true fp64 steps a wide bracket may take before the Newton kernel: 2^-7 needs 7 */
#define PT_HANDOFF_WIDTH 0.0078125   /* 2^-7: brackets wider than this never enter K3 */
#define PT_FP32_STOP_WIDTH 0.001953125 /* 2^-9: fp32 screening stops here; deeper levels are mostly uncertain anyway */

template <int N> struct PtRow32 { static const int value = (N + 2 + 3) & ~3; };

__device__ __forceinline__ float pt_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// optional row indirection: kernels walk either all m rows or a compacted list whose length lives on the device
struct PtRows { const uint32_t* list; const unsigned long long* count; size_t m; };
__device__ __forceinline__ size_t pt_rows_total(const PtRows& r) { return r.list ? (size_t)*r.count : r.m; }

// lane share of sum_j w_j 2^(c_s + c_p + q.s_j) and of the same sum with |w_j|; fp32 chunks of <= 64
// terms are flushed into fp64 accumulators; all threads of the block must call it
template <int N, int G>
__device__ __forceinline__ void pt_rbf32_block_sum(const PtFieldDev& f, const float* q, float cp, int g, float* tile,
                                                   double& acc_out, double& abs_out) {
    const int ROW = PtRow32<N>::value;
    double acc = 0.0, ab = 0.0;
    for (long long t0 = 0; t0 < f.S; t0 += PT_TILE32) {
        long long rem = f.S - t0;
        const int cnt = rem < PT_TILE32 ? (int)rem : PT_TILE32;
        __syncthreads();
        const float4* src = reinterpret_cast<const float4*>(f.sv32 + t0 * ROW);
        float4* dst = reinterpret_cast<float4*>(tile);
        for (int i = threadIdx.x; i < cnt * (ROW / 4); i += PT_EVAL_THREADS) dst[i] = src[i];
        __syncthreads();
        for (int j0 = g; j0 < cnt; j0 += G * 64) {
            float fa = 0.f, fb = 0.f;
            const int jend = (j0 + G * 64 < cnt) ? j0 + G * 64 : cnt;
            for (int j = j0; j < jend; j += G) {
                const float* row = tile + j * ROW;
                float t = row[N] + cp;
#pragma unroll
                for (int d = 0; d < N; ++d) t = fmaf(q[d], row[d], t);
                const float e = pt_ex2(t);
                const float w = row[N + 1];
                fa = fmaf(w, e, fa);
                fb = fmaf(fabsf(w), e, fb);
            }
            acc += (double)fa; ab += (double)fb;
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        ab += __shfl_xor_sync(0xffffffffu, ab, off);
    }
    acc_out = acc; abs_out = ab;
}

// F, dF/dt, d2F/dt2 of the kernel sum along p(t) = a + t*diff at the point p
template <int N, int G>
__device__ __forceinline__ void pt_rbf_block_sum_d(const PtFieldDev& f, const double* p, const double* diff, double seg2,
                                                   int g, double* tile, double& F, double& D1, double& D2, double& AB) {
    const int ROW = PT_ROW64(N);
    const double* tab = tile + PT_EVAL_TILE * ROW;
    PtPoint64<N> pp;
    pp.set(p, f.gamma * PT_L2E);
    double pd = 0.0, dd[N];
    const double inv2gl = 1.0 / (2.0 * f.gamma * PT_L2E);   // rows hold 2*gamma*log2e*s_d
#pragma unroll
    for (int d = 0; d < N; ++d) { pd = fma(p[d], diff[d], pd); dd[d] = diff[d] * inv2gl; }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double ng2 = -2.0 * f.gamma, c2 = 2.0 * f.gamma * seg2;
    for (long long t0 = 0; t0 < f.S; t0 += PT_EVAL_TILE) {
        long long rem = f.S - t0;
        const int cnt = rem < PT_EVAL_TILE ? (int)rem : PT_EVAL_TILE;
        __syncthreads();
        const double* src = f.sv + t0 * ROW;
        for (int i = threadIdx.x; i < cnt * ROW; i += PT_EVAL_THREADS) tile[i] = src[i];
        __syncthreads();
        for (int j = g; j < cnt; j += G) {
            const double* row = tile + j * ROW;
            double x = pd;                           // (p - s) . diff
#pragma unroll
            for (int d = 0; d < N; ++d) x = fma(-dd[d], row[d], x);
            const double e = pt_rbf_term<N>(row, pp, tab);
            const double gx = ng2 * x;
            a0 += e; a1 = fma(e, gx, a1); a2 = fma(e, fma(gx, gx, -c2), a2); a3 += fabs(e);
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, off);
        a1 += __shfl_xor_sync(0xffffffffu, a1, off);
        a2 += __shfl_xor_sync(0xffffffffu, a2, off);
        a3 += __shfl_xor_sync(0xffffffffu, a3, off);
    }
    F = a0 + pp.poison; D1 = a1; D2 = a2; AB = a3;
}

// first and second t-derivatives of the box barrier along p(t) = a + t*diff
template <int N>
__device__ __forceinline__ void pt_barrier_derivs(const PtFieldDev& f, const double* p, const double* diff, double& B1, double& B2) {
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) {
        const double sl = 1.0 / (1.0 + exp(-(f.b_lo[d] - p[d]) / f.b_scale));
        const double sh = 1.0 / (1.0 + exp(-(p[d] - f.b_hi[d]) / f.b_scale));
        b1 = fma(diff[d], sh - sl, b1);
        b2 = fma(diff[d] * diff[d], sh * (1.0 - sh) + sl * (1.0 - sl), b2);
    }
    B1 = f.b_gain * b1; B2 = f.b_gain / f.b_scale * b2;
}

#include "pt_field_tc.cuh"

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_bisect32_kernel(PtFieldDev f, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                   const int8_t* __restrict__ signs_a, double eps, int fresh, double* __restrict__ lo_io,
                   double* __restrict__ hi_io, unsigned long long* work) {
    extern __shared__ float tile32[];
    const int PB = PT_EVAL_THREADS / G;
    const size_t total = pt_rows_total(rows);
    if ((size_t)blockIdx.x * PB >= total) return;
    const size_t idx = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = idx < total;
    const size_t ei = valid ? (rows.list ? (size_t)rows.list[idx] : idx) : 0;
    double a[N], diff[N], p[N];
    double seg = 0.0, lo = 0.0, hi = 1.0;
    int sa = 1;
    if (valid) {
        double b[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
        seg = pt_segment<N>(a, b, diff);
        sa = signs_a[ei];
        if (!fresh) { lo = lo_io[ei]; hi = hi_io[ei]; }
    } else {
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; }
    }
    const double gl = f.gamma * PT_L2E;
    bool active = valid && __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
    unsigned iters = 0;
    while (__syncthreads_or(active ? 1 : 0)) {
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
        double p2 = 0.0;
        float q[N];
#pragma unroll
        for (int d = 0; d < N; ++d) {
            p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d]));
            p2 = fma(p[d], p[d], p2);
            q[d] = (float)(2.0 * gl * p[d]);
        }
        const float cp = (float)(-gl * p2);
        // |arg32 - arg| <= (N+3) u T with T = gamma*log2(e) (|p| + max|s|)^2 (input roundings + fma chain);
        // ex2.approx, weight rounding, products and the <=64-term fp32 chunks add < 80 u relative
        const double pn = sqrt(p2) + f.smax;
        const double rel = 1.01 * ((double)(N + 4) * PT_U32 * gl * pn * pn * PT_LN2) + 80.0 * PT_U32;
        double acc, ab;
        pt_rbf32_block_sum<N, G>(f, q, cp, g, tile32, acc, ab);
        double F = f.bias + acc;
        if (f.has_barrier) F -= pt_barrier_group<N, G>(f, p, g);
        const double E = 2.0 * rel * ab + 1e-280;
        if (active) {
            if (fabs(F) > E) {
                if ((F > 0.0 ? 1 : -1) == sa) lo = mid; else hi = mid;
                ++iters;
                const double w = __dsub_rn(hi, lo);
                active = __dmul_rn(seg, w) > eps && w > PT_FP32_STOP_WIDTH;
            } else {
                active = false;   // sign not certain in fp32 (or NaN): stop with the current bracket
            }
        }
    }
    {
        unsigned mine = (g == 0) ? iters : 0u;
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&work[2], (unsigned long long)mine);
    }
    if (valid && g == 0) { lo_io[ei] = lo; hi_io[ei] = hi; }
}

// rows still active whose bracket is wider than the hand-off width -> compacted list
template <int N>
__global__ void pt_select_shallow_kernel(PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                                         const double* __restrict__ lo_, const double* __restrict__ hi_, double eps,
                                         uint32_t* __restrict__ list_out, unsigned long long* count_out) {
    const size_t total = pt_rows_total(rows);
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool take = false; size_t ei = 0;
    if (idx < total) {
        ei = rows.list ? (size_t)rows.list[idx] : idx;
        double a[N], b[N], diff[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
        const double seg = pt_segment<N>(a, b, diff);
        const double w = hi_[ei] - lo_[ei];
        take = (w > PT_HANDOFF_WIDTH) && (__dmul_rn(seg, w) > eps);
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, take);
    if (ballot) {
        const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(count_out, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (take) list_out[base + __popc(ballot & ((1u << lane) - 1u))] = (uint32_t)ei;
    }
}

__global__ void pt_select_flag_kernel(const uint8_t* __restrict__ flag, uint8_t want, size_t m, uint32_t* __restrict__ list_out,
                                      unsigned long long* count_out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool take = i < m && (want == 0xFF ? flag[i] != 0 : flag[i] == want);      // 0xFF: any set flag
    const unsigned ballot = __ballot_sync(0xffffffffu, take);
    if (ballot) {
        const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(count_out, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (take) list_out[base + __popc(ballot & ((1u << lane) - 1u))] = (uint32_t)i;
    }
}

// K2: one true fp64 bisection step for the listed rows
template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_bisect_resolve_kernel(PtFieldDev f, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                         const int8_t* __restrict__ signs_a, double* __restrict__ lo_io, double* __restrict__ hi_io,
                         unsigned long long* work) {
    extern __shared__ double tile[];
    pt_exp_table_init(tile + PT_EVAL_TILE * PT_ROW64(N));
    const int PB = PT_EVAL_THREADS / G;
    const size_t total = pt_rows_total(rows);
    if ((size_t)blockIdx.x * PB >= total) return;
    const size_t idx = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = idx < total;
    const size_t ei = valid ? (rows.list ? (size_t)rows.list[idx] : idx) : 0;
    double p[N];
    double lo = 0.0, hi = 1.0;
    int sa = 1;
#pragma unroll
    for (int d = 0; d < N; ++d) p[d] = 0.0;
    if (valid) {
        lo = lo_io[ei]; hi = hi_io[ei]; sa = signs_a[ei];
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
        for (int d = 0; d < N; ++d) {
            const double av = a_[ei * N + d];
            p[d] = __dadd_rn(av, __dmul_rn(mid, __dsub_rn(b_[ei * N + d], av)));
        }
    }
    double F = f.bias + pt_rbf_block_sum<N, G>(f, p, g, tile);
    if (f.has_barrier) F -= pt_barrier_group<N, G>(f, p, g);
    if (valid && g == 0) {
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
        if ((F > 0.0 ? 1 : -1) == sa) lo_io[ei] = mid; else hi_io[ei] = mid;
    }
    unsigned mine = (valid && g == 0) ? 1u : 0u;
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&work[5], (unsigned long long)mine);
}

// K3: monotonicity proof + Halley/Newton root location with a rigorous enclosure (see the block comment above).
// Exactly two block-wide evaluation passes, no data-dependent loops:
//   pass 1  F, F', F'' and A = sum|w_j|k_j at the bracket midpoint (a true bisection step);
//           s_min = |F'| - w|F''| - w^2 M3/2 - noise > 0 proves F monotone on the halved bracket (one root r)
//   pass 2  F at the Halley iterate x_h; x2 = x_h - F/(F'(m) + F''(m)(x_h - m)) and
//           |x2 - r| <= [eta + (|F|+eta) Delta/s_min] / |D|  (mean-value form of the Newton error),
//           eta = bound on the fp64 evaluation noise of BOTH this kernel and the reference loop.
//   The reference's final cell is the depth-I dyadic cell containing r; it is accepted only when the enclosure
//   of r stays eta/s_min away from both cell ends (there every sign the reference bisection can see is certain).
//   Everything else (<1 % of the rows) is flagged for the plain fp64 bisection kernel.
#define PT_U64 1.1102230246251565e-16   /* 2^-53 */
#ifndef PT_NEWTON_MINB
#define PT_NEWTON_MINB 4
#endif

#include "pt_field_taylor.cuh"

// two points per thread, each lane walks all support rows (G = 1): the row loads and the loop overhead are shared
// by four independent chains (2 rows x 2 points), so the FP64 pipe rather than the issue slot is the limiter
template <int N, int THREADS, bool DERIV>
__device__ __forceinline__ void pt_rbf_block_sum_x2(const PtFieldDev& f, const double (&p)[2][N], const double (&diff)[2][N],
                                                    const double (&seg2)[2], double* tile, double (&F)[2], double (&D1)[2],
                                                    double (&D2)[2], double (&AB)[2]) {
    const int ROW = PT_ROW64(N);
    const double* tab = tile + PT_EVAL_TILE * ROW;
    PtPoint64<N> pp[2];
    double pd[2], c2[2], dd[2][N];
    const double ng2 = -2.0 * f.gamma;
    const double inv2gl = 1.0 / (2.0 * f.gamma * PT_L2E);   // rows hold 2*gamma*log2e*s_d
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        pp[k].set(p[k], f.gamma * PT_L2E);
        double t = 0.0;
#pragma unroll
        for (int d = 0; d < N; ++d) { t = fma(p[k][d], diff[k][d], t); if (DERIV) dd[k][d] = diff[k][d] * inv2gl; }
        pd[k] = t; c2[k] = 2.0 * f.gamma * seg2[k];
    }
    double a0[2] = {0.0, 0.0}, b0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0}, a2[2] = {0.0, 0.0}, ab[2] = {0.0, 0.0};
    for (long long t0 = 0; t0 < f.S; t0 += PT_EVAL_TILE) {
        long long rem = f.S - t0;
        const int cnt = rem < PT_EVAL_TILE ? (int)rem : PT_EVAL_TILE;
        __syncthreads();
        const double* src = f.sv + t0 * ROW;
        for (int i = threadIdx.x; i < cnt * ROW; i += THREADS) tile[i] = src[i];
        if ((cnt & 1) && threadIdx.x < ROW) tile[cnt * ROW + threadIdx.x] = 0.0;   // zero-weight pad row
        __syncthreads();
        for (int j = 0; j < cnt; j += 2) {
            const double* r0 = tile + j * ROW;
            const double* r1 = r0 + ROW;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double e0 = pt_rbf_term<N>(r0, pp[k], tab);
                const double e1 = pt_rbf_term<N>(r1, pp[k], tab);
                a0[k] += e0; b0[k] += e1;
                if (DERIV) {
                    double x0 = pd[k], x1 = pd[k];
#pragma unroll
                    for (int d = 0; d < N; ++d) { x0 = fma(-dd[k][d], r0[d], x0); x1 = fma(-dd[k][d], r1[d], x1); }
                    const double g0 = ng2 * x0, g1 = ng2 * x1;
                    a1[k] = fma(e0, g0, a1[k]); a1[k] = fma(e1, g1, a1[k]);
                    a2[k] = fma(e0, fma(g0, g0, -c2[k]), a2[k]); a2[k] = fma(e1, fma(g1, g1, -c2[k]), a2[k]);
                    ab[k] += fabs(e0) + fabs(e1);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) { F[k] = (a0[k] + b0[k]) + pp[k].poison; D1[k] = a1[k]; D2[k] = a2[k]; AB[k] = ab[k]; }
}

template <int N, int G>
__global__ void __launch_bounds__(G == 1 ? 128 : PT_EVAL_THREADS, G == 1 ? PT_NEWTON_MINB : 1)
pt_bisect_newton_kernel(PtFieldDev f, double sum_abs_w, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                        const int8_t* __restrict__ signs_a, double* __restrict__ lo_io, double* __restrict__ hi_io,
                        double eps, double* __restrict__ out, uint8_t* __restrict__ slow,
                        double* __restrict__ jlo_out, double* __restrict__ jhi_out, double retry_ratio, unsigned long long* work) {
    constexpr int PPT = (G == 1) ? 2 : 1;
    constexpr int THREADS = (G == 1) ? 128 : PT_EVAL_THREADS;
    constexpr int GROUPS = THREADS / G;
    extern __shared__ double tile[];
    const size_t m = pt_rows_total(rows);                      // all rows, or a compacted list with a device-side count
    if ((size_t)blockIdx.x * (GROUPS * PPT) >= m) return;
    pt_exp_table_init(tile + PT_EVAL_TILE * PT_ROW64(N));
    const int g = threadIdx.x % G;
    size_t ei[PPT];
    bool valid[PPT];
    double p[PPT][N], diff[PPT][N], seg[PPT], seg2[PPT], lo[PPT], hi[PPT], mid[PPT];
    int sa[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        ei[k] = (size_t)blockIdx.x * (GROUPS * PPT) + (size_t)k * GROUPS + threadIdx.x / G;
        valid[k] = ei[k] < m;
        if (valid[k] && rows.list) ei[k] = rows.list[ei[k]];
        seg[k] = 0.0; lo[k] = 0.0; hi[k] = 1.0; sa[k] = 1;
        if (valid[k]) {
            double a[N], b[N];
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[ei[k] * N + d]; b[d] = b_[ei[k] * N + d]; }
            seg[k] = pt_segment<N>(a, b, diff[k]);
            sa[k] = signs_a[ei[k]];
            lo[k] = lo_io[ei[k]]; hi[k] = hi_io[ei[k]];
            mid[k] = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
#pragma unroll
            for (int d = 0; d < N; ++d) p[k][d] = __dadd_rn(a[d], __dmul_rn(mid[k], diff[k][d]));
        } else {
            mid[k] = 0.5;
#pragma unroll
            for (int d = 0; d < N; ++d) { p[k][d] = 0.0; diff[k][d] = 0.0; }
        }
        seg2[k] = seg[k] * seg[k];
    }
    // ---- pass 1: F, F', F'', sum|w|k at the midpoint ---------------------------------------------------------
    double F0[PPT], D1[PPT], D2[PPT], AB[PPT];
    if constexpr (G == 1) {
        pt_rbf_block_sum_x2<N, THREADS, true>(f, p, diff, seg2, tile, F0, D1, D2, AB);
    } else {
        pt_rbf_block_sum_d<N, G>(f, p[0], diff[0], seg2[0], g, tile, F0[0], D1[0], D2[0], AB[0]);
    }
    // per-row state that must survive pass 2 lives in shared memory (keeps the evaluation loop's registers free)
    double* st = tile + PT_EVAL_TILE * PT_ROW64(N) + PT_EXP_TAB;
#define PT_ST(field, k) st[((field) * PPT + (k)) * THREADS + threadIdx.x]
    enum { ST_LO, ST_W, ST_DL, ST_SMIN, ST_ETA, ST_AD2, ST_K, ST_DT, ST_XH, ST_TF, ST_FIELDS };
    bool need[PPT], to_slow[PPT], one_step[PPT];
    unsigned evals = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        one_step[k] = false;
        double B0 = 0.0;
        F0[k] += f.bias;
        if (f.has_barrier) {
            B0 = pt_barrier_group<N, G>(f, p[k], g);
            F0[k] -= B0;
            double B1, B2;
            pt_barrier_derivs<N>(f, p[k], diff[k], B1, B2);
            D1[k] -= B1; D2[k] -= B2;
        }
        // depth of the reference's final bracket: smallest I with seg * 2^-I <= eps
        double dl = 1.0;
        if (valid[k]) while (__dmul_rn(seg[k], dl) > eps) dl *= 0.5;
        double w = hi[k] - lo[k];
        const bool finished0 = valid[k] && !(__dmul_rn(seg[k], w) > eps);
        const bool shallow = valid[k] && !finished0 && w > PT_HANDOFF_WIDTH;
        need[k] = valid[k] && !finished0 && !shallow;
        to_slow[k] = shallow;
        double tf = mid[k], x = mid[k], smin = 1.0, eta = 0.0, ad2 = 0.0, K = 0.0, Dt = 1.0;
        if (shallow) {
            // too wide for a proof attempt: the midpoint evaluation is still a true bisection step
            ++evals;
            if ((F0[k] > 0.0 ? 1 : -1) == sa[k]) lo[k] = mid[k]; else hi[k] = mid[k];
            w = hi[k] - lo[k];
            if (!(__dmul_rn(seg[k], w) > eps)) { to_slow[k] = false; tf = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k])); }
        }
        if (need[k]) {
            ++evals;
            if ((F0[k] > 0.0 ? 1 : -1) == sa[k]) lo[k] = mid[k]; else hi[k] = mid[k];
            w = hi[k] - lo[k];
            if (!(__dmul_rn(seg[k], w) > eps)) { need[k] = false; tf = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k])); }
            // third-derivative bound along the edge: kernel sum (max |H3| exp < 4 gamma^1.5) + barrier, 1.5x safety
            double t3 = 4.0 * f.gamma * sqrt(f.gamma) * sum_abs_w * seg2[k] * seg[k];
            if (f.has_barrier) {
                double s3 = 0.0;
#pragma unroll
                for (int d = 0; d < N; ++d) { const double r = fabs(diff[k][d]) / f.b_scale; s3 += r * r * r; }
                t3 += 0.2 * f.b_gain * f.b_scale * s3;
            }
            const double m3 = 1.5 * t3;
            // evaluation noise anywhere in the bracket: this kernel's expanded exponent (cancellation at scale
            // T = gamma log2e (|p|+max|s|)^2) plus the reference's sequential sum, relative to A = sum|w|k
            double p2 = 0.0;
#pragma unroll
            for (int d = 0; d < N; ++d) p2 = fma(p[k][d], p[k][d], p2);
            const double pn = sqrt(p2) + f.smax + w * seg[k];
            const double T = f.gamma * PT_L2E * pn * pn;
            const double ceta = PT_U64 * (1.01 * (double)(4 * N + 3) * T * PT_LN2 + 1.25 * (double)f.S + 400.0);
            // A >= sum|w|k anywhere in the bracket: between the midpoint and a point at |x - m| <= w (in t) a kernel term
            // grows by at most exp(gamma | |x-s|^2 - |m-s|^2 |) <= exp(2 gamma pn seg w + gamma seg^2 w^2)
            const double A = 1.0001 * exp(w * (2.0 * f.gamma * pn * seg[k] + f.gamma * seg2[k] * w)) * AB[k];
            eta = ceta * A + 64.0 * PT_U64 * (1.1 * fabs(B0) + fabs(f.bias)) + 1e-290;
            const double gmax = 2.0 * f.gamma * pn * seg[k];
            const double etaD = (ceta + 16.0 * PT_U64) * gmax * A;
            const double etaD2 = (ceta + 32.0 * PT_U64) * (gmax * gmax + 2.0 * f.gamma * seg2[k]) * A;
            ad2 = fabs(D2[k]) + etaD2;
            K = 0.5 * m3 * w * w + etaD + etaD2 * w;
            smin = fabs(D1[k]) - etaD - w * ad2 - 0.5 * w * w * m3;
            if (need[k] && !(smin > 0.0)) { to_slow[k] = true; need[k] = false; }
            if (need[k]) {
                const double nt = F0[k] / D1[k];
                x = mid[k] - nt * (1.0 + 0.5 * nt * (D2[k] / D1[k]));   // Halley step from the midpoint
                if (!(x > lo[k] && x < hi[k])) x = 0.5 * (lo[k] + hi[k]);
                Dt = D1[k] + D2[k] * (x - mid[k]);                       // extrapolated slope at the iterate
            }
        }
        PT_ST(ST_LO, k) = lo[k]; PT_ST(ST_W, k) = w; PT_ST(ST_DL, k) = dl; PT_ST(ST_SMIN, k) = smin; PT_ST(ST_ETA, k) = eta;
        PT_ST(ST_AD2, k) = ad2; PT_ST(ST_K, k) = K; PT_ST(ST_DT, k) = Dt; PT_ST(ST_XH, k) = x; PT_ST(ST_TF, k) = tf;
        // the point of pass 2
#pragma unroll
        for (int d = 0; d < N; ++d) {
            const double av = valid[k] ? a_[ei[k] * N + d] : 0.0;
            p[k][d] = __dadd_rn(av, __dmul_rn(x, diff[k][d]));
        }
    }
    // ---- pass 2: F at the Halley iterate ------------------------------------------------------------------
    bool any = false;
#pragma unroll
    for (int k = 0; k < PPT; ++k) any = any || need[k];
    if (__syncthreads_or(any ? 1 : 0)) {
        double F1[PPT];
        if constexpr (G == 1) {
            double u1[2], u2[2], u3[2];
            pt_rbf_block_sum_x2<N, THREADS, false>(f, p, diff, seg2, tile, F1, u1, u2, u3);
        } else {
            F1[0] = pt_rbf_block_sum<N, G>(f, p[0], g, tile);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            F1[k] += f.bias;
            if (f.has_barrier) F1[k] -= pt_barrier_group<N, G>(f, p[k], g);
            if (need[k]) {
                ++evals;
                const double lo_ = PT_ST(ST_LO, k), w = PT_ST(ST_W, k), dl = PT_ST(ST_DL, k), smin = PT_ST(ST_SMIN, k);
                const double eta = PT_ST(ST_ETA, k), Dt = PT_ST(ST_DT, k), x = PT_ST(ST_XH, k);
                const double aF = fabs(F1[k]);
                const double rho = (aF + eta) / smin;                            // |x_h - r| <= rho
                const double x2 = x - F1[k] / Dt;
                const double Delta = PT_ST(ST_AD2, k) * rho + PT_ST(ST_K, k);    // >= |F'(xi) - Dt|
                const double err = 1.01 * (eta + (aF + eta) * Delta / smin) / fabs(Dt) + 4e-16;
                const double zeta = eta / smin;
                // Every midpoint the reference bisection visits OUTSIDE the enclosure J = [x2 - err - zeta, x2 + err + zeta]
                // has a certain sign (F is monotone, the root is in J, and the point is at least zeta = eta/s_min
                // from it), so the bisection is replayed in exact dyadic arithmetic until a midpoint falls inside J.
                const bool sane = fabs(Dt) >= smin && x2 > lo_ && x2 < lo_ + w;
                const double Jlo = x2 - err - zeta, Jhi = x2 + err + zeta;
                double L = lo_, H = lo_ + w;
                bool open = false;
                if (sane) {
                    while (__dmul_rn(seg[k], __dsub_rn(H, L)) > eps) {
                        const double mq = __dmul_rn(0.5, __dadd_rn(L, H));
                        if (mq < Jlo) L = mq;
                        else if (mq > Jhi) H = mq;
                        else { open = true; break; }
                    }
                } else open = true;
                if (!open) PT_ST(ST_TF, k) = __dmul_rn(0.5, __dadd_rn(L, H));
                else {
                    // a midpoint inside J needs a true fp64 evaluation: the rest kernels continue from [L, H],
                    // still skipping every midpoint outside J
                    // ... unless the enclosure is limited by the model error of this attempt (a wide starting bracket) rather
                    // than by the evaluation noise: then the row retries from the replayed bracket, which costs two
                    // evaluations and normally closes it
                    to_slow[k] = true;
                    PT_ST(ST_LO, k) = L; PT_ST(ST_W, k) = H - L;
                    one_step[k] = sane && !(err > retry_ratio * zeta);
                    if (sane) { PT_ST(ST_AD2, k) = Jlo; PT_ST(ST_K, k) = Jhi; }
                }
            }
        }
    }
    {
        unsigned mine = (g == 0) ? evals : 0u;
        unsigned sl = 0;
#pragma unroll
        for (int k = 0; k < PPT; ++k) sl += (g == 0 && to_slow[k]) ? 1u : 0u;
        for (int off = 16; off > 0; off >>= 1) { mine += __shfl_xor_sync(0xffffffffu, mine, off); sl += __shfl_xor_sync(0xffffffffu, sl, off); }
        if ((threadIdx.x & 31) == 0) {
            if (mine) atomicAdd(&work[0], (unsigned long long)mine);
            if (sl) atomicAdd(&work[3], (unsigned long long)sl);
        }
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        if (valid[k] && g == 0) {
            slow[ei[k]] = to_slow[k] ? (one_step[k] ? 2 : 1) : 0;      // open rows: 2 = root enclosed, 1 = no proof
            if (to_slow[k]) {
                const double l = PT_ST(ST_LO, k);
                lo_io[ei[k]] = l; hi_io[ei[k]] = l + PT_ST(ST_W, k);
                jlo_out[ei[k]] = one_step[k] ? PT_ST(ST_AD2, k) : -1e300;
                jhi_out[ei[k]] = one_step[k] ? PT_ST(ST_K, k) : 1e300;
            }
            else {
                const double tf = PT_ST(ST_TF, k);
#pragma unroll
                for (int d = 0; d < N; ++d) {
                    const double av = a_[ei[k] * N + d];
                    out[ei[k] * N + d] = __dadd_rn(av, __dmul_rn(tf, __dsub_rn(b_[ei[k] * N + d], av)));
                }
            }
        }
    }
#undef PT_ST
}

// K4 with the whole support set resident in shared memory and one WARP per row: rows need very different numbers
// of true evaluations (0..30), so nothing here is block-synchronous -- a warp takes a row, replays the certain
// midpoints, evaluates the open ones with its 32 lanes splitting the support set, writes the point, takes the next.
#define PT_RESTW_THREADS 512
// Same idea for support sets larger than shared memory: the support set passes through shared memory in chunks, so an
// evaluation round is block-synchronous (all 16 warps evaluate their current row's open midpoint against chunk after
// chunk), but every warp still owns its row: it replays, decides, finishes and pulls the next row on its own.
template <int N>
__global__ void __launch_bounds__(PT_RESTW_THREADS, 1)
pt_bisect_rest_warp_kernel(PtFieldDev f, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                           const int8_t* __restrict__ signs_a, const double* __restrict__ lo_in, const double* __restrict__ hi_in,
                           const double* __restrict__ jlo_in, const double* __restrict__ jhi_in,
                           double eps, double* __restrict__ out, int chunk_rows, unsigned long long* next_row,
                           unsigned long long* work) {
    extern __shared__ double tile[];
    const int ROW = PT_ROW64(N);
    const size_t total = pt_rows_total(rows);
    const int warps_per_block = PT_RESTW_THREADS / 32;
    if ((size_t)blockIdx.x * warps_per_block >= total) return;
    const int S = (int)f.S;
    const int nchunks = (S + chunk_rows - 1) / chunk_rows;
    double* tab = tile + (size_t)chunk_rows * ROW;
    for (int i = threadIdx.x; i < PT_EXP_TAB; i += PT_RESTW_THREADS) tab[i] = exp2((double)i * (1.0 / PT_EXP_TAB));
    if (nchunks == 1) for (long long i = threadIdx.x; i < (long long)S * ROW; i += PT_RESTW_THREADS) tile[i] = f.sv[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned iters = 0;
    // per-warp row state (replicated over the lanes)
    size_t ei = 0;
    double a[N], diff[N], p[N];
    double seg = 0.0, lo = 0.0, hi = 1.0, jlo = -1e300, jhi = 1e300, mid = 0.5;
    int sa = 1;
    bool have = false, exhausted = false;
#pragma unroll
    for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; p[d] = 0.0; }
    for (;;) {
        // bring this warp to a row with an open midpoint: replay certain steps, retire finished rows, pull new ones
        while (!exhausted) {
            if (!have) {
                unsigned long long take = 0;
                if (lane == 0) take = atomicAdd(next_row, 1ull);
                const size_t idx = (size_t)__shfl_sync(0xffffffffu, take, 0);
                if (idx >= total) { exhausted = true; break; }
                ei = rows.list ? (size_t)rows.list[idx] : idx;
                double b[N];
#pragma unroll
                for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
                seg = pt_segment<N>(a, b, diff);
                sa = signs_a[ei]; lo = lo_in[ei]; hi = hi_in[ei];
                jlo = jlo_in ? jlo_in[ei] : -1e300; jhi = jhi_in ? jhi_in[ei] : 1e300;
                have = true;
            }
            // midpoints outside [jlo, jhi] have a proven sign (see pt_bisect_newton_kernel): replay those steps exactly
            bool open = false;
            while (__dmul_rn(seg, __dsub_rn(hi, lo)) > eps) {
                mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
                if (mid < jlo) lo = mid; else if (mid > jhi) hi = mid; else { open = true; break; }
            }
            if (open) break;
            if (lane == 0) {
                const double t = __dmul_rn(0.5, __dadd_rn(lo, hi));
#pragma unroll
                for (int d = 0; d < N; ++d) out[ei * N + d] = __dadd_rn(a[d], __dmul_rn(t, diff[d]));
            }
            have = false;
        }
        const bool work_here = have && !exhausted;
        if (nchunks > 1) { if (!__syncthreads_or(work_here ? 1 : 0)) break; }
        else if (!work_here) break;
#pragma unroll
        for (int d = 0; d < N; ++d) p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d]));
        PtPoint64<N> pp;
        pp.set(p, f.gamma * PT_L2E);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const int j0 = c * chunk_rows;
            const int cnt = (S - j0) < chunk_rows ? (S - j0) : chunk_rows;
            if (nchunks > 1) {
                __syncthreads();
                const double* src = f.sv + (size_t)j0 * ROW;
                for (int i = threadIdx.x; i < cnt * ROW; i += PT_RESTW_THREADS) tile[i] = src[i];
                __syncthreads();
            }
            if (work_here) {
                int j = lane;
                for (; j + 96 < cnt; j += 128) {
                    s0 += pt_rbf_term<N>(tile + (size_t)j * ROW, pp, tab);
                    s1 += pt_rbf_term<N>(tile + (size_t)(j + 32) * ROW, pp, tab);
                    s2 += pt_rbf_term<N>(tile + (size_t)(j + 64) * ROW, pp, tab);
                    s3 += pt_rbf_term<N>(tile + (size_t)(j + 96) * ROW, pp, tab);
                }
                for (; j < cnt; j += 32) s0 += pt_rbf_term<N>(tile + (size_t)j * ROW, pp, tab);
            }
        }
        if (work_here) {
            double acc = ((s0 + s1) + (s2 + s3)) + pp.poison;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            double F = f.bias + acc;
            if (f.has_barrier) F -= pt_barrier_group<N, 32>(f, p, lane);
            if ((F > 0.0 ? 1 : -1) == sa) lo = mid; else hi = mid;
            ++iters;
        }
    }
    if (lane == 0 && iters) atomicAdd(&work[4], (unsigned long long)iters);
}

// K4 for support sets that do not fit in shared memory: step-synchronous.  One launch = ONE true evaluation for every
// listed row (two rows per thread, support tiles through shared memory like the Newton kernel): replay the certain
// midpoints, evaluate the open one, decide, replay again; rows that still have an open midpoint go to the next list
// (device-side counts, no host synchronisation), finished rows write their point.
template <int N>
__global__ void __launch_bounds__(128, 4)
pt_bisect_step_kernel(PtFieldDev f, const uint32_t* __restrict__ list_in, const unsigned long long* __restrict__ count_in,
                      const double* __restrict__ a_, const double* __restrict__ b_, const int8_t* __restrict__ signs_a,
                      double* __restrict__ lo_io, double* __restrict__ hi_io, const double* __restrict__ jlo_in,
                      const double* __restrict__ jhi_in, double eps, double* __restrict__ out,
                      uint32_t* __restrict__ list_out, unsigned long long* count_out, unsigned long long* work) {
    extern __shared__ double tile[];
    const size_t total = (size_t)*count_in;
    if ((size_t)blockIdx.x * 256 >= total) return;
    pt_exp_table_init(tile + PT_EVAL_TILE * PT_ROW64(N));
    uint32_t ei[2]; bool valid[2], active[2] = {false, false};
    double p[2][N], diff[2][N], seg[2], seg2[2], lo[2], hi[2], jlo[2], jhi[2], mid[2];
    int sa[2];
    auto replay = [&](int k) {
        // midpoints outside [jlo, jhi] have a proven sign (see pt_bisect_newton_kernel): take those steps exactly
        while (active[k]) {
            const double mq = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
            if (mq < jlo[k]) lo[k] = mq; else if (mq > jhi[k]) hi[k] = mq; else break;
            active[k] = __dmul_rn(seg[k], __dsub_rn(hi[k], lo[k])) > eps;
        }
    };
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const size_t idx = (size_t)blockIdx.x * 256 + (size_t)k * 128 + threadIdx.x;
        valid[k] = idx < total;
        ei[k] = valid[k] ? list_in[idx] : 0u;
        seg[k] = 0.0; lo[k] = 0.0; hi[k] = 1.0; jlo[k] = -1e300; jhi[k] = 1e300; sa[k] = 1;
#pragma unroll
        for (int d = 0; d < N; ++d) { p[k][d] = 0.0; diff[k][d] = 0.0; }
        if (valid[k]) {
            double a[N], b[N];
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[(size_t)ei[k] * N + d]; b[d] = b_[(size_t)ei[k] * N + d]; }
            seg[k] = pt_segment<N>(a, b, diff[k]);
            sa[k] = signs_a[ei[k]]; lo[k] = lo_io[ei[k]]; hi[k] = hi_io[ei[k]];
            jlo[k] = jlo_in[ei[k]]; jhi[k] = jhi_in[ei[k]];
        }
        seg2[k] = seg[k] * seg[k];
        active[k] = valid[k] && __dmul_rn(seg[k], __dsub_rn(hi[k], lo[k])) > eps;
        replay(k);
        mid[k] = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
        if (valid[k]) {
#pragma unroll
            for (int d = 0; d < N; ++d) p[k][d] = __dadd_rn(a_[(size_t)ei[k] * N + d], __dmul_rn(mid[k], diff[k][d]));
        }
    }
    unsigned iters = 0;
    if (__syncthreads_or((active[0] || active[1]) ? 1 : 0)) {
        double F[2], u1[2], u2[2], u3[2];
        pt_rbf_block_sum_x2<N, 128, false>(f, p, diff, seg2, tile, F, u1, u2, u3);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            double Fk = f.bias + F[k];
            if (f.has_barrier) Fk -= pt_barrier_value<N>(f, p[k]);
            if (active[k]) {
                if ((Fk > 0.0 ? 1 : -1) == sa[k]) lo[k] = mid[k]; else hi[k] = mid[k];
                active[k] = __dmul_rn(seg[k], __dsub_rn(hi[k], lo[k])) > eps;
                ++iters;
                replay(k);
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) iters += __shfl_xor_sync(0xffffffffu, iters, off);
    if ((threadIdx.x & 31) == 0 && iters) atomicAdd(&work[4], (unsigned long long)iters);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (valid[k]) {
            if (active[k]) { lo_io[ei[k]] = lo[k]; hi_io[ei[k]] = hi[k]; }
            else {
                const double t = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
#pragma unroll
                for (int d = 0; d < N; ++d) {
                    const double av = a_[(size_t)ei[k] * N + d];
                    out[(size_t)ei[k] * N + d] = __dadd_rn(av, __dmul_rn(t, diff[k][d]));
                }
            }
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, active[k]);
        if (ballot) {
            const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(count_out, (unsigned long long)__popc(ballot));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (active[k]) list_out[base + __popc(ballot & ((1u << lane) - 1u))] = ei[k];
        }
    }
}

// pack raw (support[S][n], weights[S]) into the fp64 row layout [2*gl*s_0.., w, -gl*|s|^2, pad] and the fp32
// screening copy [s_0.., -gl*|s|^2, w, pad]; record max |s_j| and sum |w_j|
__global__ void pt_pack_sv_kernel(const double* __restrict__ support, const double* __restrict__ weights,
                                  long long S, int n, int row, int row32, double gl, double* __restrict__ sv,
                                  float* __restrict__ sv32, unsigned long long* rmax_bits, double* sum_abs_w) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    double s2 = 0.0;
    for (int d = 0; d < n; ++d) {
        const double v = support[j * n + d];
        sv[j * row + d] = (2.0 * gl) * v;
        sv32[j * row32 + d] = (float)v;
        s2 = fma(v, v, s2);
    }
    const double w = weights[j];
    sv[j * row + n] = w;
    sv[j * row + n + 1] = -gl * s2;
    for (int d = n + 2; d < row; ++d) sv[j * row + d] = 0.0;
    sv32[j * row32 + n] = (float)(-gl * s2);
    sv32[j * row32 + n + 1] = (float)w;
    for (int d = n + 2; d < row32; ++d) sv32[j * row32 + d] = 0.f;
    atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(sqrt(s2)));
    atomicAdd(sum_abs_w, fabs(w));
}

// lanes per item so that small batches still fill the machine
static int pt_pick_group(pt_ctx* ctx, size_t m, long long S) {
    size_t target = (size_t)ctx->sm_count * 2048;
    if (S < 64) return 1;
    if (m >= target) return 1;
    if (m * 4 >= target || S < 256) return 4;
    return 32;
}

template <int N, int MODE>
static int pt_screen_tc_launch(pt_ctx* ctx, const pt_field* f, const PtRows& rows, const double* a, const double* b,
                               const int8_t* sa, double eps, int fresh, double* lo, double* hi, int8_t* sign_out);

template <int N>
static int pt_eval_launch(pt_ctx* ctx, const pt_field* f, const double* pts, size_t m, double* vals, int8_t* signs, float* vals32) {
    if (f->d.kind != PT_FIELD_RBF) {
        PT_LAUNCH(ctx, "eval_analytic");
        pt_eval_analytic_kernel<N><<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(f->d, pts, m, vals, signs);
        return pt_check_launch(ctx, "pt_eval_analytic_kernel");
    }
    const size_t smem = PT_SMEM64(N);
    const PtRowList none{nullptr, nullptr};
    // Signs of a large batch (lattice vertices of a BFS wave / of the refinement): the kernel sum runs on the tensor
    // cores in fp32 (pt_field_tc.cuh, MODE 2) with the screen's rigorous error bound; rows whose fp32 sign is not
    // proven are rechecked by the fp64 kernel through a compacted list.
    if (!vals && signs && f->tc_resident && f->precision != 0 && m >= (size_t)PT_TC_M * 32) {
        if constexpr (N <= 6) {
            PtBuf<uint32_t> list; PtBuf<unsigned long long> cnt;
            PT_TRY(list.alloc(ctx, m));
            PT_TRY(cnt.alloc(ctx, 1));
            PT_CUDA(ctx, cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
            const PtRows all{nullptr, nullptr, m};
            {
                PT_LAUNCH(ctx, "eval_signs_tc");
                PT_TRY((pt_screen_tc_launch<N, 2>(ctx, f, all, pts, nullptr, nullptr, 1.0, 1, nullptr, reinterpret_cast<double*>(vals32), signs)));
            }
            {
                PT_LAUNCH(ctx, "eval_select");
                pt_select_flag_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>((const uint8_t*)signs, (uint8_t)0, m, list.p, cnt.p);
                PT_TRY(pt_check_launch(ctx, "pt_select_flag_kernel"));
            }
            PT_LAUNCH(ctx, "eval_rbf");
            const PtRowList sub{list.p, cnt.p};
            pt_eval_rbf_kernel<N, 4><<<pt_grid_for(m, PT_EVAL_THREADS / 4), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, sub, pts, m, nullptr, signs, ctx->work, ctx->amb_sink, vals32);
            return pt_check_launch(ctx, "pt_eval_rbf_kernel");
        }
    }
    const int G = pt_pick_group(ctx, m, f->d.S);
    PT_LAUNCH(ctx, "eval_rbf");
    if (G == 1)
        pt_eval_rbf_kernel<N, 1><<<pt_grid_for(m, PT_EVAL_THREADS), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, none, pts, m, vals, signs, ctx->work, ctx->amb_sink, vals32);
    else if (G == 4)
        pt_eval_rbf_kernel<N, 4><<<pt_grid_for(m, PT_EVAL_THREADS / 4), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, none, pts, m, vals, signs, ctx->work, ctx->amb_sink, vals32);
    else
        pt_eval_rbf_kernel<N, 32><<<pt_grid_for(m, PT_EVAL_THREADS / 32), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, none, pts, m, vals, signs, ctx->work, ctx->amb_sink, vals32);
    return pt_check_launch(ctx, "pt_eval_rbf_kernel");
}

template <int N, int MODE>
static int pt_screen_tc_launch(pt_ctx* ctx, const pt_field* f, const PtRows& rows, const double* a, const double* b,
                               const int8_t* sa, double eps, int fresh, double* lo, double* hi, int8_t* sign_out) {
    if constexpr (N > 6) {
        return pt_fail(ctx, PT_E_STATE, "tensor-core screen is built for n <= 6");
    } else {
        const size_t smem = pt_tc_smem_bytes(N, f->d.S);
        // per launch: the attribute is per device, and a process may hold contexts on several devices (~1 us)
        PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect32_tc_kernel<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_TC_SMEM_LIMIT));
        if constexpr (N == 6 && MODE == 0) {
            if (f->tc4) {
                const size_t smem4 = (size_t)5 * f->tc.spad * 16 + 4 * (size_t)6 * PT_TC_M * 16 + (size_t)f->tc.spad * 4 + 64;
                // per launch: the attribute is per device, and a process may hold contexts on several devices (~1 us)
                PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect32_tc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_TC_SMEM_LIMIT));
                const unsigned grid4 = pt_grid_for(rows.m, 4 * PT_TC_M, (unsigned)ctx->sm_count);
                pt_bisect32_tc4_kernel<<<grid4, PT_TC4_THREADS, smem4, ctx->stream>>>(f->d, f->tc, rows, a, b, sa, eps, fresh, lo, hi, ctx->work);
                return pt_check_launch(ctx, "pt_bisect32_tc4_kernel");
            }
        }
        const unsigned grid = pt_grid_for(rows.m, 2 * PT_TC_M, (unsigned)ctx->sm_count);
        const PtTcLevel whole{0, f->tc.spad, nullptr, nullptr, 1};
        pt_bisect32_tc_kernel<N, MODE><<<grid, PT_TC_THREADS, smem, ctx->stream>>>(f->d, f->tc, rows, a, b, sa, eps, fresh, lo, hi, sign_out, whole, ctx->work);
        return pt_check_launch(ctx, "pt_bisect32_tc_kernel");
    }
}

// Level-synchronous screen (pt_field_tc.cuh, MODE 3): per bisection level one launch per support chunk over the rows
// that are still active (compacted, device-side counts -- no host synchronisation), then the decision kernel.  Serves
// support sets that do not fit one CTA's shared memory; every launch re-stages its chunk (<= 192 KB per CTA from L2).
#define PT_SCREEN_MAX_LEVELS 10
template <int N>
static int pt_screen_levels_launch(pt_ctx* ctx, const pt_field* f, const PtRows& rows, const double* a, const double* b,
                                   const int8_t* sa, double eps, int fresh, double* lo, double* hi) {
    if constexpr (N > 6) {
        return pt_fail(ctx, PT_E_STATE, "tensor-core screen is built for n <= 6");
    } else {
        const size_t m = rows.m;
        const int spad = f->tc.spad;
        const int cmax = pt_tc_chunk_rows(N);
        const int nchunks = (spad + cmax - 1) / cmax;
        int cs = (((spad + nchunks - 1) / nchunks) + PT_TC_N - 1) / PT_TC_N * PT_TC_N;
        // per launch: the attribute is per device, and a process may hold contexts on several devices (~1 us)
        PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect32_tc_kernel<N, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_TC_SMEM_LIMIT));
        PtBuf<double> acc, ab; PtBuf<uint32_t> la, lb; PtBuf<unsigned long long> cnt;
        PT_TRY(acc.alloc(ctx, m)); PT_TRY(ab.alloc(ctx, m));
        PT_TRY(la.alloc(ctx, m)); PT_TRY(lb.alloc(ctx, m));
        PT_TRY(cnt.alloc(ctx, PT_SCREEN_MAX_LEVELS + 2));
        PT_CUDA(ctx, cudaMemsetAsync(cnt.p, 0, (PT_SCREEN_MAX_LEVELS + 2) * sizeof(unsigned long long), ctx->stream));
        pt_screen_filter_kernel<N><<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(rows, a, b, eps, fresh, lo, hi, la.p, cnt.p);
        PT_TRY(pt_check_launch(ctx, "pt_screen_filter_kernel"));
        uint32_t* lin = la.p; uint32_t* lout = lb.p;
        const unsigned grid = pt_grid_for(m, 2 * PT_TC_M, (unsigned)ctx->sm_count);
        for (int level = 0; level < PT_SCREEN_MAX_LEVELS; ++level) {
            const PtRows sub{lin, cnt.p + level, m};
            for (int c = 0; c < nchunks; ++c) {
                const int j0 = c * cs;
                const int rows_c = (j0 + cs <= spad) ? cs : (spad - j0);
                if (rows_c <= 0) break;
                const size_t kc = (size_t)pt_tc_kt(N) / 4;
                const size_t smem = kc * (size_t)rows_c * 16 + 2 * kc * PT_TC_M * 16 + (size_t)rows_c * 4 + 64;
                const PtTcLevel lv{j0, rows_c, acc.p, ab.p, c == 0 ? 1 : 0};
                pt_bisect32_tc_kernel<N, 3><<<grid, PT_TC_THREADS, smem, ctx->stream>>>(f->d, f->tc, sub, a, b, sa, eps, 0, lo, hi,
                                                                                         nullptr, lv, ctx->work);
                PT_TRY(pt_check_launch(ctx, "pt_bisect32_tc_kernel"));
            }
            pt_screen_decide_kernel<N><<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(f->d, lin, cnt.p + level, a, b, sa, eps, lo, hi,
                                                                                      acc.p, ab.p, lout, cnt.p + level + 1, ctx->work);
            PT_TRY(pt_check_launch(ctx, "pt_screen_decide_kernel"));
            uint32_t* sw = lin; lin = lout; lout = sw;
        }
        return PT_OK;
    }
}

template <int N>
static int pt_bisect_launch(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, const int8_t* sa,
                            size_t m, double eps, double* out, const float* hint) {
    if (f->d.kind != PT_FIELD_RBF) {
        PT_LAUNCH(ctx, "bisect_analytic");
        pt_bisect_analytic_kernel<N><<<pt_grid_for(m, 128), 128, 0, ctx->stream>>>(f->d, a, b, sa, m, eps, out);
        return pt_check_launch(ctx, "pt_bisect_analytic_kernel");
    }
    const int G = pt_pick_group(ctx, m, f->d.S);
    const size_t smem = PT_SMEM64(N);
    const unsigned grid = pt_grid_for(m, PT_EVAL_THREADS / G);
    if (f->precision == 0 || f->d.S == 0) {
        PT_LAUNCH(ctx, "bisect_rbf");
        if (G == 1) pt_bisect_rbf_kernel<N, 1><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        else if (G == 4) pt_bisect_rbf_kernel<N, 4><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        else pt_bisect_rbf_kernel<N, 32><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        return pt_check_launch(ctx, "pt_bisect_rbf_kernel");
    }
    PtBuf<double> lo, hi, jlo, jhi; PtBuf<uint32_t> list; PtBuf<unsigned long long> cnt; PtBuf<uint8_t> slow;
    PT_TRY(lo.alloc(ctx, m));
    PT_TRY(hi.alloc(ctx, m));
    PT_TRY(jlo.alloc(ctx, m));
    PT_TRY(jhi.alloc(ctx, m));
    PT_TRY(list.alloc(ctx, m));
    PT_TRY(slow.alloc(ctx, m));
    PT_TRY(cnt.alloc(ctx, PT_RESOLVE_ROUNDS + 2));
    PT_CUDA(ctx, cudaMemsetAsync(cnt.p, 0, (PT_RESOLVE_ROUNDS + 2) * sizeof(unsigned long long), ctx->stream));
    const size_t smem32 = (size_t)PT_TILE32 * PtRow32<N>::value * sizeof(float);
    const PtRows all{nullptr, nullptr, m};
#define PT_G_LAUNCH(KERNEL, SMEM, ...)                                                            \
    do {                                                                                            \
        if (G == 1) KERNEL<N, 1><<<grid, PT_EVAL_THREADS, SMEM, ctx->stream>>>(__VA_ARGS__);        \
        else if (G == 4) KERNEL<N, 4><<<grid, PT_EVAL_THREADS, SMEM, ctx->stream>>>(__VA_ARGS__);   \
        else KERNEL<N, 32><<<grid, PT_EVAL_THREADS, SMEM, ctx->stream>>>(__VA_ARGS__);              \
        PT_TRY(pt_check_launch(ctx, #KERNEL));                                                      \
    } while (0)
    // batches that fill the machine take the one-pass Taylor-model kernel: it either finishes a row or leaves a valid
    // dyadic bracket (flag 1: no enclosure, flag 2: root enclosed) for the evaluation-based kernels below
    static const long long taylor_min = getenv("PERMATRACE_B200_TAYLOR_MIN") ? atoll(getenv("PERMATRACE_B200_TAYLOR_MIN")) : 0;
    const bool use_taylor = f->taylor && m >= (taylor_min > 0 ? (size_t)taylor_min : (size_t)ctx->sm_count * 64);
    // batches that fill the machine screen on the tensor cores (tcgen05), small ones on the SIMT kernel
    const bool use_tc = f->tc_ok && m >= (size_t)PT_TC_M * 32;
    const bool by_level = use_tc && (!f->tc_resident || f->tc_levels);
    if (use_taylor) {
        // With a secant hint of the root's position (fp32 vertex values kept by the refinement) the model is centred there
        // and 12 moments do what 20 do about the edge midpoint; without one, 20 about the midpoint.
        // OFF by default: the hint comes from fp32 vertex values whose last bits depend on the size of the batch they were
        // evaluated in (tensor-core or SIMT path), so a hinted centre -- and with it the decision at an AMBIGUOUS midpoint --
        // is not invariant under how cells are sliced over batches / ranks.  Measured with it on: dof6-stress 262 -> 239 ms,
        // dof6 29.0 -> 30.3 ms (longer fine edges: more rows need the second pass).  PERMATRACE_B200_TAYLOR_HINT=1 enables it.
        static const bool hints_on = getenv("PERMATRACE_B200_TAYLOR_HINT") && getenv("PERMATRACE_B200_TAYLOR_HINT")[0] == '1';
        const bool hinted = hint != nullptr && hints_on;
        const PtTaylorDev td{f->svt.p, f->t_pos, f->t_tot, f->taylor_dir ? f->dirtab.p : nullptr};
        const PtTaylorGroup nogrp{nullptr, nullptr};
        auto launch = [&](const PtRows& rws, size_t count, int recentre, const float* h) -> int {
            const unsigned grid = pt_grid_for(count, PT_TAYLOR_THREADS);
            if (hinted) {
                PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q_HINT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PT_TAYLOR_SMEM(N, PT_TAYLOR_Q_HINT)));
                PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q_HINT, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                pt_bisect_taylor_kernel<N, PT_TAYLOR_Q_HINT, false><<<grid, PT_TAYLOR_THREADS, PT_TAYLOR_SMEM(N, PT_TAYLOR_Q_HINT), ctx->stream>>>(
                    f->d, f->sum_abs_w, td, rws, nogrp, a, b, sa, eps, out, lo.p, hi.p, slow.p, jlo.p, jhi.p, ctx->work, recentre, h);
            } else {
                // tiny batches (at most one block per SM: recentred passes of a few thousand rows, late waves of a trace): the
                // per-edge loop over the support set is the launch's latency, so G lanes share an edge.  Measured on B200: a
                // 111-row pass 0.16 -> 0.09 ms with G = 4; from ~50 k rows on the launch is throughput-sized and sharing LOSES
                // (4x the blocks, each staging the whole support set: 47.6 k rows 0.73 -> 1.24 ms, 95 k rows 1.4 -> 2.5 ms)
                int G = 1;
                for (int g = 2; g <= 4; g *= 2)
                    if ((double)count * g / PT_TAYLOR_THREADS <= (double)ctx->sm_count) G = g;
                const char* g_env = getenv("PERMATRACE_B200_TAYLOR_SHARE");          // tests / A-B timing: force 1, 2 or 4
                if (g_env) G = atoi(g_env) == 4 ? 4 : atoi(g_env) == 2 ? 2 : 1;
#define PT_TAYLOR_GEN_LAUNCH(GG)                                                                                                          \
                do {                                                                                                                  \
                    const unsigned gridg = pt_grid_for(count, PT_TAYLOR_THREADS / GG);                                                \
                    PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, false, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PT_TAYLOR_SMEM(N, PT_TAYLOR_Q)));   \
                    PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, false, GG>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));                            \
                    pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, false, GG><<<gridg, PT_TAYLOR_THREADS, PT_TAYLOR_SMEM(N, PT_TAYLOR_Q), ctx->stream>>>(                                          \
                        f->d, f->sum_abs_w, td, rws, nogrp, a, b, sa, eps, out, lo.p, hi.p, slow.p, jlo.p, jhi.p, ctx->work, recentre, nullptr);                                          \
                } while (0)
                if (G == 4) PT_TAYLOR_GEN_LAUNCH(4);
                else if (G == 2) PT_TAYLOR_GEN_LAUNCH(2);
                else PT_TAYLOR_GEN_LAUNCH(1);
#undef PT_TAYLOR_GEN_LAUNCH
            }
            return pt_check_launch(ctx, "pt_bisect_taylor_kernel");
        };
        // Rows grouped by direction (lattice edges move along h * 1_mask): blocks whose rows share the mask get the first
        // log-derivative from the direction table with one FMA per pair.  Rows that are not lattice edges (class 0) and
        // hinted batches keep the generic kernel.
        bool grouped = false;
        // (batches of up to two waves of blocks skip the grouping: they are latency-sized and take the shared-row generic kernel)
        if (f->taylor_dir && !hinted && m < 0xFFFFFFFFull - (size_t)(PT_TAYLOR_THREADS << N) &&
            m > (getenv("PERMATRACE_B200_TAYLOR_GROUP_MIN") ? (size_t)atoll(getenv("PERMATRACE_B200_TAYLOR_GROUP_MIN"))
                                                            : (size_t)2 * ctx->sm_count * PT_TAYLOR_MINB_DIR * PT_TAYLOR_THREADS)) {
            constexpr int NC = 1 << N;
            PtBuf<uint8_t> cls, bmask; PtBuf<unsigned> hist; PtBuf<uint32_t> glist;
            PT_TRY(cls.alloc(ctx, m));
            PT_TRY(hist.alloc(ctx, 2 * NC + 2));
            PT_CUDA(ctx, cudaMemsetAsync(hist.p, 0, (2 * NC + 2) * sizeof(unsigned), ctx->stream));
            {
                PT_LAUNCH(ctx, "bisect_taylor_group");
                pt_taylor_classify_kernel<N><<<pt_grid_for(m, PT_TAYLOR_CLS_THREADS), PT_TAYLOR_CLS_THREADS, 0, ctx->stream>>>(a, b, m, cls.p, hist.p);
                PT_TRY(pt_check_launch(ctx, "pt_taylor_classify_kernel"));
            }
            unsigned* hh = (unsigned*)ctx->pinned;
            PT_CUDA(ctx, cudaMemcpyAsync(hh, hist.p, NC * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            PtTaylorOffsets offs;
            memset(&offs, 0, sizeof(offs));
            // class 0 first (unpadded: it is walked as a plain row list), then the masks, each padded to whole blocks
            size_t slot = ((size_t)hh[0] + PT_TAYLOR_THREADS - 1) / PT_TAYLOR_THREADS * PT_TAYLOR_THREADS;
            const size_t n0 = hh[0];
            for (int c = 1; c < NC; ++c) {
                offs.off[c] = (unsigned)slot;
                slot += ((size_t)hh[c] + PT_TAYLOR_THREADS - 1) / PT_TAYLOR_THREADS * PT_TAYLOR_THREADS;
            }
            const size_t first_slot = offs.off[1], total_slots = slot;
            const size_t nblocks = (total_slots - first_slot) / PT_TAYLOR_THREADS;
            PT_TRY(glist.alloc(ctx, total_slots > 0 ? total_slots : 1));
            PT_TRY(bmask.alloc(ctx, nblocks > 0 ? nblocks : 1));
            PT_CUDA(ctx, cudaMemsetAsync(glist.p, 0xFF, (total_slots > 0 ? total_slots : 1) * sizeof(uint32_t), ctx->stream));
            {
                PT_LAUNCH(ctx, "bisect_taylor_group");
                pt_taylor_scatter_kernel<N><<<pt_grid_for(m, PT_TAYLOR_CLS_THREADS), PT_TAYLOR_CLS_THREADS, 0, ctx->stream>>>(cls.p, m, offs, hist.p + NC, glist.p);
                PT_TRY(pt_check_launch(ctx, "pt_taylor_scatter_kernel"));
                if (nblocks > 0) {
                    pt_taylor_bmask_kernel<<<pt_grid_for(nblocks, 256), 256, 0, ctx->stream>>>(offs, NC, (unsigned)first_slot, nblocks, bmask.p);
                    PT_TRY(pt_check_launch(ctx, "pt_taylor_bmask_kernel"));
                }
            }
            {
                PT_LAUNCH(ctx, "bisect_fp64_taylor");
                if (nblocks > 0) {
                    const PtTaylorGroup grp{glist.p + first_slot, bmask.p};
                    PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PT_TAYLOR_SMEM_DIR(N, PT_TAYLOR_Q)));
                    PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                    pt_bisect_taylor_kernel<N, PT_TAYLOR_Q, true><<<(unsigned)nblocks, PT_TAYLOR_THREADS, PT_TAYLOR_SMEM_DIR(N, PT_TAYLOR_Q), ctx->stream>>>(
                        f->d, f->sum_abs_w, td, all, grp, a, b, sa, eps, out, lo.p, hi.p, slow.p, jlo.p, jhi.p, ctx->work, 0, nullptr);
                    PT_TRY(pt_check_launch(ctx, "pt_bisect_taylor_kernel"));
                }
                if (n0 > 0) {
                    PtBuf<unsigned long long> c0;
                    PT_TRY(c0.alloc(ctx, 1));
                    const unsigned long long n0v = n0;
                    PT_CUDA(ctx, cudaMemcpyAsync(c0.p, &n0v, sizeof(n0v), cudaMemcpyHostToDevice, ctx->stream));
                    const PtRows rest_l{glist.p, c0.p, m};
                    PT_TRY(launch(rest_l, n0, 0, nullptr));
                    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));      // c0 leaves scope
                }
            }
            grouped = true;
        }
        if (!grouped) {
            PT_LAUNCH(ctx, "bisect_fp64_taylor");
            PT_TRY(launch(all, m, 0, hint));
        }
        // rows it left open (root far from the model centre on a long edge: truncation, not rounding, limits the model
        // there): one more pass, the model recentred on the bracket each row stopped at
        PtBuf<unsigned long long> tcnt;
        PT_TRY(tcnt.alloc(ctx, 1));
        PT_CUDA(ctx, cudaMemsetAsync(tcnt.p, 0, sizeof(unsigned long long), ctx->stream));
        pt_select_flag_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(slow.p, (uint8_t)0xFF, m, list.p, tcnt.p);
        PT_TRY(pt_check_launch(ctx, "pt_select_flag_kernel"));
        unsigned long long left = 0;
        PT_CUDA(ctx, cudaMemcpyAsync(&left, tcnt.p, sizeof(left), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (left > 0) {
            PT_LAUNCH(ctx, "bisect_fp64_taylor2");
            const PtRows again{list.p, tcnt.p, m};
            PT_TRY(launch(again, (size_t)left, 1, nullptr));
        }
    }
    if (!use_taylor) {
        PT_LAUNCH(ctx, use_tc ? "bisect_fp32_screen_tc" : "bisect_fp32_screen");
        if (by_level) PT_TRY((pt_screen_levels_launch<N>(ctx, f, all, a, b, sa, eps, 1, lo.p, hi.p)));
        else if (use_tc) PT_TRY((pt_screen_tc_launch<N, 0>(ctx, f, all, a, b, sa, eps, 1, lo.p, hi.p, nullptr)));
        else PT_G_LAUNCH(pt_bisect32_kernel, smem32, f->d, all, a, b, sa, eps, 1, lo.p, hi.p, ctx->work);
    }
    // Rows that stopped while their bracket is still wider than the Newton hand-off width take true fp64 bisection steps
    // (one evaluation per listed row and round) until they are narrow enough; after the first two steps they go back
    // through the fp32 screen -- unless the screen is not getting anywhere on this field (ill-conditioned weights make
    // its error bound larger than |F| almost everywhere: seen with S = 16 384), which one look at the first list's size
    // tells.  Lists shrink round by round (device-side counts).
    PtBuf<uint32_t> list_b; PtBuf<unsigned long long> ncnt;
    PT_TRY(list_b.alloc(ctx, m));
    PT_TRY(ncnt.alloc(ctx, PT_NEWTON_RETRIES));
    PT_CUDA(ctx, cudaMemsetAsync(ncnt.p, 0, PT_NEWTON_RETRIES * sizeof(unsigned long long), ctx->stream));
    bool screen_pays = true;
    uint32_t* lcur = list.p; uint32_t* lnext = list_b.p;
    for (int round = 0; !use_taylor && round < (screen_pays ? 2 : PT_RESOLVE_ROUNDS); ++round) {
        unsigned long long* c = cnt.p + round;
        const PtRows prev = round == 0 ? all : PtRows{lcur, cnt.p + round - 1, m};
        uint32_t* lout = round == 0 ? lcur : lnext;
        const PtRows sub{lout, c, m};
        {
            PT_LAUNCH(ctx, "bisect_select");
            pt_select_shallow_kernel<N><<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(prev, a, b, lo.p, hi.p, eps, lout, c);
            PT_TRY(pt_check_launch(ctx, "pt_select_shallow_kernel"));
        }
        if (round == 0) {
            unsigned long long shallow = 0;
            PT_CUDA(ctx, cudaMemcpyAsync(&shallow, c, sizeof(shallow), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            if (shallow == 0) break;
            screen_pays = 10 * shallow < 9 * (unsigned long long)m;     // the first pass left > 90 % of the rows wide: it will not get better
        } else {
            uint32_t* sw = lcur; lcur = lnext; lnext = sw;
        }
        {
            PT_LAUNCH(ctx, "bisect_fp64_resolve");
            PT_G_LAUNCH(pt_bisect_resolve_kernel, smem, f->d, sub, a, b, sa, lo.p, hi.p, ctx->work);
        }
        if (round < 2 && screen_pays) {
            PT_LAUNCH(ctx, use_tc ? "bisect_fp32_screen_tc" : "bisect_fp32_screen");
            if (by_level) PT_TRY((pt_screen_levels_launch<N>(ctx, f, sub, a, b, sa, eps, 0, lo.p, hi.p)));
            else if (use_tc) PT_TRY((pt_screen_tc_launch<N, 0>(ctx, f, sub, a, b, sa, eps, 0, lo.p, hi.p, nullptr)));
            else PT_G_LAUNCH(pt_bisect32_kernel, smem32, f->d, sub, a, b, sa, eps, 0, lo.p, hi.p, ctx->work);
        }
    }
    {
        static const double retry_ratio = getenv("PERMATRACE_B200_RETRY_RATIO") ? atof(getenv("PERMATRACE_B200_RETRY_RATIO")) : PT_RETRY_ERR_RATIO;
        const size_t smem_nt = smem + 10 * 256 * sizeof(double);   // + per-row state (10 fields x rows per block)
        // mid-size batches (a trace's coarse edges): 4 lanes per row give several blocks per SM, 32 lanes waste the tiles
        const int Gn = G == 32 && m >= 16384 ? 4 : G;
        const unsigned grid = pt_grid_for(m, PT_EVAL_THREADS / Gn);
#define PT_NEWTON_LAUNCH(ROWS)                                                                                                     \
        do {                                                                                                                       \
            if (Gn == 1) pt_bisect_newton_kernel<N, 1><<<pt_grid_for(m, 256), 128, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, ROWS, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work); \
            else if (Gn == 4) pt_bisect_newton_kernel<N, 4><<<grid, PT_EVAL_THREADS, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, ROWS, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work); \
            else pt_bisect_newton_kernel<N, 32><<<grid, PT_EVAL_THREADS, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, ROWS, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work);       \
        } while (0)
        if (!use_taylor) {
            PT_LAUNCH(ctx, "bisect_fp64_newton");
            PT_NEWTON_LAUNCH(all);
            PT_TRY(pt_check_launch(ctx, "pt_bisect_newton_kernel"));
        }
        // Rows without a proof yet (bracket still too wide for the monotonicity bound: flat or strongly curved stretches,
        // ill-conditioned weights) come back: every attempt is a true bisection step plus a new proof attempt on the
        // halved bracket, over the shrinking list of such rows.
        for (int retry = 0; retry < PT_NEWTON_RETRIES; ++retry) {
            unsigned long long* c = ncnt.p + retry;
            pt_select_flag_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(slow.p, (uint8_t)1, m, list.p, c);
            PT_TRY(pt_check_launch(ctx, "pt_select_flag_kernel"));
            unsigned long long left = 0;
            PT_CUDA(ctx, cudaMemcpyAsync(&left, c, sizeof(left), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            if (left == 0) break;
            // lanes per row by the size of the list: small lists would leave a thread-per-row launch latency-bound
            PT_LAUNCH(ctx, "bisect_fp64_retry");
            const PtRows again{list.p, c, m};
            const int Gr = pt_pick_group(ctx, (size_t)left, f->d.S);
            const int Gl = Gr == 32 && left >= 16384 ? 4 : Gr;
            const unsigned gl_ = pt_grid_for((size_t)left, PT_EVAL_THREADS / Gl);
            if (Gl == 1) pt_bisect_newton_kernel<N, 1><<<pt_grid_for((size_t)left, 256), 128, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, again, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work + 8);
            else if (Gl == 4) pt_bisect_newton_kernel<N, 4><<<gl_, PT_EVAL_THREADS, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, again, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work + 8);
            else pt_bisect_newton_kernel<N, 32><<<gl_, PT_EVAL_THREADS, smem_nt, ctx->stream>>>(f->d, f->sum_abs_w, again, a, b, sa, lo.p, hi.p, eps, out, slow.p, jlo.p, jhi.p, retry_ratio, ctx->work + 8);
            PT_TRY(pt_check_launch(ctx, "pt_bisect_newton_kernel"));
        }
#undef PT_NEWTON_LAUNCH
    }
    PtBuf<unsigned long long> steps;
    unsigned long long* steps_dbg = nullptr;
    // open rows: (2) root enclosed, a few midpoints inside the enclosure need a true evaluation; (1) no proof -- plain
    // bisection.  The bulk of the enclosed rows needs 1..4 evaluations: a few step-synchronous launches over the
    // compacted list of rows that still have an open midpoint (two rows per thread, Newton-kernel efficiency).  The long
    // tail and the unproven rows (~20 evaluations each, few rows) finish in the warp-per-row kernel.
    {
        PtBuf<uint32_t> list2, list3;
        // with the support set resident in shared memory the warp-per-row kernel takes the enclosed rows directly (a few
        // hundred 256-row blocks would not fill the machine); otherwise four step launches thin the list out first
        const bool resident = ((size_t)f->d.S * PT_ROW64(N) + PT_EXP_TAB) * sizeof(double) <= PT_TC_SMEM_LIMIT;
        const int max_steps = 4;
        const int n_steps = resident ? 0 : max_steps;
        PT_TRY(list2.alloc(ctx, m)); PT_TRY(list3.alloc(ctx, m));
        PT_TRY(steps.alloc(ctx, max_steps + 5));
        PT_CUDA(ctx, cudaMemsetAsync(steps.p, 0, (max_steps + 5) * sizeof(unsigned long long), ctx->stream));
        steps_dbg = steps.p;
        {
            PT_LAUNCH(ctx, "bisect_select");
            pt_select_flag_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(slow.p, (uint8_t)2, m, list.p, steps.p);
            PT_TRY(pt_check_launch(ctx, "pt_select_flag_kernel"));
            pt_select_flag_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(slow.p, (uint8_t)1, m, list3.p, steps.p + max_steps + 1);
            PT_TRY(pt_check_launch(ctx, "pt_select_flag_kernel"));
        }
        PT_LAUNCH(ctx, "bisect_fp64_rest");
        uint32_t* lin = list.p; uint32_t* lout = list2.p;
        for (int step = 0; step < n_steps; ++step) {
            pt_bisect_step_kernel<N><<<pt_grid_for(m, 256), 128, smem, ctx->stream>>>(f->d, lin, steps.p + step, a, b, sa, lo.p, hi.p, jlo.p, jhi.p,
                                                                                      eps, out, lout, steps.p + step + 1, ctx->work);
            PT_TRY(pt_check_launch(ctx, "pt_bisect_step_kernel"));
            uint32_t* sw = lin; lin = lout; lout = sw;
        }
        // support rows per shared-memory chunk of the warp-per-row kernel (the whole set when it fits)
        const size_t row_bytes = (size_t)PT_ROW64(N) * sizeof(double);
        long long chunk_rows = (long long)((PT_TC_SMEM_LIMIT - PT_EXP_TAB * sizeof(double)) / row_bytes);
        if (chunk_rows > f->d.S) chunk_rows = f->d.S;
        const size_t smem_w = (size_t)chunk_rows * row_bytes + PT_EXP_TAB * sizeof(double);
        // per launch: the attribute is per device, and a process may hold contexts on several devices (~1 us)
        PT_CUDA(ctx, cudaFuncSetAttribute(pt_bisect_rest_warp_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_TC_SMEM_LIMIT));
        const unsigned gridw = pt_grid_for(m, PT_RESTW_THREADS / 32, (unsigned)ctx->sm_count);
        const PtRows tail{lin, steps.p + n_steps, m}, unproven{list3.p, steps.p + max_steps + 1, m};
        pt_bisect_rest_warp_kernel<N><<<gridw, PT_RESTW_THREADS, smem_w, ctx->stream>>>(f->d, tail, a, b, sa, lo.p, hi.p, jlo.p, jhi.p, eps, out,
                                                                                        (int)chunk_rows, steps.p + max_steps + 2, ctx->work);
        PT_TRY(pt_check_launch(ctx, "pt_bisect_rest_warp_kernel"));
        pt_bisect_rest_warp_kernel<N><<<gridw, PT_RESTW_THREADS, smem_w, ctx->stream>>>(f->d, unproven, a, b, sa, lo.p, hi.p, jlo.p, jhi.p, eps, out,
                                                                                        (int)chunk_rows, steps.p + max_steps + 3, ctx->work);
        PT_TRY(pt_check_launch(ctx, "pt_bisect_rest_warp_kernel"));
    }
#undef PT_G_LAUNCH
    if (getenv("PT_DEBUG_COUNTS")) {
        unsigned long long hs[16];
        cudaMemcpyAsync(hs, steps_dbg, 9 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        fprintf(stderr, "[pt] open rows: enclosed=%llu unproven=%llu after-steps=%llu\n", hs[0], hs[5], hs[4]);
        unsigned long long hn[PT_NEWTON_RETRIES];
        cudaMemcpyAsync(hn, ncnt.p, sizeof(hn), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        fprintf(stderr, "[pt] proof retries:");
        for (int i = 0; i < PT_NEWTON_RETRIES; ++i) fprintf(stderr, " %llu", hn[i]);
        fprintf(stderr, "\n");
        unsigned long long h[2];
        cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        fprintf(stderr, "[pt] root solve m=%zu resolve_round1=%llu resolve_round2=%llu tc=%d\n", m, h[0], h[1], (int)use_tc);
    }
    return PT_OK;
}

#define PT_DISPATCH_N(n, CALL)                                                   \
    switch (n) {                                                                 \
        case 2: return CALL(2);                                                  \
        case 3: return CALL(3);                                                  \
        case 4: return CALL(4);                                                  \
        case 5: return CALL(5);                                                  \
        case 6: return CALL(6);                                                  \
        case 7: return CALL(7);                                                  \
        default: return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", (n)); \
    }

int pt_field_eval_dev(pt_ctx* ctx, const pt_field* f, const double* pts_dev, size_t m, double* vals_dev,
                      int8_t* signs_dev, float* vals32_dev) {
    if (m == 0) return PT_OK;
#define CALL(N) pt_eval_launch<N>(ctx, f, pts_dev, m, vals_dev, signs_dev, vals32_dev)
    PT_DISPATCH_N(f->d.n, CALL)
#undef CALL
}

int pt_field_bisect_dev(pt_ctx* ctx, const pt_field* f, const double* a_dev, const double* b_dev,
                        const int8_t* signs_a_dev, size_t m, double eps, double* out_dev, const float* hint_dev) {
    if (m == 0) return PT_OK;
#define CALL(N) pt_bisect_launch<N>(ctx, f, a_dev, b_dev, signs_a_dev, m, eps, out_dev, hint_dev)
    PT_DISPATCH_N(f->d.n, CALL)
#undef CALL
}

extern "C" int pt_debug_tc_arg_error(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, long long m, double* out);

static int pt_field_build_rbf(pt_ctx* ctx, int n, long long S, const double* support, const double* weights,
                              double gamma, double bias, const double* barrier_host, pt_field** out) {
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", n);
    if (S < 0) return pt_fail(ctx, PT_E_INVALID, "negative support count");
    pt_field* f = new pt_field();
    f->ctx = ctx;
    memset(&f->d, 0, sizeof(f->d));
    f->d.kind = PT_FIELD_RBF; f->d.n = n; f->d.S = S; f->d.row = pt_sv_row(n);
    {
        const char* env = getenv("PERMATRACE_B200_PRECISION");
        f->precision = (env && env[0] == '0') ? 0 : 1;
    }
    f->d.gamma = gamma; f->d.bias = bias;
    if (barrier_host) {
        f->d.has_barrier = 1;
        f->d.b_scale = barrier_host[0]; f->d.b_gain = barrier_host[1];
        for (int d = 0; d < n; ++d) { f->d.b_lo[d] = barrier_host[2 + d]; f->d.b_hi[d] = barrier_host[2 + n + d]; }
    }
    int rc = f->sv.alloc(ctx, (size_t)(S > 0 ? S : 1) * f->d.row);
    if (rc != PT_OK) { delete f; return rc; }
    if (S > 0) {
        PtBuf<double> tmp_s, tmp_w;
        const double *sdev, *wdev;
        rc = pt_stage_in(ctx, support, (size_t)S * n, tmp_s, &sdev);
        if (rc == PT_OK) rc = pt_stage_in(ctx, weights, (size_t)S, tmp_w, &wdev);
        if (rc != PT_OK) { delete f; return rc; }
        f->d.row32 = pt_sv_row32(n);
        rc = f->sv32.alloc(ctx, (size_t)S * f->d.row32);
        PtBuf<unsigned long long> rmax;
        if (rc == PT_OK) rc = rmax.alloc(ctx, 2);
        if (rc != PT_OK) { delete f; return rc; }
        cudaMemsetAsync(rmax.p, 0, 2 * sizeof(unsigned long long), ctx->stream);
        pt_pack_sv_kernel<<<pt_grid_for((size_t)S, 256), 256, 0, ctx->stream>>>(sdev, wdev, S, n, f->d.row, f->d.row32, gamma * PT_L2E,
                                                                              f->sv.p, f->sv32.p, rmax.p, (double*)(rmax.p + 1));
        rc = pt_check_launch(ctx, "pt_pack_sv_kernel");
        if (rc != PT_OK) { delete f; return rc; }
        unsigned long long bits[2] = {0, 0};
        cudaMemcpyAsync(bits, rmax.p, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        memcpy(&f->d.smax, &bits[0], sizeof(double));
        memcpy(&f->sum_abs_w, &bits[1], sizeof(double));
        f->d.amb_tol = 1e-12 * (f->sum_abs_w + fabs(bias));
        f->d.sv32 = f->sv32.p;
        // sign-sorted rows of the Taylor-model root solve (stable partition by an exclusive scan of the sign flags)
        {
            const char* ty_env = getenv("PERMATRACE_B200_TAYLOR");
            if (!(ty_env && ty_env[0] == '0') && f->precision != 0) {
                PtBuf<unsigned> flag, rank; PtBuf<uint8_t> tmp;
                size_t tb = 0;
                rc = flag.alloc(ctx, (size_t)S);
                if (rc == PT_OK) rc = rank.alloc(ctx, (size_t)S);
                if (rc != PT_OK) { delete f; return rc; }
                pt_taylor_flag_kernel<<<pt_grid_for((size_t)S, 256), 256, 0, ctx->stream>>>(wdev, S, flag.p);
                cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, rank.p, (long long)S, ctx->stream);
                rc = tmp.alloc(ctx, tb);
                if (rc != PT_OK) { delete f; return rc; }
                cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, rank.p, (long long)S, ctx->stream);
                unsigned last[2] = {0, 0};
                cudaMemcpyAsync(&last[0], rank.p + (S - 1), sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
                cudaMemcpyAsync(&last[1], flag.p + (S - 1), sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
                cudaStreamSynchronize(ctx->stream);
                const long long n_pos = (long long)last[0] + (long long)last[1], n_neg = S - n_pos;
                f->t_pos = (n_pos + 1) & ~1ll;
                f->t_tot = f->t_pos + ((n_neg + 1) & ~1ll);
                const int rowt = (n + 2) & ~1;
                rc = f->svt.alloc(ctx, (size_t)f->t_tot * rowt);
                if (rc != PT_OK) { delete f; return rc; }
                const long long span = f->t_tot > S ? f->t_tot : S;
                pt_taylor_pack_kernel<<<pt_grid_for((size_t)span, 256), 256, 0, ctx->stream>>>(sdev, wdev, S, n, rowt, gamma * PT_L2E, flag.p,
                                                                                              rank.p, f->t_pos, f->t_tot, f->svt.p);
                rc = pt_check_launch(ctx, "pt_taylor_pack_kernel");
                if (rc != PT_OK) { delete f; return rc; }
                cudaStreamSynchronize(ctx->stream);
                f->taylor = true;
                // direction sums for the grouped variant (2^n x t_tot doubles: 1 MB at n = 6, S = 2048)
                const char* dir_env = getenv("PERMATRACE_B200_TAYLOR_DIR");
                if (!(dir_env && dir_env[0] == '0') && n <= 7 && ((size_t)f->t_tot << n) * sizeof(double) <= ((size_t)1 << 30)) {
                    rc = f->dirtab.alloc(ctx, (size_t)f->t_tot << n);
                    if (rc != PT_OK) { delete f; return rc; }
                    const dim3 dgrid(pt_grid_for((size_t)f->t_tot, 256), 1u << n);
                    pt_taylor_dirtab_kernel<<<dgrid, 256, 0, ctx->stream>>>(f->svt.p, rowt, n, f->t_tot, f->dirtab.p);
                    rc = pt_check_launch(ctx, "pt_taylor_dirtab_kernel");
                    if (rc != PT_OK) { delete f; return rc; }
                    cudaStreamSynchronize(ctx->stream);
                    f->taylor_dir = true;
                }
            }
        }
        // tensor-core screen operand, when the whole packed support set fits one CTA's shared memory
        const char* tc_env = getenv("PERMATRACE_B200_TC");
        if (!(tc_env && tc_env[0] == '0') && n <= 6) {
            const int kt = pt_tc_kt(n), spad = (int)pt_tc_spad(S);
            rc = f->tc_bt.alloc(ctx, (size_t)kt * spad);
            if (rc == PT_OK) rc = f->tc_wt.alloc(ctx, (size_t)spad);
            if (rc != PT_OK) { delete f; return rc; }
            pt_pack_tc_kernel<<<pt_grid_for((size_t)spad, 256), 256, 0, ctx->stream>>>(sdev, wdev, S, n, spad, kt, gamma * PT_L2E,
                                                                                     f->tc_bt.p, f->tc_wt.p);
            rc = pt_check_launch(ctx, "pt_pack_tc_kernel");
            if (rc != PT_OK) { delete f; return rc; }
            f->tc.bt = f->tc_bt.p; f->tc.wt = f->tc_wt.p; f->tc.spad = spad; f->tc.kt = kt;
            f->tc_ok = true;
            f->tc_resident = pt_tc_smem_bytes(n, S) <= PT_TC_SMEM_LIMIT;
            const char* lv_env = getenv("PERMATRACE_B200_TC_LEVELS");
            f->tc_levels = lv_env && lv_env[0] == '1';
            const char* g4_env = getenv("PERMATRACE_B200_TC4");
            const size_t smem4 = (size_t)5 * spad * 16 + 4 * (size_t)6 * PT_TC_M * 16 + (size_t)spad * 4 + 64;
            f->tc4 = n == 6 && smem4 <= PT_TC_SMEM_LIMIT && !(g4_env && g4_env[0] == '0');
            cudaStreamSynchronize(ctx->stream);   // sdev/wdev may be staging buffers released on return
            // The tensor-core accumulation error is not specified by PTX; PT_TC_ARG_ULPS is calibrated.  Spot-check it on
            // THIS field (exponents of up to 4096 support vectors against all of them, in fp64): a field whose measured
            // error passes half the bound does not get the tensor-core paths at all.
            if (f->tc_resident && S >= 64) {
                const long long ms = S < 4096 ? S : 4096;
                std::vector<double> errs((size_t)ms);
                f->d.sv = f->sv.p;
                const int src = pt_debug_tc_arg_error(ctx, f, sdev, sdev, ms, errs.data());
                double worst = 0.0;
                for (double e : errs) worst = (e == e && e > worst) ? e : (e == e ? worst : 1e300);
                if (src != PT_OK || !(worst < 0.5 * PT_TC_ARG_ULPS)) {
                    fprintf(stderr, "[permatrace_b200] tensor-core exponent error %.3g u32*T on this field (bound %.1f): "
                                    "tensor-core paths disabled for it\n", worst, (double)PT_TC_ARG_ULPS);
                    f->tc_ok = false; f->tc_resident = false; f->tc4 = false;
                }
            }
        }
    }
    f->d.sv = f->sv.p;
    *out = f;
    return PT_OK;
}

template <int N>
static int pt_gradient_launch(pt_ctx* ctx, const pt_field* f, const double* pts, size_t m, double* out) {
    pt_gradient_rbf_kernel<N><<<pt_grid_for(m, PT_EVAL_THREADS), PT_EVAL_THREADS, PT_SMEM64(N), ctx->stream>>>(f->d, pts, m, out);
    return pt_check_launch(ctx, "pt_gradient_rbf_kernel");
}

static int pt_gradient_dispatch(pt_ctx* ctx, const pt_field* f, const double* pts, size_t m, double* out) {
#define CALL(N) pt_gradient_launch<N>(ctx, f, pts, m, out)
    PT_DISPATCH_N(f->d.n, CALL)
#undef CALL
}

extern "C" {

int pt_field_create_rbf(pt_ctx* ctx, int n, long long S, const double* support, const double* weights,
                        double gamma, double bias, const double* barrier, pt_field** out) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_field_create_rbf: NULL argument");
    if (S > 0 && (!support || !weights)) return pt_fail(ctx, PT_E_INVALID, "support/weights are NULL");
    if (!(gamma > 0.0)) return pt_fail(ctx, PT_E_INVALID, "gamma must be positive");
    return pt_field_build_rbf(ctx, n, S, support, weights, gamma, bias, barrier, out);
}

int pt_field_create_analytic(pt_ctx* ctx, int kind, int n, const double* params, pt_field** out) {
    if (!ctx || !out || !params) return pt_fail(ctx, PT_E_INVALID, "pt_field_create_analytic: NULL argument");
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", n);
    if (kind != PT_FIELD_SPHERE && kind != PT_FIELD_ELLIPSOID && kind != PT_FIELD_PLANE)
        return pt_fail(ctx, PT_E_INVALID, "unknown analytic field kind %d", kind);
    pt_field* f = new pt_field();
    f->ctx = ctx;
    memset(&f->d, 0, sizeof(f->d));
    f->d.kind = kind; f->d.n = n;
    for (int d = 0; d < n; ++d) f->d.p0[d] = params[d];
    if (kind == PT_FIELD_ELLIPSOID) for (int d = 0; d < n; ++d) f->d.p1[d] = params[n + d];
    else f->d.c0 = params[n];
    *out = f;
    return PT_OK;
}

void pt_field_destroy(pt_field* f) { delete f; }

int pt_field_set_precision(pt_field* f, int mode) {
    if (!f) return pt_fail(nullptr, PT_E_INVALID, "field is NULL");
    if (mode != 0 && mode != 1) return pt_fail(f->ctx, PT_E_INVALID, "precision mode must be 0 (fp64) or 1 (fp32-screened)");
    f->precision = mode;
    return PT_OK;
}

int pt_field_values(pt_ctx* ctx, const pt_field* f, const double* points, long long m, double* out_values,
                    int8_t* out_signs) {
    if (!ctx || !f) return pt_fail(ctx, PT_E_INVALID, "pt_field_values: NULL argument");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative point count");
    if (m == 0) return PT_OK;
    if (!points) return pt_fail(ctx, PT_E_INVALID, "points is NULL");
    const int n = f->d.n;
    PtBuf<double> tmp_p, tmp_v; PtBuf<int8_t> tmp_s;
    const double* pdev;
    PT_TRY(pt_stage_in(ctx, points, (size_t)m * n, tmp_p, &pdev));
    double* vdev = nullptr; int8_t* sdev = nullptr;
    if (out_values) { if (pt_is_device_ptr(out_values)) vdev = out_values; else { PT_TRY(tmp_v.alloc(ctx, m)); vdev = tmp_v.p; } }
    if (out_signs) { if (pt_is_device_ptr(out_signs)) sdev = out_signs; else { PT_TRY(tmp_s.alloc(ctx, m)); sdev = tmp_s.p; } }
    PT_TRY(pt_field_eval_dev(ctx, f, pdev, (size_t)m, vdev, sdev));
    if (out_values && vdev != out_values) PT_TRY(pt_copy_out(ctx, out_values, vdev, (size_t)m, false));
    if (out_signs && sdev != out_signs) PT_TRY(pt_copy_out(ctx, out_signs, sdev, (size_t)m, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_field_gradients(pt_ctx* ctx, const pt_field* f, const double* points, long long m, double* out) {
    if (!ctx || !f) return pt_fail(ctx, PT_E_INVALID, "pt_field_gradients: NULL argument");
    if (f->d.kind != PT_FIELD_RBF) return pt_fail(ctx, PT_E_INVALID, "pt_field_gradients serves KernelClassifierManifold fields");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative point count");
    if (m == 0) return PT_OK;
    if (!points || !out) return pt_fail(ctx, PT_E_INVALID, "points/out is NULL");
    const int n = f->d.n;
    PtBuf<double> tmp_p, tmp_o;
    const double* pdev;
    PT_TRY(pt_stage_in(ctx, points, (size_t)m * n, tmp_p, &pdev));
    double* odev = out;
    if (!pt_is_device_ptr(out)) { PT_TRY(tmp_o.alloc(ctx, (size_t)m * n)); odev = tmp_o.p; }
    {
        PT_LAUNCH(ctx, "gradient_rbf");
        PT_TRY(pt_gradient_dispatch(ctx, f, pdev, (size_t)m, odev));
    }
    if (odev != out) PT_TRY(pt_copy_out(ctx, out, odev, (size_t)m * n, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_intersection_points(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, long long m,
                           double eps, const int8_t* signs_a, double* out) {
    if (!ctx || !f) return pt_fail(ctx, PT_E_INVALID, "pt_intersection_points: NULL argument");
    if (!(eps > 0.0)) return pt_fail(ctx, PT_E_INVALID, "eps must be positive");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative segment count");
    if (m == 0) return PT_OK;
    if (!a || !b || !out) return pt_fail(ctx, PT_E_INVALID, "endpoint/output arrays are NULL");
    const int n = f->d.n;
    PtBuf<double> ta, tb, to; PtBuf<int8_t> ts;
    const double *adev, *bdev; const int8_t* sdev;
    PT_TRY(pt_stage_in(ctx, a, (size_t)m * n, ta, &adev));
    PT_TRY(pt_stage_in(ctx, b, (size_t)m * n, tb, &bdev));
    if (signs_a) PT_TRY(pt_stage_in(ctx, signs_a, (size_t)m, ts, &sdev));
    else {
        PT_TRY(ts.alloc(ctx, m));
        PT_TRY(pt_field_eval_dev(ctx, f, adev, (size_t)m, nullptr, ts.p));
        sdev = ts.p;
    }
    double* odev = out;
    if (!pt_is_device_ptr(out)) { PT_TRY(to.alloc(ctx, (size_t)m * n)); odev = to.p; }
    PT_TRY(pt_field_bisect_dev(ctx, f, adev, bdev, sdev, (size_t)m, eps, odev));
    if (odev != out) PT_TRY(pt_copy_out(ctx, out, odev, (size_t)m * n, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_debug_tc_arg_error(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, long long m, double* out) {
    if (!ctx || !f || !a || !b || !out || m <= 0) return pt_fail(ctx, PT_E_INVALID, "pt_debug_tc_arg_error: bad argument");
    if (f->d.kind != PT_FIELD_RBF || !f->tc_resident) return pt_fail(ctx, PT_E_STATE, "field has no resident tensor-core operand");
    const int n = f->d.n;
    PtBuf<double> ta, tb, lo, hi; PtBuf<int8_t> sa;
    const double *adev, *bdev;
    PT_TRY(pt_stage_in(ctx, a, (size_t)m * n, ta, &adev));
    PT_TRY(pt_stage_in(ctx, b, (size_t)m * n, tb, &bdev));
    PT_TRY(lo.alloc(ctx, m)); PT_TRY(hi.alloc(ctx, m)); PT_TRY(sa.alloc(ctx, m));
    PT_CUDA(ctx, cudaMemsetAsync(sa.p, 1, (size_t)m, ctx->stream));
    const PtRows all{nullptr, nullptr, (size_t)m};
    int rc;
    switch (n) {
        case 2: rc = pt_screen_tc_launch<2, 1>(ctx, f, all, adev, bdev, sa.p, 1e-9, 1, lo.p, hi.p, nullptr); break;
        case 3: rc = pt_screen_tc_launch<3, 1>(ctx, f, all, adev, bdev, sa.p, 1e-9, 1, lo.p, hi.p, nullptr); break;
        case 4: rc = pt_screen_tc_launch<4, 1>(ctx, f, all, adev, bdev, sa.p, 1e-9, 1, lo.p, hi.p, nullptr); break;
        case 5: rc = pt_screen_tc_launch<5, 1>(ctx, f, all, adev, bdev, sa.p, 1e-9, 1, lo.p, hi.p, nullptr); break;
        case 6: rc = pt_screen_tc_launch<6, 1>(ctx, f, all, adev, bdev, sa.p, 1e-9, 1, lo.p, hi.p, nullptr); break;
        default: return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported by the tensor-core screen", n);
    }
    PT_TRY(rc);
    return pt_copy_out(ctx, out, hi.p, (size_t)m, true);
}

int pt_rbf_values(pt_ctx* ctx, const double* points, long long m, int n, const double* support, long long S,
                  const double* weights, double gamma, double bias, double* out) {
    if (!ctx) return pt_fail(ctx, PT_E_INVALID, "ctx is NULL");
    if (m < 0 || S < 0) return pt_fail(ctx, PT_E_INVALID, "negative size");
    if (m == 0) return PT_OK;
    if (!out || !points) return pt_fail(ctx, PT_E_INVALID, "points/out is NULL");
    pt_field* f = nullptr;
    // gamma sign is the caller's business at this seam (the reference kernel accepts any double)
    PT_TRY(pt_field_build_rbf(ctx, n, S, support, weights, gamma, bias, nullptr, &f));
    int rc = pt_field_values(ctx, f, points, m, out, nullptr);
    pt_field_destroy(f);
    return rc;
}

}  // extern "C"
