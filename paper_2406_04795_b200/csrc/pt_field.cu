// Field evaluation and per-edge root solve (bisection) kernels + their C ABI.
//
//   pt_eval_rbf_kernel<N,G>    values/signs of the kernel-SVM field at m points; G lanes share a
//                              point and split the support set, support rows staged in shared memory
//   pt_bisect_rbf_kernel<N,G>  intersection_points_batch: every segment halves its own bracket
//                              until seg*(hi-lo) <= eps  (manifold.py:368-383)
//   *_analytic_*               same for sphere/ellipsoid/plane fields, arithmetic ordered like numpy
#include <stdlib.h>
#include "pt_internal.cuh"
#include "pt_field.cuh"

struct pt_field {
    pt_ctx* ctx = nullptr;
    PtFieldDev d;
    PtBuf<double> sv;
    PtBuf<float> sv32;
    int precision = 0;
    double sum_abs_w = 0.0;
};

int pt_field_dim(const pt_field* f) { return f->d.n; }

#define PT_EVAL_THREADS 256
#define PT_EVAL_TILE 256

template <int N>
__device__ __forceinline__ double pt_rbf_term(const double* __restrict__ row, const double* p, double neg_gamma) {
    double d2 = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) { double df = p[d] - row[d]; d2 = fma(df, df, d2); }
    return row[N] * exp(neg_gamma * d2);
}

// accumulate this lane's share of sum_j w_j k(p, s_j); all threads of the block must call it
template <int N, int G>
__device__ __forceinline__ double pt_rbf_block_sum(const PtFieldDev& f, const double* p, int g, double* tile) {
    const int ROW = (N + 1) | 1;
    double acc = 0.0;
    const double ng = -f.gamma;
    for (long long t0 = 0; t0 < f.S; t0 += PT_EVAL_TILE) {
        long long rem = f.S - t0;
        int cnt = rem < PT_EVAL_TILE ? (int)rem : PT_EVAL_TILE;
        __syncthreads();
        const double* src = f.sv + t0 * ROW;
        for (int i = threadIdx.x; i < cnt * ROW; i += PT_EVAL_THREADS) tile[i] = src[i];
        __syncthreads();
        for (int j = g; j < cnt; j += G) acc += pt_rbf_term<N>(tile + j * ROW, p, ng);
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    return acc;
}

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_eval_rbf_kernel(PtFieldDev f, const double* __restrict__ pts, size_t m, double* __restrict__ vals,
                   int8_t* __restrict__ signs, unsigned long long* work) {
    extern __shared__ double tile[];
    const int PB = PT_EVAL_THREADS / G;
    const size_t pi = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = pi < m;
    double p[N];
#pragma unroll
    for (int d = 0; d < N; ++d) p[d] = valid ? pts[pi * N + d] : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&work[1], (unsigned long long)m);
    double acc = pt_rbf_block_sum<N, G>(f, p, g, tile);
    if (valid && g == 0) {
        double F = f.bias + acc;
        if (f.has_barrier) F -= pt_barrier_value<N>(f, p);
        if (vals) vals[pi] = F;
        if (signs) signs[pi] = F > 0.0 ? (int8_t)1 : (int8_t)-1;
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


// ==== fast root solve: fp32-screened bisection + fp64 secant endgame ================================
// Phase 1 (pt_bisect32_kernel) replays the reference's bisection with the field evaluated in fp32; a
// step is taken only when |F32| exceeds a rigorous bound on |F32 - F| (so the decision equals the
// fp64 one), otherwise the row stops with its current dyadic bracket.
// Phase 2 (pt_bisect_finish_kernel) finds the root inside that bracket by two fp64 secant steps,
// maps it to the depth-I dyadic cell the reference's bisection would end in, and VERIFIES the cell
// by evaluating the field at its two ends with exactly the midpoints' arithmetic (sign(a side) ==
// signs_a, other side differs).  A failed verification falls back to plain fp64 bisection from the
// phase-1 bracket, so the returned point is always the reference's a + (lo+hi)/2 * (b-a).
#define PT_TILE32 512

template <int N> struct PtRow32 { static const int value = (N + 2 + 3) & ~3; };

__device__ __forceinline__ float pt_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

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

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_bisect32_kernel(PtFieldDev f, const double* __restrict__ a_, const double* __restrict__ b_,
                   const int8_t* __restrict__ signs_a, size_t m, double eps, double* __restrict__ lo_out,
                   double* __restrict__ hi_out, unsigned long long* work) {
    extern __shared__ float tile32[];
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
    const double gl = f.gamma * PT_L2E;
    double lo = 0.0, hi = 1.0;
    bool active = valid && seg > eps;
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
        // |arg32 - arg| <= (N+4) u T with T = gamma*log2(e) (|p| + max|s|)^2 (input roundings + fma chain);
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
                active = __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
            } else {
                active = false;   // sign not certain in fp32 (or NaN): hand the bracket to phase 2
            }
        }
    }
    {
        unsigned mine = (g == 0) ? iters : 0u;
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&work[2], (unsigned long long)mine);
    }
    if (valid && g == 0) { lo_out[ei] = lo; hi_out[ei] = hi; }
}

template <int N, int G>
__global__ void __launch_bounds__(PT_EVAL_THREADS)
pt_bisect_finish_kernel(PtFieldDev f, const double* __restrict__ a_, const double* __restrict__ b_,
                        const int8_t* __restrict__ signs_a, const double* __restrict__ lo_in,
                        const double* __restrict__ hi_in, size_t m, double eps, double* __restrict__ out,
                        unsigned long long* work) {
    extern __shared__ double tile[];
    const int PB = PT_EVAL_THREADS / G;
    const size_t ei = (size_t)blockIdx.x * PB + threadIdx.x / G;
    const int g = threadIdx.x % G;
    const bool valid = ei < m;
    double a[N], diff[N], p[N];
    double seg = 0.0, lo = 0.0, hi = 1.0;
    int sa = 1;
    if (valid) {
        double b[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
        seg = pt_segment<N>(a, b, diff);
        sa = signs_a[ei];
        lo = lo_in[ei]; hi = hi_in[ei];
    } else {
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; }
    }
    unsigned evals = 0;
    // F at parameter t with the reference's point arithmetic; every thread of the block calls it
    auto eval = [&](double t, bool count) -> double {
#pragma unroll
        for (int d = 0; d < N; ++d) p[d] = __dadd_rn(a[d], __dmul_rn(t, diff[d]));
        double F = f.bias + pt_rbf_block_sum<N, G>(f, p, g, tile);
        if (f.has_barrier) F -= pt_barrier_group<N, G>(f, p, g);
        if (count) ++evals;
        return F;
    };
    auto sgn = [](double F) -> int { return F > 0.0 ? 1 : -1; };
    // depth of the reference's final bracket: smallest I with seg * 2^-I <= eps
    double delta = 1.0;
    if (valid) while (__dmul_rn(seg, delta) > eps) delta *= 0.5;
    const double width = hi - lo;
    const bool need = valid && width > delta;       // phase 1 did not reach the final depth
    double t_final = __dmul_rn(0.5, __dadd_rn(lo, hi));
    bool fallback = false;
    if (__syncthreads_or(need ? 1 : 0)) {
        const double F_lo = eval(lo, need);
        const double F_hi = eval(hi, need);
        const bool ok = need && sgn(F_lo) == sa && sgn(F_hi) != sa;
        // safeguarded secant on (x0,f0),(x1,f1); [blo,bhi] is the sign bracket.  The next iterate is
        // used WITHOUT being evaluated once its predicted error 10*e_cur*e_prev (e = |f / slope|, the
        // secant's error recursion with a generous curvature constant) is far below the cell width.
        double x0 = lo, f0 = F_lo, x1 = hi, f1 = F_hi, blo = lo, bhi = hi;
        const double slope = fabs((F_hi - F_lo) / width) + 1e-300;
        double e_prev = width, e_cur = width;
        double x2 = lo + 0.5 * width;
        bool searching = ok;
        for (int it = 0; it < 8; ++it) {
            if (searching) {
                const double den = f1 - f0;
                x2 = (den != 0.0) ? x1 - f1 * ((x1 - x0) / den) : 0.5 * (blo + bhi);
                if (!(x2 > blo && x2 < bhi)) x2 = 0.5 * (blo + bhi);
                if (10.0 * e_cur * e_prev < 0.0625 * delta) searching = false;
            }
            if (!__syncthreads_or(searching ? 1 : 0)) break;
            const double f2 = eval(x2, searching);
            if (searching) {
                if (sgn(f2) == sa) blo = x2; else bhi = x2;
                x0 = x1; f0 = f1; x1 = x2; f1 = f2;
                e_prev = e_cur; e_cur = fabs(f2) / slope;
            }
        }
        const double nsub = width / delta;            // exact: both are powers of two
        double j = floor((x2 - lo) / delta);
        if (!(j >= 0.0)) j = 0.0;
        if (j > nsub - 1.0) j = nsub - 1.0;
        double c = lo + j * delta;                    // exact dyadic arithmetic
        const int sc = sgn(eval(c, need));
        const int sd = sgn(eval(c + delta, need));
        bool accepted = ok && sc == sa && sd != sa;
        // one neighbouring cell when the secant landed within rounding of a cell boundary
        const bool try_left = ok && !accepted && sc != sa && j > 0.0;
        const bool try_right = ok && !accepted && sc == sa && sd == sa && j < nsub - 1.0;
        if (__syncthreads_or((try_left || try_right) ? 1 : 0)) {
            const double tq = try_left ? c - delta : c + 2.0 * delta;
            const int sq = sgn(eval(tq, try_left || try_right));
            if (try_left && sq == sa) { c = c - delta; accepted = true; }
            if (try_right && sq != sa) { c = c + delta; accepted = true; }
        }
        if (need) {
            if (accepted) t_final = c + 0.5 * delta;
            else {
                fallback = true;
                // a bracket whose ends do not show the expected signs cannot be trusted: replay from [0,1]
                if (!ok) { lo = 0.0; hi = 1.0; }
            }
        }
    }
    // plain fp64 bisection from the phase-1 bracket for the rows that could not be verified
    bool active = fallback;
    while (__syncthreads_or(active ? 1 : 0)) {
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
        const int s = sgn(eval(mid, active));
        if (active) {
            if (s == sa) lo = mid; else hi = mid;
            active = __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
            if (!active) t_final = __dmul_rn(0.5, __dadd_rn(lo, hi));
        }
    }
    {
        unsigned mine = (g == 0) ? evals : 0u;
        unsigned fb = (g == 0 && fallback) ? 1u : 0u;
        for (int off = 16; off > 0; off >>= 1) { mine += __shfl_xor_sync(0xffffffffu, mine, off); fb += __shfl_xor_sync(0xffffffffu, fb, off); }
        if ((threadIdx.x & 31) == 0) {
            if (mine) atomicAdd(&work[0], (unsigned long long)mine);
            if (fb) atomicAdd(&work[3], (unsigned long long)fb);
        }
    }
    if (valid && g == 0) {
#pragma unroll
        for (int d = 0; d < N; ++d) out[ei * N + d] = __dadd_rn(a[d], __dmul_rn(t_final, diff[d]));
    }
}

// pack the fp32 screening copy and record max |s_j|
__global__ void pt_pack_sv32_kernel(const double* __restrict__ sv, long long S, int n, int row, int row32, double gl,
                                    float* __restrict__ sv32, unsigned long long* rmax_bits) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    double s2 = 0.0;
    for (int d = 0; d < n; ++d) { double v = sv[j * row + d]; s2 = fma(v, v, s2); sv32[j * row32 + d] = (float)v; }
    sv32[j * row32 + n] = (float)(-gl * s2);
    sv32[j * row32 + n + 1] = (float)sv[j * row + n];
    for (int d = n + 2; d < row32; ++d) sv32[j * row32 + d] = 0.f;
    atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(sqrt(s2)));
}

// pack raw (support[S][n], weights[S]) into the padded row layout
__global__ void pt_pack_sv_kernel(const double* __restrict__ support, const double* __restrict__ weights,
                                  long long S, int n, int row, double* __restrict__ sv) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    for (int d = 0; d < n; ++d) sv[j * row + d] = support[j * n + d];
    sv[j * row + n] = weights[j];
    for (int d = n + 1; d < row; ++d) sv[j * row + d] = 0.0;
}

// lanes per item so that small batches still fill the machine
static int pt_pick_group(pt_ctx* ctx, size_t m, long long S) {
    size_t target = (size_t)ctx->sm_count * 2048;
    if (S < 64) return 1;
    if (m >= target) return 1;
    if (m * 4 >= target || S < 256) return 4;
    return 32;
}

template <int N>
static int pt_eval_launch(pt_ctx* ctx, const pt_field* f, const double* pts, size_t m, double* vals, int8_t* signs) {
    if (f->d.kind != PT_FIELD_RBF) {
        PT_LAUNCH(ctx, "eval_analytic");
        pt_eval_analytic_kernel<N><<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(f->d, pts, m, vals, signs);
        return pt_check_launch(ctx, "pt_eval_analytic_kernel");
    }
    const int G = pt_pick_group(ctx, m, f->d.S);
    const size_t smem = (size_t)PT_EVAL_TILE * ((N + 1) | 1) * sizeof(double);
    PT_LAUNCH(ctx, "eval_rbf");
    if (G == 1)
        pt_eval_rbf_kernel<N, 1><<<pt_grid_for(m, PT_EVAL_THREADS), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, pts, m, vals, signs, ctx->work);
    else if (G == 4)
        pt_eval_rbf_kernel<N, 4><<<pt_grid_for(m, PT_EVAL_THREADS / 4), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, pts, m, vals, signs, ctx->work);
    else
        pt_eval_rbf_kernel<N, 32><<<pt_grid_for(m, PT_EVAL_THREADS / 32), PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, pts, m, vals, signs, ctx->work);
    return pt_check_launch(ctx, "pt_eval_rbf_kernel");
}

template <int N>
static int pt_bisect_launch(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, const int8_t* sa,
                            size_t m, double eps, double* out) {
    if (f->d.kind != PT_FIELD_RBF) {
        PT_LAUNCH(ctx, "bisect_analytic");
        pt_bisect_analytic_kernel<N><<<pt_grid_for(m, 128), 128, 0, ctx->stream>>>(f->d, a, b, sa, m, eps, out);
        return pt_check_launch(ctx, "pt_bisect_analytic_kernel");
    }
    const int G = pt_pick_group(ctx, m, f->d.S);
    const size_t smem = (size_t)PT_EVAL_TILE * ((N + 1) | 1) * sizeof(double);
    const unsigned grid = pt_grid_for(m, PT_EVAL_THREADS / G);
    if (f->precision == 0 || f->d.S == 0) {
        PT_LAUNCH(ctx, "bisect_rbf");
        if (G == 1) pt_bisect_rbf_kernel<N, 1><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        else if (G == 4) pt_bisect_rbf_kernel<N, 4><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        else pt_bisect_rbf_kernel<N, 32><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, m, eps, out, ctx->work);
        return pt_check_launch(ctx, "pt_bisect_rbf_kernel");
    }
    PtBuf<double> lo, hi;
    PT_TRY(lo.alloc(ctx, m));
    PT_TRY(hi.alloc(ctx, m));
    const size_t smem32 = (size_t)PT_TILE32 * PtRow32<N>::value * sizeof(float);
    {
        PT_LAUNCH(ctx, "bisect_fp32_screen");
        if (G == 1) pt_bisect32_kernel<N, 1><<<grid, PT_EVAL_THREADS, smem32, ctx->stream>>>(f->d, a, b, sa, m, eps, lo.p, hi.p, ctx->work);
        else if (G == 4) pt_bisect32_kernel<N, 4><<<grid, PT_EVAL_THREADS, smem32, ctx->stream>>>(f->d, a, b, sa, m, eps, lo.p, hi.p, ctx->work);
        else pt_bisect32_kernel<N, 32><<<grid, PT_EVAL_THREADS, smem32, ctx->stream>>>(f->d, a, b, sa, m, eps, lo.p, hi.p, ctx->work);
        PT_TRY(pt_check_launch(ctx, "pt_bisect32_kernel"));
    }
    {
        PT_LAUNCH(ctx, "bisect_fp64_finish");
        if (G == 1) pt_bisect_finish_kernel<N, 1><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, lo.p, hi.p, m, eps, out, ctx->work);
        else if (G == 4) pt_bisect_finish_kernel<N, 4><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, lo.p, hi.p, m, eps, out, ctx->work);
        else pt_bisect_finish_kernel<N, 32><<<grid, PT_EVAL_THREADS, smem, ctx->stream>>>(f->d, a, b, sa, lo.p, hi.p, m, eps, out, ctx->work);
        PT_TRY(pt_check_launch(ctx, "pt_bisect_finish_kernel"));
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
                      int8_t* signs_dev) {
    if (m == 0) return PT_OK;
#define CALL(N) pt_eval_launch<N>(ctx, f, pts_dev, m, vals_dev, signs_dev)
    PT_DISPATCH_N(f->d.n, CALL)
#undef CALL
}

int pt_field_bisect_dev(pt_ctx* ctx, const pt_field* f, const double* a_dev, const double* b_dev,
                        const int8_t* signs_a_dev, size_t m, double eps, double* out_dev) {
    if (m == 0) return PT_OK;
#define CALL(N) pt_bisect_launch<N>(ctx, f, a_dev, b_dev, signs_a_dev, m, eps, out_dev)
    PT_DISPATCH_N(f->d.n, CALL)
#undef CALL
}

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
        f->precision = (env && env[0] == '1') ? 1 : 0;
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
        pt_pack_sv_kernel<<<pt_grid_for((size_t)S, 256), 256, 0, ctx->stream>>>(sdev, wdev, S, n, f->d.row, f->sv.p);
        rc = pt_check_launch(ctx, "pt_pack_sv_kernel");
        if (rc != PT_OK) { delete f; return rc; }
        f->d.row32 = pt_sv_row32(n);
        rc = f->sv32.alloc(ctx, (size_t)S * f->d.row32);
        PtBuf<unsigned long long> rmax;
        if (rc == PT_OK) rc = rmax.alloc(ctx, 1);
        if (rc != PT_OK) { delete f; return rc; }
        cudaMemsetAsync(rmax.p, 0, sizeof(unsigned long long), ctx->stream);
        pt_pack_sv32_kernel<<<pt_grid_for((size_t)S, 256), 256, 0, ctx->stream>>>(f->sv.p, S, n, f->d.row, f->d.row32,
                                                                                gamma * PT_L2E, f->sv32.p, rmax.p);
        rc = pt_check_launch(ctx, "pt_pack_sv32_kernel");
        if (rc != PT_OK) { delete f; return rc; }
        unsigned long long bits = 0;
        cudaMemcpyAsync(&bits, rmax.p, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        memcpy(&f->d.smax, &bits, sizeof(double));
        f->d.sv32 = f->sv32.p;
    }
    f->d.sv = f->sv.p;
    *out = f;
    return PT_OK;
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
