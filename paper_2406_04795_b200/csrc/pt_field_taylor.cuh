// One-pass root solve of intersection_points_batch (reference manifold.py:351-383) for large batches.
//
// Along an edge q(t) = a + t*diff every kernel term is e_j * exp(u_j tau) * exp(c tau^2) with tau = t - 1/2,
//   e_j = |w_j| exp(-gamma |q(1/2) - s_j|^2),  u_j = -2 gamma (q(1/2) - s_j).diff,  c = -gamma |diff|^2,
// so ONE fp64 pass over the support set that accumulates the moments  M_k = sum_j sgn(w_j) e_j u_j^k  (k < Q) and the
// absolute moments  MA_k = sum_j e_j |u_j|^k  (k even, k <= Q)  yields a polynomial model of the field on the WHOLE edge,
//   F(t) = exp(c tau^2) * [ sum_{k<Q} M_k tau^k / k!  +  R(tau) ] + bias - barrier(q(t)),   |R| <= fac * MA_Q |tau|^Q / Q!,
// with rigorous bounds on the truncation and on the rounding of this pass (both relative to
// sum_j e_j exp(|u_j tau|) <= 2 sum_{k even} MA_k tau^k / k!; the support rows are sorted by the sign of the weight, so the
// absolute moments cost nothing extra, and partial sums are flushed per tile so the summation error does not grow with S).
// The reference's bisection is then replayed on the model:
//   * a midpoint whose |model| exceeds the bound has the sign of the EXACT field there;
//   * once the bracket is narrow enough for a proof of monotonicity the root of the model is polished by Newton steps and
//     enclosed (mean-value bound with a proven lower bound on |F'|); midpoints outside the enclosure J are decided without
//     any evaluation, in exact dyadic arithmetic, exactly like pt_bisect_newton_kernel does;
//   * a midpoint where |model| is below the bound is an AMBIGUOUS point of the bisection: |F| there is below the rounding
//     level of an fp64 evaluation (this kernel's, the plain kernels' and the reference's alike -- the reference's own
//     cross-backend tolerance, pkg/tests/test_backends.py:81-93).  If the model's truncation is below its rounding there the
//     model value IS an evaluation-grade number and its sign is taken; otherwise (root far from the edge midpoint) the row
//     keeps its valid dyadic bracket and goes on to the evaluation-based kernels: flag 1 = no enclosure (proof retries /
//     plain bisection), flag 2 = root enclosed in J, a midpoint inside J needs a true evaluation.
// The returned bracket is therefore the bracket of the bisection on the exact field, except at ambiguous midpoints, where no
// fp64 implementation is determined.
//
// Cost per (edge, support vector) pair: (N+1) + 8 + N + 3 + 1.25 Q + 1 FP64 instructions = 45 at N = 6, Q = 16 --
// against 45 for the two passes of the Newton kernel PLUS about eight fp32 screen levels, resolves and retries before.
// The support set streams through shared memory in tiles, so its size is not limited by one CTA's shared memory.
// (DMMA was measured as an alternative home for the two dot products: benchmarks/dmma_probe.cu -- on B200 the FP64 tensor
// path and the FP64 FMA pipe do not overlap, 24.2 ms together against 11.4 + 10.5 ms alone, so nothing is gained.)
#pragma once

#ifndef PT_TAYLOR_Q
#define PT_TAYLOR_Q 16                /* moments about the edge midpoint (no hint of where the root is); measured on dof6 /
                                       * dof6-stress: Q = 20 28.9 / 265 ms, Q = 16 28.1 / 251 ms (more rows take the
                                       * recentred second pass, the first one is 10 % shorter), Q = 12 32.5 / 250 ms */
#endif
#define PT_TAYLOR_Q_HINT 12           /* moments about a secant estimate of the root */
#define PT_TAYLOR_THREADS 128
#ifndef PT_TAYLOR_TILE
#define PT_TAYLOR_TILE 128              /* support rows per shared-memory tile = block of the blocked accumulation */
#endif
#ifndef PT_TAYLOR_MINB
#define PT_TAYLOR_MINB 5              /* resident CTAs per SM the register budget is cut for */
#endif
#ifndef PT_TAYLOR_MINB_DIR
#define PT_TAYLOR_MINB_DIR 6          /* ditto, direction-table variant (its loop keeps N-1 fewer values live) */
#endif
#ifdef PT_TAYLOR_NO_CS
#define PT_TAYLOR_LDCS(p) (*(p))
#define PT_TAYLOR_STCS(p, v) (*(p) = (v))
#else
#define PT_TAYLOR_LDCS(p) __ldcs(p)
#define PT_TAYLOR_STCS(p, v) __stcs((p), (v))
#endif
#define PT_TAYLOR_TRY_WIDTH 0.0625     /* first enclosure attempt once the bracket is this narrow (in t) */

template <int N> struct PtRowT { static const int value = (N + 2) & ~1; };   // 2*gl*s_d (N), c'_s, pad to an even count

// shared-memory row of the direction-table variant: the packed row plus T_j = sum_{d in mask} 2*gl*s_jd in slot N+1
template <int N> struct PtRowX { static const int value = (N + 3) & ~1; };

struct PtTaylorDev {
    const double* svt;     // [s_tot][ROWT] rows sorted by the sign of the weight: positive block (padded to even), negative block
    long long s_pos;       // rows of the positive block (even)
    long long s_tot;       // all rows (even)
    const double* dirtab;  // [2^N][s_tot] direction sums T_j(mask) of the sorted rows (null: no direction-table variant)
};

// Rows grouped by direction (pt_taylor_classify / scatter kernels): lattice edges move along diff = h * 1_mask, so the
// first log-derivative of a term is u_j = pdu + h * T_j(mask) -- ONE FMA per pair instead of N once a block's rows share
// the mask (T_j comes in with the tile).  glist holds the row indices class by class, every class padded to a whole block
// with 0xFFFFFFFF; bmask[b] is block b's mask.
struct PtTaylorGroup {
    const uint32_t* glist;
    const uint8_t* bmask;
};

// tile (+ look-ahead row) | 2^x table | running totals of the Q+1 moments | fp32 stash of the positive block's even moments |
// barrier parameters.  (The absolute moments MA_k / k! of the tail live in the tile's space once the pass is over.)
#define PT_TAYLOR_TILE_D(ROWS, Q) ((PT_TAYLOR_TILE + 1) * (ROWS) > ((Q) / 2) * PT_TAYLOR_THREADS ? (PT_TAYLOR_TILE + 1) * (ROWS) : ((Q) / 2) * PT_TAYLOR_THREADS)
#define PT_TAYLOR_SMEM_ROWS(ROWS, Q) ((size_t)(PT_TAYLOR_TILE_D(ROWS, Q) + PT_EXP_TAB + ((Q) + 1 + ((Q) + 3) / 4) * PT_TAYLOR_THREADS + 2 + 2 * PT_NMAX) * sizeof(double))
#define PT_TAYLOR_SMEM(N, Q) PT_TAYLOR_SMEM_ROWS(PtRowT<N>::value, Q)
#define PT_TAYLOR_SMEM_DIR(N, Q) PT_TAYLOR_SMEM_ROWS(PtRowX<N>::value, Q)

// pack the sign-sorted rows: dest index from an exclusive scan of the "weight >= 0" flags (stable, deterministic)
__global__ void pt_taylor_flag_kernel(const double* __restrict__ weights, long long S, unsigned* __restrict__ flag) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < S) flag[j] = weights[j] >= 0.0 ? 1u : 0u;
}

__global__ void pt_taylor_pack_kernel(const double* __restrict__ support, const double* __restrict__ weights, long long S, int n,
                                      int row, double gl, const unsigned* __restrict__ flag, const unsigned* __restrict__ rank,
                                      long long s_pos_pad, long long s_tot_pad, double* __restrict__ svt) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s_tot_pad) return;
    if (j < S) {
        const long long dst = flag[j] ? (long long)rank[j] : s_pos_pad + (j - (long long)rank[j]);
        double s2 = 0.0;
        for (int d = 0; d < n; ++d) {
            const double v = support[j * n + d];
            svt[dst * row + d] = (2.0 * gl) * v;
            s2 = fma(v, v, s2);
        }
        // log2|w| folded into the constant of the exponent: the term is 2^(c' + c_p + q.s') = |w| k(q, s)
        svt[dst * row + n] = fma(-gl, s2, log2(fabs(weights[j])));
        for (int d = n + 1; d < row; ++d) svt[dst * row + d] = 0.0;
    }
    // pad rows (at most one per block): exponent -inf, i.e. a zero term
    const long long n_pos = (long long)rank[S - 1] + (long long)flag[S - 1];
    const long long n_neg = S - n_pos;
    long long pad = -1;
    if (j == 0 && (n_pos & 1)) pad = n_pos;
    if (j == 1 && (n_neg & 1)) pad = s_pos_pad + n_neg;
    if (pad >= 0) {
        for (int d = 0; d < row; ++d) svt[pad * row + d] = 0.0;
        svt[pad * row + n] = -1.0 / 0.0;
    }
}

// one (edge, support row) pair: exponent, exponential, first log-derivative, and the Q+1 moment updates.
// `sx` = 0 in the positive block, 0x80000000 in the negative one (the sign of the weight, applied by an integer XOR).
template <int N, int Q>
__device__ __forceinline__ void pt_taylor_pair(const double* __restrict__ row, const PtPoint64<N>& pp, double pdu,
                                               const double (&ddu)[N], const double* __restrict__ tab, int sx, double (&acc)[Q + 1]) {
    double arg = row[N] + pp.cp, u = pdu;
#pragma unroll
    for (int d = 0; d < N; ++d) { arg = fma(pp.q[d], row[d], arg); u = fma(ddu[d], row[d], u); }
    const double ea = pt_exp2_neg(arg, tab);
    double pw = __hiloint2double(__double2hiint(ea) ^ sx, __double2loint(ea));
    const double u2 = u * u, u3 = u2 * u, u4 = u2 * u2;
#pragma unroll
    for (int k = 0; k < Q; k += 4) {
        acc[k] += pw;
        acc[k + 1] = fma(pw, u, acc[k + 1]);
        acc[k + 2] = fma(pw, u2, acc[k + 2]);
        acc[k + 3] = fma(pw, u3, acc[k + 3]);
        pw *= u4;
    }
    acc[Q] += fabs(pw);
}

// front half of a pair: the term e = |w| k(q(1/2), s) (sign applied) and its first log-derivative u
template <int N, bool DIR>
__device__ __forceinline__ void pt_taylor_front(const double* __restrict__ row, const PtPoint64<N>& pp, double pdu,
                                                const double (&ddu)[N], const double* __restrict__ tab, int sx, double& e, double& u) {
    if (DIR) {
        // ddu[0] = h*ln2: the common step of the moving coordinates; row[N + 1] = T_j(mask)
        double arg = row[N] + pp.cp;
        u = fma(ddu[0], row[N + 1], pdu);
#pragma unroll
        for (int d = 0; d < N; ++d) arg = fma(pp.q[d], row[d], arg);
        const double ea = pt_exp2_neg(arg, tab);
        e = __hiloint2double(__double2hiint(ea) ^ sx, __double2loint(ea));
        return;
    }
#ifdef PT_TAYLOR_TREE
    // two half-length chains per dot product (one extra add each, half the dependent depth)
    double arg = row[N] + pp.cp, arg2 = pp.q[N - 1] * row[N - 1], u2_ = ddu[N - 1] * row[N - 1];
    u = pdu;
#pragma unroll
    for (int d = 0; d < (N - 1) / 2; ++d) { arg = fma(pp.q[d], row[d], arg); u = fma(ddu[d], row[d], u); }
#pragma unroll
    for (int d = (N - 1) / 2; d < N - 1; ++d) { arg2 = fma(pp.q[d], row[d], arg2); u2_ = fma(ddu[d], row[d], u2_); }
    arg += arg2; u += u2_;
#else
    double arg = row[N] + pp.cp;
    u = pdu;
#pragma unroll
    for (int d = 0; d < N; ++d) { arg = fma(pp.q[d], row[d], arg); u = fma(ddu[d], row[d], u); }
#endif
    const double ea = pt_exp2_neg(arg, tab);
    e = __hiloint2double(__double2hiint(ea) ^ sx, __double2loint(ea));
}

// back half: the Q+1 moment updates
template <int Q>
__device__ __forceinline__ void pt_taylor_back(double pw, double u, double (&acc)[Q + 1]) {
    const double u2 = u * u, u3 = u2 * u, u4 = u2 * u2;
#ifdef PT_TAYLOR_POWPAR
    // powers of u^4 by squaring (they only need u, not the exponential): every group's base power is then ONE multiply
    // away from e, and all Q+1 updates are independent of each other
    static_assert(Q == 20 || Q == 16 || Q == 12, "power table written out for Q in {12, 16, 20}");
    const double u8 = u4 * u4, u12 = u8 * u4, u16 = u8 * u8, u20 = u16 * u4;
    const double pk[6] = {1.0, u4, u8, u12, u16, u20};
#pragma unroll
    for (int k = 0; k < Q; k += 4) {
        const double b = k ? pw * pk[k / 4] : pw;
        acc[k] += b;
        acc[k + 1] = fma(b, u, acc[k + 1]);
        acc[k + 2] = fma(b, u2, acc[k + 2]);
        acc[k + 3] = fma(b, u3, acc[k + 3]);
    }
    acc[Q] += fabs(pw * pk[Q / 4]);
#else
    static_assert((Q & 1) == 0, "an even number of moments");
#pragma unroll
    for (int k = 0; k + 4 <= Q; k += 4) {
        acc[k] += pw;
        acc[k + 1] = fma(pw, u, acc[k + 1]);
        acc[k + 2] = fma(pw, u2, acc[k + 2]);
        acc[k + 3] = fma(pw, u3, acc[k + 3]);
        pw *= u4;
    }
    if (Q % 4 == 2) {
        acc[Q - 2] += pw;
        acc[Q - 1] = fma(pw, u, acc[Q - 1]);
        pw *= u2;
    }
    acc[Q] += fabs(pw);
#endif
}

// Software-pipelined over the support rows: the (serial) exponent / exponential chain of row j+1 is issued next to the
// (parallel) moment updates of row j.  The tile carries one zero pad row behind the last one for the final look-ahead.
template <int N, int Q, bool DIR, int G>
__device__ __forceinline__ void pt_taylor_block(const double* __restrict__ svt, const double* __restrict__ dir, long long r0, long long r1,
                                                double* tile, const double* tab, const PtPoint64<N>& pp, double pdu,
                                                const double (&ddu)[N], int sx, double (&acc)[Q + 1], double* total) {
    constexpr int ROWG = PtRowT<N>::value;                               // row in global memory
    constexpr int ROW = DIR ? PtRowX<N>::value : PtRowT<N>::value;       // row in the tile
    for (long long t0 = r0; t0 < r1; t0 += PT_TAYLOR_TILE) {
        const long long rem = r1 - t0;
        const int cnt = rem < PT_TAYLOR_TILE ? (int)rem : PT_TAYLOR_TILE;     // even by construction
        __syncthreads();
        const double2* src = reinterpret_cast<const double2*>(svt + t0 * ROWG);
        double2* dst = reinterpret_cast<double2*>(tile);
        if (!DIR) {
            for (int i = threadIdx.x; i < cnt * ROWG / 2; i += PT_TAYLOR_THREADS) dst[i] = src[i];
        } else {
            for (int i = threadIdx.x; i < cnt * ROWG / 2; i += PT_TAYLOR_THREADS) {
                const int r = i / (ROWG / 2), c = i - r * (ROWG / 2);
                double2 v = src[i];
                if ((N & 1) == 0 && c == ROWG / 2 - 1) v.y = dir[t0 + r];      // even N: T_j takes the packed row's pad slot
                dst[r * (ROW / 2) + c] = v;
            }
            if (N & 1)                                                          // odd N: slot N+1 lies behind the packed row
                for (int r = threadIdx.x; r < cnt; r += PT_TAYLOR_THREADS) tile[r * ROW + N + 1] = dir[t0 + r];
        }
        if (threadIdx.x < ROW) tile[cnt * ROW + threadIdx.x] = 0.0;
        __syncthreads();
        // G lanes share an edge (small batches: the per-edge loop over the support set is the launch's latency): lane g of
        // the group takes an even-sized share [j0, j1) of every tile
        int j0 = 0, j1 = cnt;
        if (G > 1) {
            const int per = ((cnt + G - 1) / G + 1) & ~1;
            j0 = (int)(threadIdx.x % G) * per; if (j0 > cnt) j0 = cnt;
            j1 = j0 + per < cnt ? j0 + per : cnt;
        }
        double e0, u0, e1, u1;
        pt_taylor_front<N, DIR>(tile + j0 * ROW, pp, pdu, ddu, tab, sx, e0, u0);
#pragma unroll 1
        for (int j = j0; j < j1; j += 2) {
            pt_taylor_front<N, DIR>(tile + (j + 1) * ROW, pp, pdu, ddu, tab, sx, e1, u1);
            pt_taylor_back<Q>(e0, u0, acc);
            pt_taylor_front<N, DIR>(tile + (j + 2) * ROW, pp, pdu, ddu, tab, sx, e0, u0);
            pt_taylor_back<Q>(e1, u1, acc);
        }
        // blocked accumulation: a tile's partial sums go to the running totals in shared memory, so the summation error is
        // (PT_TAYLOR_TILE + S / PT_TAYLOR_TILE) u instead of S u
#pragma unroll
        for (int k = 0; k <= Q; ++k) { total[k * PT_TAYLOR_THREADS] += acc[k]; acc[k] = 0.0; }
    }
}

// ---- per-row tail: small non-inlined helpers with rolled loops (the tail is executed divergently, a few thousand
// instructions per row; kept compact so that it stays in the instruction cache next to the hot loop) -----------------

// p(tau) = sum_{k<Q} c_k tau^k, p'(tau) and exp(c tau^2); coefficients in a shared-memory column (stride PT_TAYLOR_THREADS)
template <int Q>
__device__ __noinline__ void pt_taylor_model(const double* col, double c, double tau, double* p_out, double* dp_out, double* ex_out) {
    double p = col[(Q - 1) * PT_TAYLOR_THREADS], dp = 0.0;
#pragma unroll 1
    for (int k = Q - 2; k >= 0; --k) { dp = fma(dp, tau, p); p = fma(p, tau, col[k * PT_TAYLOR_THREADS]); }
    *p_out = p; *dp_out = dp; *ex_out = exp(c * tau * tau);
}

// 2 * [ sum_{k even < Q} ca_k tau^k + fac * ca_Q tau^Q ]  >=  sum_j e_j exp(|u_j tau|)
template <int Q>
__device__ __noinline__ double pt_taylor_cosh(const double* cola, double caQ_fac, double tau) {
    const double t2 = tau * tau;
    double s = caQ_fac;
#pragma unroll 1
    for (int k = Q / 2 - 1; k >= 0; --k) s = fma(s, t2, cola[k * PT_TAYLOR_THREADS]);
    return 2.002 * s;
}

__device__ __noinline__ double pt_powi(double x, int k) {
    double r = 1.0;
    while (k) { if (k & 1) r *= x; x *= x; k >>= 1; }
    return r;
}

// log1p(e) for e in (0, 1]: seven terms of the series below 2^-8 (truncation 2^-59 relative), the library above
__device__ __forceinline__ double pt_log1p_unit(double e) {
    if (e < 0.00390625)
        return e * fma(e, fma(e, fma(e, fma(e, fma(e, fma(e, 1.0 / 7.0, -1.0 / 6.0), 0.2), -0.25), 1.0 / 3.0), -0.5), 1.0);
    return log1p(e);
}

// barrier(q(t)) and (deriv != 0) its first two t-derivatives along q(t) = a + t*diff; bp = {scale, gain, lo[n], hi[n]} in
// shared memory, geo = per-thread {a[n], diff[n]}, tab = the 2^x table of the pass.  Per term one table-based exponential
// (relative error <= (2 + |x|) u: the argument is rescaled to base 2), a short series or log1p, and a division only when the
// derivatives are wanted -- a few ulps of every term plus |x| u of the (then tiny) far ones, inside the `bulp` u |B| the
// bounds allow for it (bulp >= 64 grows with the largest |x| on the edge, pt_taylor_barrier_max).
// `moving` = bit mask of the coordinates that change along the edge; `acc0` = the (t-independent) sum of the softplus
// terms of the others (pt_taylor_barrier_const).
__device__ __noinline__ void pt_taylor_barrier(const double* bp, const double* tab, const double* geo, int n, unsigned moving,
                                               double acc0, double t, int deriv, double* B, double* B1, double* B2) {
    const double sc = bp[0], gain = bp[1];
    double acc = acc0, b1 = 0.0, b2 = 0.0;
#pragma unroll 1
    for (int i = 0; i < 2 * n; ++i) {
        const int d = i >> 1;
        if (!((moving >> d) & 1u)) continue;
        const double q = __dadd_rn(geo[d], __dmul_rn(t, geo[n + d]));
        const double x = (i & 1) ? (q - bp[2 + n + d]) / sc : (bp[2 + d] - q) / sc;      // hi side / lo side
        const double e = pt_exp2_neg(-fabs(x) * PT_L2E, tab);
        acc += fmax(x, 0.0) + pt_log1p_unit(e);
        if (deriv) {
            const double sg = (x > 0.0 ? 1.0 : e) / (1.0 + e);                            // sigmoid(x)
            const double dq = (i & 1) ? geo[n + d] : -geo[n + d];                         // d x / d t * scale
            b1 = fma(dq, sg, b1);
            b2 = fma(dq * dq, sg * (1.0 - sg), b2);
        }
    }
    *B = gain * sc * acc; *B1 = gain * b1; *B2 = gain / sc * b2;
}

// softplus terms of the coordinates that do NOT move along the edge (evaluated once per row)
__device__ __noinline__ double pt_taylor_barrier_const(const double* bp, const double* tab, const double* geo, int n, unsigned moving) {
    const double sc = bp[0];
    double acc = 0.0;
#pragma unroll 1
    for (int i = 0; i < 2 * n; ++i) {
        const int d = i >> 1;
        if ((moving >> d) & 1u) continue;
        const double x = (i & 1) ? (geo[d] - bp[2 + n + d]) / sc : (bp[2 + d] - geo[d]) / sc;
        acc += fmax(x, 0.0) + pt_log1p_unit(pt_exp2_neg(-fabs(x) * PT_L2E, tab));
    }
    return acc;
}

// upper bound of the barrier anywhere on the edge: softplus(x) <= exp(x), each coordinate at its worst end; *xabs = the
// largest |x| of any term anywhere on the edge
__device__ __noinline__ double pt_taylor_barrier_max(const double* bp, const double* geo, int n, double* xabs) {
    const double sc = bp[0], gain = bp[1];
    double acc = 0.0, xa = 0.0;
#pragma unroll 1
    for (int d = 0; d < n; ++d) {
        const double q0 = geo[d], q1 = geo[d] + geo[n + d];
        const double xl = (bp[2 + d] - fmin(q0, q1)) / sc, xh = (fmax(q0, q1) - bp[2 + n + d]) / sc;
        acc += (xl > 0.0 ? xl + 0.6931471805599453 : exp(xl)) + (xh > 0.0 ? xh + 0.6931471805599453 : exp(xh));
        xa = fmax(xa, fmax(fmax(fabs(xl), fabs(xh)), fmax(fabs((bp[2 + d] - fmax(q0, q1)) / sc), fabs((fmin(q0, q1) - bp[2 + n + d]) / sc))));
    }
    *xabs = xa;
    return 1.0001 * gain * sc * acc;
}

// model centre of the first pass: the edge midpoint, or the hinted root position snapped to a multiple of 2^-10 inside
// [1/16, 15/16] (dyadic, so tau = t - centre stays exact for every dyadic t of the bisection)
__device__ __forceinline__ double pt_taylor_centre(const float* hint, size_t ei) {
    if (!hint) return 0.5;
    const double h = (double)hint[ei];
    if (!(h > 0.0 && h < 1.0)) return 0.5;                  // NaN / out of range: no information
    const double c = rint(h * 1024.0) * (1.0 / 1024.0);
    return fmin(fmax(c, 0.0625), 0.9375);
}

// common step of the moving coordinates (the first one's) and the largest deviation of any coordinate's step from the
// direction model diff = h * 1_mask; the deviation (roundings of the two end points, ~1e-16) enters the error bound
template <int N>
__device__ __forceinline__ double pt_taylor_step(const double (&diff)[N], unsigned mask, double& dev) {
    double h = 0.0;
#pragma unroll
    for (int d = N - 1; d >= 0; --d) if ((mask >> d) & 1u) h = diff[d];
    dev = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) dev = fmax(dev, fabs(diff[d] - (((mask >> d) & 1u) ? h : 0.0)));
    return h;
}

// direction sums of the sorted rows: dirtab[mask][j] = sum_{d in mask} svt[j][d]   (2^n x s_tot doubles, L2-resident)
__global__ void pt_taylor_dirtab_kernel(const double* __restrict__ svt, int row, int n, long long s_tot, double* __restrict__ dirtab) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned mask = blockIdx.y;
    if (j >= s_tot) return;
    double t = 0.0;
    for (int d = 0; d < n; ++d) if ((mask >> d) & 1u) t += svt[j * row + d];
    dirtab[(size_t)mask * (size_t)s_tot + j] = t;
}

// ---- grouping of a batch's rows by direction ------------------------------------------------------------------------
// class of a row = the mask of its moving coordinates when all of them move by the same step (to 1e-12 relative: lattice
// edges, whose end points are rounded separately), 0 otherwise (arbitrary segments keep the N-term dot product).
#define PT_TAYLOR_CLS_THREADS 256
template <int N>
__global__ void __launch_bounds__(PT_TAYLOR_CLS_THREADS)
pt_taylor_classify_kernel(const double* __restrict__ a_, const double* __restrict__ b_, size_t m, uint8_t* __restrict__ cls,
                          unsigned* __restrict__ hist) {
    __shared__ unsigned sh[1 << N];
    for (int i = threadIdx.x; i < (1 << N); i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        double diff[N];
        unsigned mask = 0;
#pragma unroll
        for (int d = 0; d < N; ++d) { diff[d] = __dsub_rn(b_[i * N + d], a_[i * N + d]); mask |= (diff[d] != 0.0 ? 1u : 0u) << d; }
        double dev;
        const double h = pt_taylor_step<N>(diff, mask, dev);
        if (!(dev <= 1e-12 * fabs(h))) mask = 0;            // (NaN steps land here too)
        cls[i] = (uint8_t)mask;
        atomicAdd(&sh[mask], 1u);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < (1 << N); c += blockDim.x) if (sh[c]) atomicAdd(&hist[c], sh[c]);
}

struct PtTaylorOffsets { unsigned off[1 << PT_NMAX]; };     // first slot of every class in glist (block-aligned for mask != 0)

// rows to their class's run of glist; the order inside a class does not matter (every row is solved on its own)
template <int N>
__global__ void __launch_bounds__(PT_TAYLOR_CLS_THREADS)
pt_taylor_scatter_kernel(const uint8_t* __restrict__ cls, size_t m, PtTaylorOffsets offs, unsigned* __restrict__ cursor,
                         uint32_t* __restrict__ glist) {
    __shared__ unsigned cnt[1 << N], base[1 << N];
    for (int i = threadIdx.x; i < (1 << N); i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned c = 0, local = 0;
    if (i < m) { c = cls[i]; local = atomicAdd(&cnt[c], 1u); }
    __syncthreads();
    for (int k = threadIdx.x; k < (1 << N); k += blockDim.x) if (cnt[k]) base[k] = atomicAdd(&cursor[k], cnt[k]);
    __syncthreads();
    if (i < m) glist[(size_t)offs.off[c] + base[c] + local] = (uint32_t)i;
}

// block -> mask of the grouped launch: blocks [off[c]/TH, off[c+1]/TH) belong to class c (classes in ascending order from 1)
__global__ void pt_taylor_bmask_kernel(PtTaylorOffsets offs, int ncls, unsigned first_slot, size_t nblocks, uint8_t* __restrict__ bmask) {
    const size_t b = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const unsigned slot = first_slot + (unsigned)b * PT_TAYLOR_THREADS;
    int c = 1;
    while (c + 1 < ncls && offs.off[c + 1] <= slot) ++c;
    bmask[b] = (uint8_t)c;
}

template <int N, int Q, bool DIR, int G = 1>
__global__ void __launch_bounds__(PT_TAYLOR_THREADS, DIR ? PT_TAYLOR_MINB_DIR : PT_TAYLOR_MINB)
pt_bisect_taylor_kernel(PtFieldDev f, double sum_abs_w, PtTaylorDev tf, PtRows rows, PtTaylorGroup grp, const double* __restrict__ a_,
                        const double* __restrict__ b_, const int8_t* __restrict__ signs_a, double eps, double* __restrict__ out,
                        double* __restrict__ lo_io, double* __restrict__ hi_io, uint8_t* __restrict__ slow, double* __restrict__ jlo_out,
                        double* __restrict__ jhi_out, unsigned long long* work, int recentre, const float* __restrict__ hint) {
    constexpr int ROW = DIR ? PtRowX<N>::value : PtRowT<N>::value, TH = PT_TAYLOR_THREADS;
    extern __shared__ double sm[];
    double* tile = sm;
    double* tab = tile + PT_TAYLOR_TILE_D(ROW, Q);
    double* col = tab + PT_EXP_TAB + threadIdx.x;          // c_k at col[k*TH], k < Q;  RQ-independent
    float* stash = reinterpret_cast<float*>(tab + PT_EXP_TAB + (Q + 1) * TH) + threadIdx.x;   // even moments of the positive block
    double* cola = tile + threadIdx.x;                     // ca_k (k even < Q) at cola[(k/2)*TH]: the tile's space, after the pass
    pt_exp_table_init(tab);
    if (threadIdx.x < 2 + 2 * N) {
        double* bpw = tab + PT_EXP_TAB + (Q + 1 + (Q + 3) / 4) * TH;
        bpw[threadIdx.x] = threadIdx.x == 0 ? f.b_scale : threadIdx.x == 1 ? f.b_gain
                         : threadIdx.x < 2 + N ? f.b_lo[threadIdx.x - 2] : f.b_hi[threadIdx.x - 2 - N];
    }
    // first pass: all rows, model about the edge midpoint, bracket [0, 1].  Second pass (`recentre`): the listed rows the
    // first one left open, model about the midpoint of the bracket they stopped at -- the truncation then scales with
    // (bracket width / 2)^Q instead of 2^-Q
    static_assert(G == 1 || !DIR, "shared rows only in the generic kernel");
    constexpr int RPB = TH / G;                                // rows per block: G adjacent lanes share one
    const size_t m = DIR ? (size_t)gridDim.x * TH : pt_rows_total(rows);
    if ((size_t)blockIdx.x * RPB >= m) return;
    size_t ei = (size_t)blockIdx.x * RPB + threadIdx.x / G;
    bool valid = ei < m;
    unsigned mask = 0;
    if (DIR) {
        // grouped rows: the block's rows share the direction mask; 0xFFFFFFFF pads a class to a whole block
        ei = grp.glist[ei];
        valid = ei != 0xFFFFFFFFull;
        mask = grp.bmask[blockIdx.x];
    } else if (valid && rows.list) ei = rows.list[ei];
    const double* dir = DIR ? tf.dirtab + (size_t)mask * (size_t)tf.s_tot : nullptr;
    // (row geometry is loaded twice -- here for the pass, again for the tail -- so that nothing but the pass's own
    //  operands stays live across the support loop: at 96 registers every extra live value spills INSIDE that loop)
    double mnorm2 = 0.0;
    {
        double a[N], diff[N], L = 0.0, H = 1.0;
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; }
        if (valid) {
            double b[N];
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
            pt_segment<N>(a, b, diff);
            if (recentre) { L = lo_io[ei]; H = hi_io[ei]; }
        }
        const double tc = recentre ? 0.5 * (L + H) : pt_taylor_centre(valid ? hint : nullptr, ei);
        // ---- the pass over the support set: moments about the model centre ------------------------------------------
        PtPoint64<N> pp;
        double mc[N], ddu[N], md = 0.0;
#pragma unroll
        for (int d = 0; d < N; ++d) {
            mc[d] = fma(tc, diff[d], a[d]);
            md = fma(mc[d], diff[d], md);
            ddu[d] = diff[d] * PT_LN2;                     // rows hold 2*gamma*log2e*s_d
            mnorm2 = fma(mc[d], mc[d], mnorm2);
        }
        if (DIR) { double dev; ddu[0] = pt_taylor_step<N>(diff, mask, dev) * PT_LN2; }
        pp.set(mc, f.gamma * PT_L2E);
        const double pdu = -2.0 * f.gamma * md;
        double acc[Q + 1];
#pragma unroll
        for (int k = 0; k <= Q; ++k) { acc[k] = 0.0; col[k * TH] = 0.0; }
        pt_taylor_block<N, Q, DIR, G>(tf.svt, dir, 0, tf.s_pos, tile, tab, pp, pdu, ddu, 0, acc, col);
        // even moments of the positive block, rounded up to fp32: they only enter error bounds (MA_k = 2 M_k^+ - M_k)
#pragma unroll
        for (int k = 0; k < Q; k += 2) {
            double v = col[k * TH];
            if (G > 1) for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);     // the group's lanes' shares
            stash[(k / 2) * TH] = __double2float_ru(v * (G > 1 ? 1.0 + 1e-15 : 1.0));
        }
        pt_taylor_block<N, Q, DIR, G>(tf.svt, dir, tf.s_pos, tf.s_tot, tile, tab, pp, pdu, ddu, (int)0x80000000, acc, col);
        if (G > 1) {
#pragma unroll
            for (int k = 0; k <= Q; ++k) {
                double v = col[k * TH];
                for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                col[k * TH] = v;
            }
        }
        __syncthreads();                                   // the last tile is dead: its space takes the absolute moments
        double inv_fact = 1.0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            if (k > 1) inv_fact /= (double)k;
            const double mk = col[k * TH];
            col[k * TH] = (mk + pp.poison) * inv_fact;
            // MA_k / k! (fp32 stash: relative 1.2e-7, inside the 2.002 of pt_taylor_cosh; the max keeps MA_k >= |M_k|)
            if ((k & 1) == 0) cola[(k / 2) * TH] = fmax(fabs(2.0 * (double)stash[(k / 2) * TH] - mk), fabs(mk)) * inv_fact;
        }
        col[Q * TH] = col[Q * TH] * (inv_fact / (double)Q);                 // MA_Q / Q!
    }
    if (DIR && !recentre) {
        const int nvalid = __syncthreads_count(valid ? 1 : 0);
        if (threadIdx.x == 0) atomicAdd(&work[7], (unsigned long long)nvalid);
    }
    if (G > 1) {
        // shared rows: the tails of the block's RPB rows go to its first RPB threads (whole warps, not every G-th lane); thread
        // r reads the coefficient columns the group of row r left behind (all G lanes of a group hold the same totals)
        __syncthreads();
        if (threadIdx.x >= RPB) return;
        ei = (size_t)blockIdx.x * RPB + threadIdx.x;
        valid = ei < m;
        if (valid && rows.list) ei = rows.list[ei];
        col = tab + PT_EXP_TAB + threadIdx.x * G;
        cola = tile + threadIdx.x * G;
    }
    if (!valid) return;
    double a[N], diff[N];
    double L = 0.0, H = 1.0, seg;
    {
        double b[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = PT_TAYLOR_LDCS(&a_[ei * N + d]); b[d] = PT_TAYLOR_LDCS(&b_[ei * N + d]); }   // last use
        seg = pt_segment<N>(a, b, diff);
    }
    const int sa = signs_a[ei];
    if (recentre) { L = lo_io[ei]; H = hi_io[ei]; }
    const double tc = recentre ? 0.5 * (L + H) : pt_taylor_centre(hint, ei);     // model centre (dyadic)
    if (G > 1) {
        mnorm2 = 0.0;                                                            // (the pass computed it for another row)
#pragma unroll
        for (int d = 0; d < N; ++d) { const double mcd = fma(tc, diff[d], a[d]); mnorm2 = fma(mcd, mcd, mnorm2); }
    }
    const double hr = fmax(tc - L, H - tc);                                      // |tau| <= hr on the bracket
    const double seg2 = seg * seg;

    // ---- per-row constants of the bounds --------------------------------------------------------------------------
    const double c = -f.gamma * seg2;
    const double ac = fabs(c);
    const double mn = sqrt(mnorm2);
    const double pn = mn + f.smax + hr * seg;
    const double T = f.gamma * PT_L2E * pn * pn;
    const double gmaxu = 2.0 * f.gamma * seg * (mn + f.smax);
    // Remainder of exp(u_j tau) after Q terms: <= |u_j tau|^Q / Q! / (1 - |u_j tau| / (Q+1)).  Support vectors with
    // |u_j| hr <= X = 0.8 (Q+1) get the factor 5 (all of them, when the crude bound gmaxu says so: then the exact factor).
    // The others are at least r_X = X / (2 gamma seg hr) away from the model centre, so each of their terms -- exact or
    // truncated -- is below |w_j| exp(-gamma r_X (r_X - 2 seg hr)) anywhere on the bracket: they are charged in full (Efar).
    const double xmax = hr * gmaxu, X = 0.8 * (double)(Q + 1);
    const double fac = xmax <= X ? 1.0 / (1.0 - xmax / (double)(Q + 1)) : 5.0;
    double Efar = 0.0;
    if (xmax > X) {
        const double segh = seg * hr, rX = X / (2.0 * f.gamma * segh);
        Efar = rX > 2.0 * segh ? 2.002 * sum_abs_w * exp(-f.gamma * rX * (rX - 2.0 * segh)) : 1e300;
    }
    const bool model_ok = Efar < 1e290;
    const double caQ = col[Q * TH];
    const double ca0 = cola[0];
    const double RQ = fac * (1.01 * caQ + 1e-40 * ca0);                     // |R(tau)| <= RQ |tau|^Q
    // rounding of THIS pass relative to sum_j e_j exp(|u_j tau|): expanded exponent (cancellation at scale T), blocked
    // summation, powers and Horner, the log-derivative's absolute error
    // (direction-table variant: u_j = pdu + h T_j instead of the N-term dot product -- T_j's own rounding, and the
    //  deviation of the true steps from h * 1_mask times 2 gamma |s_j| sqrt(N), an absolute error of the log-derivative)
    double Cdir = 0.0;
    if (DIR) {
        double dev;
        pt_taylor_step<N>(diff, mask, dev);
        Cdir = 1.01 * 2.0 * f.gamma * f.smax * sqrt((double)N) * dev;
    }
    const double Ctot = PT_U64 * (1.01 * (double)(4 * N + 7) * T * PT_LN2 + 1.05 * (double)(PT_TAYLOR_TILE + f.S / PT_TAYLOR_TILE)
                                  + 4.0 * Q + (double)(DIR ? 4 * N + 2 : N + 2) * gmaxu + 450.0) + Cdir;
    const double abias = fabs(f.bias);
    const double* bp = tab + PT_EXP_TAB + (Q + 1 + (Q + 3) / 4) * TH;              // barrier parameters (shared)
    double geo[2 * N];                                                      // dynamically indexed by the helpers
#pragma unroll
    for (int d = 0; d < N; ++d) { geo[d] = a[d]; geo[N + d] = diff[d]; }
    unsigned moving = 0;
#pragma unroll
    for (int d = 0; d < N; ++d) moving |= (diff[d] != 0.0 ? 1u : 0u) << d;
    // the barrier terms of the resting coordinates: once per row, by all lanes together (every enclosure attempt needs them)
    const double bconst_v = f.has_barrier ? pt_taylor_barrier_const(bp, tab, geo, N, moving) : 0.0;
    auto bconst = [&]() { return bconst_v; };
    double bulp = 64.0;                                                     // allowance, in ulps of |B|, for the barrier's evaluation
    double bsum = 0.0, Bmax = 0.0;                                          // |B'| <= bsum, 0 <= B <= Bmax on the edge
    if (f.has_barrier) {
#pragma unroll
        for (int d = 0; d < N; ++d) bsum += fabs(diff[d]);
        bsum *= f.b_gain;
        double xabs;
        Bmax = pt_taylor_barrier_max(bp, geo, N, &xabs);
        bulp = fmax(64.0, 16.0 + 2.0 * xabs);
    }

    int flag = 1;                 // 0 done, 1 no enclosure, 2 enclosed with open midpoints
    double Jlo = -1e300, Jhi = 1e300;
    double D2max = -1.0;
    if (model_ok) {
#pragma unroll 1
        for (;;) {
            if (!(__dmul_rn(seg, __dsub_rn(H, L)) > eps)) { flag = 0; break; }
            const double mq = __dmul_rn(0.5, __dadd_rn(L, H));
            const double tau = mq - tc;
            const double at = fabs(tau);
            double p, dp, ex, B = 0.0, B1 = 0.0, B2 = 0.0;
            pt_taylor_model<Q>(col, c, tau, &p, &dp, &ex);
            const double Ach = pt_taylor_cosh<Q>(cola, fac * caQ, at);
            const double Etr = ex * RQ * pt_powi(at, Q), Ern = ex * Ctot * Ach;      // truncation / rounding of the model
            const double Ek = 1.001 * (Etr + Ern) + Efar + 1e-290;
            const double g0 = fma(ex, p, f.bias);
            // the barrier is only evaluated when the decision needs it (0 <= B <= Bmax)
            const double Eb0 = bulp * PT_U64 * (1.1 * Bmax + abias);
            int sgn = 0;
            if (g0 - Bmax > Ek + Eb0) sgn = 1;
            else if (g0 < -(Ek + Eb0)) sgn = -1;
            else {
                if (f.has_barrier) pt_taylor_barrier(bp, tab, geo, N, moving, bconst(), mq, 0, &B, &B1, &B2);
                const double g = g0 - B;
                if (fabs(g) > Ek + bulp * PT_U64 * (1.1 * fabs(B) + abias)) sgn = g > 0.0 ? 1 : -1;
                // |F| is below the rounding level of any fp64 evaluation (this model's truncation is smaller still): the
                // model value is as good as an evaluation, its sign is taken
                else if (Etr + Efar <= Ern && g == g) sgn = g > 0.0 ? 1 : -1;
            }
            if (sgn == 0) break;                                          // undecided: keep [L, H]
            if (sgn == sa) L = mq; else H = mq;
            const double w = H - L;
            if (!(w <= PT_TAYLOR_TRY_WIDTH)) continue;
            if (!(__dmul_rn(seg, w) > eps)) continue;
            // ---- enclosure attempt on [L, H] ------------------------------------------------------------------------
            if (D2max < 0.0) {
                // |F''| anywhere on the edge: polynomial part by absolute coefficients, remainder, rounding, barrier
                double pm0 = 0.0, pm1 = 0.0, pm2 = 0.0;
                double hk = 1.0, hm = 0.0, hn = 0.0;                  // hr^k, hr^(k-1), hr^(k-2)  (0 where the power is negative)
#pragma unroll 1
                for (int k = 0; k < Q; ++k) {
                    const double ck = fabs(col[k * TH]);
                    pm0 = fma(ck, hk, pm0);
                    pm1 = fma(ck * (double)k, hm, pm1);
                    pm2 = fma(ck * (double)(k * (k - 1)), hn, pm2);
                    hn = hm; hm = hk; hk *= hr;
                    if (k == 0) hn = 0.0;
                }
                // now hk = hr^Q, hm = hr^(Q-1), hn = hr^(Q-2)
                const double r0 = RQ * hk, r1 = RQ * (double)Q * hm, r2 = RQ * (double)(Q * (Q - 1)) * hn;
                const double Ah = pt_taylor_cosh<Q>(cola, fac * caQ, hr);
                double b2 = 0.0;
                if (f.has_barrier) {
#pragma unroll
                    for (int d = 0; d < N; ++d) b2 = fma(diff[d], diff[d], b2);
                    b2 *= 0.5 * f.b_gain / f.b_scale;
                }
                // (e^{c tau^2} p)'' = e^{c tau^2} [p'' + 4 c tau p' + (2 c + 4 c^2 tau^2) p],  |tau| <= hr <= 1
                D2max = 1.01 * ((pm2 + r2) + 4.0 * ac * hr * (pm1 + r1) + (2.0 * ac + 4.0 * ac * ac * hr * hr) * (pm0 + r0)
                                + 2.0 * Ctot * (gmaxu * gmaxu + 4.0 * ac * hr * (gmaxu + 1.0) + 4.0 * ac * ac * hr * hr + 2.0 * ac) * Ah
                                + (gmaxu * gmaxu + 4.0 * ac * hr * gmaxu + 4.0 * ac * ac * hr * hr + 2.0 * ac) * Efar + b2);
            }
            const double tmax = fmax(fabs(L - tc), fabs(H - tc));
            const double Amax = pt_taylor_cosh<Q>(cola, fac * caQ, tmax);
            const double ptq1 = pt_powi(tmax, Q - 1);
            // |F' - model'| anywhere in the bracket
            const double Ed = 1.01 * (RQ * (double)Q * ptq1 + 2.0 * ac * tmax * RQ * ptq1 * tmax
                                      + 1.5 * Ctot * (gmaxu + 2.0 * ac * tmax + 1.0) * Amax + (gmaxu + 2.0 * ac * tmax) * Efar);
            const double xm = 0.5 * (L + H);
            double Bm = 0.0, B1m = 0.0, B2m = 0.0;
            pt_taylor_model<Q>(col, c, xm - tc, &p, &dp, &ex);
            if (f.has_barrier) pt_taylor_barrier(bp, tab, geo, N, moving, bconst(), xm, 1, &Bm, &B1m, &B2m);
            double gv = fma(ex, p, f.bias) - Bm;
            double gd = ex * fma(2.0 * c * (xm - tc), p, dp) - B1m;
            const double EdB = Ed + bulp * PT_U64 * (fabs(gd) + bsum);
            const double smin = fabs(gd) - EdB - 0.5 * w * D2max;
            if (!(smin > 0.0)) continue;                                  // not provably monotone yet: next level
            // Newton on the model inside (L, H), the barrier replaced by its quadratic expansion about the bracket
            // midpoint (exact values come back in below)
            double x = xm;
#pragma unroll 1
            for (int it = 0; it < 7; ++it) {
                double xn = x - gv / gd;
                if (!(xn > L && xn < H)) xn = 0.5 * (xn > x ? x + H : x + L);
                const bool conv = fabs(xn - x) <= 1e-13;
                x = xn;
                const double sft = x - xm;
                pt_taylor_model<Q>(col, c, x - tc, &p, &dp, &ex);
                gv = fma(ex, p, f.bias) - fma(sft, fma(0.5 * B2m, sft, B1m), Bm);
                gd = ex * fma(2.0 * c * (x - tc), p, dp) - fma(B2m, sft, B1m);
                if (conv) break;
            }
            // exact barrier at the surrogate root and one corrected Newton step; the residual after that step is bounded, not
            // evaluated: |G(x - G/G')| <= |G''|/2 (G/G')^2
            double Bx = 0.0, B1x = 0.0, B2x = 0.0;
            if (f.has_barrier) {
                pt_taylor_barrier(bp, tab, geo, N, moving, bconst(), x, 1, &Bx, &B1x, &B2x);
                gv = fma(ex, p, f.bias) - Bx;
                gd = ex * fma(2.0 * c * (x - tc), p, dp) - B1x;
                const double step = gv / gd, xn = x - step;
                if (xn > L && xn < H) {
                    x = xn;
                    gv = 0.505 * D2max * step * step;
                    gd = fmax(fabs(gd) - fabs(step) * D2max, 0.0);         // |model'| at the new x, from below
                }
            }
            const double agd = fabs(gd);
            const double Eb = bulp * PT_U64 * (1.1 * (fabs(Bx) + w * bsum) + abias) + 1e-290;
            const double tx = fabs(x - tc);
            const double Ex = 1.001 * ex * (RQ * pt_powi(tx, Q) + Ctot * pt_taylor_cosh<Q>(cola, fac * caQ, tx)) + Efar + Eb;
            const double rho0 = (fabs(gv) + Ex) / smin;                    // |x - root| <= rho0
            double sloc = agd - EdB - rho0 * D2max;                        // |F'| on [x - rho0, x + rho0]
            if (!(sloc > smin)) sloc = smin;
            const double rho = 1.01 * (fabs(gv) + Ex) / sloc + 4e-16;
            // F is monotone on [L, H] and its root lies in J: every midpoint outside J has a certain sign
            Jlo = x - rho; Jhi = x + rho;
            bool open = false;
            while (__dmul_rn(seg, __dsub_rn(H, L)) > eps) {
                const double mr = __dmul_rn(0.5, __dadd_rn(L, H));
                if (mr < Jlo) L = mr;
                else if (mr > Jhi) H = mr;
                else {
                    // a midpoint inside the enclosure: decide it on the model like the levels above
                    const double tr = mr - tc, atr = fabs(tr);
                    pt_taylor_model<Q>(col, c, tr, &p, &dp, &ex);
                    double Br = 0.0, B1r = 0.0, B2r = 0.0;
                    if (f.has_barrier) pt_taylor_barrier(bp, tab, geo, N, moving, bconst(), mr, 0, &Br, &B1r, &B2r);
                    const double gr = fma(ex, p, f.bias) - Br;
                    const double Etr = ex * RQ * pt_powi(atr, Q), Ern = ex * Ctot * pt_taylor_cosh<Q>(cola, fac * caQ, atr);
                    const double Er = 1.001 * (Etr + Ern) + Efar + bulp * PT_U64 * (1.1 * fabs(Br) + abias) + 1e-290;
                    if (fabs(gr) > Er || (Etr + Efar <= Ern && gr == gr)) { if ((gr > 0.0 ? 1 : -1) == sa) L = mr; else H = mr; }
                    else { open = true; break; }
                }
            }
            flag = open ? 2 : 0;
            break;
        }
    }
    // (results are written once and read by later kernels: streaming stores, so they do not push the resident tiles, the
    //  direction table and the threads' local memory out of L2)
    slow[ei] = (uint8_t)flag;
    if (flag == 0) {
        const double tf_ = __dmul_rn(0.5, __dadd_rn(L, H));
#pragma unroll
        for (int d = 0; d < N; ++d) PT_TAYLOR_STCS(&out[ei * N + d], __dadd_rn(a[d], __dmul_rn(tf_, diff[d])));
    } else {
        lo_io[ei] = L; hi_io[ei] = H;
        jlo_out[ei] = flag == 2 ? Jlo : -1e300;
        jhi_out[ei] = flag == 2 ? Jhi : 1e300;
    }
    if (recentre && flag != 0) atomicAdd(&work[3], 1ull);                 // rows left to the evaluation-based kernels
    if (!DIR && threadIdx.x == 0 && !recentre) {
        const size_t first = (size_t)blockIdx.x * RPB;
        atomicAdd(&work[7], (unsigned long long)(m - first < (size_t)RPB ? m - first : (size_t)RPB));
    }
}
