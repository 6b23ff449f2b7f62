// Tensor-core (tcgen05 / TMEM) version of the fp32 bisection screen.
//
// The exponent of every (point, support vector) pair,
//     arg_ij = -gamma*log2(e)*|p_i - s_j|^2 = c_s(j) + c_p(i) + q_i . s_j ,   q = 2*gamma*log2(e)*p ,
// is a [128 points] x [S support vectors] x [K] contraction.  It runs on the 5th-generation tensor cores as
// kind::tf32 UMMA instructions (M = 128, N = 128, K = 8) with the fp32 accumulator in tensor memory.  TF32
// carries 11 significant bits, so both operands are split into tf32 pieces (x = x_h + x_l, residual <= 2^-24|x|)
// and the contraction is widened to K = 3n + 6 columns
//     q_h.s_h + c_p,h*1 + 1*c_s,h  |  q_h.s_l + c_p,l*1 + 1*c_s,l  |  q_l.s_h + c_p,ll*1 + 1*c_s,ll
// (every product of two 11-bit pieces is exact in fp32; the dropped q_l.s_l term and the split residuals are
// <= 3*2^-24 sum_d |q_d s_d|).  The epilogue reads the accumulator back with tcgen05.ld, one point per thread
// (TMEM lane = point, column = support vector), and does 2^arg (MUFU ex2) and the weighted fp32 sums exactly
// like the SIMT screen (pt_bisect32_kernel); the decision rule |F32| > E with E a bound on |F32 - F| is the same.
//
// Shared memory (one CTA per SM, persistent over chunks of 128 rows):
//     B  : the whole packed support set, K-major canonical no-swizzle UMMA layout, loaded once per CTA
//     A  : the 128 points of the current bisection level, rewritten by the epilogue threads every level
//     W  : the fp32 weights
// TMEM: 512 columns = four 128 x 128 fp32 accumulators (two per row group), so the MMAs of tile t+1 overlap the
// epilogue of tile t.
#pragma once
#include "pt_field.cuh"

#ifdef __CUDACC__
__device__ __forceinline__ float pt_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// x = h + l (+ ll): tf32 pieces, each exactly representable with 11 significant bits
__device__ __forceinline__ void pt_tf32_split3(double x, float& h, float& l, float& ll) {
    h = pt_tf32((float)x);
    const double r = x - (double)h;
    l = pt_tf32((float)r);
    ll = pt_tf32((float)(r - (double)l));
}

// column k of the widened contraction for the support side (see the header comment)
__global__ void pt_pack_tc_kernel(const double* __restrict__ support, const double* __restrict__ weights, long long S,
                                  int n, int spad, int kt, double gl, float* __restrict__ bt, float* __restrict__ wt) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= spad) return;
    float col[32];
    for (int k = 0; k < kt; ++k) col[k] = 0.f;
    float w = 0.f;
    if (j < S) {
        double s2 = 0.0;
        for (int d = 0; d < n; ++d) {
            const double v = support[j * n + d];
            s2 = fma(v, v, s2);
            float h, l, ll;
            pt_tf32_split3(v, h, l, ll);
            col[d] = h;                   // q_h . s_h
            col[(n + 2) + d] = l;         // q_h . s_l
            col[2 * (n + 2) + d] = h;     // q_l . s_h
        }
        float ch, cl, cll;
        pt_tf32_split3(-gl * s2, ch, cl, cll);
        col[n] = 1.f;             col[n + 1] = ch;                 // c_p,h * 1 ; 1 * c_s,h
        col[(n + 2) + n] = 1.f;   col[(n + 2) + n + 1] = cl;
        col[2 * (n + 2) + n] = 1.f; col[2 * (n + 2) + n + 1] = cll;
        w = (float)weights[j];
    }
    for (int k = 0; k < kt; ++k) bt[((size_t)(k >> 2) * spad + j) * 4 + (k & 3)] = col[k];
    wt[j] = w;
}

// 2^x on the FMA pipe (the MUFU pipe is the screen's limiter, so every fourth exponential goes here): round to
// nearest integer by the magic-number trick, degree-5 polynomial on [-1/2, 1/2] (relative error 3.7 u32 including the
// fp32 Horner rounding -- same class as ex2.approx), exponent field add.  Arguments below -125 flush to 2^-125 ~ 0.
__device__ __forceinline__ float pt_ex2_poly(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;             // 1.5 * 2^23: low mantissa bits of t hold round(x)
    const float f = x - (t - 12582912.0f);
    float p = 0.0013266970636323094f;
    p = fmaf(p, f, 0.009675459936261177f);
    p = fmaf(p, f, 0.05550742521882057f);
    p = fmaf(p, f, 0.24022121727466583f);
    p = fmaf(p, f, 0.6931469440460205f);
    p = fmaf(p, f, 1.0000001192092896f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// ---- raw PTX wrappers ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pt_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pt_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void pt_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "PT_MBAR_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra PT_MBAR_DONE;\n\t"
        "bra PT_MBAR_WAIT;\n\t"
        "PT_MBAR_DONE:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void pt_fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void pt_tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void pt_tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// K-major, no swizzle: core matrix = 8 rows x 16 bytes, contiguous (128 B); lbo = byte distance between the two
// 16-byte K halves of one instruction, sbo = byte distance between successive 8-row groups
__device__ __forceinline__ uint64_t pt_umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, issued by one thread for the whole CTA
__device__ __forceinline__ void pt_umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void pt_umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void pt_tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void pt_tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// instruction descriptor: D = f32, A = B = tf32, both K-major, N = PT_TC_N, M = 128
#define PT_TC_IDESC ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(PT_TC_N >> 3) << 17) | ((uint32_t)(PT_TC_M >> 4) << 24))

// sync / OR-reduce over the 128 threads of one row group (named barriers 1 and 2; barrier 0 stays __syncthreads)
__device__ __forceinline__ void pt_group_sync(int group) {
    asm volatile("bar.sync %0, 128;" ::"r"(group + 1) : "memory");
}
__device__ __forceinline__ bool pt_group_or(int group, bool pred) {
    uint32_t out;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 q, %1, 0;\n\t"
        "bar.red.or.pred p, %2, 128, q;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(out) : "r"((uint32_t)pred), "r"(group + 1) : "memory");
    return out != 0;
}

// box barrier in fp32 (fast exp/log): value and a bound on its error; the screen only needs F to within E
template <int N>
__device__ __forceinline__ double pt_barrier_fast(const PtFieldDev& f, const double* p, double inv_scale, double& err) {
    float acc = 0.f, mag = 0.f;
#pragma unroll
    for (int d = 0; d < N; ++d) {
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const float v = (float)((side ? (p[d] - f.b_hi[d]) : (f.b_lo[d] - p[d])) * inv_scale);
            const float t = __logf(1.f + __expf(-fabsf(v)));     // log1p(exp(-|v|)): __expf <= 4 u32 abs, 1+e 2 u32, __logf on [1,2] 2^-21.41 = 6 u32
            acc += fmaxf(v, 0.f) + t;
            mag += 1.f + fmaxf(v, 0.f);
        }
    }
    const double gs = f.b_gain * f.b_scale;
    // per term: 12 u32 (t) + u32*v (conversion) <= 13 u32 (1 + max(v,0)); the 4N fp32 additions round at u32 of a partial
    // sum <= mag each, whichever term dominates and wherever it enters the sum: (13 + 4N) u32 mag in all; 16 + 4N is used
    err = (16.0 + 4.0 * N) * PT_U32 * gs * (double)mag;
    return gs * (double)acc;
}

// MODE 3 arguments: one bisection level of the listed rows against ONE chunk [j0, j0+cs) of the support set; the
// partial sums are stored (first chunk) or added to acc[row] / ab[row].  Other modes: j0 = 0, cs = spad.
struct PtTcLevel {
    int j0, cs;
    double* acc;
    double* ab;
    int first_chunk;
};

// MODE 0: the bisection screen (same contract as pt_bisect32_kernel).
// MODE 1: calibration -- one evaluation at t = 0.5 per row; hi_io[row] receives max_j |arg_tc - arg_fp64| / (u32*T).
// MODE 2: sign evaluation at the points a_[row] (lattice vertices): sign_out[row] = +1 / -1 when |F32| > E, i.e. the
//         fp32 sign is PROVEN equal to the fp64 one, and 0 when it is not -- those rows are rechecked in fp64.
// MODE 3: level-synchronous screen for support sets larger than one CTA's shared memory (and, optionally, for all):
//         ONE evaluation at the midpoint of every listed row's current bracket against one support chunk; the
//         decision is taken by pt_screen_decide_kernel once all chunks of the level have been added.
//
// Two independent row groups per CTA (warps 0-3 and 4-7, 128 rows each, one row per thread = one TMEM lane): every
// bisection level ends in a serial stretch (decide, move the bracket, rewrite A, wait for the first MMA), and while
// one group is there the other one keeps the MUFU pipe busy.  Each group owns two 128-column accumulators.
template <int N, int MODE>
__global__ void __launch_bounds__(PT_TC_THREADS, 1)
pt_bisect32_tc_kernel(PtFieldDev f, PtTcDev tc, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                      const int8_t* __restrict__ signs_a, double eps, int fresh, double* __restrict__ lo_io,
                      double* __restrict__ hi_io, int8_t* __restrict__ sign_out, PtTcLevel lv, unsigned long long* work) {
    extern __shared__ __align__(1024) unsigned char pt_tc_smem[];
    constexpr int KT = ((3 * N + 6) + 7) & ~7;
    constexpr int KC = KT / 4;           // 16-byte K chunks
    const int spad = tc.spad;            // row stride of the packed operand in global memory
    const int cs = lv.cs;                // support rows resident in this launch
    const int ntiles = cs / PT_TC_N;
    float* sB = reinterpret_cast<float*>(pt_tc_smem);
    float* sA0 = sB + (size_t)KC * cs * 4;                      // A of group 0, then group 1
    float* sW = sA0 + 2 * (size_t)KC * PT_TC_M * 4;
    unsigned long long* sBar = reinterpret_cast<unsigned long long*>(sW + cs);
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBar + 4);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = tid & (PT_TC_M - 1), group = tid >> 7;
    const size_t total = pt_rows_total(rows);
    if ((size_t)blockIdx.x * (2 * PT_TC_M) >= total) return;

    // ---- one-time setup: barriers, TMEM, the packed support set ---------------------------------------------
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) pt_mbar_init(pt_smem_u32(&sBar[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(pt_smem_u32(sTmem)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(tc.bt);
        uint4* dst = reinterpret_cast<uint4*>(sB);
        for (int i = tid; i < KC * cs; i += PT_TC_THREADS) {
            const int c = i / cs, j = i - c * cs;
            dst[i] = src[(size_t)c * spad + lv.j0 + j];
        }
        const uint4* ws = reinterpret_cast<const uint4*>(tc.wt + lv.j0);
        uint4* wd = reinterpret_cast<uint4*>(sW);
        for (int i = tid; i < cs / 4; i += PT_TC_THREADS) wd[i] = ws[i];
    }
    pt_fence_async_smem();
    pt_tc_fence_before();
    __syncthreads();
    pt_tc_fence_after();
    const uint32_t tmem_base = *sTmem + (uint32_t)group * (2 * PT_TC_N);
    float* sA = sA0 + (size_t)group * KC * PT_TC_M * 4;
    const uint32_t sA_u32 = pt_smem_u32(sA), sB_u32 = pt_smem_u32(sB);
    const uint32_t bar_u32[2] = {pt_smem_u32(&sBar[group * 2]), pt_smem_u32(&sBar[group * 2 + 1])};
    uint32_t phase[2] = {0u, 0u};
    const double gl = f.gamma * PT_L2E;
    const double inv_scale = f.has_barrier ? 1.0 / f.b_scale : 0.0;
    const bool leader = row == 0;

    // one MMA tile: accumulator buffer `buf` <- A (128 x KT) * B[tile]^T (KT x PT_TC_N)
    auto issue_tile = [&](int tile, int buf) {
#pragma unroll
        for (int ks = 0; ks < KT / 8; ++ks) {
            const uint64_t da = pt_umma_desc(sA_u32 + (uint32_t)(2 * ks) * (PT_TC_M * 16), PT_TC_M * 16, 128);
            const uint64_t db = pt_umma_desc(sB_u32 + (uint32_t)(2 * ks) * (uint32_t)(cs * 16) + (uint32_t)tile * (PT_TC_N * 16),
                                             (uint32_t)(cs * 16), 128);
            pt_umma_tf32(tmem_base + (uint32_t)buf * PT_TC_N, da, db, PT_TC_IDESC, ks > 0 ? 1u : 0u);
        }
        pt_umma_commit(bar_u32[buf]);
    };

    for (size_t chunk = (size_t)blockIdx.x * 2 + group; chunk * PT_TC_M < total; chunk += (size_t)gridDim.x * 2) {
        const size_t idx = chunk * PT_TC_M + row;
        const bool valid = idx < total;
        const size_t ei = valid ? (rows.list ? (size_t)rows.list[idx] : idx) : 0;
        double a[N], diff[N], p[N];
        double seg = 0.0, lo = 0.0, hi = 1.0;
        int sa = 1;
        if (valid && MODE == 2) {
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; diff[d] = 0.0; }
        } else if (valid) {
            double b[N];
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
            seg = pt_segment<N>(a, b, diff);
            sa = signs_a[ei];
            if ((!fresh && MODE == 0) || MODE == 3) { lo = lo_io[ei]; hi = hi_io[ei]; }
        } else {
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = 0.0; diff[d] = 0.0; }
        }
        bool active = valid && (MODE != 0 || __dmul_rn(seg, __dsub_rn(hi, lo)) > eps);
        int8_t sign_certain = 0;
        float f32_value = 0.f;
        unsigned iters = 0;
        double calib = 0.0;
        while (pt_group_or(group, active)) {
            const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
            double p2 = 0.0;
#pragma unroll
            for (int d = 0; d < N; ++d) {
                p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d]));
                p2 = fma(p[d], p[d], p2);
            }
            {
                // this point's row of A: tf32 pieces of q = 2 gl p and of c_p = -gl |p|^2, column order as in pt_pack_tc_kernel
                float col[KT];
#pragma unroll
                for (int k = 0; k < KT; ++k) col[k] = 0.f;
#pragma unroll
                for (int d = 0; d < N; ++d) {
                    float h, l, ll;
                    pt_tf32_split3(2.0 * gl * p[d], h, l, ll);
                    col[d] = h; col[(N + 2) + d] = h; col[2 * (N + 2) + d] = l;
                }
                float ch, cl, cll;
                pt_tf32_split3(-gl * p2, ch, cl, cll);
                col[N] = ch;               col[N + 1] = 1.f;
                col[(N + 2) + N] = cl;     col[(N + 2) + N + 1] = 1.f;
                col[2 * (N + 2) + N] = cll; col[2 * (N + 2) + N + 1] = 1.f;
#pragma unroll
                for (int c = 0; c < KC; ++c)
                    *reinterpret_cast<float4*>(sA + ((size_t)c * PT_TC_M + row) * 4) =
                        make_float4(col[4 * c], col[4 * c + 1], col[4 * c + 2], col[4 * c + 3]);
            }
            pt_fence_async_smem();
            pt_group_sync(group);
            if (leader) {
                pt_tc_fence_after();
                issue_tile(0, 0);
                if (ntiles > 1) issue_tile(1, 1);
            }
            double acc = 0.0, ab = 0.0;
            const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
            for (int t = 0; t < ntiles; ++t) {
                const int buf = t & 1;
                pt_mbar_wait(bar_u32[buf], phase[buf]);
                phase[buf] ^= 1u;
                pt_tc_fence_after();
                const uint32_t taddr = tmem_base + lane_base + (uint32_t)(buf * PT_TC_N);
                const float* wrow = sW + t * PT_TC_N;
                uint32_t r0[32], r1[32];
                float fa_t[PT_TC_N / 32], fb_t[PT_TC_N / 32];
                pt_tmem_ld32(taddr, r0);
#pragma unroll
                for (int blk = 0; blk < PT_TC_N / 32; ++blk) {
                    pt_tmem_wait_ld();
                    uint32_t (&cur)[32] = (blk & 1) ? r1 : r0;
                    uint32_t (&nxt)[32] = (blk & 1) ? r0 : r1;
                    if (blk + 1 < PT_TC_N / 32) pt_tmem_ld32(taddr + (uint32_t)(blk + 1) * 32, nxt);
                    if (MODE != 1) {
                        float fa = 0.f, fb = 0.f;
#pragma unroll
                        for (int c4 = 0; c4 < 8; ++c4) {
                            const float4 w4 = *reinterpret_cast<const float4*>(wrow + blk * 32 + c4 * 4);
                            const float e0 = pt_ex2(__uint_as_float(cur[c4 * 4 + 0]));
                            const float e1 = pt_ex2(__uint_as_float(cur[c4 * 4 + 1]));
                            const float e2 = pt_ex2(__uint_as_float(cur[c4 * 4 + 2]));
                            const float e3 = pt_ex2_poly(__uint_as_float(cur[c4 * 4 + 3]));
                            fa = fmaf(w4.x, e0, fa); fb = fmaf(fabsf(w4.x), e0, fb);
                            fa = fmaf(w4.y, e1, fa); fb = fmaf(fabsf(w4.y), e1, fb);
                            fa = fmaf(w4.z, e2, fa); fb = fmaf(fabsf(w4.z), e2, fb);
                            fa = fmaf(w4.w, e3, fa); fb = fmaf(fabsf(w4.w), e3, fb);
                        }
                        fa_t[blk] = fa; fb_t[blk] = fb;        // 32-term fp32 chains
                    } else {
                        // calibration: exact exponent from the fp64 rows (row layout: 2 gl s_d, w, -gl |s|^2)
                        const int ROW = PT_ROW64(N);
                        for (int c = 0; c < 32; ++c) {
                            const long long j = (long long)lv.j0 + (long long)t * PT_TC_N + blk * 32 + c;
                            if (j < f.S) {
                                const double* srow = f.sv + j * ROW;
                                double ex = srow[N + 1] - gl * p2;
#pragma unroll
                                for (int d = 0; d < N; ++d) ex = fma(p[d], srow[d], ex);
                                calib = fmax(calib, fabs((double)__uint_as_float(cur[c]) - ex));
                            }
                        }
                    }
                }
                if (MODE != 1) {
                    // pairwise fp32 sum of the four chains (34 roundings at most), one conversion per tile
                    acc += (double)((fa_t[0] + fa_t[1]) + (fa_t[2] + fa_t[3]));
                    ab += (double)((fb_t[0] + fb_t[1]) + (fb_t[2] + fb_t[3]));
                }
                pt_tc_fence_before();
                if (t + 2 < ntiles) {
                    pt_group_sync(group);
                    if (leader) { pt_tc_fence_after(); issue_tile(t + 2, buf); }
                }
            }
            const double pn = sqrt(p2) + f.smax;
            if (MODE == 3) {
                if (valid) {
                    if (lv.first_chunk) { lv.acc[ei] = acc; lv.ab[ei] = ab; }
                    else { lv.acc[ei] += acc; lv.ab[ei] += ab; }
                }
                active = false;
            } else if (MODE == 1) {
                calib = calib / (PT_U32 * gl * pn * pn);
                active = false;
            } else {
                double F = f.bias + acc, eb = 0.0;
                if (f.has_barrier) F -= pt_barrier_fast<N>(f, p, inv_scale, eb);
                // |arg_tc - arg| <= PT_TC_ARG_ULPS u T (tf32 splits + tensor-core accumulation, calibrated);
                // ex2.approx, weight rounding, products and the 32-term fp32 chains (+2 pairwise levels) add < 80 u relative
                const double rel = 1.01 * (PT_TC_ARG_ULPS * PT_U32 * gl * pn * pn * PT_LN2) + 80.0 * PT_U32;
                const double E = 2.0 * rel * ab + eb + 1e-280;
                if (MODE == 2) {
                    // + amb_tol: a vertex within the ambiguity band of zero always reaches the fp64 kernel, which counts it
                    if (active && fabs(F) > E + f.amb_tol) sign_certain = F > 0.0 ? (int8_t)1 : (int8_t)-1;
                    if (active) f32_value = (float)F;
                    active = false;
                } else if (active) {
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
        }
        if (MODE == 0) {
            unsigned mine = iters;
            for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
            if ((tid & 31) == 0 && mine) atomicAdd(&work[2], (unsigned long long)mine);
            if (valid) { lo_io[ei] = lo; hi_io[ei] = hi; }
        } else if (MODE == 1) {
            if (valid) hi_io[ei] = calib;
        } else if (MODE == 2) {
            if (valid) sign_out[ei] = sign_certain;
            // MODE 2 has no brackets: hi_io, when given, receives the fp32 field VALUES (as floats) -- the refinement keeps
            // them per fine vertex as a secant hint for the root solve's model centre
            if (valid && hi_io) reinterpret_cast<float*>(hi_io)[ei] = f32_value;
        }
    }
    pt_tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*sTmem), "r"(512u));
}

// ---- four row groups per CTA (n = 6) ---------------------------------------------------------------------------
// Same screen with FOUR independent 128-row groups per CTA (16 warps, four per SM sub-partition instead of two), so that
// the serial stretches of a group (level boundary, waiting for its MMA) are covered by three others.  What makes it fit:
//   * shared memory: the K = 24 operand of n = 6 has an exact duplicate 16-byte chunk (columns 16..19 = s_h[0..3] =
//     columns 0..3), so B is stored as 5 chunks instead of 6 (160 KB at S = 2048) and the third k-step's descriptor
//     simply points at chunk 0 with a leading-byte offset that reaches chunk 4;
//   * TMEM: one 128-column accumulator per group (4 x 128 = 512 columns); the MMA of a group's next tile is issued when
//     the group has drained the current one -- the wait is hidden by the other groups;
//   * registers (128 per thread): the segment endpoints are re-read from L2 at every level instead of living in
//     registers, and the accumulator is read through one 32-register window.
#define PT_TC4_THREADS 512
static_assert(PT_TC_N == 128, "the four-group kernel assumes 128-column tiles");

__global__ void __launch_bounds__(PT_TC4_THREADS, 1)
pt_bisect32_tc4_kernel(PtFieldDev f, PtTcDev tc, PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_,
                       const int8_t* __restrict__ signs_a, double eps, int fresh, double* __restrict__ lo_io,
                       double* __restrict__ hi_io, unsigned long long* work) {
    constexpr int N = 6, KT = 24, KC = 6, BC = 5;     // BC: distinct B chunks
    extern __shared__ __align__(1024) unsigned char pt_tc_smem[];
    const int spad = tc.spad;
    const int ntiles = spad / PT_TC_N;
    float* sB = reinterpret_cast<float*>(pt_tc_smem);
    float* sA0 = sB + (size_t)BC * spad * 4;
    float* sW = sA0 + 4 * (size_t)KC * PT_TC_M * 4;
    unsigned long long* sBar = reinterpret_cast<unsigned long long*>(sW + spad);
    uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBar + 4);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = tid & (PT_TC_M - 1), group = tid >> 7;
    const size_t total = pt_rows_total(rows);
    if ((size_t)blockIdx.x * (4 * PT_TC_M) >= total) return;

    if (tid == 0) {
        for (int i = 0; i < 4; ++i) pt_mbar_init(pt_smem_u32(&sBar[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(pt_smem_u32(sTmem)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(tc.bt);
        uint4* dst = reinterpret_cast<uint4*>(sB);
        for (int i = tid; i < BC * spad; i += PT_TC4_THREADS) {
            const int c = i / spad, j = i - c * spad;
            dst[i] = src[(size_t)(c < 4 ? c : 5) * spad + j];          // global chunk 4 duplicates chunk 0
        }
        const uint4* ws = reinterpret_cast<const uint4*>(tc.wt);
        uint4* wd = reinterpret_cast<uint4*>(sW);
        for (int i = tid; i < spad / 4; i += PT_TC4_THREADS) wd[i] = ws[i];
    }
    pt_fence_async_smem();
    pt_tc_fence_before();
    __syncthreads();
    pt_tc_fence_after();
    const uint32_t tmem_base = *sTmem + (uint32_t)group * PT_TC_N;
    float* sA = sA0 + (size_t)group * KC * PT_TC_M * 4;
    const uint32_t sA_u32 = pt_smem_u32(sA), sB_u32 = pt_smem_u32(sB);
    const uint32_t bar_u32 = pt_smem_u32(&sBar[group]);
    uint32_t phase = 0u;
    const double gl = f.gamma * PT_L2E;
    const double inv_scale = f.has_barrier ? 1.0 / f.b_scale : 0.0;
    const bool leader = row == 0;
    const uint32_t chunk_bytes = (uint32_t)spad * 16u;

    auto issue_tile = [&](int tile) {
        const uint32_t tb = sB_u32 + (uint32_t)tile * (PT_TC_N * 16);
        // k-step 0: chunks (0, 1); k-step 1: chunks (2, 3); k-step 2: chunks (0, 4) -- chunk 0 doubles as columns 16..19
        pt_umma_tf32(tmem_base, pt_umma_desc(sA_u32, PT_TC_M * 16, 128), pt_umma_desc(tb, chunk_bytes, 128), PT_TC_IDESC, 0u);
        pt_umma_tf32(tmem_base, pt_umma_desc(sA_u32 + 2 * (PT_TC_M * 16), PT_TC_M * 16, 128),
                     pt_umma_desc(tb + 2 * chunk_bytes, chunk_bytes, 128), PT_TC_IDESC, 1u);
        pt_umma_tf32(tmem_base, pt_umma_desc(sA_u32 + 4 * (PT_TC_M * 16), PT_TC_M * 16, 128),
                     pt_umma_desc(tb, 4 * chunk_bytes, 128), PT_TC_IDESC, 1u);
        pt_umma_commit(bar_u32);
    };

    for (size_t chunk = (size_t)blockIdx.x * 4 + group; chunk * PT_TC_M < total; chunk += (size_t)gridDim.x * 4) {
        const size_t idx = chunk * PT_TC_M + row;
        const bool valid = idx < total;
        const size_t ei = valid ? (rows.list ? (size_t)rows.list[idx] : idx) : 0;
        double seg = 0.0, lo = 0.0, hi = 1.0;
        int sa = 1;
        if (valid) {
            double a[N], b[N], diff[N];
#pragma unroll
            for (int d = 0; d < N; ++d) { a[d] = a_[ei * N + d]; b[d] = b_[ei * N + d]; }
            seg = pt_segment<N>(a, b, diff);
            sa = signs_a[ei];
            if (!fresh) { lo = lo_io[ei]; hi = hi_io[ei]; }
        }
        bool active = valid && __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
        unsigned iters = 0;
        while (pt_group_or(group, active)) {
            const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
            double p2 = 0.0;
            {
                // this point's row of A (endpoints re-read from L2: they must not live in registers across the epilogue)
                float col[KT];
#pragma unroll
                for (int k = 0; k < KT; ++k) col[k] = 0.f;
#pragma unroll
                for (int d = 0; d < N; ++d) {
                    const double av = valid ? a_[ei * N + d] : 0.0, bv = valid ? b_[ei * N + d] : 0.0;
                    const double pd = __dadd_rn(av, __dmul_rn(mid, __dsub_rn(bv, av)));
                    p2 = fma(pd, pd, p2);
                    float h, l, ll;
                    pt_tf32_split3(2.0 * gl * pd, h, l, ll);
                    col[d] = h; col[(N + 2) + d] = h; col[2 * (N + 2) + d] = l;
                }
                float ch, cl, cll;
                pt_tf32_split3(-gl * p2, ch, cl, cll);
                col[N] = ch;               col[N + 1] = 1.f;
                col[(N + 2) + N] = cl;     col[(N + 2) + N + 1] = 1.f;
                col[2 * (N + 2) + N] = cll; col[2 * (N + 2) + N + 1] = 1.f;
#pragma unroll
                for (int c = 0; c < KC; ++c)
                    *reinterpret_cast<float4*>(sA + ((size_t)c * PT_TC_M + row) * 4) =
                        make_float4(col[4 * c], col[4 * c + 1], col[4 * c + 2], col[4 * c + 3]);
            }
            pt_fence_async_smem();
            pt_group_sync(group);
            if (leader) { pt_tc_fence_after(); issue_tile(0); }
            double acc = 0.0, ab = 0.0;
            const uint32_t taddr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
            for (int t = 0; t < ntiles; ++t) {
                pt_mbar_wait(bar_u32, phase);
                phase ^= 1u;
                pt_tc_fence_after();
                const float* wrow = sW + t * PT_TC_N;
                float fa_t[4], fb_t[4];
#pragma unroll
                for (int blk = 0; blk < 4; ++blk) {
                    uint32_t cur[32];
                    pt_tmem_ld32(taddr + (uint32_t)blk * 32, cur);
                    pt_tmem_wait_ld();
                    float fa = 0.f, fb = 0.f;
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(wrow + blk * 32 + c4 * 4);
                        const float e0 = pt_ex2(__uint_as_float(cur[c4 * 4 + 0]));
                        const float e1 = pt_ex2(__uint_as_float(cur[c4 * 4 + 1]));
                        const float e2 = pt_ex2(__uint_as_float(cur[c4 * 4 + 2]));
                        const float e3 = pt_ex2_poly(__uint_as_float(cur[c4 * 4 + 3]));
                        fa = fmaf(w4.x, e0, fa); fb = fmaf(fabsf(w4.x), e0, fb);
                        fa = fmaf(w4.y, e1, fa); fb = fmaf(fabsf(w4.y), e1, fb);
                        fa = fmaf(w4.z, e2, fa); fb = fmaf(fabsf(w4.z), e2, fb);
                        fa = fmaf(w4.w, e3, fa); fb = fmaf(fabsf(w4.w), e3, fb);
                    }
                    fa_t[blk] = fa; fb_t[blk] = fb;
                }
                acc += (double)((fa_t[0] + fa_t[1]) + (fa_t[2] + fa_t[3]));
                ab += (double)((fb_t[0] + fb_t[1]) + (fb_t[2] + fb_t[3]));
                pt_tc_fence_before();
                if (t + 1 < ntiles) {
                    pt_group_sync(group);
                    if (leader) { pt_tc_fence_after(); issue_tile(t + 1); }
                }
            }
            // decision (the midpoint is recomputed from the endpoints)
            double p[N];
            p2 = 0.0;
#pragma unroll
            for (int d = 0; d < N; ++d) {
                const double av = valid ? a_[ei * N + d] : 0.0, bv = valid ? b_[ei * N + d] : 0.0;
                p[d] = __dadd_rn(av, __dmul_rn(mid, __dsub_rn(bv, av)));
                p2 = fma(p[d], p[d], p2);
            }
            const double pn = sqrt(p2) + f.smax;
            double F = f.bias + acc, eb = 0.0;
            if (f.has_barrier) F -= pt_barrier_fast<N>(f, p, inv_scale, eb);
            const double rel = 1.01 * (PT_TC_ARG_ULPS * PT_U32 * gl * pn * pn * PT_LN2) + 80.0 * PT_U32;
            const double E = 2.0 * rel * ab + eb + 1e-280;
            if (active) {
                if (fabs(F) > E) {
                    if ((F > 0.0 ? 1 : -1) == sa) lo = mid; else hi = mid;
                    ++iters;
                    const double w = __dsub_rn(hi, lo);
                    active = __dmul_rn(seg, w) > eps && w > PT_FP32_STOP_WIDTH;
                } else {
                    active = false;
                }
            }
        }
        unsigned mine = iters;
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        if ((tid & 31) == 0 && mine) atomicAdd(&work[2], (unsigned long long)mine);
        if (valid) { lo_io[ei] = lo; hi_io[ei] = hi; }
    }
    pt_tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*sTmem), "r"(512u));
}

// ---- level-synchronous driver kernels (MODE 3) ------------------------------------------------------------------
// rows of `rows` whose bracket still needs a step -> list_out (fresh: brackets start at [0, 1])
template <int N>
__global__ void pt_screen_filter_kernel(PtRows rows, const double* __restrict__ a_, const double* __restrict__ b_, double eps,
                                        int fresh, double* __restrict__ lo_io, double* __restrict__ hi_io,
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
        double lo = 0.0, hi = 1.0;
        if (fresh) { lo_io[ei] = lo; hi_io[ei] = hi; } else { lo = lo_io[ei]; hi = hi_io[ei]; }
        take = __dmul_rn(seg, __dsub_rn(hi, lo)) > eps;
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

// the decision of one level: F32 = bias + acc - barrier against E; certain -> move the bracket, still active -> list_out
template <int N>
__global__ void pt_screen_decide_kernel(PtFieldDev f, const uint32_t* __restrict__ list_in, const unsigned long long* count_in,
                                        const double* __restrict__ a_, const double* __restrict__ b_,
                                        const int8_t* __restrict__ signs_a, double eps, double* __restrict__ lo_io,
                                        double* __restrict__ hi_io, const double* __restrict__ acc_, const double* __restrict__ ab_,
                                        uint32_t* __restrict__ list_out, unsigned long long* count_out, unsigned long long* work) {
    const size_t total = (size_t)*count_in;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool active = false; uint32_t ei = 0; unsigned stepped = 0;
    if (idx < total) {
        ei = list_in[idx];
        double a[N], b[N], diff[N], p[N];
#pragma unroll
        for (int d = 0; d < N; ++d) { a[d] = a_[(size_t)ei * N + d]; b[d] = b_[(size_t)ei * N + d]; }
        const double seg = pt_segment<N>(a, b, diff);
        double lo = lo_io[ei], hi = hi_io[ei];
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
        double p2 = 0.0;
#pragma unroll
        for (int d = 0; d < N; ++d) { p[d] = __dadd_rn(a[d], __dmul_rn(mid, diff[d])); p2 = fma(p[d], p[d], p2); }
        const double gl = f.gamma * PT_L2E;
        const double pn = sqrt(p2) + f.smax;
        double F = f.bias + acc_[ei], eb = 0.0;
        if (f.has_barrier) F -= pt_barrier_fast<N>(f, p, 1.0 / f.b_scale, eb);
        const double rel = 1.01 * (PT_TC_ARG_ULPS * PT_U32 * gl * pn * pn * PT_LN2) + 80.0 * PT_U32;
        const double E = 2.0 * rel * ab_[ei] + eb + 1e-280;
        if (fabs(F) > E) {
            if ((F > 0.0 ? 1 : -1) == signs_a[ei]) { lo = mid; lo_io[ei] = mid; } else { hi = mid; hi_io[ei] = mid; }
            stepped = 1;
            const double w = __dsub_rn(hi, lo);
            active = __dmul_rn(seg, w) > eps && w > PT_FP32_STOP_WIDTH;
        }
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, active);
    const unsigned sb = __ballot_sync(0xffffffffu, stepped != 0);
    const int lane = threadIdx.x & 31;
    if (lane == 0 && sb) atomicAdd(&work[2], (unsigned long long)__popc(sb));
    if (ballot) {
        const int leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(count_out, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (active) list_out[base + __popc(ballot & ((1u << lane) - 1u))] = ei;
    }
}
#endif
