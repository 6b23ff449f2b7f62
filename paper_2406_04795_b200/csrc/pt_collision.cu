// Fused forward kinematics + sphere-vs-{box, cylinder, sphere} tests, one thread per configuration,
// robot chain and scene primitives staged in shared memory.
//   fk_batch                collision.py:204-225   (serial chain, Rodrigues per revolute joint :191-201)
//   Pose.to_local           collision.py:83-84     local = (c - t) @ R
//   sphere_box_hits         _kernels.pyx:43-76     octant fold, prune, 3 edge regions, vertex region
//   sphere_cylinder_hits    _kernels.pyx:79-104
//   sphere_sphere_hits      _kernels.pyx:107-122   touching counts
//   batch_check/_batch_hits collision.py:278-329 ; _not_free_checker pipeline.py:256-270
#include <stdlib.h>
#include <math.h>
#include "pt_internal.cuh"

#define PT_MAX_JOINTS 16

// flat double layout of the model in device memory / shared memory
//   joint j  (PT_JSTRIDE doubles): kind, axis[3], rot[9], trans[3], lim_lo, lim_hi
//   sphere s (PT_SSTRIDE doubles): link, off[3], radius
//   obst  o  (PT_OSTRIDE doubles): type, rot[9], trans[3], dims[3]
#define PT_JSTRIDE 18
#define PT_SSTRIDE 5
#define PT_OSTRIDE 16

struct pt_checker {
    pt_ctx* ctx = nullptr;
    int nj = 0, ns = 0, no = 0;
    PtBuf<double> model;       // joints | spheres (sorted by link) | obstacles
    std::vector<int> sphere_order;   // position in link-sorted order -> original sphere index
    PtBuf<int> sphere_orig;    // same, on device (for fk output ordering)
    size_t model_doubles = 0;
    // fp32 screen (pt_check32_kernel): bound on |gap32 - gap| for every (sphere, obstacle) pair of this model; 0 = off
    float gap_margin = 0.f;
};

__device__ __forceinline__ bool pt_hit_box(double cx, double cy, double cz, double r, double lx, double ly, double lz) {
    const double hx = 0.5 * lx, hy = 0.5 * ly, hz = 0.5 * lz;
    const double px = fabs(cx), py = fabs(cy), pz = fabs(cz);
    const double dx = __dsub_rn(px, hx), dy = __dsub_rn(py, hy), dz = __dsub_rn(pz, hz);
    if (dx > r || dy > r || dz > r) return false;
    const double r2 = __dmul_rn(r, r);
    const double dx2 = __dmul_rn(dx, dx), dy2 = __dmul_rn(dy, dy), dz2 = __dmul_rn(dz, dz);
    if (px <= hx && dy > 0 && dz > 0 && __dadd_rn(dy2, dz2) > r2) return false;
    if (py <= hy && dx > 0 && dz > 0 && __dadd_rn(dx2, dz2) > r2) return false;
    if (pz <= hz && dx > 0 && dy > 0 && __dadd_rn(dx2, dy2) > r2) return false;
    if (dx > 0 && dy > 0 && dz > 0 && __dadd_rn(__dadd_rn(dx2, dy2), dz2) > r2) return false;
    return true;
}
__device__ __forceinline__ bool pt_hit_cylinder(double cx, double cy, double cz, double r, double height, double radius) {
    const double hh = 0.5 * height;
    const double pz = fabs(cz);
    const double rad = sqrt(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)));
    const double dz = __dsub_rn(pz, hh), dr = __dsub_rn(rad, radius);
    if (dz > r || dr > r) return false;
    if (dz > 0 && dr > 0 && __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dz, dz)) > __dmul_rn(r, r)) return false;
    return true;
}
__device__ __forceinline__ bool pt_hit_sphere(double cx, double cy, double cz, double r, double radius) {
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz));
    const double rr = __dadd_rn(r, radius);
    return d2 <= __dmul_rn(rr, rr);
}

__global__ void pt_sphere_box_kernel(const double* __restrict__ c, const double* __restrict__ r, size_t m,
                                     double lx, double ly, double lz, uint8_t* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = pt_hit_box(c[3 * i], c[3 * i + 1], c[3 * i + 2], r[i], lx, ly, lz) ? 1 : 0;
}
__global__ void pt_sphere_cyl_kernel(const double* __restrict__ c, const double* __restrict__ r, size_t m,
                                     double height, double radius, uint8_t* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = pt_hit_cylinder(c[3 * i], c[3 * i + 1], c[3 * i + 2], r[i], height, radius) ? 1 : 0;
}
__global__ void pt_sphere_sph_kernel(const double* __restrict__ c, const double* __restrict__ r, size_t m,
                                     double radius, uint8_t* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = pt_hit_sphere(c[3 * i], c[3 * i + 1], c[3 * i + 2], r[i], radius) ? 1 : 0;
}

// y = R x (row-major R), separately rounded products summed left to right
__device__ __forceinline__ void pt_matvec(const double* R, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        y[i] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * i], x[0]), __dmul_rn(R[3 * i + 1], x[1])), __dmul_rn(R[3 * i + 2], x[2]));
}
__device__ __forceinline__ void pt_matmul(const double* A, const double* B, double* C) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            C[3 * i + k] = __dadd_rn(__dadd_rn(__dmul_rn(A[3 * i], B[k]), __dmul_rn(A[3 * i + 1], B[3 + k])), __dmul_rn(A[3 * i + 2], B[6 + k]));
}

// advance the frame through joint j (collision.py:213-220)
__device__ __forceinline__ void pt_fk_step(const double* J, double q, double* R, double* t) {
    double v[3], Rn[9];
    pt_matvec(R, J + 13, v);                       // rot @ origin.translation
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] = __dadd_rn(v[i], t[i]);
    pt_matmul(R, J + 4, Rn);                       // rot @ origin.rotation
    if (J[0] == 0.0) {                             // revolute: Rodrigues
        const double kx = J[1], ky = J[2], kz = J[3];
        double s, c;
        sincos(q, &s, &c);
        const double omc = __dsub_rn(1.0, c);
        double A[9];
        // c*I + s*skew + (1-c)*outer(k,k), summed in that order
        const double skew[9] = {0.0, -kz, ky, kz, 0.0, -kx, -ky, kx, 0.0};
        const double k[3] = {kx, ky, kz};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
                const double ident = (i == jj) ? 1.0 : 0.0;
                A[3 * i + jj] = __dadd_rn(__dadd_rn(__dmul_rn(c, ident), __dmul_rn(s, skew[3 * i + jj])),
                                          __dmul_rn(omc, __dmul_rn(k[i], k[jj])));
            }
        pt_matmul(Rn, A, R);
    } else {                                       // prismatic: trans += (rot @ axis) * q
#pragma unroll
        for (int i = 0; i < 9; ++i) R[i] = Rn[i];
        pt_matvec(R, J + 1, v);
#pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = __dadd_rn(t[i], __dmul_rn(v[i], q));
    }
}

__device__ __forceinline__ bool pt_sphere_vs_scene(const double* obs, int no, const double* c, double radius) {
    for (int o = 0; o < no; ++o) {
        const double* O = obs + o * PT_OSTRIDE;
        const double dx = __dsub_rn(c[0], O[10]), dy = __dsub_rn(c[1], O[11]), dz = __dsub_rn(c[2], O[12]);
        // (c - t) @ R : local_k = sum_i d_i R[i][k]
        const double lx = __dadd_rn(__dadd_rn(__dmul_rn(dx, O[1]), __dmul_rn(dy, O[4])), __dmul_rn(dz, O[7]));
        const double ly = __dadd_rn(__dadd_rn(__dmul_rn(dx, O[2]), __dmul_rn(dy, O[5])), __dmul_rn(dz, O[8]));
        const double lz = __dadd_rn(__dadd_rn(__dmul_rn(dx, O[3]), __dmul_rn(dy, O[6])), __dmul_rn(dz, O[9]));
        const int type = (int)O[0];
        bool hit;
        if (type == 0) hit = pt_hit_box(lx, ly, lz, radius, O[13], O[14], O[15]);
        else if (type == 1) hit = pt_hit_cylinder(lx, ly, lz, radius, O[13], O[14]);
        else hit = pt_hit_sphere(lx, ly, lz, radius, O[13]);
        if (hit) return true;
    }
    return false;
}

// ---- fp32 screen ------------------------------------------------------------------------------------------
// The same walk in fp32: FK, obstacle-frame transform and the signed gap (distance to the primitive minus the sphere
// radius; the reference's branch tests are exactly "gap <= 0") of every (sphere, obstacle) pair.  With `margin` a
// bound on |gap32 - gap|, gap32 < -margin is a certain hit and gap32 > margin a certain miss; a configuration with an
// undecided pair (and no certain hit) is marked 2 and decided by the fp64 kernel.
__device__ __forceinline__ float pt_gap_box32(float cx, float cy, float cz, float r, float lx, float ly, float lz) {
    const float dx = fabsf(cx) - 0.5f * lx, dy = fabsf(cy) - 0.5f * ly, dz = fabsf(cz) - 0.5f * lz;
    const float ox = fmaxf(dx, 0.f), oy = fmaxf(dy, 0.f), oz = fmaxf(dz, 0.f);
    const float outside = sqrtf(ox * ox + oy * oy + oz * oz);
    const float inside = fminf(fmaxf(dx, fmaxf(dy, dz)), 0.f);
    return outside + inside - r;
}
__device__ __forceinline__ float pt_gap_cylinder32(float cx, float cy, float cz, float r, float height, float radius) {
    const float dz = fabsf(cz) - 0.5f * height, dr = sqrtf(cx * cx + cy * cy) - radius;
    const float oz = fmaxf(dz, 0.f), orr = fmaxf(dr, 0.f);
    return sqrtf(oz * oz + orr * orr) + fminf(fmaxf(dz, dr), 0.f) - r;
}

__global__ void __launch_bounds__(128)
pt_check32_kernel(const double* __restrict__ model, int nj, int ns, int no, const double* __restrict__ q_, size_t m,
                  int mode, float margin, uint8_t* __restrict__ out) {
    extern __shared__ __align__(16) float smf[];
    // joints and spheres as in the fp64 layout; every obstacle repacked into four float4 (one LDS.128 each):
    //   (R00, R10, R20, tx) (R01, R11, R21, ty) (R02, R12, R22, tz) (dim0, dim1, dim2, type)
    const int head = nj * PT_JSTRIDE + ns * PT_SSTRIDE;
    const int head4 = (head + 3) & ~3;
    for (int i = threadIdx.x; i < head; i += blockDim.x) smf[i] = (float)model[i];
    float4* OB4 = reinterpret_cast<float4*>(smf + head4);
    for (int i = threadIdx.x; i < no * 4; i += blockDim.x) {
        const double* O = model + head + (i >> 2) * PT_OSTRIDE;
        const int part = i & 3;
        OB4[i] = part < 3 ? make_float4((float)O[1 + part], (float)O[4 + part], (float)O[7 + part], (float)O[10 + part])
                          : make_float4((float)O[13], (float)O[14], (float)O[15], (float)O[0]);
    }
    __syncthreads();
    const float* J = smf;
    const float* SP = smf + nj * PT_JSTRIDE;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float q[PT_MAX_JOINTS];
    bool inside = true;
    for (int j = 0; j < nj; ++j) {
        const double qd = q_[i * nj + j];
        // the limit test stays exact: compare the fp64 value with the fp64 limits
        inside = inside && (qd >= model[j * PT_JSTRIDE + 16]) && (qd <= model[j * PT_JSTRIDE + 17]);
        q[j] = (float)qd;
    }
    if (mode != PT_LIMIT_IGNORE && !inside) { out[i] = 1; return; }
    float R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    float t[3] = {0, 0, 0};
    int sp = 0;
    bool hit = false, undecided = false;
    for (int link = 0; link <= nj && !hit; ++link) {
        if (link > 0) {
            const float* Jp = J + (link - 1) * PT_JSTRIDE;
            float Rn[9];
#pragma unroll
            for (int a = 0; a < 3; ++a) t[a] += R[3 * a] * Jp[13] + R[3 * a + 1] * Jp[14] + R[3 * a + 2] * Jp[15];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int k = 0; k < 3; ++k) Rn[3 * a + k] = R[3 * a] * Jp[4 + k] + R[3 * a + 1] * Jp[7 + k] + R[3 * a + 2] * Jp[10 + k];
            if (Jp[0] == 0.f) {
                const float kx = Jp[1], ky = Jp[2], kz = Jp[3];
                float sn, cs;
                sincosf(q[link - 1], &sn, &cs);
                const float omc = 1.f - cs;
                const float A[9] = {cs + omc * kx * kx, -sn * kz + omc * kx * ky, sn * ky + omc * kx * kz,
                                    sn * kz + omc * ky * kx, cs + omc * ky * ky, -sn * kx + omc * ky * kz,
                                    -sn * ky + omc * kz * kx, sn * kx + omc * kz * ky, cs + omc * kz * kz};
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int k = 0; k < 3; ++k) R[3 * a + k] = Rn[3 * a] * A[k] + Rn[3 * a + 1] * A[3 + k] + Rn[3 * a + 2] * A[6 + k];
            } else {
#pragma unroll
                for (int a = 0; a < 9; ++a) R[a] = Rn[a];
#pragma unroll
                for (int a = 0; a < 3; ++a) t[a] += (R[3 * a] * Jp[1] + R[3 * a + 1] * Jp[2] + R[3 * a + 2] * Jp[3]) * q[link - 1];
            }
        }
        while (sp < ns && (int)SP[sp * PT_SSTRIDE] == link && !hit) {
            const float* S = SP + sp * PT_SSTRIDE;
            const float cx = R[0] * S[1] + R[1] * S[2] + R[2] * S[3] + t[0];
            const float cy = R[3] * S[1] + R[4] * S[2] + R[5] * S[3] + t[1];
            const float cz = R[6] * S[1] + R[7] * S[2] + R[8] * S[3] + t[2];
            const float r = S[4];
            for (int o = 0; o < no; ++o) {
                const float4 A = OB4[4 * o], B = OB4[4 * o + 1], Cc = OB4[4 * o + 2], D = OB4[4 * o + 3];
                const float dx = cx - A.w, dy = cy - B.w, dz = cz - Cc.w;
                const float lx = dx * A.x + dy * A.y + dz * A.z;
                const float ly = dx * B.x + dy * B.y + dz * B.z;
                const float lz = dx * Cc.x + dy * Cc.y + dz * Cc.z;
                const int type = (int)D.w;
                float gap;
                if (type == 0) gap = pt_gap_box32(lx, ly, lz, r, D.x, D.y, D.z);
                else if (type == 1) gap = pt_gap_cylinder32(lx, ly, lz, r, D.x, D.y);
                else gap = sqrtf(lx * lx + ly * ly + lz * lz) - (r + D.x);
                if (gap < -margin) { hit = true; break; }
                if (!(gap > margin)) undecided = true;     // also catches NaN
            }
            ++sp;
        }
    }
    out[i] = hit ? 1 : (undecided ? 2 : 0);
}

__global__ void pt_check_select_kernel(const uint8_t* __restrict__ flag, size_t m, uint32_t* __restrict__ list,
                                       unsigned long long* count) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool take = i < m && flag[i] == 2;
    const unsigned ballot = __ballot_sync(0xffffffffu, take);
    if (ballot) {
        const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (take) list[base + __popc(ballot & ((1u << lane) - 1u))] = (uint32_t)i;
    }
}

// mode: PT_LIMIT_ERROR -> out-of-limit rows recorded in *first_bad (atomicMin) and marked 1
//       PT_LIMIT_UNFREE -> out-of-limit rows marked 1 without testing; PT_LIMIT_IGNORE -> always test
__global__ void __launch_bounds__(128)
pt_check_kernel(const double* __restrict__ model, int nj, int ns, int no, const double* __restrict__ q_, size_t m_all,
                int mode, uint8_t* __restrict__ out, unsigned long long* first_bad, const uint32_t* __restrict__ list,
                const unsigned long long* __restrict__ list_count) {
    extern __shared__ double sm[];
    const size_t m = list ? (size_t)*list_count : m_all;        // optional compacted row list (device-side count)
    if ((size_t)blockIdx.x * blockDim.x >= m) return;
    const int total = nj * PT_JSTRIDE + ns * PT_SSTRIDE + no * PT_OSTRIDE;
    for (int i = threadIdx.x; i < total; i += blockDim.x) sm[i] = model[i];
    __syncthreads();
    const double* J = sm;
    const double* SP = sm + nj * PT_JSTRIDE;
    const double* OB = SP + ns * PT_SSTRIDE;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= m) return;
    const size_t i = list ? (size_t)list[idx] : idx;
    double q[PT_MAX_JOINTS];
    bool inside = true;
    for (int j = 0; j < nj; ++j) {
        q[j] = q_[i * nj + j];
        inside = inside && (q[j] >= J[j * PT_JSTRIDE + 16]) && (q[j] <= J[j * PT_JSTRIDE + 17]);
    }
    if (mode != PT_LIMIT_IGNORE && !inside) {
        out[i] = 1;
        if (mode == PT_LIMIT_ERROR) atomicMin(first_bad, (unsigned long long)i);
        return;
    }
    double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double t[3] = {0, 0, 0};
    int sp = 0;
    bool hit = false;
    for (int link = 0; link <= nj && !hit; ++link) {
        if (link > 0) pt_fk_step(J + (link - 1) * PT_JSTRIDE, q[link - 1], R, t);
        while (sp < ns && (int)SP[sp * PT_SSTRIDE] == link) {
            const double* S = SP + sp * PT_SSTRIDE;
            double c[3];
            pt_matvec(R, S + 1, c);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = __dadd_rn(c[k], t[k]);
            if (pt_sphere_vs_scene(OB, no, c, S[4])) { hit = true; break; }
            ++sp;
        }
    }
    out[i] = hit ? 1 : 0;
}

__global__ void __launch_bounds__(128)
pt_fk_kernel(const double* __restrict__ model, int nj, int ns, const int* __restrict__ sphere_orig,
             const double* __restrict__ q_, size_t m, double* __restrict__ centers) {
    extern __shared__ double sm[];
    const int total = nj * PT_JSTRIDE + ns * PT_SSTRIDE;
    for (int i = threadIdx.x; i < total; i += blockDim.x) sm[i] = model[i];
    __syncthreads();
    const double* J = sm;
    const double* SP = sm + nj * PT_JSTRIDE;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double t[3] = {0, 0, 0};
    int sp = 0;
    for (int link = 0; link <= nj; ++link) {
        if (link > 0) pt_fk_step(J + (link - 1) * PT_JSTRIDE, q_[i * nj + link - 1], R, t);
        while (sp < ns && (int)SP[sp * PT_SSTRIDE] == link) {
            const double* S = SP + sp * PT_SSTRIDE;
            double c[3];
            pt_matvec(R, S + 1, c);
            const int orig = sphere_orig[sp];
#pragma unroll
            for (int k = 0; k < 3; ++k) centers[(i * ns + orig) * 3 + k] = __dadd_rn(c[k], t[k]);
            ++sp;
        }
    }
}

int pt_checker_run_dev(pt_ctx* ctx, const pt_checker* ck, const double* q_dev, size_t m, int mode,
                       uint8_t* out_dev, long long* first_bad_host) {
    if (first_bad_host) *first_bad_host = -1;
    if (m == 0) return PT_OK;
    PtBuf<unsigned long long> bad;
    PT_TRY(bad.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), ctx->stream));
    const size_t smem = ck->model_doubles * sizeof(double);
    if (ck->gap_margin > 0.f && mode != PT_LIMIT_ERROR && m >= 4096 && m < (1ull << 32)) {
        // fp32 screen, then the fp64 kernel on the undecided configurations only
        PtBuf<uint32_t> list; PtBuf<unsigned long long> cnt;
        PT_TRY(list.alloc(ctx, m));
        PT_TRY(cnt.alloc(ctx, 1));
        PT_CUDA(ctx, cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
        {
            PT_LAUNCH(ctx, "collision_screen_fp32");
            pt_check32_kernel<<<pt_grid_for(m, 128), 128, (ck->model_doubles + 4) * sizeof(float), ctx->stream>>>(
                ck->model.p, ck->nj, ck->ns, ck->no, q_dev, m, mode, ck->gap_margin, out_dev);
            PT_TRY(pt_check_launch(ctx, "pt_check32_kernel"));
            pt_check_select_kernel<<<pt_grid_for(m, 256), 256, 0, ctx->stream>>>(out_dev, m, list.p, cnt.p);
            PT_TRY(pt_check_launch(ctx, "pt_check_select_kernel"));
        }
        PT_LAUNCH(ctx, "collision_check");
        pt_check_kernel<<<pt_grid_for(m, 128), 128, smem, ctx->stream>>>(ck->model.p, ck->nj, ck->ns, ck->no, q_dev, m,
                                                                           mode, out_dev, bad.p, list.p, cnt.p);
        PT_TRY(pt_check_launch(ctx, "pt_check_kernel"));
        return PT_OK;
    }
    {
        PT_LAUNCH(ctx, "collision_check");
        pt_check_kernel<<<pt_grid_for(m, 128), 128, smem, ctx->stream>>>(ck->model.p, ck->nj, ck->ns, ck->no, q_dev, m,
                                                                           mode, out_dev, bad.p, nullptr, nullptr);
        PT_TRY(pt_check_launch(ctx, "pt_check_kernel"));
    }
    if (mode == PT_LIMIT_ERROR) {
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, bad.p, sizeof(*h), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (*h != ~0ull) {
            if (first_bad_host) *first_bad_host = (long long)*h;
            return pt_fail(ctx, PT_E_LIMIT, "configuration %llu violates the joint limits", *h);
        }
    }
    return PT_OK;
}

template <typename K, typename... Args>
static int pt_hits_common(pt_ctx* ctx, const char* name, K kernel, const double* centers, const double* radii,
                          long long m, uint8_t* out, Args... args) {
    if (!ctx) return pt_fail(ctx, PT_E_INVALID, "ctx is NULL");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative sphere count");
    if (m == 0) return PT_OK;
    if (!centers || !radii || !out) return pt_fail(ctx, PT_E_INVALID, "%s: NULL array", name);
    PtBuf<double> tc, tr; PtBuf<uint8_t> to;
    const double *cdev, *rdev;
    PT_TRY(pt_stage_in(ctx, centers, (size_t)m * 3, tc, &cdev));
    PT_TRY(pt_stage_in(ctx, radii, (size_t)m, tr, &rdev));
    uint8_t* odev = out;
    if (!pt_is_device_ptr(out)) { PT_TRY(to.alloc(ctx, m)); odev = to.p; }
    {
        PT_LAUNCH(ctx, name);
        kernel<<<pt_grid_for((size_t)m, 256), 256, 0, ctx->stream>>>(cdev, rdev, (size_t)m, args..., odev);
        PT_TRY(pt_check_launch(ctx, name));
    }
    if (odev != out) PT_TRY(pt_copy_out(ctx, out, odev, (size_t)m, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

extern "C" {

int pt_sphere_box_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m, double lx, double ly,
                       double lz, uint8_t* out) {
    return pt_hits_common(ctx, "sphere_box_hits", pt_sphere_box_kernel, centers, radii, m, out, lx, ly, lz);
}
int pt_sphere_cylinder_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m, double height,
                            double radius, uint8_t* out) {
    return pt_hits_common(ctx, "sphere_cylinder_hits", pt_sphere_cyl_kernel, centers, radii, m, out, height, radius);
}
int pt_sphere_sphere_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m, double radius,
                          uint8_t* out) {
    return pt_hits_common(ctx, "sphere_sphere_hits", pt_sphere_sph_kernel, centers, radii, m, out, radius);
}

int pt_checker_create(pt_ctx* ctx, int nj, const int* joint_kind, const double* joint_axis, const double* joint_rot,
                      const double* joint_trans, const double* joint_limits, int ns, const int* sphere_link,
                      const double* sphere_offset, const double* sphere_radius, int no, const int* obs_type,
                      const double* obs_rot, const double* obs_trans, const double* obs_dims, pt_checker** out) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_checker_create: NULL argument");
    if (nj < 1 || nj > PT_MAX_JOINTS) return pt_fail(ctx, PT_E_INVALID, "robot needs 1..%d joints, got %d", PT_MAX_JOINTS, nj);
    if (ns < 1) return pt_fail(ctx, PT_E_INVALID, "robot needs at least one collision sphere");
    if (no < 0) return pt_fail(ctx, PT_E_INVALID, "negative obstacle count");
    for (int s = 0; s < ns; ++s)
        if (sphere_link[s] < 0 || sphere_link[s] > nj) return pt_fail(ctx, PT_E_INVALID, "sphere attached to unknown link %d", sphere_link[s]);
    pt_checker* ck = new pt_checker();
    ck->ctx = ctx; ck->nj = nj; ck->ns = ns; ck->no = no;
    ck->model_doubles = (size_t)nj * PT_JSTRIDE + (size_t)ns * PT_SSTRIDE + (size_t)no * PT_OSTRIDE;
    if (ck->model_doubles * sizeof(double) > 200 * 1024) {
        delete ck;
        return pt_fail(ctx, PT_E_INVALID, "robot+scene model (%zu doubles) exceeds the shared-memory staging limit", ck->model_doubles);
    }
    std::vector<double> h(ck->model_doubles, 0.0);
    for (int j = 0; j < nj; ++j) {
        double* J = &h[(size_t)j * PT_JSTRIDE];
        J[0] = (double)joint_kind[j];
        for (int k = 0; k < 3; ++k) J[1 + k] = joint_axis[3 * j + k];
        for (int k = 0; k < 9; ++k) J[4 + k] = joint_rot[9 * j + k];
        for (int k = 0; k < 3; ++k) J[13 + k] = joint_trans[3 * j + k];
        J[16] = joint_limits[2 * j]; J[17] = joint_limits[2 * j + 1];
    }
    // stable sort of spheres by link so the kernel walks the chain once
    ck->sphere_order.resize(ns);
    {
        int w = 0;
        for (int link = 0; link <= nj; ++link)
            for (int s = 0; s < ns; ++s)
                if (sphere_link[s] == link) ck->sphere_order[w++] = s;
    }
    double* SP = &h[(size_t)nj * PT_JSTRIDE];
    for (int w = 0; w < ns; ++w) {
        int s = ck->sphere_order[w];
        SP[w * PT_SSTRIDE] = (double)sphere_link[s];
        for (int k = 0; k < 3; ++k) SP[w * PT_SSTRIDE + 1 + k] = sphere_offset[3 * s + k];
        SP[w * PT_SSTRIDE + 4] = sphere_radius[s];
    }
    double* OB = SP + (size_t)ns * PT_SSTRIDE;
    for (int o = 0; o < no; ++o) {
        double* O = OB + (size_t)o * PT_OSTRIDE;
        O[0] = (double)obs_type[o];
        for (int k = 0; k < 9; ++k) O[1 + k] = obs_rot[9 * o + k];
        for (int k = 0; k < 3; ++k) O[10 + k] = obs_trans[3 * o + k];
        for (int k = 0; k < 3; ++k) O[13 + k] = obs_dims[3 * o + k];
    }
    int rc = ck->model.alloc(ctx, ck->model_doubles);
    if (rc == PT_OK) rc = ck->sphere_orig.alloc(ctx, ns);
    if (rc != PT_OK) { delete ck; return rc; }
    cudaMemcpyAsync(ck->model.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(ck->sphere_orig.p, ck->sphere_order.data(), ns * sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { delete ck; return pt_fail(ctx, PT_E_CUDA, "model upload failed: %s", cudaGetErrorString(e)); }
    {
        // |gap32 - gap| <= 64 u32 (nj + 2) * (chain reach + farthest obstacle + largest primitive): every fp32
        // operation of the walk errs by at most u32 times a coordinate bounded by that length; 64 covers the op count
        // per joint (two 3x3 products, Rodrigues, sincosf) with a wide allowance
        double reach = 0.0, far = 0.0, dims = 0.0;
        for (int j = 0; j < nj; ++j) {
            double tn = 0.0;
            for (int k = 0; k < 3; ++k) tn += joint_trans[3 * j + k] * joint_trans[3 * j + k];
            reach += sqrt(tn);
            if (joint_kind[j] != 0) reach += fmax(fabs(joint_limits[2 * j]), fabs(joint_limits[2 * j + 1]));
        }
        double off = 0.0;
        for (int sidx = 0; sidx < ns; ++sidx) {
            double on = 0.0;
            for (int k = 0; k < 3; ++k) on += sphere_offset[3 * sidx + k] * sphere_offset[3 * sidx + k];
            off = fmax(off, sqrt(on) + fabs(sphere_radius[sidx]));
        }
        for (int o = 0; o < no; ++o) {
            double tn = 0.0;
            for (int k = 0; k < 3; ++k) { tn += obs_trans[3 * o + k] * obs_trans[3 * o + k]; dims = fmax(dims, fabs(obs_dims[3 * o + k])); }
            far = fmax(far, sqrt(tn));
        }
        const double length = reach + off + far + dims + 1.0;
        const char* env = getenv("PERMATRACE_B200_PRECISION");
        const bool plain = env && env[0] == '0';
        ck->gap_margin = plain ? 0.f : (float)(64.0 * 5.9604644775390625e-08 * (nj + 2) * length);
        if (!(ck->gap_margin < 1e-2f)) ck->gap_margin = 0.f;     // hopelessly large model: fp64 only
    }
    if (ck->model_doubles * sizeof(double) > 48 * 1024) {
        cudaFuncSetAttribute(pt_check32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((ck->model_doubles + 4) * sizeof(float)));
        cudaFuncSetAttribute(pt_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ck->model_doubles * sizeof(double)));
        cudaFuncSetAttribute(pt_fk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ck->model_doubles * sizeof(double)));
    }
    *out = ck;
    return PT_OK;
}

void pt_checker_destroy(pt_checker* ck) { delete ck; }

int pt_fk_batch(pt_ctx* ctx, const pt_checker* ck, const double* configs, long long m, double* out_centers) {
    if (!ctx || !ck) return pt_fail(ctx, PT_E_INVALID, "pt_fk_batch: NULL argument");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative configuration count");
    if (m == 0) return PT_OK;
    if (!configs || !out_centers) return pt_fail(ctx, PT_E_INVALID, "pt_fk_batch: NULL array");
    PtBuf<double> tq, to;
    const double* qdev;
    PT_TRY(pt_stage_in(ctx, configs, (size_t)m * ck->nj, tq, &qdev));
    double* odev = out_centers;
    const size_t outn = (size_t)m * ck->ns * 3;
    if (!pt_is_device_ptr(out_centers)) { PT_TRY(to.alloc(ctx, outn)); odev = to.p; }
    const size_t smem = ((size_t)ck->nj * PT_JSTRIDE + (size_t)ck->ns * PT_SSTRIDE) * sizeof(double);
    {
        PT_LAUNCH(ctx, "fk_batch");
        pt_fk_kernel<<<pt_grid_for((size_t)m, 128), 128, smem, ctx->stream>>>(ck->model.p, ck->nj, ck->ns, ck->sphere_orig.p,
                                                                                qdev, (size_t)m, odev);
        PT_TRY(pt_check_launch(ctx, "pt_fk_kernel"));
    }
    if (odev != out_centers) PT_TRY(pt_copy_out(ctx, out_centers, odev, outn, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_batch_check(pt_ctx* ctx, const pt_checker* ck, const double* configs, long long m, int on_limit, uint8_t* out,
                   long long* first_bad) {
    if (!ctx || !ck) return pt_fail(ctx, PT_E_INVALID, "pt_batch_check: NULL argument");
    if (on_limit < 0 || on_limit > 2) return pt_fail(ctx, PT_E_INVALID, "on_limit must be 0 (error), 1 (unfree) or 2 (ignore)");
    if (m < 0) return pt_fail(ctx, PT_E_INVALID, "negative configuration count");
    if (first_bad) *first_bad = -1;
    if (m == 0) return PT_OK;
    if (!configs || !out) return pt_fail(ctx, PT_E_INVALID, "pt_batch_check: NULL array");
    PtBuf<double> tq; PtBuf<uint8_t> to;
    const double* qdev;
    PT_TRY(pt_stage_in(ctx, configs, (size_t)m * ck->nj, tq, &qdev));
    uint8_t* odev = out;
    if (!pt_is_device_ptr(out)) { PT_TRY(to.alloc(ctx, m)); odev = to.p; }
    PT_TRY(pt_checker_run_dev(ctx, ck, qdev, (size_t)m, on_limit, odev, first_bad));
    if (odev != out) PT_TRY(pt_copy_out(ctx, out, odev, (size_t)m, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

}  // extern "C"
