/* CPU oracle: C restatement of the reference's compiled inner loops.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2406_04795_b200/ may link or call this file; it is
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs as
 * the checker and as the timed CPU baseline.
 *
 * Each function follows /root/reference/pkg/src/permatrace/_kernels.pyx (cited per function):
 * plain double arithmetic, the same loop order, the same branch order, libm exp/sqrt/fabs.
 * The *_mt variants only add an OpenMP split over independent rows (the reference releases the
 * GIL around these loops but never threads them); per-row arithmetic is unchanged.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* _kernels.pyx:18-40  acc = bias; for j: dist2 = sum_d (p_d - s_jd)^2; acc += w_j exp(-gamma dist2) */
static void rbf_rows(const double* points, ptrdiff_t lo, ptrdiff_t hi, int n, const double* support,
                     ptrdiff_t s, const double* weights, double gamma, double bias, double* out) {
    for (ptrdiff_t i = lo; i < hi; ++i) {
        double acc = bias;
        const double* p = points + i * n;
        for (ptrdiff_t j = 0; j < s; ++j) {
            const double* q = support + j * n;
            double dist2 = 0.0;
            for (int d = 0; d < n; ++d) {
                double diff = p[d] - q[d];
                dist2 += diff * diff;
            }
            acc += weights[j] * exp(-gamma * dist2);
        }
        out[i] = acc;
    }
}

void oracle_rbf_values(const double* points, ptrdiff_t m, int n, const double* support, ptrdiff_t s,
                       const double* weights, double gamma, double bias, double* out) {
    rbf_rows(points, 0, m, n, support, s, weights, gamma, bias, out);
}

void oracle_rbf_values_mt(const double* points, ptrdiff_t m, int n, const double* support, ptrdiff_t s,
                          const double* weights, double gamma, double bias, double* out, int threads) {
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (ptrdiff_t blk = 0; blk < (m + 255) / 256; ++blk) {
        ptrdiff_t lo = blk * 256, hi = lo + 256 < m ? lo + 256 : m;
        rbf_rows(points, lo, hi, n, support, s, weights, gamma, bias, out);
    }
}

/* _kernels.pyx:43-76 */
void oracle_sphere_box_hits(const double* centers, const double* radii, ptrdiff_t m, double lx, double ly,
                            double lz, uint8_t* out) {
    const double hx = 0.5 * lx, hy = 0.5 * ly, hz = 0.5 * lz;
    for (ptrdiff_t i = 0; i < m; ++i) {
        double px = fabs(centers[3 * i]), py = fabs(centers[3 * i + 1]), pz = fabs(centers[3 * i + 2]);
        double r = radii[i];
        double dx = px - hx, dy = py - hy, dz = pz - hz;
        out[i] = 0;
        if (dx > r || dy > r || dz > r) continue;
        if (px <= hx && dy > 0 && dz > 0 && dy * dy + dz * dz > r * r) continue;
        if (py <= hy && dx > 0 && dz > 0 && dx * dx + dz * dz > r * r) continue;
        if (pz <= hz && dx > 0 && dy > 0 && dx * dx + dy * dy > r * r) continue;
        if (dx > 0 && dy > 0 && dz > 0 && dx * dx + dy * dy + dz * dz > r * r) continue;
        out[i] = 1;
    }
}

/* _kernels.pyx:79-104 */
void oracle_sphere_cylinder_hits(const double* centers, const double* radii, ptrdiff_t m, double height,
                                 double radius, uint8_t* out) {
    const double hh = 0.5 * height;
    for (ptrdiff_t i = 0; i < m; ++i) {
        double pz = fabs(centers[3 * i + 2]);
        double r = radii[i];
        double rad = sqrt(centers[3 * i] * centers[3 * i] + centers[3 * i + 1] * centers[3 * i + 1]);
        double dz = pz - hh, dr = rad - radius;
        out[i] = 0;
        if (dz > r || dr > r) continue;
        if (dz > 0 && dr > 0 && dr * dr + dz * dz > r * r) continue;
        out[i] = 1;
    }
}

/* _kernels.pyx:107-122 */
void oracle_sphere_sphere_hits(const double* centers, const double* radii, ptrdiff_t m, double radius,
                               uint8_t* out) {
    for (ptrdiff_t i = 0; i < m; ++i) {
        double d2 = centers[3 * i] * centers[3 * i] + centers[3 * i + 1] * centers[3 * i + 1] +
                    centers[3 * i + 2] * centers[3 * i + 2];
        double rr = radii[i] + radius;
        out[i] = d2 <= rr * rr ? 1 : 0;
    }
}
