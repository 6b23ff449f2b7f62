// Host-executable mirrors of the device lattice arithmetic: the same inline functions the kernels
// use (pt_common.cuh), callable without a GPU so the CPU test-suite can pin them against the
// reference's expansion plans and cell-coface templates.
#include "pt_internal.cuh"

extern "C" {

int pt_host_expansion_plan(int n, uint32_t mask, int32_t* out, int cap) {
    if (n < 2 || n > 7 || mask == 0 || mask >= (1u << n)) return pt_fail(nullptr, PT_E_INVALID, "bad edge type");
    const int nc = pt_ncofaces(n, mask);
    if (!out) return nc;
    if (cap < nc) return pt_fail(nullptr, PT_E_INVALID, "plan buffer too small");
    for (int j = 0; j < nc; ++j) {
        PtCoface f = pt_coface(n, mask, j);
        int32_t* r = out + 10 * j;
        r[0] = (int32_t)f.c_plus; r[1] = (int32_t)f.c_minus;
        r[2] = (int32_t)f.bc_bplus; r[3] = (int32_t)f.bc_bminus; r[4] = (int32_t)f.bc_mask; r[5] = f.bc_shared;
        r[6] = (int32_t)f.ac_bplus; r[7] = (int32_t)f.ac_bminus; r[8] = (int32_t)f.ac_mask; r[9] = f.ac_shared;
    }
    return nc;
}

int pt_host_cellcofaces(int n, uint32_t mask, int32_t* out, int cap) {
    if (n < 2 || n > 7 || mask == 0 || mask >= (1u << n)) return pt_fail(nullptr, PT_E_INVALID, "bad edge type");
    const int nc = pt_ncellcofaces(n, mask);
    if (!out) return nc;
    if (cap < nc) return pt_fail(nullptr, PT_E_INVALID, "cell buffer too small");
    for (int t = 0; t < nc; ++t) {
        uint32_t y; uint8_t perm[PT_NMAX];
        pt_cellcoface(n, mask, t, y, perm);
        int32_t* r = out + (size_t)(1 + n) * t;
        r[0] = (int32_t)y;
        for (int d = 0; d < n; ++d) r[1 + d] = perm[d];
    }
    return nc;
}

int pt_host_perm_rank(int n, const uint8_t* perm) {
    if (n < 1 || n > 7 || !perm) return pt_fail(nullptr, PT_E_INVALID, "bad permutation");
    return (int)pt_perm_rank(n, perm);
}

int pt_host_perm_unrank(int n, int rank, uint8_t* perm) {
    if (n < 1 || n > 7 || !perm || rank < 0 || rank >= pt_factorial(n)) return pt_fail(nullptr, PT_E_INVALID, "bad rank");
    pt_perm_unrank(n, (uint32_t)rank, perm);
    return PT_OK;
}

}  // extern "C"
