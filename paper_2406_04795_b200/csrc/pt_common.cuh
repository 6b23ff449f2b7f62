// Shared device/host primitives: packed lattice keys, Freudenthal-Kuhn (Coxeter A~_n)
// edge/coface combinatorics as pure bit arithmetic, and the 16-byte-entry open-addressing
// HBM hash table used by the tracer and the refiner.
//
// Reference behaviour restated here (never copied):
//   canonical edge  = (base u, step mask s)          /root/reference/pkg/src/permatrace/lattice.py:125-127,156-166
//   coface order    = ordered splits of p1 then p2   /root/reference/pkg/src/permatrace/lattice.py:210-230
//   partner edges   = (a,c) / (b,c) of each coface   /root/reference/pkg/src/permatrace/tracer.py:123-149
//   cell cofaces    = |p1|!*|p2|! cells per edge     /root/reference/pkg/src/permatrace/lattice.py:245-266
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PT_NMAX 8
#define PT_HD __host__ __device__ __forceinline__

typedef unsigned long long u64;

#define PT_EMPTY (~0ull)
// value-word conventions of the visited-edge table
#define PT_VAL_PENDING_BASE (1ull << 40)   // val >= base: tentative slot id of the current wave
#define PT_VAL_DEAD (~0ull - 1ull)          // inserted but rejected by the max_edges cap

// error bits accumulated in PtCounters::error
#define PT_ERR_KEY_RANGE 1u   // lattice coordinate left the packed-key window
#define PT_ERR_TABLE_FULL 2u  // probe sequence wrapped (host sizing bug)

struct PtGeom {
    int n;                    // ambient dimension (2..7)
    int bits;                 // bits per packed coordinate
    int origin[PT_NMAX];      // window origin in lattice units (packed coord = v - origin >= 0)
    double scale;             // lattice edge scale
    double offset[PT_NMAX];   // lattice origin offset
    int has_box;              // clamp box present?
    int box_lo[PT_NMAX];      // inclusive integer bounds (ceil((lo-offset)/scale))
    int box_hi[PT_NMAX];      // inclusive integer bounds (floor((hi-offset)/scale))
};

PT_HD int pt_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __popc(x);
#else
    return __builtin_popcount(x);
#endif
}

PT_HD u64 pt_mix(u64 x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// ---- packed keys ---------------------------------------------------------------------------
// vertex key: coordinate 0 in the most significant field so that numeric order == lexicographic
// order of the integer vectors (needed for the sorted coarse_cells output).
PT_HD bool pt_pack_vertex(const PtGeom& g, const int* v, u64& key) {
    u64 k = 0; bool ok = true;
    const uint32_t lim = 1u << g.bits;
    for (int d = 0; d < g.n; ++d) {
        uint32_t r = (uint32_t)(v[d] - g.origin[d]);
        ok = ok && (r < lim);
        k = (k << g.bits) | (u64)(r & (lim - 1u));
    }
    key = k;
    return ok;
}
PT_HD void pt_unpack_vertex(const PtGeom& g, u64 key, int* v) {
    const u64 m = (1ull << g.bits) - 1ull;
    for (int d = g.n - 1; d >= 0; --d) { v[d] = (int)(key & m) + g.origin[d]; key >>= g.bits; }
}
PT_HD u64 pt_edge_key(const PtGeom& g, u64 vkey, uint32_t mask) { return (vkey << g.n) | (u64)mask; }
PT_HD u64 pt_edge_vkey(const PtGeom& g, u64 ekey) { return ekey >> g.n; }
PT_HD uint32_t pt_edge_mask(const PtGeom& g, u64 ekey) { return (uint32_t)(ekey & ((1ull << g.n) - 1ull)); }
#define PT_CELL_RANK_BITS 13   // 7! = 5040 < 2^13
PT_HD u64 pt_cell_key(u64 vkey, uint32_t rank) { return (vkey << PT_CELL_RANK_BITS) | (u64)rank; }

// adding a 0/1 mask to a packed vertex key (no carries can cross fields while in range)
PT_HD u64 pt_mask_to_packed(const PtGeom& g, uint32_t mask) {
    u64 k = 0;
    for (int d = 0; d < g.n; ++d) k = (k << g.bits) | (u64)((mask >> d) & 1u);
    return k;
}

PT_HD bool pt_in_box(const PtGeom& g, const int* v) {
    if (!g.has_box) return true;
    bool ok = true;
    for (int d = 0; d < g.n; ++d) ok = ok && (v[d] >= g.box_lo[d]) && (v[d] <= g.box_hi[d]);
    return ok;
}

// ---- coface enumeration --------------------------------------------------------------------
// deposit the low bits of `bits` into the set positions of `mask`, ascending (software PDEP)
PT_HD uint32_t pt_pdep(uint32_t bits, uint32_t mask) {
    uint32_t out = 0;
    while (mask) {
        uint32_t low = mask & (0u - mask);
        if (bits & 1u) out |= low;
        bits >>= 1; mask ^= low;
    }
    return out;
}

PT_HD int pt_ncofaces(int n, uint32_t s) {
    int m1 = pt_popc(s), m2 = n + 1 - m1;
    return ((1 << m1) - 2) + ((1 << m2) - 2);
}

// One 2-simplex coface of the canonical edge (u, s) in the reference's plan order.
//   third vertex c = u + 1_{c_plus} - 1_{c_minus}
//   partner edge (b,c) [taken when sign(c)==sign(a)] and (a,c) [otherwise], each canonical:
//   base = u + 1_{*_bplus} - 1_{*_bminus}, step mask *_mask, *_shared = base is the shared endpoint
struct PtCoface {
    uint32_t c_plus, c_minus;
    uint32_t bc_bplus, bc_bminus, bc_mask; int bc_shared;
    uint32_t ac_bplus, ac_bminus, ac_mask; int ac_shared;
};

PT_HD PtCoface pt_coface(int n, uint32_t s, int j) {
    PtCoface f;
    const uint32_t full = (1u << n) - 1u;
    const uint32_t comp = full & ~s;
    const int m1 = pt_popc(s);
    const int na = (1 << m1) - 2;
    if (j < na) {
        // ordered split (s1, s2) of p1: c = u + s1
        uint32_t s1 = pt_pdep((uint32_t)(j + 1), s);
        f.c_plus = s1; f.c_minus = 0;
        f.ac_bplus = 0; f.ac_bminus = 0; f.ac_mask = s1; f.ac_shared = 1;          // (a, c), base a
        f.bc_bplus = s1; f.bc_bminus = 0; f.bc_mask = s & ~s1; f.bc_shared = 0;    // (c, b), base c
    } else {
        // ordered split (t1, t2) of p2 = comp labels ascending followed by the wrap label n
        const int m2 = n + 1 - m1;
        uint32_t bits = (uint32_t)(j - na + 1);
        uint32_t t1 = pt_pdep(bits & ((1u << (m2 - 1)) - 1u), comp);
        if (!((bits >> (m2 - 1)) & 1u)) {
            // wrap label in t2: c = u + s + t1
            f.c_plus = s | t1; f.c_minus = 0;
            f.bc_bplus = s; f.bc_bminus = 0; f.bc_mask = t1; f.bc_shared = 1;      // (b, c), base b
            f.ac_bplus = 0; f.ac_bminus = 0; f.ac_mask = s | t1; f.ac_shared = 1;  // (a, c), base a
        } else {
            // wrap label in t1: c = u - t2, t2 = comp \ t1
            uint32_t t2 = comp & ~t1;
            f.c_plus = 0; f.c_minus = t2;
            f.ac_bplus = 0; f.ac_bminus = t2; f.ac_mask = t2; f.ac_shared = 0;       // (c, a), base c
            f.bc_bplus = 0; f.bc_bminus = t2; f.bc_mask = s | t2; f.bc_shared = 0;   // (c, b), base c
        }
    }
    return f;
}

PT_HD void pt_apply_masks(int n, const int* u, uint32_t plus, uint32_t minus, int* out) {
    for (int d = 0; d < n; ++d) out[d] = u[d] + (int)((plus >> d) & 1u) - (int)((minus >> d) & 1u);
}

// ---- permutations (cells) ------------------------------------------------------------------
PT_HD int pt_factorial(int m) { int f = 1; for (int i = 2; i <= m; ++i) f *= i; return f; }

// lexicographic rank of a permutation of {0..n-1}
PT_HD uint32_t pt_perm_rank(int n, const uint8_t* perm) {
    uint32_t rank = 0; uint32_t used = 0;
    for (int i = 0; i < n; ++i) {
        uint32_t p = perm[i];
        uint32_t smaller = (uint32_t)pt_popc(((1u << p) - 1u) & ~used);
        rank = rank * (uint32_t)(n - i) + smaller;
        used |= 1u << p;
    }
    return rank;
}
PT_HD void pt_perm_unrank(int n, uint32_t rank, uint8_t* perm) {
    // digits of the factorial number system, most significant first
    uint32_t digits[PT_NMAX];
    for (int i = n - 1; i >= 0; --i) { uint32_t base = (uint32_t)(n - i); digits[i] = rank % base; rank /= base; }
    uint32_t avail = (1u << n) - 1u;
    for (int i = 0; i < n; ++i) {
        uint32_t m = avail; uint32_t dsel = digits[i];
        while (dsel--) m &= m - 1u;          // drop the dsel lowest available labels
        uint32_t low = m & (0u - m);
        int lab = 0; while (!((low >> lab) & 1u)) ++lab;
        perm[i] = (uint8_t)lab; avail ^= low;
    }
}

// t-th ordering (any fixed bijection) of the labels in `set`; writes popc(set) labels
PT_HD void pt_subset_perm(uint32_t set, int t, uint8_t* out) {
    int m = pt_popc(set);
    uint32_t avail = set;
    for (int i = 0; i < m; ++i) {
        int base = m - i;
        int f = pt_factorial(base - 1);
        int dsel = t / f; t -= dsel * f;
        uint32_t mm = avail;
        while (dsel--) mm &= mm - 1u;
        uint32_t low = mm & (0u - mm);
        int lab = 0; while (!((low >> lab) & 1u)) ++lab;
        out[i] = (uint8_t)lab; avail ^= low;
    }
}

// Number of full-dimensional cells containing edge (u, s): |p1|! * |p2|!
PT_HD int pt_ncellcofaces(int n, uint32_t s) {
    int m1 = pt_popc(s);
    return pt_factorial(m1) * pt_factorial(n + 1 - m1);
}

// t-th cell containing the canonical edge (u, s).  A canonical cell is (base', pi) with the wrap
// label last; the edge's step labels form a contiguous block of pi, preceded by the labels Y that
// the cell walks before reaching u (base' = u - 1_Y) and followed by the rest X of comp(s).
PT_HD void pt_cellcoface(int n, uint32_t s, int t, uint32_t& y_mask, uint8_t* perm) {
    const uint32_t full = (1u << n) - 1u;
    const uint32_t comp = full & ~s;
    const int m1 = pt_popc(s);
    const int mc = n - m1;                 // |comp|
    const int f1 = pt_factorial(m1);
    int t1 = t % f1; int t2 = t / f1;      // t2 in [0, (mc+1)!)
    // ordering of comp plus the wrap marker: unrank a permutation of mc+1 items, item mc = marker
    uint8_t ord[PT_NMAX + 1];
    {
        uint32_t avail = (1u << (mc + 1)) - 1u;
        for (int i = 0; i <= mc; ++i) {
            int base = mc + 1 - i;
            int f = pt_factorial(base - 1);
            int dsel = t2 / f; t2 -= dsel * f;
            uint32_t mm = avail;
            while (dsel--) mm &= mm - 1u;
            uint32_t low = mm & (0u - mm);
            int idx = 0; while (!((low >> idx) & 1u)) ++idx;
            ord[i] = (uint8_t)idx; avail ^= low;
        }
    }
    // map item index -> comp label
    uint8_t comp_lab[PT_NMAX];
    { int c = 0; for (int d = 0; d < n; ++d) if ((comp >> d) & 1u) comp_lab[c++] = (uint8_t)d; }
    int pos_marker = 0;
    for (int i = 0; i <= mc; ++i) if (ord[i] == mc) pos_marker = i;
    // X = items before the marker (walked after the edge block), Y = items after the marker
    int w = 0; y_mask = 0;
    for (int i = pos_marker + 1; i <= mc; ++i) { uint8_t lab = comp_lab[ord[i]]; perm[w++] = lab; y_mask |= 1u << lab; }
    pt_subset_perm(s, t1, perm + w); w += m1;
    for (int i = 0; i < pos_marker; ++i) perm[w++] = comp_lab[ord[i]];
}

// ---- 16-byte-entry open-addressing table (key, val), linear probing --------------------------
struct PtTable {
    u64* ent;        // 2 * capacity words, interleaved (key, val); memset 0xFF == all empty
    u64 cap_mask;    // capacity - 1 (capacity is a power of two)
};

#ifdef __CUDACC__
__device__ __forceinline__ u64 pt_ld_cg(const u64* p) { return __ldcg(p); }

// insert-if-absent; returns the slot index; *inserted tells whether this thread claimed it
__device__ __forceinline__ u64 pt_table_insert(const PtTable& t, u64 key, bool& inserted, unsigned* err) {
    u64 slot = pt_mix(key) & t.cap_mask;
    for (u64 probes = 0; probes <= t.cap_mask; ++probes) {
        u64 cur = pt_ld_cg(&t.ent[2 * slot]);
        if (cur == key) { inserted = false; return slot; }
        if (cur == PT_EMPTY) {
            u64 prev = atomicCAS(&t.ent[2 * slot], PT_EMPTY, key);
            if (prev == PT_EMPTY) { inserted = true; return slot; }
            if (prev == key) { inserted = false; return slot; }
        }
        slot = (slot + 1) & t.cap_mask;
    }
    atomicOr(err, PT_ERR_TABLE_FULL);
    inserted = false;
    return 0;
}
__device__ __forceinline__ bool pt_table_find(const PtTable& t, u64 key, u64& slot_out) {
    u64 slot = pt_mix(key) & t.cap_mask;
    for (u64 probes = 0; probes <= t.cap_mask; ++probes) {
        u64 cur = pt_ld_cg(&t.ent[2 * slot]);
        if (cur == key) { slot_out = slot; return true; }
        if (cur == PT_EMPTY) return false;
        slot = (slot + 1) & t.cap_mask;
    }
    return false;
}
#endif
