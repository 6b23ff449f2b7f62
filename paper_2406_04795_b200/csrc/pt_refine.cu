// Batch refinement of coarse cells (subdivision.py:220-301), fully on the device:
//   R1  warp per cell: template vertices -> fine-lattice integer keys -> shared sign table
//       (each distinct fine vertex is evaluated once; for k = 2 the evaluated coordinates are
//       bit-identical to the reference's per-cell einsum, see pt_fine_point)
//   R2  per-cell crossing counts over the template edges + exclusive scan  (global crossing index
//       = the reference's cell-major, template-edge-major order, subdivision.py:263-266)
//   R3  crossing fine edges -> canonical fine-lattice edge keys, atomicMin(first crossing index)
//   R4  distinct fine edges sorted by first occurrence; one bisection each (manifold.py:351-383)
//   R5  greedy eps-dedup in that order == _PointRegistry (subdivision.py:195-217), resolved in
//       parallel rounds over a sorted spatial hash
//   R6  collision labels for the kept points (pipeline.py:256-270)
#include <cub/cub.cuh>
#include "pt_trace.cuh"
#include "pt_field.cuh"

#define PT_MAX_TV 256      // template vertices
#define PT_SIGN_WORDS (PT_MAX_TV / 32)

struct PtFineCounters {
    unsigned long long n_pending;   // fine vertices queued for evaluation
    unsigned long long n_edges;     // distinct fine edges inserted
    unsigned long long undecided;   // dedup round bookkeeping
    unsigned long long ambiguous;   // fine vertices with |F| < 1e-12*(sum|w|+|b|)
    unsigned int error;
    unsigned int pad;
};

struct pt_refine {
    pt_ctx* ctx = nullptr;
    int n = 0;
    pt_refine_stats stats;
    PtBuf<double> points;
    PtBuf<uint8_t> labels;
    PtBuf<long long> first_tag;
    long long n_points = 0;
    std::vector<long long> batch_rows;   // nb x 2
};

struct PtRefGeom {
    PtGeom coarse;   // window of the cell keys
    PtGeom fine;     // fine lattice window (scale/offset of the COARSE lattice kept for X(i))
    int k, V, E, W;
};

// fine-lattice coordinate of template vertex v inside cell (base, perm): axis perm[j] gets
// k*base[perm[j]] + tv[v][j]
__device__ __forceinline__ void pt_fine_vertex(const PtRefGeom& rg, const int* base, const uint8_t* perm,
                                               const int8_t* tv_row, int* f) {
    for (int j = 0; j < rg.coarse.n; ++j) { int ax = perm[j]; f[ax] = rg.k * base[ax] + (int)tv_row[j]; }
}

// Cartesian point of a fine-lattice vertex: per axis f = k*q + r;  x = (1 - r/k) X(q) + (r/k) X(q+1),
// X(i) = i*scale + offset (two roundings, like the tracer).  For r == 0 this is exactly X(q); for
// k == 2 it is exactly the reference's 0.5*corner + 0.5*corner (subdivision.py:256-260).
__device__ __forceinline__ void pt_fine_point(const PtRefGeom& rg, const int* f, double* x) {
    const PtGeom& g = rg.fine;
    for (int d = 0; d < g.n; ++d) {
        int q = f[d] / rg.k; int r = f[d] - q * rg.k;
        if (r < 0) { r += rg.k; q -= 1; }
        const double x0 = __dadd_rn(__dmul_rn((double)q, g.scale), g.offset[d]);
        if (r == 0) { x[d] = x0; continue; }
        const double x1 = __dadd_rn(__dmul_rn((double)(q + 1), g.scale), g.offset[d]);
        const double w1 = __ddiv_rn((double)r, (double)rg.k);
        const double w0 = __dsub_rn(1.0, w1);
        x[d] = __dadd_rn(__dmul_rn(w0, x0), __dmul_rn(w1, x1));
    }
}

__device__ __forceinline__ void pt_decode_cell(const PtGeom& g, u64 key, int* base, uint8_t* perm) {
    pt_unpack_vertex(g, key >> PT_CELL_RANK_BITS, base);
    pt_perm_unrank(g.n, (uint32_t)(key & ((1u << PT_CELL_RANK_BITS) - 1u)), perm);
}

// ---- array-free cell decoding for the warp-per-cell kernels (runtime-indexed int arrays live in local memory) ----------
// Packed fine key of the cell's base corner, k*base - fine origin per axis, and the cell's permutation as nibbles
// (axis perm[j] in bits 4j..4j+3); same digits / label selection as pt_perm_unrank.
__device__ __forceinline__ void pt_cell_fast(const PtRefGeom& rg, u64 cell_key, u64& base_key, uint32_t& perm_nib) {
    const PtGeom& g = rg.coarse;
    const int n = g.n;
    u64 vk = cell_key >> PT_CELL_RANK_BITS;
    const u64 cm = (1ull << g.bits) - 1ull;
    u64 bk = 0;
    for (int d = n - 1; d >= 0; --d) {
        const int b = (int)(vk & cm) + g.origin[d];
        vk >>= g.bits;
        bk |= (u64)(uint32_t)(rg.k * b - rg.fine.origin[d]) << ((n - 1 - d) * rg.fine.bits);
    }
    base_key = bk;
    uint32_t rank = (uint32_t)(cell_key & ((1u << PT_CELL_RANK_BITS) - 1u));
    // factorial digits, least significant first: digit i (position i of the permutation) has base n - i
    uint32_t digits = 0;                       // 3 bits each
    for (int i = n - 1; i >= 0; --i) { const uint32_t b = (uint32_t)(n - i); digits |= (rank % b) << (3 * i); rank /= b; }
    uint32_t avail = (1u << n) - 1u, nib = 0;
    for (int i = 0; i < n; ++i) {
        uint32_t m = avail, dsel = (digits >> (3 * i)) & 7u;
        while (dsel--) m &= m - 1u;
        const uint32_t low = m & (0u - m);
        nib |= (uint32_t)(__ffs(low) - 1) << (4 * i);
        avail ^= low;
    }
    perm_nib = nib;
}

// packed fine key of template vertex `tv_row` (n int8 template coordinates) of that cell
__device__ __forceinline__ u64 pt_fine_vertex_key(const PtRefGeom& rg, u64 base_key, uint32_t perm_nib, const int8_t* __restrict__ tv_row) {
    const int n = rg.coarse.n;
    u64 k = base_key;
    for (int j = 0; j < n; ++j) {
        const int ax = (int)((perm_nib >> (4 * j)) & 15u);
        k += (u64)(uint32_t)tv_row[j] << ((n - 1 - ax) * rg.fine.bits);
    }
    return k;
}

__device__ __forceinline__ unsigned long long pt_warp_append64(unsigned long long* counter, bool pred) {
    unsigned ballot = __ballot_sync(0xffffffffu, pred);
    if (ballot == 0) return 0;
    int lane = threadIdx.x & 31;
    int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + (unsigned long long)__popc(ballot & ((1u << lane) - 1u));
}

// R1a: insert fine vertices, queue unknown ones
__global__ void __launch_bounds__(256)
pt_ref_vertices_kernel(PtRefGeom rg, PtTable fv, const u64* __restrict__ cell_keys, size_t ncells,
                       const int8_t* __restrict__ tv, uint32_t* __restrict__ vslot, uint32_t* __restrict__ pending,
                       PtFineCounters* ctr) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= ncells) return;
    const int n = rg.coarse.n;
    u64 base_key; uint32_t perm_nib;
    pt_cell_fast(rg, cell_keys[w], base_key, perm_nib);      // (the host checked that the fine window holds every cell)
    for (int v0 = 0; v0 < rg.V; v0 += 32) {
        const int v = v0 + lane;
        bool inserted = false; u64 slot = 0;
        if (v < rg.V) {
            slot = pt_table_insert(fv, pt_fine_vertex_key(rg, base_key, perm_nib, tv + v * n), inserted, &ctr->error);
            vslot[w * rg.V + v] = (uint32_t)slot;
        }
        unsigned long long pos = pt_warp_append64(&ctr->n_pending, inserted);
        if (inserted) pending[pos] = (uint32_t)slot;
    }
}

__global__ void pt_ref_pending_points_kernel(PtRefGeom rg, PtTable fv, const uint32_t* __restrict__ pending, size_t count,
                                             double* __restrict__ pts) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    int f[PT_NMAX]; double x[PT_NMAX];
    pt_unpack_vertex(rg.fine, fv.ent[2 * (u64)pending[i]], f);
    pt_fine_point(rg, f, x);
    for (int d = 0; d < rg.fine.n; ++d) pts[i * rg.fine.n + d] = x[d];
}
// value word of a fine vertex: bit 0 = sign (1: F > 0), bits 32..63 = the field value as fp32 (0 when the evaluator gives
// none) -- only a hint for where on a crossing edge the root sits
__global__ void pt_ref_pending_store_kernel(PtTable fv, const uint32_t* __restrict__ pending, size_t count,
                                            const int8_t* __restrict__ s, const float* __restrict__ v32) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 bits = v32 ? (u64)__float_as_uint(v32[i]) : 0ull;
    fv.ent[2 * (u64)pending[i] + 1] = (s[i] > 0 ? 1ull : 0ull) | (bits << 32);
}

// R1c + R2: per-cell sign words and crossing counts
__global__ void __launch_bounds__(256)
pt_ref_signs_kernel(PtRefGeom rg, PtTable fv, size_t ncells, const int16_t* __restrict__ te,
                    const uint32_t* __restrict__ vslot, uint32_t* __restrict__ csign, unsigned long long* __restrict__ ccount) {
    __shared__ uint32_t sw[8][PT_SIGN_WORDS];
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    if (w >= ncells) return;
    for (int v0 = 0, word = 0; v0 < rg.V; v0 += 32, ++word) {
        const int v = v0 + lane;
        bool pos = false;
        if (v < rg.V) pos = (pt_ld_cg(&fv.ent[2 * (u64)vslot[w * rg.V + v] + 1]) & 1ull) != 0ull;
        unsigned ballot = __ballot_sync(0xffffffffu, pos);
        if (lane == 0) { sw[wib][word] = ballot; csign[w * rg.W + word] = ballot; }
    }
    __syncwarp();
    int count = 0;
    for (int e0 = 0; e0 < rg.E; e0 += 32) {
        const int e = e0 + lane;
        bool cross = false;
        if (e < rg.E) {
            const int i0 = te[2 * e], i1 = te[2 * e + 1];
            cross = ((sw[wib][i0 >> 5] >> (i0 & 31)) & 1u) != ((sw[wib][i1 >> 5] >> (i1 & 31)) & 1u);
        }
        count += __popc(__ballot_sync(0xffffffffu, cross));
    }
    if (lane == 0) ccount[w] = (unsigned long long)count;
}

// R3: canonical fine edges, first-occurrence tag.  The kernel is instruction-bound, and only ~20 % of a cell's template
// edges cross: each warp first compacts the crossing edge indices of its cell into shared memory (cheap: two sign-bit
// tests per edge), then runs the expensive part (fine vertices, key packing, table insert, atomicMin) on dense lanes.
#define PT_RE_SEG 1024    /* template edges per compaction segment */
__global__ void __launch_bounds__(256)
pt_ref_edges_kernel(PtRefGeom rg, PtTable fe, const u64* __restrict__ cell_keys, size_t ncells, const int8_t* __restrict__ tv,
                    const int16_t* __restrict__ te, const uint32_t* __restrict__ csign, const unsigned long long* __restrict__ coff,
                    unsigned long long tag_base, PtFineCounters* ctr) {
    __shared__ uint16_t clist[8][PT_RE_SEG];
    __shared__ u64 vkey[8][PT_MAX_TV];           // packed fine keys of the cell's template vertices
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (w >= ncells) return;
    const int n = rg.coarse.n;
    {
        u64 base_key; uint32_t perm_nib;
        pt_cell_fast(rg, cell_keys[w], base_key, perm_nib);
        for (int v = lane; v < rg.V; v += 32) vkey[wib][v] = pt_fine_vertex_key(rg, base_key, perm_nib, tv + v * n);
    }
    __syncwarp();
    const int fbits = rg.fine.bits;
    uint32_t sw[PT_SIGN_WORDS];
    for (int i = 0; i < rg.W; ++i) sw[i] = csign[w * rg.W + i];
    unsigned long long running = tag_base + coff[w];
    unsigned int fresh = 0;
    for (int seg0 = 0; seg0 < rg.E; seg0 += PT_RE_SEG) {
        const int seg1 = seg0 + PT_RE_SEG < rg.E ? seg0 + PT_RE_SEG : rg.E;
        int total = 0;
        for (int e0 = seg0; e0 < seg1; e0 += 32) {
            const int e = e0 + lane;
            bool cross = false;
            if (e < seg1) {
                const int i0 = te[2 * e], i1 = te[2 * e + 1];
                cross = ((sw[i0 >> 5] >> (i0 & 31)) & 1u) != ((sw[i1 >> 5] >> (i1 & 31)) & 1u);
            }
            const unsigned ballot = __ballot_sync(0xffffffffu, cross);
            if (cross) clist[wib][total + __popc(ballot & ((1u << lane) - 1u))] = (uint16_t)e;
            total += __popc(ballot);
        }
        __syncwarp();
        for (int c0 = 0; c0 < total; c0 += 32) {
            const int c = c0 + lane;
            bool inserted = false;
            if (c < total) {
                const int e = clist[wib][c];
                const int i0 = te[2 * e], i1 = te[2 * e + 1];
                const unsigned s0 = (sw[i0 >> 5] >> (i0 & 31)) & 1u, s1 = (sw[i1 >> 5] >> (i1 & 31)) & 1u;
                const unsigned long long tag = running + (unsigned long long)c;
                // a template edge is a unit step of the fine lattice in some axes, all of one sign: the packed keys of its end
                // points order like the points, and their difference holds one bit per stepped axis
                const u64 ka = vkey[wib][i0], kb = vkey[wib][i1];
                const bool neg = kb < ka;
                const u64 bk = neg ? kb : ka, dk = neg ? ka - kb : kb - ka;
                uint32_t mask = 0;
                for (int d = 0; d < n; ++d) mask |= (uint32_t)((dk >> ((n - 1 - d) * fbits)) & 1ull) << d;
                const unsigned sbase = neg ? s1 : s0;
                u64 slot = pt_table_insert(fe, pt_edge_key(rg.fine, bk, mask), inserted, &ctr->error);
                atomicMin(&fe.ent[2 * slot + 1], (tag << 1) | (u64)sbase);
            }
            fresh += __popc(__ballot_sync(0xffffffffu, inserted));
        }
        running += (unsigned long long)total;
        __syncwarp();
    }
    if (lane == 0 && fresh) atomicAdd(&ctr->n_edges, (unsigned long long)fresh);
}

// R4: pull (val, key) pairs out of the fine-edge table.  Each thread scans a few slots; positions come from a
// block-wide scan and ONE atomic per block (a per-warp atomic on the single counter serialises at this table size).
#define PT_EXTRACT_THREADS 256
#define PT_EXTRACT_PER_THREAD 4
__global__ void __launch_bounds__(PT_EXTRACT_THREADS)
pt_ref_extract_kernel(PtTable fe, u64* __restrict__ vals, u64* __restrict__ keys, unsigned long long* counter) {
    typedef cub::BlockScan<int, PT_EXTRACT_THREADS> Scan;
    __shared__ typename Scan::TempStorage temp;
    __shared__ unsigned long long block_base;
    const u64 first = ((u64)blockIdx.x * PT_EXTRACT_THREADS + threadIdx.x) * PT_EXTRACT_PER_THREAD;
    u64 k[PT_EXTRACT_PER_THREAD], v[PT_EXTRACT_PER_THREAD];
    int mine = 0;
#pragma unroll
    for (int q = 0; q < PT_EXTRACT_PER_THREAD; ++q) {
        const u64 i = first + q;
        k[q] = PT_EMPTY; v[q] = 0;
        if (i <= fe.cap_mask) { k[q] = fe.ent[2 * i]; v[q] = fe.ent[2 * i + 1]; }
        mine += k[q] != PT_EMPTY;
    }
    int offset, total;
    Scan(temp).ExclusiveSum(mine, offset, total);
    if (threadIdx.x == 0) block_base = total ? atomicAdd(counter, (unsigned long long)total) : 0ull;
    __syncthreads();
    unsigned long long pos = block_base + (unsigned long long)offset;
#pragma unroll
    for (int q = 0; q < PT_EXTRACT_PER_THREAD; ++q)
        if (k[q] != PT_EMPTY) { vals[pos] = v[q]; keys[pos] = k[q]; ++pos; }
}

__global__ void pt_ref_endpoints_kernel(PtRefGeom rg, const u64* __restrict__ vals, const u64* __restrict__ keys, size_t first,
                                        size_t count, double* __restrict__ a, double* __restrict__ b, int8_t* __restrict__ sa,
                                        PtTable fv, float* __restrict__ hint) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const PtGeom& g = rg.fine;
    const u64 ek = keys[first + i];
    if (hint) {
        // secant estimate of the root from the fp32 values the vertex pass left in the fine-vertex table
        float h = 0.5f;
        u64 sa_, sb_;
        const u64 ka = pt_edge_vkey(g, ek), kb = ka + pt_mask_to_packed(g, pt_edge_mask(g, ek));
        if (pt_table_find(fv, ka, sa_) && pt_table_find(fv, kb, sb_)) {
            const float fa = __uint_as_float((unsigned)(fv.ent[2 * sa_ + 1] >> 32)), fb = __uint_as_float((unsigned)(fv.ent[2 * sb_ + 1] >> 32));
            const float t = fa / (fa - fb);
            if (t > 0.f && t < 1.f) h = t;
        }
        hint[i] = h;
    }
    int u[PT_NMAX], v[PT_NMAX]; double x[PT_NMAX];
    pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
    pt_apply_masks(g.n, u, pt_edge_mask(g, ek), 0u, v);
    pt_fine_point(rg, u, x);
    for (int d = 0; d < g.n; ++d) a[i * g.n + d] = x[d];
    pt_fine_point(rg, v, x);
    for (int d = 0; d < g.n; ++d) b[i * g.n + d] = x[d];
    sa[i] = (vals[first + i] & 1ull) ? (int8_t)1 : (int8_t)-1;
}

// ---- R5: greedy eps-dedup ----------------------------------------------------------------------
// hash of a grid cell: a linear form of the coordinates (odd 64-bit multipliers) through one mixing round -- the search
// gets a neighbouring cell's form by adding one multiplier per stepped axis
__device__ __constant__ u64 pt_grid_mult[PT_NMAX] = {
    0x9e3779b97f4a7c15ULL, 0xc2b2ae3d27d4eb4fULL, 0x165667b19e3779f9ULL, 0xd6e8feb86659fd93ULL,
    0xff51afd7ed558ccdULL, 0xc4ceb9fe1a85ec53ULL, 0x2545f4914f6cdd1dULL, 0x94d049bb133111ebULL};
__device__ __forceinline__ u64 pt_grid_form(int n, const long long* c) {
    u64 h = 0;
    for (int d = 0; d < n; ++d) h += (u64)c[d] * pt_grid_mult[d];
    return h;
}
__device__ __forceinline__ u64 pt_grid_finish(u64 form) { return pt_mix(form) & 0x7fffffffffffffffULL; }
__device__ __forceinline__ u64 pt_grid_hash(int n, const long long* c) { return pt_grid_finish(pt_grid_form(n, c)); }

__global__ void pt_dedup_hash_kernel(int n, const double* __restrict__ pts, size_t count, double cell, u64* __restrict__ gkey,
                                     uint32_t* __restrict__ idx) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    long long c[PT_NMAX];
    const double inv = 1.0 / cell;   // the grid only has to be monotone and identical in the hash and search kernels
    for (int d = 0; d < n; ++d) c[d] = (long long)floor(pts[i * n + d] * inv);
    gkey[i] = pt_grid_hash(n, c);
    idx[i] = (uint32_t)i;
}

// directory of the sorted grid keys: hash(cell) -> (first position of the cell's run) << 32 | the run's smallest point index
// (the sort is stable, so that is the run's first entry): a probe from a point that precedes everything in the cell -- the
// usual case, the cell holds the point itself or nothing earlier -- ends at the directory entry
// An occupancy bitmap (one bit per 2^-4 of a point: a few MB, L2-resident) stands in front of it: the eps-ball of a point
// touches ~3.8 cells of which ~2.8 are empty, and those probes end at a 4-byte read instead of a probe into the 16 U-entry table.
__global__ void pt_dedup_directory_kernel(const u64* __restrict__ gkey_sorted, const uint32_t* __restrict__ idx_sorted, size_t count,
                                          PtTable dir, uint32_t* __restrict__ bmp, u64 bmp_mask, unsigned* err) {
    const size_t a = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= count) return;
    const u64 gk = gkey_sorted[a];
    if (a > 0 && gkey_sorted[a - 1] == gk) return;
    { const u64 bit = (gk >> 20) & bmp_mask; atomicOr(&bmp[bit >> 5], 1u << (bit & 31)); }
    bool ins;
    const u64 slot = pt_table_insert(dir, gk, ins, err);
    dir.ent[2 * slot + 1] = ((u64)a << 32) | (u64)idx_sorted[a];
}

#define PT_DD_UNDECIDED 0
#define PT_DD_KEPT 1
#define PT_DD_REMOVED 2

// Greedy first-keeper resolution: a point is removed if an earlier kept point lies within eps, kept once every
// earlier point within eps is removed.
// Round 1 (all points) does the spatial search and decides every point that has no undecided earlier neighbour;
// the others go to a compacted list together with their neighbour COUNT.  A second pass over that list writes
// the neighbours into a CSR array (exclusive scan of the counts), and the follow-up rounds only look at the
// states of a point's recorded neighbours -- no spatial search, no launch over all points.
template <bool COLLECT>
__device__ __forceinline__ int pt_dedup_search(int n, const double* __restrict__ pts, size_t count, double cell, double eps,
                                               const u64* __restrict__ gkey_sorted, const uint32_t* __restrict__ idx_sorted,
                                               const PtTable& dir, const uint32_t* __restrict__ bmp, u64 bmp_mask,
                                               const uint8_t* state, size_t i, uint32_t* nbr, int& nbc) {
    // returns 2 if an earlier KEPT point is within eps, 1 if an earlier undecided one is, else 0 (COLLECT: states are
    // ignored and every earlier neighbour within eps is written to nbr); nbc = earlier neighbours within eps seen
    double p[PT_NMAX]; long long lo[PT_NMAX], hi[PT_NMAX];
    int ncomb = 1;
    const double inv = 1.0 / cell;
    for (int d = 0; d < n; ++d) {
        p[d] = pts[i * n + d];
        lo[d] = (long long)floor((p[d] - eps) * inv);
        hi[d] = (long long)floor((p[d] + eps) * inv);
        if (hi[d] != lo[d]) ncomb <<= 1;
    }
    bool any_kept = false, any_undecided = false;
    nbc = 0;
    const u64 form_lo = pt_grid_form(n, lo);
    for (int comb = 0; comb < ncomb && !any_kept; ++comb) {
        u64 form = form_lo; int bit = 0;
        for (int d = 0; d < n; ++d)
            if (hi[d] != lo[d]) { if ((comb >> bit) & 1) form += (u64)(hi[d] - lo[d]) * pt_grid_mult[d]; ++bit; }
        const u64 gk = pt_grid_finish(form);
        { const u64 bit = (gk >> 20) & bmp_mask; if (!((__ldg(&bmp[bit >> 5]) >> (bit & 31)) & 1u)) continue; }   // empty for sure
        u64 slot;
        if (!pt_table_find(dir, gk, slot)) continue;          // no point in that cell
        const u64 entry = dir.ent[2 * slot + 1];
        if ((size_t)(uint32_t)entry >= i) continue;           // nothing earlier than i in that cell
        size_t a = (size_t)(entry >> 32);
        for (; a < count && gkey_sorted[a] == gk; ++a) {
            const size_t j = idx_sorted[a];
            if (j >= i) break;           // the sort is stable: a cell's run is in ascending point order
            double s = 0.0;
            for (int d = 0; d < n; ++d) { double df = __dsub_rn(pts[j * n + d], p[d]); s = __dadd_rn(s, __dmul_rn(df, df)); }
            if (sqrt(s) <= eps) {
                if (COLLECT) { nbr[nbc++] = (uint32_t)j; continue; }
                ++nbc;
                const uint8_t sj = ((volatile const uint8_t*)state)[j];
                if (sj == PT_DD_REMOVED) continue;
                if (sj == PT_DD_KEPT) { any_kept = true; break; }
                any_undecided = true;
            }
        }
    }
    return any_kept ? 2 : (any_undecided ? 1 : 0);
}

__global__ void pt_dedup_force_kernel(const int8_t* __restrict__ forced, size_t count, uint8_t* __restrict__ state) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count && forced[i] >= 0) state[i] = forced[i] ? PT_DD_KEPT : PT_DD_REMOVED;
}

__global__ void pt_dedup_round_kernel(int n, const double* __restrict__ pts, size_t count, double cell, double eps,
                                      const u64* __restrict__ gkey_sorted, const uint32_t* __restrict__ idx_sorted, PtTable dir,
                                      const uint32_t* __restrict__ bmp, u64 bmp_mask,
                                      uint8_t* state, uint32_t* __restrict__ undecided, uint32_t* __restrict__ nbc_out,
                                      PtFineCounters* ctr) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool pending = false;
    int nbc = 0;
    if (i < count && state[i] == PT_DD_UNDECIDED) {      // (pre-decided: states forced by the caller)
        const int verdict = pt_dedup_search<false>(n, pts, count, cell, eps, gkey_sorted, idx_sorted, dir, bmp, bmp_mask, state, i, nullptr, nbc);
        if (verdict == 2) state[i] = PT_DD_REMOVED;
        else if (verdict == 0) state[i] = PT_DD_KEPT;
        else pending = true;
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, pending);
    if (ballot) {
        const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&ctr->undecided, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (pending) {
            const unsigned long long pos = base + __popc(ballot & ((1u << lane) - 1u));
            undecided[pos] = (uint32_t)i; nbc_out[pos] = (uint32_t)nbc;
        }
    }
}

// neighbours of the listed points into csr[off[pos] ...] (same search, same order as the counting pass)
__global__ void pt_dedup_collect_kernel(int n, const double* __restrict__ pts, size_t count, double cell, double eps,
                                        const u64* __restrict__ gkey_sorted, const uint32_t* __restrict__ idx_sorted, PtTable dir,
                                        const uint32_t* __restrict__ bmp, u64 bmp_mask,
                                        const uint32_t* __restrict__ list, size_t list_count, const uint32_t* __restrict__ off,
                                        uint32_t* __restrict__ csr) {
    const size_t pos = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= list_count) return;
    int nbc;
    pt_dedup_search<true>(n, pts, count, cell, eps, gkey_sorted, idx_sorted, dir, bmp, bmp_mask, nullptr, (size_t)list[pos], csr + off[pos], nbc);
}

// one follow-up round over list positions: decided points drop out, the rest goes to list_out
__global__ void pt_dedup_follow_kernel(uint8_t* state, const uint32_t* __restrict__ point_of, const uint32_t* __restrict__ off,
                                       const uint32_t* __restrict__ csr, const uint32_t* __restrict__ list_in, size_t list_count,
                                       uint32_t* __restrict__ list_out, PtFineCounters* ctr) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool pending = false;
    uint32_t pos = 0;
    if (t < list_count) {
        pos = list_in[t];
        const uint32_t i = point_of[pos];
        bool any_kept = false, any_undecided = false;
        for (uint32_t q = off[pos]; q < off[pos + 1]; ++q) {
            const uint8_t sj = ((volatile const uint8_t*)state)[csr[q]];
            if (sj == PT_DD_KEPT) { any_kept = true; break; }
            if (sj != PT_DD_REMOVED) any_undecided = true;
        }
        if (any_kept) state[i] = PT_DD_REMOVED;
        else if (!any_undecided) state[i] = PT_DD_KEPT;
        else pending = true;
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, pending);
    if (ballot) {
        const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&ctr->undecided, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (pending) list_out[base + __popc(ballot & ((1u << lane) - 1u))] = pos;
    }
}

__global__ void pt_flag_kept_kernel(const uint8_t* __restrict__ state, size_t count, uint8_t* __restrict__ flag) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) flag[i] = state[i] == PT_DD_KEPT ? 1 : 0;
}
__global__ void pt_gather_points_kernel(int n, const double* __restrict__ pts, const u64* __restrict__ vals,
                                        const uint32_t* __restrict__ sel, size_t count, double* __restrict__ out_pts,
                                        long long* __restrict__ out_tag) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const size_t src = sel[i];
    for (int d = 0; d < n; ++d) out_pts[i * n + d] = pts[src * n + d];
    out_tag[i] = vals ? (long long)(vals[src] >> 1) : (long long)src;
}
__global__ void pt_iota32_kernel(uint32_t* out, size_t count) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = (uint32_t)i;
}
__global__ void pt_batch_bins_kernel(const long long* __restrict__ tags, size_t count, const unsigned long long* __restrict__ bounds,
                                     int nb, unsigned long long* __restrict__ bins) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const unsigned long long t = (unsigned long long)tags[i];
    int a = 0, b = nb;   // largest batch index with bounds[idx] <= t
    while (b - a > 1) { int mid = (a + b) >> 1; if (bounds[mid] <= t) a = mid; else b = mid; }
    atomicAdd(&bins[a], 1ull);
}
__global__ void pt_count_labels_kernel(const uint8_t* __restrict__ labels, size_t count, unsigned long long* out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hit = i < count && labels[i] != 0;
    unsigned b = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, (unsigned long long)__popc(b));
}

static int pt_read_fine_counters(pt_ctx* ctx, PtFineCounters* dev, PtFineCounters* host, const PtRefGeom& rg) {
    PT_CUDA(ctx, cudaMemcpyAsync(ctx->pinned, dev, sizeof(PtFineCounters), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(host, ctx->pinned, sizeof(PtFineCounters));
    if (host->error & PT_ERR_KEY_RANGE)
        return pt_fail(ctx, PT_E_RANGE, "fine lattice coordinates exceed the packed-key window (%d bits per axis at n=%d, k=%d)",
                       rg.fine.bits, rg.fine.n, rg.k);
    if (host->error & PT_ERR_TABLE_FULL) return pt_fail(ctx, PT_E_STATE, "hash table overflow (sizing bug)");
    return PT_OK;
}

// Greedy first-keeper dedup at eps over `U` points given in priority order, then collision labels.
// vals (optional) carries (tag << 1 | sign) per point; without it the tag is the input position.
static int pt_dedup_label_impl(pt_ctx* ctx, int n, const double* upts, const u64* vals, size_t U, double eps_dedup,
                               const pt_checker* checker, pt_refine* r, const int8_t* forced = nullptr) {
    PtBuf<PtFineCounters> ctr;
    PT_TRY(ctr.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(ctr.p, 0, sizeof(PtFineCounters), ctx->stream));
    PtFineCounters hc;
    PtRefGeom rg;
    memset(&rg, 0, sizeof(rg));
    rg.fine.n = n;
    PtBuf<uint8_t> state;
    PT_TRY(state.alloc(ctx, U > 0 ? U : 1));
    long long rounds = 0;
    size_t P = 0;
    PtBuf<uint32_t> sel;
    if (U > 0) {
        if (U >= (1ull << 32)) return pt_fail(ctx, PT_E_NOMEM, "more than 2^32 distinct fine edges in one refine call");
        PT_CUDA(ctx, cudaMemsetAsync(state.p, PT_DD_UNDECIDED, U, ctx->stream));
        if (forced) {
            // ghost copies of points another rank owns enter with that rank's verdict (multi-GPU eps-dedup)
            pt_dedup_force_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(forced, U, state.p);
            PT_TRY(pt_check_launch(ctx, "pt_dedup_force_kernel"));
        }
        // 8 eps cells: a point's eps-ball touches ~(1 + 1/4)^n cells (3.8 at n = 6) holding about one point each
        const double cell = 8.0 * eps_dedup;
        PtBuf<u64> gk, gks; PtBuf<uint32_t> gi, gis;
        PT_TRY(gk.alloc(ctx, U)); PT_TRY(gks.alloc(ctx, U)); PT_TRY(gi.alloc(ctx, U)); PT_TRY(gis.alloc(ctx, U));
        {
            PT_LAUNCH(ctx, "dedup_hash");
            pt_dedup_hash_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(n, upts, U, cell, gk.p, gi.p);
            PT_TRY(pt_check_launch(ctx, "pt_dedup_hash_kernel"));
        }
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, gk.p, gks.p, gi.p, gis.p, (long long)U, 0, 64, ctx->stream);
        PtBuf<uint8_t> tmp;
        PT_TRY(tmp.alloc(ctx, tb));
        {
            PT_LAUNCH(ctx, "dedup_sort");
            PT_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tb, gk.p, gks.p, gi.p, gis.p, (long long)U, 0, 64, ctx->stream));
            ctx->launches++;
        }
        PtHashTable dir;
        PT_TRY(pt_table_init(ctx, dir, 2 * (u64)U));
        // occupancy bitmap: the smallest power of two of at least 16 bits per point
        u64 bmp_bits = 1024;
        while (bmp_bits < 16 * (u64)U) bmp_bits <<= 1;
        const u64 bmp_mask = bmp_bits - 1;
        PtBuf<uint32_t> bmp;
        PT_TRY(bmp.alloc(ctx, bmp_bits / 32));
        PT_CUDA(ctx, cudaMemsetAsync(bmp.p, 0, bmp_bits / 8, ctx->stream));
        {
            PT_LAUNCH(ctx, "dedup_directory");
            pt_dedup_directory_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(gks.p, gis.p, U, dir.view(), bmp.p, bmp_mask, &ctr.p->error);
            PT_TRY(pt_check_launch(ctx, "pt_dedup_directory_kernel"));
        }
        PtBuf<uint32_t> point_of, nbc, off, csr, list_a, list_b;
        PT_TRY(point_of.alloc(ctx, U)); PT_TRY(nbc.alloc(ctx, U + 1));
        PT_CUDA(ctx, cudaMemsetAsync(&ctr.p->undecided, 0, sizeof(unsigned long long), ctx->stream));
        {
            PT_LAUNCH(ctx, "dedup_round");
            pt_dedup_round_kernel<<<pt_grid_for(U, 128), 128, 0, ctx->stream>>>(n, upts, U, cell, eps_dedup, gks.p, gis.p, dir.view(), bmp.p, bmp_mask, state.p,
                                                                                point_of.p, nbc.p, ctr.p);
            PT_TRY(pt_check_launch(ctx, "pt_dedup_round_kernel"));
        }
        ++rounds;
        PT_TRY(pt_read_fine_counters(ctx, ctr.p, &hc, rg));
        const size_t pending1 = (size_t)hc.undecided;
        if (pending1 > 0) {
            // CSR of the undecided points' earlier neighbours
            PT_TRY(off.alloc(ctx, pending1 + 1));
            PT_TRY(list_a.alloc(ctx, pending1)); PT_TRY(list_b.alloc(ctx, pending1));
            PT_CUDA(ctx, cudaMemsetAsync(nbc.p + pending1, 0, sizeof(uint32_t), ctx->stream));
            size_t tb3 = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb3, nbc.p, off.p, (int)(pending1 + 1), ctx->stream);
            PT_TRY(tmp.alloc(ctx, tb3));
            {
                PT_LAUNCH(ctx, "dedup_follow");
                PT_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp.p, tb3, nbc.p, off.p, (int)(pending1 + 1), ctx->stream));
                ctx->launches++;
            }
            uint32_t* h32 = (uint32_t*)ctx->pinned;
            PT_CUDA(ctx, cudaMemcpyAsync(h32, off.p + pending1, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            const size_t total_nbr = (size_t)*h32;
            PT_TRY(csr.alloc(ctx, total_nbr + 1));
            {
                PT_LAUNCH(ctx, "dedup_follow");
                pt_dedup_collect_kernel<<<pt_grid_for(pending1, 128), 128, 0, ctx->stream>>>(n, upts, U, cell, eps_dedup, gks.p, gis.p, dir.view(),
                                                                                             bmp.p, bmp_mask, point_of.p, pending1, off.p, csr.p);
                PT_TRY(pt_check_launch(ctx, "pt_dedup_collect_kernel"));
                pt_iota32_kernel<<<pt_grid_for(pending1, 256), 256, 0, ctx->stream>>>(list_a.p, pending1);
                PT_TRY(pt_check_launch(ctx, "pt_iota32_kernel"));
            }
            uint32_t* lin = list_a.p; uint32_t* lout = list_b.p;
            size_t pending = pending1;
            while (pending != 0) {
                PT_CUDA(ctx, cudaMemsetAsync(&ctr.p->undecided, 0, sizeof(unsigned long long), ctx->stream));
                {
                    PT_LAUNCH(ctx, "dedup_follow");
                    pt_dedup_follow_kernel<<<pt_grid_for(pending, 128), 128, 0, ctx->stream>>>(state.p, point_of.p, off.p, csr.p, lin, pending, lout, ctr.p);
                    PT_TRY(pt_check_launch(ctx, "pt_dedup_follow_kernel"));
                }
                ++rounds;
                PT_TRY(pt_read_fine_counters(ctx, ctr.p, &hc, rg));
                pending = (size_t)hc.undecided;
                uint32_t* sw = lin; lin = lout; lout = sw;
                if (rounds > 100000) return pt_fail(ctx, PT_E_STATE, "eps-dedup did not converge");
            }
        }
        // compact the kept points, order preserved
        PtBuf<uint8_t> flag; PtBuf<uint32_t> iota; PtBuf<long long> nsel;
        PT_TRY(flag.alloc(ctx, U)); PT_TRY(iota.alloc(ctx, U)); PT_TRY(sel.alloc(ctx, U)); PT_TRY(nsel.alloc(ctx, 1));
        pt_flag_kept_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(state.p, U, flag.p);
        PT_TRY(pt_check_launch(ctx, "pt_flag_kept_kernel"));
        pt_iota32_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(iota.p, U);
        PT_TRY(pt_check_launch(ctx, "pt_iota32_kernel"));
        size_t tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb2, iota.p, flag.p, sel.p, nsel.p, (long long)U, ctx->stream);
        PT_TRY(tmp.alloc(ctx, tb2));
        {
            PT_LAUNCH(ctx, "dedup_compact");
            PT_CUDA(ctx, cub::DeviceSelect::Flagged(tmp.p, tb2, iota.p, flag.p, sel.p, nsel.p, (long long)U, ctx->stream));
            ctx->launches++;
        }
        long long* h = (long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        P = (size_t)*h;
    }
    r->stats.dedup_rounds = rounds;
    r->n_points = (long long)P;
    r->stats.points = (long long)P;
    PT_TRY(r->points.alloc(ctx, (P > 0 ? P : 1) * n));
    PT_TRY(r->labels.alloc(ctx, P > 0 ? P : 1));
    PT_TRY(r->first_tag.alloc(ctx, P > 0 ? P : 1));
    if (P > 0) {
        PT_LAUNCH(ctx, "refine_gather");
        pt_gather_points_kernel<<<pt_grid_for(P, 256), 256, 0, ctx->stream>>>(n, upts, vals, sel.p, P, r->points.p, r->first_tag.p);
        PT_TRY(pt_check_launch(ctx, "pt_gather_points_kernel"));
    }

    // ---- R6: labels --------------------------------------------------------------------------
    PT_CUDA(ctx, cudaMemsetAsync(r->labels.p, 0, P > 0 ? P : 1, ctx->stream));
    if (checker && P > 0) {
        PT_TRY(pt_checker_run_dev(ctx, checker, r->points.p, P, PT_LIMIT_UNFREE, r->labels.p, nullptr));
        PtBuf<unsigned long long> nh;
        PT_TRY(nh.alloc(ctx, 1));
        PT_CUDA(ctx, cudaMemsetAsync(nh.p, 0, sizeof(unsigned long long), ctx->stream));
        pt_count_labels_kernel<<<pt_grid_for(P, 256), 256, 0, ctx->stream>>>(r->labels.p, P, nh.p);
        PT_TRY(pt_check_launch(ctx, "pt_count_labels_kernel"));
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, nh.p, sizeof(*h), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        r->stats.in_collision = (long long)*h;
        r->stats.free_points = (long long)P - r->stats.in_collision;
    } else {
        r->stats.free_points = (long long)P;
    }

    return PT_OK;
}

static int pt_refine_impl(pt_ctx* ctx, const pt_field* field, const pt_cells* cells, int n, double scale, const double* offset, int k,
                          int V, const int32_t* tv_host, int E, const int32_t* te_host, double eps, double eps_dedup,
                          const pt_checker* checker, const long long* batch_bounds, int nb, bool candidates_only,
                          pt_refine** out) {
    if (!ctx || !field || !cells || !out) return pt_fail(ctx, PT_E_INVALID, "pt_refine_run: NULL argument");
    if (cells->n != n || pt_field_dim(field) != n) return pt_fail(ctx, PT_E_INVALID, "template and lattice dimension mismatch");
    if (k < 1 || k > 64) return pt_fail(ctx, PT_E_INVALID, "subdivision factor must be in 1..64");
    if (V < 1 || V > PT_MAX_TV) return pt_fail(ctx, PT_E_INVALID, "template has %d vertices; this build supports up to %d", V, PT_MAX_TV);
    if (E < 0 || E > 32767) return pt_fail(ctx, PT_E_INVALID, "template has too many edges (%d)", E);
    if (!(eps > 0.0) || !(eps_dedup > 0.0)) return pt_fail(ctx, PT_E_INVALID, "eps and eps_dedup must be positive");
    if (!(scale > 0.0)) return pt_fail(ctx, PT_E_INVALID, "lattice scale must be positive");

    pt_refine* r = new pt_refine();
    r->ctx = ctx; r->n = n;
    memset(&r->stats, 0, sizeof(r->stats));
    struct Guard { pt_refine* r; bool keep = false; ~Guard() { if (!keep) delete r; } } guard{r};

    PtRefGeom rg;
    memset(&rg, 0, sizeof(rg));
    rg.coarse = cells->geom; rg.k = k; rg.V = V; rg.E = E; rg.W = (V + 31) / 32;
    rg.fine.n = n; rg.fine.bits = (63 - n) / n > 20 ? 20 : (63 - n) / n;
    rg.fine.scale = scale;
    for (int d = 0; d < n; ++d) {
        rg.fine.offset[d] = offset ? offset[d] : 0.0;
        rg.fine.origin[d] = k * cells->base_min[d] - 1;
        long long span = (long long)k * (cells->base_max[d] + 1) + 1 - rg.fine.origin[d];
        if (span >= (1ll << rg.fine.bits))
            return pt_fail(ctx, PT_E_RANGE, "fine lattice spans %lld units on axis %d; packed keys hold %lld at n=%d", span, d,
                           (1ll << rg.fine.bits), n);
    }
    const size_t C = (size_t)cells->count;
    r->stats.cells = (long long)C;
    r->stats.fine_vertices = (long long)C * V;
    r->batch_rows.assign((size_t)(nb > 0 ? nb : 0) * 2, 0);

    // template to the device (int8 coordinates, int16 edge indices)
    std::vector<int8_t> tv8((size_t)V * n);
    for (size_t i = 0; i < tv8.size(); ++i) tv8[i] = (int8_t)tv_host[i];
    std::vector<int16_t> te16((size_t)(E > 0 ? E : 1) * 2, 0);
    for (int e = 0; e < E; ++e) {
        if (te_host[2 * e] < 0 || te_host[2 * e] >= V || te_host[2 * e + 1] < 0 || te_host[2 * e + 1] >= V)
            return pt_fail(ctx, PT_E_INVALID, "template edge %d references a missing vertex", e);
        te16[2 * e] = (int16_t)te_host[2 * e]; te16[2 * e + 1] = (int16_t)te_host[2 * e + 1];
    }
    PtBuf<int8_t> tv; PtBuf<int16_t> te;
    PT_TRY(tv.alloc(ctx, tv8.size()));
    PT_TRY(te.alloc(ctx, te16.size()));
    PT_CUDA(ctx, cudaMemcpyAsync(tv.p, tv8.data(), tv8.size(), cudaMemcpyHostToDevice, ctx->stream));
    PT_CUDA(ctx, cudaMemcpyAsync(te.p, te16.data(), te16.size() * sizeof(int16_t), cudaMemcpyHostToDevice, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));

    PtBuf<PtFineCounters> ctr;
    PT_TRY(ctr.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(ctr.p, 0, sizeof(PtFineCounters), ctx->stream));
    PtFineCounters hc;
    memset(&hc, 0, sizeof(hc));

    PtHashTable fvt, fet;
    PT_TRY(pt_table_init(ctx, fvt, 1 << 16));
    PT_TRY(pt_table_init(ctx, fet, 1 << 16));

    // global crossing offsets (cell-major order)
    PtBuf<unsigned long long> ccount, coff;
    PT_TRY(ccount.alloc(ctx, C + 1));
    PT_TRY(coff.alloc(ctx, C + 1));
    PtBuf<uint32_t> csign;
    PT_TRY(csign.alloc(ctx, (C > 0 ? C : 1) * rg.W));

    // ---- pass 1 over cell batches: signs + crossing counts ------------------------------------
    size_t batch_cells = ((size_t)1 << 25) / (size_t)V;
    if (batch_cells < 4096) batch_cells = 4096;
    {
        PtBuf<uint32_t> vslot, pending; PtBuf<double> pts; PtBuf<int8_t> sg; PtBuf<float> vf;
        for (size_t c0 = 0; c0 < C; c0 += batch_cells) {
            const size_t bc = (C - c0) < batch_cells ? (C - c0) : batch_cells;
            PT_TRY(vslot.ensure(ctx, bc * V, 0));
            PT_TRY(pending.ensure(ctx, bc * V, 0));
            PT_TRY(pt_table_reserve(ctx, fvt, bc * V));
            PT_CUDA(ctx, cudaMemsetAsync(&ctr.p->n_pending, 0, sizeof(unsigned long long), ctx->stream));
            {
                PT_LAUNCH(ctx, "refine_vertices");
                pt_ref_vertices_kernel<<<pt_grid_for(bc * 32, 256), 256, 0, ctx->stream>>>(rg, fvt.view(), cells->keys.p + c0, bc, tv.p,
                                                                                             vslot.p, pending.p, ctr.p);
                PT_TRY(pt_check_launch(ctx, "pt_ref_vertices_kernel"));
            }
            PT_TRY(pt_read_fine_counters(ctx, ctr.p, &hc, rg));
            const size_t np = (size_t)hc.n_pending;
            if (np) {
                PT_TRY(pts.ensure(ctx, np * n, 0));
                PT_TRY(sg.ensure(ctx, np, 0));
                PT_TRY(vf.ensure(ctx, np, 0));
                {
                    PT_LAUNCH(ctx, "refine_pending_points");
                    pt_ref_pending_points_kernel<<<pt_grid_for(np, 256), 256, 0, ctx->stream>>>(rg, fvt.view(), pending.p, np, pts.p);
                    PT_TRY(pt_check_launch(ctx, "pt_ref_pending_points_kernel"));
                }
                {
                    PtAmbScope amb(ctx, &ctr.p->ambiguous);
                    PT_CUDA(ctx, cudaMemsetAsync(vf.p, 0, np * sizeof(float), ctx->stream));
                    PT_TRY(pt_field_eval_dev(ctx, field, pts.p, np, nullptr, sg.p, vf.p));
                }
                {
                    PT_LAUNCH(ctx, "refine_pending_store");
                    pt_ref_pending_store_kernel<<<pt_grid_for(np, 256), 256, 0, ctx->stream>>>(fvt.view(), pending.p, np, sg.p, vf.p);
                    PT_TRY(pt_check_launch(ctx, "pt_ref_pending_store_kernel"));
                }
                fvt.count += np;
                r->stats.unique_fine_vertices += (long long)np;
                r->stats.field_evaluations += (long long)np;
            }
            {
                PT_LAUNCH(ctx, "refine_signs");
                pt_ref_signs_kernel<<<pt_grid_for(bc * 32, 256), 256, 0, ctx->stream>>>(rg, fvt.view(), bc, te.p, vslot.p,
                                                                                          csign.p + c0 * rg.W, ccount.p + c0);
                PT_TRY(pt_check_launch(ctx, "pt_ref_signs_kernel"));
            }
        }
    }
    PT_CUDA(ctx, cudaMemsetAsync(ccount.p + C, 0, sizeof(unsigned long long), ctx->stream));
    PT_TRY(pt_read_fine_counters(ctx, ctr.p, &hc, rg));     // final ambiguous-sign count of pass 1
    r->stats.ambiguous_signs = (long long)hc.ambiguous;
    {
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, ccount.p, coff.p, (long long)(C + 1), ctx->stream);
        PtBuf<uint8_t> tmp;
        PT_TRY(tmp.alloc(ctx, tb));
        PT_LAUNCH(ctx, "refine_scan");
        PT_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp.p, tb, ccount.p, coff.p, (long long)(C + 1), ctx->stream));
        ctx->launches++;
    }
    unsigned long long total_cross = 0;
    {
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, coff.p + C, sizeof(*h), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        total_cross = *h;
    }
    r->stats.crossing_edges = (long long)total_cross;

    // ---- pass 2 over cell batches: distinct fine edges with first-occurrence tags --------------
    {
        // batches bounded by crossings so the table reservation stays proportionate
        std::vector<unsigned long long> hoff;
        const size_t step = batch_cells;
        for (size_t c0 = 0; c0 < C; c0 += step) {
            const size_t bc = (C - c0) < step ? (C - c0) : step;
            unsigned long long ends[2];
            PT_CUDA(ctx, cudaMemcpyAsync(&ends[0], coff.p + c0, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaMemcpyAsync(&ends[1], coff.p + c0 + bc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            const unsigned long long bcross = ends[1] - ends[0];
            if (bcross == 0) continue;
            PT_TRY(pt_table_reserve(ctx, fet, bcross));
            {
                PT_LAUNCH(ctx, "refine_edges");
                pt_ref_edges_kernel<<<pt_grid_for(bc * 32, 256), 256, 0, ctx->stream>>>(rg, fet.view(), cells->keys.p + c0, bc, tv.p, te.p,
                                                                                          csign.p + c0 * rg.W, coff.p + c0, 0ull, ctr.p);
                PT_TRY(pt_check_launch(ctx, "pt_ref_edges_kernel"));
            }
            PT_TRY(pt_read_fine_counters(ctx, ctr.p, &hc, rg));
            fet.count = hc.n_edges;
        }
    }
    const size_t U = (size_t)hc.n_edges;
    r->stats.unique_fine_edges = (long long)U;

    // ---- R4: order the distinct edges by first occurrence, bisect each once --------------------
    PtBuf<u64> vals, keys;
    PtBuf<double> upts;
    PT_TRY(upts.alloc(ctx, (U > 0 ? U : 1) * n));
    if (U > 0) {
        PtBuf<u64> vraw, kraw; PtBuf<unsigned long long> cnt;
        PT_TRY(vraw.alloc(ctx, U)); PT_TRY(kraw.alloc(ctx, U));
        PT_TRY(vals.alloc(ctx, U)); PT_TRY(keys.alloc(ctx, U));
        PT_TRY(cnt.alloc(ctx, 1));
        PT_CUDA(ctx, cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
        {
            PT_LAUNCH(ctx, "refine_extract");
            pt_ref_extract_kernel<<<pt_grid_for(fet.capacity, PT_EXTRACT_THREADS * PT_EXTRACT_PER_THREAD), PT_EXTRACT_THREADS, 0, ctx->stream>>>(fet.view(), vraw.p, kraw.p, cnt.p);
            PT_TRY(pt_check_launch(ctx, "pt_ref_extract_kernel"));
        }
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, vraw.p, vals.p, kraw.p, keys.p, (long long)U, 0, 64, ctx->stream);
        PtBuf<uint8_t> tmp;
        PT_TRY(tmp.alloc(ctx, tb));
        {
            PT_LAUNCH(ctx, "refine_sort_edges");
            PT_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tb, vraw.p, vals.p, kraw.p, keys.p, (long long)U, 0, 64, ctx->stream));
            ctx->launches++;
        }
        vraw.release(); kraw.release();
        fet.ent.release();
        const size_t chunk = (size_t)1 << 22;
        PtBuf<double> a, b; PtBuf<int8_t> sa; PtBuf<float> hint;
        PT_TRY(a.alloc(ctx, (U < chunk ? U : chunk) * n));
        PT_TRY(b.alloc(ctx, (U < chunk ? U : chunk) * n));
        PT_TRY(sa.alloc(ctx, (U < chunk ? U : chunk)));
        PT_TRY(hint.alloc(ctx, (U < chunk ? U : chunk)));
        for (size_t u0 = 0; u0 < U; u0 += chunk) {
            const size_t uc = (U - u0) < chunk ? (U - u0) : chunk;
            {
                PT_LAUNCH(ctx, "refine_endpoints");
                pt_ref_endpoints_kernel<<<pt_grid_for(uc, 256), 256, 0, ctx->stream>>>(rg, vals.p, keys.p, u0, uc, a.p, b.p, sa.p, fvt.view(), hint.p);
                PT_TRY(pt_check_launch(ctx, "pt_ref_endpoints_kernel"));
            }
            PT_TRY(pt_field_bisect_dev(ctx, field, a.p, b.p, sa.p, uc, eps, upts.p + u0 * n, hint.p));
        }
    }

    // ---- R5 + R6: greedy eps-dedup in first-occurrence order, labels --------------------------------
    if (candidates_only) {
        // hand back the root-solved points of the distinct fine edges (multi-GPU merge happens upstream)
        r->n_points = (long long)U;
        r->stats.points = (long long)U;
        PT_TRY(r->points.alloc(ctx, (U > 0 ? U : 1) * n));
        PT_TRY(r->labels.alloc(ctx, U > 0 ? U : 1));
        PT_TRY(r->first_tag.alloc(ctx, U > 0 ? U : 1));
        PT_CUDA(ctx, cudaMemsetAsync(r->labels.p, 0, U > 0 ? U : 1, ctx->stream));
        if (U > 0) {
            PtBuf<uint32_t> iota;
            PT_TRY(iota.alloc(ctx, U));
            pt_iota32_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(iota.p, U);
            PT_TRY(pt_check_launch(ctx, "pt_iota32_kernel"));
            pt_gather_points_kernel<<<pt_grid_for(U, 256), 256, 0, ctx->stream>>>(n, upts.p, vals.p, iota.p, U, r->points.p, r->first_tag.p);
            PT_TRY(pt_check_launch(ctx, "pt_gather_points_kernel"));
        }
    } else {
        PT_TRY(pt_dedup_label_impl(ctx, n, upts.p, vals.p, U, eps_dedup, checker, r));
    }

    // ---- per-batch statistics ------------------------------------------------------------------
    if (nb > 0 && batch_bounds) {
        std::vector<unsigned long long> hb((size_t)nb + 1);
        for (int i = 0; i <= nb; ++i) {
            long long cidx = batch_bounds[i];
            if (cidx < 0 || (size_t)cidx > C) return pt_fail(ctx, PT_E_INVALID, "batch boundary %lld out of range", cidx);
            PT_CUDA(ctx, cudaMemcpyAsync(&hb[(size_t)i], coff.p + cidx, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        }
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<unsigned long long> bins((size_t)nb, 0);
        const size_t P = (size_t)r->n_points;
        if (P > 0) {
            PtBuf<unsigned long long> db, dbins;
            PT_TRY(db.alloc(ctx, (size_t)nb + 1));
            PT_TRY(dbins.alloc(ctx, (size_t)nb));
            PT_CUDA(ctx, cudaMemcpyAsync(db.p, hb.data(), hb.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->stream));
            PT_CUDA(ctx, cudaMemsetAsync(dbins.p, 0, (size_t)nb * sizeof(unsigned long long), ctx->stream));
            pt_batch_bins_kernel<<<pt_grid_for(P, 256), 256, 0, ctx->stream>>>(r->first_tag.p, P, db.p, nb, dbins.p);
            PT_TRY(pt_check_launch(ctx, "pt_batch_bins_kernel"));
            PT_CUDA(ctx, cudaMemcpyAsync(bins.data(), dbins.p, (size_t)nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
            PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        }
        for (int i = 0; i < nb; ++i) {
            r->batch_rows[(size_t)2 * i] = (long long)(hb[(size_t)i + 1] - hb[(size_t)i]);
            r->batch_rows[(size_t)2 * i + 1] = (long long)bins[(size_t)i];
        }
    }
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    guard.keep = true;
    *out = r;
    return PT_OK;
}

extern "C" {

int pt_refine_run(pt_ctx* ctx, const pt_field* field, const pt_cells* cells, int n, double scale, const double* offset, int k,
                  int V, const int32_t* tv_host, int E, const int32_t* te_host, double eps, double eps_dedup,
                  const pt_checker* checker, const long long* batch_bounds, int nb, pt_refine** out) {
    return pt_refine_impl(ctx, field, cells, n, scale, offset, k, V, tv_host, E, te_host, eps, eps_dedup, checker,
                          batch_bounds, nb, false, out);
}

int pt_refine_candidates(pt_ctx* ctx, const pt_field* field, const pt_cells* cells, int n, double scale, const double* offset,
                         int k, int V, const int32_t* tv_host, int E, const int32_t* te_host, double eps, pt_refine** out) {
    return pt_refine_impl(ctx, field, cells, n, scale, offset, k, V, tv_host, E, te_host, eps, 1.0, nullptr, nullptr, 0, true, out);
}

int pt_dedup_label(pt_ctx* ctx, int n, const double* points, long long count, double eps_dedup, const pt_checker* checker,
                   pt_refine** out) {
    return pt_dedup_label_forced(ctx, n, points, count, eps_dedup, nullptr, checker, out);
}

int pt_dedup_label_forced(pt_ctx* ctx, int n, const double* points, long long count, double eps_dedup, const int8_t* forced,
                          const pt_checker* checker, pt_refine** out) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_dedup_label: NULL argument");
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", n);
    if (count < 0) return pt_fail(ctx, PT_E_INVALID, "negative point count");
    if (!(eps_dedup > 0.0)) return pt_fail(ctx, PT_E_INVALID, "eps_dedup must be positive");
    if (count > 0 && !points) return pt_fail(ctx, PT_E_INVALID, "points is NULL");
    pt_refine* r = new pt_refine();
    r->ctx = ctx; r->n = n;
    memset(&r->stats, 0, sizeof(r->stats));
    PtBuf<double> tmp;
    const double* pdev;
    PtBuf<int8_t> ftmp;
    const int8_t* fdev = nullptr;
    int rc = pt_stage_in(ctx, points, (size_t)count * n, tmp, &pdev);
    if (rc == PT_OK && forced && count > 0) rc = pt_stage_in(ctx, forced, (size_t)count, ftmp, &fdev);
    if (rc == PT_OK) rc = pt_dedup_label_impl(ctx, n, pdev, nullptr, (size_t)count, eps_dedup, checker, r, fdev);
    if (rc == PT_OK) rc = (cudaStreamSynchronize(ctx->stream) == cudaSuccess) ? PT_OK : pt_fail(ctx, PT_E_CUDA, "dedup failed");
    if (rc != PT_OK) { delete r; return rc; }
    *out = r;
    return PT_OK;
}

void pt_refine_destroy(pt_refine* r) { delete r; }

int pt_refine_get_stats(const pt_refine* r, pt_refine_stats* out) {
    if (!r || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_refine_get_stats: NULL argument");
    *out = r->stats;
    return PT_OK;
}

int pt_refine_points(const pt_refine* r, double* points, uint8_t* labels, long long* first_tag) {
    if (!r) return pt_fail(nullptr, PT_E_INVALID, "refine result is NULL");
    pt_ctx* ctx = r->ctx;
    const size_t P = (size_t)r->n_points;
    if (P == 0) return PT_OK;
    if (points) PT_TRY(pt_copy_out(ctx, points, r->points.p, P * r->n, false));
    if (labels) PT_TRY(pt_copy_out(ctx, labels, r->labels.p, P, false));
    if (first_tag) PT_TRY(pt_copy_out(ctx, first_tag, r->first_tag.p, P, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_refine_batch_stats(const pt_refine* r, long long* out, int nb) {
    if (!r || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_refine_batch_stats: NULL argument");
    size_t rows = r->batch_rows.size() / 2;
    if ((size_t)nb < rows) rows = (size_t)nb;
    memcpy(out, r->batch_rows.data(), rows * 2 * sizeof(long long));
    return PT_OK;
}

int pt_refine_set_labels(pt_refine* r, const uint8_t* labels) {
    if (!r) return pt_fail(nullptr, PT_E_INVALID, "refine result is NULL");
    pt_ctx* ctx = r->ctx;
    const size_t P = (size_t)r->n_points;
    if (P == 0) return PT_OK;
    if (!labels) return pt_fail(ctx, PT_E_INVALID, "labels is NULL");
    cudaMemcpyKind kind = pt_is_device_ptr(labels) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    PT_CUDA(ctx, cudaMemcpyAsync(r->labels.p, labels, P, kind, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    long long hits = 0;
    if (!pt_is_device_ptr(labels)) for (size_t i = 0; i < P; ++i) hits += labels[i] != 0;
    r->stats.in_collision = hits; r->stats.free_points = (long long)P - hits;
    return PT_OK;
}

}  // extern "C"
