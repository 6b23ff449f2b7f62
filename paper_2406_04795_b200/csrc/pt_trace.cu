// Batched BFS manifold tracing on the Freudenthal-Kuhn lattice (tracer.py:152-452).
//
// One wave (= _Tracer.expand, tracer.py:322-380) over a chunk of frontier edges:
//   pt_wave_probe_kernel    warp per frontier edge enumerates its 2-simplex cofaces, inserts the third
//                           vertices into the vertex-sign table, queues the unknown ones
//   (field evaluation of the queued vertices -- _ensure_signs, tracer.py:195-209)
//   pt_wave_partner_kernel  partner rule + box clamp + visited insert with atomicMin(slot id)
//   pt_wave_count_kernel    winners (first occurrence in slot order) per frontier edge
//   pt_wave_admit_kernel    admission in slot order: edge index = visited + rank (tracer.py:239-252)
// Slot id = frontier position * stride + coface ordinal reproduces the reference's admission order.
#include <cub/cub.cuh>
#include <limits.h>
#include "pt_trace.cuh"
#include "pt_field.cuh"

#define PT_NONE32 0xFFFFFFFFu

int pt_bits_for_dim(int n) {
    int b = (63 - PT_CELL_RANK_BITS) / n;
    return b > 20 ? 20 : b;
}

// ---- table management ----------------------------------------------------------------------
__global__ void pt_rehash_kernel(PtTable src, PtTable dst, unsigned* err) {
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > src.cap_mask) return;
    u64 key = src.ent[2 * i];
    if (key == PT_EMPTY) return;
    bool ins;
    u64 slot = pt_table_insert(dst, key, ins, err);
    dst.ent[2 * slot + 1] = src.ent[2 * i + 1];
}

int pt_table_init(pt_ctx* ctx, PtHashTable& t, u64 capacity) {
    u64 cap = 1024;
    while (cap < capacity) cap <<= 1;
    PT_TRY(t.ent.alloc(ctx, 2 * cap));
    PT_CUDA(ctx, cudaMemsetAsync(t.ent.p, 0xFF, 2 * cap * sizeof(u64), ctx->stream));
    t.capacity = cap; t.count = 0;
    return PT_OK;
}

int pt_table_reserve(pt_ctx* ctx, PtHashTable& t, u64 extra) {
    // worst case every one of `extra` probes inserts a new key: the table must never fill up
    // (count + extra <= capacity); the usual case inserts far fewer, keep the load at <= 1/2 for it
    u64 need = t.count + extra + (t.count + extra) / 8;
    if (need < 2 * t.count + 1024) need = 2 * t.count + 1024;
    if (need <= t.capacity) return PT_OK;
    u64 cap = t.capacity;
    while (cap < need) cap <<= 1;
    if (cap > (1ull << 31)) return pt_fail(ctx, PT_E_NOMEM, "hash table would exceed 2^31 entries");
    PtBuf<u64> fresh;
    PT_TRY(fresh.alloc(ctx, 2 * cap));
    PT_CUDA(ctx, cudaMemsetAsync(fresh.p, 0xFF, 2 * cap * sizeof(u64), ctx->stream));
    PtTable dst; dst.ent = fresh.p; dst.cap_mask = cap - 1;
    PtBuf<unsigned> err;
    PT_TRY(err.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(err.p, 0, sizeof(unsigned), ctx->stream));
    {
        PT_LAUNCH(ctx, "table_rehash");
        pt_rehash_kernel<<<pt_grid_for(t.capacity, 256), 256, 0, ctx->stream>>>(t.view(), dst, err.p);
        PT_TRY(pt_check_launch(ctx, "pt_rehash_kernel"));
    }
    // swap storage
    u64* old = t.ent.p;
    t.ent.p = fresh.p; t.ent.count = 2 * cap; t.ent.ctx = ctx;
    fresh.p = old; fresh.count = 2 * t.capacity; fresh.ctx = ctx;
    t.capacity = cap;
    return PT_OK;
}

// ---- small helpers -------------------------------------------------------------------------
__device__ __forceinline__ void pt_vertex_point(const PtGeom& g, const int* v, double* x) {
    // numpy: asarray(v, f64) * scale + offset, two roundings (tracer.py:204)
    for (int d = 0; d < g.n; ++d) x[d] = __dadd_rn(__dmul_rn((double)v[d], g.scale), g.offset[d]);
}

// warp-aggregated counter bump; returns this lane's position (valid where pred)
__device__ __forceinline__ unsigned long long pt_warp_append(unsigned long long* counter, bool pred) {
    unsigned ballot = __ballot_sync(0xffffffffu, pred);
    if (ballot == 0) return 0;
    int lane = threadIdx.x & 31;
    int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + (unsigned long long)__popc(ballot & ((1u << lane) - 1u));
}

// ---- locate (tracer.py:256-301) ---------------------------------------------------------------
// locate_point (lattice.py:135-153): base = floor((p - offset)/scale); labels by (-frac, index)
__global__ void pt_locate_cells_kernel(PtGeom g, const double* __restrict__ seeds, size_t m,
                                       int* __restrict__ cell_base, uint8_t* __restrict__ cell_perm) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double frac[PT_NMAX]; uint8_t ord[PT_NMAX];
    for (int d = 0; d < g.n; ++d) {
        double y = __ddiv_rn(__dsub_rn(seeds[i * g.n + d], g.offset[d]), g.scale);
        double b = floor(y);
        frac[d] = __dsub_rn(y, b);
        cell_base[i * g.n + d] = (int)b;
        ord[d] = (uint8_t)d;
    }
    // stable insertion sort, descending fraction (ties keep ascending index)
    for (int a = 1; a < g.n; ++a) {
        uint8_t key = ord[a]; int b = a - 1;
        while (b >= 0 && frac[ord[b]] < frac[key]) { ord[b + 1] = ord[b]; --b; }
        ord[b + 1] = key;
    }
    for (int d = 0; d < g.n; ++d) cell_perm[i * g.n + d] = ord[d];
}

// insert the n+1 vertices of each seed cell into the sign table, queue unknown ones
__global__ void pt_cell_vertices_kernel(PtGeom g, PtTable sgn, const int* __restrict__ cell_base,
                                        const uint8_t* __restrict__ cell_perm, size_t m,
                                        uint32_t* __restrict__ pending, PtCounters* ctr) {
    size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t i = tid / (g.n + 1);
    int j = (int)(tid % (g.n + 1));
    bool live = i < m;
    bool inserted = false; u64 slot = 0;
    if (live) {
        int v[PT_NMAX];
        for (int d = 0; d < g.n; ++d) v[d] = cell_base[i * g.n + d];
        for (int a = 0; a < j; ++a) v[cell_perm[i * g.n + a]] += 1;
        u64 key;
        if (!pt_pack_vertex(g, v, key)) atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
        else slot = pt_table_insert(sgn, key, inserted, &ctr->error);
    }
    unsigned long long pos = pt_warp_append(&ctr->n_pending, inserted);
    if (inserted) pending[pos] = (uint32_t)slot;
}

// cell_edges stage (tracer.py:272-285): sign-changing in-box edges of each seed cell, slot order
// = (cell, pair ordinal) with pairs (a<b), a outer (lattice.py:182-193)
__global__ void pt_cell_edges_kernel(PtGeom g, PtTable sgn, PtTable vis, const int* __restrict__ cell_base,
                                     const uint8_t* __restrict__ cell_perm, size_t m, int bound,
                                     uint32_t* __restrict__ vis_slot, PtCounters* ctr) {
    size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t i = tid / bound;
    int ord = (int)(tid % bound);
    if (i >= m) return;
    // ordinal -> (a, b)
    int a = 0, rem = ord;
    while (rem >= g.n - a) { rem -= g.n - a; ++a; }
    int b = a + 1 + rem;
    int va[PT_NMAX], vb[PT_NMAX];
    for (int d = 0; d < g.n; ++d) va[d] = cell_base[i * g.n + d];
    for (int k = 0; k < a; ++k) va[cell_perm[i * g.n + k]] += 1;
    uint32_t mask = 0;
    for (int d = 0; d < g.n; ++d) vb[d] = va[d];
    for (int k = a; k < b; ++k) { int lab = cell_perm[i * g.n + k]; vb[lab] += 1; mask |= 1u << lab; }
    u64 ka, kb;
    uint32_t marker = PT_NONE32;
    if (pt_pack_vertex(g, va, ka) && pt_pack_vertex(g, vb, kb)) {
        u64 sa_slot, sb_slot;
        if (pt_table_find(sgn, ka, sa_slot) && pt_table_find(sgn, kb, sb_slot)) {
            const int sa = pt_ld_cg(&sgn.ent[2 * sa_slot + 1]) ? 1 : -1;
            const int sb = pt_ld_cg(&sgn.ent[2 * sb_slot + 1]) ? 1 : -1;
            if (sa != sb) {
                atomicAdd(&ctr->markers, 1ull);
                if (pt_in_box(g, va) && pt_in_box(g, vb)) {
                    bool ins;
                    u64 slot = pt_table_insert(vis, pt_edge_key(g, ka, mask), ins, &ctr->error);
                    const u64 mine = PT_VAL_PENDING_BASE + (u64)tid;
                    if (atomicMin(&vis.ent[2 * slot + 1], mine) > mine) marker = (uint32_t)slot | (sa > 0 ? 0x80000000u : 0u);
                } else {
                    atomicAdd(&ctr->dropped, 1ull);
                }
            }
        }
    } else {
        atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
    }
    vis_slot[tid] = marker;
}

// ---- pending vertex evaluation --------------------------------------------------------------
__global__ void pt_pending_points_kernel(PtGeom g, PtTable sgn, const uint32_t* __restrict__ pending, size_t count,
                                         double* __restrict__ pts) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    u64 key = sgn.ent[2 * (u64)pending[i]];
    int v[PT_NMAX]; double x[PT_NMAX];
    pt_unpack_vertex(g, key, v);
    pt_vertex_point(g, v, x);
    for (int d = 0; d < g.n; ++d) pts[i * g.n + d] = x[d];
}
__global__ void pt_pending_store_kernel(PtTable sgn, const uint32_t* __restrict__ pending, size_t count,
                                        const int8_t* __restrict__ s) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    sgn.ent[2 * (u64)pending[i] + 1] = s[i] > 0 ? 1ull : 0ull;
}

// ---- wave kernels ----------------------------------------------------------------------------
// Packed-key arithmetic for the wave kernels.  Every vertex a frontier edge (u, s) touches is u + 1_P - 1_M with disjoint
// coordinate sets P, M (its cofaces' third vertices and partner-edge end points), so with
//   * the packed key of u,
//   * a per-block table `pk[mask]` = packed image of a 0/1 coordinate mask (shared memory, 2^n entries),
//   * two per-edge bit sets: the coordinates where u sits on the upper / lower face of the clamp box,
// a candidate costs a few adds and bit tests instead of unpacking into runtime-indexed int arrays (local memory):
//   key(u + 1_P - 1_M) = key(u) + pk[P] - pk[M]     (no carry crosses a field while every coordinate stays in the window)
//   in box  <=>  P misses the upper-face set and M misses the lower-face set.
// `safe` (all coordinates of u at least one unit inside the key window) guards the arithmetic; the few edges on the window
// border take the array path below.
struct PtEdgeFast { u64 vk; uint32_t at_hi, at_lo; bool safe; };

__device__ __forceinline__ void pt_fill_packmask(const PtGeom& g, u64* pk) {
    for (uint32_t m = threadIdx.x; m < (1u << g.n); m += blockDim.x) pk[m] = pt_mask_to_packed(g, m);
}

__device__ __forceinline__ PtEdgeFast pt_edge_fast(const PtGeom& g, u64 ek) {
    PtEdgeFast e;
    e.vk = pt_edge_vkey(g, ek);
    e.at_hi = 0; e.at_lo = 0; e.safe = true;
    const u64 fm = (1ull << g.bits) - 1ull;
    u64 k = e.vk;
    for (int d = g.n - 1; d >= 0; --d) {
        const int r = (int)(k & fm);
        k >>= g.bits;
        e.safe = e.safe && r >= 1 && r <= (int)fm - 1;
        if (g.has_box) {
            const int v = r + g.origin[d];
            if (v >= g.box_hi[d]) e.at_hi |= 1u << d;
            if (v <= g.box_lo[d]) e.at_lo |= 1u << d;
        }
    }
    return e;
}

__global__ void __launch_bounds__(256)
pt_wave_probe_kernel(PtGeom g, PtTable sgn, const u64* __restrict__ edge_key, const uint32_t* __restrict__ frontier,
                     size_t fcount, int stride, uint32_t* __restrict__ sgn_slot, uint32_t* __restrict__ pending,
                     PtCounters* ctr) {
    __shared__ u64 pk[1 << PT_NMAX];
    pt_fill_packmask(g, pk);
    __syncthreads();
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= fcount) return;
    const u64 ek = edge_key[frontier[w]];
    const uint32_t s = pt_edge_mask(g, ek);
    const PtEdgeFast ef = pt_edge_fast(g, ek);
    const int nc = pt_ncofaces(g.n, s);
    if (lane == 0) atomicAdd(&ctr->candidates, (unsigned long long)nc);
    for (int j0 = 0; j0 < nc; j0 += 32) {
        const int j = j0 + lane;
        bool inserted = false; u64 slot = 0;
        if (j < nc) {
            PtCoface f = pt_coface(g.n, s, j);
            if (ef.safe) {
                slot = pt_table_insert(sgn, ef.vk + pk[f.c_plus] - pk[f.c_minus], inserted, &ctr->error);
            } else {
                int u[PT_NMAX], c[PT_NMAX];
                pt_unpack_vertex(g, ef.vk, u);
                pt_apply_masks(g.n, u, f.c_plus, f.c_minus, c);
                u64 ck;
                if (!pt_pack_vertex(g, c, ck)) atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
                else slot = pt_table_insert(sgn, ck, inserted, &ctr->error);
            }
            sgn_slot[w * stride + j] = (uint32_t)slot;
        }
        unsigned long long pos = pt_warp_append(&ctr->n_pending, inserted);
        if (inserted) pending[pos] = (uint32_t)slot;
    }
}

// new canonical edge produced by coface j of edge (u, s, sa) given sign(c) = sc (tracer.py:340-350)
struct PtPartner { int base[PT_NMAX]; uint32_t mask; int sign_base; };
__device__ __forceinline__ PtPartner pt_partner(int n, const int* u, uint32_t s, int sa, int j, int sc) {
    PtCoface f = pt_coface(n, s, j);
    PtPartner p;
    if (sc == sa) {   // (b, c) crosses; shared endpoint b carries -sa
        pt_apply_masks(n, u, f.bc_bplus, f.bc_bminus, p.base);
        p.mask = f.bc_mask;
        p.sign_base = f.bc_shared ? -sa : sc;
    } else {          // (a, c) crosses; shared endpoint a carries sa
        pt_apply_masks(n, u, f.ac_bplus, f.ac_bminus, p.base);
        p.mask = f.ac_mask;
        p.sign_base = f.ac_shared ? sa : sc;
    }
    return p;
}

__global__ void __launch_bounds__(256)
pt_wave_partner_kernel(PtGeom g, PtTable sgn, PtTable vis, const u64* __restrict__ edge_key,
                       const int8_t* __restrict__ edge_sa, const uint32_t* __restrict__ frontier, size_t fcount,
                       int stride, const uint32_t* __restrict__ sgn_slot, uint32_t* __restrict__ vis_slot,
                       PtCounters* ctr) {
    __shared__ u64 pk[1 << PT_NMAX];
    pt_fill_packmask(g, pk);
    __syncthreads();
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= fcount) return;
    const uint32_t e = frontier[w];
    const u64 ek = edge_key[e];
    const int sa = edge_sa[e];
    const uint32_t s = pt_edge_mask(g, ek);
    const PtEdgeFast ef = pt_edge_fast(g, ek);
    const int nc = pt_ncofaces(g.n, s);
    for (int j0 = 0; j0 < stride; j0 += 32) {
        const int j = j0 + lane;
        uint32_t marker = PT_NONE32;
        bool dropped = false;
        if (j < nc) {
            const int sc = pt_ld_cg(&sgn.ent[2 * (u64)sgn_slot[w * stride + j] + 1]) ? 1 : -1;
            u64 bk = 0; uint32_t pmask = 0; int sign_base = 0; bool ok = true;
            if (ef.safe) {
                // partner edge (tracer.py:340-350): base = u + 1_bplus - 1_bminus, other end = base + 1_mask; both are
                // u plus / minus disjoint coordinate sets, so the box test is two bit tests
                const PtCoface f = pt_coface(g.n, s, j);
                uint32_t bplus, bminus;
                if (sc == sa) { bplus = f.bc_bplus; bminus = f.bc_bminus; pmask = f.bc_mask; sign_base = f.bc_shared ? -sa : sc; }
                else { bplus = f.ac_bplus; bminus = f.ac_bminus; pmask = f.ac_mask; sign_base = f.ac_shared ? sa : sc; }
                const uint32_t up = bplus | (pmask & ~bminus), down = bminus & ~pmask;      // all vertices: u + 1_up' - 1_down', up' <= up
                if (((bplus | up) & ef.at_hi) || ((bminus | down) & ef.at_lo)) dropped = true;
                else bk = ef.vk + pk[bplus] - pk[bminus];
            } else {
                int u[PT_NMAX];
                pt_unpack_vertex(g, ef.vk, u);
                PtPartner p = pt_partner(g.n, u, s, sa, j, sc);
                int other[PT_NMAX];
                pt_apply_masks(g.n, p.base, p.mask, 0u, other);
                pmask = p.mask; sign_base = p.sign_base;
                if (!(pt_in_box(g, p.base) && pt_in_box(g, other))) dropped = true;
                else if (!pt_pack_vertex(g, p.base, bk)) { atomicOr(&ctr->error, PT_ERR_KEY_RANGE); ok = false; }
            }
            if (!dropped && ok) {
                bool ins;
                u64 slot = pt_table_insert(vis, pt_edge_key(g, bk, pmask), ins, &ctr->error);
                const u64 mine = PT_VAL_PENDING_BASE + (u64)(w * stride + j);
                const u64 old = atomicMin(&vis.ent[2 * slot + 1], mine);
                // an already admitted edge or a smaller pending slot beats this candidate for good:
                // only candidates that lowered the value stay in the winner scan
                if (old > mine) marker = (uint32_t)slot | (sign_base > 0 ? 0x80000000u : 0u);
            }
        }
        unsigned db = __ballot_sync(0xffffffffu, dropped);
        if (lane == 0 && db) atomicAdd(&ctr->dropped, (unsigned long long)__popc(db));
        if (j < stride) vis_slot[w * stride + j] = marker;
    }
}

// winners of each item (frontier edge or seed cell): val still equals this slot's pending id
__global__ void __launch_bounds__(256)
pt_wave_count_kernel(PtTable vis, size_t items, int stride, const uint32_t* __restrict__ vis_slot,
                     uint32_t* __restrict__ wcount) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= items) return;
    int count = 0;
    for (int j0 = 0; j0 < stride; j0 += 32) {
        const int j = j0 + lane;
        bool win = false;
        if (j < stride) {
            uint32_t mk = vis_slot[w * stride + j];
            if (mk != PT_NONE32)
                win = pt_ld_cg(&vis.ent[2 * (u64)(mk & 0x7fffffffu) + 1]) == PT_VAL_PENDING_BASE + (u64)(w * stride + j);
        }
        count += __popc(__ballot_sync(0xffffffffu, win));
    }
    if (lane == 0) wcount[w] = (uint32_t)count;
}

__global__ void __launch_bounds__(256)
pt_wave_admit_kernel(PtTable vis, size_t items, int stride, const uint32_t* __restrict__ vis_slot,
                     const uint32_t* __restrict__ woff, long long n_edges, long long max_edges,
                     u64* __restrict__ edge_key, int8_t* __restrict__ edge_sa) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= items) return;
    long long running = n_edges + (long long)woff[w];
    for (int j0 = 0; j0 < stride; j0 += 32) {
        const int j = j0 + lane;
        bool win = false; uint32_t mk = PT_NONE32;
        if (j < stride) {
            mk = vis_slot[w * stride + j];
            if (mk != PT_NONE32)
                win = pt_ld_cg(&vis.ent[2 * (u64)(mk & 0x7fffffffu) + 1]) == PT_VAL_PENDING_BASE + (u64)(w * stride + j);
        }
        unsigned ballot = __ballot_sync(0xffffffffu, win);
        if (win) {
            const long long idx = running + __popc(ballot & ((1u << lane) - 1u));
            const u64 slot = (u64)(mk & 0x7fffffffu);
            if (idx < max_edges) {
                edge_key[idx] = vis.ent[2 * slot];
                edge_sa[idx] = (mk & 0x80000000u) ? (int8_t)1 : (int8_t)-1;
                vis.ent[2 * slot + 1] = (u64)idx;
            } else {
                vis.ent[2 * slot + 1] = PT_VAL_DEAD;
            }
        }
        running += __popc(ballot);
    }
}

__global__ void pt_iota_kernel(uint32_t* out, size_t count, uint32_t first) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = first + (uint32_t)i;
}

// ---- host orchestration ----------------------------------------------------------------------
int pt_read_counters(pt_trace* t) {
    pt_ctx* ctx = t->ctx;
    PT_CUDA(ctx, cudaMemcpyAsync(ctx->pinned, t->counters.p, sizeof(PtCounters), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(&t->host_counters, ctx->pinned, sizeof(PtCounters));
    if (t->host_counters.error & PT_ERR_KEY_RANGE)
        return pt_fail(ctx, PT_E_RANGE, "lattice coordinates left the packed-key window (%d bits per axis at n=%d)",
                       t->geom.bits, t->geom.n);
    if (t->host_counters.error & PT_ERR_TABLE_FULL) return pt_fail(ctx, PT_E_STATE, "hash table overflow (sizing bug)");
    return PT_OK;
}

static int pt_reset_pending(pt_trace* t) {
    // n_pending is the first field of PtCounters
    PT_CUDA(t->ctx, cudaMemsetAsync(t->counters.p, 0, sizeof(unsigned long long), t->ctx->stream));
    return PT_OK;
}

// evaluate the `count` queued vertices (slots in `pending`) and store their signs
static int pt_eval_pending(pt_trace* t, const uint32_t* pending, size_t count) {
    if (count == 0) return PT_OK;
    pt_ctx* ctx = t->ctx;
    PtBuf<double> pts; PtBuf<int8_t> sg;
    PT_TRY(pts.alloc(ctx, count * t->geom.n));
    PT_TRY(sg.alloc(ctx, count));
    {
        PT_LAUNCH(ctx, "trace_pending_points");
        pt_pending_points_kernel<<<pt_grid_for(count, 256), 256, 0, ctx->stream>>>(t->geom, t->signs.view(), pending, count, pts.p);
        PT_TRY(pt_check_launch(ctx, "pt_pending_points_kernel"));
    }
    {
        PtAmbScope amb(ctx, &t->counters.p->ambiguous);
        PT_TRY(pt_field_eval_dev(ctx, t->field, pts.p, count, nullptr, sg.p));
    }
    {
        PT_LAUNCH(ctx, "trace_pending_store");
        pt_pending_store_kernel<<<pt_grid_for(count, 256), 256, 0, ctx->stream>>>(t->signs.view(), pending, count, sg.p);
        PT_TRY(pt_check_launch(ctx, "pt_pending_store_kernel"));
    }
    t->field_evaluations += (long long)count;
    t->signs.count += count;
    return PT_OK;
}

// count winners, scan, admit; returns number admitted (after the cap)
static int pt_admit_items(pt_trace* t, size_t items, int stride, const uint32_t* vis_slot, long long* admitted,
                          long long* winners = nullptr) {
    pt_ctx* ctx = t->ctx;
    *admitted = 0;
    if (winners) *winners = 0;
    if (items == 0) return PT_OK;
    PtBuf<uint32_t> wcount, woff;
    PT_TRY(wcount.alloc(ctx, items + 1));
    PT_TRY(woff.alloc(ctx, items + 1));
    PT_CUDA(ctx, cudaMemsetAsync(wcount.p + items, 0, sizeof(uint32_t), ctx->stream));
    {
        PT_LAUNCH(ctx, "trace_wave_count");
        pt_wave_count_kernel<<<pt_grid_for(items * 32, 256), 256, 0, ctx->stream>>>(t->visited.view(), items, stride, vis_slot, wcount.p);
        PT_TRY(pt_check_launch(ctx, "pt_wave_count_kernel"));
    }
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, wcount.p, woff.p, (int)(items + 1), ctx->stream);
    PtBuf<uint8_t> tmp;
    PT_TRY(tmp.alloc(ctx, tmp_bytes));
    {
        PT_LAUNCH(ctx, "trace_wave_scan");
        PT_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, wcount.p, woff.p, (int)(items + 1), ctx->stream));
        ctx->launches++;
    }
    uint32_t* h = (uint32_t*)ctx->pinned;
    PT_CUDA(ctx, cudaMemcpyAsync(h, woff.p + items, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const long long total = (long long)*h;
    if (winners) *winners = total;
    t->visited.count += (u64)total;   // every winner owns a fresh table entry (admitted or dead)
    if (total == 0) return PT_OK;
    long long room = t->max_edges - t->n_edges;
    if (room < 0) room = 0;
    const long long take = total < room ? total : room;
    if (take < total) t->complete = false;
    PT_TRY(t->edge_key.ensure(ctx, (size_t)(t->n_edges + take + 1), (size_t)t->n_edges));
    PT_TRY(t->edge_sa.ensure(ctx, (size_t)(t->n_edges + take + 1), (size_t)t->n_edges));
    {
        PT_LAUNCH(ctx, "trace_wave_admit");
        pt_wave_admit_kernel<<<pt_grid_for(items * 32, 256), 256, 0, ctx->stream>>>(
            t->visited.view(), items, stride, vis_slot, woff.p, t->n_edges, t->max_edges, t->edge_key.p, t->edge_sa.p);
        PT_TRY(pt_check_launch(ctx, "pt_wave_admit_kernel"));
    }
    t->n_edges += take;
    *admitted = take;
    return PT_OK;
}

// bounding box of the seeds' lattice cells: out[d] = min, out[PT_NMAX + d] = max, out[2 PT_NMAX] = 1 if a coordinate is not finite
__global__ void pt_seed_bounds_kernel(PtGeom g, const double* __restrict__ seeds, size_t m, int* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int d = 0; d < g.n; ++d) {
        const double y = (seeds[i * g.n + d] - g.offset[d]) / g.scale;
        if (!(y == y) || y > 1e9 || y < -1e9) { out[2 * PT_NMAX] = 1; continue; }
        const int c = (int)floor(y);
        atomicMin(&out[d], c);
        atomicMax(&out[PT_NMAX + d], c);
    }
}

static int pt_set_window(pt_trace* t, const int* first_cell_base) {
    PtGeom& g = t->geom;
    if (g.has_box) {
        for (int d = 0; d < g.n; ++d) {
            g.origin[d] = g.box_lo[d] - 2;
            long long span = (long long)g.box_hi[d] + 2 - g.origin[d];
            if (span >= (1ll << g.bits))
                return pt_fail(t->ctx, PT_E_RANGE, "clamp box spans %lld lattice units on axis %d; packed keys hold %lld at n=%d",
                               span, d, (1ll << g.bits), g.n);
        }
    } else {
        for (int d = 0; d < g.n; ++d) g.origin[d] = first_cell_base[d] - (1 << (g.bits - 1));
    }
    t->window_set = true;
    return PT_OK;
}

static int pt_stride_for(int n) {
    // max over edge types of (2^m1 - 2) + (2^(n+1-m1) - 2): attained at m1 = 1 or n
    return (1 << n) - 2;
}

static int pt_set_range_frontier(pt_trace* t, long long first, long long count) {
    pt_ctx* ctx = t->ctx;
    PT_TRY(t->frontier.ensure(ctx, (size_t)(count > 0 ? count : 1), 0));
    if (count > 0) {
        pt_iota_kernel<<<pt_grid_for((size_t)count, 256), 256, 0, ctx->stream>>>(t->frontier.p, (size_t)count, (uint32_t)first);
        PT_TRY(pt_check_launch(ctx, "pt_iota_kernel"));
    }
    t->n_frontier = count;
    t->range_frontier = true;
    return PT_OK;
}

static int pt_trace_locate_impl(pt_trace* t, const double* seeds, long long m) {
    pt_ctx* ctx = t->ctx;
    PtGeom& g = t->geom;
    const int n = g.n;
    if (m <= 0 || !seeds) return pt_fail(ctx, PT_E_INVALID, "seeds must be a non-empty (m, n) array");
    PtBuf<double> tmp;
    const double* sdev;
    PT_TRY(pt_stage_in(ctx, seeds, (size_t)m * n, tmp, &sdev));
    if (!t->window_set) {
        // without a clamp box the key window is centred on the bounding box of ALL seed cells (a zero set narrower than
        // the window then fits wherever the first seed happens to sit on it)
        PtBuf<int> bounds;
        PT_TRY(bounds.alloc(ctx, 2 * PT_NMAX + 1));
        int init[2 * PT_NMAX + 1];
        for (int d = 0; d < PT_NMAX; ++d) { init[d] = INT_MAX; init[PT_NMAX + d] = INT_MIN; }
        init[2 * PT_NMAX] = 0;
        PT_CUDA(ctx, cudaMemcpyAsync(bounds.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
        pt_seed_bounds_kernel<<<pt_grid_for((size_t)m, 256), 256, 0, ctx->stream>>>(g, sdev, (size_t)m, bounds.p);
        PT_TRY(pt_check_launch(ctx, "pt_seed_bounds_kernel"));
        PT_CUDA(ctx, cudaMemcpyAsync(init, bounds.p, sizeof(init), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (init[2 * PT_NMAX]) return pt_fail(ctx, PT_E_INVALID, "point coordinates must be finite");
        int cb[PT_NMAX];
        for (int d = 0; d < n; ++d) cb[d] = (int)(((long long)init[d] + (long long)init[PT_NMAX + d]) >> 1);
        PT_TRY(pt_set_window(t, cb));
    }
    t->seeds += m;
    PtBuf<int> cell_base; PtBuf<uint8_t> cell_perm;
    PT_TRY(cell_base.alloc(ctx, (size_t)m * n));
    PT_TRY(cell_perm.alloc(ctx, (size_t)m * n));
    {
        PT_LAUNCH(ctx, "trace_locate_cells");
        pt_locate_cells_kernel<<<pt_grid_for((size_t)m, 128), 128, 0, ctx->stream>>>(g, sdev, (size_t)m, cell_base.p, cell_perm.p);
        PT_TRY(pt_check_launch(ctx, "pt_locate_cells_kernel"));
    }
    t->stages.insert(t->stages.end(), {0, t->levels, m, m, m});
    const size_t nverts = (size_t)m * (n + 1);
    PT_TRY(pt_table_reserve(ctx, t->signs, nverts));
    PtBuf<uint32_t> pending;
    PT_TRY(pending.alloc(ctx, nverts));
    PT_TRY(pt_reset_pending(t));
    {
        PT_LAUNCH(ctx, "trace_cell_vertices");
        pt_cell_vertices_kernel<<<pt_grid_for(nverts, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), cell_base.p, cell_perm.p,
                                                                                     (size_t)m, pending.p, t->counters.p);
        PT_TRY(pt_check_launch(ctx, "pt_cell_vertices_kernel"));
    }
    PT_TRY(pt_read_counters(t));
    PT_TRY(pt_eval_pending(t, pending.p, (size_t)t->host_counters.n_pending));
    const int bound = (n + 1) * n / 2;
    const size_t nslots = (size_t)m * bound;
    PT_TRY(pt_table_reserve(ctx, t->visited, nslots));
    PtBuf<uint32_t> vis_slot;
    PT_TRY(vis_slot.alloc(ctx, nslots));
    const unsigned long long markers_before = t->host_counters.markers;
    {
        PT_LAUNCH(ctx, "trace_cell_edges");
        pt_cell_edges_kernel<<<pt_grid_for(nslots, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->visited.view(), cell_base.p,
                                                                                  cell_perm.p, (size_t)m, bound, vis_slot.p, t->counters.p);
        PT_TRY(pt_check_launch(ctx, "pt_cell_edges_kernel"));
    }
    const long long before = t->n_edges;
    long long admitted = 0;
    PT_TRY(pt_admit_items(t, (size_t)m, bound, vis_slot.p, &admitted));
    PT_TRY(pt_read_counters(t));
    t->stages.insert(t->stages.end(), {1, t->levels, m, (long long)nslots, (long long)(t->host_counters.markers - markers_before)});
    PT_TRY(pt_set_range_frontier(t, before, admitted));
    return PT_OK;
}

static int pt_trace_expand_impl(pt_trace* t, long long* frontier_out) {
    pt_ctx* ctx = t->ctx;
    PtGeom& g = t->geom;
    t->levels += 1;
    const long long F = t->n_frontier;
    const int stride = pt_stride_for(g.n);
    const long long before = t->n_edges;
    const unsigned long long cand_before = t->host_counters.candidates;
    // chunk the frontier: bounds the per-slot scratch and the worst-case table growth per chunk (~2^24 slots)
    size_t chunk_edges = ((size_t)1 << 24) / (size_t)stride;
    if (chunk_edges < 1024) chunk_edges = 1024;
    PtBuf<uint32_t> sgn_slot, vis_slot, pending;
    // the frontier buffer is replaced at the end; chunks read the current one
    for (long long f0 = 0; f0 < F; f0 += (long long)chunk_edges) {
        const size_t fc = (size_t)((F - f0) < (long long)chunk_edges ? (F - f0) : (long long)chunk_edges);
        const size_t nslots = fc * (size_t)stride;
        PT_TRY(sgn_slot.ensure(ctx, nslots, 0));
        PT_TRY(vis_slot.ensure(ctx, nslots, 0));
        PT_TRY(pending.ensure(ctx, nslots, 0));
        PT_TRY(pt_table_reserve(ctx, t->signs, nslots));
        PT_TRY(pt_table_reserve(ctx, t->visited, nslots));
        PT_TRY(pt_reset_pending(t));
        const uint32_t* fr = t->frontier.p + f0;
        {
            PT_LAUNCH(ctx, "trace_wave_probe");
            pt_wave_probe_kernel<<<pt_grid_for(fc * 32, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->edge_key.p, fr, fc, stride,
                                                                                       sgn_slot.p, pending.p, t->counters.p);
            PT_TRY(pt_check_launch(ctx, "pt_wave_probe_kernel"));
        }
        PT_TRY(pt_read_counters(t));
        PT_TRY(pt_eval_pending(t, pending.p, (size_t)t->host_counters.n_pending));
        {
            PT_LAUNCH(ctx, "trace_wave_partner");
            pt_wave_partner_kernel<<<pt_grid_for(fc * 32, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->visited.view(), t->edge_key.p,
                                                                                         t->edge_sa.p, fr, fc, stride, sgn_slot.p,
                                                                                         vis_slot.p, t->counters.p);
            PT_TRY(pt_check_launch(ctx, "pt_wave_partner_kernel"));
        }
        long long admitted = 0;
        PT_TRY(pt_admit_items(t, fc, stride, vis_slot.p, &admitted));
    }
    PT_TRY(pt_read_counters(t));
    const long long cands = (long long)(t->host_counters.candidates - cand_before);
    t->stages.insert(t->stages.end(), {2, t->levels, F, cands, cands});
    t->stages.insert(t->stages.end(), {3, t->levels, cands, cands, cands});
    if (t->range_frontier) t->expanded_upto = before;   // everything before the new frontier is expanded
    PT_TRY(pt_set_range_frontier(t, before, t->n_edges - before));
    t->n_adj = -1;
    if (frontier_out) *frontier_out = t->n_frontier;
    return PT_OK;
}

// ---- result assembly ------------------------------------------------------------------------
__global__ void pt_edge_endpoints_kernel(PtGeom g, const u64* __restrict__ edge_key, size_t first, size_t count,
                                         double* __restrict__ a, double* __restrict__ b) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 ek = edge_key[first + i];
    int u[PT_NMAX], v[PT_NMAX]; double x[PT_NMAX];
    pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
    pt_apply_masks(g.n, u, pt_edge_mask(g, ek), 0u, v);
    pt_vertex_point(g, u, x);
    for (int d = 0; d < g.n; ++d) a[i * g.n + d] = x[d];
    pt_vertex_point(g, v, x);
    for (int d = 0; d < g.n; ++d) b[i * g.n + d] = x[d];
}

__global__ void pt_edge_unpack_kernel(PtGeom g, const u64* __restrict__ edge_key, size_t first, size_t count,
                                      int32_t* __restrict__ base, uint32_t* __restrict__ mask) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 ek = edge_key[first + i];
    if (base) {
        int u[PT_NMAX];
        pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
        for (int d = 0; d < g.n; ++d) base[i * g.n + d] = u[d];
    }
    if (mask) mask[i] = pt_edge_mask(g, ek);
}

// adjacency (tracer.py:249-251): pairs (edge, partner) for every coface of every expanded edge
__global__ void __launch_bounds__(256)
pt_adjacency_kernel(PtGeom g, PtTable sgn, PtTable vis, const u64* __restrict__ edge_key, const int8_t* __restrict__ edge_sa,
                    size_t count, int stride, u64* __restrict__ pairs) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= count) return;
    const u64 ek = edge_key[w];
    const int sa = edge_sa[w];
    const uint32_t s = pt_edge_mask(g, ek);
    int u[PT_NMAX];
    pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
    const int nc = pt_ncofaces(g.n, s);
    for (int j = lane; j < stride; j += 32) {
        u64 out = PT_EMPTY;
        if (j < nc) {
            PtCoface f = pt_coface(g.n, s, j);
            int c[PT_NMAX]; u64 ck, cslot;
            pt_apply_masks(g.n, u, f.c_plus, f.c_minus, c);
            if (pt_pack_vertex(g, c, ck) && pt_table_find(sgn, ck, cslot)) {
                u64 sv = sgn.ent[2 * cslot + 1];
                if (sv <= 1ull) {
                    PtPartner p = pt_partner(g.n, u, s, sa, j, sv ? 1 : -1);
                    u64 bk, eslot;
                    if (pt_pack_vertex(g, p.base, bk) && pt_table_find(vis, pt_edge_key(g, bk, p.mask), eslot)) {
                        u64 idx = vis.ent[2 * eslot + 1];
                        if (idx < PT_VAL_PENDING_BASE && idx != (u64)w) {
                            u64 lo = idx < (u64)w ? idx : (u64)w, hi = idx < (u64)w ? (u64)w : idx;
                            out = (lo << 32) | hi;
                        }
                    }
                }
            }
        }
        pairs[w * stride + j] = out;
    }
}

// ---- seeding from explicit edges (expand_frontier, tracer.py:418-433) ---------------------------
__global__ void pt_seed_insert_kernel(PtGeom g, PtTable vis, const int32_t* __restrict__ base, const uint32_t* __restrict__ mask,
                                      size_t m, uint32_t* __restrict__ vis_slot, PtCounters* ctr) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int u[PT_NMAX];
    for (int d = 0; d < g.n; ++d) u[d] = base[i * g.n + d];
    u64 bk; uint32_t marker = PT_NONE32;
    if (!pt_pack_vertex(g, u, bk)) atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
    else {
        bool ins;
        u64 slot = pt_table_insert(vis, pt_edge_key(g, bk, mask[i]), ins, &ctr->error);
        atomicMin(&vis.ent[2 * slot + 1], PT_VAL_PENDING_BASE + (u64)i);
        marker = (uint32_t)slot;
    }
    vis_slot[i] = marker;
}
// resolve frontier rows to edge indices and queue their endpoints for sign evaluation
__global__ void pt_seed_frontier_kernel(PtGeom g, PtTable vis, PtTable sgn, const int32_t* __restrict__ base,
                                        const uint32_t* __restrict__ mask, size_t count, uint32_t* __restrict__ frontier,
                                        uint32_t* __restrict__ pending, PtCounters* ctr) {
    size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t i = tid >> 1; int which = (int)(tid & 1);
    bool inserted = false; u64 slot = 0;
    if (i < count) {
        int u[PT_NMAX], v[PT_NMAX];
        for (int d = 0; d < g.n; ++d) u[d] = base[i * g.n + d];
        pt_apply_masks(g.n, u, which ? mask[i] : 0u, 0u, v);
        u64 vk;
        if (!pt_pack_vertex(g, v, vk)) atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
        else {
            slot = pt_table_insert(sgn, vk, inserted, &ctr->error);
            if (!which) {
                u64 es;
                if (pt_table_find(vis, pt_edge_key(g, vk, mask[i]), es)) frontier[i] = (uint32_t)vis.ent[2 * es + 1];
                else { frontier[i] = 0; atomicOr(&ctr->error, PT_ERR_TABLE_FULL); }
            }
        }
    }
    unsigned long long pos = pt_warp_append(&ctr->n_pending, inserted);
    if (inserted) pending[pos] = (uint32_t)slot;
}
__global__ void pt_seed_signs_kernel(PtGeom g, PtTable sgn, const u64* __restrict__ edge_key, const uint32_t* __restrict__ frontier,
                                     size_t count, int8_t* __restrict__ edge_sa) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t e = frontier[i];
    u64 slot;
    if (pt_table_find(sgn, pt_edge_vkey(g, edge_key[e]), slot)) edge_sa[e] = sgn.ent[2 * slot + 1] ? (int8_t)1 : (int8_t)-1;
}

extern "C" {

int pt_trace_seed_edges(pt_trace* t, const int32_t* base, const uint32_t* mask, long long n_visited, long long n_frontier) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    pt_ctx* ctx = t->ctx;
    PtGeom& g = t->geom;
    const int n = g.n;
    const long long m = n_visited + n_frontier;
    if (n_visited < 0 || n_frontier < 0) return pt_fail(ctx, PT_E_INVALID, "negative edge count");
    if (m == 0) { t->n_frontier = 0; return PT_OK; }
    if (!base || !mask) return pt_fail(ctx, PT_E_INVALID, "edge arrays are NULL");
    PtBuf<int32_t> tb; PtBuf<uint32_t> tm;
    const int32_t* bdev; const uint32_t* mdev;
    PT_TRY(pt_stage_in(ctx, base, (size_t)m * n, tb, &bdev));
    PT_TRY(pt_stage_in(ctx, mask, (size_t)m, tm, &mdev));
    if (!t->window_set) {
        int32_t first[PT_NMAX];
        PT_CUDA(ctx, cudaMemcpyAsync(first, bdev, n * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        int cb[PT_NMAX];
        for (int d = 0; d < n; ++d) cb[d] = first[d];
        PT_TRY(pt_set_window(t, cb));
    }
    PT_TRY(pt_table_reserve(ctx, t->visited, (u64)m));
    PtBuf<uint32_t> vis_slot;
    PT_TRY(vis_slot.alloc(ctx, (size_t)m));
    {
        PT_LAUNCH(ctx, "trace_seed_insert");
        pt_seed_insert_kernel<<<pt_grid_for((size_t)m, 256), 256, 0, ctx->stream>>>(g, t->visited.view(), bdev, mdev, (size_t)m,
                                                                                      vis_slot.p, t->counters.p);
        PT_TRY(pt_check_launch(ctx, "pt_seed_insert_kernel"));
    }
    long long admitted = 0;
    PT_TRY(pt_admit_items(t, (size_t)m, 1, vis_slot.p, &admitted));
    PT_TRY(t->frontier.ensure(ctx, (size_t)(n_frontier > 0 ? n_frontier : 1), 0));
    t->n_frontier = n_frontier;
    t->range_frontier = false;
    if (n_frontier > 0) {
        PT_TRY(pt_table_reserve(ctx, t->signs, (u64)(2 * n_frontier)));
        PtBuf<uint32_t> pending;
        PT_TRY(pending.alloc(ctx, (size_t)(2 * n_frontier)));
        PT_TRY(pt_reset_pending(t));
        {
            PT_LAUNCH(ctx, "trace_seed_frontier");
            pt_seed_frontier_kernel<<<pt_grid_for((size_t)(2 * n_frontier), 256), 256, 0, ctx->stream>>>(
                g, t->visited.view(), t->signs.view(), bdev + (size_t)n_visited * n, mdev + n_visited, (size_t)n_frontier,
                t->frontier.p, pending.p, t->counters.p);
            PT_TRY(pt_check_launch(ctx, "pt_seed_frontier_kernel"));
        }
        PT_TRY(pt_read_counters(t));
        PT_TRY(pt_eval_pending(t, pending.p, (size_t)t->host_counters.n_pending));
        {
            PT_LAUNCH(ctx, "trace_seed_signs");
            pt_seed_signs_kernel<<<pt_grid_for((size_t)n_frontier, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->edge_key.p,
                                                                                                  t->frontier.p, (size_t)n_frontier, t->edge_sa.p);
            PT_TRY(pt_check_launch(ctx, "pt_seed_signs_kernel"));
        }
    }
    PT_TRY(pt_read_counters(t));
    return PT_OK;
}

}  // extern "C"

extern "C" {

int pt_trace_create(pt_ctx* ctx, const pt_field* field, int n, double scale, const double* offset, const double* box_lo,
                    const double* box_hi, long long max_edges, double eps, pt_trace** out) {
    if (!ctx || !field || !out) return pt_fail(ctx, PT_E_INVALID, "pt_trace_create: NULL argument");
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "lattice dimension %d unsupported (2..7)", n);
    if (pt_field_dim(field) != n) return pt_fail(ctx, PT_E_INVALID, "manifold and lattice dimension mismatch");
    if (!(scale > 0.0)) return pt_fail(ctx, PT_E_INVALID, "lattice scale must be positive");
    if (max_edges < 1) return pt_fail(ctx, PT_E_INVALID, "max_edges must be positive");
    if (max_edges > (1ll << 31) - 2) return pt_fail(ctx, PT_E_INVALID, "max_edges above 2^31-2 is not supported");
    if (!(eps > 0.0)) return pt_fail(ctx, PT_E_INVALID, "eps must be positive");
    if ((box_lo == nullptr) != (box_hi == nullptr)) return pt_fail(ctx, PT_E_INVALID, "box needs both bounds");
    pt_trace* t = new pt_trace();
    t->ctx = ctx; t->field = field; t->max_edges = max_edges; t->eps = eps;
    memset(&t->geom, 0, sizeof(t->geom));
    memset(&t->host_counters, 0, sizeof(t->host_counters));
    PtGeom& g = t->geom;
    g.n = n; g.bits = pt_bits_for_dim(n); g.scale = scale;
    for (int d = 0; d < n; ++d) g.offset[d] = offset ? offset[d] : 0.0;
    if (box_lo) {
        g.has_box = 1;
        for (int d = 0; d < n; ++d) {
            if (!(box_lo[d] < box_hi[d])) { delete t; return pt_fail(ctx, PT_E_INVALID, "box must be a (lower, upper) pair with lower < upper"); }
            // vertex bounds in lattice units (tracer.py:174-175); integer v passes iff lo <= v <= hi
            double lo = (box_lo[d] - g.offset[d]) / scale, hi = (box_hi[d] - g.offset[d]) / scale;
            if (lo < -2e9 || hi > 2e9) { delete t; return pt_fail(ctx, PT_E_RANGE, "clamp box too large for 32-bit lattice coordinates"); }
            g.box_lo[d] = (int)ceil(lo); g.box_hi[d] = (int)floor(hi);
            t->box_lo_f[d] = lo; t->box_hi_f[d] = hi;
        }
        int rc = pt_set_window(t, nullptr);
        if (rc != PT_OK) { delete t; return rc; }
    }
    int rc = t->counters.alloc(ctx, 1);
    if (rc == PT_OK) { cudaMemsetAsync(t->counters.p, 0, sizeof(PtCounters), ctx->stream); }
    if (rc == PT_OK) rc = pt_table_init(ctx, t->visited, 1 << 16);
    if (rc == PT_OK) rc = pt_table_init(ctx, t->signs, 1 << 16);
    if (rc == PT_OK) rc = t->edge_key.alloc(ctx, 1 << 12);
    if (rc == PT_OK) rc = t->edge_sa.alloc(ctx, 1 << 12);
    if (rc != PT_OK) { delete t; return rc; }
    *out = t;
    return PT_OK;
}

void pt_trace_destroy(pt_trace* t) { delete t; }

int pt_trace_locate(pt_trace* t, const double* seeds, long long m) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    return pt_trace_locate_impl(t, seeds, m);
}

int pt_trace_expand(pt_trace* t, long long* frontier_out) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    if (!t->window_set) return pt_fail(t->ctx, PT_E_STATE, "expand before locate/seed");
    return pt_trace_expand_impl(t, frontier_out);
}

int pt_trace_run(pt_trace* t, const double* seeds, long long m) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    PT_TRY(pt_trace_locate_impl(t, seeds, m));
    while (t->n_frontier > 0 && t->complete) PT_TRY(pt_trace_expand_impl(t, nullptr));
    if (t->n_frontier == 0) t->expanded_upto = t->n_edges;
    return PT_OK;
}

int pt_trace_get_stats(pt_trace* t, pt_trace_stats* out) {
    if (!t || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_trace_get_stats: NULL argument");
    PT_TRY(pt_read_counters(t));
    out->levels = t->levels; out->seeds = t->seeds; out->visited_edges = t->n_edges;
    out->field_evaluations = t->field_evaluations;
    out->dropped_out_of_box = (long long)t->host_counters.dropped;
    out->candidates = (long long)t->host_counters.candidates;
    out->frontier = t->n_frontier;
    out->complete = t->complete ? 1 : 0;
    out->closure_ok = (t->n_edges > 0 && t->complete && t->host_counters.dropped == 0) ? 1 : 0;
    out->table_capacity = (long long)t->visited.capacity;
    out->sign_table_capacity = (long long)t->signs.capacity;
    out->n_stages = (long long)(t->stages.size() / 5);
    out->ambiguous_signs = (long long)t->host_counters.ambiguous;
    return PT_OK;
}

int pt_trace_stages(pt_trace* t, long long* out, long long rows) {
    if (!t || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_trace_stages: NULL argument");
    long long have = (long long)(t->stages.size() / 5);
    if (rows > have) rows = have;
    memcpy(out, t->stages.data(), (size_t)rows * 5 * sizeof(long long));
    return PT_OK;
}

int pt_trace_edges(pt_trace* t, long long first, long long count, int32_t* base, uint32_t* mask, int8_t* sign_a) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    pt_ctx* ctx = t->ctx;
    if (first < 0 || count < 0 || first + count > t->n_edges) return pt_fail(ctx, PT_E_INVALID, "edge range out of bounds");
    if (count == 0) return PT_OK;
    const int n = t->geom.n;
    PtBuf<int32_t> tb; PtBuf<uint32_t> tm;
    int32_t* bdev = nullptr; uint32_t* mdev = nullptr;
    if (base) { if (pt_is_device_ptr(base)) bdev = base; else { PT_TRY(tb.alloc(ctx, (size_t)count * n)); bdev = tb.p; } }
    if (mask) { if (pt_is_device_ptr(mask)) mdev = mask; else { PT_TRY(tm.alloc(ctx, (size_t)count)); mdev = tm.p; } }
    if (bdev || mdev) {
        pt_edge_unpack_kernel<<<pt_grid_for((size_t)count, 256), 256, 0, ctx->stream>>>(t->geom, t->edge_key.p, (size_t)first,
                                                                                          (size_t)count, bdev, mdev);
        PT_TRY(pt_check_launch(ctx, "pt_edge_unpack_kernel"));
    }
    if (base && bdev != base) PT_TRY(pt_copy_out(ctx, base, bdev, (size_t)count * n, false));
    if (mask && mdev != mask) PT_TRY(pt_copy_out(ctx, mask, mdev, (size_t)count, false));
    if (sign_a) PT_TRY(pt_copy_out(ctx, sign_a, t->edge_sa.p + first, (size_t)count, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_trace_frontier(pt_trace* t, long long* first, long long* count) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    if (!t->range_frontier) return pt_fail(t->ctx, PT_E_STATE, "frontier is not an index range");
    if (first) *first = t->n_edges - t->n_frontier;
    if (count) *count = t->n_frontier;
    return PT_OK;
}

int pt_trace_points(pt_trace* t, double* out) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    pt_ctx* ctx = t->ctx;
    const size_t E = (size_t)t->n_edges;
    if (E == 0) return PT_OK;
    if (!out) return pt_fail(ctx, PT_E_INVALID, "points output is NULL");
    const int n = t->geom.n;
    PtBuf<double> a, b, o;
    PT_TRY(a.alloc(ctx, E * n));
    PT_TRY(b.alloc(ctx, E * n));
    double* odev = out;
    if (!pt_is_device_ptr(out)) { PT_TRY(o.alloc(ctx, E * n)); odev = o.p; }
    {
        PT_LAUNCH(ctx, "trace_edge_endpoints");
        pt_edge_endpoints_kernel<<<pt_grid_for(E, 256), 256, 0, ctx->stream>>>(t->geom, t->edge_key.p, 0, E, a.p, b.p);
        PT_TRY(pt_check_launch(ctx, "pt_edge_endpoints_kernel"));
    }
    PT_TRY(pt_field_bisect_dev(ctx, t->field, a.p, b.p, t->edge_sa.p, E, t->eps, odev));
    if (odev != out) PT_TRY(pt_copy_out(ctx, out, odev, E * n, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

long long pt_trace_adjacency(pt_trace* t, long long* pairs, long long cap) {
    if (!t) { pt_fail(nullptr, PT_E_INVALID, "trace is NULL"); return PT_E_INVALID; }
    pt_ctx* ctx = t->ctx;
    if (t->n_adj < 0) {
        const size_t count = (size_t)t->expanded_upto;
        t->n_adj = 0;
        if (count > 0) {
            const int stride = pt_stride_for(t->geom.n);
            const size_t total = count * (size_t)stride;
            PtBuf<u64> raw, sorted;
            if (raw.alloc(ctx, total) != PT_OK || sorted.alloc(ctx, total) != PT_OK) return PT_E_NOMEM;
            {
                PT_LAUNCH(ctx, "trace_adjacency");
                pt_adjacency_kernel<<<pt_grid_for(count * 32, 256), 256, 0, ctx->stream>>>(t->geom, t->signs.view(), t->visited.view(),
                                                                                             t->edge_key.p, t->edge_sa.p, count, stride, raw.p);
                if (pt_check_launch(ctx, "pt_adjacency_kernel") != PT_OK) return PT_E_CUDA;
            }
            size_t tb = 0, tb2 = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, raw.p, sorted.p, (long long)total, 0, 64, ctx->stream);
            PtBuf<long long> nsel;
            if (nsel.alloc(ctx, 1) != PT_OK) return PT_E_NOMEM;
            cub::DeviceSelect::Unique(nullptr, tb2, sorted.p, raw.p, nsel.p, (long long)total, ctx->stream);
            PtBuf<uint8_t> tmp;
            if (tmp.alloc(ctx, tb > tb2 ? tb : tb2) != PT_OK) return PT_E_NOMEM;
            cub::DeviceRadixSort::SortKeys(tmp.p, tb, raw.p, sorted.p, (long long)total, 0, 64, ctx->stream);
            cub::DeviceSelect::Unique(tmp.p, tb2, sorted.p, raw.p, nsel.p, (long long)total, ctx->stream);
            ctx->launches += 2;
            long long* h = (long long*)ctx->pinned;
            cudaMemcpyAsync(h, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream);
            if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { pt_fail(ctx, PT_E_CUDA, "adjacency sort failed"); return PT_E_CUDA; }
            long long uniq = *h;
            // the EMPTY sentinel (all ones) sorts last; drop it if present
            if (uniq > 0) {
                u64 last;
                cudaMemcpy(&last, raw.p + (uniq - 1), sizeof(u64), cudaMemcpyDeviceToHost);
                if (last == PT_EMPTY) uniq -= 1;
            }
            if (t->adj.alloc(ctx, (size_t)(uniq > 0 ? uniq : 1)) != PT_OK) return PT_E_NOMEM;
            cudaMemcpyAsync(t->adj.p, raw.p, (size_t)uniq * sizeof(u64), cudaMemcpyDeviceToDevice, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
            t->n_adj = uniq;
        }
    }
    if (pairs) {
        long long take = t->n_adj < cap ? t->n_adj : cap;
        std::vector<u64> h((size_t)take);
        if (take > 0) cudaMemcpy(h.data(), t->adj.p, (size_t)take * sizeof(u64), cudaMemcpyDeviceToHost);
        for (long long i = 0; i < take; ++i) { pairs[2 * i] = (long long)(h[(size_t)i] >> 32); pairs[2 * i + 1] = (long long)(h[(size_t)i] & 0xffffffffull); }
    }
    return t->n_adj;
}

}  // extern "C"

// ==== owner-hashed sharded BFS (multi-GPU) =============================================================
// Rank r of W owns the canonical edges whose base lattice vertex hashes to r.  One wave:
//   pt_trace_wave_candidates  expand the local frontier (probe signs, evaluate unknown vertices, partner rule,
//                             box clamp) and emit one 16-byte record per surviving candidate,
//                             (edge key, tag) with tag = (parent's GLOBAL admission index * stride + coface ordinal)*2
//                             + (sign at base > 0), bucketed by owner rank  -> all_to_all by the caller
//   pt_trace_wave_admit       the owner inserts the records it received into its visited shard with atomicMin(tag):
//                             the winner of a new edge is its first occurrence in the reference's slot order;
//                             winners come back sorted by tag
//   pt_trace_wave_commit      after the caller ranked all ranks' winner tags (global admission indices), the
//                             winners join the local edge list and form the next local frontier
// Tags are comparable across ranks, so the union of the ranks' edge lists ordered by global index IS the
// single-GPU (= reference) admission order.
PT_HD int pt_owner_of(const PtGeom& g, u64 edge_key, int world) {
    return (int)(pt_mix(pt_edge_vkey(g, edge_key) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull) % (u64)world);
}

__global__ void pt_shard_select_kernel(PtGeom g, const u64* __restrict__ edge_key, const int8_t* __restrict__ edge_sa,
                                       size_t count, int rank, int world, u64* __restrict__ out_gidx,
                                       u64* __restrict__ out_key, int8_t* __restrict__ out_sa, unsigned long long* counter) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool mine = i < count && pt_owner_of(g, edge_key[i], world) == rank;
    const unsigned long long pos = pt_warp_append(counter, mine);
    if (mine) { out_gidx[pos] = (u64)i; out_key[pos] = edge_key[i]; out_sa[pos] = edge_sa[i]; }
}

__global__ void pt_shard_fill_kernel(PtTable vis, const u64* __restrict__ gidx_sorted, const uint32_t* __restrict__ order,
                                     const u64* __restrict__ key_in, const int8_t* __restrict__ sa_in, size_t count,
                                     u64* __restrict__ edge_key, int8_t* __restrict__ edge_sa, u64* __restrict__ edge_gidx,
                                     unsigned* err) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t src = order[i];
    const u64 key = key_in[src];
    edge_key[i] = key; edge_sa[i] = sa_in[src]; edge_gidx[i] = gidx_sorted[i];
    bool ins;
    const u64 slot = pt_table_insert(vis, key, ins, err);
    vis.ent[2 * slot + 1] = (u64)i;
}

// partner stage of a sharded wave: emit (edge key, tag) instead of touching a visited table
__global__ void __launch_bounds__(256)
pt_wave_emit_kernel(PtGeom g, PtTable sgn, const u64* __restrict__ edge_key, const int8_t* __restrict__ edge_sa,
                    const u64* __restrict__ edge_gidx, const uint32_t* __restrict__ frontier, size_t fcount, int stride,
                    const uint32_t* __restrict__ sgn_slot, u64* __restrict__ cand, unsigned long long* cand_count,
                    PtCounters* ctr) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= fcount) return;
    const uint32_t e = frontier[w];
    const u64 ek = edge_key[e];
    const int sa = edge_sa[e];
    const u64 parent = edge_gidx[e];
    const uint32_t s = pt_edge_mask(g, ek);
    int u[PT_NMAX];
    pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
    const int nc = pt_ncofaces(g.n, s);
    for (int j0 = 0; j0 < nc; j0 += 32) {
        const int j = j0 + lane;
        bool emit = false, dropped = false;
        u64 key = 0, tag = 0;
        if (j < nc) {
            const int sc = pt_ld_cg(&sgn.ent[2 * (u64)sgn_slot[w * stride + j] + 1]) ? 1 : -1;
            PtPartner p = pt_partner(g.n, u, s, sa, j, sc);
            int other[PT_NMAX];
            pt_apply_masks(g.n, p.base, p.mask, 0u, other);
            if (!(pt_in_box(g, p.base) && pt_in_box(g, other))) dropped = true;
            else {
                u64 bk;
                if (!pt_pack_vertex(g, p.base, bk)) atomicOr(&ctr->error, PT_ERR_KEY_RANGE);
                else {
                    key = pt_edge_key(g, bk, p.mask);
                    tag = ((parent * (u64)stride + (u64)j) << 1) | (p.sign_base > 0 ? 1ull : 0ull);
                    emit = true;
                }
            }
        }
        const unsigned db = __ballot_sync(0xffffffffu, dropped);
        if (lane == 0 && db) atomicAdd(&ctr->dropped, (unsigned long long)__popc(db));
        const unsigned long long pos = pt_warp_append(cand_count, emit);
        if (emit) { cand[2 * pos] = key; cand[2 * pos + 1] = tag; }
    }
}

__global__ void pt_owner_count_kernel(PtGeom g, const u64* __restrict__ cand, size_t count, int world,
                                      unsigned long long* __restrict__ hist) {
    __shared__ unsigned int local[64];
    if (threadIdx.x < 64) local[threadIdx.x] = 0;
    __syncthreads();
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) atomicAdd(&local[pt_owner_of(g, cand[2 * i], world)], 1u);
    __syncthreads();
    if (threadIdx.x < world && local[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)local[threadIdx.x]);
}

__global__ void pt_owner_scatter_kernel(PtGeom g, const u64* __restrict__ cand, size_t count, int world,
                                        unsigned long long* __restrict__ cursor, u64* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 key = cand[2 * i], tag = cand[2 * i + 1];
    const unsigned long long pos = atomicAdd(&cursor[pt_owner_of(g, key, world)], 1ull);
    out[2 * pos] = key; out[2 * pos + 1] = tag;
}

// owner side: claim the edge for the smallest tag seen this wave (already admitted edges keep their small index)
__global__ void pt_shard_insert_kernel(PtTable vis, const u64* __restrict__ rec, size_t count, uint32_t* __restrict__ slot_out,
                                       unsigned* err) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    bool ins;
    const u64 slot = pt_table_insert(vis, rec[2 * i], ins, err);
    atomicMin(&vis.ent[2 * slot + 1], PT_VAL_PENDING_BASE + rec[2 * i + 1]);
    slot_out[i] = (uint32_t)slot;
}

__global__ void pt_shard_winners_kernel(PtTable vis, const u64* __restrict__ rec, const uint32_t* __restrict__ slot_in,
                                        size_t count, u64* __restrict__ win_tag, u64* __restrict__ win_key,
                                        unsigned long long* counter) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool win = false;
    if (i < count) win = pt_ld_cg(&vis.ent[2 * (u64)slot_in[i] + 1]) == PT_VAL_PENDING_BASE + rec[2 * i + 1];
    const unsigned long long pos = pt_warp_append(counter, win);
    if (win) { win_tag[pos] = rec[2 * i + 1]; win_key[pos] = rec[2 * i]; }
}

__global__ void pt_shard_commit_kernel(PtTable vis, const u64* __restrict__ win, const long long* __restrict__ gidx,
                                       size_t count, long long first_local, u64* __restrict__ edge_key,
                                       int8_t* __restrict__ edge_sa, u64* __restrict__ edge_gidx) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 tag = win[2 * i], key = win[2 * i + 1];
    u64 slot;
    if (!pt_table_find(vis, key, slot)) return;
    if (gidx[i] >= 0) {
        const long long idx = first_local + (long long)i;      // dead winners (cap) are a suffix in tag order
        edge_key[idx] = key; edge_sa[idx] = (tag & 1ull) ? (int8_t)1 : (int8_t)-1; edge_gidx[idx] = (u64)gidx[i];
        vis.ent[2 * slot + 1] = (u64)idx;
    } else {
        vis.ent[2 * slot + 1] = PT_VAL_DEAD;
    }
}

__global__ void pt_interleave_kernel(const u64* __restrict__ a, const u64* __restrict__ b, size_t count, u64* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) { out[2 * i] = a[i]; out[2 * i + 1] = b[i]; }
}

extern "C" {

int pt_trace_shard(pt_trace* t, int rank, int world) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    pt_ctx* ctx = t->ctx;
    if (world < 1 || world > 64 || rank < 0 || rank >= world) return pt_fail(ctx, PT_E_INVALID, "bad rank/world (%d/%d; at most 64 ranks)", rank, world);
    if (!t->geom.has_box) return pt_fail(ctx, PT_E_STATE, "the sharded trace needs a clamp box (every rank must pack keys in the same window)");
    if (t->levels != 0 || !t->range_frontier) return pt_fail(ctx, PT_E_STATE, "pt_trace_shard must follow pt_trace_locate directly");
    const size_t E = (size_t)t->n_edges;
    t->rank = rank; t->world = world; t->n_global = (long long)E;
    PtBuf<u64> gidx, key, gidx_sorted; PtBuf<int8_t> sa; PtBuf<uint32_t> order_in, order; PtBuf<unsigned long long> counter;
    PT_TRY(gidx.alloc(ctx, E + 1)); PT_TRY(key.alloc(ctx, E + 1)); PT_TRY(sa.alloc(ctx, E + 1));
    PT_TRY(gidx_sorted.alloc(ctx, E + 1)); PT_TRY(order_in.alloc(ctx, E + 1)); PT_TRY(order.alloc(ctx, E + 1));
    PT_TRY(counter.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), ctx->stream));
    size_t mine = 0;
    if (E) {
        PT_LAUNCH(ctx, "trace_shard");
        pt_shard_select_kernel<<<pt_grid_for(E, 256), 256, 0, ctx->stream>>>(t->geom, t->edge_key.p, t->edge_sa.p, E, rank, world,
                                                                             gidx.p, key.p, sa.p, counter.p);
        PT_TRY(pt_check_launch(ctx, "pt_shard_select_kernel"));
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, counter.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        mine = (size_t)*h;
    }
    // restore admission order among the kept edges, rebuild the visited shard from empty
    PT_CUDA(ctx, cudaMemsetAsync(t->visited.ent.p, 0xFF, (size_t)t->visited.capacity * 2 * sizeof(u64), ctx->stream));
    t->visited.count = 0;
    PT_TRY(t->edge_gidx.ensure(ctx, mine + 1, 0));
    if (mine) {
        pt_iota_kernel<<<pt_grid_for(mine, 256), 256, 0, ctx->stream>>>(order_in.p, mine, 0u);
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, gidx.p, gidx_sorted.p, order_in.p, order.p, (int)mine, 0, 64, ctx->stream);
        PtBuf<uint8_t> tmp;
        PT_TRY(tmp.alloc(ctx, tmp_bytes));
        PT_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, gidx.p, gidx_sorted.p, order_in.p, order.p, (int)mine, 0, 64, ctx->stream));
        PT_TRY(pt_table_reserve(ctx, t->visited, (u64)mine));
        pt_shard_fill_kernel<<<pt_grid_for(mine, 256), 256, 0, ctx->stream>>>(t->visited.view(), gidx_sorted.p, order.p, key.p, sa.p, mine,
                                                                              t->edge_key.p, t->edge_sa.p, t->edge_gidx.p, &t->counters.p->error);
        PT_TRY(pt_check_launch(ctx, "pt_shard_fill_kernel"));
        t->visited.count = (u64)mine;
    }
    t->n_edges = (long long)mine;
    PT_TRY(pt_set_range_frontier(t, 0, (long long)mine));
    t->n_adj = -1;
    // locate ran identically on every rank: its out-of-box drops are reported by rank 0 only
    if (rank != 0)
        PT_CUDA(ctx, cudaMemsetAsync((char*)t->counters.p + offsetof(PtCounters, dropped), 0, sizeof(unsigned long long), ctx->stream));
    return pt_read_counters(t);
}

int pt_trace_wave_candidates(pt_trace* t, long long* counts) {
    if (!t || !counts) return pt_fail(t ? t->ctx : nullptr, PT_E_INVALID, "pt_trace_wave_candidates: NULL argument");
    pt_ctx* ctx = t->ctx;
    PtGeom& g = t->geom;
    const long long F = t->n_frontier;
    const int stride = pt_stride_for(g.n), world = t->world;
    const unsigned long long cand_before = t->host_counters.candidates;
    for (int r = 0; r < world; ++r) counts[r] = 0;
    t->n_cand = 0;
    PtBuf<unsigned long long> cc;          // [0] candidate cursor, [1..world] histogram, [1+world..] scatter cursors
    PT_TRY(cc.alloc(ctx, 2 * (size_t)world + 2));
    PT_CUDA(ctx, cudaMemsetAsync(cc.p, 0, (2 * (size_t)world + 2) * sizeof(unsigned long long), ctx->stream));
    PtBuf<u64> raw;
    size_t chunk_edges = ((size_t)1 << 24) / (size_t)stride;
    if (chunk_edges < 1024) chunk_edges = 1024;
    PtBuf<uint32_t> sgn_slot, pending;
    size_t emitted_bound = 0;
    for (long long f0 = 0; f0 < F; f0 += (long long)chunk_edges) {
        const size_t fc = (size_t)((F - f0) < (long long)chunk_edges ? (F - f0) : (long long)chunk_edges);
        const size_t nslots = fc * (size_t)stride;
        PT_TRY(sgn_slot.ensure(ctx, nslots, 0));
        PT_TRY(pending.ensure(ctx, nslots, 0));
        PT_TRY(pt_table_reserve(ctx, t->signs, nslots));
        PT_TRY(pt_reset_pending(t));
        const uint32_t* fr = t->frontier.p + f0;
        {
            PT_LAUNCH(ctx, "trace_wave_probe");
            pt_wave_probe_kernel<<<pt_grid_for(fc * 32, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->edge_key.p, fr, fc, stride,
                                                                                       sgn_slot.p, pending.p, t->counters.p);
            PT_TRY(pt_check_launch(ctx, "pt_wave_probe_kernel"));
        }
        PT_TRY(pt_read_counters(t));
        PT_TRY(pt_eval_pending(t, pending.p, (size_t)t->host_counters.n_pending));
        // every candidate of the chunks so far may survive the box clamp
        emitted_bound = (size_t)(t->host_counters.candidates - cand_before);
        PT_TRY(raw.ensure(ctx, 2 * emitted_bound + 2, 2 * (size_t)t->n_cand));
        {
            PT_LAUNCH(ctx, "trace_wave_emit");
            pt_wave_emit_kernel<<<pt_grid_for(fc * 32, 256), 256, 0, ctx->stream>>>(g, t->signs.view(), t->edge_key.p, t->edge_sa.p,
                                                                                      t->edge_gidx.p, fr, fc, stride, sgn_slot.p, raw.p,
                                                                                      cc.p, t->counters.p);
            PT_TRY(pt_check_launch(ctx, "pt_wave_emit_kernel"));
        }
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, cc.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        t->n_cand = (long long)*h;
    }
    PT_TRY(pt_read_counters(t));
    const long long cands = (long long)(t->host_counters.candidates - cand_before);
    t->levels += 1;
    t->stages.insert(t->stages.end(), {2, t->levels, F, cands, cands});
    t->stages.insert(t->stages.end(), {3, t->levels, cands, cands, cands});
    const size_t C = (size_t)t->n_cand;
    PT_TRY(t->cand.ensure(ctx, 2 * C + 2, 0));
    if (C) {
        {
            PT_LAUNCH(ctx, "trace_owner_bucket");
            pt_owner_count_kernel<<<pt_grid_for(C, 256), 256, 0, ctx->stream>>>(g, raw.p, C, world, cc.p + 1);
            PT_TRY(pt_check_launch(ctx, "pt_owner_count_kernel"));
        }
        unsigned long long* h = (unsigned long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(h, cc.p + 1, (size_t)world * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        unsigned long long offs[64], run = 0;
        for (int r = 0; r < world; ++r) { counts[r] = (long long)h[r]; offs[r] = run; run += h[r]; }
        PT_CUDA(ctx, cudaMemcpyAsync(cc.p + 1 + world, offs, (size_t)world * sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->stream));
        {
            PT_LAUNCH(ctx, "trace_owner_bucket");
            pt_owner_scatter_kernel<<<pt_grid_for(C, 256), 256, 0, ctx->stream>>>(g, raw.p, C, world, cc.p + 1 + world, t->cand.p);
            PT_TRY(pt_check_launch(ctx, "pt_owner_scatter_kernel"));
        }
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));   // offs lives on this stack frame
    }
    return PT_OK;
}

int pt_trace_wave_fetch(pt_trace* t, long long* out) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    if (t->n_cand == 0) return PT_OK;
    if (!out) return pt_fail(t->ctx, PT_E_INVALID, "output is NULL");
    return pt_copy_out(t->ctx, (u64*)out, t->cand.p, 2 * (size_t)t->n_cand, true);
}

int pt_trace_wave_admit(pt_trace* t, const long long* records, long long count, long long* n_winners) {
    if (!t || !n_winners) return pt_fail(t ? t->ctx : nullptr, PT_E_INVALID, "pt_trace_wave_admit: NULL argument");
    pt_ctx* ctx = t->ctx;
    *n_winners = 0; t->n_win = 0;
    if (count < 0) return pt_fail(ctx, PT_E_INVALID, "negative record count");
    if (count == 0) return PT_OK;
    if (!records) return pt_fail(ctx, PT_E_INVALID, "records is NULL");
    PtBuf<u64> tmp_rec; const u64* rec;
    PT_TRY(pt_stage_in(ctx, (const u64*)records, 2 * (size_t)count, tmp_rec, &rec));
    PT_TRY(pt_table_reserve(ctx, t->visited, (u64)count));
    PtBuf<uint32_t> slot; PtBuf<u64> wtag, wkey, wtag_s, wkey_s; PtBuf<unsigned long long> counter;
    PT_TRY(slot.alloc(ctx, (size_t)count));
    PT_TRY(wtag.alloc(ctx, (size_t)count)); PT_TRY(wkey.alloc(ctx, (size_t)count));
    PT_TRY(counter.alloc(ctx, 1));
    PT_CUDA(ctx, cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), ctx->stream));
    {
        PT_LAUNCH(ctx, "trace_shard_admit");
        pt_shard_insert_kernel<<<pt_grid_for((size_t)count, 256), 256, 0, ctx->stream>>>(t->visited.view(), rec, (size_t)count, slot.p,
                                                                                          &t->counters.p->error);
        PT_TRY(pt_check_launch(ctx, "pt_shard_insert_kernel"));
        pt_shard_winners_kernel<<<pt_grid_for((size_t)count, 256), 256, 0, ctx->stream>>>(t->visited.view(), rec, slot.p, (size_t)count,
                                                                                           wtag.p, wkey.p, counter.p);
        PT_TRY(pt_check_launch(ctx, "pt_shard_winners_kernel"));
    }
    unsigned long long* h = (unsigned long long*)ctx->pinned;
    PT_CUDA(ctx, cudaMemcpyAsync(h, counter.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const size_t V = (size_t)*h;
    PT_TRY(pt_read_counters(t));
    t->visited.count += (u64)V;
    t->n_win = (long long)V; *n_winners = (long long)V;
    PT_TRY(t->win.ensure(ctx, 2 * V + 2, 0));
    if (V) {
        PT_TRY(wtag_s.alloc(ctx, V)); PT_TRY(wkey_s.alloc(ctx, V));
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, wtag.p, wtag_s.p, wkey.p, wkey_s.p, (int)V, 0, 64, ctx->stream);
        PtBuf<uint8_t> tmp;
        PT_TRY(tmp.alloc(ctx, tmp_bytes));
        PT_LAUNCH(ctx, "trace_shard_admit");
        PT_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, wtag.p, wtag_s.p, wkey.p, wkey_s.p, (int)V, 0, 64, ctx->stream));
        pt_interleave_kernel<<<pt_grid_for(V, 256), 256, 0, ctx->stream>>>(wtag_s.p, wkey_s.p, V, t->win.p);
        PT_TRY(pt_check_launch(ctx, "pt_interleave_kernel"));
    }
    return PT_OK;
}

int pt_trace_wave_winner_tags(pt_trace* t, long long* out) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    if (t->n_win == 0) return PT_OK;
    if (!out) return pt_fail(t->ctx, PT_E_INVALID, "output is NULL");
    pt_ctx* ctx = t->ctx;
    cudaMemcpyKind kind = pt_is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    PT_CUDA(ctx, cudaMemcpy2DAsync(out, sizeof(u64), t->win.p, 2 * sizeof(u64), sizeof(u64), (size_t)t->n_win, kind, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_trace_wave_commit(pt_trace* t, const long long* gidx, long long alive, long long global_total) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    pt_ctx* ctx = t->ctx;
    const size_t V = (size_t)t->n_win;
    if (alive < 0 || (size_t)alive > V) return pt_fail(ctx, PT_E_INVALID, "alive count out of range");
    const long long before = t->n_edges;
    if (V) {
        if (!gidx) return pt_fail(ctx, PT_E_INVALID, "gidx is NULL");
        PtBuf<long long> tmp; const long long* gdev;
        PT_TRY(pt_stage_in(ctx, gidx, V, tmp, &gdev));
        PT_TRY(t->edge_key.ensure(ctx, (size_t)(before + alive + 1), (size_t)before));
        PT_TRY(t->edge_sa.ensure(ctx, (size_t)(before + alive + 1), (size_t)before));
        PT_TRY(t->edge_gidx.ensure(ctx, (size_t)(before + alive + 1), (size_t)before));
        PT_LAUNCH(ctx, "trace_shard_commit");
        pt_shard_commit_kernel<<<pt_grid_for(V, 256), 256, 0, ctx->stream>>>(t->visited.view(), t->win.p, gdev, V, before,
                                                                             t->edge_key.p, t->edge_sa.p, t->edge_gidx.p);
        PT_TRY(pt_check_launch(ctx, "pt_shard_commit_kernel"));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    if ((size_t)alive < V) t->complete = false;
    t->n_edges = before + alive;
    t->n_global = global_total;
    t->n_win = 0;
    t->expanded_upto = before;
    PT_TRY(pt_set_range_frontier(t, before, alive));
    t->n_adj = -1;
    return PT_OK;
}

int pt_trace_gidx(pt_trace* t, long long first, long long count, long long* out) {
    if (!t) return pt_fail(nullptr, PT_E_INVALID, "trace is NULL");
    if (first < 0 || count < 0 || first + count > t->n_edges) return pt_fail(t->ctx, PT_E_INVALID, "edge range out of bounds");
    if (count == 0) return PT_OK;
    if (!out) return pt_fail(t->ctx, PT_E_INVALID, "output is NULL");
    if (t->world == 1 && t->edge_gidx.count < (size_t)t->n_edges) return pt_fail(t->ctx, PT_E_STATE, "trace is not sharded");
    return pt_copy_out(t->ctx, (u64*)out, t->edge_gidx.p + first, (size_t)count, true);
}

}  // extern "C"
