// coarse_cells (subdivision.py:132-141): every full-dimensional cell containing a traced edge,
// deduplicated and sorted by (base vertex, permutation).  A warp per traced edge enumerates the
// |p1|!*|p2|! cell cofaces (lattice.py:245-266) as packed 64-bit keys whose numeric order equals the
// reference's tuple order; a radix sort + unique finishes the job.
#include <cub/cub.cuh>
#include "pt_trace.cuh"

__global__ void pt_cell_counts_kernel(PtGeom g, const u64* __restrict__ edge_key, size_t count, unsigned long long* __restrict__ ncell) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) ncell[i] = (unsigned long long)pt_ncellcofaces(g.n, pt_edge_mask(g, edge_key[i]));
    if (i == count) ncell[i] = 0;
}

// A cell is a coface of many traced edges (dof6: 14 M emitted keys for 1.3 M distinct cells).  Before the sort a
// direct-mapped "last key seen" table (no probing, L2-resident) drops a key whose slot already holds it; distinct keys
// sharing a slot just pass through more than once.  Whatever survives is compacted through a warp-aggregated counter
// and still goes through sort + unique, so the filter can only shrink the sort, never change the result.
__global__ void __launch_bounds__(256)
pt_cell_cofaces_kernel(PtGeom g, const u64* __restrict__ edge_key, size_t count, u64* __restrict__ seen, unsigned seen_mask,
                       u64* __restrict__ keys, unsigned long long* __restrict__ n_out, unsigned* err) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= count) return;
    const u64 ek = edge_key[w];
    const uint32_t s = pt_edge_mask(g, ek);
    int u[PT_NMAX];
    pt_unpack_vertex(g, pt_edge_vkey(g, ek), u);
    const int nc = pt_ncellcofaces(g.n, s);
    for (int t0 = 0; t0 < nc; t0 += 32) {
        const int t = t0 + lane;
        bool emit = false;
        u64 key = 0;
        if (t < nc) {
            uint32_t y; uint8_t perm[PT_NMAX];
            pt_cellcoface(g.n, s, t, y, perm);
            int base[PT_NMAX];
            pt_apply_masks(g.n, u, 0u, y, base);
            u64 bk;
            if (!pt_pack_vertex(g, base, bk)) { atomicOr(err, PT_ERR_KEY_RANGE); bk = 0; }
            key = pt_cell_key(bk, pt_perm_rank(g.n, perm));
            const unsigned slot = (unsigned)(pt_mix(key) & seen_mask);
            emit = atomicExch((unsigned long long*)&seen[slot], (unsigned long long)(key + 1)) != (unsigned long long)(key + 1);
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, emit);
        if (ballot) {
            const int leader = __ffs(ballot) - 1;
            unsigned long long base_out = 0;
            if (lane == leader) base_out = atomicAdd(n_out, (unsigned long long)__popc(ballot));
            base_out = __shfl_sync(0xffffffffu, base_out, leader);
            if (emit) keys[base_out + __popc(ballot & ((1u << lane) - 1u))] = key;
        }
    }
}

__global__ void pt_cell_unpack_kernel(PtGeom g, const u64* __restrict__ keys, size_t first, size_t count,
                                      int32_t* __restrict__ base, uint8_t* __restrict__ perm) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 k = keys[first + i];
    if (base) {
        int u[PT_NMAX];
        pt_unpack_vertex(g, k >> PT_CELL_RANK_BITS, u);
        for (int d = 0; d < g.n; ++d) base[i * g.n + d] = u[d];
    }
    if (perm) {
        uint8_t p[PT_NMAX];
        pt_perm_unrank(g.n, (uint32_t)(k & ((1u << PT_CELL_RANK_BITS) - 1u)), p);
        for (int d = 0; d < g.n; ++d) perm[i * g.n + d] = p[d];
    }
}

// per-axis min/max of the cell bases (one block, tiny output)
__global__ void pt_cell_bounds_kernel(PtGeom g, const u64* __restrict__ keys, size_t count, int* __restrict__ mn, int* __restrict__ mx) {
    int lmn[PT_NMAX], lmx[PT_NMAX];
    for (int d = 0; d < g.n; ++d) { lmn[d] = 0x7fffffff; lmx[d] = -0x7fffffff; }
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        int u[PT_NMAX];
        pt_unpack_vertex(g, keys[i] >> PT_CELL_RANK_BITS, u);
        for (int d = 0; d < g.n; ++d) { lmn[d] = min(lmn[d], u[d]); lmx[d] = max(lmx[d], u[d]); }
    }
    for (int d = 0; d < g.n; ++d) { atomicMin(&mn[d], lmn[d]); atomicMax(&mx[d], lmx[d]); }
}

static int pt_cells_bounds(pt_cells* c) {
    pt_ctx* ctx = c->ctx;
    for (int d = 0; d < PT_NMAX; ++d) { c->base_min[d] = 0; c->base_max[d] = 0; }
    if (c->count == 0) return PT_OK;
    PtBuf<int> mm;
    PT_TRY(mm.alloc(ctx, 2 * PT_NMAX));
    int init[2 * PT_NMAX];
    for (int d = 0; d < PT_NMAX; ++d) { init[d] = 0x7fffffff; init[PT_NMAX + d] = -0x7fffffff; }
    PT_CUDA(ctx, cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    pt_cell_bounds_kernel<<<pt_grid_for((size_t)c->count, 256, 1024), 256, 0, ctx->stream>>>(c->geom, c->keys.p, (size_t)c->count, mm.p, mm.p + PT_NMAX);
    PT_TRY(pt_check_launch(ctx, "pt_cell_bounds_kernel"));
    int out[2 * PT_NMAX];
    PT_CUDA(ctx, cudaMemcpyAsync(out, mm.p, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int d = 0; d < c->n; ++d) { c->base_min[d] = out[d]; c->base_max[d] = out[PT_NMAX + d]; }
    return PT_OK;
}

static int pt_cells_build(pt_ctx* ctx, const PtGeom& geom, const u64* edge_key_dev, size_t n_edges, pt_cells** out) {
    pt_cells* c = new pt_cells();
    c->ctx = ctx; c->n = geom.n; c->geom = geom;
    // cell bases may sit one unit below an edge base: widen the window by shifting the origin
    // (keys are re-packed relative to the shifted origin; the trace window keeps a 2-unit margin)
    const size_t E = n_edges;
    if (E == 0) { c->count = 0; int rc = c->keys.alloc(ctx, 1); if (rc != PT_OK) { delete c; return rc; } *out = c; return PT_OK; }
    PtBuf<unsigned long long> ncell, off;
    int rc = ncell.alloc(ctx, E + 1);
    if (rc == PT_OK) rc = off.alloc(ctx, E + 1);
    if (rc != PT_OK) { delete c; return rc; }
    {
        PT_LAUNCH(ctx, "cells_counts");
        pt_cell_counts_kernel<<<pt_grid_for(E + 1, 256), 256, 0, ctx->stream>>>(geom, edge_key_dev, E, ncell.p);
        rc = pt_check_launch(ctx, "pt_cell_counts_kernel");
    }
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ncell.p, off.p, (long long)(E + 1), ctx->stream);
    PtBuf<uint8_t> tmp;
    if (rc == PT_OK) rc = tmp.alloc(ctx, tb);
    if (rc != PT_OK) { delete c; return rc; }
    cub::DeviceScan::ExclusiveSum(tmp.p, tb, ncell.p, off.p, (long long)(E + 1), ctx->stream);
    ctx->launches++;
    unsigned long long* h = (unsigned long long*)ctx->pinned;
    cudaMemcpyAsync(h, off.p + E, sizeof(*h), cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { delete c; return pt_fail(ctx, PT_E_CUDA, "cell count scan failed"); }
    const size_t emitted = (size_t)*h;
    PtBuf<u64> raw, sorted, seen; PtBuf<unsigned> err; PtBuf<long long> nsel; PtBuf<unsigned long long> nkept;
    // "last key seen" filter: a power of two of 8-byte slots around the number of emitted keys / 4, at most 32 MB (L2)
    size_t slots = 1u << 12;
    while (slots < emitted / 4 && slots < ((size_t)1 << 22)) slots <<= 1;
    rc = raw.alloc(ctx, emitted);
    if (rc == PT_OK) rc = seen.alloc(ctx, slots);
    if (rc == PT_OK) rc = err.alloc(ctx, 1);
    if (rc == PT_OK) rc = nsel.alloc(ctx, 1);
    if (rc == PT_OK) rc = nkept.alloc(ctx, 1);
    if (rc != PT_OK) { delete c; return rc; }
    cudaMemsetAsync(err.p, 0, sizeof(unsigned), ctx->stream);
    cudaMemsetAsync(nkept.p, 0, sizeof(unsigned long long), ctx->stream);
    cudaMemsetAsync(seen.p, 0, slots * sizeof(u64), ctx->stream);          // stored values are key + 1, so 0 = empty
    {
        PT_LAUNCH(ctx, "cells_cofaces");
        pt_cell_cofaces_kernel<<<pt_grid_for(E * 32, 256), 256, 0, ctx->stream>>>(geom, edge_key_dev, E, seen.p, (unsigned)(slots - 1),
                                                                                 raw.p, nkept.p, err.p);
        rc = pt_check_launch(ctx, "pt_cell_cofaces_kernel");
        if (rc != PT_OK) { delete c; return rc; }
    }
    cudaMemcpyAsync(h, nkept.p, sizeof(*h), cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { delete c; return pt_fail(ctx, PT_E_CUDA, "cell coface enumeration failed"); }
    const size_t total = (size_t)*h;
    rc = sorted.alloc(ctx, total > 0 ? total : 1);
    if (rc != PT_OK) { delete c; return rc; }
    const int key_bits = geom.n * geom.bits + PT_CELL_RANK_BITS;
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, raw.p, sorted.p, (long long)total, 0, key_bits, ctx->stream);
    cub::DeviceSelect::Unique(nullptr, tb2, sorted.p, raw.p, nsel.p, (long long)total, ctx->stream);
    rc = tmp.alloc(ctx, tb1 > tb2 ? tb1 : tb2);
    if (rc != PT_OK) { delete c; return rc; }
    {
        PT_LAUNCH(ctx, "cells_sort");
        cub::DeviceRadixSort::SortKeys(tmp.p, tb1, raw.p, sorted.p, (long long)total, 0, key_bits, ctx->stream);
        ctx->launches++;
    }
    {
        PT_LAUNCH(ctx, "cells_unique");
        cub::DeviceSelect::Unique(tmp.p, tb2, sorted.p, raw.p, nsel.p, (long long)total, ctx->stream);
        ctx->launches++;
    }
    long long* hs = (long long*)ctx->pinned;
    unsigned* he = (unsigned*)((char*)ctx->pinned + 64);
    cudaMemcpyAsync(hs, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(he, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { delete c; return pt_fail(ctx, PT_E_CUDA, "cell sort failed: %s", cudaGetErrorString(cudaGetLastError())); }
    if (*he & PT_ERR_KEY_RANGE) { delete c; return pt_fail(ctx, PT_E_RANGE, "cell bases left the packed-key window"); }
    c->count = *hs;
    rc = c->keys.alloc(ctx, (size_t)(c->count > 0 ? c->count : 1));
    if (rc != PT_OK) { delete c; return rc; }
    cudaMemcpyAsync(c->keys.p, raw.p, (size_t)c->count * sizeof(u64), cudaMemcpyDeviceToDevice, ctx->stream);
    rc = pt_cells_bounds(c);
    if (rc != PT_OK) { delete c; return rc; }
    *out = c;
    return PT_OK;
}


extern "C" {

int pt_cells_from_trace(pt_trace* t, pt_cells** out) {
    if (!t || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_cells_from_trace: NULL argument");
    return pt_cells_build(t->ctx, t->geom, t->edge_key.p, (size_t)t->n_edges, out);
}

int pt_cells_from_edges(pt_ctx* ctx, int n, const int32_t* base, const uint32_t* mask, long long count, pt_cells** out) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_cells_from_edges: NULL argument");
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", n);
    if (count < 0) return pt_fail(ctx, PT_E_INVALID, "negative edge count");
    if (count > 0 && (!base || !mask)) return pt_fail(ctx, PT_E_INVALID, "edge arrays are NULL");
    if (pt_is_device_ptr(base) || pt_is_device_ptr(mask)) return pt_fail(ctx, PT_E_INVALID, "pt_cells_from_edges expects host arrays");
    PtGeom g;
    memset(&g, 0, sizeof(g));
    g.n = n; g.bits = pt_bits_for_dim(n); g.scale = 1.0;
    int mn[PT_NMAX], mx[PT_NMAX];
    for (int d = 0; d < n; ++d) { mn[d] = 0x7fffffff; mx[d] = -0x7fffffff; }
    for (long long i = 0; i < count; ++i)
        for (int d = 0; d < n; ++d) { int v = base[i * n + d]; if (v < mn[d]) mn[d] = v; if (v > mx[d]) mx[d] = v; }
    if (count == 0) for (int d = 0; d < n; ++d) { mn[d] = 0; mx[d] = 0; }
    for (int d = 0; d < n; ++d) {
        g.origin[d] = mn[d] - 2;
        if ((long long)mx[d] + 2 - g.origin[d] >= (1ll << g.bits))
            return pt_fail(ctx, PT_E_RANGE, "edges span more than %lld lattice units on axis %d (n=%d)", (1ll << g.bits), d, n);
    }
    std::vector<u64> keys((size_t)(count > 0 ? count : 1));
    for (long long i = 0; i < count; ++i) {
        int v[PT_NMAX];
        for (int d = 0; d < n; ++d) v[d] = base[i * n + d];
        if (mask[i] == 0 || mask[i] >= (1u << n)) return pt_fail(ctx, PT_E_INVALID, "edge %lld: bad step mask", i);
        u64 bk;
        pt_pack_vertex(g, v, bk);
        keys[(size_t)i] = pt_edge_key(g, bk, mask[i]);
    }
    PtBuf<u64> dev;
    PT_TRY(dev.alloc(ctx, keys.size()));
    PT_CUDA(ctx, cudaMemcpyAsync(dev.p, keys.data(), keys.size() * sizeof(u64), cudaMemcpyHostToDevice, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return pt_cells_build(ctx, g, dev.p, (size_t)count, out);
}

int pt_cells_from_host(pt_ctx* ctx, int n, const int32_t* base, const uint8_t* perm, long long count, pt_cells** out) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_cells_from_host: NULL argument");
    if (n < 2 || n > 7) return pt_fail(ctx, PT_E_INVALID, "dimension %d unsupported (2..7)", n);
    if (count < 0) return pt_fail(ctx, PT_E_INVALID, "negative cell count");
    if (count > 0 && (!base || !perm)) return pt_fail(ctx, PT_E_INVALID, "cell arrays are NULL");
    if (pt_is_device_ptr(base) || pt_is_device_ptr(perm)) return pt_fail(ctx, PT_E_INVALID, "pt_cells_from_host expects host arrays");
    pt_cells* c = new pt_cells();
    c->ctx = ctx; c->n = n; c->count = count;
    memset(&c->geom, 0, sizeof(c->geom));
    c->geom.n = n; c->geom.bits = pt_bits_for_dim(n); c->geom.scale = 1.0;
    for (int d = 0; d < n; ++d) { c->base_min[d] = 0x7fffffff; c->base_max[d] = -0x7fffffff; }
    for (long long i = 0; i < count; ++i)
        for (int d = 0; d < n; ++d) {
            int v = base[i * n + d];
            if (v < c->base_min[d]) c->base_min[d] = v;
            if (v > c->base_max[d]) c->base_max[d] = v;
        }
    if (count == 0) for (int d = 0; d < n; ++d) { c->base_min[d] = 0; c->base_max[d] = 0; }
    for (int d = 0; d < n; ++d) {
        c->geom.origin[d] = c->base_min[d] - 1;
        if ((long long)c->base_max[d] - c->geom.origin[d] + 1 >= (1ll << c->geom.bits)) {
            delete c;
            return pt_fail(ctx, PT_E_RANGE, "cells span more than %lld lattice units on axis %d (n=%d)", (1ll << pt_bits_for_dim(n)), d, n);
        }
    }
    std::vector<u64> keys((size_t)(count > 0 ? count : 1));
    for (long long i = 0; i < count; ++i) {
        int v[PT_NMAX]; uint8_t p[PT_NMAX]; uint32_t seen = 0;
        for (int d = 0; d < n; ++d) { v[d] = base[i * n + d]; p[d] = perm[i * n + d]; if (p[d] < n) seen |= 1u << p[d]; }
        if (seen != (1u << n) - 1u) { delete c; return pt_fail(ctx, PT_E_INVALID, "cell %lld: labels are not a permutation of 0..%d", i, n - 1); }
        u64 bk;
        pt_pack_vertex(c->geom, v, bk);
        keys[(size_t)i] = pt_cell_key(bk, pt_perm_rank(n, p));
    }
    int rc = c->keys.alloc(ctx, keys.size());
    if (rc != PT_OK) { delete c; return rc; }
    cudaMemcpyAsync(c->keys.p, keys.data(), keys.size() * sizeof(u64), cudaMemcpyHostToDevice, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { delete c; return pt_fail(ctx, PT_E_CUDA, "cell upload failed"); }
    *out = c;
    return PT_OK;
}

int pt_cells_slice(const pt_cells* c, long long first, long long count, pt_cells** out) {
    if (!c || !out) return pt_fail(nullptr, PT_E_INVALID, "pt_cells_slice: NULL argument");
    pt_ctx* ctx = c->ctx;
    if (first < 0 || count < 0 || first + count > c->count) return pt_fail(ctx, PT_E_INVALID, "cell range out of bounds");
    pt_cells* s = new pt_cells();
    s->ctx = ctx; s->n = c->n; s->geom = c->geom; s->count = count;
    for (int d = 0; d < PT_NMAX; ++d) { s->base_min[d] = c->base_min[d]; s->base_max[d] = c->base_max[d]; }
    int rc = s->keys.alloc(ctx, (size_t)(count > 0 ? count : 1));
    if (rc != PT_OK) { delete s; return rc; }
    cudaMemcpyAsync(s->keys.p, c->keys.p + first, (size_t)count * sizeof(u64), cudaMemcpyDeviceToDevice, ctx->stream);
    *out = s;
    return PT_OK;
}

int pt_cells_keys(const pt_cells* c, long long first, long long count, unsigned long long* out) {
    if (!c || (count > 0 && !out)) return pt_fail(c ? c->ctx : nullptr, PT_E_INVALID, "pt_cells_keys: NULL argument");
    pt_ctx* ctx = c->ctx;
    if (first < 0 || count < 0 || first + count > c->count) return pt_fail(ctx, PT_E_INVALID, "cell range out of bounds");
    if (count == 0) return PT_OK;
    PT_CUDA(ctx, cudaMemcpyAsync(out, c->keys.p + first, (size_t)count * sizeof(u64), cudaMemcpyDefault, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_cells_merge_keys(const pt_cells* like, const unsigned long long* keys, long long count, pt_cells** out) {
    if (!like || !out || (count > 0 && !keys)) return pt_fail(like ? like->ctx : nullptr, PT_E_INVALID, "pt_cells_merge_keys: NULL argument");
    pt_ctx* ctx = like->ctx;
    if (count < 0) return pt_fail(ctx, PT_E_INVALID, "negative key count");
    pt_cells* c = new pt_cells();
    c->ctx = ctx; c->n = like->n; c->geom = like->geom; c->count = 0;
    struct Guard { pt_cells* c; bool keep = false; ~Guard() { if (!keep) delete c; } } guard{c};
    PT_TRY(c->keys.alloc(ctx, (size_t)(count > 0 ? count : 1)));
    if (count > 0) {
        PtBuf<u64> in, sorted; PtBuf<long long> nsel; PtBuf<uint8_t> tmp;
        const u64* kdev;
        PT_TRY(pt_stage_in(ctx, (const u64*)keys, (size_t)count, in, &kdev));
        PT_TRY(sorted.alloc(ctx, (size_t)count));
        PT_TRY(nsel.alloc(ctx, 1));
        const int key_bits = c->geom.n * c->geom.bits + PT_CELL_RANK_BITS;
        size_t tb1 = 0, tb2 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb1, kdev, sorted.p, count, 0, key_bits, ctx->stream);
        cub::DeviceSelect::Unique(nullptr, tb2, sorted.p, c->keys.p, nsel.p, count, ctx->stream);
        PT_TRY(tmp.alloc(ctx, tb1 > tb2 ? tb1 : tb2));
        {
            PT_LAUNCH(ctx, "cells_sort");
            PT_CUDA(ctx, cub::DeviceRadixSort::SortKeys(tmp.p, tb1, kdev, sorted.p, count, 0, key_bits, ctx->stream));
            ctx->launches++;
        }
        {
            PT_LAUNCH(ctx, "cells_unique");
            PT_CUDA(ctx, cub::DeviceSelect::Unique(tmp.p, tb2, sorted.p, c->keys.p, nsel.p, count, ctx->stream));
            ctx->launches++;
        }
        long long* hs = (long long*)ctx->pinned;
        PT_CUDA(ctx, cudaMemcpyAsync(hs, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        c->count = *hs;
    }
    PT_TRY(pt_cells_bounds(c));
    guard.keep = true;
    *out = c;
    return PT_OK;
}

void pt_cells_destroy(pt_cells* c) { delete c; }
long long pt_cells_count(const pt_cells* c) { return c ? c->count : -1; }

int pt_cells_get(const pt_cells* c, long long first, long long count, int32_t* base, uint8_t* perm) {
    if (!c) return pt_fail(nullptr, PT_E_INVALID, "cells is NULL");
    pt_ctx* ctx = c->ctx;
    if (first < 0 || count < 0 || first + count > c->count) return pt_fail(ctx, PT_E_INVALID, "cell range out of bounds");
    if (count == 0) return PT_OK;
    const int n = c->n;
    PtBuf<int32_t> tb; PtBuf<uint8_t> tp;
    int32_t* bdev = nullptr; uint8_t* pdev = nullptr;
    if (base) { if (pt_is_device_ptr(base)) bdev = base; else { PT_TRY(tb.alloc(ctx, (size_t)count * n)); bdev = tb.p; } }
    if (perm) { if (pt_is_device_ptr(perm)) pdev = perm; else { PT_TRY(tp.alloc(ctx, (size_t)count * n)); pdev = tp.p; } }
    pt_cell_unpack_kernel<<<pt_grid_for((size_t)count, 256), 256, 0, ctx->stream>>>(c->geom, c->keys.p, (size_t)first, (size_t)count, bdev, pdev);
    PT_TRY(pt_check_launch(ctx, "pt_cell_unpack_kernel"));
    if (base && bdev != base) PT_TRY(pt_copy_out(ctx, base, bdev, (size_t)count * n, false));
    if (perm && pdev != perm) PT_TRY(pt_copy_out(ctx, perm, pdev, (size_t)count * n, false));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

}  // extern "C"
