// Internal state of one BFS trace and of a cell list (shared by pt_trace.cu / pt_cells.cu /
// pt_refine.cu).  Not part of the C ABI.
#pragma once
#include "pt_internal.cuh"

struct PtCounters {
    unsigned long long n_pending;    // vertices queued for evaluation in the current chunk
    unsigned long long dropped;      // dropped_out_of_box (cumulative)
    unsigned long long candidates;   // (edge, coface) records (cumulative)
    unsigned long long markers;      // cell_edges stage outputs (cumulative)
    unsigned long long ambiguous;    // evaluated vertices with |F| < 1e-12*(sum|w|+|b|) (cumulative)
    unsigned int error;              // PT_ERR_* bits
    unsigned int pad;
};

struct PtHashTable {
    PtBuf<u64> ent;
    u64 capacity = 0;     // entries (power of two)
    u64 count = 0;        // host-tracked upper bound of occupied entries
    PtTable view() const { PtTable t; t.ent = ent.p; t.cap_mask = capacity - 1; return t; }
};

int pt_table_init(pt_ctx* ctx, PtHashTable& t, u64 capacity);
// make room for `extra` more keys at load factor <= 1/2 (rehashes when growing)
int pt_table_reserve(pt_ctx* ctx, PtHashTable& t, u64 extra);

struct pt_trace {
    pt_ctx* ctx = nullptr;
    const pt_field* field = nullptr;
    PtGeom geom;
    bool window_set = false;
    double box_lo_f[PT_NMAX], box_hi_f[PT_NMAX];
    long long max_edges = 0;
    double eps = 1e-9;

    PtHashTable visited;   // edge key -> admission index | pending slot | dead
    PtHashTable signs;     // vertex key -> 1 (F>0) / 0 (F<=0)

    PtBuf<u64> edge_key;       // admission order
    PtBuf<int8_t> edge_sa;     // sign at the base vertex
    long long n_edges = 0;
    PtBuf<uint32_t> frontier;  // indices into the edge list
    long long n_frontier = 0;
    long long expanded_upto = 0;   // edges [0, expanded_upto) have been expanded (trace() flow)
    bool range_frontier = true;    // frontier is the index range [n_edges - n_frontier, n_edges)

    PtBuf<PtCounters> counters;
    PtCounters host_counters;

    long long levels = 0, seeds = 0, field_evaluations = 0;
    bool complete = true;
    std::vector<long long> stages;   // rows of 5

    // adjacency cache
    PtBuf<u64> adj;
    long long n_adj = -1;

    // owner-hashed sharded BFS (pt_trace_shard / pt_trace_wave_*): this rank keeps the edges whose base lattice
    // vertex hashes to it; every local edge carries its GLOBAL admission index
    int rank = 0, world = 1;
    PtBuf<u64> edge_gidx;
    long long n_global = 0;        // edges admitted by all ranks so far
    PtBuf<u64> cand;               // [n_cand][2] (edge key, tag) of the current wave, bucketed by owner rank
    long long n_cand = 0;
    PtBuf<u64> win;                // [n_win][2] (tag, edge key) winners of the last admit, ascending tag
    long long n_win = 0;
};

struct pt_cells {
    pt_ctx* ctx = nullptr;
    int n = 0;
    PtGeom geom;            // window used to pack the cell keys
    PtBuf<u64> keys;        // pt_cell_key(vkey(base), perm_rank)
    long long count = 0;
    int base_min[PT_NMAX], base_max[PT_NMAX];
};

int pt_bits_for_dim(int n);
int pt_read_counters(pt_trace* t);
