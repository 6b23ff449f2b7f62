/* libpermatrace_b200 -- C ABI of the B200-native (sm_100a) manifold-tracing / refinement /
 * collision-checking hot path.  This is the drop-in boundary: plain pointers and sizes, no
 * exceptions, no torch types.  Every data pointer may be HOST or DEVICE memory (classified with
 * cudaPointerGetAttributes); results are written to the memory space of the output pointer.
 *
 * Each entry point names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/permatrace/).  Return value: PT_OK (0) or a negative PT_E_* code;
 * pt_last_error() returns the message of the calling thread's last failure.
 */
#ifndef PERMATRACE_B200_H
#define PERMATRACE_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PT_OK 0
#define PT_E_INVALID (-1)    /* bad argument (maps to ValueError) */
#define PT_E_CUDA (-2)       /* CUDA runtime failure (maps to RuntimeError) */
#define PT_E_RANGE (-3)      /* lattice window exceeds the packed-key range */
#define PT_E_LIMIT (-4)      /* configuration outside joint limits (maps to LimitError) */
#define PT_E_NOMEM (-5)      /* device memory exhausted */
#define PT_E_STATE (-6)      /* call sequence error */

typedef struct pt_ctx pt_ctx;
typedef struct pt_field pt_field;       /* an implicit manifold resident on the device */
typedef struct pt_checker pt_checker;   /* robot + scene resident on the device */
typedef struct pt_trace pt_trace;       /* one BFS trace (visited table, sign table, frontier) */
typedef struct pt_cells pt_cells;       /* sorted, deduplicated full-dimensional cells */
typedef struct pt_refine pt_refine;     /* result of one batch refinement */

/* ---- context ------------------------------------------------------------------------------ */
const char* pt_last_error(void);
int pt_version(void);
int pt_ctx_create(int device, pt_ctx** out);
void pt_ctx_destroy(pt_ctx* ctx);
/* run all work of this context on an existing CUDA stream (e.g. torch's current stream) */
int pt_ctx_set_stream(pt_ctx* ctx, void* cuda_stream);
int pt_ctx_synchronize(pt_ctx* ctx);
/* device blocks freed by the library are cached per context for reuse by the next step; this returns them
 * to the driver (bytes released, or -1) */
long long pt_ctx_trim(pt_ctx* ctx);
/* page-locked host blocks for large results (device->host copies into them run at full PCIe speed and need no
 * staging); freed blocks are cached per context.  pt_host_free may be called from any thread. */
void* pt_host_alloc(pt_ctx* ctx, long long bytes);
void pt_host_free(pt_ctx* ctx, void* p);
/* per-kernel CUDA-event profiler (events on the launching stream) */
int pt_ctx_profile_enable(pt_ctx* ctx, int on);
int pt_ctx_profile_reset(pt_ctx* ctx);
/* writes "name,launches,total_ms\n" lines; returns bytes needed (call with cap=0 to size) */
long long pt_ctx_profile_dump(pt_ctx* ctx, char* buf, long long cap);
long long pt_ctx_launch_count(pt_ctx* ctx);
/* device-side work counters, out[6]: [0] fp64 field evaluations of the main root-solve kernel (Newton
 * path, or plain bisection in fp64 mode), [1] points evaluated by the batch evaluator, [2] fp32-screened
 * bisection evaluations, [3] root solves handed to plain fp64 bisection, [4] fp64 evaluations spent there,
 * [5] fp64 single-step resolves; reset != 0 zeroes them */
int pt_ctx_work_counters(pt_ctx* ctx, long long* out, int reset);
/* fp64 field evaluations spent in proof retries of the root solve (rows whose first enclosure attempt failed),
 * as of the last pt_ctx_work_counters call */
long long pt_ctx_retry_evaluations(pt_ctx* ctx);
/* root solves (edges) that went through the one-pass Taylor-model kernel (csrc/pt_field_taylor.cuh), and of those the
 * ones it left to the evaluation-based kernels: out[3] of pt_ctx_work_counters; as of the last pt_ctx_work_counters call */
long long pt_ctx_taylor_rows(pt_ctx* ctx);
/* DFMA-chain microbenchmark: measured FP64 peak of this device in TFLOP/s (roofline denominator) */
double pt_peak_fp64(pt_ctx* ctx);
/* MUFU.EX2 microbenchmark: measured special-function peak in T ex2/s (roofline denominator of the fp32 screen) */
double pt_peak_ex2(pt_ctx* ctx);

/* ---- B1: the reference's kernel plugin seam (backend.py:30-33, _kernels.pyx) ---------------- */
/* _kernels.pyx:18-40 rbf_values(points[m,n], support[S,n], weights[S], gamma, bias) -> out[m] */
int pt_rbf_values(pt_ctx* ctx, const double* points, long long m, int n, const double* support,
                  long long S, const double* weights, double gamma, double bias, double* out);
/* _kernels.pyx:43-76 sphere_box_hits(centers[m,3], radii[m], lx, ly, lz) -> out[m] (uint8) */
int pt_sphere_box_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m,
                       double lx, double ly, double lz, uint8_t* out);
/* _kernels.pyx:79-104 sphere_cylinder_hits(centers, radii, height, radius) */
int pt_sphere_cylinder_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m,
                            double height, double radius, uint8_t* out);
/* _kernels.pyx:107-122 sphere_sphere_hits(centers, radii, radius) */
int pt_sphere_sphere_hits(pt_ctx* ctx, const double* centers, const double* radii, long long m,
                          double radius, uint8_t* out);

/* ---- implicit manifolds (manifold.py:49-217) ------------------------------------------------ */
#define PT_FIELD_RBF 0        /* KernelClassifierManifold (manifold.py:177-208) */
#define PT_FIELD_SPHERE 1     /* SphereManifold (manifold.py:75-95) */
#define PT_FIELD_ELLIPSOID 2  /* EllipsoidManifold (manifold.py:98-120) */
#define PT_FIELD_PLANE 3      /* PlaneManifold (manifold.py:123-140) */
/* KernelClassifierManifold(support, weights, gamma, bias, barrier); barrier = NULL or
 * [scale, gain, lower[n], upper[n]] (BoxBarrier, manifold.py:143-169).  Host pointers. */
int pt_field_create_rbf(pt_ctx* ctx, int n, long long S, const double* support,
                        const double* weights, double gamma, double bias, const double* barrier,
                        pt_field** out);
/* analytic fields: params = sphere [center[n], radius^2]; ellipsoid [center[n], semi_axes[n]];
 * plane [normal[n], offset].  Host pointers. */
int pt_field_create_analytic(pt_ctx* ctx, int kind, int n, const double* params, pt_field** out);
void pt_field_destroy(pt_field* f);
/* precision policy (default 1; environment PERMATRACE_B200_PRECISION overrides at creation):
 *   0 = plain FP64 everywhere (bisection exactly as the reference loop, manifold.py:368-383);
 *   1 = fast path with the same results: FP32 screening on the tensor cores (tcgen05, tf32 x3 split) where the FP32 sign
 *       is PROVEN equal to the FP64 one, FP64 recheck of every unproven value, Newton root location with a rigorous
 *       enclosure that replays the reference's bisection decisions.
 * PERMATRACE_B200_TC=0 keeps mode 1 on the SIMT kernels; PERMATRACE_B200_TC_LEVELS=1 forces the level-synchronous
 * tensor-core driver that serves support sets beyond one CTA's shared memory; PERMATRACE_B200_TC4=0 selects the
 * two-group screen kernel where the four-group one (n = 6, resident support set) would run;
 * PERMATRACE_B200_RETRY_RATIO (default 8) is the enclosure-width / noise-width ratio above which an open row retries
 * the proof from its replayed bracket instead of evaluating its open midpoints one by one.  None of these changes a
 * result. */
int pt_field_set_precision(pt_field* f, int mode);
/* ImplicitManifold.values / .signs (manifold.py:54-72): out_values (f64) and out_signs (i8, +1/-1)
 * may each be NULL */
int pt_field_values(pt_ctx* ctx, const pt_field* f, const double* points, long long m,
                    double* out_values, int8_t* out_signs);
/* KernelClassifierManifold.gradient (manifold.py:210-217), batched: out[m, n] */
int pt_field_gradients(pt_ctx* ctx, const pt_field* f, const double* points, long long m, double* out);
/* intersection_points_batch(manifold, a, b, eps, signs_a) (manifold.py:351-383); signs_a NULL ->
 * evaluated at a */
int pt_intersection_points(pt_ctx* ctx, const pt_field* f, const double* a, const double* b,
                           long long m, double eps, const int8_t* signs_a, double* out);

/* test hook of the tensor-core (tcgen05) fp32 screen: for the midpoint of each segment a[i]..b[i], out[i] =
 * max over the support set of |exponent computed on the tensor cores - exponent in fp64|, in units of
 * 2^-24 * gamma*log2(e)*(|p|+max|s|)^2 (the unit of the screen's error bound).  PT_E_STATE if the field has no
 * tensor-core operand (support set too large for one CTA's shared memory, n > 6, or PERMATRACE_B200_TC=0). */
int pt_debug_tc_arg_error(pt_ctx* ctx, const pt_field* f, const double* a, const double* b, long long m,
                          double* out);

/* ---- collision (collision.py:191-329, pipeline.py:256-270) --------------------------------- */
/* Robot: joints[nj]: kind (0 revolute, 1 prismatic), axis[3] (unit), origin rotation[9] row-major,
 * origin translation[3], limits[2]; spheres[ns]: link, offset[3], radius.
 * Scene: obstacles[no]: type (0 box, 1 cylinder, 2 sphere), rotation[9], translation[3],
 * dims[3] (box lx,ly,lz | cylinder height,radius,- | sphere radius,-,-).  Host pointers. */
int pt_checker_create(pt_ctx* ctx, int nj, const int* joint_kind, const double* joint_axis,
                      const double* joint_rot, const double* joint_trans, const double* joint_limits,
                      int ns, const int* sphere_link, const double* sphere_offset,
                      const double* sphere_radius, int no, const int* obs_type,
                      const double* obs_rot, const double* obs_trans, const double* obs_dims,
                      pt_checker** out);
void pt_checker_destroy(pt_checker* ck);
/* fk_batch (collision.py:204-225): centers out[m, ns, 3] */
int pt_fk_batch(pt_ctx* ctx, const pt_checker* ck, const double* configs, long long m,
                double* out_centers);
#define PT_LIMIT_ERROR 0   /* batch_check(on_limit="error"): PT_E_LIMIT, *first_bad = row */
#define PT_LIMIT_UNFREE 1  /* batch_check(on_limit="unfree") == _not_free_checker */
#define PT_LIMIT_IGNORE 2  /* _batch_hits: no limit test */
/* batch_check (collision.py:306-329): out[m] uint8 in-collision mask */
int pt_batch_check(pt_ctx* ctx, const pt_checker* ck, const double* configs, long long m,
                   int on_limit, uint8_t* out, long long* first_bad);

/* ---- tracer (tracer.py:152-452) ------------------------------------------------------------- */
typedef struct pt_trace_stats {
    long long levels, seeds, visited_edges, field_evaluations, dropped_out_of_box;
    long long candidates;        /* sum of (edge, coface) records expanded */
    long long frontier;          /* current frontier size */
    int complete, closure_ok;
    long long table_capacity, sign_table_capacity;
    long long n_stages;          /* StageStat rows available through pt_trace_stages */
    /* evaluated lattice vertices with |F| < 1e-12*(sum|w|+|bias|), the reference's own cross-backend tolerance on the
     * kernel sum (pkg/tests/test_backends.py:81-93): only there can a sign -- hence the traced set -- differ from the
     * reference's.  0 for analytic fields. */
    long long ambiguous_signs;
} pt_trace_stats;

/* TraceConfig(lattice=LatticeConfig(n, scale, offset), box, max_edges, eps) (tracer.py:43-59).
 * box_lo/box_hi NULL -> no clamp.  window_center: lattice-unit centre of the packed-key window
 * when no box is given (NULL -> centred on the first seed). */
int pt_trace_create(pt_ctx* ctx, const pt_field* field, int n, double scale, const double* offset,
                    const double* box_lo, const double* box_hi, long long max_edges, double eps,
                    pt_trace** out);
void pt_trace_destroy(pt_trace* t);
/* _Tracer.locate + admit_frontier (tracer.py:256-306) */
int pt_trace_locate(pt_trace* t, const double* seeds, long long m);
/* _Tracer.expand (tracer.py:322-380): one BFS wave; *frontier_out = new frontier size */
int pt_trace_expand(pt_trace* t, long long* frontier_out);
/* trace() (tracer.py:436-452): locate, then expand until the frontier empties or the cap hits */
int pt_trace_run(pt_trace* t, const double* seeds, long long m);
/* seed the visited set + frontier directly from canonical edges (expand_frontier, tracer.py:418-433):
 * base[m,n] int32, mask[m] uint32; the first n_visited rows are "visited", the rest the frontier
 * (rows already present are skipped). */
int pt_trace_seed_edges(pt_trace* t, const int32_t* base, const uint32_t* mask, long long n_visited,
                        long long n_frontier);
int pt_trace_get_stats(pt_trace* t, pt_trace_stats* out);
/* StageStat rows (tracer.py:74-80): out[rows,5] = kind (0 locate_cells,1 cell_edges,2 edge_cofaces,
 * 3 coface_partner), level, items, capacity, produced */
int pt_trace_stages(pt_trace* t, long long* out, long long rows);
/* edges in admission order: base[E,n] int32, mask[E] uint32 (bit d set <=> label d in p1),
 * sign_a[E] int8 (sign at the base vertex); any pointer may be NULL.  Rows [first, first+count). */
int pt_trace_edges(pt_trace* t, long long first, long long count, int32_t* base, uint32_t* mask,
                   int8_t* sign_a);
/* frontier rows (indices into the edge list) of the current frontier */
int pt_trace_frontier(pt_trace* t, long long* first, long long* count);
/* _Tracer.result (tracer.py:384-395): one bisection point per edge, out[E,n] */
int pt_trace_points(pt_trace* t, double* out);
/* sorted unique adjacency pairs (tracer.py:249-251,398): returns count; pairs[count,2] int64 when
 * pairs != NULL (call once with NULL to size) */
long long pt_trace_adjacency(pt_trace* t, long long* pairs, long long cap);

/* ---- owner-hashed sharded BFS (multi-GPU) ------------------------------------------
 * Rank r of `world` owns the canonical edges whose base lattice vertex hashes to r.  Per wave the caller runs
 * candidates -> all_to_all of the 16-byte records -> admit -> rank the winner tags across ranks -> commit.
 * A record is two 64-bit words (packed edge key, tag); tag = ((global admission index of the parent edge * stride
 * + coface ordinal) << 1) | (sign at base > 0), i.e. the reference's slot order (tracer.py:359-375), comparable
 * across ranks.  The trace must have a clamp box (all ranks pack keys in the same window). */
/* after pt_trace_locate (run identically on every rank): keep the owned edges, remember their global indices */
int pt_trace_shard(pt_trace* t, int rank, int world);
/* expand the local frontier; counts[world] = records per owner rank (bucketed in that order) */
int pt_trace_wave_candidates(pt_trace* t, long long* counts);
/* the bucketed records of the last pt_trace_wave_candidates: out[sum(counts)][2] (host or device) */
int pt_trace_wave_fetch(pt_trace* t, long long* out);
/* owner side: records[count][2] received from all ranks (host or device); *n_winners = new edges owned here */
int pt_trace_wave_admit(pt_trace* t, const long long* records, long long count, long long* n_winners);
/* tags of the winners of the last admit, ascending: out[n_winners] */
int pt_trace_wave_winner_tags(pt_trace* t, long long* out);
/* gidx[n_winners] = global admission index of each winner (tag order), -1 for winners beyond max_edges (they
 * must be a suffix); alive = number of non-negative entries; global_total = edges admitted by all ranks so far */
int pt_trace_wave_commit(pt_trace* t, const long long* gidx, long long alive, long long global_total);
/* global admission indices of local edges [first, first+count) */
int pt_trace_gidx(pt_trace* t, long long first, long long count, long long* out);

/* ---- coarse cells (subdivision.py:132-141, lattice.py:245-266) ------------------------------ */
int pt_cells_from_trace(pt_trace* t, pt_cells** out);
/* same from canonical edges given on the host: base[E,n] int32, mask[E] uint32 */
int pt_cells_from_edges(pt_ctx* ctx, int n, const int32_t* base, const uint32_t* mask, long long count,
                        pt_cells** out);
/* cells given by the caller in processing order: base[C,n] int32, perm[C,n] uint8 */
int pt_cells_from_host(pt_ctx* ctx, int n, const int32_t* base, const uint8_t* perm, long long count,
                       pt_cells** out);
/* contiguous sub-range of a cell list (multi-GPU sharding of refine) */
int pt_cells_slice(const pt_cells* c, long long first, long long count, pt_cells** out);
/* packed 64-bit keys of cells [first, first+count) (numeric order = the reference's (base, parts) tuple order inside one
 * key window); `out` may be host or device memory.  With pt_cells_merge_keys -- sort + unique of keys packed in the window
 * of `like` -- this is what the range-partitioned (sample-sort) build of the sorted cell list across GPUs exchanges
 * (order contract: reference subdivision.py:141) */
int pt_cells_keys(const pt_cells* c, long long first, long long count, unsigned long long* out);
int pt_cells_merge_keys(const pt_cells* like, const unsigned long long* keys, long long count, pt_cells** out);
void pt_cells_destroy(pt_cells* c);
long long pt_cells_count(const pt_cells* c);
int pt_cells_get(const pt_cells* c, long long first, long long count, int32_t* base, uint8_t* perm);

/* ---- refine (subdivision.py:220-301) -------------------------------------------------------- */
typedef struct pt_refine_stats {
    long long cells, fine_vertices, crossing_edges, unique_fine_vertices, unique_fine_edges,
        points, in_collision, free_points, dedup_rounds, field_evaluations;
    long long ambiguous_signs;   /* fine vertices with |F| below the same tolerance as pt_trace_stats.ambiguous_signs */
} pt_refine_stats;
/* template: tv[V,n] int32 vertices (lex sorted), te[E,2] int32 edges; k subdivision factor;
 * lattice (n, scale, offset) is the COARSE lattice of the cells; checker NULL -> labels all 0 and
 * the caller labels the points itself.  batch_bounds[nb+1] (cell index boundaries, may be NULL)
 * only shapes the per-batch statistics: results never depend on it. */
int pt_refine_run(pt_ctx* ctx, const pt_field* field, const pt_cells* cells, int n, double scale,
                  const double* offset, int k, int V, const int32_t* tv, int E, const int32_t* te,
                  double eps, double eps_dedup, const pt_checker* checker,
                  const long long* batch_bounds, int nb, pt_refine** out);
/* multi-GPU building blocks: (1) refinement of a cell slice up to and including the root solves --
 * the result holds one point per distinct fine edge in first-crossing order (first_tag = crossing index
 * local to the slice), no dedup, no labels; (2) greedy first-keeper dedup at eps_dedup over points given
 * in priority order + collision labels (first_tag = position in the input). */
int pt_refine_candidates(pt_ctx* ctx, const pt_field* field, const pt_cells* cells, int n, double scale,
                         const double* offset, int k, int V, const int32_t* tv, int E, const int32_t* te,
                         double eps, pt_refine** out);
int pt_dedup_label(pt_ctx* ctx, int n, const double* points, long long count, double eps_dedup,
                   const pt_checker* checker, pt_refine** out);
/* same, with the state of some points given: forced[i] = 1 kept, 0 removed, -1 decide here.  A rank of the sharded
 * eps-dedup runs it over its own candidates plus ghost copies of its neighbours' boundary points, the ghosts pinned to
 * their owners' verdicts (distributed.py; the greedy rule of reference subdivision.py:195-217 has one fixed point) */
int pt_dedup_label_forced(pt_ctx* ctx, int n, const double* points, long long count, double eps_dedup,
                          const int8_t* forced, const pt_checker* checker, pt_refine** out);
void pt_refine_destroy(pt_refine* r);
int pt_refine_get_stats(const pt_refine* r, pt_refine_stats* out);
/* points[P,n] f64, labels[P] uint8 (1 = not free), first_tag[P] int64 (global crossing index of the
 * point's first occurrence); any may be NULL */
int pt_refine_points(const pt_refine* r, double* points, uint8_t* labels, long long* first_tag);
/* per-batch rows out[nb,2] = crossing_edges, new_points */
int pt_refine_batch_stats(const pt_refine* r, long long* out, int nb);
/* overwrite labels (used when the checker is an arbitrary host callable) */
int pt_refine_set_labels(pt_refine* r, const uint8_t* labels);

/* ---- host-executable mirrors of the device lattice arithmetic (tests, no GPU needed) -------- */
/* expansion plan of edge type `mask` in dimension n (tracer.py:123-149): rows of 10 int32:
 * c_plus,c_minus, bc_bplus,bc_bminus,bc_mask,bc_shared, ac_bplus,ac_bminus,ac_mask,ac_shared */
int pt_host_expansion_plan(int n, uint32_t mask, int32_t* out, int cap);
/* cell cofaces of edge type `mask` (lattice.py:245-258): rows of (1+n) int32: y_mask, perm[n] */
int pt_host_cellcofaces(int n, uint32_t mask, int32_t* out, int cap);
int pt_host_perm_rank(int n, const uint8_t* perm);
int pt_host_perm_unrank(int n, int rank, uint8_t* perm);

#ifdef __cplusplus
}
#endif
#endif
