// Host-side internals of libpermatrace_b200: context, error plumbing, stream-ordered device
// buffers, per-kernel CUDA-event profiler.  Nothing here crosses the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <string>
#include <vector>
#include <map>
#include <mutex>
#include "pt_common.cuh"
#include "../../include/permatrace_b200.h"

struct PtProfEntry {
    double total_ms = 0.0;
    long long launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

struct pt_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string last_error;
    bool profiling = false;
    std::map<std::string, PtProfEntry> prof;
    std::vector<cudaEvent_t> event_pool;
    long long launches = 0;            // total kernel launches issued by this library
    int sm_count = 148;
    // device-side work counters: [0] bisection field evaluations (rows x iterations), [1] points evaluated
    unsigned long long* work = nullptr;
    long long retry_evals = 0;           // snapshot taken by pt_ctx_work_counters
    long long taylor_rows = 0;           // ditto: rows of the one-pass Taylor-model root solve (work[7])
    // where the sign evaluator counts ambiguous vertices (|F| < 1e-12*(sum|w|+|b|)); work + 6 unless a trace / refinement
    // points it at its own counter block for the duration of a call (PtAmbScope)
    unsigned long long* amb_sink = nullptr;
    // size-bucketed cache of device blocks (all work is ordered on `stream`, so a freed block can be handed
    // out again at once): after the first step the hot path makes no driver allocation calls at all
    std::multimap<size_t, void*> free_blocks;
    std::map<void*, size_t> live_blocks;
    size_t cached_bytes = 0;
    // cache of pinned host blocks handed to the caller for large results (pt_host_alloc); finalizers of the host
    // language may free from another thread, hence the lock
    std::mutex host_lock;
    std::multimap<size_t, void*> host_free_blocks;
    std::map<void*, size_t> host_live_blocks;
    // pinned scratch for small device->host readbacks (counters)
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
};

extern thread_local std::string g_pt_last_error;

int pt_fail(pt_ctx* ctx, int code, const char* fmt, ...);

#define PT_CUDA(ctx, expr)                                                                  \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return pt_fail((ctx), PT_E_CUDA, "%s failed: %s (%s:%d)", #expr,                \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                     \
    } while (0)

#define PT_TRY(expr)                                \
    do {                                            \
        int _rc = (expr);                           \
        if (_rc != PT_OK) return _rc;               \
    } while (0)

// stream-ordered allocation; the default pool keeps freed blocks (release threshold = max)
int pt_dev_alloc(pt_ctx* ctx, void** p, size_t bytes);
void pt_dev_free(pt_ctx* ctx, void* p);

// RAII device buffer (stream-ordered)
template <typename T>
struct PtBuf {
    pt_ctx* ctx = nullptr;
    T* p = nullptr;
    size_t count = 0;
    PtBuf() {}
    PtBuf(const PtBuf&) = delete;
    PtBuf& operator=(const PtBuf&) = delete;
    ~PtBuf() { release(); }
    void release() { if (p) { pt_dev_free(ctx, p); p = nullptr; count = 0; } }
    int alloc(pt_ctx* c, size_t n) {
        release(); ctx = c; count = n;
        if (n == 0) n = 1;
        return pt_dev_alloc(c, (void**)&p, n * sizeof(T));
    }
    // grow keeping contents
    int ensure(pt_ctx* c, size_t n, size_t keep) {
        if (n <= count && p) return PT_OK;
        size_t want = count ? count : 1;
        while (want < n) want *= 2;
        T* q = nullptr; ctx = c;
        int rc = pt_dev_alloc(c, (void**)&q, want * sizeof(T));
        if (rc != PT_OK) return rc;
        if (p && keep) cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, c->stream);
        if (p) pt_dev_free(c, p);
        p = q; count = want;
        return PT_OK;
    }
};

// classify a user pointer: true if it is device (or managed) memory
bool pt_is_device_ptr(const void* p);

// copy-in helper: returns a device pointer for `src` (staging through `tmp` if src is host memory)
template <typename T>
int pt_stage_in(pt_ctx* ctx, const T* src, size_t count, PtBuf<T>& tmp, const T** out) {
    if (count == 0) { PT_TRY(tmp.alloc(ctx, 1)); *out = tmp.p; return PT_OK; }
    if (pt_is_device_ptr(src)) { *out = src; return PT_OK; }
    PT_TRY(tmp.alloc(ctx, count));
    PT_CUDA(ctx, cudaMemcpyAsync(tmp.p, src, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    *out = tmp.p;
    return PT_OK;
}
// copy-out helper: dst may be host or device
template <typename T>
int pt_copy_out(pt_ctx* ctx, T* dst, const T* src_dev, size_t count, bool sync = true) {
    if (count) {
        cudaMemcpyKind kind = pt_is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        PT_CUDA(ctx, cudaMemcpyAsync(dst, src_dev, count * sizeof(T), kind, ctx->stream));
    }
    if (sync) PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

// redirect the ambiguous-sign counter for the lifetime of the scope
struct PtAmbScope {
    pt_ctx* ctx; unsigned long long* prev;
    PtAmbScope(pt_ctx* c, unsigned long long* sink) : ctx(c), prev(c->amb_sink) { c->amb_sink = sink; }
    ~PtAmbScope() { ctx->amb_sink = prev; }
};

// profiler: bracket one launch with events when ctx->profiling
struct PtProfScope {
    pt_ctx* ctx; const char* name; cudaEvent_t e0 = nullptr, e1 = nullptr;
    PtProfScope(pt_ctx* c, const char* n);
    ~PtProfScope();
};
#define PT_LAUNCH(ctx, name) PtProfScope _pt_scope_##__LINE__((ctx), (name))

int pt_check_launch(pt_ctx* ctx, const char* what);

static inline unsigned pt_grid_for(size_t items, unsigned block, unsigned max_blocks = 0x7fffffffu) {
    size_t g = (items + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (unsigned)g;
}

// ---- internal device-level services used across translation units ------------------------------
struct PtFieldDev;   // pt_field.cuh
struct pt_field;
struct pt_checker;

// evaluate field at m device points (row-major m x n); vals/signs may be null
// (vals32_dev: optional fp32 copy of the values -- whatever precision the sign evaluation ran in; learned fields only)
int pt_field_eval_dev(pt_ctx* ctx, const pt_field* f, const double* pts_dev, size_t m,
                      double* vals_dev, int8_t* signs_dev, float* vals32_dev = nullptr);
// bisection on m device segments (hint_dev: optional estimate of the root's position on each segment, in [0, 1]; it only
// places the centre of the Taylor model and never changes the result)
int pt_field_bisect_dev(pt_ctx* ctx, const pt_field* f, const double* a_dev, const double* b_dev,
                        const int8_t* signs_a_dev, size_t m, double eps, double* out_dev, const float* hint_dev = nullptr);
// non-free mask for m device configurations (limits + collision), out_dev: uint8
int pt_checker_run_dev(pt_ctx* ctx, const pt_checker* ck, const double* q_dev, size_t m, int mode,
                       uint8_t* out_dev, long long* first_bad_host);
int pt_field_dim(const pt_field* f);
