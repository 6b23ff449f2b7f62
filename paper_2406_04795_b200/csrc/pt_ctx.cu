// Context, error reporting, stream-ordered allocation and the CUDA-event kernel profiler.
#include <stdarg.h>
#include "pt_internal.cuh"

thread_local std::string g_pt_last_error;

int pt_fail(pt_ctx* ctx, int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_pt_last_error = buf;
    if (ctx) ctx->last_error = buf;
    return code;
}

bool pt_is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

int pt_dev_alloc(pt_ctx* ctx, void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(p, bytes, ctx->stream);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return pt_fail(ctx, PT_E_NOMEM, "device allocation of %zu bytes failed", bytes);
    }
    if (e != cudaSuccess) return pt_fail(ctx, PT_E_CUDA, "cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
    return PT_OK;
}
void pt_dev_free(pt_ctx* ctx, void* p) {
    if (p) cudaFreeAsync(p, ctx ? ctx->stream : nullptr);
}

int pt_check_launch(pt_ctx* ctx, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return pt_fail(ctx, PT_E_CUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
    ctx->launches++;
    return PT_OK;
}

PtProfScope::PtProfScope(pt_ctx* c, const char* n) : ctx(c), name(n) {
    if (!ctx->profiling) return;
    auto get = [&]() {
        cudaEvent_t e;
        if (!ctx->event_pool.empty()) { e = ctx->event_pool.back(); ctx->event_pool.pop_back(); }
        else cudaEventCreate(&e);
        return e;
    };
    e0 = get(); e1 = get();
    cudaEventRecord(e0, ctx->stream);
}
PtProfScope::~PtProfScope() {
    if (!e0) return;
    cudaEventRecord(e1, ctx->stream);
    ctx->prof[name].pending.emplace_back(e0, e1);
}

static void pt_prof_collect(pt_ctx* ctx) {
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->prof) {
        for (auto& pr : kv.second.pending) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
                kv.second.total_ms += ms; kv.second.launches++;
            } else cudaGetLastError();
            ctx->event_pool.push_back(pr.first); ctx->event_pool.push_back(pr.second);
        }
        kv.second.pending.clear();
    }
}

extern "C" {

const char* pt_last_error(void) { return g_pt_last_error.c_str(); }
int pt_version(void) { return 100; }

int pt_ctx_create(int device, pt_ctx** out) {
    if (!out) return pt_fail(nullptr, PT_E_INVALID, "pt_ctx_create: out is NULL");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return pt_fail(nullptr, PT_E_CUDA, "no CUDA device available (%s); this library has no CPU path",
                       e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0");
    }
    if (device < 0 || device >= count) return pt_fail(nullptr, PT_E_INVALID, "device %d out of range (have %d)", device, count);
    pt_ctx* ctx = new pt_ctx();
    ctx->device = device;
    PT_CUDA(ctx, cudaSetDevice(device));
    PT_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) ctx->sm_count = prop.multiProcessorCount;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    ctx->pinned_bytes = 1 << 16;
    PT_CUDA(ctx, cudaMallocHost(&ctx->pinned, ctx->pinned_bytes));
    *out = ctx;
    return PT_OK;
}

void pt_ctx_destroy(pt_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->prof)
        for (auto& pr : kv.second.pending) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int pt_ctx_set_stream(pt_ctx* ctx, void* cuda_stream) {
    if (!ctx) return pt_fail(nullptr, PT_E_INVALID, "ctx is NULL");
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) { cudaStreamDestroy(ctx->stream); ctx->own_stream = false; }
    ctx->stream = (cudaStream_t)cuda_stream;
    return PT_OK;
}

int pt_ctx_synchronize(pt_ctx* ctx) {
    if (!ctx) return pt_fail(nullptr, PT_E_INVALID, "ctx is NULL");
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}

int pt_ctx_profile_enable(pt_ctx* ctx, int on) {
    if (!ctx) return pt_fail(nullptr, PT_E_INVALID, "ctx is NULL");
    pt_prof_collect(ctx);
    ctx->profiling = on != 0;
    return PT_OK;
}
int pt_ctx_profile_reset(pt_ctx* ctx) {
    if (!ctx) return pt_fail(nullptr, PT_E_INVALID, "ctx is NULL");
    pt_prof_collect(ctx);
    for (auto& kv : ctx->prof) { kv.second.total_ms = 0; kv.second.launches = 0; }
    ctx->launches = 0;
    return PT_OK;
}
long long pt_ctx_profile_dump(pt_ctx* ctx, char* buf, long long cap) {
    if (!ctx) return -1;
    pt_prof_collect(ctx);
    std::string s;
    char line[256];
    for (auto& kv : ctx->prof) {
        if (kv.second.launches == 0) continue;
        snprintf(line, sizeof(line), "%s,%lld,%.6f\n", kv.first.c_str(), kv.second.launches, kv.second.total_ms);
        s += line;
    }
    long long need = (long long)s.size() + 1;
    if (buf && cap >= need) memcpy(buf, s.c_str(), (size_t)need);
    return need;
}
long long pt_ctx_launch_count(pt_ctx* ctx) { return ctx ? ctx->launches : -1; }

}  // extern "C"
