// Context, error reporting, stream-ordered allocation and the CUDA-event kernel profiler.
#include <stdarg.h>
#include <stdlib.h>
#include "pt_internal.cuh"

// FP64 peak microbenchmark: 8 independent DFMA chains per thread, enough blocks to fill the chip
__global__ void __launch_bounds__(256) pt_peak_fp64_kernel(double* out, int iters, double seed) {
    double a0 = seed, a1 = seed + 1, a2 = seed + 2, a3 = seed + 3, a4 = seed + 4, a5 = seed + 5, a6 = seed + 6, a7 = seed + 7;
    const double m = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 123.456) out[0] = r;   // never true; keeps the chains alive
}

// MUFU.EX2 peak microbenchmark: 8 independent ex2.approx chains per thread
__global__ void __launch_bounds__(256) pt_peak_ex2_kernel(float* out, int iters, float seed) {
    float a0 = seed, a1 = seed - 0.1f, a2 = seed - 0.2f, a3 = seed - 0.3f, a4 = seed - 0.4f, a5 = seed - 0.5f, a6 = seed - 0.6f, a7 = seed - 0.7f;
    for (int i = 0; i < iters; ++i) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a4)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a5));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a6)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a7));
    }
    float r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 123.456f) out[0] = r;
}

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

// Allocation sizes are rounded up to 4 significant bits (<= 6.25 % slack) so that the slightly different
// buffer sizes of successive waves / steps land in the same bucket; blocks above PT_CACHE_MAX_BLOCK bypass
// the cache (they are the per-proof giants whose size follows the problem, not the step).
#define PT_CACHE_MAX_BLOCK ((size_t)4 << 30)
static size_t pt_round_block(size_t bytes) {
    if (bytes < 512) return 512;
    int top = 63 - __builtin_clzll((unsigned long long)bytes);
    const size_t gran = (size_t)1 << (top > 4 ? top - 4 : 0);
    return (bytes + gran - 1) & ~(gran - 1);
}
static void pt_cache_release(pt_ctx* ctx) {
    for (auto& kv : ctx->free_blocks) cudaFreeAsync(kv.second, ctx->stream);
    ctx->free_blocks.clear();
    ctx->cached_bytes = 0;
}
int pt_dev_alloc(pt_ctx* ctx, void** p, size_t bytes) {
    const size_t want = pt_round_block(bytes);
    auto it = ctx->free_blocks.lower_bound(want);
    if (it != ctx->free_blocks.end() && it->first <= want + want / 4) {
        *p = it->second;
        ctx->cached_bytes -= it->first;
        ctx->live_blocks[*p] = it->first;
        ctx->free_blocks.erase(it);
        return PT_OK;
    }
    cudaError_t e = cudaMallocAsync(p, want, ctx->stream);
    if (e == cudaErrorMemoryAllocation && !ctx->free_blocks.empty()) {
        cudaGetLastError();
        pt_cache_release(ctx);
        cudaStreamSynchronize(ctx->stream);
        e = cudaMallocAsync(p, want, ctx->stream);
    }
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return pt_fail(ctx, PT_E_NOMEM, "device allocation of %zu bytes failed", bytes);
    }
    if (e != cudaSuccess) return pt_fail(ctx, PT_E_CUDA, "cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
    ctx->live_blocks[*p] = want;
    return PT_OK;
}
void pt_dev_free(pt_ctx* ctx, void* p) {
    if (!p) return;
    if (!ctx) { cudaFreeAsync(p, nullptr); return; }
    auto it = ctx->live_blocks.find(p);
    if (it == ctx->live_blocks.end()) { cudaFreeAsync(p, ctx->stream); return; }
    const size_t size = it->second;
    ctx->live_blocks.erase(it);
    if (size > PT_CACHE_MAX_BLOCK) { cudaFreeAsync(p, ctx->stream); return; }
    ctx->free_blocks.emplace(size, p);
    ctx->cached_bytes += size;
    // the cache is a working-set optimisation, not a reservation: a loop whose batch sizes keep growing (solve() at 6 DoF)
    // leaves ever larger free blocks behind; past the cap everything cached goes back to the driver's pool
    static const size_t cap = (size_t)(getenv("PERMATRACE_B200_CACHE_GB") ? atof(getenv("PERMATRACE_B200_CACHE_GB")) : 48.0) << 30;
    if (ctx->cached_bytes > cap) {
        pt_cache_release(ctx);
        // cudaFreeAsync only hands the blocks to the stream-ordered pool; trimming the pool is what gives the memory back
        cudaStreamSynchronize(ctx->stream);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    }
}

extern "C" void* pt_host_alloc(pt_ctx* ctx, long long bytes) {
    if (!ctx || bytes < 0) return nullptr;
    const size_t want = pt_round_block((size_t)bytes);
    {
        std::lock_guard<std::mutex> g(ctx->host_lock);
        auto it = ctx->host_free_blocks.lower_bound(want);
        if (it != ctx->host_free_blocks.end() && it->first <= want + want / 4) {
            void* p = it->second;
            ctx->host_live_blocks[p] = it->first;
            ctx->host_free_blocks.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        pt_fail(ctx, PT_E_NOMEM, "pinned host allocation of %lld bytes failed", bytes);
        return nullptr;
    }
    std::lock_guard<std::mutex> g(ctx->host_lock);
    ctx->host_live_blocks[p] = want;
    return p;
}

extern "C" void pt_host_free(pt_ctx* ctx, void* p) {
    if (!ctx || !p) return;
    std::lock_guard<std::mutex> g(ctx->host_lock);
    auto it = ctx->host_live_blocks.find(p);
    if (it == ctx->host_live_blocks.end()) return;
    ctx->host_free_blocks.emplace(it->second, p);
    ctx->host_live_blocks.erase(it);
}

static void pt_host_cache_release(pt_ctx* ctx) {
    std::lock_guard<std::mutex> g(ctx->host_lock);
    for (auto& kv : ctx->host_free_blocks) cudaFreeHost(kv.second);
    ctx->host_free_blocks.clear();
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
    PT_CUDA(ctx, cudaMalloc((void**)&ctx->work, 16 * sizeof(unsigned long long)));
    PT_CUDA(ctx, cudaMemset(ctx->work, 0, 16 * sizeof(unsigned long long)));
    ctx->amb_sink = ctx->work + 6;
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
    pt_cache_release(ctx);
    cudaStreamSynchronize(ctx->stream);
    pt_host_cache_release(ctx);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->work) cudaFree(ctx->work);
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

long long pt_ctx_trim(pt_ctx* ctx) {
    if (!ctx) return -1;
    const long long released = (long long)ctx->cached_bytes;
    pt_cache_release(ctx);
    cudaStreamSynchronize(ctx->stream);
    pt_host_cache_release(ctx);
    return released;
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

int pt_ctx_work_counters(pt_ctx* ctx, long long* out, int reset) {
    if (!ctx || !out) return pt_fail(ctx, PT_E_INVALID, "pt_ctx_work_counters: NULL argument");
    unsigned long long h[16];
    PT_CUDA(ctx, cudaMemcpyAsync(h, ctx->work, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 6; ++i) out[i] = (long long)h[i];
    ctx->retry_evals = (long long)h[8];          // the proof retries count into a second bank (work + 8)
    ctx->taylor_rows = (long long)h[7];          // rows that went through the one-pass Taylor-model kernel
    if (reset) PT_CUDA(ctx, cudaMemsetAsync(ctx->work, 0, sizeof(h), ctx->stream));
    return PT_OK;
}

long long pt_ctx_retry_evaluations(pt_ctx* ctx) { return ctx ? ctx->retry_evals : -1; }
long long pt_ctx_taylor_rows(pt_ctx* ctx) { return ctx ? ctx->taylor_rows : -1; }

double pt_peak_ex2(pt_ctx* ctx) {
    if (!ctx) return -1.0;
    float* d = nullptr;
    if (cudaMalloc((void**)&d, sizeof(float)) != cudaSuccess) return -1.0;
    const int iters = 1 << 14, blocks = ctx->sm_count * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, ctx->stream);
        pt_peak_ex2_kernel<<<blocks, threads, 0, ctx->stream>>>(d, iters, -0.5f);
        cudaEventRecord(e1, ctx->stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double rate = 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
        if (rep > 0 && rate > best) best = rate;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    cudaFree(d);
    return best;   // T ex2/s
}

double pt_peak_fp64(pt_ctx* ctx) {
    if (!ctx) return -1.0;
    double* d = nullptr;
    if (cudaMalloc((void**)&d, sizeof(double)) != cudaSuccess) return -1.0;
    const int iters = 1 << 15, blocks = ctx->sm_count * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, ctx->stream);
        pt_peak_fp64_kernel<<<blocks, threads, 0, ctx->stream>>>(d, iters, 0.5);
        cudaEventRecord(e1, ctx->stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double tf = 2.0 * 8.0 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
        if (rep > 0 && tf > best) best = tf;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    cudaFree(d);
    return best;
}

}  // extern "C"
