// Library context: errors, stream-ordered buffers, host/device staging, cuFFT plan cache.
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <map>
#include <set>
#include <mutex>
#include <tuple>


#include "common.cuh"

namespace uotk {

thread_local std::string g_last_error = "no error";
thread_local int64_t g_launches = 0;
thread_local int g_slot = 0;
int comm_slot(void* comm);  // comm.cu
SlotScope::SlotScope(void* comm) : prev(g_slot) { g_slot = comm_slot(comm); }

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    fail(e == cudaErrorMemoryAllocation ? UOTK_ENOMEM : UOTK_ECUDA, buf);
}

void check_cufft(cufftResult r, const char* what, const char* file, int line) {
    if (r == CUFFT_SUCCESS) return;
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed: cufftResult %d (%s:%d)", what, (int)r, file, line);
    fail(r == CUFFT_ALLOC_FAILED ? UOTK_ENOMEM : UOTK_ECUFFT, buf);
}

void note_launch(const char* file, int line) {
    ++g_launches;
    check_cuda(cudaGetLastError(), "kernel launch", file, line);
}

void add_launches(int k) { g_launches += k; }

void set_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({func, dev})) return;
    UOTK_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({func, dev});
}

void trace_mark(const char* what) {
    // UOTK_TRACE=1: host time between marks; =2: the device is synchronised first, so a
    // mark's time includes the GPU work of its phase
    static const int level = [] {
        const char* e = getenv("UOTK_TRACE");
        return (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
    }();
    if (!level) return;
    if (level == 2) cudaDeviceSynchronize();
    unsigned long long reserved = 0;
    if (level == 2) {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaGetLastError();
    }
    static thread_local auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[uotk] %-28s %9.1f us  pool %.2f GB\n", what,
            std::chrono::duration<double, std::micro>(now - last).count(), reserved / 1e9);
    last = now;
}

// ------------------------------------------------------------------ block cache
// Device buffers of a call are recycled through a small library-level cache instead of
// being returned to the stream-ordered pool: cudaMallocAsync occasionally blocks the
// host for tens of milliseconds even when the pool does not grow (measured, DESIGN.md
// §10), and a solve makes ~40 allocations.  A freed block records an event on its stream;
// it is reused by the same stream at once, by another stream once the event completed.
// Inside CUDA-graph capture the stream-ordered allocator is used (graph memory nodes).
namespace {
struct CachedBlock {
    void* p;
    size_t bytes;
    int dev;
    cudaStream_t s;
    cudaEvent_t ev;
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;
size_t g_cache_bytes = 0;
constexpr size_t kCacheMaxBytes = size_t(48) << 30;

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st != cudaStreamCaptureStatusNone;
}

size_t round_bytes(size_t b) { return (b + 4095) & ~size_t(4095); }

// ---- guard mode (UOTK_GUARD=1; the memcheck substitute of DESIGN.md §12): every device
// buffer gets kGuard bytes of a fixed pattern before and after it; when the buffer is
// freed the stream is synchronised and both bands are checked.  A kernel writing out of
// bounds into any library buffer is reported (stderr + the next API call fails).
constexpr size_t kGuard = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_mode() {
    static const bool on = [] {
        const char* e = getenv("UOTK_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}
std::atomic<int64_t> g_guard_violations{0};

void* guard_alloc(size_t bytes, cudaStream_t s) {
    char* base = nullptr;
    UOTK_CUDA(cudaMallocAsync((void**)&base, bytes + 2 * kGuard, s));
    UOTK_CUDA(cudaMemsetAsync(base, kGuardByte, kGuard, s));
    UOTK_CUDA(cudaMemsetAsync(base + kGuard + bytes, kGuardByte, kGuard, s));
    return base + kGuard;
}

void guard_free(void* p, size_t bytes, cudaStream_t s) {
    char* base = static_cast<char*>(p) - kGuard;
    std::vector<unsigned char> h(2 * kGuard);
    if (cudaMemcpyAsync(h.data(), base, kGuard, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaMemcpyAsync(h.data() + kGuard, base + kGuard + bytes, kGuard, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaStreamSynchronize(s) == cudaSuccess) {
        size_t bad = 0;
        for (unsigned char c : h) bad += c != kGuardByte;
        if (bad) {
            fprintf(stderr, "[uotk] GUARD VIOLATION: %zu bytes overwritten around a %zu-byte buffer\n", bad, bytes);
            ++g_guard_violations;
        }
    }
    cudaGetLastError();
    cudaFreeAsync(base, s);
}

// Give a cached block back to the pool.  The stream that freed it may no longer exist
// (a caller's stream), so wait for its event on the host and free on the legacy stream.
void release_block(const CachedBlock& b) {
    cudaEventSynchronize(b.ev);
    cudaFreeAsync(b.p, 0);
    cudaEventDestroy(b.ev);
    cudaGetLastError();
}

void* cache_alloc(size_t bytes, cudaStream_t s, bool* from_pool) {
    bytes = round_bytes(bytes);
    *from_pool = capturing(s);
    if (!*from_pool && guard_mode()) return guard_alloc(bytes, s);
    if (*from_pool) {
        void* p = nullptr;
        UOTK_CUDA(cudaMallocAsync(&p, bytes, s));
        return p;
    }
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        int best = -1;
        for (int i = 0; i < (int)g_cache.size(); ++i) {
            const CachedBlock& b = g_cache[i];
            if (b.dev != dev || b.bytes < bytes || b.bytes > 2 * bytes + (size_t(4) << 20)) continue;
            if (best >= 0 && g_cache[best].bytes <= b.bytes) continue;
            if (b.s != s && cudaEventQuery(b.ev) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            best = i;
        }
        if (best >= 0) {
            CachedBlock b = g_cache[best];
            g_cache.erase(g_cache.begin() + best);
            g_cache_bytes -= b.bytes;
            cudaEventDestroy(b.ev);
            return b.p;
        }
    }
    void* p = nullptr;
    UOTK_CUDA(cudaMallocAsync(&p, bytes, s));
    return p;
}

void cache_free(void* p, size_t bytes, cudaStream_t s, bool from_pool) {
    if (from_pool || capturing(s)) {
        cudaFreeAsync(p, s);
        return;
    }
    bytes = round_bytes(bytes);
    if (guard_mode()) return guard_free(p, bytes, s);
    int dev = 0;
    cudaEvent_t ev = nullptr;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, s) != cudaSuccess) {
        cudaGetLastError();
        if (ev) cudaEventDestroy(ev);
        cudaFreeAsync(p, s);
        return;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.push_back({p, bytes, dev, s, ev});
    g_cache_bytes += bytes;
    while (g_cache_bytes > kCacheMaxBytes && !g_cache.empty()) {  // evict the oldest
        CachedBlock b = g_cache.front();
        g_cache.erase(g_cache.begin());
        g_cache_bytes -= b.bytes;
        release_block(b);
    }
}
}  // namespace

int64_t guard_violations() { return g_guard_violations.load(); }

// bytes held by the block cache on the current device, and releasing them to the pool
size_t block_cache_bytes() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t b = 0;
    for (const CachedBlock& c : g_cache)
        if (c.dev == dev) b += c.bytes;
    return b;
}

void block_cache_release() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t i = 0; i < g_cache.size();) {
        CachedBlock& b = g_cache[i];
        if (b.dev != dev) {
            ++i;
            continue;
        }
        g_cache_bytes -= b.bytes;
        release_block(b);
        g_cache.erase(g_cache.begin() + i);
    }
}

template <typename T>
void DevBuf<T>::alloc(size_t count, cudaStream_t stream) {
    if (p) cache_free(p, n * sizeof(T), s, pooled);
    p = nullptr;
    n = count;
    s = stream;
    if (count) p = static_cast<T*>(cache_alloc(count * sizeof(T), stream, &pooled));
}

template <typename T>
DevBuf<T>::~DevBuf() {
    if (p) cache_free(p, n * sizeof(T), s, pooled);
}

template <typename T>
DevBuf<T>& DevBuf<T>::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (p) cache_free(p, n * sizeof(T), s, pooled);
        p = o.p; n = o.n; s = o.s; pooled = o.pooled;
        o.p = nullptr; o.n = 0;
    }
    return *this;
}

template struct DevBuf<double>;
template struct DevBuf<double2>;
template struct DevBuf<int32_t>;
template struct DevBuf<uint32_t>;
template struct DevBuf<int64_t>;
template struct DevBuf<unsigned long long>;
template struct DevBuf<uint8_t>;
template struct DevBuf<int4>;

bool is_device_pointer(const void* ptr) {
    if (!ptr) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear: older drivers flag unregistered host memory
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void InArr::bind(const double* user, size_t count, cudaStream_t s) {
    if (count == 0 || is_device_pointer(user)) {
        d = user;
        return;
    }
    staged.alloc(count, s);
    UOTK_CUDA(cudaMemcpyAsync(staged.p, user, count * sizeof(double), cudaMemcpyHostToDevice, s));
    d = staged.p;
    host = true;
}

void OutArr::bind(double* user_ptr, size_t cnt, cudaStream_t stream) {
    user = user_ptr;
    count = cnt;
    s = stream;
    host = cnt > 0 && !is_device_pointer(user_ptr);
    if (host) {
        staged.alloc(cnt, stream);
        d = staged.p;
    } else {
        d = user_ptr;
    }
}

void OutArr::flush() {
    if (host && count)
        UOTK_CUDA(cudaMemcpyAsync(user, staged.p, count * sizeof(double), cudaMemcpyDeviceToHost, s));
}

// ------------------------------------------------------------------ context
struct Context {
    std::mutex mu;
    // (device, slot, d, n) -> (r2c, c2r)
    std::map<std::tuple<int, int, int, int>, std::pair<cufftHandle, cufftHandle>> fft;
    bool pool_configured[64] = {};
    // (device, slot, n, w, H) -> pruned-transform plans (pass z R2C, pass y C2C, pass x C2C)
    std::map<std::tuple<int, int, int, int, int>, std::array<cufftHandle, 4>> pruned;
    std::map<int, cudaStream_t> streams;
};

Context& ctx() {
    static Context* c = new Context();  // intentionally leaked: lives until process exit
    return *c;
}

static void configure_pool(int dev) {
    Context& c = ctx();
    if (dev < 0 || dev >= 64 || c.pool_configured[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep freed blocks cached between calls
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    c.pool_configured[dev] = true;
}

void release_fft_plans() {
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto& e : c.fft) {
        cufftDestroy(e.second.first);
        cufftDestroy(e.second.second);
    }
    c.fft.clear();
    for (auto& e : c.pruned)
        for (cufftHandle h : e.second) cufftDestroy(h);
    c.pruned.clear();
}

void get_fft_plans(int d, int n, cufftHandle* r2c, cufftHandle* c2r) {
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    configure_pool(dev);
    auto key = std::make_tuple(dev, g_slot, d, n);
    auto it = c.fft.find(key);
    if (it != c.fft.end()) {
        *r2c = it->second.first;
        *c2r = it->second.second;
        return;
    }
    cufftHandle a, b;
    if (d == 1) {
        UOTK_CUFFT(cufftPlan1d(&a, n, CUFFT_D2Z, 1));
        UOTK_CUFFT(cufftPlan1d(&b, n, CUFFT_Z2D, 1));
    } else if (d == 2) {
        UOTK_CUFFT(cufftPlan2d(&a, n, n, CUFFT_D2Z));
        UOTK_CUFFT(cufftPlan2d(&b, n, n, CUFFT_Z2D));
    } else {
        UOTK_CUFFT(cufftPlan3d(&a, n, n, n, CUFFT_D2Z));
        UOTK_CUFFT(cufftPlan3d(&b, n, n, n, CUFFT_Z2D));
    }
    c.fft[key] = {a, b};
    trace_mark("full cuFFT plans created");
    *r2c = a;
    *c2r = b;
}

void get_pruned_plans(int n, int w, int H, cufftHandle* pz, cufftHandle* py, cufftHandle* px, cufftHandle* pzi) {
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    auto key = std::make_tuple(dev, g_slot, n, w, H);
    auto it = c.pruned.find(key);
    if (it == c.pruned.end()) {
        std::array<cufftHandle, 4> h{};
        int len = n;
        const int half = n / 2 + 1;
        // z: R2C of the w * n rows g[o + x'][y][.], contiguous
        UOTK_CUFFT(cufftPlanMany(&h[0], 1, &len, nullptr, 1, n, nullptr, 1, half, CUFFT_D2Z, w * n));
        // y: C2C of w * (H + 1) rows of length n
        UOTK_CUFFT(cufftPlanMany(&h[1], 1, &len, nullptr, 1, n, nullptr, 1, n, CUFFT_Z2Z, w * (H + 1)));
        // x: C2C of (2H + 1) * (H + 1) rows of length n
        UOTK_CUFFT(cufftPlanMany(&h[2], 1, &len, nullptr, 1, n, nullptr, 1, n, CUFFT_Z2Z, (2 * H + 1) * (H + 1)));
        // z inverse (kernel-sum chain): C2R of the w * n rows back into the box slab
        UOTK_CUFFT(cufftPlanMany(&h[3], 1, &len, nullptr, 1, half, nullptr, 1, n, CUFFT_Z2D, w * n));
        it = c.pruned.emplace(key, h).first;
        trace_mark("pruned cuFFT plans created");
    }
    *pz = it->second[0];
    *py = it->second[1];
    *px = it->second[2];
    *pzi = it->second[3];
}

cudaStream_t private_stream() {
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.streams.find(dev);
    if (it == c.streams.end()) {
        cudaStream_t st;
        UOTK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        it = c.streams.emplace(dev, st).first;
    }
    return it->second;
}

void ensure_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return; }
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    configure_pool(dev);
}

}  // namespace uotk
