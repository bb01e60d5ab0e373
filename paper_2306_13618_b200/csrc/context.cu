// Library context: errors, stream-ordered buffers, host/device staging, cuFFT plan cache.
#include <chrono>
#include <cstdlib>
#include <map>
#include <set>
#include <mutex>
#include <tuple>

#include <cublas_v2.h>

#include "common.cuh"

namespace uotk {

thread_local std::string g_last_error = "no error";
thread_local int64_t g_launches = 0;

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
    static thread_local auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[uotk] %-28s %9.1f us\n", what,
            std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
}

template <typename T>
void DevBuf<T>::alloc(size_t count, cudaStream_t stream) {
    if (p) UOTK_CUDA(cudaFreeAsync(p, s));
    p = nullptr;
    n = count;
    s = stream;
    if (count) UOTK_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
}

template <typename T>
DevBuf<T>::~DevBuf() {
    if (p) cudaFreeAsync(p, s);
}

template <typename T>
DevBuf<T>& DevBuf<T>::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (p) cudaFreeAsync(p, s);
        p = o.p; n = o.n; s = o.s;
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
    // (device, d, n) -> (r2c, c2r)
    std::map<std::tuple<int, int, int>, std::pair<cufftHandle, cufftHandle>> fft;
    bool pool_configured[64] = {};
    std::map<int, cublasHandle_t> blas;
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

void get_fft_plans(int d, int n, cufftHandle* r2c, cufftHandle* c2r) {
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    configure_pool(dev);
    auto key = std::make_tuple(dev, d, n);
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
    *r2c = a;
    *c2r = b;
}

void get_cublas(void** handle) {
    int dev = 0;
    UOTK_CUDA(cudaGetDevice(&dev));
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.blas.find(dev);
    if (it == c.blas.end()) {
        cublasHandle_t h;
        if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) fail(UOTK_ECUDA, "cublasCreate failed");
        it = c.blas.emplace(dev, h).first;
    }
    *handle = it->second;
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
