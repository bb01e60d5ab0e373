// Multi-GPU exchange: one process per GPU, NCCL loaded at run
// time.  The fast summation is linear in the source weights, so with the sources
// sharded over ranks the oversampled Fourier coefficients of every kernel sum are the
// sum of the ranks' partial coefficients (factorisation (4.6), is linear in
// alpha~): one all-reduce per kernel sum (between the D_k multiplication and the inverse
// FFT), after which each rank interpolates at its own targets.  Setup needs a global
// bounding box (min/max all-reduce) and the objective scalars a sum all-reduce.
//
// A second communicator kind, the LOOPBACK group, stands in for P ranks inside one
// process on one GPU (tests of the multi-rank path with a single device): each of P host
// threads calls the library with its own rank handle and stream; an all-reduce publishes
// every rank's buffer, and each rank reduces all P buffers in rank order (0..P-1) with
// one kernel into a scratch buffer, then copies the result back.  The ordering between
// ranks is CUDA events (stream waits) plus two host barriers per all-reduce; no kernel
// ever waits on another rank's kernel, so nothing depends on concurrent residency.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>

#include "common.cuh"

namespace uotk {

namespace {

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (!api.lib) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.lib, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.lib, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.lib, "ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))dlsym(api.lib, "ncclAllReduce");
        api.ReduceScatter = (decltype(api.ReduceScatter))dlsym(api.lib, "ncclReduceScatter");
        api.AllGather = (decltype(api.AllGather))dlsym(api.lib, "ncclAllGather");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.lib, "ncclGetErrorString");
        api.GetVersion = (decltype(api.GetVersion))dlsym(api.lib, "ncclGetVersion");
    });
    if (!api.lib || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.ReduceScatter || !api.AllGather)
        fail(UOTK_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
    return api;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    std::string msg = std::string(what) + " failed: ";
    msg += nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error";
    fail(UOTK_ENCCL, msg);
}

constexpr int kMaxLoopRanks = 16;
constexpr double kLoopTimeoutS = 120.0;  // a rank that never arrives (it failed): error, not a hang

// element types and reduction ops of the all-reduces (NCCL's enums are not used for the
// loopback path so that it does not depend on libnccl)
enum { kF64 = 0, kI32 = 1 };
enum { kSum = 0, kMax = 1, kMin = 2 };

struct LoopGroup {
    int P = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool aborted = false;
    std::string abort_msg;
    // published by each rank for the all-reduce in flight
    void* buf[kMaxLoopRanks] = {};
    size_t count[kMaxLoopRanks] = {};
    int op[kMaxLoopRanks] = {};
    int type[kMaxLoopRanks] = {};
    cudaEvent_t ready[kMaxLoopRanks] = {};  // rank's buffer complete on its stream
    cudaEvent_t done[kMaxLoopRanks] = {};   // rank finished reading every buffer

    // all P ranks arrive (or an error / timeout aborts the group for everyone)
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) fail(UOTK_ENCCL, "loopback communicator aborted: " + abort_msg);
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(kLoopTimeoutS);
        while (gen == g && !aborted) {
            if (cv.wait_until(lk, deadline) == std::cv_status::timeout && gen == g) {
                aborted = true;
                abort_msg = "a rank did not reach the collective within the timeout";
                cv.notify_all();
            }
        }
        if (gen == g) fail(UOTK_ENCCL, "loopback communicator aborted: " + abort_msg);
    }
    void abort(const std::string& why) {
        std::lock_guard<std::mutex> lk(mu);
        if (!aborted) {
            aborted = true;
            abort_msg = why;
        }
        cv.notify_all();
    }
};

struct LoopPtrs {
    const void* p[kMaxLoopRanks];
};

// out[i] = op over ranks k = 0..P-1 (fixed order) of in_k[i]
template <class T>
__global__ void loop_reduce_k(LoopPtrs in, int P, size_t n, int op, T* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T acc = static_cast<const T*>(in.p[0])[i];
        for (int k = 1; k < P; ++k) {
            const T v = static_cast<const T*>(in.p[k])[i];
            acc = op == kSum ? acc + v : (op == kMax ? (v > acc ? v : acc) : (v < acc ? v : acc));
        }
        out[i] = acc;
    }
}

// all-gather: out[k * n + i] = in_k[i]
__global__ void loop_gather_k(LoopPtrs in, int P, size_t n, double* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n * P; i += (size_t)gridDim.x * blockDim.x)
        out[i] = static_cast<const double*>(in.p[i / n])[i % n];
}

}  // namespace

struct Comm {
    bool loopback = false;
    ncclComm_t comm = nullptr;
    int nranks = 1;
    int rank = 0;
    std::shared_ptr<LoopGroup> group;
};

void comm_unique_id(void* id128) {
    ncclUniqueId id;
    check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(id128, &id, sizeof id);
}

void* comm_create(const void* id128, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(UOTK_EINVAL, "bad nranks / rank");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    Comm* c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        check_nccl(r, "ncclCommInitRank");
    }
    if (getenv("UOTK_COMM_VERBOSE")) {
        int v = 0;
        if (nccl().GetVersion) nccl().GetVersion(&v);
        int dev = -1;
        cudaGetDevice(&dev);
        fprintf(stderr, "[uotk] NCCL communicator: rank %d of %d on device %d (NCCL %d)\n", rank, nranks, dev, v);
    }
    return c;
}

void comm_create_loopback(int nranks, void** out) {
    if (nranks < 1 || nranks > kMaxLoopRanks) fail(UOTK_EINVAL, "loopback communicator: 1 <= nranks <= 16");
    auto g = std::make_shared<LoopGroup>();
    g->P = nranks;
    for (int k = 0; k < nranks; ++k) {
        UOTK_CUDA(cudaEventCreateWithFlags(&g->ready[k], cudaEventDisableTiming));
        UOTK_CUDA(cudaEventCreateWithFlags(&g->done[k], cudaEventDisableTiming));
    }
    for (int k = 0; k < nranks; ++k) {
        Comm* c = new Comm();
        c->loopback = true;
        c->nranks = nranks;
        c->rank = k;
        c->group = g;
        out[k] = c;
    }
}

void comm_destroy(void* comm) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) return;
    if (!c->loopback && c->comm && nccl().CommDestroy) nccl().CommDestroy(c->comm);
    if (c->loopback && c->group.use_count() == 1) {
        for (int k = 0; k < c->group->P; ++k) {
            cudaEventDestroy(c->group->ready[k]);
            cudaEventDestroy(c->group->done[k]);
        }
    }
    delete c;
}

namespace {

// kind 0: all-reduce of `count` elements in place (buf); 1: reduce-scatter (fp64 sum): rank r
// receives the sum of the ranks' buf[r count .. (r + 1) count) in out; 2: all-gather (fp64):
// out[k count ..] = rank k's buf[0 .. count)
void loop_collective(Comm* c, int kind, void* buf, void* out, size_t count, int type, int op, cudaStream_t s) {
    LoopGroup& g = *c->group;
    const int r = c->rank;
    try {
        UOTK_CUDA(cudaEventRecord(g.ready[r], s));
        g.buf[r] = buf;
        g.count[r] = count;
        g.op[r] = op + 16 * kind;
        g.type[r] = type;
        g.barrier();  // (1) every rank's buffer and event are published
        for (int k = 0; k < g.P; ++k)
            if (g.count[k] != count || g.op[k] != op + 16 * kind || g.type[k] != type)
                fail(UOTK_ENCCL, "loopback collective: ranks disagree on kind / count / op / type (rank " +
                                     std::to_string(k) + ": " + std::to_string(g.count[k]) + " vs " +
                                     std::to_string(count) + ")");
        LoopPtrs ptrs{};
        for (int k = 0; k < g.P; ++k) {
            ptrs.p[k] = g.buf[k];
            if (kind == 1) ptrs.p[k] = static_cast<const double*>(g.buf[k]) + (size_t)r * count;
            if (k != r) UOTK_CUDA(cudaStreamWaitEvent(s, g.ready[k], 0));
        }
        const size_t esz = type == kF64 ? sizeof(double) : sizeof(int32_t);
        DevBuf<double> tmp;
        const int blocks = (int)std::min<size_t>(1184, (count * (kind == 2 ? g.P : 1) + 255) / 256);
        if (kind == 0) {
            tmp.alloc((count * esz + 7) / 8, s);
            if (count) {
                if (type == kF64) loop_reduce_k<double><<<blocks, 256, 0, s>>>(ptrs, g.P, count, op, tmp.p);
                else loop_reduce_k<int32_t><<<blocks, 256, 0, s>>>(ptrs, g.P, count, op, reinterpret_cast<int32_t*>(tmp.p));
                UOTK_LAUNCHED();
            }
        } else if (kind == 1) {  // into `out` (not a published buffer): no copy-back needed
            if (count) {
                loop_reduce_k<double><<<blocks, 256, 0, s>>>(ptrs, g.P, count, kSum, static_cast<double*>(out));
                UOTK_LAUNCHED();
            }
        } else {
            if (count) {
                loop_gather_k<<<blocks, 256, 0, s>>>(ptrs, g.P, count, static_cast<double*>(out));
                UOTK_LAUNCHED();
            }
        }
        UOTK_CUDA(cudaEventRecord(g.done[r], s));
        g.barrier();  // (2) every rank's reads are enqueued: no buffer is overwritten before all read it
        for (int k = 0; k < g.P; ++k)
            if (k != r) UOTK_CUDA(cudaStreamWaitEvent(s, g.done[k], 0));
        if (kind == 0 && count) UOTK_CUDA(cudaMemcpyAsync(buf, tmp.p, count * esz, cudaMemcpyDeviceToDevice, s));
    } catch (const Error& e) {
        g.abort(e.msg);
        throw;
    }
}

void loop_allreduce(Comm* c, void* buf, size_t count, int type, int op, cudaStream_t s) {
    loop_collective(c, 0, buf, nullptr, count, type, op, s);
}

}  // namespace

void comm_allreduce(double* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) return;  // a 1-rank communicator still goes through NCCL (tested on 1 GPU)
    if (c->loopback) return loop_allreduce(c, buf, count, kF64, op_max_min_sum, s);
    if (count == 0) return;
    ncclRedOp_t op = op_max_min_sum == 1 ? ncclMax : (op_max_min_sum == 2 ? ncclMin : ncclSum);
    check_nccl(nccl().AllReduce(buf, buf, count, ncclDouble, op, c->comm, s), "ncclAllReduce");
}

void comm_allreduce_i32(int32_t* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) return;
    if (c->loopback) return loop_allreduce(c, buf, count, kI32, op_max_min_sum, s);
    if (count == 0) return;
    ncclRedOp_t op = op_max_min_sum == 1 ? ncclMax : (op_max_min_sum == 2 ? ncclMin : ncclSum);
    check_nccl(nccl().AllReduce(buf, buf, count, ncclInt32, op, c->comm, s), "ncclAllReduce");
}

// rank r receives out[0 .. count) = sum over ranks of their in[r count .. (r + 1) count)
void comm_reduce_scatter(const double* in, double* out, size_t count, void* comm, cudaStream_t s) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) fail(UOTK_EINVAL, "internal: reduce-scatter without a communicator");
    if (c->loopback) return loop_collective(c, 1, const_cast<double*>(in), out, count, kF64, kSum, s);
    if (count == 0) return;
    check_nccl(nccl().ReduceScatter(in, out, count, ncclDouble, ncclSum, c->comm, s), "ncclReduceScatter");
}

// out[k count .. (k + 1) count) = rank k's in[0 .. count)
void comm_all_gather(const double* in, double* out, size_t count, void* comm, cudaStream_t s) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) fail(UOTK_EINVAL, "internal: all-gather without a communicator");
    if (c->loopback) return loop_collective(c, 2, const_cast<double*>(in), out, count, kF64, kSum, s);
    if (count == 0) return;
    check_nccl(nccl().AllGather(in, out, count, ncclDouble, c->comm, s), "ncclAllGather");
}

int comm_rank(void* comm) { return comm ? static_cast<Comm*>(comm)->rank : 0; }

void comm_allreduce_minmax(double* dmin, int nmin, double* dmax, int nmax, void* comm, cudaStream_t s) {
    if (dmin) comm_allreduce(dmin, nmin, 2, comm, s);
    if (dmax) comm_allreduce(dmax, nmax, 1, comm, s);
}

void comm_allreduce_spectrum(double2* buf, size_t count, void* comm, cudaStream_t s) {
    comm_allreduce(reinterpret_cast<double*>(buf), 2 * count, 0, comm, s);
}

int comm_nranks(void* comm) { return comm ? static_cast<Comm*>(comm)->nranks : 1; }

// The CUDA-graph capture of the iteration loop may contain the exchange step only when it
// is an NCCL call (capturable); the loopback group's host barriers are not.
bool comm_capturable(void* comm) { return !comm || !static_cast<Comm*>(comm)->loopback; }

// Library-internal per-thread resources (cuFFT plans, the cuBLAS handle) are keyed by a
// slot: the rank of a loopback communicator (its ranks run concurrently on one device
// from several host threads), else 0.
int comm_slot(void* comm) {
    Comm* c = static_cast<Comm*>(comm);
    return (c && c->loopback) ? c->rank : 0;
}

void comm_abort(void* comm, const std::string& why) {
    Comm* c = static_cast<Comm*>(comm);
    if (c && c->loopback) c->group->abort(why);
}

}  // namespace uotk
