// Multi-GPU exchange: one process per GPU, NCCL loaded at run
// time.  The fast summation is linear in the source weights, so with the sources
// sharded over ranks the oversampled Fourier coefficients of every kernel sum are the
// sum of the ranks' partial coefficients: one all-reduce per kernel sum (between the
// D_k multiplication and the inverse FFT), after which each rank interpolates at its
// own targets.  Setup needs a global bounding box (min/max all-reduce) and the
// objective scalars a sum all-reduce.
#include <dlfcn.h>
#include <nccl.h>

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
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
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
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.lib, "ncclGetErrorString");
    });
    if (!api.lib || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce)
        fail(UOTK_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
    return api;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    std::string msg = std::string(what) + " failed: ";
    msg += nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error";
    fail(UOTK_ENCCL, msg);
}

}  // namespace

struct Comm {
    ncclComm_t comm = nullptr;
    int nranks = 1;
    int rank = 0;
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
    return c;
}

void comm_destroy(void* comm) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c) return;
    if (c->comm && nccl().CommDestroy) nccl().CommDestroy(c->comm);
    delete c;
}

void comm_allreduce(double* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s) {
    Comm* c = static_cast<Comm*>(comm);
    if (!c || count == 0) return;  // a 1-rank communicator still goes through NCCL (tested on 1 GPU)
    ncclRedOp_t op = op_max_min_sum == 1 ? ncclMax : (op_max_min_sum == 2 ? ncclMin : ncclSum);
    check_nccl(nccl().AllReduce(buf, buf, count, ncclDouble, op, c->comm, s), "ncclAllReduce");
}

void comm_allreduce_minmax(double* dmin, int nmin, double* dmax, int nmax, void* comm, cudaStream_t s) {
    if (dmin) comm_allreduce(dmin, nmin, 2, comm, s);
    if (dmax) comm_allreduce(dmax, nmax, 1, comm, s);
}

void comm_allreduce_spectrum(double2* buf, size_t count, void* comm, cudaStream_t s) {
    comm_allreduce(reinterpret_cast<double*>(buf), 2 * count, 0, comm, s);
}

int comm_nranks(void* comm) { return comm ? static_cast<Comm*>(comm)->nranks : 1; }

}  // namespace uotk
