// NCCL plumbing for the velocity-sharded collision.
//
// Velocities are independent during transport (L_h is block-diagonal over
// velocities), so each rank sweeps its own contiguous block of nv/nranks velocities.
// The only exchange is the sum of the partial moments w over ranks, once per
// collision (the paper's commutative reduction task).  libnccl.so.2 is
// loaded with dlopen: torch has already mapped its bundled copy into the process, so
// the same library instance serves torch.distributed and this communicator.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <string>

namespace pdg {

struct NcclApi {
    typedef int (*GetUniqueId_t)(void *);
    typedef int (*CommInitRank_t)(void **, int, const void *, int);  // (comm*, nranks, id (by value: 128 B), rank)
    typedef int (*AllReduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
    typedef int (*AllGather_t)(const void *, void *, size_t, int, void *, cudaStream_t);
    typedef int (*CommDestroy_t)(void *);
    typedef const char *(*GetErrorString_t)(int);
    void *handle = nullptr;
    GetUniqueId_t getUniqueId = nullptr;
    void *commInitRank = nullptr;
    AllReduce_t allReduce = nullptr;
    AllGather_t allGather = nullptr;
    CommDestroy_t commDestroy = nullptr;
    GetErrorString_t getErrorString = nullptr;

    bool load(std::string *err)
    {
        if (handle) return true;
        handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!handle) handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!handle) {
            *err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return false;
        }
        getUniqueId = (GetUniqueId_t)dlsym(handle, "ncclGetUniqueId");
        commInitRank = dlsym(handle, "ncclCommInitRank");
        allReduce = (AllReduce_t)dlsym(handle, "ncclAllReduce");
        allGather = (AllGather_t)dlsym(handle, "ncclAllGather");
        commDestroy = (CommDestroy_t)dlsym(handle, "ncclCommDestroy");
        getErrorString = (GetErrorString_t)dlsym(handle, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !allReduce || !allGather || !commDestroy) {
            *err = "libnccl.so.2 lacks a required symbol";
            return false;
        }
        return true;
    }
    std::string message(int r) const
    {
        return getErrorString ? std::string(getErrorString(r)) : ("nccl error " + std::to_string(r));
    }
};

inline NcclApi &nccl_api()
{
    static NcclApi api;
    return api;
}

struct NcclUid {
    char internal[128];
};

struct NcclComm {
    void *comm = nullptr;

    static bool unique_id(void *out, std::string *err)
    {
        NcclApi &a = nccl_api();
        if (!a.load(err)) return false;
        int r = a.getUniqueId(out);
        if (r != 0) {
            *err = "ncclGetUniqueId: " + a.message(r);
            return false;
        }
        return true;
    }

    bool init(const void *id, int nranks, int rank, std::string *err)
    {
        NcclApi &a = nccl_api();
        if (!a.load(err)) return false;
        NcclUid uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        typedef int (*Init_t)(void **, int, NcclUid, int);
        int r = ((Init_t)a.commInitRank)(&comm, nranks, uid, rank);
        if (r != 0) {
            comm = nullptr;
            *err = "ncclCommInitRank: " + a.message(r);
            return false;
        }
        return true;
    }

    // in-place fp64 sum over ranks (ncclFloat64 = 8, ncclSum = 0 in nccl.h)
    bool allreduce_sum(double *buf, size_t count, cudaStream_t stream, std::string *err)
    {
        NcclApi &a = nccl_api();
        int r = a.allReduce(buf, buf, count, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm, stream);
        if (r != 0) {
            *err = "ncclAllReduce: " + a.message(r);
            return false;
        }
        return true;
    }

    // in-place fp64 all-gather: rank r's block of `count` doubles sits at buf + r * count
    bool allgather(double *buf, size_t count, int rank, cudaStream_t stream, std::string *err)
    {
        NcclApi &a = nccl_api();
        int r = a.allGather(buf + (size_t)rank * count, buf, count, /*ncclFloat64*/ 8, comm, stream);
        if (r != 0) {
            *err = "ncclAllGather: " + a.message(r);
            return false;
        }
        return true;
    }

    void destroy()
    {
        if (comm) nccl_api().commDestroy(comm);
        comm = nullptr;
    }
};

}  // namespace pdg
