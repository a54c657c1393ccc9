// comm.cu -- runtime binding of NCCL (see comm.hpp).
#include <dlfcn.h>

#include <mutex>

#include "comm.hpp"
#include "common.cuh"

namespace picgpu {

namespace {

Nccl g_nccl;
bool g_loaded = false;
std::mutex g_mu;

template <class F>
void bind(void* h, F& f, const char* name) {
    f = reinterpret_cast<F>(dlsym(h, name));
    if (!f) throw Status{PICGPU_ENCCL, "libnccl.so.2 lacks a required symbol"};
}

}  // namespace

const Nccl& nccl() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_loaded) return g_nccl;
    // the process's own NCCL first (a communicator must be driven by the library that made it)
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Status{PICGPU_ENCCL, "cannot load libnccl.so.2"};
    bind(h, g_nccl.GetUniqueId, "ncclGetUniqueId");
    bind(h, g_nccl.CommInitRank, "ncclCommInitRank");
    bind(h, g_nccl.CommDestroy, "ncclCommDestroy");
    bind(h, g_nccl.CommCount, "ncclCommCount");
    bind(h, g_nccl.CommUserRank, "ncclCommUserRank");
    bind(h, g_nccl.Send, "ncclSend");
    bind(h, g_nccl.Recv, "ncclRecv");
    bind(h, g_nccl.GroupStart, "ncclGroupStart");
    bind(h, g_nccl.GroupEnd, "ncclGroupEnd");
    bind(h, g_nccl.GetErrorString, "ncclGetErrorString");
    g_loaded = true;
    return g_nccl;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Status{PICGPU_ENCCL, what};
}

}  // namespace picgpu
