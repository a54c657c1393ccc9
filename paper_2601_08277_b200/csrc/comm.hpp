// comm.hpp -- NCCL behind the C ABI (x-slab exchanges over NVLink/NVSwitch).
//
// The library does not link NCCL: it binds the libnccl.so.2 ALREADY LOADED in
// the process (dlopen RTLD_NOLOAD -- e.g. the one torch.distributed uses, so a
// communicator created there can be handed over as a raw ncclComm_t), else
// loads libnccl.so.2 itself.  Only the types come from <nccl.h>.
#pragma once

#include <nccl.h>

namespace picgpu {

struct Nccl {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

// The bound NCCL; throws Status{PICGPU_ECUDA} when no libnccl.so.2 can be loaded.
const Nccl& nccl();
// ncclResult_t -> Status (PICGPU_ENCCL) with NCCL's message.
void nccl_check(ncclResult_t r, const char* what);

}  // namespace picgpu

// The opaque communicator of the C ABI (include/picgpu.h).
struct picgpu_comm {
    ncclComm_t comm = nullptr;
    int rank = 0;
    int nranks = 1;
    int device = 0;
    bool owned = false;  // created by picgpu_comm_init (destroyed with it)
};
