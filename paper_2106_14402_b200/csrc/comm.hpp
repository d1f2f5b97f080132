// comm.hpp -- the NCCL communicator handle behind slapcu_comm (shared by the
// SUMMA / 3D drivers in dist.cu and the redistributions in redist.cu).
#pragma once
#include <nccl.h>

#include <map>
#include <string>

#include "ctx.hpp"

#define SLAPCU_NCCL(call)                                                                               \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess)                                                                          \
            throw ::slapcu::Fail{SLAPCU_ERR_COMM, std::string(#call) + ": " + ncclGetErrorString(r_)};  \
    } while (0)

struct slapcu_comm_s {
    slapcu_ctx ctx = nullptr;
    int rank = 0, nranks = 1;
    ncclComm_t world = nullptr;
    std::map<std::string, ncclComm_t> splits;
    cudaStream_t comm_stream = nullptr;
    int64_t calls[4] = {0, 0, 0, 0};
    int64_t bytes[4] = {0, 0, 0, 0};
};

namespace slapcu {
enum { kBcast = 0, kAlltoallv = 1, kReduce = 2, kAllgatherv = 3 };
}
