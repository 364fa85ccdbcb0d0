// comm.h — NCCL communicator of the engine (row a9; see comm.cpp).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>   // types only; the library is dlopen()ed

#include <string>

namespace galois {

bool nccl_load(std::string *why);
bool nccl_unique_id(void *out128, std::string *why);

struct Comm {
    int rank = 0;
    int world = 1;
    ncclComm_t comm = nullptr;

    bool init(int rank, int world, const unsigned char *id128, std::string *why);
    bool allreduce_min_u64(const unsigned long long *send, unsigned long long *recv, cudaStream_t st,
                           std::string *why);
    bool broadcast_bytes(void *buf, size_t bytes, int root, cudaStream_t st, std::string *why);
    void destroy(bool abort);
};

}  // namespace galois
