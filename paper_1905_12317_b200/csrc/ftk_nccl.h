// NCCL glue (ftk_nccl.cpp): run-time-loaded libnccl.so.2; see include/ftk.h for the public calls.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/ftk.h"

namespace ftk {
int nccl_unique_id(void* id_out /* 128 bytes */, std::string& msg);
int nccl_comm_create(const void* id /* 128 bytes */, int world, int rank, void** comm_out, std::string& msg);
int nccl_comm_destroy(void* comm);
// FTK_EINVAL if the communicator's size / rank differ from (world, rank)
int nccl_comm_check(void* comm, int world, int rank, std::string& msg);
// recv[r][i] = rank r's send[i] (16-byte ftk_best_t records), asynchronous on s
int nccl_allgather_bests(void* comm, const void* send, void* recv, int64_t n_records, cudaStream_t s,
                         std::string& msg);
}  // namespace ftk
