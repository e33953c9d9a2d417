// Collective hook used by the stage loops of the head-sharded (tensor-parallel) prefill.
#pragma once
#include "common.cuh"

namespace pkv {
struct LocalGroup;
// in-place sum over the ranks of c (no-op when c is null or has one rank)
int comm_allreduce(pkv_comm* c, void* buf, size_t count, int dtype, cudaStream_t st);
// recv = the W ranks' send buffers of `bytes` each, in rank order
int comm_allgather(pkv_comm* c, const void* send, void* recv, size_t bytes, cudaStream_t st);
int comm_rank(const pkv_comm* c);
int comm_world(const pkv_comm* c);
}  // namespace pkv
