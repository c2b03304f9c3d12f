// xport.h -- the exchange primitives of the z-slab plan (points
// move to their owners, halos are accumulated / filled between z-neighbours, the
// distributed FFT transposes with an all-to-all).  Private to libnufft.so.
//
// Two transports implement them:
//   NCCL      one process (rank) per GPU over NVLink / NVSwitch (the product path);
//   loopback  P ranks on ONE GPU, each driven by its own host thread: every message
//             is a device-to-device cudaMemcpyAsync on the receiver's stream, ordered
//             after the sender's data by events and host-side rendezvous.  It runs
//             the same dist.cpp code at any P on a single device (tests, P = 8 without
//             an 8-GPU box); it is not a performance path.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace nufft {

struct Xport {
    int P = 1, r = 0;
    virtual ~Xport() = default;
    // grouped point-to-point messages (NCCL group semantics: all sends / recvs of a
    // group are posted, then the group completes on stream s)
    virtual int group_start() = 0;
    virtual int send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual int recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual int group_end(cudaStream_t s) = 0;
    // block q of `send` (bytes_per_rank each) -> rank q's `recv` block r
    virtual int alltoall(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t s) = 0;
    // in-place max over the ranks of one device-resident u64
    virtual int allreduce_max_u64(unsigned long long* dev_val, cudaStream_t s) = 0;
};

// NCCL communicator from a 128-byte unique id (nufft_comm_unique_id); nullptr on failure
Xport* xport_nccl(const char id[128], int nranks, int rank);
void xport_nccl_unique_id(char id[128], int* status);
// nranks loopback transports sharing one rendezvous (all on the current device)
int xport_loopback(int nranks, Xport** out);

}  // namespace nufft
