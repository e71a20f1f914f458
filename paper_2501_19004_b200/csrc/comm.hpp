// Library-owned NCCL communicator for lvn_louvain_sharded.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": inside a PyTorch process
// that is the torch-bundled NCCL already mapped, in a plain C++ host the
// system one), so liblvn.so carries no link-time NCCL dependency and
// single-GPU users never touch it. Collectives are enqueued on the engine
// stream: no host synchronisation around them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "lvn.h"

namespace lvn {

struct NcclComm;  // opaque; defined in comm.cu

// the NcclComm behind an lvn_comm made by lvn_comm_nccl_create, else nullptr
NcclComm* nccl_of(const lvn_comm* c);

// stream-ordered collectives (fail(kCuda, ...) on an NCCL error)
void nccl_allreduce(NcclComm* nc, void* buf, uint64_t count, int dtype, int op, cudaStream_t s);
// rank r contributes counts[r] bytes; recv holds them concatenated in rank order
// (send may alias recv at this rank's position)
void nccl_allgatherv(NcclComm* nc, const void* send, void* recv, const uint64_t* counts, cudaStream_t s);
// all-to-all of bytes: send_counts[k] bytes for rank k back to back in send,
// recv_counts[k] bytes from rank k back to back in recv
void nccl_alltoallv(NcclComm* nc, const void* send, const uint64_t* send_counts, void* recv,
                    const uint64_t* recv_counts, cudaStream_t s);

}  // namespace lvn
