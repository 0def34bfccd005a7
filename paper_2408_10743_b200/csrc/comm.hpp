// NCCL for the multi-GPU level exchange, loaded at run time (dlopen "libnccl.so.2": the copy
// torch already loaded when there is one, else the system's), so the library itself loads
// on hosts without NCCL. One min-allreduce of the per-weight best keys per sharded level,
// stream-ordered between the level kernel and level_close: no host round trip.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace sdb {

constexpr int kCommIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES

void comm_unique_id(unsigned char *out);
void *comm_create(const unsigned char *id, int rank, int world, int device);
void comm_destroy(void *comm);
// elementwise min of n uint64 values across the communicator, in place, on `stream`
void comm_allreduce_min_u64(void *comm, unsigned long long *buf, size_t n, cudaStream_t stream);

}  // namespace sdb
