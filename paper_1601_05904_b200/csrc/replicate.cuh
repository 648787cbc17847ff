// replicate.cuh — data replication across the devices of a single-process
// multi-device run (replicate.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace aidwb {

enum { kReplicateNone = 0, kReplicateNccl = 1, kReplicatePeer = 2 };

// One replica of the data arrays per distinct device (first-appearance
// order); freed on destruction, each on its own device.
struct Replicas {
    std::vector<int> devs;
    std::vector<double*> x, y, z;
    std::vector<cudaStream_t> streams;
    size_t m = 0;
    int kind = kReplicateNone;
    int slot_of(int dev) const;
    Replicas() = default;
    Replicas(const Replicas&) = delete;
    Replicas& operator=(const Replicas&) = delete;
    ~Replicas();
};

// Host data -> first device (one H2D), then ncclBroadcast to the others
// (ncclCommInitAll, communicators cached per device set); CUDA peer copies
// when NCCL cannot be loaded.  Synchronous.
void replicate_data(const std::vector<int>& devices, const double* hx, const double* hy,
                    const double* hz, size_t m, Replicas& out);

long long nccl_broadcast_count();  // grouped broadcasts issued so far
int last_replication_kind();       // kReplicate* of the latest replication
int nccl_version();                // 0 if NCCL is not loadable
}  // namespace aidwb
