// comm.h — the collective seam under the FSDP path (F0 / B11 of §8(a)).
//
// The runtime issues exactly three collectives per parameter group: an all-gather of the
// bf16 compute shards before a layer's forward and backward, a reduce-scatter (fp32 sum) of its gradients,
// and, in the replicated-DP debug mode, an all-reduce.  Two backends implement them:
//   * NCCL (one process per GPU over NVLink / NVSwitch) — the product path;
//   * loopback — G virtual ranks inside ONE process on one GPU (one host thread per rank, each with its own
//     dhen_ctx and streams).  Every collective is a host rendezvous of the G threads; the last arriver's
//     communication stream waits on every rank's "input ready" event, performs the copies / the fixed-order
//     (rank 0, 1, ...) sums, and records a "done" event every rank's communication stream then waits on.  No
//     kernel ever waits on another rank's kernel: ordering is stream / event dependencies only.  It exists
//     so the real event / stream / sharding logic of the FSDP path runs and is checked against world = 1 on a
//     one-GPU machine (tests/test_gpu_fsdp.py).
// Both count the bytes each rank moves with the ring-collective convention: an all-gather of `count`
// elements per rank receives (G - 1) count elements, a reduce-scatter to `count` per rank sends
// (G - 1) count, an all-reduce of n elements moves 2 (G - 1) / G n, an all-to-all of `count` per peer sends
// (G - 1) count.  The reductions take fp32 or bf16
// operands (bf16: the paper's quantized collectives, P:158 / P:277; the loopback sums in fp32 in rank order
// and rounds once, NCCL rounds per ring hop).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace dhen {

struct Comm {
  int rank = 0, world = 1;
  unsigned long long bytes = 0;   // bytes moved by this rank's collectives so far (convention above)
  std::string err;                // message of the last failure
  virtual ~Comm() = default;
  // recv[k * count + i] = send of rank k [i]; dt: 0 fp32, 1 bf16.  0 = ok, else err is set.
  virtual int all_gather(const void* send, void* recv, size_t count, int dt, cudaStream_t st) = 0;
  // recv[i] = sum over ranks k (in rank order) of send_k[rank * count + i]  (dt: 0 fp32, 1 bf16)
  virtual int reduce_scatter(const void* send, void* recv, size_t count, int dt, cudaStream_t st) = 0;
  // recv[i] = sum over ranks k (in rank order) of send_k[i]
  virtual int all_reduce(const void* send, void* recv, size_t count, int dt, cudaStream_t st) = 0;
  // recv[k * count + i] = send of rank k [rank * count + i] (equal blocks; the feature-processing layer's pooled
  // embedding exchange)
  virtual int all_to_all(const void* send, void* recv, size_t count, int dt, cudaStream_t st) = 0;
  virtual const char* name() const = 0;
};

// backend 0: NCCL communicator from a ncclUniqueId (128 bytes); backend 1: loopback group keyed by an id from
// loopback_new_id().  nullptr on failure (*err set).
Comm* comm_create(int backend, const unsigned char id[128], int world, int rank, std::string* err);
void loopback_new_id(unsigned char out[128]);

}  // namespace dhen
