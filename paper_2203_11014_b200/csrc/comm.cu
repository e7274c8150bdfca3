// comm.cu — collective backends of the FSDP path (comm.h): NCCL, and the in-process loopback.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "kernels.h"

namespace dhen {

// ------------------------------------------------------------------ NCCL
namespace {

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  int chk(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return 0;
    err = std::string(what) + ": " + ncclGetErrorString(r);
    return 1;
  }
  int all_gather(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2);
    return chk(ncclAllGather(send, recv, count, dt == F32 ? ncclFloat32 : ncclBfloat16, c, st), "ncclAllGather");
  }
  int reduce_scatter(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2);
    return chk(ncclReduceScatter(send, recv, count, dt == F32 ? ncclFloat32 : ncclBfloat16, ncclSum, c, st),
               "ncclReduceScatter");
  }
  int all_reduce(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += 2ull * (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2) / (unsigned long long)world;
    return chk(ncclAllReduce(send, recv, count, dt == F32 ? ncclFloat32 : ncclBfloat16, ncclSum, c, st), "ncclAllReduce");
  }
  int all_to_all(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    const size_t es = dt == F32 ? 4 : 2;
    bytes += (unsigned long long)(world - 1) * count * es;
    const ncclDataType_t t = dt == F32 ? ncclFloat32 : ncclBfloat16;
    if (chk(ncclGroupStart(), "ncclGroupStart")) return 1;
    for (int k = 0; k < world; ++k) {
      if (chk(ncclSend((const char*)send + k * count * es, count, t, k, c, st), "ncclSend")) return 1;
      if (chk(ncclRecv((char*)recv + k * count * es, count, t, k, c, st), "ncclRecv")) return 1;
    }
    return chk(ncclGroupEnd(), "ncclGroupEnd");
  }
  const char* name() const override { return "nccl"; }
};

// ------------------------------------------------------------------ loopback (virtual ranks, one process)
constexpr int kMaxLoop = 16;
constexpr int kAG = 0, kRS = 1, kAR = 2, kA2A = 3;

struct SumSrc {
  const void* p[kMaxLoop];
  int n;
};
// dst[i] = src_0[i] + src_1[i] + ... (rank order: deterministic), in fp32; bf16 operands rounded once at the end
template <typename T>
__global__ void loop_sum_k(SumSrc s, T* __restrict__ dst, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float a = tof<T>(static_cast<const T*>(s.p[0])[i]);
    for (int k = 1; k < s.n; ++k) a += tof<T>(static_cast<const T*>(s.p[k])[i]);
    dst[i] = fromf<T>(a);
  }
}

struct LoopGroup {
  int world = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  unsigned long long gen = 0;
  int arrived = 0;
  struct Slot {
    int kind;
    const void* send;
    void* recv;
    size_t count;
    int dt;
    cudaEvent_t ready;
  };
  std::vector<Slot> slot;
  cudaEvent_t done[2] = {nullptr, nullptr};
  bool broken = false;
  std::string why;
};
std::mutex g_groups_mu;
std::map<std::string, LoopGroup*> g_groups;

struct LoopComm final : Comm {
  LoopGroup* g = nullptr;
  std::string key;
  cudaEvent_t ready = nullptr;
  ~LoopComm() override {
    if (ready) cudaEventDestroy(ready);
    if (!g) return;
    std::lock_guard<std::mutex> lk(g_groups_mu);
    if (g && --g->refs == 0) {
      for (auto& e : g->done) if (e) cudaEventDestroy(e);
      g_groups.erase(key);
      delete g;
    }
  }
  // the last arriver enqueues the whole collective on its stream (every rank's input ready before)
  int perform(cudaStream_t st) {
    const auto& s0 = g->slot[0];
    for (int k = 0; k < world; ++k) {
      const auto& sk = g->slot[k];
      if (sk.kind != s0.kind || sk.count != s0.count || sk.dt != s0.dt) {
        char b[256];
        snprintf(b, sizeof b, "loopback: mismatched collectives (rank 0 kind %d count %zu, rank %d kind %d count %zu)",
                 s0.kind, s0.count, k, sk.kind, sk.count);
        err = b;
        return 1;
      }
      if (cudaStreamWaitEvent(st, sk.ready, 0) != cudaSuccess) { err = "loopback: cudaStreamWaitEvent"; return 1; }
    }
    const size_t n = s0.count;
    if (s0.kind == kA2A) {
      const size_t es = s0.dt == F32 ? 4 : 2;
      for (int r = 0; r < world; ++r)
        for (int k = 0; k < world; ++k)
          if (n && cudaMemcpyAsync((char*)g->slot[r].recv + k * n * es, (const char*)g->slot[k].send + r * n * es, n * es,
                                   cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
            err = "loopback: all-to-all copy";
            return 1;
          }
    } else if (s0.kind == kAG) {
      const size_t es = s0.dt == F32 ? 4 : 2;
      for (int r = 0; r < world; ++r)
        for (int k = 0; k < world; ++k)
          if (cudaMemcpyAsync((char*)g->slot[r].recv + k * n * es, g->slot[k].send, n * es, cudaMemcpyDeviceToDevice,
                              st) != cudaSuccess) {
            err = "loopback: all-gather copy";
            return 1;
          }
    } else {
      const size_t es = s0.dt == F32 ? 4 : 2;
      for (int r = 0; r < world; ++r) {
        SumSrc src;
        src.n = world;
        for (int k = 0; k < world; ++k)
          src.p[k] = (const char*)g->slot[k].send + (s0.kind == kRS ? (size_t)r * n * es : 0);
        const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
        if (n) {
          if (s0.dt == F32) loop_sum_k<float><<<grid > 0 ? grid : 1, 256, 0, st>>>(src, (float*)g->slot[r].recv, n);
          else loop_sum_k<__nv_bfloat16><<<grid > 0 ? grid : 1, 256, 0, st>>>(src, (__nv_bfloat16*)g->slot[r].recv, n);
        }
        ++g_launches;
      }
      if (cudaGetLastError() != cudaSuccess) { err = "loopback: sum kernel launch"; return 1; }
    }
    return 0;
  }
  int collective(int kind, const void* send, void* recv, size_t count, int dt, cudaStream_t st) {
    if (cudaEventRecord(ready, st) != cudaSuccess) { err = "loopback: cudaEventRecord"; return 1; }
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->broken) { err = "loopback group broken: " + g->why; return 1; }
    g->slot[rank] = {kind, send, recv, count, dt, ready};
    const unsigned long long my = g->gen;
    int rc = 0;
    if (++g->arrived == world) {
      rc = perform(st);
      if (rc == 0 && cudaEventRecord(g->done[my & 1], st) != cudaSuccess) { err = "loopback: done record"; rc = 1; }
      if (rc) { g->broken = true; g->why = err; }
      g->arrived = 0;
      ++g->gen;
      g->cv.notify_all();
      return rc;
    }
    // every rank's next collective needs this one complete, so two alternating done events suffice
    if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->gen != my || g->broken; })) {
      g->broken = true;
      g->why = "rendezvous timeout (a rank never reached this collective)";
      g->cv.notify_all();
    }
    if (g->broken) { err = "loopback group broken: " + g->why; return 1; }
    const cudaEvent_t d = g->done[my & 1];
    lk.unlock();
    if (cudaStreamWaitEvent(st, d, 0) != cudaSuccess) { err = "loopback: cudaStreamWaitEvent(done)"; return 1; }
    return 0;
  }
  int all_gather(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2);
    return collective(kAG, send, recv, count, dt, st);
  }
  int reduce_scatter(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2);
    return collective(kRS, send, recv, count, dt, st);
  }
  int all_reduce(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += 2ull * (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2) / (unsigned long long)world;
    return collective(kAR, send, recv, count, dt, st);
  }
  int all_to_all(const void* send, void* recv, size_t count, int dt, cudaStream_t st) override {
    bytes += (unsigned long long)(world - 1) * count * (dt == F32 ? 4 : 2);
    return collective(kA2A, send, recv, count, dt, st);
  }
  const char* name() const override { return "loopback"; }
};

}  // namespace

void loopback_new_id(unsigned char out[128]) {
  static std::mutex mu;
  static std::mt19937_64 rng(std::random_device{}());
  std::lock_guard<std::mutex> lk(mu);
  memset(out, 0, 128);
  memcpy(out, "dhen-loopback:", 14);
  for (int i = 16; i < 48; i += 8) {
    const unsigned long long v = rng();
    memcpy(out + i, &v, 8);
  }
}

Comm* comm_create(int backend, const unsigned char id[128], int world, int rank, std::string* err) {
  if (backend == 0) {
    auto* c = new NcclComm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId uid;
    memcpy(uid.internal, id, 128);
    const ncclResult_t r = ncclCommInitRank(&c->c, world, uid, rank);
    if (r != ncclSuccess) {
      *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      c->c = nullptr;
      delete c;
      return nullptr;
    }
    return c;
  }
  if (backend == 1) {
    if (world > kMaxLoop || memcmp(id, "dhen-loopback:", 14) != 0) {
      *err = "loopback: world > 16 or the id is not from dhen_loopback_id";
      return nullptr;
    }
    auto* c = new LoopComm();
    c->rank = rank;
    c->world = world;
    c->key.assign((const char*)id, 128);
    if (cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming) != cudaSuccess) {
      *err = "loopback: event creation";
      delete c;
      return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_groups_mu);
    LoopGroup*& g = g_groups[c->key];
    if (!g) {
      g = new LoopGroup();
      g->world = world;
      g->slot.resize(world);
      for (auto& e : g->done)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
          *err = "loopback: event creation";
          delete c;
          return nullptr;
        }
    }
    if (g->world != world) {
      *err = "loopback: world differs from the group's";
      delete c;
      return nullptr;
    }
    ++g->refs;
    c->g = g;
    return c;
  }
  *err = "unknown collective backend";
  return nullptr;
}

}  // namespace dhen
