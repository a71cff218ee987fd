// fake_nccl.cpp -- TEST INFRASTRUCTURE ONLY: an in-process loopback stand-in
// for libnccl.so.2 (the subset comm.cu uses), so that the library's
// multi-rank code path (rank slabs, NCCL halo rows, allgather of partial sums,
// cross-rank finalize) runs with several ranks = host threads of ONE process
// on ONE GPU.  Loaded instead of NCCL via env CHB_NCCL_LIB.  Every group is
// executed on the host: each rank synchronizes its streams, posts its
// operations, meets the other ranks at a barrier, copies what it receives
// (cudaMemcpy, device to device), and meets them again.  Host-synchronous and
// slow by design; it proves the index and ordering logic, not performance.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace {

enum Kind { SEND, RECV, ALLGATHER, ALLREDUCE };

struct Fabric;
struct Comm {
  Fabric* f;
  int rank, nranks;
};

struct Op {
  Kind kind;
  const void* src;
  void* dst;
  size_t bytes;
  int peer;
  cudaStream_t st;
  Comm* comm;
};

struct Fabric {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<std::vector<Op>> posted;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_mu;
std::map<std::string, Fabric*> g_fabrics;
thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;
long g_counter = 0;

size_t dtype_size(int dt) {
  switch (dt) {
    case 0: case 1: return 1;   // int8 / uint8
    case 2: case 3: case 4: return 4;  // int32 / uint32 / float32? (int32=2, uint32=3)
    case 5: return 8;   // int64
    case 6: return 2;   // float16
    case 7: return 4;   // float32
    case 8: return 8;   // float64
    default: return 8;
  }
}

int run_group(std::vector<Op>& ops) {
  if (ops.empty()) return 0;
  Comm* c = ops[0].comm;
  Fabric* f = c->f;
  for (auto& o : ops)
    if (cudaStreamSynchronize(o.st) != cudaSuccess) return 3;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    f->posted[c->rank] = ops;
  }
  f->barrier();
  int bad = 0;
  std::map<int, int> recv_seen;  // peer -> receives matched so far
  int ag_seen = 0, ar_seen = 0;
  for (auto& o : ops) {
    if (o.kind == RECV) {
      const int k = recv_seen[o.peer]++;
      int n = 0;
      const Op* match = nullptr;
      for (auto& s : f->posted[o.peer])
        if (s.kind == SEND && s.peer == c->rank && n++ == k) { match = &s; break; }
      if (!match || match->bytes != o.bytes) { bad = 1; continue; }
      bad |= cudaMemcpy(o.dst, match->src, o.bytes, cudaMemcpyDeviceToDevice) != cudaSuccess;
    } else if (o.kind == ALLGATHER) {
      const int k = ag_seen++;
      for (int r = 0; r < c->nranks; ++r) {
        int n = 0;
        const Op* m = nullptr;
        for (auto& s : f->posted[r])
          if (s.kind == ALLGATHER && n++ == k) { m = &s; break; }
        if (!m || m->bytes != o.bytes) { bad = 1; continue; }
        bad |= cudaMemcpy(static_cast<char*>(o.dst) + r * o.bytes, m->src, o.bytes,
                          cudaMemcpyDeviceToDevice) != cudaSuccess;
      }
    } else if (o.kind == ALLREDUCE) {  // float64 sum
      const int k = ar_seen++;
      const size_t n8 = o.bytes / 8;
      std::vector<double> acc(n8, 0.0), tmp(n8);
      for (int r = 0; r < c->nranks; ++r) {
        int n = 0;
        const Op* m = nullptr;
        for (auto& s : f->posted[r])
          if (s.kind == ALLREDUCE && n++ == k) { m = &s; break; }
        if (!m) { bad = 1; continue; }
        bad |= cudaMemcpy(tmp.data(), m->src, o.bytes, cudaMemcpyDeviceToHost) != cudaSuccess;
        for (size_t i = 0; i < n8; ++i) acc[i] += tmp[i];
      }
      bad |= cudaMemcpy(o.dst, acc.data(), o.bytes, cudaMemcpyHostToDevice) != cudaSuccess;
    }
  }
  f->barrier();  // nobody reuses a posted buffer before every copy is done
  return bad ? 3 : 0;
}

int submit(const Op& o) {
  if (t_depth > 0) {
    t_ops.push_back(o);
    return 0;
  }
  std::vector<Op> one{o};
  return run_group(one);
}

}  // namespace

extern "C" {

struct FakeUniqueId {
  char internal[128];
};

int ncclGetVersion(int* v) {
  *v = 0;
  return 0;
}

int ncclGetUniqueId(FakeUniqueId* id) {
  std::lock_guard<std::mutex> lk(g_mu);
  memset(id->internal, 0, 128);
  snprintf(id->internal, 128, "fake-nccl-%ld", ++g_counter);
  return 0;
}

int ncclCommInitRank(Comm** comm, int nranks, FakeUniqueId id, int rank) {
  std::lock_guard<std::mutex> lk(g_mu);
  const std::string key(id.internal, strnlen(id.internal, 128));
  Fabric*& f = g_fabrics[key];
  if (!f) {
    f = new Fabric();
    f->nranks = nranks;
    f->posted.resize(nranks);
  }
  if (f->nranks != nranks || rank < 0 || rank >= nranks) return 4;
  *comm = new Comm{f, rank, nranks};
  return 0;
}

int ncclCommDestroy(Comm* c) {
  delete c;
  return 0;
}

int ncclAllGather(const void* send, void* recv, size_t count, int dt, Comm* c, cudaStream_t st) {
  return submit(Op{ALLGATHER, send, recv, count * dtype_size(dt), -1, st, c});
}

int ncclAllReduce(const void* send, void* recv, size_t count, int dt, int op, Comm* c,
                  cudaStream_t st) {
  if (dt != 8 || op != 0) return 4;  // float64 sum only
  return submit(Op{ALLREDUCE, send, recv, count * 8, -1, st, c});
}

int ncclSend(const void* buf, size_t count, int dt, int peer, Comm* c, cudaStream_t st) {
  return submit(Op{SEND, buf, nullptr, count * dtype_size(dt), peer, st, c});
}

int ncclRecv(void* buf, size_t count, int dt, int peer, Comm* c, cudaStream_t st) {
  return submit(Op{RECV, nullptr, buf, count * dtype_size(dt), peer, st, c});
}

int ncclGroupStart() {
  ++t_depth;
  return 0;
}

int ncclGroupEnd() {
  if (t_depth <= 0) return 5;
  if (--t_depth > 0) return 0;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return run_group(ops);
}

const char* ncclGetErrorString(int r) { return r ? "fake nccl error" : "no error"; }

}  // extern "C"
