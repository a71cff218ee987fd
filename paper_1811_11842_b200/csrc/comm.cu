// comm.cu -- NCCL transport (dlopen) for halos and reduction partials.
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "comm.h"
#include "common.cuh"

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  if (a.lib || a.ok) return a;
  // CHB_NCCL_LIB: another NCCL build (or the tests' in-process loopback stand-in)
  const char* path = getenv("CHB_NCCL_LIB");
  a.lib = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!a.lib) return a;
#define CHB_SYM(name) a.name = reinterpret_cast<decltype(a.name)>(dlsym(a.lib, "nccl" #name))
  CHB_SYM(GetUniqueId);
  CHB_SYM(CommInitRank);
  CHB_SYM(CommDestroy);
  CHB_SYM(AllGather);
  CHB_SYM(AllReduce);
  CHB_SYM(Send);
  CHB_SYM(Recv);
  CHB_SYM(GroupStart);
  CHB_SYM(GroupEnd);
  CHB_SYM(GetErrorString);
#undef CHB_SYM
  a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.AllReduce && a.Send && a.Recv &&
         a.GroupStart && a.GroupEnd && a.CommDestroy;
  return a;
}

}  // namespace

struct Comm {
  ncclComm_t comm;
  int rank, nranks;
};

int comm_unique_id(void* out, size_t len) {
  if (len < sizeof(ncclUniqueId)) return 1;
  NcclApi& a = api();
  if (!a.ok) return 5;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return 5;
  memcpy(out, &id, sizeof id);
  return 0;
}

Comm* comm_create(const void* id, size_t len, int rank, int nranks, int device, std::string* err) {
  NcclApi& a = api();
  if (!a.ok) {
    if (err) *err = "NCCL (libnccl.so.2) not loadable";
    return nullptr;
  }
  if (len < sizeof(ncclUniqueId)) {
    if (err) *err = "unique id too short";
    return nullptr;
  }
  cudaSetDevice(device);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  Comm* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = a.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    if (err) *err = std::string("ncclCommInitRank: ") + (a.GetErrorString ? a.GetErrorString(r) : "?");
    delete c;
    return nullptr;
  }
  return c;
}

int comm_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st) {
  return api().AllGather(send, recv, count, ncclFloat64, c->comm, st) == ncclSuccess ? 0 : 1;
}

int comm_halo(Comm* c, double* first_base, int first_nyl, double* last_base, int last_nyl,
              int pitch, int w, cudaStream_t st) {
  NcclApi& a = api();
  const size_t n = (size_t)w * pitch;
  const int GH = chb::GH;
  if (a.GroupStart() != ncclSuccess) return 1;
  if (c->rank > 0) {
    // my bottom rows -> rank-1's top ghosts; rank-1's top rows -> my bottom ghosts
    a.Send(first_base + (size_t)GH * pitch, n, ncclFloat64, c->rank - 1, c->comm, st);
    a.Recv(first_base + (size_t)(GH - w) * pitch, n, ncclFloat64, c->rank - 1, c->comm, st);
  }
  if (c->rank + 1 < c->nranks) {
    a.Send(last_base + (size_t)(last_nyl + GH - w) * pitch, n, ncclFloat64, c->rank + 1, c->comm, st);
    a.Recv(last_base + (size_t)(last_nyl + GH) * pitch, n, ncclFloat64, c->rank + 1, c->comm, st);
  }
  (void)first_nyl;
  return a.GroupEnd() == ncclSuccess ? 0 : 1;
}

int comm_iter_exchange(Comm* c, const double* send, double* recv, size_t count,
                       const HaloSpec* halos, int nhalo, int pitch, cudaStream_t st) {
  NcclApi& a = api();
  const int GH = chb::GH;
  if (a.GroupStart() != ncclSuccess) return 1;
  int bad = 0;
  if (count) bad |= a.AllGather(send, recv, count, ncclFloat64, c->comm, st) != ncclSuccess;
  for (int k = 0; k < nhalo; ++k) {
    const HaloSpec& h = halos[k];
    const size_t n = (size_t)h.w * pitch;
    if (c->rank > 0) {
      bad |= a.Send(h.first_base + (size_t)GH * pitch, n, ncclFloat64, c->rank - 1, c->comm, st) !=
             ncclSuccess;
      bad |= a.Recv(h.first_base + (size_t)(GH - h.w) * pitch, n, ncclFloat64, c->rank - 1,
                    c->comm, st) != ncclSuccess;
    }
    if (c->rank + 1 < c->nranks) {
      bad |= a.Send(h.last_base + (size_t)(h.last_nyl + GH - h.w) * pitch, n, ncclFloat64,
                    c->rank + 1, c->comm, st) != ncclSuccess;
      bad |= a.Recv(h.last_base + (size_t)(h.last_nyl + GH) * pitch, n, ncclFloat64, c->rank + 1,
                    c->comm, st) != ncclSuccess;
    }
  }
  bad |= a.GroupEnd() != ncclSuccess;
  return bad ? 1 : 0;
}

int comm_allreduce_sum(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st) {
  return api().AllReduce(send, recv, count, ncclFloat64, ncclSum, c->comm, st) == ncclSuccess ? 0
                                                                                              : 1;
}

int comm_allgather_host(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  char* d = nullptr;
  const size_t n = (size_t)c->nranks * bytes;
  if (cudaMalloc(&d, n + bytes) != cudaSuccess) return 1;
  int bad = cudaMemcpyAsync(d + n, send, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess;
  if (!bad) bad = api().AllGather(d + n, d, bytes, ncclUint8, c->comm, st) != ncclSuccess;
  if (!bad) bad = cudaMemcpyAsync(recv, d, n, cudaMemcpyDeviceToHost, st) != cudaSuccess;
  if (!bad) bad = cudaStreamSynchronize(st) != cudaSuccess;
  cudaFree(d);
  return bad;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  api().CommDestroy(c->comm);
  delete c;
}
