// comm.h -- inter-process transport for the slab decomposition (internal).
// NCCL is loaded at run time (dlopen "libnccl.so.2", the library torch already
// uses) only when a handle has nranks > 1, so single-GPU use has no NCCL
// dependency.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <string>

struct Comm;

int comm_unique_id(void* out, size_t len);
Comm* comm_create(const void* id, size_t len, int rank, int nranks, int device, std::string* err);
// recv[r * count .. (r+1) * count) = send of rank r (rank-ordered, deterministic)
int comm_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st);
// y-slab halo: the first local slab exchanges its bottom w rows with rank-1,
// the last local slab its top w rows with rank+1 (non-periodic in y).
int comm_halo(Comm* c, double* first_base, int first_nyl, double* last_base, int last_nyl,
              int pitch, int w, cudaStream_t st);
// One NCCL group per CG iteration: the allgather of the per-slab partial sums
// and the halo rows of up to 4 arrays (first/last local slab bases, width w[k])
// travel together, so an iteration costs one NCCL launch instead of three.
struct HaloSpec {
  double* first_base;
  double* last_base;
  int last_nyl;
  int w;
};
int comm_iter_exchange(Comm* c, const double* send, double* recv, size_t count,
                       const HaloSpec* halos, int nhalo, int pitch, cudaStream_t st);
// recv = sum over ranks of send (`count` device doubles, distinct buffers), on stream st (0 = ok)
int comm_allreduce_sum(Comm* c, const double* send, double* recv, size_t count, cudaStream_t st);
// recv[r * bytes .. (r+1) * bytes) = send of rank r; host buffers (staged
// through device memory, synchronous on st): setup-time metadata only
int comm_allgather_host(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t st);
void comm_destroy(Comm* c);
