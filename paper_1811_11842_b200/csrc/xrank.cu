// xrank.cu -- self-test of the peer-memory combine protocol of the multi-slab
// CG sweep (common.cuh xrank_combine), run on ONE GPU as one cooperative
// launch in which R groups of CTAs play R ranks (each group with its own
// totals area, flags and peer table pointing at the other groups' areas).
// The product sweep runs the very same device function: across processes the
// areas are NVLink peer mappings (ch_comm_init), within one process R = 1.
// Emulating the ranks inside one launch is how blocks that wait on one another
// may share a GPU (separate launches that spin on each other may not).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "ch_b200.h"
#include "common.cuh"

namespace chb {

// block b: rank b / nloc, local slab b % nloc (one warp per block).  Each slab
// waits a pseudo-random time, stores its totals (vals[global slab][k]), takes
// its rank's ticket; the rank's last slab runs the combine.  A rank equal to
// `absent` never arrives (the others must report a timeout, not hang).
__global__ void __launch_bounds__(32) k_xrank_selftest(const XPeers* xps, double* loc,
                                                        unsigned* tickets, int nloc,
                                                        unsigned epoch, const double* vals,
                                                        int absent, double* out, int* fail) {
  const int lane = threadIdx.x;
  const int r = blockIdx.x / nloc, s = blockIdx.x % nloc;
  const XPeers* xp = xps + r;
  if (r == absent) return;
  unsigned x = (epoch * 2654435761u) ^ (blockIdx.x * 40503u + 12345u);
  x ^= x >> 13;
  x *= 0x5bd1e995u;
  x ^= x >> 15;
  const unsigned wait_ns = x % 20000u;   // up to 20 us: arrival orders differ per epoch
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < wait_ns);
  double* myloc = loc + (size_t)r * MS_MAX * 8;
  if (lane < 3) myloc[s * 8 + lane] = vals[(size_t)(xp->slab0 + s) * 3 + lane];
  __syncwarp();
  unsigned prev = 0;
  if (lane == 0)
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(tickets + r) : "memory");
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != (unsigned)(nloc - 1)) return;
  if (lane == 0) tickets[r] = 0u;
  double t[8];
  const bool ok = xrank_combine<3>(xp, epoch, myloc, nloc, t);
  if (lane == 0) {
    if (!ok) atomicAdd(fail + r, 1);
    for (int k = 0; k < 3; ++k) out[r * 8 + k] = ok ? t[k] : 0.0;
  }
}

// Probe of a freshly mapped clique (ch_comm_init, before any sweep uses it):
// the same stores and the same combine as one multi-slab CG iteration.  Every
// thread writes the pattern row * 1e6 + column + 0.25 of the first two rows of
// its first slab into the lower neighbour's ghost rows and of the last two rows
// of its last slab into the upper neighbour's (through `lo` / `hi`, offset like
// the sweep's zlo / zhi), fences at system scope, then warp 0 runs
// xrank_combine on the totals (r + 1) * (k + 1) of each local slab.  The
// caller checks its own ghost rows and the sums after the kernel.
__global__ void __launch_bounds__(256) k_peer_probe(const XPeers* xp, unsigned epoch, double* loc,
                                                     int nloc, Geom g0, double* lo, Geom g1,
                                                     double* hi, double* out) {
  const int t = threadIdx.x;
  for (int c = t; c < g0.nx; c += blockDim.x) {
    if (lo)
      for (int r = 0; r < 2; ++r) {
        const int gq = g0.j0 + r;
        lo[off(g0, gq, c)] = gq * 1e6 + c + 0.25;
      }
    if (hi)
      for (int r = 0; r < 2; ++r) {
        const int gq = g1.j0 + g1.nyl - 2 + r;
        hi[off(g1, gq, c)] = gq * 1e6 + c + 0.25;
      }
  }
  if (t < nloc * 3) loc[(t / 3) * 8 + t % 3] = (xp->rank + 1.0) * (t % 3 + 1.0);
  __threadfence_system();
  __syncthreads();
  if (t < 32) {
    double r[8];
    const bool ok = xrank_combine<3>(xp, epoch, loc, nloc, r);
    if (t == 0)
      for (int k = 0; k < 3; ++k) out[k] = ok ? r[k] : -1.0;
  }
}

void launch_peer_probe(const XPeers* xp, unsigned epoch, double* loc, int nloc, const Geom& g0,
                       double* lo, const Geom& g1, double* hi, double* out, cudaStream_t st) {
  k_peer_probe<<<1, 256, 0, st>>>(xp, epoch, loc, nloc, g0, lo, g1, hi, out);
}

}  // namespace chb

using namespace chb;

extern "C" int ch_selftest_xrank(int device, int nranks, int nloc, int epochs, int absent_epoch,
                                 double* last) {
  if (nranks < 1 || nranks > XR_MAX || nloc < 1 || nloc > MS_MAX || nranks * nloc > XS_MAX ||
      epochs < 1)
    return -CH_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return -CH_ERR_CUDA;
  const int R = nranks, N = nranks * nloc;
  const size_t tot_bytes = (size_t)2 * XS_MAX * 8 * sizeof(double), area = tot_bytes + 256;
  char* areas = nullptr;
  XPeers* xps = nullptr;
  double *loc = nullptr, *vals = nullptr, *out = nullptr;
  unsigned* tickets = nullptr;
  int* fail = nullptr;
  int bad = 0;
  bad |= cudaMalloc(&areas, area * R) != cudaSuccess;
  bad |= cudaMalloc(&xps, sizeof(XPeers) * R) != cudaSuccess;
  bad |= cudaMalloc(&loc, sizeof(double) * R * MS_MAX * 8) != cudaSuccess;
  bad |= cudaMalloc(&vals, sizeof(double) * N * 3) != cudaSuccess;
  bad |= cudaMalloc(&out, sizeof(double) * R * 8) != cudaSuccess;
  bad |= cudaMalloc(&tickets, sizeof(unsigned) * R) != cudaSuccess;
  bad |= cudaMalloc(&fail, sizeof(int) * R) != cudaSuccess;
  int mismatches = 0;
  if (!bad) {
    cudaMemset(areas, 0, area * R);
    cudaMemset(tickets, 0, sizeof(unsigned) * R);
    std::vector<XPeers> hx(R);
    for (int r = 0; r < R; ++r) {
      memset(&hx[r], 0, sizeof(XPeers));
      hx[r].R = R;
      hx[r].rank = r;
      hx[r].slab0 = r * nloc;
      hx[r].nslab_all = N;
      for (int q = 0; q < R; ++q) {
        hx[r].tot[q] = reinterpret_cast<double*>(areas + area * q);
        hx[r].flag[q] = reinterpret_cast<unsigned*>(areas + area * q + tot_bytes);
      }
    }
    cudaMemcpy(xps, hx.data(), sizeof(XPeers) * R, cudaMemcpyHostToDevice);
    std::vector<double> hv((size_t)N * 3), ho((size_t)R * 8);
    std::vector<int> hf(R);
    for (int e = 1; e <= epochs && !bad; ++e) {
      // totals with rounding-sensitive magnitudes: the sum must follow slab order
      for (int g = 0; g < N; ++g)
        for (int k = 0; k < 3; ++k)
          hv[(size_t)g * 3 + k] = (g & 1 ? 1e16 : 1.0) * (1.0 + 0.1 * g + 1e-3 * e) / (k + 3.0);
      cudaMemcpy(vals, hv.data(), sizeof(double) * N * 3, cudaMemcpyHostToDevice);
      cudaMemset(fail, 0, sizeof(int) * R);
      const int absent = (e == absent_epoch) ? R - 1 : -1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)N);
      cfg.blockDim = dim3(32);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;   // all blocks co-resident
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      bad |= cudaLaunchKernelEx(&cfg, k_xrank_selftest, (const XPeers*)xps, loc, tickets, nloc,
                                (unsigned)e, (const double*)vals, absent, out, fail) != cudaSuccess;
      bad |= cudaDeviceSynchronize() != cudaSuccess;
      cudaMemcpy(ho.data(), out, sizeof(double) * R * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hf.data(), fail, sizeof(int) * R, cudaMemcpyDeviceToHost);
      for (int r = 0; r < R; ++r) {
        if (r == absent) continue;
        if (absent >= 0) {   // every present rank must have timed out
          mismatches += hf[r] != 1;
          continue;
        }
        mismatches += hf[r] != 0;
        for (int k = 0; k < 3; ++k) {
          double a = 0.0;
          for (int g = 0; g < N; ++g) a += hv[(size_t)g * 3 + k];
          mismatches += memcmp(&a, &ho[(size_t)r * 8 + k], sizeof a) != 0;
        }
      }
      if (absent >= 0) {
        // the absent rank's flag stays behind: restart the flags for the next epoch
        cudaMemset(areas, 0, area * R);
        cudaMemset(tickets, 0, sizeof(unsigned) * R);
      }
      if (last && e == epochs)
        for (int i = 0; i < R * 8; ++i) last[i] = ho[i];
    }
  }
  cudaFree(areas);
  cudaFree(xps);
  cudaFree(loc);
  cudaFree(vals);
  cudaFree(out);
  cudaFree(tickets);
  cudaFree(fail);
  if (bad) return -CH_ERR_CUDA;
  return mismatches;
}
