// Hardware probe for the critical-path bound of the DAG kernels (bench.py roofline): the
// latency of one dependency hop — a value published by a warp on one SM and observed by a
// polling warp on another, through L2 with the same relaxed 64-bit loads / stores as the
// value-as-flag readiness protocol (kernels.cuh).  A level-scheduled or sync-free solve of a
// DAG with L levels cannot finish in less than L such hops.
#include <cuda_runtime.h>

#include <string>

#include "../../include/kktb200.h"
#include "kernels.cuh"
#include "kkt_internal.h"

namespace kkt {

// block 0 publishes i in a[0] and waits for b[0] == i; block 1 mirrors it: 2 hops per round.
__global__ void k_pingpong(double *a, double *b, int rounds, unsigned long long *out) {
  if (threadIdx.x) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (blockIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    for (int i = 1; i <= rounds; ++i) {
      st_relaxed_f64(a, (double)i);
      while (ld_relaxed_f64(b) != (double)i) {
      }
    }
    out[0] = globaltimer() - t0;
    out[1] = smid;
  } else {
    for (int i = 1; i <= rounds; ++i) {
      while (ld_relaxed_f64(a) != (double)i) {
      }
      st_relaxed_f64(b, (double)i);
    }
    out[2] = smid;
  }
}

}  // namespace kkt

int kkt_probe_hop_ns(int device, int rounds, double *ns_per_hop) {
  if (!ns_per_hop || rounds < 1) return kkt::set_error(KKT_ERR_BAD_ARG, "bad argument");
  if (cudaSetDevice(device) != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, "cudaSetDevice");
  double *buf = nullptr;
  unsigned long long *out = nullptr, host[3] = {0, 0, 0};
  cudaError_t e = cudaMalloc(&buf, 512);
  if (e == cudaSuccess) e = cudaMalloc(&out, 64);
  if (e == cudaSuccess) e = cudaMemset(buf, 0, 512);
  if (e == cudaSuccess) {
    // the two words on different 128-byte lines; two CTAs of 120 KB dynamic shared memory
    // cannot share an SM (228 KB), so every hop crosses SMs
    const int smem = 120 * 1024;
    e = cudaFuncSetAttribute(kkt::k_pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) {
      kkt::k_pingpong<<<2, 32, smem>>>(buf, buf + 32, rounds, out);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaMemcpy(host, out, sizeof host, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  cudaFree(out);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, std::string("probe: ") + cudaGetErrorString(e));
  if (host[1] == host[2]) return kkt::set_error(KKT_ERR_CUDA, "probe: both CTAs on one SM");
  *ns_per_hop = (double)host[0] / (2.0 * rounds);
  return KKT_OK;
}
