// Local shared-memory latency under concurrent distributed-shared-memory traffic
// (development microbenchmark). Thread 0 runs a chain of dependent local ATOMS or
// LDS while W other warps issue remote DSMEM loads / stores / atomics.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void bar() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t raddr(const void* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  return ra;
}
__global__ void kern(int mode, int W, int iters, long long* out) {
  __shared__ uint32_t buf[1024];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, rank = crank(), G = gridDim.x;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = i;
  bar();
  uint32_t idx = 0, acc = 0;
  long long tsum = 0;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int k = 0; k < 16; ++k) {
        if (mode & 1) idx = atomicAdd(&buf[idx & 1023], 1u) & 1023;
        else idx = buf[(idx + 7) & 1023] & 1023;
      }
      tsum += clock64() - t0;
    } else if (warp >= 1 && warp <= (uint32_t)W) {
      const uint32_t tgt = (rank + 1 + lane) % G;
      const uint32_t ra = raddr(&buf[(lane * 32 + it) & 1007], tgt);
      for (int k = 0; k < 16; ++k) {
        if ((mode >> 1) == 0) { uint32_t v; asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra + 4 * (acc & 7)) : "memory"); acc += v; }
        else if ((mode >> 1) == 1) { asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(ra + 4 * k), "r"(k) : "memory"); }
        else { uint32_t v; asm volatile("atom.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(v) : "r"(ra + 4 * (acc & 7)), "r"(k) : "memory"); acc += v; }
      }
    }
    bar();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tsum / iters / 16;
  if (acc == 12345) buf[0] = acc;
  bar();
}
int main() {
  long long* out; cudaMalloc(&out, 64 * 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"LDS   | remote ld", "ATOMS | remote ld", "LDS   | remote st", "ATOMS | remote st", "LDS   | remote exch", "ATOMS | remote exch"};
  for (int mode = 0; mode < 6; ++mode) for (int W : {0, 1, 4, 15}) {
    cudaLaunchConfig_t lc{}; lc.gridDim = dim3(16); lc.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; lc.attrs = at; lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, kern, mode, W, 500, out);
    { cudaError_t e = cudaDeviceSynchronize(); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; } }
    long long h[16]; cudaMemcpy(h, out, 16 * 8, cudaMemcpyDeviceToHost);
    long long s = 0; for (int i = 0; i < 16; ++i) s += h[i];
    printf("%-22s W=%2d  local op latency %5lld cycles\n", names[mode], W, s / 16);
  }
}
