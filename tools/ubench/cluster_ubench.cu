// Microbenchmarks of the tier C round skeleton on B200 (development tool).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o cluster_ubench cluster_ubench.cu
// Prints cycles per iteration of: cluster barrier variants, barrier + DSMEM
// gather, L2 load / atomic latency after a barrier.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void bar_rel_acq() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void bar_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t dsmem_ld(const void* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), ra, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

// mode 0: barrier(rel/acq) only; 1: relaxed barrier; 2: barrier + dsmem gather + scan;
// 3: barrier + one dependent L2 load (lane 0); 4: barrier + global atomicExch (lane 0);
// 5: barrier + st.global by every thread then barrier; 6: __syncthreads only (no cluster)
__global__ void kern(int mode, int iters, uint32_t* gbuf, long long* out) {
  __shared__ uint32_t ctr[4];
  const uint32_t lane = threadIdx.x & 31, rank = crank();
  if (threadIdx.x < 4) ctr[threadIdx.x] = threadIdx.x + rank;
  bar_rel_acq();
  uint32_t acc = 0, idx = (blockIdx.x * 977u) & 0xFFFF;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    switch (mode) {
      case 0: bar_rel_acq(); break;
      case 1: bar_relaxed(); break;
      case 2: {
        bar_rel_acq();
        uint32_t v = lane < gridDim.x ? dsmem_ld(&ctr[0], lane) : 0;
        for (int o = 1; o < 32; o <<= 1) { uint32_t t = __shfl_up_sync(~0u, v, o); if (lane >= o) v += t; }
        acc += __shfl_sync(~0u, v, 31);
        break;
      }
      case 3: {
        bar_rel_acq();
        if (threadIdx.x == 0) { idx = gbuf[idx] & 0xFFFF; acc += idx; }
        break;
      }
      case 4: {
        bar_rel_acq();
        if (threadIdx.x == 0) { idx = atomicExch(&gbuf[idx], idx * 3 + 1) & 0xFFFF; acc += idx; }
        break;
      }
      case 5: {
        gbuf[(blockIdx.x * blockDim.x + threadIdx.x + it * 37) & 0xFFFF] = it;
        bar_rel_acq();
        break;
      }
      case 6: __syncthreads(); break;
      case 8: {  // barrier + one remote DSMEM load (thread 0)
        bar_rel_acq();
        if (threadIdx.x == 0) { idx = dsmem_ld(&ctr[idx & 3], (rank + 1) % gridDim.x); acc += idx; }
        break;
      }
      case 9: {  // barrier + 4 dependent remote DSMEM loads (lane 0 of each warp)
        bar_rel_acq();
        if (lane == 0) for (int k = 0; k < 4; ++k) idx = dsmem_ld(&ctr[idx & 3], (rank + k + 1) % gridDim.x);
        acc += idx;
        break;
      }
      case 10: {  // barrier + remote DSMEM atomic exchange (thread 0)
        bar_rel_acq();
        if (threadIdx.x == 0) {
          uint32_t a = (uint32_t)__cvta_generic_to_shared(&ctr[1]), ra, v;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((rank + 1) % gridDim.x));
          asm volatile("atom.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(v) : "r"(ra), "r"(idx) : "memory");
          idx = v & 0xFFFF; acc += v;
        }
        break;
      }
      case 11: {  // push pattern: __syncthreads, warp 0 lanes<G store to every CTA, barrier, local LDS scan
        __syncthreads();
        if (threadIdx.x < gridDim.x) {
          uint32_t a = (uint32_t)__cvta_generic_to_shared(&ctr[rank & 3]), ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(threadIdx.x));
          asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(ra), "r"(it) : "memory");
        }
        bar_rel_acq();
        uint32_t v = lane < 4 ? ctr[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) { uint32_t t = __shfl_up_sync(~0u, v, o); if (lane >= o) v += t; }
        acc += __shfl_sync(~0u, v, 31);
        break;
      }
      case 12: {  // 8 dependent local ATOMS by thread 0 (others idle at the barrier)
        if (threadIdx.x == 0) for (int k = 0; k < 8; ++k) idx = atomicAdd(&ctr[idx & 3], 1u) & 0xFFFF;
        bar_rel_acq();
        break;
      }
      case 13: {  // same, while warps 1.. hammer remote DSMEM with loads
        if (threadIdx.x == 0) for (int k = 0; k < 8; ++k) idx = atomicAdd(&ctr[idx & 3], 1u) & 0xFFFF;
        else if (threadIdx.x >= 32) for (int k = 0; k < 8; ++k) acc += dsmem_ld(&ctr[(acc + k) & 3], (rank + 1 + k) % gridDim.x);
        bar_rel_acq();
        break;
      }
      case 14: {  // 8 dependent local ATOMS by lane 0 of every warp, same address
        if (lane == 0) for (int k = 0; k < 8; ++k) idx = atomicAdd(&ctr[0], 1u) & 0xFFFF;
        bar_rel_acq();
        break;
      }
      case 15: {  // 8 dependent LDS by thread 0
        if (threadIdx.x == 0) for (int k = 0; k < 8; ++k) idx = ctr[idx & 3] & 0xFFFF;
        bar_rel_acq();
        break;
      }
      case 7: {  // dependent chain of 4 L2 loads per round by lane 0 of each warp
        bar_rel_acq();
        if (lane == 0) for (int k = 0; k < 4; ++k) { idx = gbuf[(idx + threadIdx.x) & 0xFFFF] & 0xFFFF; }
        acc += idx;
        break;
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (acc == 0xFFFFFFFF) gbuf[0] = acc;
  bar_rel_acq();
}

int main() {
  uint32_t* gbuf; long long* out;
  cudaMalloc(&gbuf, 65536 * 4); cudaMalloc(&out, 1024 * 8);
  uint32_t* h = new uint32_t[65536];
  for (int i = 0; i < 65536; ++i) h[i] = (i * 40503u + 17) & 0xFFFF;
  cudaMemcpy(gbuf, h, 65536 * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"barrier rel/acq", "barrier relaxed", "barrier+dsmem gather", "barrier+L2 load",
                         "barrier+atomicExch", "st.global+barrier", "__syncthreads", "barrier+4 dep L2 loads",
                         "barrier+dsmem load", "barrier+4 dep dsmem loads", "barrier+dsmem exch", "push counts+barrier",
                         "8 dep ATOMS + barrier", "8 dep ATOMS w/ DSMEM load + bar", "8 dep ATOMS all warps + bar",
                         "8 dep LDS + barrier"};
  for (int G : {1, 16}) for (int T : {256, 512}) for (int mode = 0; mode < 16; ++mode) {
    if (G == 1 && (mode == 2 || mode == 8 || mode == 9 || mode == 10 || mode == 11 || mode == 13)) continue;
    cudaLaunchConfig_t lc{}; lc.gridDim = dim3(G); lc.blockDim = dim3(T); lc.dynamicSmemBytes = 0;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; lc.attrs = at; lc.numAttrs = 1;
    int iters = 2000;
    cudaLaunchKernelEx(&lc, kern, mode, iters, gbuf, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("G=%d T=%d mode=%d error %s\n", G, T, mode, cudaGetErrorString(e)); return 1; }
    long long hout[16]; cudaMemcpy(hout, out, G * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < G; ++i) mx = hout[i] > mx ? hout[i] : mx;
    printf("G=%2d T=%4d %-26s %6lld cycles/iter\n", G, T, names[mode], mx);
  }
  return 0;
}
