// Flag hop latency between two CTAs on one B200 (the floor under every
// Phase-B round in team mode): CTA 0 and CTA 1 bounce a counter through two
// flags in global memory, 10000 round trips, with three signalling styles:
//   0: st.release.gpu / ld.acquire.gpu
//   1: fence.acq_rel.gpu + st.relaxed.gpu / ld.acquire.gpu  (the library's st_release/ld_acquire)
//   2: st.volatile + __threadfence / ld.volatile (relaxed polling)
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pingpong scripts/pingpong.cu && /tmp/pingpong
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_fence_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_pingpong(uint32_t* f, int iters, int style, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  uint32_t* mine = f + 32 * blockIdx.x;          // separate 128-byte lines
  uint32_t* other = f + 32 * (1 - blockIdx.x);
  unsigned long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (blockIdx.x == 0) {
      if (style == 0) st_rel(other, i); else if (style == 1) st_fence_relaxed(other, i);
      else { __threadfence(); *(volatile uint32_t*)other = i; }
      if (style == 2) { while (*(volatile uint32_t*)mine < (uint32_t)i) {} }
      else { while (ld_acq(mine) < (uint32_t)i) {} }
    } else {
      if (style == 2) { while (*(volatile uint32_t*)mine < (uint32_t)i) {} }
      else { while (ld_acq(mine) < (uint32_t)i) {} }
      if (style == 0) st_rel(other, i); else if (style == 1) st_fence_relaxed(other, i);
      else { __threadfence(); *(volatile uint32_t*)other = i; }
    }
  }
  if (blockIdx.x == 0) *out = clock64() - t0;
}

int main() {
  uint32_t* f;
  unsigned long long* out;
  cudaMalloc(&f, 4096);
  cudaMalloc(&out, 8);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int iters = 10000;
  for (int style = 0; style < 3; ++style) {
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(f, 0, 4096);
      k_pingpong<<<2, 32>>>(f, iters, style, out);
      unsigned long long cyc;
      cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      double ns_per_hop = cyc / (double)(2 * iters) / (clk_khz * 1e-6);
      best = ns_per_hop < best ? ns_per_hop : best;
    }
    printf("{\"style\": %d, \"one_way_ns\": %.0f}\n", style, best);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
