// One flag hop between two CTAs of one kernel (different SMs), by memory-model
// scope and form: what a Phase-B hand-off costs at GPU vs system scope with no
// data in flight.  Prints ns per one-way hop (round trip / 2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong_scope pingpong_scope.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int V>
__device__ __forceinline__ void sig(uint32_t* f, uint32_t v) {
  if constexpr (V == 0) asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  if constexpr (V == 1) asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  if constexpr (V == 2) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  if constexpr (V == 3) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  if constexpr (V == 4) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(f) : "memory");
  if constexpr (V == 5) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
template <int V>
__device__ __forceinline__ uint32_t poll(const uint32_t* f) {
  uint32_t x;
  if constexpr (V == 0 || V == 5)
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
  else if constexpr (V == 3)
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
  else
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
  return x;
}

template <int V>
__global__ void pp(uint32_t* flags, int iters, unsigned long long* out) {
  if (threadIdx.x) return;
  uint32_t* mine = flags + blockIdx.x * 64;
  uint32_t* theirs = flags + (1 - blockIdx.x) * 64;
  const uint64_t t0 = gt();
  for (int i = 1; i <= iters; ++i) {
    if (blockIdx.x == 0) sig<V>(theirs, i);
    while ((int)(poll<V>(mine) - (uint32_t)i) < 0) {}
    if (blockIdx.x == 1) sig<V>(theirs, i);
  }
  if (blockIdx.x == 0) out[0] = gt() - t0;
}

template <int V>
void run(const char* name, uint32_t* flags, unsigned long long* out) {
  const int iters = 5000;
  cudaMemset(flags, 0, 4096);
  pp<V><<<2, 32>>>(flags, iters, out);   // warm
  cudaMemset(flags, 0, 4096);
  pp<V><<<2, 32>>>(flags, iters, out);
  unsigned long long h = 0;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"%s\", \"ns_per_hop\": %.1f}\n", name, (double)h / iters / 2);
}

int main() {
  uint32_t* flags;
  unsigned long long* out;
  cudaMalloc(&flags, 4096);
  cudaMalloc(&out, 8);
  run<0>("fence.acq_rel.gpu+st.relaxed.gpu / ld.acquire.gpu", flags, out);
  run<1>("fence.acq_rel.sys+st.relaxed.sys / ld.acquire.sys", flags, out);
  run<2>("st.release.sys / ld.acquire.sys", flags, out);
  run<3>("st.relaxed.sys / ld.relaxed.sys (no ordering)", flags, out);
  run<4>("red.release.sys.add / ld.acquire.sys", flags, out);
  run<5>("st.release.gpu / ld.acquire.gpu", flags, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
