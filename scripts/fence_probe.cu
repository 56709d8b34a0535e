// Cost of the release that publishes a TMA-stored piece, by scope and form
// (DESIGN.md §6b "system-scope signalling").  Each CTA repeats: bulk-load a
// piece into shared memory, bulk-store it elsewhere, wait for the store
// (cp.async.bulk.wait_group 0), then publish a flag with variant V:
//   0 none, 1 fence.acq_rel.gpu + st.relaxed.gpu, 2 fence.acq_rel.sys + st.relaxed.sys,
//   3 st.release.gpu, 4 st.release.sys.
// Prints ns per iteration (whole loop) and ns spent in the publish step alone.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_probe fence_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t sm(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void probe(char* src, char* dst, uint32_t* flags, uint32_t piece, int iters, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm);
  char* buf = reinterpret_cast<char*>(dsm) + 128;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t off = (size_t)blockIdx.x * piece;
  uint64_t pub = 0;
  const uint64_t t0 = gt();
  for (int i = 0; i < iters; ++i) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm(bar)), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sm(buf)), "l"(src + off), "r"(piece), "r"(sm(bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                 ::"r"(sm(bar)), "r"(i & 1) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(sm(buf)), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const uint64_t a = gt();
    uint32_t* f = flags + blockIdx.x * 32;
    if constexpr (V == 1) asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(i) : "memory");
    if constexpr (V == 2) asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(i) : "memory");
    if constexpr (V == 3) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(i) : "memory");
    if constexpr (V == 4) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(i) : "memory");
    pub += gt() - a;
  }
  const uint64_t t1 = gt();
  atomicAdd(&out[0], (unsigned long long)(t1 - t0));
  atomicAdd(&out[1], (unsigned long long)pub);
}

template <int V>
void run(const char* name, int ctas, uint32_t piece, char* src, char* dst, uint32_t* flags, unsigned long long* out) {
  const int iters = 200;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + piece);
  cudaMemset(out, 0, 16);
  probe<V><<<ctas, 32, 128 + piece>>>(src, dst, flags, piece, iters, out);
  cudaMemset(out, 0, 16);
  probe<V><<<ctas, 32, 128 + piece>>>(src, dst, flags, piece, iters, out);
  unsigned long long h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"%s\", \"ctas\": %d, \"piece\": %u, \"ns_per_iter\": %.1f, \"ns_publish\": %.1f}\n", name, ctas,
         piece, (double)h[0] / ctas / iters, (double)h[1] / ctas / iters);
}

int main() {
  char *src, *dst;
  uint32_t* flags;
  unsigned long long* out;
  const size_t big = 600ull << 20;
  cudaMalloc(&src, big);
  cudaMalloc(&dst, big);
  cudaMalloc(&flags, 1 << 20);
  cudaMalloc(&out, 16);
  cudaMemset(src, 1, big);
  for (int ctas : {1, 148, 592})
    for (uint32_t piece : {4096u, 16384u, 65536u}) {
      run<0>("none", ctas, piece, src, dst, flags, out);
      run<1>("fence.acq_rel.gpu+st.relaxed", ctas, piece, src, dst, flags, out);
      run<2>("fence.acq_rel.sys+st.relaxed", ctas, piece, src, dst, flags, out);
      run<3>("st.release.gpu", ctas, piece, src, dst, flags, out);
      run<4>("st.release.sys", ctas, piece, src, dst, flags, out);
    }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
