// HBM ceiling of the direct completion's access mix (2 reads : 8 writes per
// element of a chunk) when moved the way the kernel moves it: TMA bulk loads of
// two operands into a 3-stage shared-memory ring, one 16-byte add per vector,
// bulk stores of the result to 8 destinations (no flags, no schedule).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_mix tma_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sm(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NDST, int STAGES, int PIECE, bool ADD>
__global__ void __launch_bounds__(256) k_mix(const char* a, const char* b, char* const* dst, size_t bytes_per_cta) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm);
  char* stage = reinterpret_cast<char*>(dsm) + 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = blockIdx.x * bytes_per_cta;
  const uint32_t np = (uint32_t)(bytes_per_cta / PIECE);
  auto issue = [&](uint32_t i) {
    const int s = i % STAGES;
    char* st = stage + (size_t)s * 2 * PIECE;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm(&bar[s])), "r"(2 * PIECE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sm(st)), "l"(a + base + (size_t)i * PIECE), "r"(PIECE), "r"(sm(&bar[s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sm(st + PIECE)), "l"(b + base + (size_t)i * PIECE), "r"(PIECE), "r"(sm(&bar[s])) : "memory");
  };
  if (threadIdx.x == 0)
    for (uint32_t i = 0; i < np && i < STAGES - 1; ++i) issue(i);
  uint32_t ph = 0;
  for (uint32_t i = 0; i < np; ++i) {
    const int s = i % STAGES;
    char* st = stage + (size_t)s * 2 * PIECE;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                 ::"r"(sm(&bar[s])), "r"((ph >> s) & 1u) : "memory");
    ph ^= 1u << s;
    if (ADD) {
      uint4* A = reinterpret_cast<uint4*>(st);
      const uint4* B = reinterpret_cast<const uint4*>(st + PIECE);
      for (int v = threadIdx.x; v < PIECE / 16; v += blockDim.x) {
        uint4 x = A[v], y = B[v];
        A[v] = make_uint4(__float_as_uint(__uint_as_float(x.x) + __uint_as_float(y.x)),
                          __float_as_uint(__uint_as_float(x.y) + __uint_as_float(y.y)),
                          __float_as_uint(__uint_as_float(x.z) + __uint_as_float(y.z)),
                          __float_as_uint(__uint_as_float(x.w) + __uint_as_float(y.w)));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int d = 0; d < NDST; ++d)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[d] + base + (size_t)i * PIECE),
                     "r"(sm(st)), "r"(PIECE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (i + STAGES - 1 < np) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        issue(i + STAGES - 1);
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int NDST, int STAGES, int PIECE, bool ADD>
void run(const char* name, int ctas, char* a, char* b, char** dd, size_t n) {
  const size_t per = n / ctas / PIECE * PIECE;
  const int smem = 128 + STAGES * 2 * PIECE;
  cudaFuncSetAttribute(k_mix<NDST, STAGES, PIECE, ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    k_mix<NDST, STAGES, PIECE, ADD><<<ctas, 256, smem>>>(a, b, dd, per);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  const double bytes = (double)per * ctas * (2 + NDST);
  printf("{\"variant\": \"%s\", \"ctas\": %d, \"stages\": %d, \"piece\": %d, \"dst\": %d, \"GBps\": %.1f}\n", name, ctas,
         STAGES, PIECE, NDST, bytes / (best * 1e-3) / 1e9);
}

int main() {
  const size_t n = 256ull << 20;   // bytes per operand / destination
  char *a, *b, *d[8];
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  for (int i = 0; i < 8; ++i) cudaMalloc(&d[i], n);
  char** dd;
  cudaMalloc(&dd, sizeof(d));
  cudaMemcpy(dd, d, sizeof(d), cudaMemcpyHostToDevice);
  cudaMemset(a, 0, n);
  cudaMemset(b, 0, n);
  for (int ctas : {518, 592, 1036})
    run<8, 3, 8192, true>("2r8w add (direct completion's mover)", ctas, a, b, dd, n);
  run<8, 3, 8192, false>("2r8w no add", 592, a, b, dd, n);
  run<8, 4, 8192, true>("2r8w add, 4 stages", 444, a, b, dd, n);
  run<8, 3, 16384, true>("2r8w add, 16 KB pieces", 296, a, b, dd, n);
  run<8, 2, 16384, true>("2r8w add, 2 x 16 KB", 444, a, b, dd, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
