// Does a system-scope release stall a CTA's TMA stream, and can it be hidden?
// (round 2: the sys-scope Phase-B gap is all in fence.acq_rel.sys.)
//
// 592 CTAs (4 per SM) each copy their own region src -> dst in 16 KB pieces
// through a 3-stage shared-memory ring (cp.async.bulk, like kernels.cuh
// tma_copy).  Every U pieces (a "unit", the library's ~128 KB sub-slice) a
// flag is published for the unit, in one of these modes:
//   0 none            no flag (pure stream: the ceiling)
//   1 drain           thread 0: wait_group 0, fence, flag; the next unit's loads
//                     start only after the flag (the library's default hand-off)
//   2 defer           thread 0 keeps loading across units; after the next unit's
//                     first store: wait_group 1, fence, flag (STRAGGLAR_DEFER_SEND)
//   3 signaller       as 2, but thread 0 only passes the unit to a thread of warp 1
//                     through shared memory (release/acquire at CTA scope); that
//                     thread issues the fence and the flag
// each with the fence at GPU or system scope.  Prints GB/s (read + write bytes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_overlap fence_overlap.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kStages = 3;
constexpr uint32_t kPiece = 16384;

__device__ __forceinline__ uint32_t sm(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void load(void* s, const void* g, uint32_t n, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm(bar)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm(s)),
               "l"(g), "r"(n), "r"(sm(bar))
               : "memory");
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   sm(bar)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void store(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sm(s)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <bool SYS>
__device__ __forceinline__ void publish(uint32_t* f, uint32_t v) {
  if constexpr (SYS)
    asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  else
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

template <int MODE, bool SYS>
__global__ void __launch_bounds__(256) stream(const char* src, char* dst, uint32_t* flags, uint64_t bytes, int U) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm);
  volatile uint32_t* mail = reinterpret_cast<volatile uint32_t*>(dsm + 64);   // units handed to the signaller
  char* ring = reinterpret_cast<char*>(dsm) + 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *mail = 0;
  }
  __syncthreads();
  const uint64_t off = (uint64_t)blockIdx.x * bytes;
  const uint32_t np = (uint32_t)(bytes / kPiece);
  const uint32_t nunits = (np + U - 1) / U;
  uint32_t* myflags = flags + (size_t)blockIdx.x * 64;
  if (MODE == 3 && threadIdx.x == 32) {
    // signaller: publish every unit thread 0 reports complete
    uint32_t done = 0;
    while (done < nunits) {
      uint32_t m;
      asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(m) : "r"(sm((const void*)mail)) : "memory");
      while (done < m) {
        publish<SYS>(myflags + (done % 64), done + 1);
        ++done;
      }
    }
    return;
  }
  if (threadIdx.x != 0) return;
  uint32_t ph = 0;
  auto issue = [&](uint32_t i) {
    const int s = i % kStages;
    load(ring + s * kPiece, src + off + (uint64_t)i * kPiece, kPiece, &bar[s]);
  };
  if (MODE == 1) {
    // unit by unit, pipeline restarted per unit
    for (uint32_t u = 0; u < nunits; ++u) {
      const uint32_t a = u * U, b = (a + U < np) ? a + U : np;
      for (uint32_t i = a; i < b && i < a + kStages - 1; ++i) issue(i);
      for (uint32_t i = a; i < b; ++i) {
        const int s = i % kStages;
        wait_bar(&bar[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        store(dst + off + (uint64_t)i * kPiece, ring + s * kPiece, kPiece);
        if (i + kStages - 1 < b) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          issue(i + kStages - 1);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      publish<SYS>(myflags + (u % 64), u + 1);
    }
    return;
  }
  // modes 0, 2, 3: one continuous pipeline over all pieces
  for (uint32_t i = 0; i < np && i < (uint32_t)kStages - 1; ++i) issue(i);
  uint32_t pending = 0;   // units whose stores are issued but not yet published (modes 2, 3)
  for (uint32_t i = 0; i < np; ++i) {
    const int s = i % kStages;
    wait_bar(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    store(dst + off + (uint64_t)i * kPiece, ring + s * kPiece, kPiece);
    if (MODE != 0 && i % U == 0 && i > 0) {
      // first store of unit i / U committed: every older group (unit i / U - 1) is complete
      asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      ++pending;
      if (MODE == 2) publish<SYS>(myflags + ((pending - 1) % 64), pending);
      if (MODE == 3) asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sm((const void*)mail)), "r"(pending) : "memory");
    }
    if (i + kStages - 1 < np) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(i + kStages - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (MODE == 2) publish<SYS>(myflags + (pending % 64), pending + 1);
  if (MODE == 3) asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sm((const void*)mail)), "r"(nunits) : "memory");
}

template <int MODE, bool SYS>
void run(const char* name, int ctas, uint64_t bytes, int U, const char* src, char* dst, uint32_t* flags) {
  const int smem = 128 + kStages * kPiece;
  cudaFuncSetAttribute(stream<MODE, SYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f, sum = 0.f;
  const int reps = 10;
  for (int r = 0; r < reps + 2; ++r) {
    cudaEventRecord(a);
    stream<MODE, SYS><<<ctas, 256, smem>>>(src, dst, flags, bytes, U);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) {
      sum += ms;
      if (ms < best) best = ms;
    }
  }
  const double moved = 2.0 * ctas * (double)bytes;
  printf("{\"mode\": \"%s\", \"scope\": \"%s\", \"ctas\": %d, \"unit_kb\": %d, \"us_mean\": %.1f, \"gbs_mean\": %.1f, \"gbs_best\": %.1f}\n",
         name, SYS ? "sys" : "gpu", ctas, U * (int)kPiece / 1024, sum / reps * 1e3, moved / (sum / reps * 1e-3) / 1e9,
         moved / (best * 1e-3) / 1e9);
  fflush(stdout);
}

int main() {
  const int ctas = 592;
  const uint64_t bytes = 4ull << 20;   // per CTA: 2.48 GB read + 2.48 GB written in total
  char *src, *dst;
  uint32_t* flags;
  cudaMalloc(&src, ctas * bytes);
  cudaMalloc(&dst, ctas * bytes);
  cudaMalloc(&flags, ctas * 64 * 4);
  cudaMemset(src, 1, ctas * bytes);
  for (int U : {8, 2, 32}) {
    run<0, false>("none", ctas, bytes, U, src, dst, flags);
    run<1, false>("drain", ctas, bytes, U, src, dst, flags);
    run<1, true>("drain", ctas, bytes, U, src, dst, flags);
    run<2, false>("defer", ctas, bytes, U, src, dst, flags);
    run<2, true>("defer", ctas, bytes, U, src, dst, flags);
    run<3, false>("signaller", ctas, bytes, U, src, dst, flags);
    run<3, true>("signaller", ctas, bytes, U, src, dst, flags);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
