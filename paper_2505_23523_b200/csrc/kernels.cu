// StragglAR host-side launchers and the non-templated kernels (delay, barrier).
// The method's kernel templates live in kernels.cuh; their per-dtype
// instantiations in kernels_{i32,f32,bf16}.cu.
#include "kernels.cuh"

namespace stragglar {

// ---------------------------------------------------------------- delay / barrier
// Spin until base + ns, base = *base_ptr if given (team: start of Phase A),
// else this kernel's own start (P:405-407 idle kernel; %globaltimer is
// independent of the SM clock).
__global__ void k_delay(const uint64_t* base_ptr, uint64_t ns, DevState* st) {
  uint64_t base = base_ptr ? *(volatile const uint64_t*)base_ptr : globaltimer();
  const uint64_t until = base + ns;
  uint64_t now;
  while ((now = globaltimer()) < until) {
    uint64_t left = until - now;
    __nanosleep(left > 2000 ? 1000 : 64);
  }
  st->t_release = globaltimer();
}

__global__ void k_barrier(const __grid_constant__ LaunchPlan P) {
  const int me = P.local_rank[0];
  const uint32_t ep = call_epoch(P);
  if (threadIdx.x < P.world && (int)threadIdx.x != me)
    st_release(flag_at(P.flags[threadIdx.x], SLOT_BARRIER + me, P.fstride, 0), ep, P.sys_scope);
  if (threadIdx.x < P.world && (int)threadIdx.x != me)
    spin_wait(flag_at(P.flags[me], SLOT_BARRIER + threadIdx.x, P.fstride, 0), ep, P, 0x800 | threadIdx.x);
  finish_call(P);
}

// ---------------------------------------------------------------- host launchers
void* select_kernel(int which, int dtype, int world, int mover) {
  switch (dtype) {
    case DT_I32: return select_kernel_i32(which, world, mover);
    case DT_F32: return select_kernel_f32(which, world, mover);
    case DT_BF16: return select_kernel_bf16(which, world, mover);
    default: return nullptr;
  }
}

int dynamic_smem(int which, int mover) { return (which <= 9 && mover == MOVER_TMA) ? kTmaSmem : 0; }

cudaError_t launch_plan_kernel(int which, int dtype, const LaunchPlan& P, int nblocks, cudaStream_t stream) {
  void* fn = select_kernel(which, dtype, P.world, P.mover);
  if (!fn) return cudaErrorInvalidValue;
  void* args[] = {(void*)&P};
  // cudaLaunchKernelEx with the cooperative attribute: co-residency of every
  // CTA is guaranteed (they spin on each other's flags) and the launch can be
  // captured into a CUDA graph.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = dynamic_smem(which, P.mover);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_delay(const uint64_t* base_ptr, uint64_t ns, DevState* st, cudaStream_t stream) {
  k_delay<<<1, 1, 0, stream>>>(base_ptr, ns, st);
  return cudaGetLastError();
}

cudaError_t launch_barrier(const LaunchPlan& P, cudaStream_t stream) {
  k_barrier<<<1, 32, 0, stream>>>(P);
  return cudaGetLastError();
}

cudaError_t occupancy_blocks_per_sm(int which, int dtype, int world, int mover, int* blocks) {
  void* fn = select_kernel(which, dtype, world, mover);
  if (!fn) return cudaErrorInvalidValue;
  const int smem = dynamic_smem(which, mover);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, kThreads, smem);
}

}  // namespace stragglar
