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
  const CallEpoch ce = call_epoch(P);
  const uint32_t ep = ce.ep;
  if (threadIdx.x < P.world && (int)threadIdx.x != me)
    st_release(flag_at(P.flags[threadIdx.x], SLOT_BARRIER + me, P.fstride, 0), ep, P.sys_scope);
  if (threadIdx.x < P.world && (int)threadIdx.x != me)
    spin_wait(flag_at(P.flags[me], SLOT_BARRIER + threadIdx.x, P.fstride, 0), ep, P, 0x800 | threadIdx.x);
  __syncwarp();
  if (threadIdx.x == 0) P.state->t_barrier = globaltimer();
  finish_call(P, ce);
}

// ---------------------------------------------------------------- K0 probes
// Device-initiated copies to / from peers: the ceiling the NVLink rooflines
// are quoted against.  MV = MOVER_LSU: 16-byte ld/st by every thread
// (copy_vecs); MOVER_TMA: cp.async.bulk through the shared-memory stage ring
// (tma_copy), the data kernels' own mover.
template <int MV>
__global__ void __launch_bounds__(kThreads) k_probe_copy(const __grid_constant__ ProbeArgs A) {
  const int pi = blockIdx.x % A.npeers, part = blockIdx.x / A.npeers;
  const int nparts = gridDim.x / A.npeers;
  const int p = A.peers[pi];
  const uint64_t nv = A.bytes / 16;
  const uint64_t lo = nv * part / nparts * 16, hi = nv * (part + 1) / nparts * 16;
  const char* src = A.pull ? A.peer[p] + (uint64_t)p * A.bytes : A.local + (uint64_t)A.me * A.bytes;
  char* dst = A.pull ? A.local + (uint64_t)p * A.bytes : A.peer[p] + (uint64_t)A.me * A.bytes;
  if constexpr (MV == MOVER_TMA) {
    Pipe pipe = make_pipe(true);
    tma_copy(pipe, dst + lo, src + lo, hi - lo);
  } else {
    copy_vecs(dst + lo, src + lo, (hi - lo) / 16);
  }
}

// Flag ping-pong between this rank and one peer at system scope with the data
// kernels' own signalling (fence.acq_rel.sys + st.relaxed.sys to the peer's
// flag, ld.acquire.sys spin on the own flag): `iters` round trips, timed on
// the device.  The initiator (lower rank) starts each round trip.
__global__ void k_probe_pingpong(uint32_t* mine, uint32_t* theirs, int initiator, int iters, DevState* st,
                                 uint64_t timeout_ns, uint32_t* host_err) {
  if (threadIdx.x != 0) return;
  const uint32_t base = st->probe_seq;
  const uint64_t t0 = globaltimer();
  bool ok = true;
  for (int i = 1; i <= iters && ok; ++i) {
    const uint32_t v = base + (uint32_t)i;
    if (initiator) st_release_sys(theirs, v);
    const uint64_t w0 = globaltimer();
    while (int32_t(ld_acquire_sys(mine) - v) < 0) {
      if (globaltimer() - w0 > timeout_ns) {
        if (atomicCAS(&st->err, 0u, (uint32_t)ERR_TIMEOUT) == 0u) {
          st->err_info = 0xF00;
          if (host_err) *(volatile uint32_t*)host_err = (uint32_t)ERR_TIMEOUT;
        }
        ok = false;
        break;
      }
    }
    if (ok && !initiator) st_release_sys(theirs, v);
  }
  st->probe_ns = globaltimer() - t0;
  st->probe_seq = base + (uint32_t)iters;
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

cudaError_t launch_probe_copy(const ProbeArgs& A, int mover, int nblocks, cudaStream_t stream) {
  if (mover == MOVER_TMA) {
    cudaError_t e = cudaFuncSetAttribute(k_probe_copy<MOVER_TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
    if (e != cudaSuccess) return e;
    k_probe_copy<MOVER_TMA><<<nblocks, kThreads, kTmaSmem, stream>>>(A);
  } else {
    k_probe_copy<MOVER_LSU><<<nblocks, kThreads, 0, stream>>>(A);
  }
  return cudaGetLastError();
}

cudaError_t launch_probe_pingpong(uint32_t* mine, uint32_t* theirs, int initiator, int iters, DevState* st,
                                  uint64_t timeout_ns, uint32_t* host_err, cudaStream_t stream) {
  k_probe_pingpong<<<1, 32, 0, stream>>>(mine, theirs, initiator, iters, st, timeout_ns, host_err);
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
