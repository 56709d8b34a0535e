// NEXT row N1(i): StragglAR with NVLink SHARP (NVLS).
//
// The paper's schedule assumes a single-port fabric ("a GPU can only
// send data to one other GPU").  An NVSwitch fabric can also reduce and
// replicate inside the switch: a load through a multicast address returns the
// sum of every member GPU's copy (multimem.ld_reduce), a store through it
// writes every member's copy (multimem.st).  With the same two phases:
//   Phase A (during the straggler's delay): owner g of chunk c_g loads c_g
//     through the non-stragglers' multicast object — the switch sums the n-1
//     non-straggler copies — and keeps the partial in its own arena
//     (owner ingress C instead of (n-2)C, P:202's ReduceScatter result);
//   completion (once the straggler arrived): owner g adds x_sigma[c_g] (one
//     unicast peer load, the exchange's single add) and stores the
//     fully reduced chunk through the all-rank multicast object: every rank's
//     copy of c_g is written by one store (owner egress C).
// Numerics reading (reading 24): the switch adds the n-1
// non-straggler values in an order the hardware does not specify (fp32
// accumulation; bf16 through .acc::f32 and one rounding), then the straggler's
// value is added once — int32 results are exact, float results match the
// canonical oracle within the north_star tolerance, not bit for bit.
//
// The arenas are library memory (VMM physical allocations bound to the
// multicast objects; api.cu stragglar_nvls_*).  Flags are the communicator's
// IPC-mapped flag arrays, epochs as everywhere else.
#include "kernels.cuh"

namespace stragglar {

template <int DT>
__device__ __forceinline__ uint4 mm_ld_reduce(const void* mc) {
  uint4 v;
  if constexpr (DT == DT_F32) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  } else if constexpr (DT == DT_BF16) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  } else {
    const uint32_t* p = static_cast<const uint32_t*>(mc);
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.x) : "l"(p) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.y) : "l"(p + 1) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.z) : "l"(p + 2) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.w) : "l"(p + 3) : "memory");
  }
  return v;
}

__device__ __forceinline__ void mm_st(void* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// One launch per rank (G CTAs): Phase A through the switch, then the completion.
// P.buf[me] = this rank's arena (+ call offset), P.mc_ns / P.mc_all = the two
// multicast mappings, P.sigma_uc = the straggler's arena (unicast peer mapping).
// count must be a multiple of 16 bytes' worth of elements (host-checked).
//
// EMU (test only, stragglar_allreduce_nvls_emulated): the same kernel — flags,
// epochs, arrivals, slices, hand-offs — with the two multicast operations
// replaced by what they do, through IPC peer pointers (P.buf[p], registered
// cudaMalloc buffers): the reducing load becomes the canonical non-straggler
// sum (ascending rank, fp32 accumulation, so the result is bit-exact to the
// oracle) and the multicast store one store per rank.  It validates the
// variant's synchronisation where no multicast object can be created (one GPU).
template <int DT, int W, bool EMU>
__global__ void __launch_bounds__(kThreads) k_nvls(const __grid_constant__ LaunchPlan P) {
  const int me = P.local_rank[0], s = blockIdx.x;
  const CallEpoch ce = call_epoch(P);
  const uint32_t ep = ce.ep;
  const int V = 16 / P.esize;
  uint64_t* stamp = P.state->stamp[ep & 1u];
  if (threadIdx.x == 0) atomicMin(reinterpret_cast<unsigned long long*>(&stamp[0]), (unsigned long long)globaltimer());
  // arrival: this rank's arena holds the call's input (every rank tells every other)
  if (threadIdx.x < W && (int)threadIdx.x != me)
    st_release(flag_at(P.flags[threadIdx.x], SLOT_ARRIVE + me, P.fstride, s), ep, true);
  bool ok = true;
  int own = -1;
  if (me != P.sigma) {
    own = P.logical_of_phys[me];
    // barrier (1) among the non-stragglers: every member's input must be in place
    int k = 1;
    if (threadIdx.x < W && (int)threadIdx.x != me && (int)threadIdx.x != P.sigma)
      k = spin_wait(flag_at(P.flags[me], SLOT_ARRIVE + threadIdx.x, P.fstride, s), ep, P, 0x1100 | threadIdx.x, true);
    ok = __syncthreads_and(k);
    const Range cr = chunk_range(P, own);
    const Range sl = slice_of(cr.lo, cr.hi, s, P.G, V);
    const uint64_t a = sl.lo * P.esize, nv = (sl.hi - sl.lo) / V;
    if (ok) {
      // Phase A in the switch: partial of the slice = sum over the non-stragglers' copies
      if constexpr (EMU) {
        const char* src[W - 1];
#pragma unroll
        for (int j = 0; j < W - 1; ++j) src[j] = P.buf[j < P.sigma ? j : j + 1];
        if constexpr (W > 2) rs_slice<DT, W>(P, src, P.buf[me], a, a + nv * 16);
      } else {
        for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x)
          st_vec(P.buf[me] + a + i * 16, mm_ld_reduce<DT>(P.mc_ns + a + i * 16));
      }
      __syncthreads();
      if (threadIdx.x == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(&stamp[1]), (unsigned long long)globaltimer());
      // the straggler arrived (barrier (2)): its input x_sigma is readable
      ok = cta_wait(flag_at(P.flags[me], SLOT_ARRIVE + P.sigma, P.fstride, s), ep, P, 0x1200);
    }
    if (ok) {
      // completion: full = partial (+) x_sigma, one multicast store to every rank's arena
      for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        if constexpr (EMU) {
          const uint4 z = add_vec<DT>(ld_vec(P.buf[me] + a + i * 16), ld_vec(P.buf[P.sigma] + a + i * 16));
#pragma unroll
          for (int d = 0; d < W; ++d) st_vec(P.buf[d] + a + i * 16, z);
        } else {
          const uint4 z = add_vec<DT>(ld_vec(P.buf[me] + a + i * 16), ld_vec(P.sigma_uc + a + i * 16));
          mm_st(P.mc_all + a + i * 16, z);
        }
      }
      __syncthreads();
      // hand-off: the multicast stores happen-before every rank's HAVE flag
      if (threadIdx.x < W && (int)threadIdx.x != me)
        st_release(flag_at(P.flags[threadIdx.x], SLOT_HAVE + own, P.fstride, s), ep, true);
    }
  }
  // postcondition: every other owner's slice has landed here
  if (ok && (int)threadIdx.x < P.nchunks && (int)threadIdx.x != own)
    spin_wait(flag_at(P.flags[me], SLOT_HAVE + threadIdx.x, P.fstride, s), ep, P, 0x1300 | threadIdx.x, true);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(&stamp[2]), (unsigned long long)globaltimer());
  finish_call(P, ce);
}

cudaError_t launch_nvls(int dtype, const LaunchPlan& P, int nblocks, cudaStream_t stream, bool emulated) {
  void* fn = nullptr;
#define STRAGGLAR_NVLS_CASE(DTV, WV) \
  if (dtype == DTV && P.world == WV) fn = emulated ? (void*)k_nvls<DTV, WV, true> : (void*)k_nvls<DTV, WV, false>;
  STRAGGLAR_NVLS_CASE(DT_I32, 2) STRAGGLAR_NVLS_CASE(DT_I32, 4) STRAGGLAR_NVLS_CASE(DT_I32, 6) STRAGGLAR_NVLS_CASE(DT_I32, 8)
  STRAGGLAR_NVLS_CASE(DT_F32, 2) STRAGGLAR_NVLS_CASE(DT_F32, 4) STRAGGLAR_NVLS_CASE(DT_F32, 6) STRAGGLAR_NVLS_CASE(DT_F32, 8)
  STRAGGLAR_NVLS_CASE(DT_BF16, 2) STRAGGLAR_NVLS_CASE(DT_BF16, 4) STRAGGLAR_NVLS_CASE(DT_BF16, 6)
  STRAGGLAR_NVLS_CASE(DT_BF16, 8)
#undef STRAGGLAR_NVLS_CASE
  if (!fn) return cudaErrorInvalidValue;
  void* args[] = {(void*)&P};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// One-GPU self-test of the multicast instructions: a multicast object with a
// single member, so a reducing load returns the member's own value and a
// multicast store writes it back.  in -> out through mc (both through the
// multicast mapping of one buffer: out = buffer + bytes).
template <int DT>
__global__ void k_nvls_selftest(char* mc, uint64_t bytes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < bytes / 16; i += (uint64_t)gridDim.x * blockDim.x)
    mm_st(mc + bytes + i * 16, mm_ld_reduce<DT>(mc + i * 16));
}

cudaError_t launch_nvls_selftest(int dtype, char* mc, uint64_t bytes, cudaStream_t stream) {
  if (dtype == DT_F32)
    k_nvls_selftest<DT_F32><<<148, 256, 0, stream>>>(mc, bytes);
  else if (dtype == DT_BF16)
    k_nvls_selftest<DT_BF16><<<148, 256, 0, stream>>>(mc, bytes);
  else
    k_nvls_selftest<DT_I32><<<148, 256, 0, stream>>>(mc, bytes);
  return cudaGetLastError();
}

}  // namespace stragglar
