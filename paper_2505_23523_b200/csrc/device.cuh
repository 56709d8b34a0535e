// Device primitives for the StragglAR kernels (sm_100a): 16-byte vector moves,
// dtype-specific adds, and cross-GPU flag signalling with release/acquire at
// system scope (valid for NVLink peer memory mapped through CUDA IPC and for
// same-device "team" ranks alike).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace stragglar {

enum DType : int { DT_I32 = 0, DT_F32 = 1, DT_BF16 = 2 };

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ uint4 ld_vec(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
#if STRAGGLAR_DIAG_ACQ_GPU
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#else
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#endif
  return v;
}
// Diagnostic A/B knobs (never on in a product build; NOT valid across GPUs):
// STRAGGLAR_DIAG_FENCE_GPU=1 issues the system-scope release fence at GPU
// scope, STRAGGLAR_DIAG_ACQ_GPU=1 the system-scope acquire polls at GPU scope
// -- to find which half of a system-scope hand-off costs (team mode only).
#ifndef STRAGGLAR_DIAG_FENCE_GPU
#define STRAGGLAR_DIAG_FENCE_GPU 0
#endif
#ifndef STRAGGLAR_DIAG_ACQ_GPU
#define STRAGGLAR_DIAG_ACQ_GPU 0
#endif
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
#if STRAGGLAR_DIAG_FENCE_GPU
  asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
// GPU-scope variants: enough when every rank lives on this device (team mode)
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a release fence followed by relaxed flag stores (several flags, one fence)
__device__ __forceinline__ void fence_release(bool sys) {
  if (sys && !STRAGGLAR_DIAG_FENCE_GPU)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_flag(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// scope-selected flag access: sys for CUDA-IPC peers on other GPUs, gpu for one device
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p, bool sys) {
  return sys ? ld_acquire_sys(p) : ld_acquire_gpu(p);
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    st_release_sys(p, v);
  else
    st_release_gpu(p, v);
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16_rn(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // .x (low 16 bits) = lo
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int DT>
__device__ __forceinline__ uint32_t add_word(uint32_t a, uint32_t b) {
  if constexpr (DT == DT_I32) {
    return a + b;  // two's-complement wrap
  } else if constexpr (DT == DT_F32) {
    return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));
  } else {
    return pack_bf16_rn(__fadd_rn(bf_lo(a), bf_lo(b)), __fadd_rn(bf_hi(a), bf_hi(b)));
  }
}
template <int DT>
__device__ __forceinline__ uint4 add_vec(const uint4& a, const uint4& b) {
  return make_uint4(add_word<DT>(a.x, b.x), add_word<DT>(a.y, b.y), add_word<DT>(a.z, b.z), add_word<DT>(a.w, b.w));
}

// Accumulator for the Phase-A reduction: fp32 lanes for float types, u32 for int.
template <int DT>
struct Acc {
  uint32_t u[4];
  float f[8];
  __device__ __forceinline__ void init(const uint4& v) {
    if constexpr (DT == DT_I32) {
      u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
    } else if constexpr (DT == DT_F32) {
      f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
      f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    } else {
      f[0] = bf_lo(v.x); f[1] = bf_hi(v.x); f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
      f[4] = bf_lo(v.z); f[5] = bf_hi(v.z); f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
    }
  }
  __device__ __forceinline__ void add(const uint4& v) {
    if constexpr (DT == DT_I32) {
      u[0] += v.x; u[1] += v.y; u[2] += v.z; u[3] += v.w;
    } else if constexpr (DT == DT_F32) {
      f[0] = __fadd_rn(f[0], __uint_as_float(v.x)); f[1] = __fadd_rn(f[1], __uint_as_float(v.y));
      f[2] = __fadd_rn(f[2], __uint_as_float(v.z)); f[3] = __fadd_rn(f[3], __uint_as_float(v.w));
    } else {
      f[0] = __fadd_rn(f[0], bf_lo(v.x)); f[1] = __fadd_rn(f[1], bf_hi(v.x));
      f[2] = __fadd_rn(f[2], bf_lo(v.y)); f[3] = __fadd_rn(f[3], bf_hi(v.y));
      f[4] = __fadd_rn(f[4], bf_lo(v.z)); f[5] = __fadd_rn(f[5], bf_hi(v.z));
      f[6] = __fadd_rn(f[6], bf_lo(v.w)); f[7] = __fadd_rn(f[7], bf_hi(v.w));
    }
  }
  __device__ __forceinline__ uint4 get() const {
    if constexpr (DT == DT_I32) {
      return make_uint4(u[0], u[1], u[2], u[3]);
    } else if constexpr (DT == DT_F32) {
      return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    } else {
      return make_uint4(pack_bf16_rn(f[0], f[1]), pack_bf16_rn(f[2], f[3]), pack_bf16_rn(f[4], f[5]),
                        pack_bf16_rn(f[6], f[7]));
    }
  }
};

// Scalar versions for the (< 16 byte) tail of the buffer.
template <int DT>
__device__ __forceinline__ void scalar_add_store(void* dst0, void* dst1, const void* a, const void* b) {
  if constexpr (DT == DT_BF16) {
    float s = __fadd_rn(__uint_as_float(uint32_t(*(const volatile uint16_t*)a) << 16),
                        __uint_as_float(uint32_t(*(const volatile uint16_t*)b) << 16));
    __nv_bfloat16 h = __float2bfloat16_rn(s);
    uint16_t bits = *reinterpret_cast<uint16_t*>(&h);
    *(volatile uint16_t*)dst0 = bits;
    if (dst1) *(volatile uint16_t*)dst1 = bits;
  } else {
    uint32_t v = add_word<DT>(*(const volatile uint32_t*)a, *(const volatile uint32_t*)b);
    *(volatile uint32_t*)dst0 = v;
    if (dst1) *(volatile uint32_t*)dst1 = v;
  }
}

}  // namespace stragglar

// ---------------------------------------------------------------- TMA bulk copies (sm_90+ / sm_100a)
// cp.async.bulk moves contiguous 16-byte-aligned byte ranges between global
// memory (local HBM or an NVLink peer mapping) and shared memory in the async
// proxy; completion of loads is tracked by an mbarrier (complete_tx), of
// stores by bulk groups.
namespace stragglar {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// L2 eviction-priority hints on the bulk copies: 0 = none, 1 = evict_first,
// 2 = evict_last (default for both).  Measured at config 2 (DESIGN.md §6b,
// profiles/r01/hint_ab/): evict_last on loads and stores takes Phase B from
// 664-666 to 655 us (forwarded slices stay in L2 for the next hop), the Ring
// -1.6 %, the fused call -0.8 %; evict_first hurts everything.
#ifndef STRAGGLAR_LOAD_HINT
#define STRAGGLAR_LOAD_HINT 2
#endif
#ifndef STRAGGLAR_STORE_HINT
#define STRAGGLAR_STORE_HINT 2
#endif
template <int H>
__device__ __forceinline__ uint64_t l2_policy() {
  uint64_t pol;
  if constexpr (H == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// HINT = false: no cache policy (the direct completion's write-heavy stream, where
// nothing is re-read, measured slightly faster without it).
template <bool HINT = true>
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
#if STRAGGLAR_LOAD_HINT
  if constexpr (HINT) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_policy<STRAGGLAR_LOAD_HINT>())
      : "memory");
  return;
  }
#endif
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
template <bool HINT = true>
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
#if STRAGGLAR_STORE_HINT
  if constexpr (HINT) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(l2_policy<STRAGGLAR_STORE_HINT>())
               : "memory");
  return;
  }
#endif
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
// L2 residency by data lifetime (Phase B, STRAGGLAR_LIFETIME_HINTS=1): a copy
// that is read again later in the call (kernels.cuh, Op::life) keeps the
// default policy above (evict_last); dead data gets STRAGGLAR_DEAD_HINT
// (1 = evict_first, 0 = no hint) so it does not crowd the forwarded slices out.
// Measured with the sub-slice-major order (profiles/r02/ab/r02ac_*): config-2
// Phase B 570 -> 541 us, DRAM reads 1.16 -> 0.62 GB (the floor is 0.54 GB:
// x_sigma and the partials); no hint on dead data: 566 us.
#ifndef STRAGGLAR_LIFETIME_HINTS
#define STRAGGLAR_LIFETIME_HINTS 1
#endif
#ifndef STRAGGLAR_DEAD_HINT
#define STRAGGLAR_DEAD_HINT 1
#endif
__device__ __forceinline__ void bulk_load_life(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                               bool keep) {
#if STRAGGLAR_LIFETIME_HINTS && STRAGGLAR_DEAD_HINT
  if (!keep) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_policy<1>())
        : "memory");
    return;
  }
#elif STRAGGLAR_LIFETIME_HINTS
  if (!keep) {
    bulk_load<false>(smem_dst, gsrc, bytes, bar);
    return;
  }
#endif
  bulk_load<true>(smem_dst, gsrc, bytes, bar);
}
__device__ __forceinline__ void bulk_store_life(void* gdst, const void* smem_src, uint32_t bytes, bool keep) {
#if STRAGGLAR_LIFETIME_HINTS && STRAGGLAR_DEAD_HINT
  if (!keep) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(l2_policy<1>())
                 : "memory");
    return;
  }
#elif STRAGGLAR_LIFETIME_HINTS
  if (!keep) {
    bulk_store<false>(gdst, smem_src, bytes);
    return;
  }
#endif
  bulk_store<true>(gdst, smem_src, bytes);
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

}  // namespace stragglar
