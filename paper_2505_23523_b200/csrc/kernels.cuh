// StragglAR kernels for sm_100a.
//
//   k_phase<..., KIND> one persistent kernel template for the method:
//     KIND 0  Phase A: owner g pulls its chunk from the
//             n-2 other non-stragglers, sums in canonical order (ascending
//             physical rank, fp32 accumulation), stores in place.  Replaces
//             ncclReduceScatter.                      [rs_body]
//     KIND 1  Phase B (Algorithm 1): round executor; each CTA owns
//             one slice of every chunk and walks its rank's op list in round
//             order; the straggler exchange is fused with its
//             reduction (P:347's separate reduction kernels become one pass).
//                                                              [complete_body]
//     KIND 3  Phase B as a one-round direct completion (NEXT N1(ii)). [direct_body]
//     KIND 4  Phase A then Phase B (schedule) in one launch (single-call API).
//     KIND 5  Phase A then direct completion in one launch.
//     KIND 6-8 the straggler-aware Broadcast baseline (NEXT N3).
//   k_ring            hand-written Ring baseline, pull-based.
//   k_rhd             recursive halving/doubling baseline (NEXT N3).
//   k_delay           the paper's idle kernel on %globaltimer.
//   k_barrier         device barrier among ranks (bench start line).
//
// One launch serves `nlocal` ranks: 1 in the per-process (NVLink) mode, all
// of them in the single-device team mode (block b works for local rank b/G,
// slice b%G).  All CTAs of a launch must be co-resident (cooperative launch),
// because they spin on flags produced by CTAs of other ranks.
#pragma once
#include "device.cuh"
#include "plan.h"

namespace stragglar {

// ---------------------------------------------------------------- flags
__device__ __forceinline__ bool flag_ok(uint32_t v, uint32_t epoch) { return int32_t(v - epoch) >= 0; }

// Spin (one thread) until *f >= epoch.  Bounded by the watchdog; gives up
// early if another CTA of this process already reported an error.
static __device__ bool spin_wait(const uint32_t* f, uint32_t epoch, const LaunchPlan& P, uint32_t where,
                                 bool sys) {
  if (flag_ok(ld_acquire(f, sys), epoch)) return true;
  const uint64_t t0 = globaltimer();
  for (uint32_t it = 1;; ++it) {
    if (flag_ok(ld_acquire(f, sys), epoch)) return true;
    if (it > 2048) __nanosleep(32);
    if ((it & 127) == 0) {
      if (*(volatile uint32_t*)&P.state->err) return false;
      if (globaltimer() - t0 > P.timeout_ns) {
        if (atomicCAS(&P.state->err, 0u, (uint32_t)ERR_TIMEOUT) == 0u) {
          atomicExch(&P.state->err_info, where);
          if (P.host_err) *(volatile uint32_t*)P.host_err = (uint32_t)ERR_TIMEOUT;   // sticky, seen by the host API
        }
        return false;
      }
    }
  }
}

// Flags written by other ranks need the communicator's scope (system scope
// across GPUs); flags a rank writes for its own CTAs (SLOT_SELF,
// SLOT_RS_LOCAL) only need GPU scope.
__device__ __forceinline__ bool spin_wait(const uint32_t* f, uint32_t epoch, const LaunchPlan& P, uint32_t where) {
  return spin_wait(f, epoch, P, where, P.sys_scope != 0);
}

// Whole-CTA wait: thread 0 spins, the barrier publishes the acquired state.
__device__ __forceinline__ bool cta_wait(const uint32_t* f, uint32_t epoch, const LaunchPlan& P, uint32_t where,
                                         bool local = false) {
  int ok = 1;
  if (threadIdx.x == 0) ok = spin_wait(f, epoch, P, where, local ? false : P.sys_scope != 0);
  return __syncthreads_and(ok);
}

// Whole-CTA signal: all prior stores of the CTA happen-before the flag store
// (the barrier orders every thread's stores — thread 0's completed bulk stores
// included — before the release fence, which is cumulative).  Issuing the
// release from a thread of warp 1, so that it overlaps thread 0's poll of the
// next flag, measured no different (profiles/r02/ab/r02g_sig*); thread 0 it is.
constexpr int kSignalThread = 0;
__device__ __forceinline__ void cta_signal(uint32_t* f, uint32_t epoch, bool sys) {
  __syncthreads();
  if (threadIdx.x == kSignalThread) st_release(f, epoch, sys);
}

// Signalling warp (Phase B, STRAGGLAR_SIGNALLER): at system scope a unit's
// release fence costs thread 0 ~2 us (profiles/r02/ab/r02aj_trace_*: a CTA's
// units move 343 us at system scope vs 270 us at GPU scope, waits unchanged).
// With the signaller, warp 1 leaves the CTA's barriers for the whole of
// complete_body and only publishes flags: thread 0 completes a unit's stores,
// posts the flag to a shared-memory queue (st.release.cta) and goes on; warp 1's
// lane 0 takes it (ld.acquire.cta), issues the system-scope fence and stores
// the flag.  Cumulativity carries thread 0's completed stores to the waiter.
// The other 7 warps synchronise on named barrier 1.
// Measured (profiles/r02/ab/r02ak_*, two repetitions): config-2 Phase B 512 -> 493 us
// (GPU scope), 526-528 -> 502-508 us (system scope), 1 GiB bf16 at system scope
// 2125-2133 -> 1918-1930 us; MPS n = 8 654 -> 648 us.
#ifndef STRAGGLAR_SIGNALLER
#define STRAGGLAR_SIGNALLER 1
#endif
constexpr int kGrp = kThreads - 32;     // threads of the CTA without warp 1
constexpr int kSigQ = 64;               // queue entries (thread 0 waits if it is full)
constexpr uint32_t kSigDone = 0xffffffffu;
__device__ __forceinline__ int grp_tid() { return threadIdx.x < 32 ? (int)threadIdx.x : (int)threadIdx.x - 32; }
__device__ __forceinline__ void grp_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kGrp) : "memory"); }
__device__ __forceinline__ int grp_sync_and(int pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred a, b;\n\tsetp.ne.s32 a, %1, 0;\n\tbar.red.and.pred b, 1, %2, a;\n\tselp.s32 %0, 1, 0, b;\n}"
      : "=r"(r)
      : "r"(pred), "n"(kGrp)
      : "memory");
  return r;
}
struct SigQ {
  uint32_t head, tail;   // entries posted by thread 0 / published by the signaller
  uint32_t e[kSigQ];     // (peer << 24) | flag index in the peer's array
};
__device__ __forceinline__ uint32_t ld_acquire_cta_smem(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_smem(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// thread 0: queue the flag (its unit's stores have completed: wait_group 0)
__device__ __forceinline__ void sig_post(SigQ& q, uint32_t entry) {
  const uint32_t h = q.head;
  while (h - ld_acquire_cta_smem(&q.tail) >= (uint32_t)kSigQ) {
  }
  q.e[h % kSigQ] = entry;
  st_release_cta_smem(&q.head, h + 1);
}
// warp 1, lane 0: publish every queued flag until kSigDone
__device__ __forceinline__ void sig_loop(SigQ& q, const LaunchPlan& P, uint32_t ep) {
  uint32_t t = 0;
  for (;;) {
    const uint32_t h = ld_acquire_cta_smem(&q.head);
    for (; t < h; ++t) {
      const uint32_t e = q.e[t % kSigQ];
      if (e == kSigDone) return;
      fence_release(P.sys_scope != 0);
      st_flag(P.flags[e >> 24] + (e & 0xffffffu), ep, P.sys_scope != 0);
      st_release_cta_smem(&q.tail, t + 1);
    }
  }
}
// group versions of cta_wait / cta_wait_range (warp 1 excluded)
__device__ __forceinline__ bool grp_wait(const uint32_t* f, uint32_t epoch, const LaunchPlan& P, uint32_t where,
                                         bool local = false) {
  int ok = 1;
  if (threadIdx.x == 0) ok = spin_wait(f, epoch, P, where, local ? false : P.sys_scope != 0);
  return grp_sync_and(ok);
}

// The call's epoch lives in device memory (state->epoch + 1), so a captured
// CUDA graph replays correctly.  It is incremented once every CTA of the
// call's final kernel has read it: thread 0 of each CTA takes a ticket from a
// counter right after its acquire read of the epoch (at kernel start), without
// waiting for the ticket; the CTA that drew the last ticket bumps the epoch and
// re-arms the next call's phase stamps when it finishes (finish_call).  The
// same-address atomics thus overlap the call's work instead of queueing on
// its tail (config 5: 22.3 -> 20.7 us vs counting CTAs at exit).
// Every thread of the CTA must call call_epoch (it has a CTA barrier).
__device__ __forceinline__ void bump_epoch(const LaunchPlan& P, uint32_t e) {
  P.state->exit_count = 0;
  uint64_t* nx = P.state->stamp[(e + 1u) & 1u];   // re-arm for the next call
  nx[0] = ~0ull;
  nx[1] = 0;
  nx[2] = 0;
  __threadfence();
  atomicAdd(&P.state->epoch, 1u);
}
struct CallEpoch {
  uint32_t ep;       // this call's epoch
  uint32_t ticket;   // thread 0: counter value drawn at start (final kernel only)
};
__device__ __forceinline__ CallEpoch call_epoch(const LaunchPlan& P) {
  __shared__ uint32_t s_ep;
  CallEpoch c{0u, 0u};
  if (threadIdx.x == 0) {
    const uint32_t e = ld_acquire_gpu(&P.state->epoch) + 1u;
    s_ep = e;
    if (P.last_kernel) c.ticket = atomicAdd(&P.state->exit_count, 1u);
  }
  __syncthreads();
  c.ep = s_ep;
  return c;
}
__device__ __forceinline__ void finish_call(const LaunchPlan& P, const CallEpoch& c) {
  if (P.last_kernel && threadIdx.x == 0 && c.ticket == gridDim.x - 1) bump_epoch(P, c.ep);
}

// Slot k of a rank's flag array spans [k * stride, (k+1) * stride) with a
// stride fixed per communicator (LaunchPlan::fstride = G_max * kMaxSub), not
// per call: a fast peer's writes for its NEXT call (a different slice layout)
// then land in the same slot as in this call, never in another slot's range.
__device__ __forceinline__ uint32_t* flag_at(uint32_t* base, int slot, int stride, int s) {
  return base + (size_t)slot * stride + s;
}

// Whole-CTA wait for `n` consecutive flags of one slot (one waiting thread each).
__device__ __forceinline__ bool cta_wait_range(uint32_t* base, int slot, int first, int n, uint32_t epoch,
                                               const LaunchPlan& P, uint32_t where, bool local = false) {
  int ok = 1;
  if ((int)threadIdx.x < n)
    ok = spin_wait(flag_at(base, slot, P.fstride, first + threadIdx.x), epoch, P, where, local ? false : P.sys_scope != 0);
  return __syncthreads_and(ok);
}

// ---------------------------------------------------------------- ranges
struct Range {
  uint64_t lo, hi;  // elements
};

// Slice s of [clo, chi): an even split of the 16-byte vectors; identical on
// every rank (it depends only on count, world and G).
__device__ __forceinline__ Range slice_of(uint64_t clo, uint64_t chi, int s, int G, int V) {
  const uint64_t nv = (chi - clo + V - 1) / V;
  const uint64_t a = nv * (uint64_t)s / G, b = nv * (uint64_t)(s + 1) / G;
  Range r;
  r.lo = clo + a * V;
  r.hi = clo + b * V < chi ? clo + b * V : chi;
  if (r.lo > r.hi) r.lo = r.hi;
  return r;
}

__device__ __forceinline__ Range chunk_range(const LaunchPlan& P, int c) {
  uint64_t lo = (uint64_t)c * P.ce, hi = lo + P.ce;
  if (lo > P.count) lo = P.count;
  if (hi > P.count) hi = P.count;
  return {lo, hi};
}

// ---------------------------------------------------------------- data movers
constexpr int kUnroll = 8;
#ifndef STRAGGLAR_MIN_BLOCKS
#define STRAGGLAR_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = STRAGGLAR_MIN_BLOCKS;  // 4 x 256 threads: <= 64 registers

// dst <- src for 16-byte vectors [0, nv)
__device__ __forceinline__ void copy_vecs(char* __restrict__ dst, const char* __restrict__ src, uint64_t nv) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  uint64_t i = threadIdx.x;
  const uint64_t step = (uint64_t)kUnroll * blockDim.x;
  for (; i + (kUnroll - 1) * blockDim.x < nv; i += step) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_vec(s + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_vec(d + i + u * blockDim.x, v[u]);
  }
  for (; i < nv; i += blockDim.x) st_vec(d + i, ld_vec(s + i));
}

// d0 = d1 = a (+) b for 16-byte vectors [0, nv)  (fused exchange-reduce)
template <int DT>
__device__ __forceinline__ void add2_vecs(char* d0, char* d1, const char* a, const char* b, uint64_t nv) {
  const uint4* pa = reinterpret_cast<const uint4*>(a);
  const uint4* pb = reinterpret_cast<const uint4*>(b);
  uint4* q0 = reinterpret_cast<uint4*>(d0);
  uint4* q1 = reinterpret_cast<uint4*>(d1);
  uint64_t i = threadIdx.x;
  constexpr int U = 4;
  const uint64_t step = (uint64_t)U * blockDim.x;
  for (; i + (U - 1) * blockDim.x < nv; i += step) {
    uint4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      va[u] = ld_vec(pa + i + u * blockDim.x);
      vb[u] = ld_vec(pb + i + u * blockDim.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 z = add_vec<DT>(va[u], vb[u]);
      st_vec(q0 + i + u * blockDim.x, z);
      if (q1) st_vec(q1 + i + u * blockDim.x, z);
    }
  }
  for (; i < nv; i += blockDim.x) {
    uint4 z = add_vec<DT>(ld_vec(pa + i), ld_vec(pb + i));
    st_vec(q0 + i, z);
    if (q1) st_vec(q1 + i, z);
  }
}

// elementwise tail (< 16 bytes) of an add2
template <int DT>
__device__ __forceinline__ void add2_tail(char* d0, char* d1, const char* a, const char* b, int nelem, int esz) {
  if ((int)threadIdx.x < nelem) {
    const int o = threadIdx.x * esz;
    scalar_add_store<DT>(d0 + o, d1 ? d1 + o : nullptr, a + o, b + o);
  }
}

__device__ __forceinline__ void copy_tail(char* dst, const char* src, int nbytes) {
  if ((int)threadIdx.x < nbytes) dst[threadIdx.x] = *(const volatile char*)(src + threadIdx.x);
}

// ---------------------------------------------------------------- TMA movers (cp.async.bulk)
// A ring of kStages shared-memory stages per CTA.  Thread 0 issues bulk loads
// (mbarrier complete_tx) kStages pieces ahead and bulk stores (bulk groups);
// for the fused exchange every thread adds the two staged operands in shared
// memory before the stores.  All threads track the per-stage mbarrier parity
// identically, so the ring persists across the ops of a kernel.
// 5 x 11 KB (round 2, with the sub-slice-major order and lifetime hints; 4 CTAs
// per SM still fit): config-2 Phase B 540 -> 513 us, 1 GiB bf16 2158 -> 2037 us
// vs 3 x 16 KB (profiles/r02/ab/r02ae_*).  Phase A keeps larger stages (kRsStages).
#ifndef STRAGGLAR_STAGES
#define STRAGGLAR_STAGES 5
#endif
#ifndef STRAGGLAR_STAGE_BYTES
#define STRAGGLAR_STAGE_BYTES 11264
#endif
constexpr int kStages = STRAGGLAR_STAGES;
// Refill lag: 1 = a stage is refilled one iteration after its stores were
// issued (wait_group.read 1: the newest piece's stores may still be reading
// shared memory while the next piece is computed); 0 = refill right after
// the stores (wait_group.read 0, serialises store reads with compute).
#ifndef STRAGGLAR_TMA_LAG
#define STRAGGLAR_TMA_LAG 1
#endif
constexpr int kAhead = kStages - STRAGGLAR_TMA_LAG;   // pieces loaded ahead

__device__ __forceinline__ void ring_release_wait() {
#if STRAGGLAR_TMA_LAG
  bulk_wait_read_1();
#else
  bulk_wait_read_all();
#endif
}
constexpr uint32_t kStageBytes = STRAGGLAR_STAGE_BYTES;
constexpr int kTmaSmem = 128 + kStages * kStageBytes;

struct Pipe {
  uint64_t* bar;
  char* stage;
  uint32_t phase;  // bit s = parity to wait for on stage s
  __device__ __forceinline__ char* buf(int s) const { return stage + (size_t)s * kStageBytes; }
};

// Shared-memory stage ring of the CTA (dynamic smem); mbarriers initialised once per launch.
__device__ __forceinline__ Pipe make_pipe(bool active) {
  extern __shared__ __align__(128) unsigned char dsm[];
  Pipe p{reinterpret_cast<uint64_t*>(dsm), reinterpret_cast<char*>(dsm) + 128, 0u};
  if (active) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < kStages; ++st) mbar_init(&p.bar[st], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  return p;
}

__device__ __forceinline__ uint32_t advance_phase(uint32_t ph, uint32_t np) {
#pragma unroll
  for (int s = 0; s < kStages; ++s) {
    const uint32_t uses = np / kStages + ((uint32_t)s < np % kStages ? 1u : 0u);
    if (uses & 1u) ph ^= 1u << s;
  }
  return ph;
}

// dst <- src, nbytes a multiple of 16.  ld_keep / st_keep: the source / the
// destination copy is read again later (L2 hints, STRAGGLAR_LIFETIME_HINTS).
static __device__ void tma_copy(Pipe& p, char* dst, const char* src, uint64_t nbytes, bool ld_keep = true,
                                bool st_keep = true) {
  const uint32_t np = (uint32_t)((nbytes + kStageBytes - 1) / kStageBytes);
  if (threadIdx.x == 0 && np) {
    fence_proxy_async_global();
    auto issue = [&](uint32_t i) {
      const int s = i % kStages;
      const uint64_t off = (uint64_t)i * kStageBytes;
      const uint32_t len = (uint32_t)((nbytes - off) < kStageBytes ? (nbytes - off) : kStageBytes);
      mbar_expect_tx(&p.bar[s], len);
      bulk_load_life(p.buf(s), src + off, len, &p.bar[s], ld_keep);
    };
    for (uint32_t i = 0; i < np && i < (uint32_t)kAhead; ++i) issue(i);
    uint32_t ph = p.phase;
    for (uint32_t i = 0; i < np; ++i) {
      const int s = i % kStages;
      mbar_wait(&p.bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      const uint64_t off = (uint64_t)i * kStageBytes;
      const uint32_t len = (uint32_t)((nbytes - off) < kStageBytes ? (nbytes - off) : kStageBytes);
      bulk_store_life(dst + off, p.buf(s), len, st_keep);
      bulk_commit();
      if (i + kAhead < np) {
        ring_release_wait();
        issue(i + kAhead);
      }
    }
    bulk_wait_all();
    fence_proxy_async_global();
  }
  p.phase = advance_phase(p.phase, np);
}

// d0 = d1 = a (+) b through shared memory, nbytes a multiple of 16
template <int DT, bool GRP = false>   // GRP: run by the CTA without warp 1 (signalling warp)
__device__ void tma_add2(Pipe& p, char* d0, char* d1, const char* a, const char* b, uint64_t nbytes,
                         bool ld_keep = true, bool st0_keep = true, bool st1_keep = true) {
  constexpr uint32_t kPiece = kStageBytes / 2;
  const uint32_t np = (uint32_t)((nbytes + kPiece - 1) / kPiece);
  auto piece_len = [&](uint32_t i) -> uint32_t {
    const uint64_t off = (uint64_t)i * kPiece;
    return (uint32_t)((nbytes - off) < kPiece ? (nbytes - off) : kPiece);
  };
  auto issue = [&](uint32_t i) {
    const int s = i % kStages;
    const uint64_t off = (uint64_t)i * kPiece;
    const uint32_t len = piece_len(i);
    mbar_expect_tx(&p.bar[s], 2 * len);
    bulk_load_life(p.buf(s), a + off, len, &p.bar[s], ld_keep);
    bulk_load_life(p.buf(s) + kPiece, b + off, len, &p.bar[s], ld_keep);
  };
  if (threadIdx.x == 0 && np) {
    fence_proxy_async_global();
    for (uint32_t i = 0; i < np && i < (uint32_t)kAhead; ++i) issue(i);
  }
  uint32_t ph = p.phase;
  for (uint32_t i = 0; i < np; ++i) {
    const int s = i % kStages;
    const uint32_t len = piece_len(i);
    mbar_wait(&p.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    uint4* A = reinterpret_cast<uint4*>(p.buf(s));
    const uint4* B = reinterpret_cast<const uint4*>(p.buf(s) + kPiece);
    if constexpr (GRP) {
      for (uint32_t v = grp_tid(); v < len / 16; v += kGrp) A[v] = add_vec<DT>(A[v], B[v]);
      fence_proxy_async_smem();
      grp_sync();
    } else {
      for (uint32_t v = threadIdx.x; v < len / 16; v += blockDim.x) A[v] = add_vec<DT>(A[v], B[v]);
      fence_proxy_async_smem();
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const uint64_t off = (uint64_t)i * kPiece;
      bulk_store_life(d0 + off, A, len, st0_keep);
      if (d1) bulk_store_life(d1 + off, A, len, st1_keep);
      bulk_commit();
      if (i + kAhead < np) {
        ring_release_wait();
        issue(i + kAhead);
      }
    }
  }
  if (threadIdx.x == 0 && np) {
    bulk_wait_all();
    fence_proxy_async_global();
  }
  p.phase = ph;
}

// Phase A through shared memory: per stage, the W-1 non-straggler operands of
// one piece (ascending physical order) are bulk-loaded, summed by the CTA in
// canonical order into operand slot 0, and bulk-stored to the owner.
// Phase A cuts the same shared memory into its own, fewer and larger stages
// (STRAGGLAR_RS_STAGES, barriers 0.. of the ring): a stage holds W-1 operand
// pieces, and the many small stages that suit the copies (5 x 11 KB) leave it
// ~1.6 KB per operand (measured: 342 -> 370 us at config 2).  The ring is
// empty between ops, and each barrier's phase bit is tracked per use, so the
// two geometries share it.
#ifndef STRAGGLAR_RS_STAGES
#define STRAGGLAR_RS_STAGES 3
#endif
constexpr int kRsStages = STRAGGLAR_RS_STAGES < kStages ? STRAGGLAR_RS_STAGES : kStages;
constexpr uint32_t kRsStageBytes = (kStages * kStageBytes / kRsStages) / 16 * 16;
constexpr int kRsAhead = kRsStages - STRAGGLAR_TMA_LAG;
template <int DT, int W>
__device__ void tma_reduce(Pipe& p, char* dst, const char* const (&src)[W - 1], uint64_t lo_b, uint64_t nbytes) {
  constexpr uint32_t kPiece = (kRsStageBytes / (W - 1)) / 16 * 16;
  auto sbuf = [&](int s) { return p.stage + (size_t)s * kRsStageBytes; };
  const uint32_t np = (uint32_t)((nbytes + kPiece - 1) / kPiece);
  auto piece_len = [&](uint32_t i) -> uint32_t {
    const uint64_t off = (uint64_t)i * kPiece;
    return (uint32_t)((nbytes - off) < kPiece ? (nbytes - off) : kPiece);
  };
  auto issue = [&](uint32_t i) {
    const int s = i % kRsStages;
    const uint64_t off = lo_b + (uint64_t)i * kPiece;
    const uint32_t len = piece_len(i);
    mbar_expect_tx(&p.bar[s], (W - 1) * len);
#pragma unroll
    for (int j = 0; j < W - 1; ++j) bulk_load<false>(sbuf(s) + j * kPiece, src[j] + off, len, &p.bar[s]);
  };
  if (threadIdx.x == 0 && np) {
    fence_proxy_async_global();
    for (uint32_t i = 0; i < np && i < (uint32_t)kRsAhead; ++i) issue(i);
  }
  uint32_t ph = p.phase;
  for (uint32_t i = 0; i < np; ++i) {
    const int s = i % kRsStages;
    const uint32_t len = piece_len(i);
    mbar_wait(&p.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    char* base = sbuf(s);
    for (uint32_t v = threadIdx.x; v < len / 16; v += blockDim.x) {
      Acc<DT> acc;
      acc.init(reinterpret_cast<const uint4*>(base)[v]);
#pragma unroll
      for (int j = 1; j < W - 1; ++j) acc.add(reinterpret_cast<const uint4*>(base + j * kPiece)[v]);
      reinterpret_cast<uint4*>(base)[v] = acc.get();
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(dst + lo_b + (uint64_t)i * kPiece, base, len);
      bulk_commit();
      if (i + kRsAhead < np) {
        ring_release_wait();
        issue(i + kRsAhead);
      }
    }
  }
  if (threadIdx.x == 0 && np) {
    bulk_wait_all();
    fence_proxy_async_global();
  }
  p.phase = ph;
}

// a (+) b through shared memory, stored at offset lo_b of all W buffers
template <int DT, int W>
__device__ void tma_add_bcast(Pipe& p, char* const* dst, const char* a, const char* b, uint64_t lo_b,
                              uint64_t nbytes) {
  constexpr uint32_t kPiece = kStageBytes / 2;
  const uint32_t np = (uint32_t)((nbytes + kPiece - 1) / kPiece);
  auto piece_len = [&](uint32_t i) -> uint32_t {
    const uint64_t off = (uint64_t)i * kPiece;
    return (uint32_t)((nbytes - off) < kPiece ? (nbytes - off) : kPiece);
  };
  auto issue = [&](uint32_t i) {
    const int s = i % kStages;
    const uint64_t off = lo_b + (uint64_t)i * kPiece;
    const uint32_t len = piece_len(i);
    mbar_expect_tx(&p.bar[s], 2 * len);
    bulk_load<false>(p.buf(s), a + off, len, &p.bar[s]);
    bulk_load<false>(p.buf(s) + kPiece, b + off, len, &p.bar[s]);
  };
  if (threadIdx.x == 0 && np) {
    fence_proxy_async_global();
    for (uint32_t i = 0; i < np && i < (uint32_t)kAhead; ++i) issue(i);
  }
  uint32_t ph = p.phase;
  for (uint32_t i = 0; i < np; ++i) {
    const int s = i % kStages;
    const uint32_t len = piece_len(i);
    mbar_wait(&p.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    uint4* A = reinterpret_cast<uint4*>(p.buf(s));
    const uint4* B = reinterpret_cast<const uint4*>(p.buf(s) + kPiece);
    for (uint32_t v = threadIdx.x; v < len / 16; v += blockDim.x) A[v] = add_vec<DT>(A[v], B[v]);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t off = lo_b + (uint64_t)i * kPiece;
#pragma unroll
      for (int d = 0; d < W; ++d) bulk_store<false>(dst[d] + off, A, len);
      bulk_commit();
      if (i + kAhead < np) {
        ring_release_wait();
        issue(i + kAhead);
      }
    }
  }
  if (threadIdx.x == 0 && np) {
    bulk_wait_all();
    fence_proxy_async_global();
  }
  p.phase = ph;
}

// LSU version of the same
template <int DT, int W>
__device__ void lsu_add_bcast(char* const* dst, const char* a, const char* b, uint64_t lo_b, uint64_t nbytes) {
  const uint64_t nv = nbytes / 16;
  constexpr int U = 4;
  uint64_t i = threadIdx.x;
  for (; i + (U - 1) * blockDim.x < nv; i += (uint64_t)U * blockDim.x) {
    uint4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      va[u] = ld_vec(a + lo_b + (i + u * blockDim.x) * 16);
      vb[u] = ld_vec(b + lo_b + (i + u * blockDim.x) * 16);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4 z = add_vec<DT>(va[u], vb[u]);
#pragma unroll
      for (int d = 0; d < W; ++d) st_vec(dst[d] + lo_b + (i + u * blockDim.x) * 16, z);
    }
  }
  for (; i < nv; i += blockDim.x) {
    const uint4 z = add_vec<DT>(ld_vec(a + lo_b + i * 16), ld_vec(b + lo_b + i * 16));
#pragma unroll
    for (int d = 0; d < W; ++d) st_vec(dst[d] + lo_b + i * 16, z);
  }
}

// ---------------------------------------------------------------- Phase A
// Canonical sum of the slice over the non-stragglers in ascending physical order.
template <int DT, int W>
__device__ void rs_slice(const LaunchPlan& P, const char* const (&src)[W - 1], char* dst, uint64_t lo_b, uint64_t hi_b) {
  const uint64_t nv = (hi_b - lo_b) / 16;
  constexpr int U = (W <= 4) ? 4 : 2;
  uint64_t i = threadIdx.x;
  const uint64_t step = (uint64_t)U * blockDim.x;
  for (; i + (U - 1) * blockDim.x < nv; i += step) {
    uint4 v[U][W - 1];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < W - 1; ++j) v[u][j] = ld_vec(src[j] + lo_b + (i + u * blockDim.x) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      Acc<DT> acc;
      acc.init(v[u][0]);
#pragma unroll
      for (int j = 1; j < W - 1; ++j) acc.add(v[u][j]);
      st_vec(dst + lo_b + (i + u * blockDim.x) * 16, acc.get());
    }
  }
  for (; i < nv; i += blockDim.x) {
    Acc<DT> acc;
    acc.init(ld_vec(src[0] + lo_b + i * 16));
#pragma unroll
    for (int j = 1; j < W - 1; ++j) acc.add(ld_vec(src[j] + lo_b + i * 16));
    st_vec(dst + lo_b + i * 16, acc.get());
  }
  // tail: fewer than 16 bytes at the very end of the buffer
  const int tail = (int)((hi_b - lo_b) % 16) / P.esize;
  if ((int)threadIdx.x < tail) {
    const uint64_t o = lo_b + nv * 16 + threadIdx.x * P.esize;
    if constexpr (DT == DT_BF16) {
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < W - 1; ++j) {
        float x = __uint_as_float(uint32_t(*(const volatile uint16_t*)(src[j] + o)) << 16);
        a = (j == 0) ? x : __fadd_rn(a, x);
      }
      __nv_bfloat16 h = __float2bfloat16_rn(a);
      *(volatile uint16_t*)(dst + o) = *reinterpret_cast<uint16_t*>(&h);
    } else {
      uint32_t a = *(const volatile uint32_t*)(src[0] + o);
#pragma unroll
      for (int j = 1; j < W - 1; ++j) a = add_word<DT>(a, *(const volatile uint32_t*)(src[j] + o));
      *(volatile uint32_t*)(dst + o) = a;
    }
  }
}

// Phase A body for non-straggler `me`, CTA slot s (slices s*sub .. s*sub+sub-1).
// BC (Broadcast baseline): the partial is announced to every other
// non-straggler (they copy it in ag_body) instead of to the straggler.
// With op lanes (small messages: LaunchPlan::lanes = L > 1, one slice per
// CTA; the split Phase-A kernel uses the same L) Phase A is split over the
// lanes too: CTA (s, q) reduces
// mini-slice m = s*L + q of the G*L equal parts of the chunk (slice s is
// exactly the union of minis s*L .. s*L+L-1) and flags it on its own, so the
// exchange of slice s waits for L flags.
template <int DT, int W, int MV, bool BC = false>
__device__ void rs_body(const LaunchPlan& P, Pipe& pipe, int s, int q, int me, uint32_t ep) {
  const int L = P.lanes;
  const int m = s * L + q;           // this CTA's Phase-A slot
  const int NV = P.G * L * P.sub;    // Phase-A slices per chunk (flag stride)
  if (blockIdx.x == 0 && threadIdx.x == 0) P.state->t_rs_start = globaltimer();
  // barrier (1) among the non-stragglers, per CTA slot
  if (threadIdx.x < W && (int)threadIdx.x != me && (int)threadIdx.x != P.sigma)
    st_release(flag_at(P.flags[threadIdx.x], SLOT_ARRIVE + me, P.fstride, m), ep, P.sys_scope);
  // one waiting thread per peer: the acquire loads overlap instead of queueing
  int ok = 1;
  if (threadIdx.x < W && (int)threadIdx.x != me && (int)threadIdx.x != P.sigma)
    ok = spin_wait(flag_at(P.flags[me], SLOT_ARRIVE + threadIdx.x, P.fstride, m), ep, P, 0x100 | threadIdx.x);
  if (!__syncthreads_and(ok)) return;

  const int g = P.logical_of_phys[me];  // owned chunk
  const Range c = chunk_range(P, g);
  // non-stragglers in ascending physical order (compile-time indices, no local memory)
  const char* src[W - 1];
#pragma unroll
  for (int j = 0; j < W - 1; ++j) src[j] = P.buf[j < P.sigma ? j : j + 1];
  // P.rs_whole: the CTA's `sub` adjacent slices are reduced as one range (no
  // pipeline drain between them) and flagged together after it, with one
  // release fence for all of them; otherwise slice by slice (the next hop can
  // start on the first slice sooner).
  const int nseg = P.rs_whole ? 1 : P.sub;
  for (int j = 0; j < nseg; ++j) {
    const int v = m * P.sub + j;
    Range r = slice_of(c.lo, c.hi, v, NV, 16 / P.esize);
    if (P.rs_whole) r.hi = slice_of(c.lo, c.hi, m * P.sub + P.sub - 1, NV, 16 / P.esize).hi;
    // with two ranks the owner's chunk already is the non-straggler "sum"
    if constexpr (W > 2) {
      if constexpr (MV == MOVER_TMA) {
        const uint64_t lo_b = r.lo * P.esize, hi_b = r.hi * P.esize;
        const uint64_t body = (hi_b - lo_b) / 16 * 16;
        tma_reduce<DT, W>(pipe, P.buf[me], src, lo_b, body);
        rs_slice<DT, W>(P, src, P.buf[me], lo_b + body, hi_b);   // < 16-byte tail only
      } else {
        rs_slice<DT, W>(P, src, P.buf[me], r.lo * P.esize, r.hi * P.esize);
      }
    }
    const int v1 = P.rs_whole ? m * P.sub + P.sub : v + 1;   // slices [v, v1) are done
    __syncthreads();
    if constexpr (BC) {
      if (threadIdx.x < W && (int)threadIdx.x != me && (int)threadIdx.x != P.sigma) {
        fence_release(P.sys_scope);
        for (int u = v; u < v1; ++u) st_flag(flag_at(P.flags[threadIdx.x], SLOT_RSDONE + g, P.fstride, u), ep, P.sys_scope);
      }
    } else if (threadIdx.x == kSignalThread) {
      // "partial ready" for the straggler's half of the exchange, and for this
      // rank's own exchange when another op lane runs it
      fence_release(P.sys_scope);
      for (int u = v; u < v1; ++u) {
        st_flag(flag_at(P.flags[P.sigma], SLOT_RSDONE + g, P.fstride, u), ep, P.sys_scope);
        if (P.lanes > 1) st_flag(flag_at(P.flags[me], SLOT_RS_LOCAL, P.fstride, u), ep, false);
      }
    }
  }
}

// ---------------------------------------------------------------- Broadcast baseline (NEXT N3)
// Straggler-aware Broadcast.  Precondition: the non-stragglers
// complete an AllReduce during the delay = rs_body<BC> (canonical partials)
// then ag_body (every non-straggler copies the other owners' partials).  Then
// bcast_body: the straggler exchanges its entire buffer with its partner
// (logical rank 0; half-split and fused with the add as in B1), and the full
// sum is copied on along the doubling tree of RankPrograms::bc_sender, s
// bytes per copy.  The precondition is chunk-sliced (CTA s: its `sub` slices of
// every chunk); the completion slices the whole buffer contiguously.

template <int MV>
__device__ __forceinline__ void move_bytes(Pipe& pipe, char* dst, const char* src, uint64_t a, uint64_t b) {
  const uint64_t body = (b - a) / 16 * 16;
  if constexpr (MV == MOVER_TMA)
    tma_copy(pipe, dst + a, src + a, body);
  else
    copy_vecs(dst + a, src + a, body / 16);
  copy_tail(dst + a + body, src + a + body, (int)((b - a) % 16));
}

// d0 = d1 = x (+) y over bytes [a, b)
template <int DT, int MV>
__device__ __forceinline__ void add_bytes(const LaunchPlan& P, Pipe& pipe, char* d0, char* d1, const char* x,
                                          const char* y, uint64_t a, uint64_t b) {
  const uint64_t body = (b - a) / 16 * 16;
  char* e1 = d1 ? d1 + a : nullptr;   // d1 == nullptr: one destination
  if constexpr (MV == MOVER_TMA)
    tma_add2<DT>(pipe, d0 + a, e1, x + a, y + a, body);
  else
    add2_vecs<DT>(d0 + a, e1, x + a, y + a, body / 16);
  add2_tail<DT>(d0 + a + body, e1 ? e1 + body : nullptr, x + a + body, y + a + body, (int)((b - a) % 16) / P.esize,
                P.esize);
}

// Non-straggler `me`: copy every other owner's partial (its CTA's slices).
template <int DT, int W, int MV>
__device__ void ag_body(const LaunchPlan& P, Pipe& pipe, int s, int me, uint32_t ep) {
  const int NV = P.G * P.sub, V = 16 / P.esize;
  const int own = P.logical_of_phys[me];
  for (int c = 0; c < P.nchunks; ++c) {
    if (c == own) continue;
    int owner = 0;
#pragma unroll
    for (int q = 0; q < W; ++q)
      if (P.logical_of_phys[q] == c) owner = q;
    const Range cr = chunk_range(P, c);
    for (int j = 0; j < P.sub; ++j) {
      const int v = s * P.sub + j;
      // the owner's partial of slice v is final (and the owner is done reading my copy of it)
      if (!cta_wait(flag_at(P.flags[me], SLOT_RSDONE + c, P.fstride, v), ep, P, 0xC00 | c)) return;
      const Range sl = slice_of(cr.lo, cr.hi, v, NV, V);
      move_bytes<MV>(pipe, P.buf[me], P.buf[owner], sl.lo * P.esize, sl.hi * P.esize);
    }
  }
  // the partner tells the straggler its operand is ready; the others tell
  // their sender in the doubling tree that they may now be overwritten
  if (me == P.bc_partner) {
    // (also to itself: its completion slices the buffer differently, so each
    // of its CTAs waits for all of them)
    __syncthreads();
    if (threadIdx.x == 0) st_release(flag_at(P.flags[P.sigma], SLOT_BC_AGDONE, P.fstride, s), ep, P.sys_scope);
    if (threadIdx.x == 1) st_release(flag_at(P.flags[me], SLOT_BC_AGDONE, P.fstride, s), ep, P.sys_scope);
  } else
    cta_signal(flag_at(P.flags[P.bc_sender[me]], SLOT_BC_READY + me, P.fstride, s), ep, P.sys_scope);
}

// Whole-CTA wait for slot `slot` of rank `me` at every CTA index 0..P.G-1 (one
// waiting thread per flag, so the acquire loads overlap).
__device__ __forceinline__ bool cta_wait_all(const LaunchPlan& P, int me, int slot, uint32_t ep, uint32_t where) {
  int ok = 1;
  for (int i = threadIdx.x; i < P.G; i += blockDim.x)
    ok &= spin_wait(flag_at(P.flags[me], slot, P.fstride, i), ep, P, where) ? 1 : 0;
  return __syncthreads_and(ok);
}

// The completion treats the buffer as a whole (the paper's Broadcast moves s
// bytes per round): CTA s owns the s-th of G contiguous slices of the
// entire buffer, so each step is one TMA pipeline over one range.  Its inputs
// come from the chunk-sliced precondition, so it starts after the peer's
// whole precondition (all G flags).
template <int DT, int W, int MV>
__device__ void bcast_body(const LaunchPlan& P, Pipe& pipe, int s, int me, uint32_t ep) {
  const int p0 = P.bc_partner, sig = P.sigma;
  char* mine = P.buf[me];
  const Range sl = slice_of(0, P.count, s, P.G, 16 / P.esize);
  const uint64_t a = sl.lo * P.esize, b = sl.hi * P.esize;
  bool ok;
  if (me == sig || me == p0) {
    const int peer = (me == sig) ? p0 : sig;
    if (me == sig) {
      // the straggler arrives (barrier (2)); its operand is the partner's full non-straggler sum
      if (threadIdx.x == 0) st_release(flag_at(P.flags[p0], SLOT_ARRIVE + sig, P.fstride, s), ep, P.sys_scope);
      ok = cta_wait_all(P, me, SLOT_BC_AGDONE, ep, 0xD00);
    } else {
      ok = cta_wait(flag_at(P.flags[me], SLOT_ARRIVE + sig, P.fstride, s), ep, P, 0xD01) &&
           cta_wait_all(P, me, SLOT_BC_AGDONE, ep, 0xD04);
    }
    if (ok) {
      // the exchange of the entire buffer: the partner computes the first half
      // of the slice, the straggler the second; both halves land at both ends
      const uint64_t nv = (b - a + 15) / 16;
      const uint64_t m = a + (nv / 2) * 16 < b ? a + (nv / 2) * 16 : b;
      if (me == p0)
        add_bytes<DT, MV>(P, pipe, mine, P.buf[peer], mine, P.buf[peer], a, m);
      else
        add_bytes<DT, MV>(P, pipe, mine, P.buf[peer], P.buf[peer], mine, m, b);
      cta_signal(flag_at(P.flags[peer], SLOT_HAVE, P.fstride, s), ep, P.sys_scope);
      ok = cta_wait(flag_at(P.flags[me], SLOT_HAVE, P.fstride, s), ep, P, 0xD02);
    }
  } else {
    ok = cta_wait(flag_at(P.flags[me], SLOT_HAVE, P.fstride, s), ep, P, 0xD03);
  }
  // holders copy the slice on, one receiver per round, once the receiver's
  // whole precondition is done (it no longer writes its own buffer)
  for (int rd = 1; ok && rd < W; ++rd)
    for (int q = 0; ok && q < W; ++q) {
      if (P.bc_sender[q] != me || P.bc_round[q] != rd) continue;
      if (!(ok = cta_wait_all(P, me, SLOT_BC_READY + q, ep, 0xD10 | q))) break;
      move_bytes<MV>(pipe, P.buf[q], mine, a, b);
      cta_signal(flag_at(P.flags[q], SLOT_HAVE, P.fstride, s), ep, P.sys_scope);
    }
}

// Phase B body (Algorithm 1 round executor) for rank `me`, CTA slot s, op
// lane q: walks the rank's ops k with k % lanes == q in round order; every op
// runs over the CTA's `sub` slices one after the other, each handed to the
// partner with its own flag.  With one lane a CTA runs all of the rank's ops
// of its slice in round order.  With several lanes (small messages, where a
// hop's latency, not bandwidth, is the cost) each op starts as soon as its
// own inputs have landed — the transfers, partners and bytes are Algorithm 1's,
// only the round barrier is replaced by the data dependencies: the straggler's
// n-1 exchanges (independent of each other) no longer queue behind one CTA.
// Lanes hand off through local flags: an exchange's own half (SLOT_SELF, for a
// later send of that chunk on another lane) and, in the fused call, the
// lanes' parts of the Phase-A partial (SLOT_RS_LOCAL, for the exchange; see
// rs_body).
template <int DT, int W, int MV, bool FUSED>
__device__ void complete_body(const LaunchPlan& P, Pipe& pipe, int s, int q, int me, uint32_t ep) {
  const int NV = P.G * P.sub;   // slices per chunk (flag stride)
  const int V = 16 / P.esize;
  const int lanes = P.lanes;
  constexpr bool tma = MV == MOVER_TMA;
  constexpr bool kLife = STRAGGLAR_LIFETIME_HINTS != 0;   // L2 hints by data lifetime (Op::life)
  // the straggler reaches barrier (2): announce per CTA slot to the others
  if (q == 0 && me == P.sigma && threadIdx.x < W && (int)threadIdx.x != me)
    st_release(flag_at(P.flags[threadIdx.x], SLOT_ARRIVE + me, P.fstride, s), ep, P.sys_scope);
  char* mine = P.buf[me];
  const int nops = P.nops[me];
  // lane of this rank's exchange op of chunk c (-1: no exchange of c here)
  auto exch_lane = [&](int c) {
    for (int k = 0; k < nops; ++k) {
      const Op o = P.ops[me][k];
      if (o.chunk == c && (o.kind == OP_EXCH_LOW || o.kind == OP_EXCH_HIGH)) return k % lanes;
    }
    return -1;
  };
  bool ok = true;
  // signalling warp (STRAGGLAR_SIGNALLER, TMA, one op lane): warp 1 only publishes flags
  const bool sig = STRAGGLAR_SIGNALLER && tma && lanes == 1;
  __shared__ SigQ sq;
  if (sig) {
    if (threadIdx.x == 0) sq.head = sq.tail = 0;
    __syncthreads();
  }
  if (sig && (threadIdx.x >> 5) == 1) {
    if (threadIdx.x == 32) sig_loop(sq, P, ep);
  } else {
  // the CTA's units (op k, sub-slice j): op by op (all sub-slices of an op,
  // then the next op), or with P.sub_major sub-slice by sub-slice
  const int nk = (nops - q + lanes - 1) / lanes;   // this lane's ops: k = q, q + lanes, ...
  int ki = 0, j = 0;   // this unit's op index (k = q + ki * lanes) and sub-slice
  for (int u = 0; u < nk * P.sub && ok;
       ++u, P.sub_major ? (++ki == nk ? (ki = 0, ++j) : 0) : (++j == P.sub ? (j = 0, ++ki) : 0)) {
    const int k = q + ki * lanes;
    const Op op = P.ops[me][k];
    const int c = op.chunk, peer = op.peer;
    const Range cr = chunk_range(P, c);
    {
      const int v = s * P.sub + j;
      const Range sl = slice_of(cr.lo, cr.hi, v, NV, V);
      // optional trace: per op and slice, when the wait began, data movement began, it was signalled
      uint64_t* tr = (P.trace && threadIdx.x == 0) ? P.trace + (((size_t)me * NV + v) * kMaxOps + k) * 3 : nullptr;
      if (tr) tr[0] = globaltimer();
      const uint64_t nvec_total = (sl.hi - sl.lo + V - 1) / V;
      const uint64_t mid = sl.lo + (nvec_total / 2) * V < sl.hi ? sl.lo + (nvec_total / 2) * V : sl.hi;
      if (op.kind == OP_EXCH_LOW) {
        // non-straggler r: [lo, mid) of c_r = partial_r (+) x_sigma, stored at both ends
        // (fused call with lanes: Phase A of this slice was split over the L lanes)
        if (FUSED && lanes > 1 &&
            !(ok = cta_wait_range(P.flags[me], SLOT_RS_LOCAL, s * lanes, lanes, ep, P, 0x210 | k, true)))
          break;
        if (!(ok = sig ? grp_wait(flag_at(P.flags[me], SLOT_ARRIVE + peer, P.fstride, s), ep, P, 0x200 | k)
                       : cta_wait(flag_at(P.flags[me], SLOT_ARRIVE + peer, P.fstride, s), ep, P, 0x200 | k)))
          break;
        if (tr) tr[1] = globaltimer();
        const uint64_t a = sl.lo * P.esize, b = mid * P.esize, body = (b - a) / 16 * 16;
        if constexpr (tma) {
          if (sig)
            tma_add2<DT, true>(pipe, mine + a, P.buf[peer] + a, mine + a, P.buf[peer] + a, body, !kLife,
                               !kLife || (op.life & LIFE_SELF_REREAD), !kLife || (op.life & LIFE_PEER_REREAD));
          else
            tma_add2<DT>(pipe, mine + a, P.buf[peer] + a, mine + a, P.buf[peer] + a, body, !kLife,
                         !kLife || (op.life & LIFE_SELF_REREAD), !kLife || (op.life & LIFE_PEER_REREAD));
        }
        else
          add2_vecs<DT>(mine + a, P.buf[peer] + a, mine + a, P.buf[peer] + a, body / 16);
        add2_tail<DT>(mine + a + body, P.buf[peer] + a + body, mine + a + body, P.buf[peer] + a + body,
                      (int)((b - a) % 16) / P.esize, P.esize);
      } else if (op.kind == OP_EXCH_HIGH) {
        // straggler: [mid, hi) of c_r; waits for rank r's Phase-A partial
        if (lanes > 1) {   // Phase A of the slice was split over the lanes (rs_body)
          if (!(ok = cta_wait_range(P.flags[me], SLOT_RSDONE + c, s * lanes, lanes, ep, P, 0x300 | k))) break;
        } else if (!(ok = sig ? grp_wait(flag_at(P.flags[me], SLOT_RSDONE + c, P.fstride, v), ep, P, 0x300 | k)
                              : cta_wait(flag_at(P.flags[me], SLOT_RSDONE + c, P.fstride, v), ep, P, 0x300 | k))) {
          break;
        }
        if (tr) tr[1] = globaltimer();
        const uint64_t a = mid * P.esize, b = sl.hi * P.esize, body = (b - a) / 16 * 16;
        if constexpr (tma) {
          if (sig)
            tma_add2<DT, true>(pipe, mine + a, P.buf[peer] + a, P.buf[peer] + a, mine + a, body, !kLife,
                               !kLife || (op.life & LIFE_SELF_REREAD), !kLife || (op.life & LIFE_PEER_REREAD));
          else
            tma_add2<DT>(pipe, mine + a, P.buf[peer] + a, P.buf[peer] + a, mine + a, body, !kLife,
                         !kLife || (op.life & LIFE_SELF_REREAD), !kLife || (op.life & LIFE_PEER_REREAD));
        }
        else
          add2_vecs<DT>(mine + a, P.buf[peer] + a, P.buf[peer] + a, mine + a, body / 16);
        add2_tail<DT>(mine + a + body, P.buf[peer] + a + body, P.buf[peer] + a + body, mine + a + body,
                      (int)((b - a) % 16) / P.esize, P.esize);
      } else {
        // copy of a fully reduced chunk (push); if this rank computed half of it
        // in an exchange on another lane, that half must have been stored too
        if (!(ok = sig ? grp_wait(flag_at(P.flags[me], SLOT_HAVE + c, P.fstride, v), ep, P, 0x400 | k)
                       : cta_wait(flag_at(P.flags[me], SLOT_HAVE + c, P.fstride, v), ep, P, 0x400 | k)))
          break;
        if (lanes > 1) {
          const int el = exch_lane(c);
          if (el >= 0 && el != q && !(ok = cta_wait(flag_at(P.flags[me], SLOT_SELF + c, P.fstride, v), ep, P, 0x410 | k, true)))
            break;
        }
        if (tr) tr[1] = globaltimer();
        const uint64_t a = sl.lo * P.esize, b = sl.hi * P.esize, body = (b - a) / 16 * 16;
        if constexpr (tma)
          tma_copy(pipe, P.buf[peer] + a, mine + a, body, !kLife || (op.life & LIFE_SRC_REREAD),
                   !kLife || (op.life & LIFE_PEER_REREAD));
        else
          copy_vecs(P.buf[peer] + a, mine + a, body / 16);
        copy_tail(P.buf[peer] + a + body, mine + a + body, (int)((b - a) % 16));
      }
      if (sig) {
        grp_sync();   // the tail threads' stores (warp 0) before thread 0's post
        if (threadIdx.x == 0) sig_post(sq, ((uint32_t)peer << 24) | (uint32_t)((SLOT_HAVE + c) * P.fstride + v));
      } else {
        cta_signal(flag_at(P.flags[peer], SLOT_HAVE + c, P.fstride, v), ep, P.sys_scope);
      }
      if (lanes > 1 && op.kind != OP_SEND && threadIdx.x == kSignalThread)
        st_release(flag_at(P.flags[me], SLOT_SELF + c, P.fstride, v), ep, false);
      if (tr) tr[2] = globaltimer();
    }
  }
  if (sig && threadIdx.x == 0) sig_post(sq, kSigDone);
  // postcondition: every chunk has landed here (one waiting thread per
  // (chunk, slice) flag, so the acquire loads overlap; lanes split the chunks)
  if (ok) {
    const int nc = (P.nchunks - q + lanes - 1) / lanes;   // chunks c = q, q + lanes, ...
    const int t = sig ? grp_tid() : (int)threadIdx.x;
    if (t < nc * P.sub) {
      const int c = q + (t / P.sub) * lanes, j = t % P.sub;
      spin_wait(flag_at(P.flags[me], SLOT_HAVE + c, P.fstride, s * P.sub + j), ep, P, 0x500 | c);
    }
  }
  }   // not the signalling warp
  __syncthreads();
}

// Direct completion body (NEXT N1(ii)): one round instead of Algorithm 1's
// n + log n - 2.  Owner g (non-straggler) fully reduces its chunk (partial +
// x_sigma, the straggler exchange's single add) and stores the
// result to every rank.  On NVSwitch every port then carries about S bytes
// (vs R*C = 9/7 S for the pairwise schedule at n = 8): the fabric is not
// single-port (the P:149-150 assumption).
template <int DT, int W, int MV>
__device__ void direct_body(const LaunchPlan& P, Pipe& pipe, int s, int me, uint32_t ep) {
  const int NV = P.G * P.sub;   // slices per chunk (flag stride)
  const int V = 16 / P.esize;
  constexpr bool tma = MV == MOVER_TMA;
  int own = -1;
  bool ok = true;
  if (me == P.sigma) {
    // the straggler arrives: its buffer may now be read by every owner
    if (threadIdx.x < W && (int)threadIdx.x != me)
      st_release(flag_at(P.flags[threadIdx.x], SLOT_ARRIVE + me, P.fstride, s), ep, P.sys_scope);
  } else {
    own = P.logical_of_phys[me];
    ok = cta_wait(flag_at(P.flags[me], SLOT_ARRIVE + P.sigma, P.fstride, s), ep, P, 0x900);
    if (ok) {
      // the CTA's sub slices are adjacent: one pass over their union (no
      // pipeline drain between them), then one flag per slice
      const Range cr = chunk_range(P, own);
      const uint64_t a = slice_of(cr.lo, cr.hi, s * P.sub, NV, V).lo * P.esize;
      const uint64_t b = slice_of(cr.lo, cr.hi, s * P.sub + P.sub - 1, NV, V).hi * P.esize;
      const uint64_t body = (b - a) / 16 * 16;
      // every rank's buffer, own included, receives the fully reduced slices
      if constexpr (tma)
        tma_add_bcast<DT, W>(pipe, P.buf, P.buf[me], P.buf[P.sigma], a, body);
      else
        lsu_add_bcast<DT, W>(P.buf, P.buf[me], P.buf[P.sigma], a, body);
      const int tail = (int)((b - a) % 16) / P.esize;
      if ((int)threadIdx.x < tail) {
        // read both operands before any store (the own buffer is a destination)
        const uint64_t o = a + body + threadIdx.x * P.esize;
        char tmp[4];
        scalar_add_store<DT>(tmp, nullptr, P.buf[me] + o, P.buf[P.sigma] + o);
#pragma unroll
        for (int d = 0; d < W; ++d) {
          if (P.esize == 2)
            *(volatile uint16_t*)(P.buf[d] + o) = *reinterpret_cast<uint16_t*>(tmp);
          else
            *(volatile uint32_t*)(P.buf[d] + o) = *reinterpret_cast<uint32_t*>(tmp);
        }
      }
      __syncthreads();
      if (threadIdx.x < W && (int)threadIdx.x != me) {   // one release fence per peer for all its flags
        fence_release(P.sys_scope);
        for (int j = 0; j < P.sub; ++j)
          st_flag(flag_at(P.flags[threadIdx.x], SLOT_HAVE + own, P.fstride, s * P.sub + j), ep, P.sys_scope);
      }
    }
  }
  // postcondition: every other chunk has landed here (one waiting thread per flag)
  if (ok && (int)threadIdx.x < P.nchunks * P.sub) {
    const int c = threadIdx.x / P.sub, j = threadIdx.x % P.sub;
    if (c != own) spin_wait(flag_at(P.flags[me], SLOT_HAVE + c, P.fstride, s * P.sub + j), ep, P, 0xA00 | c);
  }
  __syncthreads();
}

// KIND: 0 Phase A only, 1 Phase B (schedule), 3 Phase B (direct),
//       4 Phase A + schedule in one launch, 5 Phase A + direct in one launch,
//       6 Broadcast baseline precondition (non-straggler AllReduce),
//       7 Broadcast baseline completion, 8 both in one launch.
template <int DT, int W, int MV, int KIND>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_phase(const __grid_constant__ LaunchPlan P) {
  // block -> (local rank, slice slot s, op lane q); lanes > 1 only for Phase B (KIND 1 / 4)
  const int per = P.G * P.lanes;
  const int li = blockIdx.x / per, s = (blockIdx.x % per) % P.G, q = (blockIdx.x % per) / P.G;
  const int me = P.local_rank[li];
  const CallEpoch ce = call_epoch(P);
  const uint32_t ep = ce.ep;
  Pipe pipe = make_pipe(MV == MOVER_TMA);
  const bool stamps = (KIND == 4 || KIND == 5) && P.nlocal == 1;   // per-process fused call
  uint64_t* stamp = P.state->stamp[ep & 1u];   // armed by the previous call's last CTA (or at init)
  if (stamps && threadIdx.x == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&stamp[0]), (unsigned long long)globaltimer());
  if constexpr (KIND == 4 || KIND == 5) {
    // measurement only (team mode): the straggler's CTAs arrive sigma_delay_ns
    // after the launch (P:405-407 idle time, inside the kernel), so Phase B of
    // each slice can overlap the non-stragglers' Phase A tail as on real GPUs
    if (P.sigma_delay_ns && me == P.sigma && threadIdx.x == 0) {
      const uint64_t until = globaltimer() + P.sigma_delay_ns;
      while (globaltimer() < until) __nanosleep(500);
    }
    __syncthreads();
  }
  if constexpr (KIND == 0 || KIND == 4 || KIND == 5)
    if (me != P.sigma) rs_body<DT, W, MV>(P, pipe, s, q, me, ep);
  if (stamps && threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&stamp[1]), (unsigned long long)globaltimer());
  if constexpr (KIND == 1 || KIND == 4) complete_body<DT, W, MV, KIND == 4>(P, pipe, s, q, me, ep);
  if constexpr (KIND == 3 || KIND == 5) direct_body<DT, W, MV>(P, pipe, s, me, ep);
  if constexpr (KIND == 6 || KIND == 8)
    if (me != P.sigma) {
      rs_body<DT, W, MV, true>(P, pipe, s, 0, me, ep);
      ag_body<DT, W, MV>(P, pipe, s, me, ep);
    }
  if constexpr (KIND == 7 || KIND == 8) bcast_body<DT, W, MV>(P, pipe, s, me, ep);
  if (stamps && threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&stamp[2]), (unsigned long long)globaltimer());
  finish_call(P, ce);
}

// ---------------------------------------------------------------- Ring
// Physical ring 0 -> 1 -> ... -> n-1 -> 0 with n chunks.  Step t < n-1: pull
// the left neighbour's partial of chunk (j-1-t) and add the own data (RS);
// step t >= n-1: copy the left neighbour's final chunk (j-t+n-1) (AllGather).
template <int DT, int W, int MV>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_ring(const __grid_constant__ LaunchPlan P) {
  const int li = blockIdx.x / P.G, s = blockIdx.x % P.G;
  const int j = P.local_rank[li];
  const int NV = P.G * P.sub;   // slices per chunk (flag stride); CTA s covers s*sub .. s*sub+sub-1
  const int V = 16 / P.esize;
  const CallEpoch ce = call_epoch(P);
  const uint32_t ep = ce.ep;
  const int left = (j + W - 1) % W, right = (j + 1) % W;
  if (threadIdx.x == 0) st_release(flag_at(P.flags[right], SLOT_RING_ARRIVE, P.fstride, s), ep, P.sys_scope);
  constexpr bool tma = MV == MOVER_TMA;
  Pipe pipe = make_pipe(tma);
  char* mine = P.buf[j];
  const char* lbuf = P.buf[left];
  // with P.sub_major the CTA runs all steps of sub-slice 0, then of 1, ... (a
  // pipelined ring: the same per-slice dependencies, forwarded slices re-read
  // sooner), otherwise step by step over all its sub-slices
  const int nouter = P.sub_major ? P.sub : 1, ninner = P.sub_major ? 1 : P.sub;
  for (int qo = 0; qo < nouter; ++qo)
  for (int t = 0; t < 2 * (W - 1); ++t) {
    const int k = (t < W - 1) ? ((j - 1 - t) % W + 2 * W) % W : ((j - t + W - 1) % W + 2 * W) % W;
    const Range cr = chunk_range(P, k);
    for (int q = qo; q < qo + ninner; ++q) {
      const int v = s * P.sub + q;
      // step 0 waits for the left neighbour's arrival (per CTA), step t for its step t-1 on slice v
      const uint32_t* wf = (t == 0) ? flag_at(P.flags[j], SLOT_RING_ARRIVE, P.fstride, s)
                                    : flag_at(P.flags[j], SLOT_RING_READY + t - 1, P.fstride, v);
      if (!cta_wait(wf, ep, P, 0x600 | t)) {
        finish_call(P, ce);
        return;
      }
      const Range sl = slice_of(cr.lo, cr.hi, v, NV, V);
      const uint64_t a = sl.lo * P.esize, b = sl.hi * P.esize;
      const uint64_t nv = (b - a) / 16;
      if (t < W - 1) {
        if constexpr (tma)
          tma_add2<DT>(pipe, mine + a, nullptr, lbuf + a, mine + a, nv * 16);
        else
          add2_vecs<DT>(mine + a, nullptr, lbuf + a, mine + a, nv);
        add2_tail<DT>(mine + a + nv * 16, nullptr, lbuf + a + nv * 16, mine + a + nv * 16,
                      (int)((b - a) % 16) / P.esize, P.esize);
      } else {
        if constexpr (tma)
          tma_copy(pipe, mine + a, lbuf + a, nv * 16);
        else
          copy_vecs(mine + a, lbuf + a, nv);
        copy_tail(mine + a + nv * 16, lbuf + a + nv * 16, (int)((b - a) % 16));
      }
      if (t < 2 * (W - 1) - 1) cta_signal(flag_at(P.flags[right], SLOT_RING_READY + t, P.fstride, v), ep, P.sys_scope);
    }
  }
  // I am done reading the left buffer; wait until the right neighbour is done with mine
  cta_signal(flag_at(P.flags[left], SLOT_RING_DONE, P.fstride, s), ep, P.sys_scope);
  cta_wait(flag_at(P.flags[j], SLOT_RING_DONE, P.fstride, s), ep, P, 0x700);
  finish_call(P, ce);
}

// ---------------------------------------------------------------- RHD (NEXT N3)
// Recursive halving/doubling, pull-based, n chunks (the Ring's
// partition).  Step t < L (ReduceScatter): partner j ^ 2^t (round
// k pairs ranks differing in bit k); both hold the same block of n/2^t chunks;
// j keeps the lower half if bit t of j is 0 and adds the partner's copy of it
// into its own.  Step L+u (AllGather) mirrors step L-1-u: partner
// j ^ 2^(L-1-u); j copies the partner's fully reduced block (its sibling).  Step tau's partner is
// told when j finished step tau-1 (SLOT_RHD_READY + tau, per slice); AllGather
// readers report back (SLOT_RHD_DONE) so no rank leaves while its buffer is read.
template <int DT, int W, int MV>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_rhd(const __grid_constant__ LaunchPlan P) {
  constexpr int L = (W >= 8) ? 3 : (W >= 4) ? 2 : 1;
  static_assert((1 << L) == W, "RHD needs a power-of-two world");
  const int li = blockIdx.x / P.G, s = blockIdx.x % P.G;
  const int j = P.local_rank[li];
  const int NV = P.G * P.sub;
  const int V = 16 / P.esize;
  const CallEpoch ce = call_epoch(P);
  const uint32_t ep = ce.ep;
  auto partner = [&](int tau) { return j ^ (tau < L ? (1 << tau) : (1 << (2 * L - 1 - tau))); };
  if (threadIdx.x == 0) st_release(flag_at(P.flags[partner(0)], SLOT_RHD_READY, P.fstride, s), ep, P.sys_scope);
  Pipe pipe = make_pipe(MV == MOVER_TMA);
  char* mine = P.buf[j];
  bool ok = true;
  // with P.sub_major all steps of sub-slice 0, then of 1, ... (as in k_ring)
  const int nouter = P.sub_major ? P.sub : 1, ninner = P.sub_major ? 1 : P.sub;
  for (int qo = 0; qo < nouter && ok; ++qo) {
  int blo = 0, m = W;   // the block of chunks j works on
  for (int tau = 0; tau < 2 * L && ok; ++tau) {
    const int p = partner(tau);
    const char* pbuf = P.buf[p];
    int clo, cn;        // chunks moved this step
    if (tau < L) {
      m /= 2;
      blo = (j & (1 << tau)) ? blo + m : blo;
      clo = blo;
      cn = m;
    } else {
      clo = blo ^ m;    // the partner's block (aligned siblings)
      cn = m;
    }
    for (int q = qo; q < qo + ninner; ++q) {
      const int v = s * P.sub + q;
      const uint32_t* wf = flag_at(P.flags[j], SLOT_RHD_READY + tau, P.fstride, tau == 0 ? s : v);
      if (!(ok = cta_wait(wf, ep, P, 0xE00 | tau))) break;
      for (int c = clo; c < clo + cn; ++c) {
        const Range cr = chunk_range(P, c);
        const Range sl = slice_of(cr.lo, cr.hi, v, NV, V);
        const uint64_t a = sl.lo * P.esize, b = sl.hi * P.esize;
        if (tau < L)
          add_bytes<DT, MV>(P, pipe, mine, nullptr, pbuf, mine, a, b);
        else
          move_bytes<MV>(pipe, mine, pbuf, a, b);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (tau + 1 < 2 * L) st_release(flag_at(P.flags[partner(tau + 1)], SLOT_RHD_READY + tau + 1, P.fstride, v), ep, P.sys_scope);
        if (tau >= L) st_release(flag_at(P.flags[p], SLOT_RHD_DONE + tau - L, P.fstride, v), ep, P.sys_scope);
      }
    }
    if (tau >= L) {
      blo = blo < clo ? blo : clo;
      m *= 2;
    }
  }
  }
  // every AllGather partner finished reading my buffer (one waiting thread per flag)
  if (ok && (int)threadIdx.x < L * P.sub) {
    const int u = threadIdx.x / P.sub, q = threadIdx.x % P.sub;
    spin_wait(flag_at(P.flags[j], SLOT_RHD_DONE + u, P.fstride, s * P.sub + q), ep, P, 0xE10 | u);
  }
  finish_call(P, ce);
}

template <int DT, int W, int MV>
inline void* kernel_ptr_mv(int which) {
  switch (which) {
    case 0: return (void*)k_phase<DT, W, MV, 0>;   // Phase A
    case 1: return (void*)k_phase<DT, W, MV, 1>;   // Phase B, Algorithm 1 schedule
    case 2: return (void*)k_ring<DT, W, MV>;
    case 3: return (void*)k_phase<DT, W, MV, 3>;   // Phase B, direct completion
    case 4: return (void*)k_phase<DT, W, MV, 4>;   // A + B (schedule), one launch
    case 5: return (void*)k_phase<DT, W, MV, 5>;   // A + B (direct), one launch
    case 6: return (void*)k_phase<DT, W, MV, 6>;   // Broadcast baseline: non-straggler AllReduce
    case 7: return (void*)k_phase<DT, W, MV, 7>;   // Broadcast baseline: exchange + doubling copies
    case 8: return (void*)k_phase<DT, W, MV, 8>;   // Broadcast baseline, one launch
    case 9:
      if constexpr ((W & (W - 1)) == 0) return (void*)k_rhd<DT, W, MV>;   // RHD baseline
      return nullptr;
    default: return nullptr;
  }
}

template <int DT, int W>
inline void* kernel_ptr(int which, int mover) {
  return mover == MOVER_TMA ? kernel_ptr_mv<DT, W, MOVER_TMA>(which) : kernel_ptr_mv<DT, W, MOVER_LSU>(which);
}

// Per-dtype instantiation units (kernels_i32.cu, kernels_f32.cu, kernels_bf16.cu)
void* select_kernel_i32(int which, int world, int mover);
void* select_kernel_f32(int which, int world, int mover);
void* select_kernel_bf16(int which, int world, int mover);

}  // namespace stragglar
