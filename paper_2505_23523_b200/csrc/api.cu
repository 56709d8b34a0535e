// C ABI of libstragglar.so (declared in include/stragglar.h).
//
// Host side only: argument checks, the per-rank schedule programs, IPC handle
// plumbing, flag/epoch management and kernel launches.  No data is touched on
// the host; every step of the collective runs in kernels.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <unistd.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "../../include/stragglar.h"
#include "plan.h"
#include "schedule.h"

namespace stragglar {
void* select_kernel(int which, int dtype, int world, int mover);
cudaError_t launch_plan_kernel(int which, int dtype, const LaunchPlan& P, int nblocks, cudaStream_t stream);
cudaError_t launch_delay(const uint64_t* base_ptr, uint64_t ns, DevState* st, cudaStream_t stream);
cudaError_t launch_barrier(const LaunchPlan& P, cudaStream_t stream);
cudaError_t occupancy_blocks_per_sm(int which, int dtype, int world, int mover, int* blocks);
cudaError_t launch_probe_copy(const ProbeArgs& A, int mover, int nblocks, cudaStream_t stream);
cudaError_t launch_nvls(int dtype, const LaunchPlan& P, int nblocks, cudaStream_t stream, bool emulated);
cudaError_t launch_nvls_selftest(int dtype, char* mc, uint64_t bytes, cudaStream_t stream);
cudaError_t launch_probe_pingpong(uint32_t* mine, uint32_t* theirs, int initiator, int iters, DevState* st,
                                  uint64_t timeout_ns, uint32_t* host_err, cudaStream_t stream);
}  // namespace stragglar

using namespace stragglar;

namespace {

enum { K_RS = 0, K_COMPLETE = 1, K_RING = 2, K_DIRECT = 3, K_FUSED = 4, K_FUSED_DIRECT = 5,
       K_BCAST_A = 6, K_BCAST_B = 7, K_BCAST = 8, K_RHD = 9, K_NUM = 10 };
constexpr int kDefaultMover = MOVER_TMA;   // measured faster (profiles/r01)

std::atomic<uint64_t> g_launches{0};

// The communicator's layout knobs.  Every rank must use the same values (a
// flag index covers the same byte range on every rank only if they agree), so
// they travel in the flag-array blob and stragglar_import_handles rejects a
// mismatch instead of running with silently different slice layouts.
struct Layout {
  int32_t world, sigma, G_alloc, sub_max, mover, sys_scope, lanes_max, sub_major;
  uint64_t slice_bytes, sub_bytes, lane_slice_max, e2e_piece_bytes;   // e2e: every rank must cut the same pieces
  uint64_t base_sub_bytes;
  int32_t base_sub_major, pad2;
};

struct IpcBlob {          // what travels between processes, per rank
  cudaIpcMemHandle_t handle;
  uint64_t offset;        // of the registered pointer inside its allocation
  uint64_t bytes;
  Layout layout;          // flag-array blob only (zero in buffer blobs)
  int32_t rank;           // the exporting rank
  int32_t resident_ctas;  // co-resident CTA capacity of the exporter's GPU (flag blob only)
  char uuid[16];          // the exporter's GPU (ranks sharing a GPU share its SMs)
};

struct Registration {
  char* local = nullptr;
  size_t bytes = 0;
  char* peer[kMaxWorld] = {nullptr};
  void* mapped[kMaxWorld] = {nullptr};   // cudaIpcOpenMemHandle results (closed by deregister / finalize)
};

struct Comm {
  bool active = false;
  bool team = false;
  int world = 0, rank = -1, sigma = -1, device = -1;
  int G = 0;                   // CTAs per rank (the launch's co-residency budget)
  int G_alloc = 0;             // CTAs per rank the flag array was sized for (fixes the flag stride)
  int sub = 1;                 // slices per CTA at most (STRAGGLAR_SUBSLICES)
  uint64_t sub_bytes = 0;      // target slice size on large messages (STRAGGLAR_SUBSLICE_BYTES)
  uint64_t base_sub_bytes = 0; // the same for the Ring / RHD baselines (STRAGGLAR_BASELINE_SUBSLICE_BYTES)
  int base_sub_major = 1;      // their unit order (STRAGGLAR_BASELINE_SUB_MAJOR)
  int lanes_max = kMaxOps;     // Phase-B op lanes per slice at most (STRAGGLAR_OP_LANES; 1 = off)
  int rs_whole = 1;                 // Phase A over a CTA's sub slices as one range (STRAGGLAR_RS_WHOLE)
  int sub_major = 1;                // unit order of Phase B, Ring, RHD (STRAGGLAR_SUB_MAJOR; plan.h LaunchPlan::sub_major)
  uint64_t lane_slice_max = 32768;  // slices may grow to this size to make room for op lanes
                                    // (STRAGGLAR_LANE_SLICE_MAX; 0 = keep slice_bytes)
  bool rs_pending = false;     // team: a Phase A awaits its Phase B (same call epoch)
  const void* rs_buf0 = nullptr;  // team: the pending Phase A's first buffer, count and dtype
  size_t rs_count = 0;
  int rs_dtype = -1;
  bool bc_pending = false;     // team: a Broadcast-baseline precondition awaits its completion
  uint32_t* flags = nullptr;   // own flag array(s); team: world of them back to back
  uint32_t* peer_flags[kMaxWorld] = {nullptr};
  size_t rank_bytes = 0;       // flag bytes per rank
  int resident = 0;            // co-resident CTAs of all kernels on this GPU (occupancy x SMs)
  int share = 1;               // ranks of this communicator on this rank's GPU (from the blobs)
  uint32_t* host_err = nullptr;// pinned, device-mapped copy of the error word (sticky; read without sync)
  uint32_t* host_err_dev = nullptr;
  bool imported = false;
  DevState* state = nullptr;
  RankPrograms progs;
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
  int mover = MOVER_LSU;
  uint64_t* trace = nullptr;            // Phase-B op trace (optional)
  // tuning knobs, read from the environment once at init (include/stragglar.h)
  uint64_t slice_bytes = 16384;         // STRAGGLAR_SLICE_BYTES
  int sys_scope = 1;                    // STRAGGLAR_SYS_SCOPE (team mode only; default 0 there)
  uint64_t e2e_piece_bytes = 8ull << 20;// STRAGGLAR_E2E_PIECE_BYTES (8 MiB measured best)
  int e2e_streams = 1;                  // STRAGGLAR_E2E_STREAMS (1 measured best)
  int last_slices = 0;                  // slices per chunk of the last Phase-B call (trace layout)
  double alpha_s = 3e-6;               // P:450 per-message latency used in the paper's model
  double beta_s_per_byte = 1.0 / 770e9; // measured B200 peer copy per direction (B200_PROFILING.md)
  std::vector<Registration> regs;
  std::vector<void*> opened;   // IPC mappings to close
  // NEXT N1(i) (nvls.cu): the library-owned arena bound to two multicast objects
  struct Nvls {
    int stage = 0;                                   // 0 none, 1 begun, 2 imported, 3 bound (ready)
    size_t bytes = 0;                                // arena size (multicast granularity)
    unsigned long long mem = 0, mc_all = 0, mc_ns = 0, sigma_mem = 0;   // CUmemGenericAllocationHandle
    unsigned long long va = 0, mc_all_va = 0, mc_ns_va = 0, sigma_va = 0;
    int fds[3] = {-1, -1, -1};
  } nvls;
};

Comm g_proc;   // per-process communicator
Comm g_team;   // single-device team
std::mutex g_mu;

#define CK(x)                                        \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) return STRAGGLAR_ERR_CUDA;\
  } while (0)

int esize_of(int dtype) {
  switch (dtype) {
    case STRAGGLAR_INT32:
    case STRAGGLAR_FLOAT32: return 4;
    case STRAGGLAR_BFLOAT16: return 2;
    default: return 0;
  }
}

bool supported_world(int w) { return w == 2 || w == 4 || w == 6 || w == 8; }  // 6: Appendix B schedule

uint64_t chunk_elems(uint64_t count, int parts, int esize) {
  const uint64_t v = 16 / esize;
  const uint64_t per = count ? (count + parts - 1) / parts : 0;
  return (per + v - 1) / v * v;
}

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* s = std::getenv(name);
  if (!s || !*s) return dflt;
  return std::strtoull(s, nullptr, 10);
}

// Smallest occupancy over all kernels of this world size, times the SM count.
int resident_ctas(int world, int mover, int* sm_count) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  int best = 1 << 30;
  for (int which = 0; which < K_NUM; ++which)
    for (int dt = 0; dt < 3; ++dt) {
      if (!select_kernel(which, dt, world, mover)) continue;   // RHD: powers of two only
      int b = 0;
      if (occupancy_blocks_per_sm(which, dt, world, mover, &b) != cudaSuccess) return -1;
      best = b < best ? b : best;
    }
  if (sm_count) *sm_count = sms;
  return best * sms;
}

int common_init(Comm& c, int world, int rank, int sigma, bool team) {
  if (!supported_world(world)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (sigma < 0 || sigma >= world) return STRAGGLAR_ERR_INVALID_ARG;
  if (!team && (rank < 0 || rank >= world)) return STRAGGLAR_ERR_INVALID_ARG;
  try {
    c.progs = build_programs(world, sigma);
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_INTERNAL;
  }
  CK(cudaGetDevice(&c.device));
  {
    const char* m = std::getenv("STRAGGLAR_MOVER");
    c.mover = (m && std::strcmp(m, "lsu") == 0) ? MOVER_LSU : (m && std::strcmp(m, "tma") == 0) ? MOVER_TMA : kDefaultMover;
  }
  int sms = 0;
  int cap = resident_ctas(world, c.mover, &sms);
  if (cap <= 0) return STRAGGLAR_ERR_CUDA;
  const int device_cap = cap;   // the whole GPU's (what ranks sharing it divide, stragglar_import_handles)
  {
    // an MPS client capped to a share of the SMs can keep only that share resident
    const uint64_t pct = env_u64("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE", 100);
    if (pct >= 1 && pct < 100) {
      cap = (int)(cap * pct / 100);
      sms = (int)(sms * pct / 100);
      if (sms < 1) sms = 1;
      if (cap < 1) cap = 1;
    }
  }
  int G;
  if (team) {
    G = cap / world;                                   // every rank's CTAs co-resident
  } else {
    G = (int)env_u64("STRAGGLAR_SLICES", (uint64_t)(2 * sms));
    if (G > cap) G = cap;
  }
  const uint64_t forced = env_u64(team ? "STRAGGLAR_TEAM_SLICES" : "STRAGGLAR_SLICES_FORCE", 0);
  if (forced) G = (int)forced;
  if (G > kMaxSlices) G = kMaxSlices;
  if (G < 1 || (team && G * world > cap)) return STRAGGLAR_ERR_UNSUPPORTED;
  c.G = G;
  c.G_alloc = G;
  c.resident = device_cap;
  c.world = world;
  c.rank = team ? -1 : rank;
  c.sigma = sigma;
  c.team = team;
  c.rs_pending = false;
  c.bc_pending = false;
  c.timeout_ns = env_u64("STRAGGLAR_TIMEOUT_MS", 10000) * 1000000ull;
  c.slice_bytes = env_u64("STRAGGLAR_SLICE_BYTES", 16384);
  c.sys_scope = team ? (int)env_u64("STRAGGLAR_SYS_SCOPE", 0) : 1;
  // the baselines' own sub-slice target, tuned for them like ours (sub-slice-major
  // order, profiles/r02/ab/r02aa_*): Ring 1286 -> 1091 us, RHD 1386 -> 1292 us at
  // 64 KB with GPU-scope flags (config 2); 128 KB at system scope (Ring 1369 vs 1332)
  c.base_sub_bytes = env_u64("STRAGGLAR_BASELINE_SUBSLICE_BYTES", c.sys_scope ? 128 * 1024 : 64 * 1024);
  // and their own unit order: sub-slice-major helps them with GPU-scope flags
  // (Ring 1377 -> 1286 us, team config 2) but not per process under MPS (n = 8:
  // Ring 1082 -> 1278 us, RHD 1013 -> 1317 us, profiles/r02/final/r02f2_*)
  c.base_sub_major = (int)env_u64("STRAGGLAR_BASELINE_SUB_MAJOR", c.sys_scope ? 0 : 1) ? 1 : 0;
  // Sub-slices (finer hand-offs): team Phase B -3.7 % at gpu scope; at system
  // scope (per process, MPS-shared GPU, round 2) equal or better for T_post
  // (config 2 n = 8: 667-708 vs 715-716 us) and 10 % better for the Ring, once
  // Phase A no longer pays a drain and a fence per sub-slice (rs_whole;
  // DESIGN.md §10).  Round 1 chose 1 at system scope under a 12 % MPS thread cap.
  c.sub = (int)env_u64("STRAGGLAR_SUBSLICES", kMaxSub);
  c.sub_bytes = env_u64("STRAGGLAR_SUBSLICE_BYTES", 128 * 1024);
  if (c.sub < 1) c.sub = 1;
  if (c.sub > kMaxSub) c.sub = kMaxSub;
  c.lane_slice_max = env_u64("STRAGGLAR_LANE_SLICE_MAX", 32768);
  c.rs_whole = (int)env_u64("STRAGGLAR_RS_WHOLE", 1) ? 1 : 0;
  c.sub_major = (int)env_u64("STRAGGLAR_SUB_MAJOR", 1) ? 1 : 0;
  c.lanes_max = (int)env_u64("STRAGGLAR_OP_LANES", kMaxOps);
  if (c.lanes_max < 1) c.lanes_max = 1;
  c.e2e_piece_bytes = env_u64("STRAGGLAR_E2E_PIECE_BYTES", 8ull << 20);
  c.e2e_streams = (int)env_u64("STRAGGLAR_E2E_STREAMS", 1);
  c.rank_bytes = ((size_t)kSlots * G * kMaxSub * sizeof(uint32_t) + 255) / 256 * 256;
  const size_t nbytes = team ? c.rank_bytes * world : c.rank_bytes;
  auto fail_free = [&]() {
    if (c.flags) cudaFree(c.flags);
    if (c.state) cudaFree(c.state);
    if (c.host_err) cudaFreeHost(c.host_err);
    c.flags = nullptr;
    c.state = nullptr;
    c.host_err = nullptr;
    return STRAGGLAR_ERR_CUDA;
  };
  DevState init;
  std::memset(&init, 0, sizeof(init));
  init.stamp[0][0] = init.stamp[1][0] = ~0ull;   // armed: the first call's min start
  if (cudaMalloc(&c.flags, nbytes) != cudaSuccess || cudaMemset(c.flags, 0, nbytes) != cudaSuccess ||
      cudaMalloc(&c.state, sizeof(DevState)) != cudaSuccess ||
      cudaMemcpy(c.state, &init, sizeof(DevState), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaHostAlloc(&c.host_err, sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&c.host_err_dev, c.host_err, 0) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return fail_free();
  *(volatile uint32_t*)c.host_err = 0;
  for (int p = 0; p < kMaxWorld; ++p) c.peer_flags[p] = nullptr;
  if (team) {
    for (int p = 0; p < world; ++p)
      c.peer_flags[p] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c.flags) + (size_t)p * c.rank_bytes);
    c.imported = true;
  } else {
    c.peer_flags[rank] = c.flags;
    c.imported = (world == 1);
  }
  c.active = true;
  return STRAGGLAR_OK;
}

Layout layout_of(const Comm& c) {
  Layout l;
  std::memset(&l, 0, sizeof(l));
  l.world = c.world;
  l.sigma = c.sigma;
  l.G_alloc = c.G_alloc;
  l.sub_max = c.sub;
  l.mover = c.mover;
  l.sys_scope = c.sys_scope;
  l.lanes_max = c.lanes_max;
  l.lane_slice_max = c.lane_slice_max;
  l.slice_bytes = c.slice_bytes;
  l.sub_bytes = c.sub_bytes;
  l.base_sub_bytes = c.base_sub_bytes;
  l.base_sub_major = c.base_sub_major;
  l.e2e_piece_bytes = c.e2e_piece_bytes;
  l.sub_major = c.sub_major;
  return l;
}

// A watchdog timeout (or another device-side error) is sticky: the kernel that
// records it also writes the pinned host copy, and every later call returns
// STRAGGLAR_ERR_TIMEOUT without launching until stragglar_check_error clears
// it — the flags are then out of step, so the caller must re-initialize.
bool sticky_error(const Comm& c) { return c.host_err && *(volatile const uint32_t*)c.host_err != 0; }

void nvls_release(Comm& c);

void common_finalize(Comm& c) {
  if (!c.active) return;
  cudaDeviceSynchronize();
  nvls_release(c);
  for (void* p : c.opened) cudaIpcCloseMemHandle(p);
  c.opened.clear();
  for (auto& r : c.regs)
    for (int p = 0; p < c.world; ++p)
      if (r.mapped[p]) cudaIpcCloseMemHandle(r.mapped[p]);
  c.regs.clear();
  if (c.flags) cudaFree(c.flags);
  if (c.state) cudaFree(c.state);
  if (c.trace) cudaFree(c.trace);
  if (c.host_err) cudaFreeHost(c.host_err);
  c = Comm();
}

// Slices per call: about one slice per slice_bytes of a chunk.  Small messages
// use few CTAs (less flag traffic per round); large ones all G CTAs, each
// covering up to `sub` slices.  Any (G, sub) is safe call to call: flags hold
// monotone epochs, so values left at other positions by earlier calls are
// stale (< epoch); within a call every kernel uses the same layout.
void slices_for(const Comm& c, uint64_t chunk_bytes, int* G, int* sub, bool baseline = false) {
  const uint64_t per = c.slice_bytes;
  uint64_t g = per ? (chunk_bytes + per - 1) / per : (uint64_t)c.G * c.sub;
  if (g < 1) g = 1;
  if (g <= (uint64_t)c.G) {
    *G = (int)g;
    *sub = 1;
    return;
  }
  // large messages: each CTA covers ~chunk/(G*sub_bytes) slices of about
  // sub_bytes (rounded; 1 if sub_bytes is 0)
  const uint64_t unit = (uint64_t)c.G * (baseline ? c.base_sub_bytes : c.sub_bytes);
  uint64_t m = unit ? (chunk_bytes + unit / 2) / unit : 1;
  if (m < 1) m = 1;
  if (m > (uint64_t)c.sub) m = c.sub;
  *G = c.G;
  *sub = (int)m;
}

int max_ops(const Comm& c) {
  int m = 1;
  for (int p = 0; p < c.world; ++p) m = c.progs.nops[p] > m ? c.progs.nops[p] : m;
  return m;
}

// Small messages (one slice per CTA, fewer slices than the CTA budget B):
// trade slices for op lanes (set_op_lanes) — fewer, larger slices (up to
// lane_slice_max bytes) so that every op of a rank can get its own CTA:
// G = max(B / max_ops, ceil(chunk / lane_slice_max)), never more than the
// slice rule gave.  Measured (n = 8 bf16, team): 2 MiB T_post 30.9 -> 24.7 us,
// 8 MiB 45.1 -> 40.5 us with 32 KB slices and lanes (profiles/r02/ab).  Every
// StragglAR kernel of a call (Phase A, B, fused, direct) uses this same G.
void lane_slices(const Comm& c, uint64_t chunk_bytes, int* G, int sub) {
  if (sub != 1 || c.lane_slice_max == 0 || c.lanes_max <= 1) return;
  const int nops = max_ops(c);
  if ((int64_t)(*G) * nops <= c.G) return;                       // every op gets a lane already
  int64_t g = c.G / nops;
  const int64_t gmin = (int64_t)((chunk_bytes + c.lane_slice_max - 1) / c.lane_slice_max);
  if (g < gmin) g = gmin;
  if (g < 1) g = 1;
  if (g < *G && c.G / g >= 2) *G = (int)g;   // only when it buys at least two lanes
}

// The call's epoch is not a launch parameter: kernels read state->epoch + 1 and
// the last CTA of the call's final kernel bumps it (graph-capturable).
LaunchPlan base_plan(const Comm& c, size_t count, int dtype, bool last_kernel) {
  LaunchPlan P;
  std::memset(&P, 0, sizeof(P));
  P.world = c.world;
  P.sigma = c.sigma;
  P.G = c.G;
  P.fstride = c.G_alloc * kMaxSub;
  P.last_kernel = last_kernel ? 1 : 0;
  P.count = count;
  P.esize = esize_of(dtype);
  P.ce = chunk_elems(count, c.world - 1, P.esize);
  P.nchunks = c.world - 1;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
  P.timeout_ns = c.timeout_ns;
  P.mover = c.mover;
  P.trace = c.trace;
  P.sys_scope = c.sys_scope;
  P.state = c.state;
  P.host_err = c.host_err_dev;
  P.lanes = 1;
  P.rs_whole = c.rs_whole;
  P.sub_major = c.sub_major;
  P.bc_partner = c.progs.bc_partner;
  for (int p = 0; p < c.world; ++p) {
    P.flags[p] = c.peer_flags[p];
    P.logical_of_phys[p] = c.progs.logical_of_phys[p];
    P.bc_sender[p] = c.progs.bc_sender[p];
    P.bc_round[p] = c.progs.bc_round[p];
    P.nops[p] = c.progs.nops[p];
    for (int k = 0; k < c.progs.nops[p]; ++k) P.ops[p][k] = c.progs.ops[p][k];
  }
  return P;
}

// Phase-B op lanes (LaunchPlan::lanes): when a call uses few slices (small
// messages) the idle CTA budget runs a rank's ops on separate CTAs, so an op
// waits only for its own inputs instead of the rank's previous op (one slice
// per CTA only; the same value on every rank: it depends on the call and the
// agreed layout alone).
void set_op_lanes(const Comm& c, LaunchPlan& P) {
  const int maxops = max_ops(c);
  int lanes = 1;
  if (P.sub == 1 && P.G > 0) {
    lanes = c.G / P.G;
    if (lanes > maxops) lanes = maxops;
    if (lanes > c.lanes_max) lanes = c.lanes_max;
    if (lanes < 1) lanes = 1;
  }
  P.lanes = lanes;
}

// The schedule's kernels of one call (Phase A, Phase B, both fused) share one
// layout: lane-aware slices, then the op lanes.  The other algorithms keep the
// plain slice rule.
void stragglar_layout(const Comm& c, LaunchPlan& P) {
  lane_slices(c, P.ce * P.esize, &P.G, P.sub);
  set_op_lanes(c, P);
}

int check_args(const void* buf, size_t count, int dtype, int op) {
  if (op != STRAGGLAR_SUM) return STRAGGLAR_ERR_UNSUPPORTED;
  if (!esize_of(dtype)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (count == 0) return STRAGGLAR_OK;
  if (!buf) return STRAGGLAR_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(buf) % 16) return STRAGGLAR_ERR_INVALID_ARG;
  return STRAGGLAR_OK;
}

int team_check(void* const* bufs, size_t count, int dtype, int op) {
  if (!g_team.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (op != STRAGGLAR_SUM || !esize_of(dtype)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (count == 0) return STRAGGLAR_OK;
  if (!bufs) return STRAGGLAR_ERR_INVALID_ARG;
  for (int p = 0; p < g_team.world; ++p) {
    int st = check_args(bufs[p], count, dtype, op);
    if (st) return st;
  }
  return STRAGGLAR_OK;
}

int launch(int which, int dtype, const LaunchPlan& P, int nblocks, void* stream) {
  Comm& c = (g_team.active && P.state == g_team.state) ? g_team : g_proc;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;   // flags out of step: re-initialize
  if (which == K_COMPLETE || which == K_FUSED) c.last_slices = P.G * P.sub;
  cudaError_t e = launch_plan_kernel(which, dtype, P, nblocks, (cudaStream_t)stream);
  if (e != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

// team: Phase A over the non-stragglers (all in one launch)
int team_rs(void* const* bufs, size_t count, int dtype, void* stream) {
  Comm& c = g_team;
  LaunchPlan P = base_plan(c, count, dtype, false);
  stragglar_layout(c, P);
  for (int p = 0; p < c.world; ++p) P.buf[p] = (char*)bufs[p];
  int k = 0;
  for (int p = 0; p < c.world; ++p)
    if (p != c.sigma) P.local_rank[k++] = p;
  P.nlocal = k;
  return launch(K_RS, dtype, P, k * P.G * P.lanes, stream);
}

int team_b(void* const* bufs, size_t count, int dtype, void* stream, int which = K_COMPLETE, uint64_t delay_ns = 0) {
  Comm& c = g_team;
  LaunchPlan P = base_plan(c, count, dtype, true);
  if (which == K_COMPLETE || which == K_FUSED) stragglar_layout(c, P);
  P.sigma_delay_ns = delay_ns;
  for (int p = 0; p < c.world; ++p) {
    P.buf[p] = (char*)bufs[p];
    P.local_rank[p] = p;
  }
  P.nlocal = c.world;
  return launch(which, dtype, P, c.world * P.G * P.lanes, stream);
}

int read_error(Comm& c, int* code, uint32_t* where = nullptr) {
  if (!code) return STRAGGLAR_ERR_INVALID_ARG;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  CK(cudaDeviceSynchronize());
  DevState h;
  CK(cudaMemcpy(&h, c.state, sizeof(h), cudaMemcpyDeviceToHost));
  *code = (int)h.err;
  if (where) *where = h.err_info;
  // reported once from the device word; the host copy stays set, so every later
  // call on this communicator fails with TIMEOUT until it is re-initialized
  if (h.err) {
    uint32_t z[2] = {0, 0};
    CK(cudaMemcpy(c.state, z, sizeof(z), cudaMemcpyHostToDevice));
  }
  return h.err == ERR_TIMEOUT ? STRAGGLAR_ERR_TIMEOUT : STRAGGLAR_OK;
}

// Host-buffer entry points: because the SUM is elementwise, the buffers go
// through a three-stage pipeline of pieces: H2D of piece k+1 (copy engine, one
// direction), the AllReduce of piece k (SMs) and D2H of piece k-1 (copy
// engine, the other direction) overlap.  Pieces keep 16-byte alignment; every
// rank cuts the same pieces, so each piece's AllReduce is one collective call.
// Synchronous: returns after the last D2H landed.
//
// The pieces: equal, 16-byte aligned, the last one ragged.  (Ramping the first
// and last pieces down to 1/8 to shorten the pipeline's fill and drain was
// measured 0.5 % slower, profiles/r02/ab/r02y_e2e_ramp_ab.json.)  Pure host
// logic, the same on every rank for the same (count, dtype, piece).
std::vector<uint64_t> e2e_pieces(uint64_t count, int es, uint64_t piece_bytes) {
  const uint64_t v = 16 / es;
  uint64_t piece = piece_bytes / es / v * v;
  if (piece == 0) piece = v;
  std::vector<uint64_t> lens;
  for (uint64_t off = 0; off < count; off += piece) lens.push_back(count - off < piece ? count - off : piece);
  return lens;
}

template <class F>
int e2e_pipeline(int nbufs, const void* const* host_in, void* const* host_out, void* const* bufs, size_t count, int es,
                 cudaStream_t s, uint64_t piece_bytes, int ncs, F&& allreduce_piece) {
  const std::vector<uint64_t> lens = e2e_pieces(count, es, piece_bytes);
  const uint64_t npieces = lens.size();
  // copy streams per direction (several copy engines; buffers alternate between them)
  if (ncs < 1) ncs = 1;
  if (ncs > nbufs) ncs = nbufs;
  struct Res {                                      // released on every return path
    std::vector<cudaStream_t> h2d, d2h;
    std::vector<cudaEvent_t> ev;
    ~Res() {
      for (auto& e : ev)
        if (e) cudaEventDestroy(e);
      for (auto x : h2d)
        if (x) cudaStreamDestroy(x);
      for (auto x : d2h)
        if (x) cudaStreamDestroy(x);
    }
  } res;
  res.h2d.assign(ncs, nullptr);
  res.d2h.assign(ncs, nullptr);
  for (int i = 0; i < ncs; ++i) {
    CK(cudaStreamCreateWithFlags(&res.h2d[i], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&res.d2h[i], cudaStreamNonBlocking));
  }
  // events: per piece, one after each H2D stream, one after the AllReduce, one after each D2H stream
  const size_t per = 2 * ncs + 1;
  res.ev.assign(per * npieces + 1, nullptr);
  std::vector<cudaEvent_t>& ev = res.ev;
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventRecord(ev.back(), s));               // everything earlier on `stream` first
  for (int i = 0; i < ncs; ++i) CK(cudaStreamWaitEvent(res.h2d[i], ev.back(), 0));
  int st = STRAGGLAR_OK;
  uint64_t off = 0;
  for (uint64_t k = 0; k < npieces && st == STRAGGLAR_OK; off += lens[k], ++k) {
    const uint64_t n = lens[k];
    const size_t boff = off * es, bytes = n * es;
    cudaEvent_t* e = &ev[per * k];
    for (int p = 0; p < nbufs; ++p)
      CK(cudaMemcpyAsync((char*)bufs[p] + boff, (const char*)host_in[p] + boff, bytes, cudaMemcpyHostToDevice,
                         res.h2d[p % ncs]));
    for (int i = 0; i < ncs; ++i) {
      CK(cudaEventRecord(e[i], res.h2d[i]));
      CK(cudaStreamWaitEvent(s, e[i], 0));
    }
    st = allreduce_piece(off, n);
    CK(cudaEventRecord(e[ncs], s));
    for (int i = 0; i < ncs; ++i) CK(cudaStreamWaitEvent(res.d2h[i], e[ncs], 0));
    for (int p = 0; p < nbufs; ++p)
      CK(cudaMemcpyAsync((char*)host_out[p] + boff, (char*)bufs[p] + boff, bytes, cudaMemcpyDeviceToHost,
                         res.d2h[p % ncs]));
    for (int i = 0; i < ncs; ++i) CK(cudaEventRecord(e[ncs + 1 + i], res.d2h[i]));
  }
  if (npieces)
    for (int i = 0; i < ncs; ++i) CK(cudaStreamWaitEvent(s, ev[per * (npieces - 1) + ncs + 1 + i], 0));
  CK(cudaStreamSynchronize(s));
  return st;
}

// ---------------------------------------------------------------- driver API (NVLS)
// The library does not link libcuda: driver functions come through the runtime.
template <class F>
F drv(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return nullptr;
  return reinterpret_cast<F>(fn);
}
#define DRV(name) static auto p_##name = drv<decltype(&name)>(#name)
#define DCK(x)                                            \
  do {                                                    \
    if ((x) != CUDA_SUCCESS) return STRAGGLAR_ERR_CUDA;   \
  } while (0)

int map_va(size_t bytes, CUmemGenericAllocationHandle h, int dev, unsigned long long* va) {
  DRV(cuMemAddressReserve);
  DRV(cuMemMap);
  DRV(cuMemSetAccess);
  if (!p_cuMemAddressReserve || !p_cuMemMap || !p_cuMemSetAccess) return STRAGGLAR_ERR_CUDA;
  CUdeviceptr p = 0;
  DCK(p_cuMemAddressReserve(&p, bytes, 0, 0, 0));
  DCK(p_cuMemMap(p, bytes, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DCK(p_cuMemSetAccess(p, bytes, &acc, 1));
  *va = (unsigned long long)p;
  return STRAGGLAR_OK;
}

void unmap_va(unsigned long long& va, size_t bytes) {
  DRV(cuMemUnmap);
  DRV(cuMemAddressFree);
  if (va && p_cuMemUnmap && p_cuMemAddressFree) {
    p_cuMemUnmap((CUdeviceptr)va, bytes);
    p_cuMemAddressFree((CUdeviceptr)va, bytes);
  }
  va = 0;
}

void nvls_release(Comm& c) {
  auto& n = c.nvls;
  if (!n.stage) return;
  DRV(cuMemRelease);
  unmap_va(n.mc_all_va, n.bytes);
  unmap_va(n.mc_ns_va, n.bytes);
  unmap_va(n.sigma_va, n.bytes);
  unmap_va(n.va, n.bytes);
  for (unsigned long long* h : {&n.mc_all, &n.mc_ns, &n.sigma_mem, &n.mem})
    if (*h && p_cuMemRelease) p_cuMemRelease((CUmemGenericAllocationHandle)*h);
  for (int& fd : n.fds)
    if (fd >= 0) close(fd), fd = -1;
  n = Comm::Nvls();
}

int lowest_ns(const Comm& c) { return c.sigma == 0 ? 1 : 0; }

// NVLS variant: one slice per CTA, about one per slice_bytes of a chunk
int nvls_slices(const Comm& c, const LaunchPlan& P) {
  const uint64_t chunk_bytes = P.ce * P.esize, per = c.slice_bytes ? c.slice_bytes : 16384;
  uint64_t g = (chunk_bytes + per - 1) / per;
  if (g < 1) g = 1;
  return g < (uint64_t)c.G ? (int)g : c.G;
}

}  // namespace

extern "C" {

int stragglar_version(void) { return 100; }

const char* stragglar_status_string(int s) {
  switch (s) {
    case STRAGGLAR_OK: return "ok";
    case STRAGGLAR_ERR_INVALID_ARG: return "invalid argument";
    case STRAGGLAR_ERR_UNSUPPORTED: return "unsupported (world must be 2, 4, 6 or 8; dtype int32/float32/bfloat16; op SUM)";
    case STRAGGLAR_ERR_NOT_INITIALIZED: return "communicator not initialized (or peer handles not imported)";
    case STRAGGLAR_ERR_NOT_REGISTERED: return "buffer is not inside a registered, peer-mapped allocation";
    case STRAGGLAR_ERR_CUDA: return "CUDA error";
    case STRAGGLAR_ERR_TIMEOUT: return "device spin-wait timed out (a peer never arrived)";
    case STRAGGLAR_ERR_INTERNAL: return "internal error";
    default: return "unknown status";
  }
}

int stragglar_launch_count(uint64_t* n) {
  if (!n) return STRAGGLAR_ERR_INVALID_ARG;
  *n = g_launches.load();
  return STRAGGLAR_OK;
}

// ---------------------------------------------------------------- schedule
int stragglar_schedule_rounds(int world, int* rounds) {
  if (!rounds) return STRAGGLAR_ERR_INVALID_ARG;
  try {
    *rounds = (int)generate_any(world).size();
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_UNSUPPORTED;
  }
  return STRAGGLAR_OK;
}

int stragglar_schedule_round(int world, int round, int* out, int max_transfers, int* n_transfers) {
  if (!n_transfers || (!out && max_transfers > 0)) return STRAGGLAR_ERR_INVALID_ARG;
  try {
    auto s = generate_any(world);
    if (round < 0 || round >= (int)s.size()) return STRAGGLAR_ERR_INVALID_ARG;
    const auto& rd = s[round];
    *n_transfers = (int)rd.size();
    if ((int)rd.size() > max_transfers) return STRAGGLAR_ERR_INVALID_ARG;
    for (size_t i = 0; i < rd.size(); ++i) {
      out[4 * i + 0] = rd[i].src;
      out[4 * i + 1] = rd[i].dst;
      out[4 * i + 2] = rd[i].chunk;
      out[4 * i + 3] = rd[i].reduce ? 0 : 1;
    }
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_UNSUPPORTED;
  }
  return STRAGGLAR_OK;
}

// Host-only: the slice / sub-slice / op-lane layout a StragglAR call of this
// size would use, for a per-rank CTA budget and the default knobs (tests).
int stragglar_plan_layout(int world, int straggler_rank, size_t count, int dtype, int ctas_per_rank, int sys_scope,
                          int* slices, int* sub, int* lanes) {
  if (!slices || !sub || !lanes || ctas_per_rank < 1 || ctas_per_rank > kMaxSlices) return STRAGGLAR_ERR_INVALID_ARG;
  if (!supported_world(world)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (straggler_rank < 0 || straggler_rank >= world) return STRAGGLAR_ERR_INVALID_ARG;
  if (!esize_of(dtype)) return STRAGGLAR_ERR_UNSUPPORTED;
  Comm c;
  try {
    c.progs = build_programs(world, straggler_rank);
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_INTERNAL;
  }
  c.world = world;
  c.sigma = straggler_rank;
  c.G = c.G_alloc = ctas_per_rank;
  c.sys_scope = sys_scope ? 1 : 0;
  c.sub = kMaxSub;
  c.sub_bytes = 128 * 1024;
  LaunchPlan P = base_plan(c, count, dtype, true);
  stragglar_layout(c, P);
  *slices = P.G;
  *sub = P.sub;
  *lanes = P.lanes;
  return STRAGGLAR_OK;
}

int stragglar_plan_e2e_pieces(size_t count, int dtype, size_t piece_bytes, size_t* out, int max_pieces,
                              int* n_pieces) {
  if (!out || !n_pieces || max_pieces < 0) return STRAGGLAR_ERR_INVALID_ARG;
  const int es = esize_of(dtype);
  if (!es) return STRAGGLAR_ERR_UNSUPPORTED;
  const std::vector<uint64_t> lens = e2e_pieces(count, es, piece_bytes);
  if (lens.size() > (size_t)max_pieces) return STRAGGLAR_ERR_INVALID_ARG;
  for (size_t i = 0; i < lens.size(); ++i) out[i] = lens[i];
  *n_pieces = (int)lens.size();
  return STRAGGLAR_OK;
}

// ---------------------------------------------------------------- per-process communicator
int stragglar_init(int rank, int world, int straggler_rank) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_proc.active) common_finalize(g_proc);
  return common_init(g_proc, world, rank, straggler_rank, false);
}

int stragglar_handle_size(size_t* bytes) {
  if (!bytes) return STRAGGLAR_ERR_INVALID_ARG;
  *bytes = sizeof(IpcBlob);
  return STRAGGLAR_OK;
}

int device_uuid(int dev, char out[16]) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  std::memcpy(out, &prop.uuid, 16);
  return STRAGGLAR_OK;
}

int stragglar_export_handle(void* blob) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!blob) return STRAGGLAR_ERR_INVALID_ARG;
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  CK(cudaIpcGetMemHandle(&b.handle, g_proc.flags));
  b.offset = 0;
  b.bytes = g_proc.rank_bytes;
  b.layout = layout_of(g_proc);
  b.rank = g_proc.rank;
  b.resident_ctas = g_proc.resident;
  int st = device_uuid(g_proc.device, b.uuid);
  if (st) return st;
  std::memcpy(blob, &b, sizeof(b));
  return STRAGGLAR_OK;
}

int stragglar_import_handles(const void* blobs, int world) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!blobs || world != c.world) return STRAGGLAR_ERR_INVALID_ARG;
  const IpcBlob* b = static_cast<const IpcBlob*>(blobs);
  // every rank must run the same layout (slices, sub-slices, mover, scope,
  // straggler) and sit at its own index: reject before mapping anything
  const Layout mine = layout_of(c);
  for (int p = 0; p < world; ++p) {
    if (b[p].rank != p || b[p].bytes != c.rank_bytes) return STRAGGLAR_ERR_INVALID_ARG;
    if (std::memcmp(&b[p].layout, &mine, sizeof(Layout)) != 0) return STRAGGLAR_ERR_INVALID_ARG;
  }
  // Co-residency: ranks that share a GPU (several processes per device, e.g.
  // under MPS) must fit their cooperative grids side by side, or one rank's
  // CTAs cannot become resident while the others spin on its flags.  Every
  // rank derives the same CTA budget from the same blobs: the smallest
  // capacity / (ranks on that GPU) over the GPUs in use (the flag stride
  // stays G_alloc, so only the launch size changes).
  int G = c.G_alloc;
  for (int p = 0; p < world; ++p) {
    int share = 0;
    for (int q = 0; q < world; ++q) share += std::memcmp(b[p].uuid, b[q].uuid, 16) == 0;
    const int cap = b[p].resident_ctas / share;
    if (cap < G) G = cap;
    if (p == c.rank) c.share = share;
  }
  if (G < 1) return STRAGGLAR_ERR_UNSUPPORTED;
  for (int p = 0; p < world; ++p) {
    if (p == c.rank) continue;
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, b[p].handle, cudaIpcMemLazyEnablePeerAccess));
    c.opened.push_back(ptr);
    c.peer_flags[p] = reinterpret_cast<uint32_t*>(static_cast<char*>(ptr) + b[p].offset);
  }
  c.G = G;
  c.imported = true;
  return STRAGGLAR_OK;
}

int stragglar_shared_device_ranks(int* ranks_on_my_gpu, int* ctas_per_rank) {
  std::lock_guard<std::mutex> lk(g_mu);
  const Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!ranks_on_my_gpu || !ctas_per_rank) return STRAGGLAR_ERR_INVALID_ARG;
  *ranks_on_my_gpu = c.share;
  *ctas_per_rank = c.G;
  return STRAGGLAR_OK;
}

int stragglar_register_buffer(void* buf, size_t bytes, void* blob_out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!buf || !bytes || !blob_out) return STRAGGLAR_ERR_INVALID_ARG;
  // driver entry point through the runtime: the library does not link libcuda
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return STRAGGLAR_ERR_CUDA;
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)buf) != CUDA_SUCCESS) return STRAGGLAR_ERR_CUDA;
  if ((CUdeviceptr)buf + bytes > base + size) return STRAGGLAR_ERR_INVALID_ARG;
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  CK(cudaIpcGetMemHandle(&b.handle, (void*)base));
  b.offset = (uint64_t)((CUdeviceptr)buf - base);
  b.bytes = bytes;
  b.rank = g_proc.rank;
  std::memcpy(blob_out, &b, sizeof(b));
  return STRAGGLAR_OK;
}

int stragglar_import_buffer(void* buf, const void* blobs, int world) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!buf || !blobs || world != c.world) return STRAGGLAR_ERR_INVALID_ARG;
  const IpcBlob* b = static_cast<const IpcBlob*>(blobs);
  Registration r;
  r.local = static_cast<char*>(buf);
  r.bytes = b[c.rank].bytes;
  for (int p = 0; p < world; ++p)   // ranks registered different sizes, or blobs out of rank order
    if (b[p].bytes != r.bytes || b[p].rank != p) return STRAGGLAR_ERR_INVALID_ARG;
  for (int p = 0; p < world; ++p) {
    if (p == c.rank) {
      r.peer[p] = r.local;
      continue;
    }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, b[p].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      for (int q = 0; q < p; ++q)
        if (r.mapped[q]) cudaIpcCloseMemHandle(r.mapped[q]);
      return STRAGGLAR_ERR_CUDA;
    }
    r.mapped[p] = ptr;
    r.peer[p] = static_cast<char*>(ptr) + b[p].offset;
  }
  c.regs.push_back(r);
  return STRAGGLAR_OK;
}

int stragglar_deregister_buffer(void* buf) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  for (size_t i = c.regs.size(); i-- > 0;) {
    if (c.regs[i].local != buf) continue;
    CK(cudaDeviceSynchronize());   // no call of this process still uses the mappings
    for (int p = 0; p < c.world; ++p)
      if (c.regs[i].mapped[p]) cudaIpcCloseMemHandle(c.regs[i].mapped[p]);
    c.regs.erase(c.regs.begin() + i);
    return STRAGGLAR_OK;
  }
  return STRAGGLAR_ERR_NOT_REGISTERED;
}

static int proc_plan(void* buf, size_t count, int dtype, LaunchPlan* P) {
  Comm& c = g_proc;
  const size_t bytes = count * esize_of(dtype);
  const Registration* reg = nullptr;
  for (const auto& r : c.regs)
    if ((char*)buf >= r.local && (char*)buf + bytes <= r.local + r.bytes) reg = &r;
  if (!reg) return STRAGGLAR_ERR_NOT_REGISTERED;
  const size_t delta = (char*)buf - reg->local;
  *P = base_plan(c, count, dtype, true);
  for (int p = 0; p < c.world; ++p) P->buf[p] = reg->peer[p] + delta;
  P->nlocal = 1;
  P->local_rank[0] = c.rank;
  return STRAGGLAR_OK;
}

int stragglar_allreduce(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;
  // one persistent launch: non-stragglers run Phase A then Phase B, the
  // straggler Phase B only (its delay is whatever precedes it on its stream)
  stragglar_layout(c, P);
  return launch(K_FUSED, dtype, P, P.G * P.lanes, stream);
}

int stragglar_allreduce_direct(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;
  return launch(K_FUSED_DIRECT, dtype, P, P.G, stream);
}

int stragglar_allreduce_ring(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;
  P.ce = chunk_elems(count, c.world, P.esize);
  P.nchunks = c.world;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub, true);
  P.sub_major = c.base_sub_major;
  return launch(K_RING, dtype, P, P.G, stream);
}

int stragglar_allreduce_rhd(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (c.world & (c.world - 1)) return STRAGGLAR_ERR_UNSUPPORTED;   // RHD needs a power of two
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;
  P.ce = chunk_elems(count, c.world, P.esize);
  P.nchunks = c.world;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub, true);
  P.sub_major = c.base_sub_major;
  return launch(K_RHD, dtype, P, P.G, stream);
}

int stragglar_allreduce_bcast(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;
  return launch(K_BCAST, dtype, P, P.G, stream);
}

int stragglar_broadcast_tree(int world, int* sender, int* round) {
  if (!sender || !round) return STRAGGLAR_ERR_INVALID_ARG;
  try {
    broadcast_tree(world, sender, round);
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_UNSUPPORTED;
  }
  return STRAGGLAR_OK;
}

int stragglar_select(int world, double bytes, double delay_s, double alpha_s, double beta, int* use_stragglar,
                     double* critical_delay_s) {
  if (world < 2 || world > 64 || (world & 1)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (!(bytes >= 0) || !(alpha_s >= 0) || !(beta >= 0)) return STRAGGLAR_ERR_INVALID_ARG;
  double Rr;
  try {
    Rr = (double)generate_any(world).size();     // n + log2 n - 2 for powers of two (Thm 1)
  } catch (const std::exception&) {
    return STRAGGLAR_ERR_UNSUPPORTED;
  }
  const double n = world, R = Rr;
  const double t_rs = (world > 2 ? alpha_s : 0.0) + (n - 2) / (n - 1) * bytes * beta;
  const double t_sar = R * alpha_s + R / (n - 1) * bytes * beta;
  const double t_ring = 2 * (n - 1) * alpha_s + 2 * (n - 1) / n * bytes * beta;
  const double gain = t_ring - t_sar > 0 ? t_ring - t_sar : 0.0;
  double crit = t_rs - gain;
  if (crit < 0) crit = 0;
  if (critical_delay_s) *critical_delay_s = crit;
  if (use_stragglar) *use_stragglar = delay_s >= crit ? 1 : 0;
  return STRAGGLAR_OK;
}

int stragglar_select_algorithm(int world, double bytes, double delay_s, double alpha_s, double beta, int* algo,
                               double* t_pred_s) {
  if (!algo) return STRAGGLAR_ERR_INVALID_ARG;
  double crit = 0.0;
  int use = 0;
  int st = stragglar_select(world, bytes, delay_s, alpha_s, beta, &use, &crit);
  if (st) return st;
  // completion from the non-stragglers' start: StragglAR hides its
  // ReduceScatter in the delay; the bulk-synchronous baselines start after it
  const double n = world, R = (double)generate_any(world).size();
  const double t_rs = (world > 2 ? alpha_s : 0.0) + (n - 2) / (n - 1) * bytes * beta;
  const double t_sar = (delay_s > t_rs ? delay_s : t_rs) + R * alpha_s + R / (n - 1) * bytes * beta;
  const double t_ring = delay_s + 2 * (n - 1) * alpha_s + 2 * (n - 1) / n * bytes * beta;
  double best = t_sar;
  int a = STRAGGLAR_ALGO_STRAGGLAR;
  if (t_ring < best) {
    best = t_ring;
    a = STRAGGLAR_ALGO_RING;
  }
  if ((world & (world - 1)) == 0) {
    int L = 0;
    while ((1 << L) < world) ++L;
    const double t_rhd = delay_s + 2 * L * alpha_s + 2 * (n - 1) / n * bytes * beta;
    if (t_rhd < best) {
      best = t_rhd;
      a = STRAGGLAR_ALGO_RHD;
    }
  }
  *algo = a;
  if (t_pred_s) *t_pred_s = best;
  return STRAGGLAR_OK;
}

int stragglar_set_cost_model(double alpha_s, double beta) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!(alpha_s >= 0) || !(beta > 0)) return STRAGGLAR_ERR_INVALID_ARG;
  g_proc.alpha_s = alpha_s;
  g_proc.beta_s_per_byte = beta;
  return STRAGGLAR_OK;
}

int stragglar_allreduce_auto(void* buf, size_t count, int dtype, int op, void* stream, uint64_t expected_delay_ns,
                             int* used_algorithm) {
  double a, b;
  int world;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
    a = g_proc.alpha_s;
    b = g_proc.beta_s_per_byte;
    world = g_proc.world;
  }
  const int es = esize_of(dtype);
  if (!es) return STRAGGLAR_ERR_UNSUPPORTED;
  int algo = STRAGGLAR_ALGO_STRAGGLAR;
  int st = stragglar_select_algorithm(world, (double)count * es, expected_delay_ns * 1e-9, a, b, &algo, nullptr);
  if (st) return st;
  if (used_algorithm) *used_algorithm = algo;
  switch (algo) {
    case STRAGGLAR_ALGO_RING: return stragglar_allreduce_ring(buf, count, dtype, op, stream);
    case STRAGGLAR_ALGO_RHD: return stragglar_allreduce_rhd(buf, count, dtype, op, stream);
    default: return stragglar_allreduce(buf, count, dtype, op, stream);
  }
}

int stragglar_barrier(void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;
  LaunchPlan P = base_plan(c, 0, STRAGGLAR_INT32, true);
  P.nlocal = 1;
  P.local_rank[0] = c.rank;
  if (launch_barrier(P, (cudaStream_t)stream) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

// ---------------------------------------------------------------- K0 probes
int stragglar_probe_copy(void* buf, size_t bytes_per_peer, int mode, uint32_t peer_mask, int ctas, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;
  if (!buf || bytes_per_peer == 0 || bytes_per_peer % 16 || (mode & ~3)) return STRAGGLAR_ERR_INVALID_ARG;
  const size_t need = bytes_per_peer * (size_t)c.world;
  const Registration* reg = nullptr;
  for (const auto& r : c.regs)
    if ((char*)buf >= r.local && (char*)buf + need <= r.local + r.bytes) reg = &r;
  if (!reg) return STRAGGLAR_ERR_NOT_REGISTERED;
  const size_t delta = (char*)buf - reg->local;
  ProbeArgs A;
  std::memset(&A, 0, sizeof(A));
  A.local = (char*)buf;
  A.bytes = bytes_per_peer;
  A.me = c.rank;
  A.pull = mode & 1;
  for (int p = 0; p < c.world; ++p) {
    A.peer[p] = reg->peer[p] + delta;
    if (p != c.rank && ((peer_mask >> p) & 1u)) A.peers[A.npeers++] = p;
  }
  if (A.npeers == 0) return STRAGGLAR_ERR_INVALID_ARG;
  int n = ctas > 0 ? ctas : c.G;
  n = (n + A.npeers - 1) / A.npeers * A.npeers;   // every peer served by the same number of CTAs
  const int mover = (mode & 2) ? MOVER_TMA : MOVER_LSU;
  if (launch_probe_copy(A, mover, n, (cudaStream_t)stream) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_probe_pingpong(int peer, int iters, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;
  if (peer < 0 || peer >= c.world || peer == c.rank || iters < 1) return STRAGGLAR_ERR_INVALID_ARG;
  uint32_t* mine = c.peer_flags[c.rank] + (size_t)SLOT_PROBE * c.G_alloc * kMaxSub;
  uint32_t* theirs = c.peer_flags[peer] + (size_t)SLOT_PROBE * c.G_alloc * kMaxSub;
  if (launch_probe_pingpong(mine, theirs, c.rank < peer ? 1 : 0, iters, c.state, c.timeout_ns, c.host_err_dev,
                            (cudaStream_t)stream) != cudaSuccess)
    return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_probe_pingpong_result(double* us) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!us) return STRAGGLAR_ERR_INVALID_ARG;
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  CK(cudaDeviceSynchronize());
  DevState h;
  CK(cudaMemcpy(&h, g_proc.state, sizeof(h), cudaMemcpyDeviceToHost));
  if (h.err) return STRAGGLAR_ERR_TIMEOUT;
  *us = h.probe_ns * 1e-3;
  return STRAGGLAR_OK;
}

int stragglar_inject_delay(uint64_t ns, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (launch_delay(nullptr, ns, g_proc.state, (cudaStream_t)stream) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_last_barrier_ns(uint64_t* ns) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!ns) return STRAGGLAR_ERR_INVALID_ARG;
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  CK(cudaDeviceSynchronize());
  DevState h;
  CK(cudaMemcpy(&h, g_proc.state, sizeof(h), cudaMemcpyDeviceToHost));
  *ns = h.t_barrier;
  return STRAGGLAR_OK;
}

int stragglar_check_error(int* code) {
  std::lock_guard<std::mutex> lk(g_mu);
  return read_error(g_proc, code);
}

int stragglar_phase_times(double* t_a_us, double* t_total_us) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!t_a_us || !t_total_us) return STRAGGLAR_ERR_INVALID_ARG;
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  CK(cudaDeviceSynchronize());
  DevState h;
  CK(cudaMemcpy(&h, g_proc.state, sizeof(h), cudaMemcpyDeviceToHost));
  const uint64_t* t = h.stamp[h.epoch & 1u];   // the last completed call
  if (h.epoch == 0 || t[0] == ~0ull || t[2] < t[0]) return STRAGGLAR_ERR_INVALID_ARG;   // not a fused call
  *t_a_us = (t[1] - t[0]) * 1e-3;
  *t_total_us = (t[2] - t[0]) * 1e-3;
  return STRAGGLAR_OK;
}

int stragglar_check_error_where(int team, int* code, uint32_t* where) {
  std::lock_guard<std::mutex> lk(g_mu);
  return read_error(team ? g_team : g_proc, code, where);
}

int stragglar_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  common_finalize(g_proc);
  return STRAGGLAR_OK;
}

// ---------------------------------------------------------------- NEXT N1(i): NVLS multicast (nvls.cu)
int stragglar_nvls_supported(int* supported) {
  if (!supported) return STRAGGLAR_ERR_INVALID_ARG;
  *supported = 0;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  DRV(cuDeviceGetAttribute);
  if (!p_cuDeviceGetAttribute) return STRAGGLAR_ERR_CUDA;
  int v = 0;
  DCK(p_cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  *supported = v;
  return STRAGGLAR_OK;
}

int stragglar_nvls_begin(size_t bytes, int* fds, size_t* bytes_out) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!fds || !bytes_out || !bytes) return STRAGGLAR_ERR_INVALID_ARG;
  if (c.nvls.stage) return STRAGGLAR_ERR_INVALID_ARG;          // one arena per communicator
  DRV(cuMulticastGetGranularity);
  DRV(cuMemGetAllocationGranularity);
  DRV(cuMemCreate);
  DRV(cuMemExportToShareableHandle);
  DRV(cuMulticastCreate);
  if (!p_cuMulticastGetGranularity || !p_cuMemCreate || !p_cuMulticastCreate) return STRAGGLAR_ERR_UNSUPPORTED;
  auto& n = c.nvls;
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)c.world;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g_mc = 0, g_mem = 0;
  DCK(p_cuMulticastGetGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c.device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  DCK(p_cuMemGetAllocationGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = g_mc > g_mem ? g_mc : g_mem;
  n.bytes = (bytes + g - 1) / g * g;
  mp.size = n.bytes;
  CUmemGenericAllocationHandle h = 0;
  n.stage = 1;
  auto fail = [&](int st) {
    nvls_release(c);
    return st;
  };
  if (p_cuMemCreate(&h, n.bytes, &ap, 0) != CUDA_SUCCESS) return fail(STRAGGLAR_ERR_CUDA);
  n.mem = h;
  int st = map_va(n.bytes, h, c.device, &n.va);
  if (st) return fail(st);
  if (p_cuMemExportToShareableHandle(&n.fds[2], h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
    return fail(STRAGGLAR_ERR_CUDA);
  if (c.rank == 0) {   // the all-rank multicast object
    CUmemGenericAllocationHandle m = 0;
    if (p_cuMulticastCreate(&m, &mp) != CUDA_SUCCESS) return fail(STRAGGLAR_ERR_CUDA);
    n.mc_all = m;
    if (p_cuMemExportToShareableHandle(&n.fds[0], m, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
      return fail(STRAGGLAR_ERR_CUDA);
  }
  if (c.rank == lowest_ns(c)) {   // the non-stragglers' multicast object
    CUmulticastObjectProp mq = mp;
    mq.numDevices = (unsigned)(c.world - 1);
    CUmemGenericAllocationHandle m = 0;
    if (p_cuMulticastCreate(&m, &mq) != CUDA_SUCCESS) return fail(STRAGGLAR_ERR_CUDA);
    n.mc_ns = m;
    if (p_cuMemExportToShareableHandle(&n.fds[1], m, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
      return fail(STRAGGLAR_ERR_CUDA);
  }
  for (int i = 0; i < 3; ++i) fds[i] = n.fds[i];
  *bytes_out = n.bytes;
  return STRAGGLAR_OK;
}

int stragglar_nvls_import(int mc_all_fd, int mc_ns_fd, int sigma_mem_fd) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  auto& n = c.nvls;
  if (!c.active || n.stage != 1) return STRAGGLAR_ERR_NOT_INITIALIZED;
  DRV(cuMemImportFromShareableHandle);
  if (!p_cuMemImportFromShareableHandle) return STRAGGLAR_ERR_UNSUPPORTED;
  auto import = [&](int fd, unsigned long long* h) {
    CUmemGenericAllocationHandle x = 0;
    if (fd < 0) return STRAGGLAR_ERR_INVALID_ARG;
    if (p_cuMemImportFromShareableHandle(&x, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
        CUDA_SUCCESS)
      return STRAGGLAR_ERR_CUDA;
    *h = x;
    return STRAGGLAR_OK;
  };
  int st;
  const bool ns = c.rank != c.sigma;
  if ((!n.mc_all && (st = import(mc_all_fd, &n.mc_all))) || (ns && !n.mc_ns && (st = import(mc_ns_fd, &n.mc_ns))) ||
      (ns && (st = import(sigma_mem_fd, &n.sigma_mem)))) {
    nvls_release(c);
    return st;
  }
  n.stage = 2;
  return STRAGGLAR_OK;
}

int stragglar_nvls_bind(void** arena) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  auto& n = c.nvls;
  if (!c.active || n.stage != 2) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!arena) return STRAGGLAR_ERR_INVALID_ARG;
  DRV(cuMulticastAddDevice);
  DRV(cuMulticastBindMem);
  DRV(cuDeviceGet);
  if (!p_cuMulticastAddDevice || !p_cuMulticastBindMem || !p_cuDeviceGet) return STRAGGLAR_ERR_UNSUPPORTED;
  auto fail = [&](int st) {
    nvls_release(c);
    return st;
  };
  CUdevice dev;
  if (p_cuDeviceGet(&dev, c.device) != CUDA_SUCCESS) return fail(STRAGGLAR_ERR_CUDA);
  const bool ns = c.rank != c.sigma;
  // every member joins before any binds (a bind waits for the whole team)
  if (p_cuMulticastAddDevice((CUmemGenericAllocationHandle)n.mc_all, dev) != CUDA_SUCCESS) return fail(STRAGGLAR_ERR_CUDA);
  if (ns && p_cuMulticastAddDevice((CUmemGenericAllocationHandle)n.mc_ns, dev) != CUDA_SUCCESS)
    return fail(STRAGGLAR_ERR_CUDA);
  if (p_cuMulticastBindMem((CUmemGenericAllocationHandle)n.mc_all, 0, (CUmemGenericAllocationHandle)n.mem, 0, n.bytes,
                           0) != CUDA_SUCCESS)
    return fail(STRAGGLAR_ERR_CUDA);
  if (ns && p_cuMulticastBindMem((CUmemGenericAllocationHandle)n.mc_ns, 0, (CUmemGenericAllocationHandle)n.mem, 0,
                                 n.bytes, 0) != CUDA_SUCCESS)
    return fail(STRAGGLAR_ERR_CUDA);
  int st;
  if ((st = map_va(n.bytes, (CUmemGenericAllocationHandle)n.mc_all, c.device, &n.mc_all_va))) return fail(st);
  if (ns) {
    if ((st = map_va(n.bytes, (CUmemGenericAllocationHandle)n.mc_ns, c.device, &n.mc_ns_va))) return fail(st);
    // owners read the straggler's input through a unicast peer mapping of its arena
    if ((st = map_va(n.bytes, (CUmemGenericAllocationHandle)n.sigma_mem, c.device, &n.sigma_va))) return fail(st);
  }
  n.stage = 3;
  *arena = (void*)n.va;
  return STRAGGLAR_OK;
}

int stragglar_nvls_release(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  cudaDeviceSynchronize();
  nvls_release(g_proc);
  return STRAGGLAR_OK;
}

int stragglar_allreduce_nvls(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  auto& n = c.nvls;
  if (!c.active || !c.imported || n.stage != 3) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  const int es = esize_of(dtype);
  if (count % (16 / es)) return STRAGGLAR_ERR_INVALID_ARG;             // whole 16-byte vectors only
  const char* lo = (const char*)n.va;
  if ((const char*)buf < lo || (const char*)buf + count * es > lo + n.bytes) return STRAGGLAR_ERR_NOT_REGISTERED;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;
  const size_t off = (const char*)buf - lo;
  LaunchPlan P = base_plan(c, count, dtype, true);
  P.nlocal = 1;
  P.local_rank[0] = c.rank;
  P.sub = 1;
  P.G = nvls_slices(c, P);                     // one slice per CTA
  P.buf[c.rank] = (char*)buf;
  P.mc_all = (char*)n.mc_all_va + off;
  P.mc_ns = n.mc_ns_va ? (char*)n.mc_ns_va + off : nullptr;
  P.sigma_uc = n.sigma_va ? (char*)n.sigma_va + off : nullptr;
  if (launch_nvls(dtype, P, P.G, (cudaStream_t)stream, false) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_allreduce_nvls_emulated(void* buf, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
  int st = check_args(buf, count, dtype, op);
  if (st || count == 0) return st;
  if (count % (16 / esize_of(dtype))) return STRAGGLAR_ERR_INVALID_ARG;
  if (sticky_error(c)) return STRAGGLAR_ERR_TIMEOUT;
  LaunchPlan P;
  if ((st = proc_plan(buf, count, dtype, &P))) return st;   // registered: P.buf[p] = every rank's copy
  P.sub = 1;
  P.G = nvls_slices(c, P);
  if (launch_nvls(dtype, P, P.G, (cudaStream_t)stream, true) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_nvls_selftest(int dtype, size_t count, const void* host_in, void* host_out) {
  // a one-member multicast object on the current device: out = ld_reduce(in) through it
  const int es = esize_of(dtype);
  if (!es || !host_in || !host_out || !count || count % (16 / es)) return STRAGGLAR_ERR_INVALID_ARG;
  int sup = 0;
  int st = stragglar_nvls_supported(&sup);
  if (st) return st;
  if (!sup) return STRAGGLAR_ERR_UNSUPPORTED;
  DRV(cuMulticastGetGranularity);
  DRV(cuMemGetAllocationGranularity);
  DRV(cuMemCreate);
  DRV(cuMulticastCreate);
  DRV(cuMulticastAddDevice);
  DRV(cuMulticastBindMem);
  DRV(cuMemRelease);
  DRV(cuDeviceGet);
  int devi = 0;
  CK(cudaGetDevice(&devi));
  CUdevice dev;
  DCK(p_cuDeviceGet(&dev, devi));
  const size_t bytes = count * es;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = 2 * bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t g_mc = 0, g_mem = 0;
  DCK(p_cuMulticastGetGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = devi;
  DCK(p_cuMemGetAllocationGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = g_mc > g_mem ? g_mc : g_mem;
  const size_t size = (2 * bytes + g - 1) / g * g;
  mp.size = size;
  CUmemGenericAllocationHandle mem = 0, mc = 0;
  unsigned long long va = 0, mcva = 0;
  st = STRAGGLAR_ERR_CUDA;
  if (p_cuMemCreate(&mem, size, &ap, 0) != CUDA_SUCCESS) return STRAGGLAR_ERR_CUDA;
  // A GPU can report multicast support and still have no usable multicast
  // object (no NVSwitch fabric behind it: this one-GPU box answers
  // CUDA_ERROR_INVALID_VALUE for any member count): that is UNSUPPORTED here.
  if (p_cuMulticastCreate(&mc, &mp) != CUDA_SUCCESS) {
    p_cuMemRelease(mem);
    return STRAGGLAR_ERR_UNSUPPORTED;
  }
  if (p_cuMulticastAddDevice(mc, dev) == CUDA_SUCCESS && p_cuMulticastBindMem(mc, 0, mem, 0, size, 0) == CUDA_SUCCESS &&
      map_va(size, mem, devi, &va) == STRAGGLAR_OK && map_va(size, mc, devi, &mcva) == STRAGGLAR_OK &&
      cudaMemcpy((void*)va, host_in, bytes, cudaMemcpyHostToDevice) == cudaSuccess &&
      cudaMemset((char*)va + bytes, 0, bytes) == cudaSuccess &&
      launch_nvls_selftest(dtype, (char*)mcva, bytes, 0) == cudaSuccess &&
      cudaDeviceSynchronize() == cudaSuccess &&
      cudaMemcpy(host_out, (char*)va + bytes, bytes, cudaMemcpyDeviceToHost) == cudaSuccess)
    st = STRAGGLAR_OK;
  unmap_va(mcva, size);
  unmap_va(va, size);
  if (mc) p_cuMemRelease(mc);
  if (mem) p_cuMemRelease(mem);
  return st;
}

// ---------------------------------------------------------------- team
int stragglar_team_init(int world, int straggler_rank) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_team.active) common_finalize(g_team);
  return common_init(g_team, world, -1, straggler_rank, true);
}

int stragglar_team_slices(int* slices) {
  if (!slices) return STRAGGLAR_ERR_INVALID_ARG;
  if (!g_team.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  *slices = g_team.G;
  return STRAGGLAR_OK;
}

}  // extern "C"

namespace {
// The split team calls (reduce_scatter -> complete*, bcast_precondition ->
// bcast_complete) share one call epoch: a completion must run on exactly the
// buffers, count and dtype of its pending first half, or flags written under
// another slice layout would satisfy its waits.
void team_pend(Comm& c, void* const* bufs, size_t count, int dtype) {
  c.rs_buf0 = bufs[0];
  c.rs_count = count;
  c.rs_dtype = dtype;
}
bool team_matches(const Comm& c, void* const* bufs, size_t count, int dtype) {
  return c.rs_buf0 == bufs[0] && c.rs_count == count && c.rs_dtype == dtype;
}
}  // namespace

extern "C" {

int stragglar_team_reduce_scatter(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  if ((st = team_rs(bufs, count, dtype, stream))) return st;
  g_team.rs_pending = true;
  team_pend(g_team, bufs, count, dtype);
  return STRAGGLAR_OK;
}

int stragglar_team_complete(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (!g_team.rs_pending || !team_matches(g_team, bufs, count, dtype))
    return STRAGGLAR_ERR_INVALID_ARG;   // Phase B needs its own Phase A
  g_team.rs_pending = false;
  return team_b(bufs, count, dtype, stream);
}

int stragglar_team_allreduce(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;   // finish the pending Phase A first
  return team_b(bufs, count, dtype, stream, K_FUSED);        // Phase A + B in one launch
}

int stragglar_team_complete_direct(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (!g_team.rs_pending || !team_matches(g_team, bufs, count, dtype)) return STRAGGLAR_ERR_INVALID_ARG;
  g_team.rs_pending = false;
  return team_b(bufs, count, dtype, stream, K_DIRECT);
}

int stragglar_team_allreduce_direct(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  return team_b(bufs, count, dtype, stream, K_FUSED_DIRECT);
}

int stragglar_team_allreduce_delayed(void* const* bufs, size_t count, int dtype, int op, uint64_t delay_ns,
                                     void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  return team_b(bufs, count, dtype, stream, K_FUSED, delay_ns);
}

int stragglar_team_allreduce_ring(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  Comm& c = g_team;
  if (c.rs_pending || c.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;   // a Phase A awaits its Phase B
  LaunchPlan P = base_plan(c, count, dtype, true);
  P.ce = chunk_elems(count, c.world, P.esize);
  P.nchunks = c.world;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub, true);
  P.sub_major = c.base_sub_major;
  for (int p = 0; p < c.world; ++p) {
    P.buf[p] = (char*)bufs[p];
    P.local_rank[p] = p;
  }
  P.nlocal = c.world;
  return launch(K_RING, dtype, P, c.world * P.G, stream);
}

int stragglar_team_allreduce_rhd(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  Comm& c = g_team;
  if (c.world & (c.world - 1)) return STRAGGLAR_ERR_UNSUPPORTED;
  if (c.rs_pending || c.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  LaunchPlan P = base_plan(c, count, dtype, true);
  P.ce = chunk_elems(count, c.world, P.esize);
  P.nchunks = c.world;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub, true);
  P.sub_major = c.base_sub_major;
  for (int p = 0; p < c.world; ++p) {
    P.buf[p] = (char*)bufs[p];
    P.local_rank[p] = p;
  }
  P.nlocal = c.world;
  return launch(K_RHD, dtype, P, c.world * P.G, stream);
}

// Broadcast baseline in team mode: the precondition (non-straggler AllReduce,
// launched for the n-1 non-stragglers only), the completion (exchange +
// doubling copies, all ranks) or both in one launch.
int stragglar_team_bcast_precondition(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  Comm& c = g_team;
  if (c.rs_pending || c.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  LaunchPlan P = base_plan(c, count, dtype, false);
  for (int p = 0; p < c.world; ++p) P.buf[p] = (char*)bufs[p];
  int k = 0;
  for (int p = 0; p < c.world; ++p)
    if (p != c.sigma) P.local_rank[k++] = p;
  P.nlocal = k;
  if ((st = launch(K_BCAST_A, dtype, P, k * P.G, stream))) return st;
  c.bc_pending = true;
  team_pend(c, bufs, count, dtype);
  return STRAGGLAR_OK;
}

int stragglar_team_bcast_complete(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (!g_team.bc_pending || !team_matches(g_team, bufs, count, dtype))
    return STRAGGLAR_ERR_INVALID_ARG;   // needs its own precondition
  g_team.bc_pending = false;
  return team_b(bufs, count, dtype, stream, K_BCAST_B);
}

int stragglar_team_allreduce_bcast(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  return team_b(bufs, count, dtype, stream, K_BCAST);
}

int stragglar_team_inject_delay(uint64_t ns, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_team.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (launch_delay(&g_team.state->t_rs_start, ns, g_team.state, (cudaStream_t)stream) != cudaSuccess)
    return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_team_allreduce_host(const void* const* host_in, void* const* host_out, void* const* bufs,
                                  size_t count, int dtype, int op, void* stream) {
  if (!host_in || !host_out) return STRAGGLAR_ERR_INVALID_ARG;
  int st;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if ((st = team_check(bufs, count, dtype, op))) return st;
  }
  if (count == 0) return STRAGGLAR_OK;
  const int world = g_team.world;
  for (int p = 0; p < world; ++p)
    if (!host_in[p] || !host_out[p]) return STRAGGLAR_ERR_INVALID_ARG;
  const int es = esize_of(dtype);
  std::vector<void*> sub(world);
  return e2e_pipeline(world, host_in, host_out, bufs, count, es, (cudaStream_t)stream, g_team.e2e_piece_bytes,
                      g_team.e2e_streams, [&](uint64_t off, uint64_t n) {
                        for (int p = 0; p < world; ++p) sub[p] = (char*)bufs[p] + off * es;
                        return stragglar_team_allreduce(sub.data(), n, dtype, op, stream);
                      });
}

int stragglar_allreduce_host(const void* host_in, void* host_out, void* buf, size_t count, int dtype, int op,
                             void* stream) {
  int st;
  uint64_t piece;
  int ncs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    Comm& c = g_proc;
    if (!c.active || !c.imported) return STRAGGLAR_ERR_NOT_INITIALIZED;
    if ((st = check_args(buf, count, dtype, op))) return st;
    if (count == 0) return STRAGGLAR_OK;
    if (!host_in || !host_out) return STRAGGLAR_ERR_INVALID_ARG;
    LaunchPlan P;
    if ((st = proc_plan(buf, count, dtype, &P))) return st;   // the whole range must be registered
    piece = c.e2e_piece_bytes;
    ncs = c.e2e_streams;
  }
  const int es = esize_of(dtype);
  const void* hin[1] = {host_in};
  void* hout[1] = {host_out};
  void* b[1] = {buf};
  return e2e_pipeline(1, hin, hout, b, count, es, (cudaStream_t)stream, piece, ncs, [&](uint64_t off, uint64_t n) {
    return stragglar_allreduce((char*)buf + off * es, n, dtype, op, stream);
  });
}

int stragglar_team_set_trace(int enable) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_team;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (c.trace) {
    cudaDeviceSynchronize();
    cudaFree(c.trace);
    c.trace = nullptr;
  }
  if (!enable) return STRAGGLAR_OK;
  const size_t n = (size_t)c.world * c.G * kMaxSub * kMaxOps * 3;
  CK(cudaMalloc(&c.trace, n * sizeof(uint64_t)));
  CK(cudaMemset(c.trace, 0, n * sizeof(uint64_t)));
  return STRAGGLAR_OK;
}

int stragglar_team_read_trace(uint64_t* out, size_t max_entries, size_t* n_entries, int* slices) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_team;
  if (!c.active || !c.trace) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!n_entries || !slices) return STRAGGLAR_ERR_INVALID_ARG;
  const size_t n = (size_t)c.world * c.last_slices * kMaxOps * 3;
  *n_entries = n;
  *slices = c.last_slices;
  if (!out || max_entries < n) return STRAGGLAR_ERR_INVALID_ARG;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, c.trace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return STRAGGLAR_OK;
}

int stragglar_team_check_error(int* code) {
  std::lock_guard<std::mutex> lk(g_mu);
  return read_error(g_team, code);
}

int stragglar_team_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  common_finalize(g_team);
  return STRAGGLAR_OK;
}

}  // extern "C"
