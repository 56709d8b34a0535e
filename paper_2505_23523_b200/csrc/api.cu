// C ABI of libstragglar.so (declared in include/stragglar.h).
//
// Host side only: argument checks, the per-rank schedule programs, IPC handle
// plumbing, flag/epoch management and kernel launches.  No data is touched on
// the host; every step of the collective runs in kernels.cu.
#include <cuda.h>
#include <cuda_runtime.h>

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
}  // namespace stragglar

using namespace stragglar;

namespace {

enum { K_RS = 0, K_COMPLETE = 1, K_RING = 2, K_DIRECT = 3, K_FUSED = 4, K_FUSED_DIRECT = 5,
       K_BCAST_A = 6, K_BCAST_B = 7, K_BCAST = 8, K_RHD = 9, K_NUM = 10 };
constexpr int kDefaultMover = MOVER_TMA;   // measured faster (profiles/r01)

std::atomic<uint64_t> g_launches{0};

struct IpcBlob {          // what travels between processes, per rank
  cudaIpcMemHandle_t handle;
  uint64_t offset;        // of the registered pointer inside its allocation
  uint64_t bytes;
};

struct Registration {
  char* local = nullptr;
  size_t bytes = 0;
  char* peer[kMaxWorld] = {nullptr};
};

struct Comm {
  bool active = false;
  bool team = false;
  int world = 0, rank = -1, sigma = -1, device = -1;
  int G = 0;                   // CTAs per rank (the launch's co-residency budget)
  int sub = 1;                 // slices per CTA at most (STRAGGLAR_SUBSLICES)
  uint64_t sub_bytes = 0;      // target slice size on large messages (STRAGGLAR_SUBSLICE_BYTES)
  bool rs_pending = false;     // team: a Phase A awaits its Phase B (same call epoch)
  bool bc_pending = false;     // team: a Broadcast-baseline precondition awaits its completion
  uint32_t* flags = nullptr;   // own flag array(s) + LL area(s); team: world of them back to back
  uint32_t* peer_flags[kMaxWorld] = {nullptr};
  uint64_t* peer_ll[kMaxWorld] = {nullptr};
  size_t flags_bytes = 0;      // per rank, before its LL area
  size_t rank_bytes = 0;       // per rank: flags + LL
  bool imported = false;
  DevState* state = nullptr;
  RankPrograms progs;
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
  int mover = MOVER_LSU;
  uint64_t* trace = nullptr;            // Phase-B op trace (optional)
  // tuning knobs, read from the environment once at init (include/stragglar.h)
  uint64_t slice_bytes = 16384;         // STRAGGLAR_SLICE_BYTES
  uint64_t ll_max_chunk = 0;            // STRAGGLAR_LL_MAX_CHUNK (0: LL off)
  int sys_scope = 1;                    // STRAGGLAR_SYS_SCOPE (team mode only; default 0 there)
  uint64_t e2e_piece_bytes = 8ull << 20;// STRAGGLAR_E2E_PIECE_BYTES (8 MiB measured best)
  int e2e_streams = 1;                  // STRAGGLAR_E2E_STREAMS (1 measured best)
  int last_slices = 0;                  // slices per chunk of the last Phase-B call (trace layout)
  // LL layout of the previous call if it ran Phase B through the LL areas
  // (count, element size, CTAs per rank); see LaunchPlan::ll_gate
  bool ll_last = false;
  uint64_t ll_count = 0;
  int ll_esize = 0, ll_G = 0;
  double alpha_s = 3e-6;               // P:450 per-message latency used in the paper's model
  double beta_s_per_byte = 1.0 / 770e9; // measured B200 peer copy per direction (B200_PROFILING.md)
  std::vector<Registration> regs;
  std::vector<void*> opened;   // IPC mappings to close
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
  const int cap = resident_ctas(world, c.mover, &sms);
  if (cap <= 0) return STRAGGLAR_ERR_CUDA;
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
  c.world = world;
  c.rank = team ? -1 : rank;
  c.sigma = sigma;
  c.team = team;
  c.rs_pending = false;
  c.bc_pending = false;
  c.timeout_ns = env_u64("STRAGGLAR_TIMEOUT_MS", 10000) * 1000000ull;
  c.slice_bytes = env_u64("STRAGGLAR_SLICE_BYTES", 16384);
  c.sys_scope = team ? (int)env_u64("STRAGGLAR_SYS_SCOPE", 0) : 1;
  // Sub-slices (finer hand-offs) pay with gpu-scope flags (team: Phase B -3.7 %)
  // but not with system-scope ones: every extra flag costs a fence.acq_rel.sys
  // (team mode at sys scope: 693 vs 690 us; per-process under MPS, n = 2/4/8:
  // 275/554/1082 us with them, 187/431/1027 without).
  c.sub = (int)env_u64("STRAGGLAR_SUBSLICES", c.sys_scope ? 1 : kMaxSub);
  c.sub_bytes = env_u64("STRAGGLAR_SUBSLICE_BYTES", 128 * 1024);
  if (c.sub < 1) c.sub = 1;
  if (c.sub > kMaxSub) c.sub = kMaxSub;
  c.ll_max_chunk = env_u64("STRAGGLAR_LL_MAX_CHUNK", 0);       // off by default: slower on one GPU
  if (c.ll_max_chunk > kLLChunkBytes) c.ll_max_chunk = kLLChunkBytes;
  c.e2e_piece_bytes = env_u64("STRAGGLAR_E2E_PIECE_BYTES", 8ull << 20);
  c.e2e_streams = (int)env_u64("STRAGGLAR_E2E_STREAMS", 1);
  c.flags_bytes = ((size_t)kSlots * G * kMaxSub * sizeof(uint32_t) + 255) / 256 * 256;
  c.rank_bytes = c.flags_bytes + (size_t)(kMaxWorld - 1) * kLLChunkWords * sizeof(uint64_t);
  const size_t nbytes = team ? c.rank_bytes * world : c.rank_bytes;
  auto fail_free = [&]() {
    if (c.flags) cudaFree(c.flags);
    if (c.state) cudaFree(c.state);
    c.flags = nullptr;
    c.state = nullptr;
    return STRAGGLAR_ERR_CUDA;
  };
  DevState init;
  std::memset(&init, 0, sizeof(init));
  init.stamp[0][0] = init.stamp[1][0] = ~0ull;   // armed: the first call's min start
  if (cudaMalloc(&c.flags, nbytes) != cudaSuccess || cudaMemset(c.flags, 0, nbytes) != cudaSuccess ||
      cudaMalloc(&c.state, sizeof(DevState)) != cudaSuccess ||
      cudaMemcpy(c.state, &init, sizeof(DevState), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return fail_free();
  for (int p = 0; p < kMaxWorld; ++p) {
    c.peer_flags[p] = nullptr;
    c.peer_ll[p] = nullptr;
  }
  auto ll_of = [&](uint32_t* f) { return reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(f) + c.flags_bytes); };
  if (team) {
    for (int p = 0; p < world; ++p) {
      c.peer_flags[p] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c.flags) + (size_t)p * c.rank_bytes);
      c.peer_ll[p] = ll_of(c.peer_flags[p]);
    }
    c.imported = true;
  } else {
    c.peer_flags[rank] = c.flags;
    c.peer_ll[rank] = ll_of(c.flags);
    c.imported = (world == 1);
  }
  c.active = true;
  return STRAGGLAR_OK;
}

void common_finalize(Comm& c) {
  if (!c.active) return;
  cudaDeviceSynchronize();
  for (void* p : c.opened) cudaIpcCloseMemHandle(p);
  c.opened.clear();
  c.regs.clear();
  if (c.flags) cudaFree(c.flags);
  if (c.state) cudaFree(c.state);
  if (c.trace) cudaFree(c.trace);
  c = Comm();
}

// Slices per call: about one slice per slice_bytes of a chunk.  Small messages
// use few CTAs (less flag traffic per round); large ones all G CTAs, each
// covering up to `sub` slices.  Any (G, sub) is safe call to call: flags hold
// monotone epochs, so values left at other positions by earlier calls are
// stale (< epoch); within a call every kernel uses the same layout.
void slices_for(const Comm& c, uint64_t chunk_bytes, int* G, int* sub) {
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
  const uint64_t unit = (uint64_t)c.G * c.sub_bytes;
  uint64_t m = unit ? (chunk_bytes + unit / 2) / unit : 1;
  if (m < 1) m = 1;
  if (m > (uint64_t)c.sub) m = c.sub;
  *G = c.G;
  *sub = (int)m;
}

// The call's epoch is not a launch parameter: kernels read state->epoch + 1 and
// the last CTA of the call's final kernel bumps it (graph-capturable).
LaunchPlan base_plan(const Comm& c, size_t count, int dtype, bool last_kernel) {
  LaunchPlan P;
  std::memset(&P, 0, sizeof(P));
  P.world = c.world;
  P.sigma = c.sigma;
  P.G = c.G;
  P.fstride = c.G * kMaxSub;
  P.last_kernel = last_kernel ? 1 : 0;
  P.count = count;
  P.esize = esize_of(dtype);
  P.ce = chunk_elems(count, c.world - 1, P.esize);
  P.nchunks = c.world - 1;
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
  P.timeout_ns = c.timeout_ns;
  P.mover = c.mover;
  P.trace = c.trace;
  {
    // LL Phase B for small chunks (latency-bound): STRAGGLAR_LL_MAX_CHUNK bytes, 0 disables
    const uint64_t chunk_bytes = P.ce * P.esize;
    P.use_ll = (chunk_bytes > 0 && chunk_bytes <= c.ll_max_chunk) ? 1 : 0;
    if (P.use_ll) P.sub = 1;   // the LL area is laid out per CTA slice
  }
  P.sys_scope = c.sys_scope;
  P.state = c.state;
  P.bc_partner = c.progs.bc_partner;
  for (int p = 0; p < c.world; ++p) {
    P.flags[p] = c.peer_flags[p];
    P.ll[p] = c.peer_ll[p];
    P.logical_of_phys[p] = c.progs.logical_of_phys[p];
    P.bc_sender[p] = c.progs.bc_sender[p];
    P.bc_round[p] = c.progs.bc_round[p];
    P.nops[p] = c.progs.nops[p];
    for (int k = 0; k < c.progs.nops[p]; ++k) P.ops[p][k] = c.progs.ops[p][k];
  }
  return P;
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

int launch(int which, int dtype, const LaunchPlan& P0, int nblocks, void* stream) {
  Comm& c = (g_team.active && P0.state == g_team.state) ? g_team : g_proc;
  if (which == K_COMPLETE || which == K_FUSED) c.last_slices = P0.G * P0.sub;
  // A peer is at most one call ahead (every call needs every rank's arrival to
  // complete anywhere).  If the previous call ran LL Phase B with another
  // layout, this call's up-front LL pushes must wait for their receivers'
  // arrival (per-process mode only: a team launch serves every rank at once).
  const bool runs_ll = P0.use_ll && (which == K_COMPLETE || which == K_FUSED);
  LaunchPlan P = P0;
  P.ll_gate = (runs_ll && !c.team && c.ll_last &&
               (c.ll_count != P.count || c.ll_esize != P.esize || c.ll_G != P.G)) ? 1 : 0;
  cudaError_t e = launch_plan_kernel(which, dtype, P, nblocks, (cudaStream_t)stream);
  if (e != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  if (P.last_kernel) {
    c.ll_last = runs_ll;
    c.ll_count = P.count;
    c.ll_esize = P.esize;
    c.ll_G = P.G;
  }
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

// team: Phase A over the non-stragglers (all in one launch)
int team_rs(void* const* bufs, size_t count, int dtype, void* stream) {
  Comm& c = g_team;
  LaunchPlan P = base_plan(c, count, dtype, false);
  for (int p = 0; p < c.world; ++p) P.buf[p] = (char*)bufs[p];
  int k = 0;
  for (int p = 0; p < c.world; ++p)
    if (p != c.sigma) P.local_rank[k++] = p;
  P.nlocal = k;
  return launch(K_RS, dtype, P, k * P.G, stream);
}

int team_b(void* const* bufs, size_t count, int dtype, void* stream, int which = K_COMPLETE, uint64_t delay_ns = 0) {
  Comm& c = g_team;
  LaunchPlan P = base_plan(c, count, dtype, true);
  P.sigma_delay_ns = delay_ns;
  for (int p = 0; p < c.world; ++p) {
    P.buf[p] = (char*)bufs[p];
    P.local_rank[p] = p;
  }
  P.nlocal = c.world;
  return launch(which, dtype, P, c.world * P.G, stream);
}

int read_error(Comm& c, int* code, uint32_t* where = nullptr) {
  if (!code) return STRAGGLAR_ERR_INVALID_ARG;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  CK(cudaDeviceSynchronize());
  DevState h;
  CK(cudaMemcpy(&h, c.state, sizeof(h), cudaMemcpyDeviceToHost));
  *code = (int)h.err;
  if (where) *where = h.err_info;
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
template <class F>
int e2e_pipeline(int nbufs, const void* const* host_in, void* const* host_out, void* const* bufs, size_t count, int es,
                 cudaStream_t s, uint64_t piece_bytes, int ncs, F&& allreduce_piece) {
  const uint64_t v = 16 / es;
  uint64_t piece = piece_bytes / es;
  piece = piece / v * v;
  if (piece == 0) piece = v;
  const uint64_t npieces = (count + piece - 1) / piece;
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
  for (uint64_t k = 0; k < npieces && st == STRAGGLAR_OK; ++k) {
    const uint64_t off = k * piece, n = (count - off) < piece ? (count - off) : piece;
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

int stragglar_export_handle(void* blob) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!blob) return STRAGGLAR_ERR_INVALID_ARG;
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  CK(cudaIpcGetMemHandle(&b.handle, g_proc.flags));
  b.offset = 0;
  b.bytes = g_proc.rank_bytes;
  std::memcpy(blob, &b, sizeof(b));
  return STRAGGLAR_OK;
}

int stragglar_import_handles(const void* blobs, int world) {
  std::lock_guard<std::mutex> lk(g_mu);
  Comm& c = g_proc;
  if (!c.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (!blobs || world != c.world) return STRAGGLAR_ERR_INVALID_ARG;
  const IpcBlob* b = static_cast<const IpcBlob*>(blobs);
  for (int p = 0; p < world; ++p) {
    if (p == c.rank) continue;
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, b[p].handle, cudaIpcMemLazyEnablePeerAccess));
    c.opened.push_back(ptr);
    if (b[p].bytes != c.rank_bytes) return STRAGGLAR_ERR_INVALID_ARG;   // ranks disagree on G
    c.peer_flags[p] = reinterpret_cast<uint32_t*>(static_cast<char*>(ptr) + b[p].offset);
    c.peer_ll[p] = reinterpret_cast<uint64_t*>(static_cast<char*>(ptr) + b[p].offset + c.flags_bytes);
  }
  c.imported = true;
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
  for (int p = 0; p < world; ++p) {
    if (p == c.rank) {
      r.peer[p] = r.local;
      continue;
    }
    if (b[p].bytes != r.bytes) return STRAGGLAR_ERR_INVALID_ARG;
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, b[p].handle, cudaIpcMemLazyEnablePeerAccess));
    c.opened.push_back(ptr);
    r.peer[p] = static_cast<char*>(ptr) + b[p].offset;
  }
  c.regs.push_back(r);
  return STRAGGLAR_OK;
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
  return launch(K_FUSED, dtype, P, P.G, stream);
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
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
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
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
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
  LaunchPlan P = base_plan(c, 0, STRAGGLAR_INT32, true);
  P.nlocal = 1;
  P.local_rank[0] = c.rank;
  if (launch_barrier(P, (cudaStream_t)stream) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
  return STRAGGLAR_OK;
}

int stragglar_inject_delay(uint64_t ns, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_proc.active) return STRAGGLAR_ERR_NOT_INITIALIZED;
  if (launch_delay(nullptr, ns, g_proc.state, (cudaStream_t)stream) != cudaSuccess) return STRAGGLAR_ERR_CUDA;
  g_launches.fetch_add(1);
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

int stragglar_team_reduce_scatter(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (g_team.rs_pending || g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;
  if ((st = team_rs(bufs, count, dtype, stream))) return st;
  g_team.rs_pending = true;
  return STRAGGLAR_OK;
}

int stragglar_team_complete(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (!g_team.rs_pending) return STRAGGLAR_ERR_INVALID_ARG;   // Phase B needs its Phase A
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
  if (!g_team.rs_pending) return STRAGGLAR_ERR_INVALID_ARG;
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
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
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
  slices_for(c, P.ce * P.esize, &P.G, &P.sub);
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
  return STRAGGLAR_OK;
}

int stragglar_team_bcast_complete(void* const* bufs, size_t count, int dtype, int op, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int st = team_check(bufs, count, dtype, op);
  if (st || count == 0) return st;
  if (!g_team.bc_pending) return STRAGGLAR_ERR_INVALID_ARG;   // needs its precondition
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
