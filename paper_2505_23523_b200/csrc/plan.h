// Launch descriptors shared by the host API and the kernels.
#pragma once
#include <cstdint>

#include "schedule.h"

namespace stragglar {

// Flag slots.  Every rank owns kSlots * G_max * kMaxSub uint32 flags; slot k,
// slice v lives at flags[k * G_max * kMaxSub + v] (a call uses G <= G_max CTAs
// per rank, each covering `sub` consecutive slices of every chunk; see
// LaunchPlan::sub and flag_at).  Flags hold the call's epoch (monotonic, never reset):
// a waiter proceeds when (int32)(flag - epoch) >= 0.  Producers write peers'
// flags (remote store, release at system scope); consumers spin on their own
// (local load, acquire at system scope).
enum Slot : int {
  SLOT_HAVE = 0,         // + chunk: the chunk's slice has landed, fully reduced, in my buffer
  SLOT_ARRIVE = 8,       // + physical rank: that rank's kernel started (its inputs are ready)
  SLOT_RSDONE = 16,      // + chunk: the owner's Phase-A partial of the slice is ready (written at sigma)
  SLOT_RING_ARRIVE = 24, // left neighbour started the ring
  SLOT_RING_READY = 25,  // + step (0..13): left neighbour finished ring step
  SLOT_RING_DONE = 39,   // right neighbour finished reading my buffer
  SLOT_BARRIER = 40,     // + physical rank
  // NEXT N3 baselines
  SLOT_BC_AGDONE = 48,   // Broadcast: the straggler's partner finished the non-straggler AllReduce (at sigma)
  SLOT_BC_READY = 49,    // + physical rank q: q finished the non-straggler AllReduce (at q's sender)
  SLOT_RHD_READY = 57,   // + step (0..5): the step's partner finished its previous step (step 0: arrived)
  SLOT_RHD_DONE = 63,    // + AllGather step (0..2): that step's partner finished reading my buffer
  SLOT_PROBE = 66,       // K0 flag ping-pong (stragglar_probe_pingpong): the peer's latest hop
  // op lanes (LaunchPlan::lanes > 1): a rank's ops run on several CTAs per slice,
  // so the hand-offs between its own lanes need local flags
  SLOT_SELF = 67,        // + chunk: my half of my exchange of the chunk is stored (local)
  SLOT_RS_LOCAL = 75,    // my Phase-A partial of the slice is stored (local; fused call)
  kSlots = 80
};

#ifndef STRAGGLAR_THREADS
#define STRAGGLAR_THREADS 256
#endif
constexpr int kThreads = STRAGGLAR_THREADS;   // CTA size of the data kernels
constexpr int kMaxSlices = 1024;
constexpr int kMaxSub = 16;                   // slices per CTA (LaunchPlan::sub) at most

// Device-resident per-communicator state (in the launching process's memory).
struct DevState {
  uint32_t err;          // 0 = ok, else an error code (first writer wins)
  uint32_t err_info;
  uint64_t t_rs_start;   // %globaltimer at the start of the last Phase-A launch (team)
  uint64_t t_release;    // when the last injected delay released
  uint32_t epoch;        // calls completed; the running call uses epoch + 1
  uint32_t exit_count;   // CTAs that finished the call's last kernel (reset by the last one)
  // phase stamps of the per-process fused calls (%globaltimer, this GPU), by
  // call-epoch parity: [e & 1] = {min CTA start, max end of Phase A, max end of
  // Phase B} of call e.  The last CTA of call e re-arms [(e + 1) & 1] for the
  // next call (no host memset per call).
  uint64_t stamp[2][3];
  // K0 probes: the ping-pong's hop counter (advanced identically on both
  // ranks of a pair) and the duration of the last ping-pong (ns, %globaltimer)
  uint32_t probe_seq;
  uint32_t probe_pad;
  uint64_t probe_ns;
  uint64_t t_barrier;    // %globaltimer when this rank left the last device barrier (start skew)
};

enum ErrCode : uint32_t { ERR_TIMEOUT = 1, ERR_BAD_PLAN = 2 };

// How the data kernels move bytes: SM load/store instructions (16-byte vectors) or
// TMA bulk copies (cp.async.bulk through a shared-memory stage ring).
enum Mover : int { MOVER_LSU = 0, MOVER_TMA = 1 };

struct LaunchPlan {
  int world;
  int sigma;                 // physical straggler
  int G;                     // CTAs per rank
  int sub;                   // slices per CTA: every chunk is cut into G * sub slices and CTA s
                             // handles slices s*sub .. s*sub+sub-1, one flag each (finer-grained
                             // hand-offs between ranks with the same CTAs); 1 = one slice per CTA
  int lanes;                 // op lanes per slice (Phase B): CTA lane q runs the rank's ops k with
                             // k % lanes == q, each as soon as its own inputs have landed (1 = one
                             // CTA walks all ops of the slice in round order)
  int rs_whole;              // Phase A: a CTA's sub slices as one range, flagged together (kernels.cuh rs_body)
  int nlocal;                // ranks served by this launch (1, or world in team mode)
  int fstride;               // flags per slot (G_max * kMaxSub, fixed per communicator; see flag_at)
  int local_rank[kMaxWorld]; // physical rank of local index i (blockIdx.x / G)
  char* buf[kMaxWorld];      // data buffer of each physical rank (local or peer mapping)
  uint32_t* flags[kMaxWorld];// flag array of each physical rank
  int last_kernel;            // 1: the call's final kernel; its last CTA to exit bumps state->epoch
  int sub_major;             // Phase B: a CTA walks its (op, sub-slice) units sub-slice by sub-slice
                             // (all ops of sub-slice 0, then of 1, ...) instead of op by op; must agree
                             // across ranks (a mixed order can deadlock), so it is a layout knob
  uint64_t count;            // elements
  uint64_t ce;               // elements per chunk (chunks start at j*ce)
  int nchunks;
  int esize;
  int mover;
  int sys_scope;             // 1: flags/fences at system scope (peers on other GPUs); 0: gpu scope (team)
  uint64_t timeout_ns;
  DevState* state;
  uint32_t* host_err;        // pinned host word (device-mapped): the first error, sticky (api.cu)
  uint64_t sigma_delay_ns;   // team measurement only: straggler CTAs start this late (KIND 4/5)
  uint64_t* trace;           // optional: [rank][slice][op][3] %globaltimer stamps (wait, data, done) of Phase B
  int logical_of_phys[kMaxWorld];
  int bc_partner;            // Broadcast baseline: the straggler's exchange partner (physical)
  int bc_sender[kMaxWorld];  //   per physical rank: who copies the full sum to it (-1: a holder)
  int bc_round[kMaxWorld];   //   and in which round
  char* mc_all;              // NVLS (nvls.cu): multicast mapping of every rank's arena (+ call offset)
  char* mc_ns;               //   the non-stragglers' multicast mapping (+ call offset)
  char* sigma_uc;            //   the straggler's arena, unicast peer mapping (+ call offset)
  int nops[kMaxWorld];       // by physical rank
  Op ops[kMaxWorld][kMaxOps];// by physical rank
};

// K0 copy probe (stragglar_probe_copy): this rank moves `bytes` to / from
// each peer in `peers` at once.  Push: local[me*bytes ..] -> peer[me*bytes ..];
// pull: peer[p*bytes ..] -> local[p*bytes ..] (disjoint segments, so every
// rank may probe at the same time).  CTA b serves peers[b % npeers].
struct ProbeArgs {
  char* local;
  char* peer[kMaxWorld];
  uint64_t bytes;
  int me;
  int npeers;
  int peers[kMaxWorld];
  int pull;                  // 0: push (remote stores), 1: pull (remote loads)
};

}  // namespace stragglar
