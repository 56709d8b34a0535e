// Host-side StragglAR schedule (Algorithm 1) and the
// per-rank op tables the round executor consumes.  Independent of oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace stragglar {

struct Xfer {
  int src, dst, chunk;
  bool reduce;  // true: straggler exchange (both sides add); false: copy
};
using Round = std::vector<Xfer>;

// Algorithm 1 in logical ranks (straggler = n-1).  n: power of two in [2, 64].
// Throws std::runtime_error if n is unsupported or an internal invariant fails.
std::vector<Round> generate_schedule(int n);
// Algorithm 1 for powers of two, Appendix B (max-weight matching) for even n in [6, 14].
std::vector<Round> generate_any(int n);

// One step of a rank's program in the Phase-B kernel.
enum OpKind : uint8_t {
  OP_NONE = 0,
  OP_EXCH_LOW = 1,   // non-straggler side of the c_r exchange: first half of every slice
  OP_EXCH_HIGH = 2,  // straggler side of the c_r exchange: second half of every slice
  OP_SEND = 3        // push a fully reduced chunk to `peer`
};
// Op::life: which copies of the op's data are read again later in Phase B
// (L2 residency hints, kernels.cuh): the source of a SEND (this rank sends the
// chunk again), the peer's copy (the peer forwards the chunk), this rank's
// stored copy of an exchange (this rank forwards the chunk).
enum OpLife : uint8_t { LIFE_SRC_REREAD = 1, LIFE_PEER_REREAD = 2, LIFE_SELF_REREAD = 4 };
struct Op {
  uint8_t kind, chunk, peer, round;  // peer is a PHYSICAL rank
  uint8_t life;                      // OpLife bits
};

constexpr int kMaxWorld = 8;
constexpr int kMaxOps = 16;

// Per-physical-rank programs for world n with physical straggler sigma.
struct RankPrograms {
  int n = 0, sigma = 0;
  int phys_of_logical[kMaxWorld];
  int logical_of_phys[kMaxWorld];
  int nops[kMaxWorld];
  Op ops[kMaxWorld][kMaxOps];
  // straggler-aware Broadcast baseline, physical ranks: the
  // straggler's exchange partner, and per rank the rank it receives the full
  // sum from (-1: it holds it after the exchange) and that copy's round
  int bc_partner;
  int bc_sender[kMaxWorld];
  int bc_round[kMaxWorld];
};

// Broadcast baseline tree in logical ranks (straggler n-1): round 0 is the
// straggler's exchange with rank 0; in round r >= 1 the holders of the full
// sum, ascending, each copy it to the next non-holder, ascending.  sender[q]
// = -1 and round[q] = 0 for q in {0, n-1}.  n in [2, 64].
void broadcast_tree(int n, int* sender, int* round);
RankPrograms build_programs(int n, int sigma_phys);

}  // namespace stragglar
