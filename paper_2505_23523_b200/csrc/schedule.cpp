// StragglAR schedule generator (Algorithm 1; §3.1)
// written for the runtime: holder sets are 64-bit masks, one pass per round.
// Readings of the garbled passages are the ones listed in DESIGN.md
// ("Readings" 1-11); they yield the same tie-breaks as the test oracle so the
// two can be compared transfer by transfer, but no code is shared.
#include "schedule.h"

#include <stdexcept>

namespace stragglar {

namespace {

inline int lowest(uint64_t m) { return m ? __builtin_ctzll(m) : -1; }
inline bool has(uint64_t m, int i) { return (m >> i) & 1ull; }
inline uint64_t bit(int i) { return 1ull << i; }

void fail(int r, const char* what) {
  throw std::runtime_error("stragglar schedule: round " + std::to_string(r) + ": " + what);
}

}  // namespace

std::vector<Round> generate_schedule(int n) {
  if (n < 2 || n > 64 || (n & (n - 1))) throw std::runtime_error("world must be a power of two in [2, 64]");
  int L = 0;
  while ((1 << L) < n) ++L;
  const int sigma = n - 1;
  const int R = n + L - 2;                         // Thm 1
  const uint64_t NS = (n == 64) ? ~0ull >> 1 : (bit(n - 1) - 1);

  // holders[c]: non-stragglers holding c_c fully reduced; active[c]: c_c is
  // reduced but not yet on every non-straggler (Definition 1).
  std::vector<uint64_t> holders(n - 1, 0);
  std::vector<bool> active(n - 1, false);
  auto active_chunk_of = [&](int h) -> int {
    for (int c = 0; c < n - 1; ++c)
      if (active[c] && has(holders[c], h)) return c;
    return -1;
  };

  std::vector<Round> sched;
  for (int r = 0; r < R; ++r) {
    Round rd;
    uint64_t busy = 0;                             // ranks matched this round
    uint64_t gained_dst[64] = {0};                 // receivers per chunk (applied after the round)
    auto copy = [&](int s, int d, int c) {
      rd.push_back({s, d, c, false});
      busy |= bit(s) | bit(d);
      if (d != sigma) gained_dst[c] |= bit(d);
    };

    // rank r <-> sigma, exchange and fully reduce c_r
    const bool sigma_busy = r < n - 1;
    if (sigma_busy) {
      rd.push_back({r, sigma, r, true});
      rd.push_back({sigma, r, r, true});
      busy |= bit(r);
    }

    if (r > 0 && r < L) {
      // Phase 1: mandated r-1 -> r-1+L, then every other holder
      // of a fully reduced chunk feeds the lowest chunk-free rank > 2(L-1).
      copy(r - 1, r - 1 + L, r - 1);
      for (int h = 0; h < n - 1; ++h) {
        if (has(busy, h)) continue;
        int c = active_chunk_of(h);
        if (c < 0) continue;
        int g = -1;
        for (int cand = 2 * (L - 1) + 1; cand < n - 1; ++cand)
          if (!has(busy, cand) && active_chunk_of(cand) < 0) { g = cand; break; }
        if (g < 0) fail(r, "phase 1 ran out of chunk-free receivers (Lemma 1)");
        copy(h, g, c);
      }
    } else if (r >= L) {
      // Phase 2
      const int old = r - L;                       // due chunk c_{r-log n}
      uint64_t P = (old < n - 1 && active[old]) ? (holders[old] & NS & ~busy) : 0;
      uint64_t Q = 0;
      for (int c = 0; c < n - 1; ++c)
        if (active[c] && c != old) Q |= holders[c];
      Q &= NS & ~busy;
      uint64_t window = 0;                         // critical window [r+1, r+L]
      for (int g = r + 1; g <= r + L && g < n - 1; ++g) window |= bit(g);

      auto swap_active = [&](int p, int q) {       // p (in P) sends c_old, q sends its own
        int cq = active_chunk_of(q);
        if (cq < 0) fail(r, "Q rank without an active chunk");
        copy(p, q, old);
        copy(q, p, cq);
      };
      for (int g = r + 1; g <= r + L && g < n - 1; ++g) {
        if (has(busy, g)) continue;
        if (has(Q, g)) {
          // g lacks only the due chunk: any P rank outside the window
          int p = lowest(P & ~busy & ~window);
          if (p < 0) fail(r, "no P partner for a window rank");
          swap_active(p, g);
        } else if (has(P, g)) {
          // g may only receive c_j with j <= g - L, oldest first
          int partner = -1;
          for (int j = 0; j < n - 1 && partner < 0; ++j) {
            if (!active[j] || j == old || j > g - L || has(holders[j], g)) continue;
            partner = lowest(holders[j] & Q & ~busy & ~window);
          }
          if (partner < 0) fail(r, "no admissible Q partner for a window rank");
          swap_active(g, partner);
        }
      }
      // P:182 / P:279-280: remaining P and Q zip in ascending order; for
      // r >= n-1 sigma joins Q last and only sends c_{n-2} (Remark 1).
      uint64_t Pr = P & ~busy, Qr = Q & ~busy;
      while (Pr) {
        int p = lowest(Pr);
        Pr &= Pr - 1;
        int q = lowest(Qr);
        if (q >= 0) {
          Qr &= Qr - 1;
          swap_active(p, q);
        } else if (!sigma_busy && !has(busy, sigma)) {
          copy(sigma, p, n - 2);
          busy |= bit(sigma);
        } else {
          fail(r, "|P| != |Q|");
        }
      }
      if (Qr) fail(r, "|Q| > |P|");
    }
    sched.push_back(rd);

    // bookkeeping after the round
    for (int c = 0; c < n - 1; ++c) holders[c] |= gained_dst[c];
    if (r >= L && r - L < n - 1) {
      if ((holders[r - L] & NS) != NS) fail(r, "due chunk not fully propagated (Lemma 2)");
      active[r - L] = false;
    }
    if (r < n - 1) {
      holders[r] |= bit(r);
      active[r] = true;
    }
  }
  for (int c = 0; c < n - 1; ++c)
    if ((holders[c] & NS) != NS) fail(R, "postcondition: a chunk did not reach every rank");
  return sched;
}

// ---------------------------------------------------------------------------
// Appendix B: even n that is not a power of two.  Per round the
// straggler pairing of round r < n-1 is kept; every other rank (and the
// straggler once it is free) is a vertex; u needs chunk c from v iff v holds
// c fully reduced and u does not.  Edge weight = number of directions with a
// need (2 or 1).  A maximum-weight matching is found by exhaustive
// search (n <= 14 here; P:684 cites Edmonds, same optimum); ties go to the
// first optimum in the order "lowest free vertex u, partners v > u ascending,
// then u unmatched".  Each matched rank sends the lowest-index chunk its
// partner needs.  DESIGN.md readings 18-21.
namespace {

struct Matcher {
  int nv = 0;
  int verts[64];
  int w[64][64];
  int best_w = -1;
  std::vector<std::pair<int, int>> best, cur;

  void rec(uint64_t rest, int acc) {
    if (!rest) {
      if (acc > best_w) {
        best_w = acc;
        best = cur;
      }
      return;
    }
    const int ui = __builtin_ctzll(rest);
    const uint64_t tail = rest & (rest - 1);
    for (uint64_t t = tail; t; t &= t - 1) {
      const int vi = __builtin_ctzll(t);
      if (w[ui][vi] > 0) {
        cur.push_back({verts[ui], verts[vi]});
        rec(tail & ~(1ull << vi), acc + w[ui][vi]);
        cur.pop_back();
      }
    }
    rec(tail, acc);
  }
};

std::vector<Round> generate_even(int n) {
  if (n < 6 || n > 14 || (n & 1) || !(n & (n - 1))) throw std::runtime_error("even non-power-of-two world must be in [6, 14]");
  const int sigma = n - 1;
  std::vector<uint64_t> full(n, 0);             // fully reduced chunks held, per rank
  const uint64_t all = (1ull << (n - 1)) - 1;
  std::vector<Round> sched;
  for (int r = 0;; ++r) {
    bool done = true;
    for (int h = 0; h < n; ++h) done &= full[h] == all;
    if (done) break;
    if (r >= 4 * n) throw std::runtime_error("appendix-B schedule did not complete");
    Round rd;
    Matcher m;
    for (int h = 0; h < n; ++h) {
      if (r < n - 1 && (h == r || h == sigma)) continue;
      m.verts[m.nv++] = h;
    }
    if (r < n - 1) {
      rd.push_back({r, sigma, r, true});
      rd.push_back({sigma, r, r, true});
    }
    for (int i = 0; i < m.nv; ++i)
      for (int j = 0; j < m.nv; ++j) {
        const int a = m.verts[i], b = m.verts[j];
        m.w[i][j] = (i == j) ? 0 : ((full[b] & ~full[a]) ? 1 : 0) + ((full[a] & ~full[b]) ? 1 : 0);
      }
    m.rec(m.nv == 64 ? ~0ull : ((1ull << m.nv) - 1), 0);
    for (auto [u, v] : m.best)
      for (int d = 0; d < 2; ++d) {
        const int a = d ? v : u, b = d ? u : v;  // a sends to b
        const uint64_t need = full[a] & ~full[b];
        if (need) rd.push_back({a, b, __builtin_ctzll(need), false});
      }
    sched.push_back(rd);
    std::vector<uint64_t> nf = full;
    for (const Xfer& x : rd) nf[x.dst] |= 1ull << x.chunk;
    full = nf;
  }
  return sched;
}

}  // namespace

std::vector<Round> generate_any(int n) {
  if (n >= 2 && !(n & (n - 1))) return generate_schedule(n);
  return generate_even(n);
}

void broadcast_tree(int n, int* sender, int* round) {
  if (n < 2 || n > 64) throw std::runtime_error("world must be in [2, 64]");
  uint64_t held = bit(0) | bit(n - 1);
  for (int q = 0; q < n; ++q) {
    sender[q] = -1;
    round[q] = 0;
  }
  for (int r = 1; __builtin_popcountll(held) < n; ++r) {
    const uint64_t before = held;
    int q = 0;
    for (int h = 0; h < n; ++h) {
      if (!has(before, h)) continue;
      while (q < n && has(held, q)) ++q;            // next non-holder, ascending
      if (q == n) break;
      sender[q] = h;
      round[q] = r;
      held |= bit(q);
    }
  }
}

RankPrograms build_programs(int n, int sigma_phys) {
  if (n < 2 || n > kMaxWorld || (n & 1)) throw std::runtime_error("world must be 2, 4, 6 or 8");
  if (sigma_phys < 0 || sigma_phys >= n) throw std::runtime_error("straggler rank out of range");
  RankPrograms pr;
  pr.n = n;
  pr.sigma = sigma_phys;
  for (int i = 0; i < n; ++i) pr.phys_of_logical[i] = i;
  pr.phys_of_logical[n - 1] = sigma_phys;          // P:200 / P:345 swap
  pr.phys_of_logical[sigma_phys] = n - 1;
  for (int l = 0; l < n; ++l) pr.logical_of_phys[pr.phys_of_logical[l]] = l;
  for (int p = 0; p < kMaxWorld; ++p) pr.nops[p] = 0;

  const int lsig = n - 1;
  auto sched = generate_any(n);
  for (size_t r = 0; r < sched.size(); ++r) {
    for (const Xfer& x : sched[r]) {
      Op op{};
      op.round = static_cast<uint8_t>(r);
      op.chunk = static_cast<uint8_t>(x.chunk);
      int actor;
      if (x.reduce) {
        // each side of the exchange computes half of every slice and pushes it
        // to the other (same bytes per direction as the paper's exchange)
        actor = x.src;
        op.kind = (x.src == lsig) ? OP_EXCH_HIGH : OP_EXCH_LOW;
      } else {
        actor = x.src;
        op.kind = OP_SEND;
      }
      op.peer = static_cast<uint8_t>(pr.phys_of_logical[x.dst]);
      int pa = pr.phys_of_logical[actor];
      if (pr.nops[pa] >= kMaxOps) throw std::runtime_error("op table overflow");
      pr.ops[pa][pr.nops[pa]++] = op;
    }
  }
  // data lifetimes for the L2 hints: a stored copy is re-read iff its holder
  // later sends that chunk; a SEND's source iff this rank sends it once more
  auto sends_chunk = [&](int p, int c, int after) {
    for (int k = after + 1; k < pr.nops[p]; ++k)
      if (pr.ops[p][k].kind == OP_SEND && pr.ops[p][k].chunk == c) return true;
    return false;
  };
  for (int p = 0; p < n; ++p)
    for (int k = 0; k < pr.nops[p]; ++k) {
      Op& o = pr.ops[p][k];
      o.life = 0;
      if (sends_chunk(o.peer, o.chunk, -1)) o.life |= LIFE_PEER_REREAD;
      if (o.kind == OP_SEND) {
        if (sends_chunk(p, o.chunk, k)) o.life |= LIFE_SRC_REREAD;
      } else if (sends_chunk(p, o.chunk, k)) {
        o.life |= LIFE_SELF_REREAD;
      }
    }
  int snd[kMaxWorld], rnd[kMaxWorld];
  broadcast_tree(n, snd, rnd);
  pr.bc_partner = pr.phys_of_logical[0];
  for (int p = 0; p < kMaxWorld; ++p) {
    pr.bc_sender[p] = -1;
    pr.bc_round[p] = 0;
  }
  for (int l = 0; l < n; ++l) {
    pr.bc_sender[pr.phys_of_logical[l]] = snd[l] < 0 ? -1 : pr.phys_of_logical[snd[l]];
    pr.bc_round[pr.phys_of_logical[l]] = rnd[l];
  }
  return pr;
}

}  // namespace stragglar
