/*
 * stragglar.h — C ABI of libstragglar.so, a B200 (sm_100a) implementation of the
 * StragglAR straggler-aware AllReduce (arXiv 2505.23523).
 *
 * Citations: P:<line> = /root/reference/PAPER.md line (section in brackets).
 *
 * The operation (§3.1): n ranks each hold a buffer of `count`
 * elements; rank `straggler_rank` is the persistent straggler (§1
 * "Assumptions"), swapped internally with logical rank n-1.
 *   Phase A  the n-1 non-stragglers ReduceScatter among themselves while the
 *            straggler is delayed: logical rank g ends with chunk c_g summed
 *            over the non-stragglers (Alg. 1 "Initialization").
 *   Phase B  the n+log2(n)-2 rounds of Algorithm 1 (Thm 1):
 *            round r < n-1 exchanges c_r between rank r and the straggler,
 *            both fully reduce it; every other transfer
 *            copies an already fully reduced chunk.
 * Postcondition: every rank holds the elementwise SUM of all n input
 * buffers, bitwise identical on every rank.
 *
 * Numerics: the non-straggler sum is taken in
 * ascending physical rank order with fp32 accumulation (int32 wraps mod 2^32);
 * bf16 is rounded to nearest-even once after Phase A and once after adding
 * the straggler's data.
 *
 * Buffer layout: one contiguous array of `count` elements, 16-byte aligned,
 * split into n-1 chunks of Ce = roundup(ceil(count/(n-1)), 16/esize) elements
 * (the last ones shorter or empty).  Chunk j is "owned" by logical rank j.
 *
 * Two communicator kinds exist in one process at a time:
 *   - the per-process communicator (stragglar_init ...): one process per GPU,
 *     peers' buffers and flags mapped with CUDA IPC; data moves over
 *     NVLink/NVSwitch with device-initiated loads and stores;
 *   - the single-device team (stragglar_team_*): all `world` logical ranks
 *     live on the current device of this process; "peer" accesses are plain
 *     HBM accesses.  Same kernels, same flags, same schedule.
 *
 * Conventions for every function:
 *   - returns a stragglar_status_t (0 = OK) and never throws or aborts;
 *   - collective calls must be made by every rank with the same count, dtype
 *     and op, in the same order (like ncclAllReduce);
 *   - asynchronous: work is enqueued on `stream` (a cudaStream_t; NULL = the
 *     legacy default stream) and the call returns without host sync; device
 *     faults and spin-wait timeouts surface through stragglar_check_error /
 *     stragglar_team_check_error after a stream synchronize;
 *   - count == 0 is a successful no-op; buf must be 16-byte aligned;
 *   - the library owns its flags, workspace, IPC mappings and schedule tables
 *     (released by *_finalize); the caller owns buffers and streams.
 */
#ifndef STRAGGLAR_H_
#define STRAGGLAR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  STRAGGLAR_INT32 = 0,    /* wraps modulo 2^32 */
  STRAGGLAR_FLOAT32 = 1,  /* IEEE binary32, round-to-nearest-even adds */
  STRAGGLAR_BFLOAT16 = 2  /* fp32 accumulation, RNE rounding (see above) */
} stragglar_dtype_t;

typedef enum { STRAGGLAR_SUM = 0 } stragglar_op_t;

typedef enum {
  STRAGGLAR_OK = 0,
  STRAGGLAR_ERR_INVALID_ARG = 1,     /* NULL/unaligned buffer, bad rank, ... */
  STRAGGLAR_ERR_UNSUPPORTED = 2,     /* world not in {2,4,6,8}, unknown dtype/op */
  STRAGGLAR_ERR_NOT_INITIALIZED = 3, /* no communicator / handles not imported */
  STRAGGLAR_ERR_NOT_REGISTERED = 4,  /* buf not inside a registered buffer */
  STRAGGLAR_ERR_CUDA = 5,            /* a CUDA runtime/driver call failed */
  STRAGGLAR_ERR_TIMEOUT = 6,         /* a device spin-wait exceeded the watchdog; sticky:
                                        every later call on that communicator returns it
                                        until the communicator is re-initialized */
  STRAGGLAR_ERR_INTERNAL = 7
} stragglar_status_t;

/* ---- library info ------------------------------------------------------ */
int stragglar_version(void);                       /* 100*major + minor */
const char* stragglar_status_string(int status);   /* static string, never NULL */

/* ---- schedule introspection (host only; no GPU needed) -------------------
 * The library's own C++ implementation of Algorithm 1 in logical
 * ranks (straggler = world-1).  stragglar_schedule_rounds returns R =
 * world + log2(world) - 2 (Thm 1).  stragglar_schedule_round writes the
 * transfers of round `round` as int quadruples {src, dst, chunk, kind} with
 * kind 0 = Reduce (the straggler exchange), 1 = Replace (copy of a fully
 * reduced chunk), into out[0 .. 4*max_transfers), and their number into
 * *n_transfers.  Supports power-of-two world in [2, 64]. */
int stragglar_schedule_rounds(int world, int* rounds);
int stragglar_schedule_round(int world, int round, int* out, int max_transfers, int* n_transfers);
/* Host only: the layout a StragglAR call of `count` elements would use with
 * `ctas_per_rank` CTAs per rank and the default knobs — slices per chunk
 * (CTA slots), slices per CTA (sub) and Phase-B op lanes per slice (DESIGN.md
 * §5).  sys_scope selects the per-process defaults (one slice per CTA). */
int stragglar_plan_layout(int world, int straggler_rank, size_t count, int dtype, int ctas_per_rank, int sys_scope,
                          int* slices, int* sub, int* lanes);
/* Host only: the pieces the host-buffer entry points (stragglar_allreduce_host,
 * stragglar_team_allreduce_host) cut a `count`-element buffer into — element
 * counts in order, written to out[0 .. max_pieces), their number to *n_pieces
 * (INVALID_ARG if more than max_pieces).  piece_bytes is the piece size
 * (STRAGGLAR_E2E_PIECE_BYTES), rounded down to 16 bytes; every piece but the
 * last has it, the last takes the rest; the pieces add up to count. */
int stragglar_plan_e2e_pieces(size_t count, int dtype, size_t piece_bytes, size_t* out, int max_pieces,
                              int* n_pieces);

/* ---- per-process communicator (one process per GPU) ----------------------
 * stragglar_init(rank, world, straggler_rank): rank and straggler_rank in
 * [0, world), world in {2,4,8} (Algorithm 1) or 6 (the even
 * non-power-of-two schedule of Appendix B); uses the calling
 * thread's current CUDA device; allocates the flag array and builds this
 * rank's round table.  The straggler is fixed for the communicator's lifetime
 * (P:457-459). */
int stragglar_init(int rank, int world, int straggler_rank);
/* Size of the opaque per-rank blob that carries IPC handles. */
int stragglar_handle_size(size_t* bytes);
/* Writes this rank's flag-array IPC handle into blob (handle_size bytes),
 * with the rank, its GPU's UUID and co-resident CTA capacity, and the
 * communicator's layout knobs (straggler, CTAs, slice sizes, mover, scope). */
int stragglar_export_handle(void* blob);
/* blobs: world * handle_size bytes, rank order (exchanged by the caller, e.g.
 * torch.distributed all_gather); opens every peer's flag array.
 * INVALID_ARG if a blob sits at the wrong index or any rank's layout knobs
 * differ from this rank's (the environment knobs below must agree across
 * ranks: a flag covers the same bytes everywhere only then).  Ranks that
 * share a GPU (several processes per device, e.g. under MPS) split its
 * co-resident CTA capacity: the CTAs per rank become
 * min over GPUs of capacity / (ranks on that GPU), the same on every rank;
 * UNSUPPORTED if that is 0. */
int stragglar_import_handles(const void* blobs, int world);
/* After import: how many ranks of this communicator share this rank's GPU
 * and the CTAs per rank a launch uses. */
int stragglar_shared_device_ranks(int* ranks_on_my_gpu, int* ctas_per_rank);
/* Registers [buf, buf+bytes) (device memory of this process) for peer access
 * and writes its IPC blob (handle_size bytes) into blob_out.  Collective in
 * effect: every rank registers its corresponding buffer, then all ranks call
 * stragglar_import_buffer with everyone's blobs. */
int stragglar_register_buffer(void* buf, size_t bytes, void* blob_out);
/* INVALID_ARG if the ranks registered different byte counts. */
int stragglar_import_buffer(void* buf, const void* blobs, int world);
/* Closes this process's mappings of the peers' copies of the registration
 * that starts at buf (synchronizes the device first).  Local, but every rank
 * should deregister its copy before freeing it; NOT_REGISTERED if none. */
int stragglar_deregister_buffer(void* buf);
/* StragglAR AllReduce in place ("similar functionality to
 * ncclAllReduce()").  buf must lie in a registered buffer at the same offset
 * on every rank.  Non-stragglers enqueue Phase A then Phase B; the straggler
 * enqueues Phase B only (its delay is whatever precedes it on its stream). */
int stragglar_allreduce(void* buf, size_t count, int dtype, int op, void* stream);
/* Hand-written Ring AllReduce baseline on the same transport:
 * 2(n-1) pull steps of ~count/n elements; bf16 partials rounded per hop. */
int stragglar_allreduce_ring(void* buf, size_t count, int dtype, int op, void* stream);
/* NEXT row N1(ii): the same Phase A, then a one-round
 * "direct completion" — each non-straggler owner g adds x_sigma to its
 * partial c_g (the straggler exchange's single add) and stores
 * the fully reduced chunk to every rank.  Valid on switched fabrics where a
 * GPU can feed several peers at once (the paper's single-port model, P:149-150,
 * does not hold on NVSwitch): ~S bytes per port instead of
 * (n+log2 n-2)/(n-1)*S, one round instead of n+log2 n-2.  Result identical
 * to stragglar_allreduce, bit for bit. */
int stragglar_allreduce_direct(void* buf, size_t count, int dtype, int op, void* stream);
/* NEXT row N3: the paper's other baselines,
 * in-house on the same transport, in place, collective, same argument rules
 * and errors as stragglar_allreduce.
 * RHD — recursive halving/doubling ("Butterfly"): n chunks (the
 *   Ring's partition); log2 n ReduceScatter steps in which, at step t, rank j
 *   pairs with j XOR 2^t (round k pairs ranks differing in bit k)
 *   and adds the partner's copy of the half of the shared block it keeps (the
 *   lower half if bit t of j is 0), then log2 n mirror-image AllGather steps;
 *   bf16 partials rounded per step.
 *   UNSUPPORTED unless world is a power of two.
 * Broadcast — straggler-aware: the non-stragglers AllReduce
 *   among themselves (canonical order of Phase A, then every non-straggler
 *   copies the other partials), the straggler exchanges its entire buffer
 *   with logical rank 0 (one add, the same bits as stragglar_allreduce), and
 *   the full sum is copied along a doubling tree (stragglar_broadcast_tree),
 *   s bytes per copy, ceil(log2 n) rounds in all. */
int stragglar_allreduce_rhd(void* buf, size_t count, int dtype, int op, void* stream);
int stragglar_allreduce_bcast(void* buf, size_t count, int dtype, int op, void* stream);
/* The Broadcast baseline's tree in LOGICAL ranks (straggler = world-1):
 * sender[q] = the rank q receives the full sum from (-1 for ranks 0 and
 * world-1, which hold it after the exchange), round[q] = that copy's round
 * (0 for the two holders).  Arrays of `world` ints; world in [2, 64]. */
int stragglar_broadcast_tree(int world, int* sender, int* round);
/* End to end from host memory (collective): host_in (count elements) is
 * copied into the registered device buffer `buf`, AllReduced with
 * stragglar_allreduce, and the result copied to host_out (may equal
 * host_in), through a pipeline of pieces (STRAGGLAR_E2E_PIECE_BYTES, 8 MiB;
 * stragglar_plan_e2e_pieces): H2D of piece k+1, the
 * AllReduce of piece k and D2H of piece k-1 overlap.  Every rank cuts the
 * same pieces (the piece knobs are checked at import), so each piece is one
 * collective call.
 * Synchronous: returns when host_out holds the result.  host buffers should
 * be pinned for full PCIe bandwidth.  Same errors as stragglar_allreduce,
 * INVALID_ARG for NULL host pointers. */
int stragglar_allreduce_host(const void* host_in, void* host_out, void* buf, size_t count, int dtype, int op,
                             void* stream);
/* Device-side barrier among all ranks of the communicator (bench start line). */
int stragglar_barrier(void* stream);
/* %globaltimer (ns, this GPU's clock) at which this rank left its last
 * stragglar_barrier; compared across ranks it bounds the start-line skew.
 * Synchronizes the device. */
int stragglar_last_barrier_ns(uint64_t* ns);
/* ---- K0 probes: the measured ceilings of the transport (
 * the paper's link bandwidths P:386-388 and model constants P:449-451) -------
 * stragglar_probe_copy: device-initiated copies between this rank and every
 * peer p with bit p of peer_mask set, all at once.  buf lies in a registered
 * buffer of >= world * bytes_per_peer bytes (bytes_per_peer a multiple of
 * 16); segment q of every rank's copy is [q*bytes_per_peer, (q+1)*...).
 * mode bit 0: 0 = push (read own segment `rank` locally, store it into
 * segment `rank` of each peer), 1 = pull (load segment p of peer p, store it
 * into own segment p); mode bit 1: 0 = 16-byte ld/st by every thread, 1 =
 * cp.async.bulk (TMA) through shared memory, the data kernels' default mover.
 * ctas: CTAs (0 = the communicator's per-rank count), rounded up to a
 * multiple of the number of peers.  Not collective: the caller decides which
 * ranks probe at once (uni- vs bidirectional) and times the call with events
 * after stragglar_barrier. */
int stragglar_probe_copy(void* buf, size_t bytes_per_peer, int mode, uint32_t peer_mask, int ctas, void* stream);
/* Collective between this rank and `peer` (both call it, each naming the
 * other, with the same iters): `iters` flag round trips with the data
 * kernels' system-scope signalling (fence.acq_rel.sys + st.relaxed.sys to the
 * peer's flag, ld.acquire.sys on the own); the lower rank starts each trip.
 * stragglar_probe_pingpong_result (synchronizes) returns the last ping-pong's
 * device time in us (divide by 2*iters for one hop, the model's alpha). */
int stragglar_probe_pingpong(int peer, int iters, void* stream);
int stragglar_probe_pingpong_result(double* us);
/* Bench only: a one-thread kernel that spins on %globaltimer for `ns`
 * nanoseconds from its own start (the paper's idle kernel). */
int stragglar_inject_delay(uint64_t ns, void* stream);
/* Reads the device error word (watchdog timeouts) and clears the device copy.
 * *code = 0 if none.  Synchronizes the device.  A timeout leaves the ranks'
 * flags out of step, so the communicator stays failed: later calls return
 * STRAGGLAR_ERR_TIMEOUT (from a pinned host copy of the word, no sync) until
 * *_finalize and a new *_init. */
int stragglar_check_error(int* code);
/* Same, for the team (team != 0) or the per-process communicator, also
 * returning where the first failing spin-wait was: (kind << 8) | index with
 * kind 0x1 Phase-A arrival, 0x2 exchange (non-straggler side), 0x3 exchange
 * (straggler side), 0x4 copy, 0x5 completion, 0x6/0x7 ring, 0x8 barrier,
 * 0x9/0xA direct completion, 0xC/0xD Broadcast baseline, 0xE RHD. */
int stragglar_check_error_where(int team, int* code, uint32_t* where);
/* Phase breakdown of this rank's last call, which must have been
 * stragglar_allreduce(_direct) (INVALID_ARG otherwise), from %globaltimer
 * stamps inside the kernel (this GPU's clock): *t_a_us = kernel start to the
 * end of the rank's Phase A (the straggler has none: ~0), *t_total_us =
 * kernel start to the end of its Phase B.  The stamps are re-armed on the
 * device by the previous call (no per-call host work).  Synchronizes. */
int stragglar_phase_times(double* t_a_us, double* t_total_us);
int stragglar_finalize(void);

/* ---- NEXT N1(i): NVLink SHARP (NVLS) multicast variant ---
 * The paper assumes a single-port fabric; an NVSwitch fabric can
 * also reduce and replicate in the switch.  Same two phases, same straggler
 * roles: Phase A = each owner's multimem.ld_reduce of its chunk through the
 * non-stragglers' multicast object (the switch sums the n-1 copies: owner
 * ingress C instead of (n-2)C); completion = the owner adds x_sigma (one
 * unicast peer load; the exchange's single add) and writes the
 * fully reduced chunk to every rank with one multimem.st through the all-rank
 * multicast object.  Numerics (reading 24): the switch's summation
 * order over the non-stragglers is unspecified (fp32 accumulation; bf16 via
 * .acc::f32, rounded once), then x_sigma is added once: int32 results are
 * exact, float results agree with stragglar_allreduce within the north_star
 * tolerance, not bit for bit.
 * Buffers must be the library's arena (VMM memory bound to the multicast
 * objects; cudaMalloc memory cannot be bound).  Setup is collective, in two
 * steps around an exchange of POSIX file descriptors that the caller performs
 * (dist.py passes them over UNIX-domain sockets, SCM_RIGHTS):
 *   nvls_begin(bytes): allocates this rank's arena (rounded up to the
 *     multicast granularity, *bytes_out) and exports fds[0] = the all-rank
 *     multicast object (rank 0; -1 elsewhere), fds[1] = the non-straggler
 *     object (the lowest non-straggler rank; -1 elsewhere), fds[2] = this
 *     rank's arena.  The fds stay owned by the library.
 *   nvls_import(mc_all_fd, mc_ns_fd, sigma_mem_fd): imports the objects (rank
 *     0 / the lowest non-straggler pass their own) and, on non-stragglers, the
 *     straggler's arena.  The caller checks that EVERY rank imported before
 *     any binds: a bind waits until the whole team joined, so a rank that
 *     failed here would leave the others waiting (stragglar_nvls_release
 *     undoes a begun / imported arena).
 *   nvls_bind(&arena): joins both objects, binds the arena, maps the multicast
 *     ranges and the straggler's arena; *arena = this rank's arena.
 * UNSUPPORTED without multicast support (stragglar_nvls_supported) or the
 * driver entry points.  Released by stragglar_nvls_release / _finalize.
 * stragglar_allreduce_nvls: in place on [buf, buf + count) inside the arena
 * (same offset on every rank), count a multiple of 16 bytes' worth of
 * elements (INVALID_ARG otherwise), NOT_REGISTERED outside the arena.
 * stragglar_nvls_selftest: one-GPU check of the multicast path — a
 * one-member multicast object on the current device; host_out = the reducing
 * load of host_in through it (equal to host_in).  No communicator needed;
 * UNSUPPORTED when the driver creates no multicast object (a GPU without an
 * NVSwitch fabric behind it, e.g. this run's one-GPU box).
 * MEASURED ONLY ON ONE GPU: the multi-GPU path needs >= 2 NVSwitch GPUs. */
int stragglar_nvls_supported(int* supported);
int stragglar_nvls_begin(size_t bytes, int* fds, size_t* bytes_out);
int stragglar_nvls_import(int mc_all_fd, int mc_ns_fd, int sigma_mem_fd);
int stragglar_nvls_bind(void** arena);
int stragglar_nvls_release(void);
int stragglar_allreduce_nvls(void* buf, size_t count, int dtype, int op, void* stream);
int stragglar_nvls_selftest(int dtype, size_t count, const void* host_in, void* host_out);
/* Test only: the NVLS kernel with its two multicast operations emulated
 * through IPC peer pointers (the reducing load as the canonical non-straggler
 * sum, the multicast store as one store per rank) on a REGISTERED buffer of
 * the per-process communicator — validates the variant's flags, epochs and
 * hand-offs where no multicast object exists.  Same arguments and errors as
 * stragglar_allreduce_nvls (count a multiple of 16 bytes' worth); the result
 * equals stragglar_allreduce's bit for bit. */
int stragglar_allreduce_nvls_emulated(void* buf, size_t count, int dtype, int op, void* stream);

/* ---- single-device team (all ranks on the current device) ---------------
 * bufs: array of `world` device pointers (physical rank order), each 16-byte
 * aligned with `count` elements; they must not overlap. */
int stragglar_team_init(int world, int straggler_rank);
int stragglar_team_allreduce(void* const* bufs, size_t count, int dtype, int op, void* stream);
/* The two phases separately (the allreduce is exactly phase A then phase B):
 * reduce_scatter = Phase A over the n-1 non-stragglers;
 * complete       = Phase B over all n ranks (requires Phase A on the same
 *                  buffers, count and dtype first: INVALID_ARG otherwise). */
int stragglar_team_reduce_scatter(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_complete(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_allreduce_ring(void* const* bufs, size_t count, int dtype, int op, void* stream);
/* Direct completion (see stragglar_allreduce_direct) after a team Phase A,
 * and the whole direct-completion AllReduce. */
int stragglar_team_complete_direct(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_allreduce_direct(void* const* bufs, size_t count, int dtype, int op, void* stream);
/* NEXT N3 baselines on the team (see stragglar_allreduce_rhd / _bcast).
 * bcast_precondition = the non-straggler AllReduce (n-1 ranks, the part the
 * paper assumes hidden in the delay); bcast_complete = the
 * straggler's exchange + doubling copies (requires the precondition on the
 * same buffers first); allreduce_bcast = both in one launch. */
int stragglar_team_allreduce_rhd(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_bcast_precondition(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_bcast_complete(void* const* bufs, size_t count, int dtype, int op, void* stream);
int stragglar_team_allreduce_bcast(void* const* bufs, size_t count, int dtype, int op, void* stream);
/* Measurement only: the whole AllReduce in one launch (Phase A + B) with the
 * straggler's CTAs arriving delay_ns after the launch, so the straggler's
 * exchanges can overlap the non-stragglers' Phase A tail slice by slice, as
 * across GPUs (the split reduce_scatter -> inject_delay -> complete sequence
 * serialises them).  Used for the partial-overlap delay sweep. */
int stragglar_team_allreduce_delayed(void* const* bufs, size_t count, int dtype, int op, uint64_t delay_ns,
                                     void* stream);
/* Bench only: spin until `ns` nanoseconds after the start of the most
 * recent team Phase A launch (the straggler's arrival time). */
int stragglar_team_inject_delay(uint64_t ns, void* stream);
/* End to end from host memory: copies host_in[p] -> bufs[p] (H2D), runs the
 * StragglAR AllReduce, copies bufs[p] -> host_out[p] (D2H), and synchronizes
 * `stream`.  The elementwise SUM lets the buffer go through a pipeline of
 * pieces (default 8 MiB, STRAGGLAR_E2E_PIECE_BYTES; stragglar_plan_e2e_pieces): H2D, AllReduce and D2H of consecutive pieces overlap on two copy-engine streams and `stream`.
 * host_in/host_out should be pinned for full PCIe bandwidth; host_out may
 * equal host_in. */
int stragglar_team_allreduce_host(const void* const* host_in, void* const* host_out, void* const* bufs,
                                  size_t count, int dtype, int op, void* stream);
/* Tracing (team mode): when enabled, thread 0 of every Phase-B CTA records
 * three %globaltimer stamps per op and slice — wait began, data movement
 * began, op signalled — at out[((rank * NS + slice) * 16 + op) * 3 + {0,1,2}],
 * NS = slices per chunk of the last call (CTAs per rank x slices per CTA,
 * written to *slices).  read_trace synchronizes the
 * device; with out == NULL it only reports the sizes. */
int stragglar_team_set_trace(int enable);
int stragglar_team_read_trace(uint64_t* out, size_t max_entries, size_t* n_entries, int* slices);
/* CTAs per rank per launch chosen at team_init (each covers 1..16 slices of
 * every chunk, by message size: STRAGGLAR_SUBSLICE_BYTES). */
int stragglar_team_slices(int* slices);
int stragglar_team_check_error(int* code);
int stragglar_team_finalize(void);

/* ---- algorithm selection for an expected delay ------
 * PAPER.md §4.2: StragglAR beats a baseline B iff
 *     T_delay >= T_RS - max{T_B - T_SAR, 0}.
 * stragglar_select evaluates it with the alpha-beta model of this
 * implementation, per port, for a buffer of `bytes` at `world` ranks:
 *     T_RS   = alpha + (n-2)/(n-1) * bytes * beta     (Phase A: one direct-pull step)
 *     T_SAR  = R alpha + R/(n-1) * bytes * beta        (R = n + log2 n - 2)
 *     T_Ring = 2(n-1) alpha + 2(n-1)/n * bytes * beta
 * Outputs the critical delay (s, >= 0) and use_stragglar = (delay_s >= critical).
 * Host only; world even in [2, 64]: powers of two use Algorithm 1, other even
 * world sizes the Appendix-B schedule (built for 6..14; UNSUPPORTED beyond). */
int stragglar_select(int world, double bytes, double delay_s, double alpha_s, double beta_s_per_byte,
                     int* use_stragglar, double* critical_delay_s);
/* Algorithm codes of stragglar_select_algorithm / stragglar_allreduce_auto. */
enum { STRAGGLAR_ALGO_RING = 0, STRAGGLAR_ALGO_STRAGGLAR = 1, STRAGGLAR_ALGO_RHD = 2 };
/* The same model over every algorithm the library has that does not need the
 * straggler-specific precondition, predicted completion from the
 * non-stragglers' start: StragglAR max(delay, T_RS) + T_SAR; the
 * bulk-synchronous Ring delay + T_Ring and RHD delay + T_RHD (T_RHD = 2 log2 n
 * alpha + 2(n-1)/n bytes beta; powers of two only).  *algo = the
 * fastest (ties: StragglAR, then Ring), *t_pred_s (may be NULL) = its time.
 * With small buffers RHD's 2 log2 n latency terms win, as the paper measured
 * (P:398-400); with a masking delay and large buffers StragglAR does. */
int stragglar_select_algorithm(int world, double bytes, double delay_s, double alpha_s, double beta_s_per_byte,
                               int* algo, double* t_pred_s);
/* Cost-model constants of the per-process communicator used by
 * stragglar_allreduce_auto (defaults: alpha = 3 us; beta = 1/(770 GB/s),
 * the measured B200 peer-copy bandwidth per direction). */
int stragglar_set_cost_model(double alpha_s, double beta_s_per_byte);
/* Collective: every rank passes the same expected straggler delay; runs the
 * algorithm stragglar_select_algorithm picks (StragglAR, Ring or RHD) with the
 * communicator's cost model; *used_algorithm (may be NULL) = its
 * STRAGGLAR_ALGO_* code (1 = StragglAR, 0 = Ring as before, 2 = RHD). */
int stragglar_allreduce_auto(void* buf, size_t count, int dtype, int op, void* stream, uint64_t expected_delay_ns,
                             int* used_algorithm);

/* Environment knobs, read once by stragglar_init / stragglar_team_init:
 * STRAGGLAR_MOVER=tma|lsu (data mover), STRAGGLAR_SLICE_BYTES (target bytes
 * per slice, 16384), STRAGGLAR_SLICES (per-process CTA cap, 2 x SMs),
 * STRAGGLAR_SUBSLICES (slices per CTA at most, 1..16; default 16) and
 * STRAGGLAR_SUBSLICE_BYTES (their target size on large messages, 131072: each
 * hop hands over ~128 KB pieces, so a forwarded slice is still in L2 when
 * the next hop reads it), STRAGGLAR_BASELINE_SUBSLICE_BYTES (the same for
 * the Ring and RHD baselines, tuned for them: 65536 with GPU-scope flags,
 * 131072 at system scope), STRAGGLAR_SUB_MAJOR (1: a CTA runs its units
 * sub-slice by sub-slice — all ops / steps of sub-slice 0, then of 1, … — in
 * Phase B, the Ring and RHD, so forwarded data is re-read while it is still in
 * L2; 0: op by op; must agree across ranks), STRAGGLAR_BASELINE_SUB_MAJOR (the
 * same for the Ring and RHD: 1 with GPU-scope flags, 0 at system scope),
 * STRAGGLAR_OP_LANES (Phase-B op lanes per slice at most, 16; 1 = off),
 * STRAGGLAR_LANE_SLICE_MAX (slices may grow to this many bytes to make room
 * for op lanes on small messages, 32768; 0 = off), STRAGGLAR_RS_WHOLE (Phase A
 * reduces a CTA's sub-slices as one range and flags them together, 1),
 * STRAGGLAR_TIMEOUT_MS (watchdog, 10000), STRAGGLAR_SYS_SCOPE (team mode: system-scope flags, 0), and for the host
 * entry point STRAGGLAR_E2E_PIECE_BYTES (8 MiB) / STRAGGLAR_E2E_STREAMS (1). */

/* Number of kernel launches the library enqueued since load (bench evidence). */
int stragglar_launch_count(uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* STRAGGLAR_H_ */
