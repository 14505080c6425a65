/*
 * vtrain_b200.h -- C ABI of the B200 (sm_100a) hot path of the vtrain
 * verifiable-training scheme (arXiv 2403.09603).
 *
 * Every entry point is stateless and stream-ordered: the caller owns all
 * device buffers (plain device pointers + sizes), passes a cudaStream_t as
 * an opaque pointer, and reads results (counters, error bits) back when it
 * synchronises.  No torch types appear here.  Status return values describe
 * argument / launch problems only; data-dependent failures (non-finite
 * input, range, bad code, corrupt log) are reported as VT_ERR_* bits OR-ed
 * into the caller's device int32 `err`, which the host wrapper turns into
 * the reference's exact exception text, in the reference's check order.
 *
 * Reference interfaces replaced (paths relative to the reference root
 * /root/reference, vtrain 0.1.0):
 *   vt_round_log      <- protocol._TrainerChannel.process   pkg/src/vtrain/protocol.py:198-202
 *                        (= fpround.direction_array :164-177 + rnd_array :127-135
 *                           + roundlog.LogWriter.write_array pkg/src/vtrain/roundlog.py:119-137),
 *                        fpround.rnd_array (no log outputs), direction_array (codes only),
 *                        protocol._PlainChannel.process      protocol.py:225-226
 *   vt_replay         <- protocol._AuditorChannel.process    protocol.py:212-216
 *                        (= roundlog.LogReader.read_array :195-201 + fpround.rev_array :227-247)
 *   vt_grid_neighbors <- fpround.grid_neighbors_array        fpround.py:185-218
 *   vt_exponent_scale <- fpround.exponent_scale_array        fpround.py:149-156
 *   vt_is_on_grid     <- fpround.is_on_grid                  fpround.py:255-264
 *   vt_norm_distance  <- the |x-rnd(x)|/max(scale,2^-126) term of direction_array :171-173
 *   vt_pack5          <- roundlog._pack_block                roundlog.py:67-70
 *   vt_unpack5        <- roundlog._unpack_block              roundlog.py:73-82
 *   vt_log_validate   <- the byte check of _unpack_block     roundlog.py:75-76
 *   vt_log_histogram  <- roundlog.LogReader.histogram        roundlog.py:203-206
 *   vt_tau_kth_key    <- protocol.search_tau predicate       protocol.py:494-506 (budget form,
 *   vt_tau_kth_begin/hist/select: the same, one pass at a time (sharded tensors)
 *   vt_tau_budget_key    SURVEY.md Appendix A.4)
 *   vt_tau_budget     <- the same budget search incl. the bisection, one read of x
 *   vt_tau_shard_*    <- the same over a tensor sharded across ranks
 *   vt_round_log_exchange / vt_counts_wait <- vt_round_log + the count all-gather of
 *                        a sharded round-and-log, fused over peer memory
 *   vt_min_f64        <- the all(p >= tau) predicate of search_tau  protocol.py:502
 *   vt_sha256_leaves  <- merkle._sha256 over 4 KiB chunks    merkle.py:24-25
 *   vt_merkle_level   <- one level of merkle.build           merkle.py:55-72
 *   vt_merkle_build   <- merkle.build over chunked leaves    merkle.py:55-72
 *   vt_tau_shard_search_x <- search_tau_budget over a sharded tensor, both
 *                        exchanges over peer memory
 *   vt_merkle_level_exchange / vt_digests_publish / vt_digests_wait
 *                     <- the block-root all-gather of a sharded merkle.build,
 *                        fused over peer memory
 *   vt_serialize_f32  <- the FP32 serialization + finiteness check of
 *                        merkle.hash_weights                 merkle.py:155-166
 */
#ifndef VTRAIN_B200_H
#define VTRAIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *vt_stream_t; /* a cudaStream_t; NULL = legacy default stream */

/* status codes */
#define VT_OK 0
#define VT_EINVAL (-1) /* bad argument (size, b_r, alignment, workspace) */
#define VT_ECUDA (-2)  /* CUDA runtime / launch failure, see vt_last_error() */

/* device error bits */
#define VT_ERR_NONFINITE 1      /* "non-finite value" */
#define VT_ERR_RANGE 2          /* rnd(x) > grid_max: "out of representable range" */
#define VT_ERR_RANGE_NEIGHBOR 4 /* |x| > grid_max (neighbour / rev semantics), same text */
#define VT_ERR_BAD_CODE 8       /* code not in {0,1,2}: "invalid direction code" */
#define VT_ERR_BAD_LOG_BYTE 16  /* packed byte > 242: "corrupt log byte" */
#define VT_ERR_BAD_SPARSE 32    /* sparse log not strictly ascending / out of range */
#define VT_ERR_EXCHANGE 64      /* vt_counts_wait: a peer's count did not arrive within 10 s */

/* output kinds for the rounded tensor */
#define VT_OUT_NONE 0
#define VT_OUT_F32 1
#define VT_OUT_F64 2

/* log kinds consumed by vt_replay */
#define VT_LOG_SPARSE 0 /* uint64 words (global_index << 1) | up, strictly ascending */
#define VT_LOG_CODES 1  /* uint8 ternary code per element (0 down, 1 ignore, 2 up) */
#define VT_LOG_PACKED 2 /* .vtrl payload bytes, 5 base-3 digits per byte */

const char *vt_version(void);
const char *vt_last_error(void);
/* host wait for `stream` (cudaStreamSynchronize); VT_ECUDA on a CUDA error */
int vt_stream_synchronize(vt_stream_t stream);
int vt_tile_elems(void); /* elements per CTA tile (shard boundaries align to it) */

/* ---- fused round-and-log (trainer) ------------------------------------ */
size_t vt_round_log_workspace(int64_t n);
/*
 * x[n] FP64 (16-byte aligned) -> out (FP32/FP64, or none) plus any of:
 *   sparse:  entries (global_base + i) << 1 | (code == UP) for every code != 1,
 *            ascending; written at *cursor_in (0 if NULL) + rank, at most
 *            sparse_cap words; *cursor_out (if not NULL) = cursor + count.
 *   codes:   uint8 ternary code per element.
 *   packed:  .vtrl bytes for the element stream starting at log position
 *            log_pos: full 5-digit groups only, byte g covers elements
 *            [head + 5g, head + 5g + 5) with head = (5 - log_pos % 5) % 5
 *            (clipped to n); edge_codes[0..7] receives the head codes then
 *            the tail codes (elements after the last full group).
 * counters[0] += number of codes != 1 (directed count / sparse entry count).
 * Workspace (>= vt_round_log_workspace(n) bytes) must be zero-filled before
 * its first use and then belong to this entry point on one stream: it keeps
 * an epoch counter so the look-back status words need no clearing per call.
 */
int vt_round_log(const double *x, int64_t n, int b_r, double tau, int out_kind, void *out,
                 uint64_t *sparse, int64_t sparse_cap, int64_t global_base,
                 const int64_t *cursor_in, int64_t *cursor_out, uint8_t *codes, uint8_t *packed,
                 int64_t log_pos, uint8_t *edge_codes, int64_t *counters, int32_t *err, void *ws,
                 size_t ws_bytes, vt_stream_t stream);

/* ---- fused replay (auditor) ------------------------------------------- */
size_t vt_replay_workspace(int64_t n);
/*
 * log_kind SPARSE: log = uint64 words, log_len = word count, log_base = global
 *   index of x[0]; counters[1] / counters[2] = first / one-past-last word consumed.
 * log_kind CODES:  log = uint8[n].
 * log_kind PACKED: log = payload bytes, log_base = stream position of x[0],
 *   log_len = payload byte count (bounds).
 * counters[0] = corrections (elements whose output differs from rnd(x)).
 * Workspace (>= vt_replay_workspace(n) bytes, SPARSE only) must be zero-filled
 * before its first use and then belong to this entry point on one stream: it
 * holds the ticket counter of the persistent kernel.
 */
int vt_replay(const double *x, int64_t n, int b_r, int log_kind, const void *log,
              int64_t log_len, int64_t log_base, int out_kind, void *out, int64_t *counters,
              int32_t *err, void *ws, size_t ws_bytes, vt_stream_t stream);

/* ---- elementwise grid helpers ----------------------------------------- */
int vt_grid_neighbors(const double *x, int64_t n, int b_r, double *below, double *above,
                      int32_t *err, vt_stream_t stream);
int vt_exponent_scale(const double *x, int64_t n, double *out, int32_t *err, vt_stream_t stream);
int vt_is_on_grid(const double *x, int64_t n, int b_r, uint8_t *out, vt_stream_t stream);
int vt_norm_distance(const double *x, int64_t n, int b_r, double *out, int32_t *err,
                     vt_stream_t stream);

/* ---- .vtrl codec -------------------------------------------------------- */
int vt_pack5(const uint8_t *codes, int64_t n_groups, uint8_t *out, int32_t *err,
             vt_stream_t stream);
/* entries [pos, pos + n) of the payload stream -> codes[n] */
int vt_unpack5(const uint8_t *payload, int64_t pos, int64_t n, uint8_t *codes, int32_t *err,
               vt_stream_t stream);
int vt_log_validate(const uint8_t *payload, int64_t nbytes, int32_t *err, vt_stream_t stream);
/* counts3[0..2] += histogram of the first n_entries digits */
int vt_log_histogram(const uint8_t *payload, int64_t n_entries, int64_t *counts3, int32_t *err,
                     vt_stream_t stream);

/* ---- adaptive threshold ------------------------------------------------- */
size_t vt_tau_workspace(int64_t n);
/*
 * *key_out = FP64 bit pattern of the (rank+1)-th largest normalized distance
 * p = |x - rnd(x)| / max(scale(x), 2^-126) (radix select; 0 if rank >= n).
 */
int vt_tau_kth_key(const double *x, int64_t n, int b_r, int64_t rank, uint64_t *key_out,
                   int32_t *err, void *ws, size_t ws_bytes, vt_stream_t stream);
/*
 * The same order statistic for one tensor sharded across ranks: begin, then
 * for pass 0..4: this rank's histogram (vt_tau_kth_hist), the caller sums
 * it over the ranks in place (vt_tau_kth_hist_bins(pass) uint32 bins at byte
 * offset vt_tau_kth_hist_offset(pass) of ws, e.g. ncclAllReduce), then the
 * selection (vt_tau_kth_select), identical on every rank.  rank = global
 * 0-based rank from the top; the caller handles rank >= total count.
 */
size_t vt_tau_kth_hist_offset(int pass);
int vt_tau_kth_hist_bins(int pass);
int vt_tau_kth_begin(int64_t rank, uint64_t *key_out, void *ws, size_t ws_bytes, vt_stream_t stream);
int vt_tau_kth_hist(const double *x, int64_t n, int b_r, int pass, int32_t *err, void *ws, size_t ws_bytes,
                    vt_stream_t stream);
int vt_tau_kth_select(int pass, uint64_t *key_out, void *ws, size_t ws_bytes, vt_stream_t stream);
/*
 * Budget form: *key_out = FP64 bits of v', the (budget+1)-th
 * largest p clamped for a bisection inside (tau_lo, tau_hi): tau_lo if
 * v <= tau_lo, +inf if v > tau_hi, else v exactly.  Two streaming passes.
 * *status_out (device int32) = 1 when done, 2 when the selected digit held
 * more candidates than the workspace: the caller then uses vt_tau_kth_key.
 */
int vt_tau_budget_key(const double *x, int64_t n, int b_r, int64_t budget, double tau_lo,
                      double tau_hi, uint64_t *key_out, int32_t *status_out, int32_t *err,
                      void *ws, size_t ws_bytes, vt_stream_t stream);
/*
 * Budget search with no host round trip (protocol.search_tau_budget, the
 * north-star form of protocol.search_tau, pkg/src/vtrain/protocol.py:494-506,
 * SURVEY.md A.4): ONE streaming read of x collects the values of the
 * candidates above a threshold below the expected tau, then one cooperative
 * launch selects the (budget+1)-th largest p among them exactly and runs the
 * 30-step FP64 bisection on the device (the exact multi-pass selection over x
 * runs in the same launch when the candidates cannot decide).  *tau_out
 * (device double) = the returned upper bound; *key_out (device, optional) =
 * FP64 bits of v' (v clamped as for vt_tau_budget_key).  x 32-byte aligned;
 * workspace vt_tau_budget_workspace(n) bytes, 256-byte aligned, zero-filled
 * before first use, one stream at a time.
 */
size_t vt_tau_budget_workspace(int64_t n);
int vt_tau_budget(const double *x, int64_t n, int b_r, int64_t budget, int iters, double *tau_out,
                  uint64_t *key_out, int32_t *err, void *ws, size_t ws_bytes, vt_stream_t stream);
/*
 * Round-and-log with the multi-GPU exchange step fused in (the
 * per-rank log counts all-gathered so each rank knows its offset in the
 * global log).  Same arguments and results as vt_round_log on the sparse path
 * (codes / packed not allowed), plus `xpeers`: a DEVICE array of `world`
 * pointers to every rank's exchange buffer of vt_exchange_words(world)
 * uint64 words (symmetric memory mapped over NVLink, zero-filled once on
 * every rank before first use).  The kernel's last CTA stores this call's
 * entry count into every rank's buffer (st.release.sys), tagged with this
 * rank's exchange sequence number; vt_counts_wait (same stream, later) spins
 * until every rank's count for that sequence number is in this rank's buffer
 * and writes them to counts_out[world] (device), or raises VT_ERR_EXCHANGE
 * in *err after 10 s.  Replaces the ncclAllGather of counts.
 */
size_t vt_exchange_words(int world);
int vt_round_log_exchange(const double *x, int64_t n, int b_r, double tau, int out_kind, void *out,
                          uint64_t *sparse, int64_t sparse_cap, int64_t global_base,
                          int64_t *counters, int32_t *err, void *ws, size_t ws_bytes,
                          uint64_t *const *xpeers, int world, int rank, vt_stream_t stream);
int vt_counts_wait(uint64_t *const *xpeers, int world, int rank, int64_t *counts_out, int32_t *err,
                   vt_stream_t stream);
/*
 * The block-root exchange of the sharded Merkle tree, fused
 * over peer memory like the count exchange.  xpeers: device array of
 * `world` pointers to every rank's buffer of vt_digest_exchange_words(world,
 * n_total) uint64 words (zero-filled once on every rank).  Rank `rank` owns
 * the block roots [dst, dst + n) of the n_total roots of all ranks:
 * vt_merkle_level_exchange hashes its last local level (as vt_merkle_level)
 * and stores every output digest into every rank's buffer; when the roots
 * need no hashing (one node, depth 0, or an empty rank) vt_digests_publish
 * stores them instead.  Either way the kernel's last CTA publishes the
 * rank's arrival (st.release.sys).  vt_digests_wait (same stream, later)
 * waits for every rank's arrival of that exchange and copies the n_total
 * roots, in block order, to out (32 bytes each), or raises VT_ERR_EXCHANGE
 * in *err after 10 s.  Replaces the ncclAllGather of the block roots.
 */
size_t vt_digest_exchange_words(int world, int64_t n_total);
int vt_merkle_level_exchange(const uint8_t *in, int64_t n_in, uint8_t *out, uint64_t *const *xpeers,
                             int world, int rank, int64_t dst, int64_t n_total, vt_stream_t stream);
int vt_digests_publish(const uint8_t *digests, int64_t n, uint64_t *const *xpeers, int world, int rank,
                       int64_t dst, int64_t n_total, vt_stream_t stream);
int vt_digests_wait(uint64_t *const *xpeers, int world, int rank, int64_t n_total, uint8_t *out,
                    int32_t *err, vt_stream_t stream);
/*
 * The same sharded budget search with both exchanges over peer memory and
 * the decision, the digit-key gather, the exact order statistic and the FP64
 * bisection on the device: one call enqueues the whole search (phases = 7)
 * and the host reads *status (0: tau_out holds tau; 1: the candidates could
 * not decide -- run the exact multi-pass path) and *tau_out once.  xpeers:
 * device array of every rank's buffer of vt_tau_shard_exchange_words(world,
 * keys_cap) uint64 words (zero-filled once), own = this rank's; keys_cap
 * bounds one rank's keys in the selected digit (more: *status = 1).  ws:
 * vt_tau_shard_search_x_workspace(n) bytes, 256-byte aligned.  phases picks
 * A (1: candidates + histogram to every rank), B (2: decision + this rank's
 * digit keys to every rank), C (4: gather + selection + bisection); every
 * wait is bounded (VT_ERR_EXCHANGE in *err after 10 s).
 */
size_t vt_tau_shard_exchange_words(int world, int64_t keys_cap);
size_t vt_tau_shard_search_x_workspace(int64_t n);
int vt_tau_shard_search_x(const double *x, int64_t n, int b_r, int64_t n_global, int64_t budget, int iters,
                          uint64_t *const *xpeers, uint64_t *own, int world, int rank, int64_t keys_cap,
                          double *tau_out, int32_t *status, int32_t *err, void *ws, size_t ws_bytes,
                          int phases, vt_stream_t stream);
/*
 * The budget search over ONE tensor sharded across ranks,
 * candidate path: vt_tau_shard_plan gives the global plan (candidate
 * threshold L as FP64 bits, digit shift) -- a function of the global n and
 * budget only; vt_tau_shard_candidates reads this rank's shard once and fills
 * xbuf (int64[2051]: 2048 top-digit counts of the candidate keys, keys above
 * tau_hi, candidates, overflow flag) for the caller to sum over the ranks;
 * vt_tau_shard_digit_keys writes this rank's keys in the selected digit for
 * the caller to gather; the exact order statistic of the gathered keys and
 * the bisection are the caller's (dist.search_tau_budget_sharded).  One
 * workspace (vt_tau_shard_workspace(n), zero-filled once) per rank and
 * stream, used by the two calls of one search.
 */
size_t vt_tau_shard_workspace(int64_t n);
int vt_tau_shard_plan(int64_t n_global, int b_r, int64_t budget, uint64_t *L_key, int *s0);
int vt_tau_shard_candidates(const double *x, int64_t n, int b_r, int64_t n_global, int64_t budget,
                            int64_t *xbuf, int32_t *err, void *ws, size_t ws_bytes, vt_stream_t stream);
int vt_tau_shard_digit_keys(int64_t n, int b_r, int64_t n_global, int64_t budget, int64_t digit,
                            uint64_t *keys_out, int64_t keys_cap, int64_t *count, void *ws, size_t ws_bytes,
                            vt_stream_t stream);
/*
 * Per-tensor adaptive round-and-log with no host round trip: budget select
 * (vt_tau_budget_key), the 30-step search_tau-skeleton bisection on the
 * device, then the sparse round-and-log at that tau.  *tau_out (device
 * double) receives the chosen tau.  Workspace 256-byte aligned, zero-filled
 * before first use.
 */
size_t vt_round_log_adaptive_workspace(int64_t n);
int vt_round_log_adaptive(const double *x, int64_t n, int b_r, int64_t budget, int iters,
                          int out_kind, void *out, uint64_t *sparse, int64_t sparse_cap,
                          int64_t global_base, const int64_t *cursor_in, int64_t *cursor_out,
                          double *tau_out, int64_t *counters, int32_t *err, void *ws,
                          size_t ws_bytes, vt_stream_t stream);
/*
 * The same per-tensor adaptive round-and-log for many independent tensors in
 * a fixed number of launches (one fused rounding pass over all of them, then
 * batched selection / filter kernels), e.g. every intermediate of one step
 * (BASELINE configs[2]).  Per segment, results are identical to
 * vt_round_log_adaptive on that tensor: *tau_out, the log words
 * (global_base + i) << 1 | up at log[0 .. flags[2]), the rounded output,
 * and the error bits OR'ed into (int32_t)flags[0].  flags must be zeroed by
 * the caller.  x 32-byte aligned, out 16 (FP32) / 32 (FP64) byte aligned, not
 * overlapping x.  Workspace 256-byte aligned, zero-filled before first use,
 * vt_round_log_adaptive_batch_workspace(ns, nseg) bytes for the sizes ns[].
 * Replaces a loop of protocol.search_tau-style selection + _TrainerChannel
 * .process calls (protocol.py:198-202, 494-506) over a step's tensors.
 */
typedef struct vt_adaptive_segment {
  const double *x;
  int64_t n;
  int64_t budget;
  void *out;
  uint64_t *log;
  int64_t log_cap;
  int64_t global_base;
  double *tau_out;
  int64_t *flags;
} vt_adaptive_segment;
size_t vt_round_log_adaptive_batch_workspace(const int64_t *ns, int nseg);
int vt_round_log_adaptive_batch(const vt_adaptive_segment *segs, int nseg, int b_r, int iters,
                                int out_kind, void *ws, size_t ws_bytes, vt_stream_t stream);
/*
 * Straddle samples of protocol.collect_divergence_samples (protocol.py:483-490)
 * for two profiles' outputs y1, y2: *count = number of samples (2 per
 * straddling element), *out_min = their minimum (+inf if none),
 * *nan_flag |= 1 if any sample is NaN.  Feeds search_tau's all(p >= tau).
 */
int vt_straddle_min(const double *y1, const double *y2, int64_t n, int b_r, double *out_min,
                    int64_t *count, int32_t *nan_flag, int32_t *err, vt_stream_t stream);
/* out[0] = min over s[n] ignoring NaN (+inf if none), *nan_flag |= 1 if any NaN */
int vt_min_f64(const double *s, int64_t n, double *out, int32_t *nan_flag, vt_stream_t stream);

/* ---- SHA-256 Merkle ---------------------------------------------------- */
/* digests[ceil(nbytes / leaf_bytes)][32] = SHA-256 of each leaf_bytes chunk */
int vt_sha256_leaves(const uint8_t *data, int64_t nbytes, int64_t leaf_bytes, uint8_t *digests,
                     vt_stream_t stream);
/* out[ceil(n_in/2)][32]: SHA-256(in[2i] || in[2i+1]); an unpaired last node is copied */
int vt_merkle_level(const uint8_t *in, int64_t n_in, uint8_t *out, vt_stream_t stream);
/* number of nodes of all levels (leaves included) for n_leaves >= 1 */
int64_t vt_merkle_node_count(int64_t n_leaves);
/*
 * Whole tree over chunked leaves: nodes = level 0 (leaves), then level 1, ...
 * concatenated, nodes_cap >= vt_merkle_node_count(ceil(nbytes / leaf_bytes)).
 */
int vt_merkle_build(const uint8_t *data, int64_t nbytes, int64_t leaf_bytes, uint8_t *nodes,
                    int64_t nodes_cap, vt_stream_t stream);
/*
 * Canonical checkpoint bytes: out[n] = (float)x[n] (RNE, overflow -> +-inf,
 * little-endian), *first_bad = min(*first_bad, index_base + first index i of
 * a non-finite x[i]).  The caller initialises *first_bad (e.g. to INT64_MAX)
 * and passes the chunk's offset in the tensor as index_base.
 * x 32-byte aligned, out 16-byte aligned.
 */
int vt_serialize_f32(const double *x, int64_t n, float *out, int64_t index_base, int64_t *first_bad,
                     vt_stream_t stream);
/* measurement support: blocks x 128 threads x reps compressions of
 * register-resident messages (compute-only SHA-256 ceiling of this chip) */
int vt_sha256_peak_bench(uint32_t *sink, int64_t blocks, int reps, vt_stream_t stream);
/*
 * Integer-pipe peak independent of compress(): register-only chains of the
 * SHA-256 op mix (6 SHF rotates + 4 LOP3 + 4 IADD3 per unit, SURVEY §8d OPS),
 * blocks x 256 threads x reps iterations of vt_int_mix_ops_per_thread_rep()
 * ops each; the denominator of the Merkle "fraction of SHA-256 int peak"
 * (BASELINE.md §3).  fma_adds != 0: the three-input adds as two IMADs each on
 * the FMA pipe (off the ALU pipe, as ptxas balances compress()); the peak of
 * the mix is the faster variant.  sink: one device uint32 (keeps the work).
 */
int vt_int_mix_peak_bench(uint32_t *sink, int64_t blocks, int reps, int fma_adds, vt_stream_t stream);
int64_t vt_int_mix_ops_per_thread_rep(void);

#ifdef __cplusplus
}
#endif
#endif /* VTRAIN_B200_H */
