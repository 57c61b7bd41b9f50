/*
 * samegibbs_b200.h -- C-ABI of the B200-native SAME Gibbs sweep.
 *
 * The reference (samegibbs 0.1.0, pure Python/NumPy) has no FFI layer: its
 * boundary is the Python function API.  Each entry point below replaces one
 * numpy hot site of that API; the Python package paper_1511_06416_b200 binds
 * them with ctypes (INTEGRATION.md shows the binding).  Conventions:
 *
 *   - every pointer argument marked [dev] is device memory, caller-allocated;
 *   - every call is stream-ordered on the caller's cudaStream_t (passed as
 *     void*), never synchronises, and returns an sg_status;
 *   - kernels report data-dependent failures through a device error word
 *     (int32, bit flags SG_ERR_*), which the caller reads after syncing;
 *   - no exceptions, no torch types, no allocation inside the library.
 *
 * Data layout in HBM:
 *   obs    int8  [n][ld_obs]        observed state or -1 (missing) per case
 *   states int8  [n][m][pitch]      lane states; lane (r, c) = replica r of
 *                                   case c (reference lane r*B + c,
 *                                   sampler.py:174-187).  Bit 7 set = latent
 *                                   cell (resampled), low 7 bits = state.
 *   cpt    f64   [cells]            all CPTs, var-major, row-major rows
 *   counts u64   [cells]            integer tallies, same indexing as cpt
 */
#ifndef SAMEGIBBS_B200_H
#define SAMEGIBBS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 2  /* 2: sg_net blanket factor tables, sg_finish read-back and range check, sg_joint_sweep prefetch flag */

typedef enum sg_status {
  SG_OK = 0,
  SG_EINVAL = 1,     /* bad argument (sizes, null pointers, unsupported shape) */
  SG_ECUDA = 2,      /* a CUDA launch failed (sg_last_error() has the text) */
  SG_ECAPACITY = 3   /* shape exceeds a compiled-in capacity */
} sg_status;

/* device error-word bits */
#define SG_ERR_ZERO_SUPPORT 1u      /* a latent cell had all-zero weights (ZeroSupport) */
#define SG_ERR_STATE_RANGE 2u       /* an observed state >= its cardinality */
#define SG_ERR_REJECT_OVERFLOW 4u   /* too many Lemire rejections in one init stream */

/* RNG modes of sg_sweep / sg_init_states */
#define SG_RNG_FAST 0      /* Philox4x32-10 under the fixed key (0x243F6A88, 0x85A308D3), counter
                              (global case, var | quad << 16 | purpose << 28, key lo, key hi):
                              purpose 0 = sweep draw, 1 = initial state; word j of the block is
                              replica 4 * quad + j.  Global cases < 2^32, m <= 16384. */
#define SG_RNG_NUMPY 1     /* numpy Philox4x64-10 stream per variable (bit-exact) */
#define SG_RNG_INJECTED 2  /* caller-supplied fp64 uniforms, reference order */

/* accumulator modes of sg_accumulate */
#define SG_ACC_MOVING 0
#define SG_ACC_EXPONENTIAL 1

/*
 * Network pack: structure of the Bayesian network flattened into device
 * arrays (built once per run by netpack.py from network.py's parents,
 * strides, child links and colour groups; reference sampler.py:190-202,
 * network.py:42-48, 147-180).  All arrays [dev].
 */
typedef struct sg_net {
  int32_t n;              /* variables */
  int32_t num_groups;     /* colour groups */
  int32_t max_card;
  int32_t max_mb;         /* largest Markov blanket */
  int32_t max_group;      /* largest colour group */
  int32_t direct_vars;    /* variables without a conditional table */
  int64_t cells;          /* total CPT cells == count cells */
  int64_t rows;           /* total CPT rows */
  int64_t ptab_size;      /* doubles in the parity conditional table */
  int64_t ftab_size;      /* uint32 in the fast conditional table */
  int64_t table_entries;  /* total Markov-blanket configurations */
  const int32_t* card;        /* [n] */
  const int32_t* group_start; /* [G+1] into order */
  const int32_t* order;       /* [n] variables in colour-group order */
  const int32_t* par_start;   /* [n+1] */
  const int32_t* par_var;     /* [P] parents of v, ascending */
  const int32_t* par_stride;  /* [P] mixed-radix stride (first parent most significant) */
  const int32_t* par_slot;    /* [P] slot of that parent in MB(v) */
  const int32_t* mb_start;    /* [n+1] */
  const int32_t* mb_var;      /* [M] Markov blanket of v, ascending */
  const int32_t* mb_stride;   /* [M] stride of that member in v's table index */
  const int32_t* chl_start;   /* [n+1] child links of v, ascending child */
  const int32_t* chl_var;     /* [K] child */
  const int32_t* chl_vstride; /* [K] stride of v inside the child's row index */
  const int32_t* chl_slot;    /* [K] slot of the child in MB(v) */
  const int32_t* chl_pstart;  /* [K+1] */
  const int32_t* chl_pslot;   /* [Q] slots of the child's other parents */
  const int32_t* chl_pstride; /* [Q] their strides in the child's row index */
  const int64_t* cpt_off;     /* [n] first cell of T_v */
  const int64_t* row_off;     /* [n+1] first row of T_v (rows prefix) */
  const int64_t* tab_entries; /* [n] MB configurations of v's table, 0 = direct */
  const int64_t* tab_start;   /* [n+1] prefix of tab_entries */
  const int64_t* ptab_off;    /* [n] first double of v's parity table */
  const int64_t* ftab_off;    /* [n] first uint32 of v's fast table */
  const int32_t* row_var;     /* [rows] variable owning each CPT row */
  /* joint-state tally: when prod(card) <= SG_JOINT_MAX the sweep histograms
     whole-lane configurations J = sum_v x_v * joint_radix[v] and expands
     them to CPT cells through joint_cell[J][v] (0 disables). */
  int64_t joint_size;
  const int32_t* joint_radix; /* [n] */
  const int32_t* joint_cell;  /* [joint_size][n] */
  /* compact per-variable draw descriptor, SG_DESC_WORDS int32 each:
     card, nmb (-1 = evaluate from CPTs), ftab offset, ptab offset,
     mb_var[SG_DESC_MB], mb_stride[SG_DESC_MB] */
  const int32_t* var_desc;    /* [n][SG_DESC_WORDS] */
  /* factored draw descriptor of v at fac_desc[fac_start[v]] (the weight
     product of sampler.py:226-240 with pre-multiplied indices): card, npar,
     nchl, cpt_off[v]; npar x (parent, stride*card); nchl x (child,
     cpt_off[child], card[child], vstride*card[child], nq, 0, nq x (other
     parent, stride*card[child])); every pair 8-byte aligned */
  const int32_t* fac_start;   /* [n+1] */
  const int32_t* fac_desc;
  /* chunked tally (large models): variables split into runs of consecutive
     variables whose cells fit a shared-memory histogram (SG_TALLY_CHUNK_CELLS);
     a single variable above that gets a run of its own (global atomics) */
  int64_t tally_chunks;
  const int32_t* tally_chunk; /* [tally_chunks+1] first variable of each run */
  /* Every int32 array above lives inside blob32 and every int64 array inside
     blob64 (the pack is two contiguous buffers), so a kernel can stage the
     whole structure in shared memory and rebase the pointers (NULL: not
     packed that way). */
  const int32_t* blob32;
  int64_t blob32_words;
  const int64_t* blob64;
  int64_t blob64_words;
  /* Blanket factor tables of the big-tile sweep (n > 32, cards <= 4; outside
     the blobs; bft_rows = 0: not built).  Row r holds 4 doubles, the CPT cells
     bft_src[2r] + t * (bft_src[2r+1] & (2^26 - 1)) for t < bft_src[2r+1] >> 26
     (zero padded): one factor of a weight product (sampler.py:226-240) as v
     runs over its states.  The program of v at bft_desc[bft_start[v]] (int4
     records): [card, npar, nchl, own row base], ceil(npar/2) x [u, stride, u,
     stride], per child [c, row base, nrec, 0] + nrec x [u, stride, u, stride]
     (child row = base + x_c + sum x_u * stride).  bft is device scratch that
     every large-network sg_sweep rewrites from its cpt argument: sweeps on
     different streams need structs with different bft buffers (the Python
     engine gives each engine its own copy, NetPack.private_ref). */
  int64_t bft_rows;
  const int32_t* bft_start;  /* [n+1] */
  const int32_t* bft_desc;
  const int32_t* bft_src;    /* [bft_rows][2] */
  double* bft;               /* [dev] [bft_rows][4] */
} sg_net;

#define SG_JOINT_MAX 128
#define SG_TALLY_CHUNK_CELLS 12288
#define SG_DESC_MB 8
#define SG_DESC_WORDS (4 + 2 * SG_DESC_MB)

/* A replicated minibatch resident on the device. */
typedef struct sg_batch {
  int8_t* states;           /* [dev] [n][m][pitch] */
  int32_t m;                /* SAME replication factor */
  int32_t cases;            /* B: cases in the minibatch incl. reference padding */
  int32_t pitch;            /* row pitch in cases, multiple of 16, >= cases */
  int32_t num_real;         /* cases with lane weight 1 (c < num_real) */
  int64_t case_base;        /* global index of case 0 (shard offset) for FAST counters */
  const int32_t* rank;      /* [dev] [n][ld_rank] latent rank of (v,c) among the
                               minibatch's latent cases of v (NUMPY / INJECTED) */
  int32_t ld_rank;
  int32_t latent_permille;  /* hint: latent share of the cells x 1000 (0 = unknown); large
                               networks with dense latent cells (>= 800) and m >= 2 take the
                               lane-per-thread sweep, the rest the big-tile sweep */
  const int64_t* nmiss;     /* [dev] [n] latent cases of v in the global minibatch */
} sg_batch;

/* Version of this ABI (SG_ABI_VERSION). */
int sg_abi_version(void);

/* Stream-ordered copy (cudaMemcpyDefault: pinned host <-> device), recorded
   as a memcpy node when `stream` is capturing a CUDA graph. */
int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* cudaMemcpy2DAsync: height rows of width bytes (pitches in bytes). */
int sg_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                    int64_t height, void* stream);

/* Small stream-ordered copy done by a kernel (8-byte aligned); dst may be
   pinned host memory (mapped through unified addressing). */
int sg_copy_small(void* dst, const void* src, int64_t bytes, void* stream);

/* Timing events usable inside CUDA-graph capture (recorded as external
   event nodes while the stream is capturing): create / record / elapsed
   milliseconds / destroy.  Handles are cudaEvent_t values. */
int sg_event_create(uint64_t* ev);
int sg_event_record(uint64_t ev, void* stream);
int sg_event_elapsed(uint64_t start, uint64_t end, float* ms);
int sg_event_destroy(uint64_t ev);

/* Empty kernel of the given launch shape (timing-floor calibration of the
   bench's event measurements). */
int sg_noop(int32_t ctas, int32_t threads, int32_t smem_bytes, void* stream);

/* L2 flush for benchmarks: writes `bytes` of wbuf, then reads `bytes` of
   rbuf [dev] (both > L2), with the sweep's max-shared carveout preference
   (no L1/shared reconfiguration in front of the next timed step). */
int sg_flush_l2(void* wbuf, void* rbuf, int64_t bytes, uint32_t tag, void* stream);

/* Text of the last failing call on this host thread ("" if none). */
const char* sg_last_error(void);

/*
 * Conditional tables: for every variable whose Markov blanket has at most
 * SG table capacity configurations, precompute the reference's fp64
 * full-conditional weights (sampler.py:226-242: parent row, then each child
 * ascending, left-to-right products, numpy pairwise norm) for every blanket
 * configuration.  ptab gets cum[0..card-2], norm per entry (bit-exact draw
 * `u*norm > cum_s`); ftab gets ceil(cum_s/norm * 2^31) thresholds (FAST).
 * ftab holds ftab_size + 1 words: the last one is set non-zero when some
 * entry has no support (all weights zero), which arms the ZeroSupport
 * check in sg_sweep.  Replaces the per-lane gathers of _resample_variable.
 */
int sg_build_tables(const sg_net* net, const double* cpt, double* ptab,
                    uint32_t* ftab, void* stream);

/*
 * Latent ranks: rank[v][c] = #{c' < c : obs[v][c'] < 0} and
 * nmiss[v] = #{c < cases : obs[v][c] < 0}; rank may be NULL (counts only).
 * scratch: [dev] int64 of
 * n * ceil(cases / 4096) words.  Replaces the ordering that
 * np.flatnonzero(values[v] < 0) imposes (sampler.py:180) on the uniforms.
 */
int sg_rank_latent(int32_t n, const int8_t* obs, int32_t ld_obs, int32_t cases,
                   int32_t* rank, int32_t ld_rank, int64_t* nmiss,
                   int64_t* scratch, void* stream);

/*
 * Replicate a minibatch into lane states and draw initial latent states
 * (replicate_minibatch sampler.py:174-187 + init_latent sampler.py:205-214).
 * rng_mode FAST: key = fast_key; NUMPY: keys [dev] [n][2] = stream_key(seed,
 * "latent_init", pass, mb, v), numpy Generator.integers(0, card) (Lemire on
 * 32-bit halves) reproduced bit-exactly.  rej_scratch: [dev] int64 of
 * n * 66 words (NUMPY only).  err: [dev] error word.
 */
int sg_init_states(const sg_net* net, const sg_batch* batch, const int8_t* obs,
                   int32_t ld_obs, int32_t rng_mode, uint64_t fast_key,
                   const uint64_t* keys, int64_t* rej_scratch, int32_t* err,
                   void* stream);

/*
 * One chromatic Gibbs sweep over every lane of the batch (gibbs_pass
 * sampler.py:251-284) and, when counts != NULL, the count tally of the final
 * assignments (tally_counts model.py:148-165, lanes c < num_real only),
 * added into counts (caller zeroes).
 *   FAST:     fast_key = derive_seed(seed, "sweep", pass, mb, s), or read from
 *             fast_key_dev [dev] when that is non-NULL (graph replay)
 *   NUMPY:    keys [dev] [n][2] = stream_key(sweep_seed, "var", v)
 *   INJECTED: uniforms [dev] concatenated per variable (ascending v), each
 *             m*nmiss[v] long in reference lane order; inj_off [dev] [n]
 */
int sg_sweep(const sg_net* net, const sg_batch* batch, const double* cpt,
             const double* ptab, const uint32_t* ftab, int32_t rng_mode,
             uint64_t fast_key, const uint64_t* fast_key_dev, const uint64_t* keys,
             const double* uniforms, const int64_t* inj_off, uint64_t* counts,
             int32_t* err, void* stream);

/* The numpy-stream uniforms of one sweep, generated ahead of it so the
   numpy-parity sweep runs as sg_sweep(SG_RNG_INJECTED, uniforms = out,
   inj_off[v] = v * ld): out[v * ld + i] = random() word i of variable v's
   stream (Philox4x64-10 under keys[2v], keys[2v + 1]; rng.py:16-25,
   sampler.py:245) for i < m * nmiss[v].  Bit-identical to SG_RNG_NUMPY;
   one Philox block per four uniforms instead of one per uniform.
   ld % 4 == 0, ld >= m * cases; out 32-byte aligned, n * ld doubles. */
int sg_np_uniforms(const sg_batch* batch, const uint64_t* keys, int32_t n, double* out, int64_t ld,
                   void* stream);

/* Count tally alone (tally_counts model.py:148-165) over lanes c < num_real. */
int sg_tally(const sg_net* net, const sg_batch* batch, uint64_t* counts,
             void* stream);

/*
 * Weighted tally with arbitrary fp64 lane weights w[m*cases] (the
 * tally_counts API with non-0/1 weights); fp64 atomics, not order-exact.
 */
int sg_tally_weighted(const sg_net* net, const sg_batch* batch,
                      const double* weights, double* counts, void* stream);

/*
 * Count accumulator (update_moving_sum / update_exponential,
 * sampler.py:337-351, CountSet.add/scale model.py:56-62), fp64 in the
 * reference's rounding order.  MOVING: total += -prev (if prev != NULL),
 * total += new.  EXPONENTIAL: total *= decay, total += new.
 */
int sg_accumulate(int32_t mode, double* total, const uint64_t* new_counts,
                  const uint64_t* prev_counts, double decay, int64_t cells,
                  void* stream);

/* Same with fp64 count deltas (CountSet objects that are not integer). */
int sg_accumulate_f64(int32_t mode, double* total, const double* new_counts,
                      const double* prev_counts, double decay, int64_t cells,
                      void* stream);

/* Posterior-mean rows (c + alpha_v) / sum (mean_cpts model.py:188-194), bit-exact. */
int sg_mean_cpts(const sg_net* net, const double* total, const double* alpha,
                 double* cpt_out, void* stream);

/*
 * Dirichlet row draws (sample_cpts model.py:179-185): gamma(c + alpha_v) by
 * Marsaglia-Tsang (shape < 1 boosted), in log space, Philox4x32 keyed by
 * key = derive_seed(seed, "cpt_update", pass, mb).  Statistical parity.
 */
int sg_sample_cpts(const sg_net* net, const double* total, const double* alpha,
                   uint64_t key, const uint64_t* key_dev, double* cpt_out, void* stream);

/*
 * Forward sampling + masking on the device (forward_sample datagen.py:91-107,
 * mask datagen.py:110-121), bit-exact with the reference for dense inputs:
 * keys [dev] [n][2] = stream_key(seed, "forward_sample", v); topo [dev] [n];
 * out int8 [n][ld_out].  mask_key = stream_key(mask_seed, "mask") (two
 * words); hide <= 0 disables masking.  Entry k of the mask stream is
 * (case k / n, variable k % n), the reference's case-major order.
 */
int sg_forward_sample(const sg_net* net, const double* cpt, const int32_t* topo,
                      const uint64_t* keys, int64_t cases, int64_t case_base,
                      int8_t* out, int64_t ld_out, double hide,
                      uint64_t mask_key0, uint64_t mask_key1, void* stream);

/*
 * Packed-lane path for small networks (FAST RNG mode): when the whole lane
 * state fits in one byte (sum of per-variable field widths <= 7), a lane is
 * a uint8 word S; the conditional table of v is indexed by S & mbmask[v];
 * cases are bucketed by latent pattern so warps run one variable loop.
 * Draws and counters equal sg_sweep's FAST mode (same states and counts).
 *   lanes   uint8 [cases][lane_ld]  lane words, slot-major: lane (r, s) at
 *                               s*lane_ld + r; lane_ld = 4, 8, 16 or 32 >= m
 *   pattern uint8 [cases]       latent-variable bit mask of each slot
 *   case_id int32 [cases]       minibatch case held by each slot
 */
#define SG_SMALL_MAXV 7
#define SG_SMALL_MAXBITS 7

typedef struct sg_small {
  int32_t n;          /* variables (<= SG_SMALL_MAXV) */
  int32_t bits;       /* lane-word bits (<= SG_SMALL_MAXBITS) */
  int32_t tab_words;  /* uint32 words of the sparse conditional table */
  int32_t pad_;
  int32_t order[SG_SMALL_MAXV];   /* colour-group order */
  int32_t off[SG_SMALL_MAXV];     /* bit offset of v's field */
  int32_t width[SG_SMALL_MAXV];   /* bit width of v's field */
  uint32_t mbmask[SG_SMALL_MAXV]; /* lane-word bits of v's Markov blanket */
  int32_t card[SG_SMALL_MAXV];
  int32_t toff[SG_SMALL_MAXV];    /* first word of v's sparse table */
  int32_t tstride[SG_SMALL_MAXV]; /* words per lane-word entry: card-1 rounded up to 1, 2 or 4 (aligned) */
} sg_small;

/* Gather sg_build_tables' FAST thresholds into the sparse per-lane-word table
   stab [tab_words]. */
int sg_small_tables(const sg_net* net, const sg_small* sp, const uint32_t* ftab,
                    uint32_t* stab, void* stream);

/* Bucket the minibatch's cases by latent pattern and (init != 0) build their
   lane words with FAST initial draws (same draws as sg_init_states; key
   derive_seed(seed, "latent_init", pass, mb), sampler.py:211 -- read from
   init_key_dev [dev] when it is not NULL, e.g. a CUDA-graph key cursor).
   scratch: [dev] int32 of 128 * 296 + ceil(cases / 2) words. */
int sg_small_prepare(const sg_small* sp, const int8_t* obs, int32_t ld_obs,
                     int32_t cases, int32_t m, int64_t case_base,
                     uint64_t init_key, int32_t init, int32_t* scratch,
                     uint8_t* pattern, int32_t* case_id, uint8_t* lanes,
                     int32_t lane_ld, const uint64_t* init_key_dev, void* stream);

/* Sweep + tally on packed lanes (m <= 32, FAST stream).  jcell [dev]
   [2^bits][n]: CPT cell of each variable for each lane word; zs_flag = ftab +
   ftab_size (arms the ZeroSupport check).  counts may be NULL.  obs (int8
   [n][ld_obs], or NULL) is the minibatch's observation block: its range check
   (sg_check_range) runs inside the same launch. */
int sg_small_sweep(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern,
                   const int32_t* case_id, uint8_t* lanes, int32_t lane_ld,
                   int32_t cases, int32_t num_real, int32_t m, int64_t case_base,
                   uint64_t key, const uint64_t* key_dev, const int32_t* jcell, int32_t cells,
                   uint64_t* counts, const uint32_t* zs_flag,
                   const int8_t* obs, int32_t ld_obs, int32_t* err,
                   void* stream);

/* ---- joint sweep (rng = "joint") ------------------------------------------
   The colour-ordered sweep of one packed lane as ONE draw from its sweep
   transition kernel K_P(S -> S') (csrc/sg_small.cu, "joint sweep"): the
   product, in colour-group order, of the full conditionals the reference's
   gibbs_pass (sampler.py:251-284) draws from one variable at a time.  Same
   Markov kernel, one uniform per lane per sweep.  Replaces
   gibbs_pass + tally_counts (sampler.py:251-304, model.py:148-165) for
   networks whose lane word has <= 6 bits.

   Blob (uint32 [words], 16-byte aligned): a static header written once by
   the host (netpack.joint_plan) -- [0,NP) byte offset of pattern P's rows,
   [NP,2NP) B_P | keep_P << 8 | dep byte offset << 16, then dep_P[2^B_P]
   (latent field bits of compact column j) -- and per pattern 2^bits rows of
   2^B_P cumulative thresholds (2^31 scale) that sg_joint_tables rewrites
   from the CPTs.  Rows are 2^B_P + 1 words apart (odd stride: the lanes of
   a warp probing the same column of different rows hit different banks). */
typedef struct sg_joint {
  int32_t words;         /* uint32 words of the blob (multiple of 4) */
  int32_t header_words;  /* static header words (multiple of 4) */
  int32_t patterns;      /* NP = 2^n latent patterns */
  int32_t max_b;         /* largest B_P (latent bits of one pattern) */
} sg_joint;

/* Rows of the joint blob from the CPTs (one CTA per pattern).  vprob: the
   conditionals sg_step_finish wrote (sg_finish.vprob), or NULL to compute
   them here from cpt. */
int sg_joint_tables(const sg_net* net, const sg_small* sp, const sg_joint* jp,
                    const double* cpt, const double* vprob, uint32_t* jblob, void* stream);

/* Shared memory one joint-sweep CTA needs (eligibility: <= 227 KB). */
int sg_joint_smem(const sg_small* sp, const sg_joint* jp, int32_t cells, int64_t* bytes);

/* Sweep + tally on packed lanes with one uniform per lane (FAST Philox
   counters with purpose 2, v = 0).  Arguments as sg_small_sweep plus the
   joint plan and blob; when zs_flag is armed the per-variable path runs
   instead (exact ZeroSupport semantics).  obs_bits 4 or 2: obs is a packed
   .sgb block (ld_obs bytes per row, 8 / obs_bits cases per byte, case
   k * (8 / obs_bits) + h in bits [h * obs_bits, (h + 1) * obs_bits) of byte
   k, all-ones = missing) and is range-checked in that form; 0 or 8: int8.
   obs_bits | SG_OBS_PREFETCH_ONLY: the block is only pulled into L2 (the
   following sg_step_tail_joint range-checks it, sg_finish.check_obs). */
#define SG_OBS_PREFETCH_ONLY 0x100
int sg_joint_sweep(const sg_small* sp, const sg_joint* jp, const uint32_t* stab,
                   const uint32_t* jblob, const uint8_t* pattern, const int32_t* case_id,
                   uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real,
                   int32_t m, int64_t case_base, uint64_t key, const uint64_t* key_dev,
                   const int32_t* jcell, int32_t cells, uint64_t* counts,
                   const uint32_t* zs_flag, const int8_t* obs, int32_t ld_obs,
                   int32_t obs_bits, int32_t* err, void* stream);

/* Layout switches between packed lanes and sg_batch int8 lane states. */
int sg_small_import(const sg_small* sp, const sg_batch* batch, const int32_t* case_id,
                    uint8_t* lanes, int32_t lane_ld, void* stream);
int sg_small_export(const sg_small* sp, const sg_batch* batch, const int32_t* case_id,
                    const uint8_t* pattern, const uint8_t* lanes, int32_t lane_ld,
                    void* stream);

/*
 * The model-sized tail of a minibatch step, fused: accumulator
 * (sg_accumulate) -> CPT update (sg_mean_cpts / sg_sample_cpts) ->
 * conditional tables (sg_build_tables) -> packed tables (sg_small_tables,
 * when sp != NULL) -> clear the next visit's count buffer -> advance the key
 * cursor (sg_keys_advance).  One single-CTA kernel when the model has at
 * most 4096 cells, else the separate launches; identical results either
 * way.  Optional members may be NULL.
 */
typedef struct sg_finish {
  int32_t acc_mode;           /* SG_ACC_MOVING / SG_ACC_EXPONENTIAL */
  int32_t map_estimate;       /* 1: posterior mean, 0: Dirichlet draw */
  double decay;               /* exponential decay */
  double* total;              /* [dev] [cells] fp64 running total */
  const uint64_t* new_counts; /* [dev] [cells] this visit's tally */
  const uint64_t* prev_counts;/* [dev] [cells] this minibatch's previous tally (moving) or NULL */
  const double* alpha;        /* [dev] [n] prior concentration per variable */
  uint64_t key;               /* Dirichlet key derive_seed(derive_seed(seed,"cpt_update",pass,mb),"sample_cpts") */
  const uint64_t* key_dev;    /* [dev] or NULL: read the key from device memory */
  double* cpt;                /* [dev] [cells] out: CPTs of the next visit */
  double* ptab;               /* [dev] parity table (sg_build_tables) */
  uint32_t* ftab;             /* [dev] fast table + zero-support flag word */
  uint32_t* stab;             /* [dev] packed table (sp != NULL) */
  uint64_t* clear_counts;     /* [dev] [cells] buffer to zero, or NULL */
  const uint64_t* key_table;  /* [dev] [steps][kps] key cursor table, or NULL */
  int32_t* key_index;         /* [dev] cursor */
  int32_t kps;                /* keys per step */
  int32_t flags;              /* SG_FINISH_* bits */
  uint64_t* key_current;      /* [dev] [kps] */
  double* vprob;              /* [dev] [n][2^bits][4] or NULL: the packed path's full conditionals
                                 p_v(x | lane word) for sg_joint_tables (sp != NULL) */
  double* cpt_host;           /* [cells] mapped pinned HOST memory or NULL: the new CPTs are also
                                 stored there by the kernel that writes them (the step's result
                                 read back without a copy node; visible once the call's work is
                                 complete) */
  /* sg_step_tail_joint only (NULL for sg_step_finish): range check of this step's
     observation block (sampler.py:429-430) by the tail's row slices, beside the model
     update (the preceding sg_joint_sweep is then called with obs = NULL): check_obs
     [dev] int8 rows or packed .sgb rows (check_bits 8 / 4 / 2), check_ld bytes per
     row, check_cases cases; out-of-range states set SG_ERR_STATE_RANGE in *check_err. */
  const void* check_obs;
  int32_t check_ld;
  int32_t check_bits;
  int32_t check_cases;
  int32_t* check_err;
} sg_finish;

/* sg_finish.flags: the packed table is the only consumer of this step's
   conditional tables (sp != NULL, packed sweep): build it straight from the
   new CPTs and leave ptab / ftab thresholds stale (the zero-support flag word
   ftab[ftab_size] is still maintained).  Packed words are identical either way. */
#define SG_FINISH_PACKED_ONLY 1

int sg_step_finish(const sg_net* net, const sg_small* sp, const sg_finish* f, void* stream);

/* The whole step tail of the joint path as ONE grid: sg_step_finish (CTA 0;
   f->stab required), which releases sync[0] as soon as the new CPTs are
   written, and sg_joint_tables (CTAs 1.., which wait for that release and
   derive the conditionals of their rows from the CPTs).  f->vprob, when not
   NULL, is scratch for an earlier hand-off: CTA 0 releases the cells' gamma
   draws and every slice normalises the CPT rows itself.  sync:
   [dev] 4 uint32 (hand-off flag, finish count, role ticket, spare), zero
   before the first call; the kernel re-arms them. */
int sg_step_tail_joint(const sg_net* net, const sg_small* sp, const sg_finish* f,
                       const sg_joint* jp, uint32_t* jblob, uint32_t* sync, const void* prep,
                       void* stream);

/* The step tail's static per-slice preparation (the conditionals' gather
   plan and every row entry's index list; they depend only on the network):
   sg_joint_prep fills `prep` [dev] (sg_joint_prep_bytes bytes, 16-byte
   aligned) once, after the blob header is in jblob; sg_step_tail_joint then
   bulk-copies each slice's part instead of building it (prep = NULL: build). */
int sg_joint_prep_bytes(const sg_small* sp, const sg_joint* jp, int64_t* bytes);
int sg_joint_prep(const sg_net* net, const sg_small* sp, const sg_joint* jp, const uint32_t* jblob,
                  void* prep, void* stream);


/* Device key cursor for CUDA-graph replay of minibatch steps:
   current[0..kps) = table[*index * kps ...]; *index += 1.  Kernels given
   key_dev = current + k then read fresh keys on every replay. */
int sg_keys_advance(const uint64_t* table, int32_t* index, int32_t kps,
                    uint64_t* current, void* stream);

/* 4-bit observation rows (.sgb nibble encoding, io.py) -> int8 rows:
   byte j of a packed row holds cases 2j (low nibble) and 2j+1 (high);
   15 = missing -> -1.  Replaces nothing in the reference (its data files
   are text, io.py:105-153); it halves the bytes an out-of-core source moves. */
int sg_unpack_nibbles(const uint8_t* packed, int64_t ld_packed, int8_t* out, int64_t ld_out,
                      int32_t rows, int64_t cases, void* stream);

/* 2-bit .sgb blocks (encoding "crumb", cards <= 3): four cases per byte, case
   4j + h in bits [2h, 2h + 2), 3 = missing -> int8 (-1 = missing). */
int sg_unpack_crumbs(const uint8_t* packed, int64_t ld_packed, int8_t* out, int64_t ld_out,
                     int32_t rows, int64_t cases, void* stream);

/* Largest state of each variable's observed cells (range check, sampler.py:429-430). */
int sg_check_range(const sg_net* net, const int8_t* obs, int32_t ld_obs,
                   int32_t cases, int32_t* err, void* stream);

/* Site keys on the device (replaces rng.stream_key, rng.py:16-20, at its
   per-variable call sites sampler.py:211 and :245, metrics.py:135):
   keys[2i], keys[2i+1] = blake2b-128 of the text
       [decimal(*seed_dev)] prefix decimal(first + i)
   read as two little-endian uint64, for i in [0, count).  seed_dev [dev]
   may be NULL (the caller then formats the seed into prefix), e.g.
   seed_dev = the sweep seed, prefix ":var:" -> stream_key(seed, "var", v). */
#define SG_SITE_TEXT_MAX 88
int sg_site_keys(const uint64_t* seed_dev, const char* prefix, int32_t prefix_len, int64_t first,
                 int32_t count, uint64_t* keys, void* stream);

/* The same BLAKE2b-128 evaluated on the host (no device needed; tests pin it
   to hashlib): out[0..1] = digest words of text[0..len), len <= 128. */
int sg_site_key_host(const char* text, int32_t len, uint64_t* out);

/* predict_missing frequency tally (metrics.py:133-137, np.add.at):
   freq[t][states[t_var[t] * var_stride + t_case[t]] & 0x7F] += 1 for every
   target t; freq int64 [targets][max_card]. */
int sg_predict_tally(const int8_t* states, int64_t var_stride, const int32_t* t_var,
                     const int32_t* t_case, int32_t targets, int32_t max_card, int64_t* freq,
                     int32_t* err, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SAMEGIBBS_B200_H */
