// Packed-lane sweep for small networks (FAST RNG mode).
//
// When every variable's state fits in a bit field and the whole lane fits in
// one byte (sum of field widths <= 7; Koller: 1+1+1+2+1 = 6 bits), a lane is
// a single uint8 word S.  Consequences that make the sweep cheap:
//
//  * the full conditional of v is a function of (S & mbmask_v), so the
//    conditional table is indexed by the masked lane word itself;
//  * the latent pattern of a case is shared by its m replicas; cases are
//    bucketed by pattern once per minibatch (counting sort,
//    sg_small_prepare) so a warp's threads run the same variable loop -- no
//    divergence, and only latent variables cost work;
//  * lane words are stored in quads: 32-bit word (q, s) holds replicas
//    4q..4q+3 of slot s (one byte each), quad rows contiguous over slots.  A
//    thread owns one (slot, quad) word -- coalesced 4-byte loads, few
//    registers, full occupancy to hide the Philox round latency -- and works
//    on its 4 lanes with byte-SIMD masking and bit insertion;
//  * the tally histograms S directly (2^bits joint states, per-thread byte
//    counters), expanded to CPT cells once per CTA.
//
// Layout: lanes uint32 [ceil(m/4)][lane_ld] (lane_ld >= cases words, slots in
// bucketed order; lane (r, s) = byte r%4 of word (r/4, s)); pattern uint8
// [cases]; case_id int32 [cases].
// Counters and draws are identical to the generic kernel's FAST mode
// (Philox4x32 on (case, variable, replica quad)), so both paths produce the
// same states and counts from the same tables (tests/test_gpu_small.py).
#include "sg_finish.cuh"

namespace sg {

static constexpr int SMALL_PATTERNS = 1 << SG_SMALL_MAXV;

// Sparse conditional tables: entry S (S & ~mbmask_v == 0) of v = generic
// table entry of the blanket configuration encoded in S.
__global__ void k_small_tables(const sg_net net, const sg_small sp, const uint32_t* __restrict__ ftab,
                               uint32_t* __restrict__ stab) {
  const int total = sp.n << sp.bits;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
    small_table_entry(net, sp, ftab, stab, i);
}

// Cases are bucketed by latent pattern with a deterministic block partition
// (no hot global atomics): block b of SMALL_PREP_BLOCKS owns the cases
// [b * chunk, (b + 1) * chunk); k_small_count writes its per-pattern counts
// cnt[P][b], k_small_scatter derives each (pattern, block) bucket's first
// slot from them and places the block's cases from there, and
// k_small_init_lanes builds the lanes slot by slot (the order inside a
// block's share of a bucket is irrelevant: results depend on case ids only).
#define SMALL_PREP_BLOCKS 296
__device__ __forceinline__ void small_chunk(int cases, int blocks, int b, int& lo, int& hi) {
  const int chunk = ((cases + blocks - 1) / blocks + 255) & ~255;
  lo = min(cases, b * chunk);
  hi = min(cases, lo + chunk);
}

// Four consecutive cases per thread: one 32-bit load per variable row.
__global__ void __launch_bounds__(1024) k_small_count(const sg_small sp, const int8_t* __restrict__ obs, int ld,
                                                      int cases, uint8_t* __restrict__ pattern_of_case,
                                                      uint8_t* __restrict__ obsw_of_case, int* __restrict__ cnt,
                                                      bool vec4) {
  __shared__ int h[SMALL_PATTERNS];
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int lo, hi;
  small_chunk(cases, gridDim.x, blockIdx.x, lo, hi);  // lo is a multiple of 256
  for (int c0 = lo; c0 < hi; c0 += 4 * int(blockDim.x)) {  // whole warps iterate (warp-aggregated counts below)
    const int c = c0 + 4 * int(threadIdx.x);
    uint32_t P[4] = {0u, 0u, 0u, 0u}, ow[4] = {0u, 0u, 0u, 0u};
    if (c < hi) {
      for (int v = 0; v < sp.n; ++v) {
        const int8_t* row = obs + int64_t(v) * ld + c;
        uint32_t w;
        if (vec4) {  // 4-byte aligned rows: c + 3 < ld since ld >= cases rounded up to 4
          w = *reinterpret_cast<const uint32_t*>(row);
        } else {
          w = 0;
          for (int k = 0; k < 4 && c + k < hi; ++k) w |= uint32_t(uint8_t(row[k])) << (8 * k);
        }
        const int card = sp.card[v], off = sp.off[v];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int o = int(int8_t(w >> (8 * k)));
          P[k] |= uint32_t(o < 0) << v;
          // observed fields of the lane word; out of range -> field 0 (the sweep's range
          // check of this block raises SG_ERR_STATE_RANGE), never a neighbouring field
          if (o >= 0 && o < card) ow[k] |= uint32_t(o) << off;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c + k < hi) {
          pattern_of_case[c + k] = uint8_t(P[k]);
          obsw_of_case[c + k] = uint8_t(ow[k]);
        }
    }
    // one shared-memory atomic per distinct pattern in the warp, per case position
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t Pk = c + k < hi ? P[k] : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, Pk);
      if (Pk != 0xFFFFFFFFu && (threadIdx.x & 31) == uint32_t(__ffs(peers) - 1)) atomicAdd(&h[Pk], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x) cnt[i * gridDim.x + blockIdx.x] = h[i];
}

// Place the block's cases into their pattern buckets (pattern[s], case_id[s]).
// The block's first slot in bucket P = the cases of patterns < P (all
// blocks) + the cases of P in blocks < this one, summed here from the
// per-block counts (no separate scan launch).  Within a warp the cases of one
// pattern claim consecutive slots with one shared atomic.
__global__ void __launch_bounds__(1024) k_small_scatter(const int cases, const uint8_t* __restrict__ pattern_of_case,
                                                        const int* __restrict__ cnt, const int patterns,
                                                        uint8_t* __restrict__ pattern, int32_t* __restrict__ case_id) {
  __shared__ int base[SMALL_PATTERNS], tot[SMALL_PATTERNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nb = gridDim.x, me = blockIdx.x;
  for (int P = warp; P < patterns; P += blockDim.x >> 5) {
    int t = 0, pre = 0;
    // all of a lane's loads in flight together (SMALL_PREP_BLOCKS / 32 of them), not one
    // L2 round trip after another
#pragma unroll
    for (int k = 0; k < (SMALL_PREP_BLOCKS + 31) / 32; ++k) {
      const int b = lane + 32 * k;
      const int x = b < nb ? cnt[P * nb + b] : 0;
      t += x;
      pre += b < me ? x : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
    }
    if (lane == 0) {
      tot[P] = t;
      base[P] = pre;
    }
  }
  __syncthreads();
  if (warp == 0) {  // + the exclusive scan of the pattern totals
    int carry = 0;
    for (int P0 = 0; P0 < patterns; P0 += 32) {
      const int P = P0 + lane;
      const int x = P < patterns ? tot[P] : 0;
      int inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (P < patterns) base[P] += carry + inc - x;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  int lo, hi;
  small_chunk(cases, nb, me, lo, hi);
  for (int c0 = lo; c0 < hi; c0 += blockDim.x) {  // whole warps iterate
    const int c = c0 + int(threadIdx.x);
    const bool valid = c < hi;
    const uint32_t P = valid ? uint32_t(pattern_of_case[c]) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, P);
    const int leader = __ffs(peers) - 1;
    int first = 0;
    if (valid && lane == leader) first = atomicAdd(&base[P], __popc(peers));
    first = __shfl_sync(0xffffffffu, first, leader);
    if (!valid) continue;
    const int s = first + __popc(peers & lanemask_lt());
    SG_DCHECK(P < uint32_t(patterns) && s >= 0 && s < cases);
    pattern[s] = uint8_t(P);
    case_id[s] = c;
  }
}

// Build the lanes of every slot (in bucket order, so a warp's slots share a
// latent pattern and its variable loop does not diverge): observed fields
// from the data, latent fields from the FAST init stream (same draw as
// k_init_states: Philox4x32(key, (case, v, r/4, purpose 1))[r%4] * card >> 32;
// the key's and the case's part of the first round computed once per slot).
template <int N>  // variables (compile-time: the variable loop unrolls, latent tests are warp-uniform)
__global__ void __launch_bounds__(256) k_small_init_lanes(
    const sg_small sp, const uint8_t* __restrict__ obsw_of_case, int cases, int m, int64_t case_base,
    uint64_t init_key, const uint8_t* __restrict__ pattern, const int32_t* __restrict__ case_id,
    uint8_t* __restrict__ lanes, int lane_ld, const uint64_t* __restrict__ init_key_dev) {
  if (init_key_dev) init_key = *init_key_dev;  // graph replay: the key cursor's init key
  const FastKey fk = fast_key(init_key);
  uint32_t* out = reinterpret_cast<uint32_t*>(lanes);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < cases; s += gridDim.x * blockDim.x) {
    const uint32_t P = pattern[s];
    const int c = case_id[s];
    const uint32_t obsw = obsw_of_case[c];
    const FastCase fc = fast_case(fk, uint32_t(case_base + c));
    for (int q = 0; q < (m + 3) / 4; ++q) {
      uint32_t S[4] = {obsw, obsw, obsw, obsw};
#pragma unroll
      for (int v = 0; v < N; ++v) {
        if (!((P >> v) & 1u)) continue;
        const u32x4 w = fast_draw(fc, fast_word(uint32_t(v), uint32_t(q), 1u));
        const uint32_t card = uint32_t(sp.card[v]), off = uint32_t(sp.off[v]);
        // (w * card) >> 32 of the 64-bit product: its high word
        S[0] |= __umulhi(w.a, card) << off;
        S[1] |= __umulhi(w.b, card) << off;
        S[2] |= __umulhi(w.c, card) << off;
        S[3] |= __umulhi(w.d, card) << off;
      }
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) word |= (q * 4 + j < m ? (S[j] & 0xFFu) : 0u) << (8 * j);
      out[int64_t(q) * lane_ld + s] = word;
    }
  }
}

// Layout switches with generic int8 lane states.
__global__ void k_small_import(const sg_small sp, const sg_batch bt, const int32_t* __restrict__ case_id,
                               uint8_t* __restrict__ lanes, int lane_ld) {
  const int64_t total = int64_t(bt.m) * bt.cases;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int s = int(i / bt.m), r = int(i - int64_t(s) * bt.m);
    const int c = case_id[s];
    uint32_t S = 0;
    for (int v = 0; v < sp.n; ++v)
      S |= uint32_t(bt.states[(int64_t(v) * bt.m + r) * bt.pitch + c] & 0x7F) << sp.off[v];
    lanes[(int64_t(r >> 2) * lane_ld + s) * 4 + (r & 3)] = uint8_t(S);
  }
}

__global__ void k_small_export(const sg_small sp, const sg_batch bt, const int32_t* __restrict__ case_id,
                               const uint8_t* __restrict__ pattern, const uint8_t* __restrict__ lanes, int lane_ld) {
  const int64_t total = int64_t(bt.m) * bt.cases;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int s = int(i / bt.m), r = int(i - int64_t(s) * bt.m);
    const int c = case_id[s];
    const uint32_t S = lanes[(int64_t(r >> 2) * lane_ld + s) * 4 + (r & 3)];
    const uint32_t P = pattern[s];
    for (int v = 0; v < sp.n; ++v)
      bt.states[(int64_t(v) * bt.m + r) * bt.pitch + c] =
          int8_t(small_field(S, sp, v) | (((P >> v) & 1u) ? 0x80 : 0));
  }
}

__device__ __forceinline__ uint32_t byte_of(uint32_t w, int j) { return __byte_perm(w, 0u, 0x4440 | j); }

#ifndef SG_SMALL_MINB
#define SG_SMALL_MINB(QG) ((QG) <= 3 ? 4 : 3)  // CTAs per SM the register budget targets (64 regs: no spills up to QG = 3)
#endif
#ifndef SG_VAR_UNROLL
#define SG_VAR_UNROLL 1
#endif
// Colour-position loop unrolling.  1 (a loop) measured faster on B200 than a
// full unroll: the unrolled body (~8.3k SASS instructions for N=5, QG=3)
// overflows the instruction cache; the loop (~3.4k) does not.
constexpr int kVarUnroll = SG_VAR_UNROLL;

// u >= t as 0/1 for 31-bit u and thresholds t <= 2^31 (sentinel 0xFFFFFFFF never passes).
__device__ __forceinline__ uint32_t ge(uint32_t u, uint32_t t) { return u >= t ? 1u : 0u; }

// Per-variable constants in colour order, passed by value so that every use
// is a constant-bank operand with an immediate offset (no dynamic indexing,
// no registers held across the unit loop).
struct SmallOrd {
  uint32_t var[SG_SMALL_MAXV];   // variable at colour position i (its pattern bit, counter word)
  uint32_t sh[SG_SMALL_MAXV];    // field offset
  uint32_t k1[SG_SMALL_MAXV];    // card - 1 (1..3)
  uint32_t msk[SG_SMALL_MAXV];   // blanket mask, replicated into the 4 bytes
  uint32_t clr[SG_SMALL_MAXV];   // ~field mask, replicated
  uint32_t toff[SG_SMALL_MAXV];  // table offset (words)
};

// Quad geometry of one thread: quads q0 .. q0 + QG - 1 of its slot.  Quads
// past the last real one alias it (same word, same draws; never stored or
// tallied); only the last real quad can have fewer than 4 real lanes.
struct QuadSet {
  uint32_t row0;    // word offset of quad q0's row
  uint32_t ld;      // lane_ld (words between quad rows)
  uint32_t q0w;     // q0 << 16 (counter word)
  int last;         // index (0-based in the group) of the last real quad
  int last_nl;      // real lanes of that quad (1..4)
  uint32_t last_valid;
};

// One byte counter += 1 at shared address a (a thread's own slot: no races).
__device__ __forceinline__ void hist_inc(uint32_t a) {
  asm volatile("{\n\t.reg .u16 t;\n\tld.shared.u8 t, [%0];\n\tadd.u16 t, t, 1;\n\tst.shared.u8 [%0], t;\n\t}"
               :: "r"(a));
}

// First slot of this thread in the joint sweep: warp-major across the CTAs
// ((warp * grid + cta) * 32 + lane, stride grid * NT), so the ragged last
// wave of 32-slot chunks is spread over every CTA instead of the first ones.
__device__ __forceinline__ int joint_first_slot() {
  return int(((threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32u + (threadIdx.x & 31u));
}

// Tally of the joint sweep: per-warp u32 histograms (65 bins: 64 lane
// states + a trash bin) updated with shared-memory reductions.  Lanes that
// must not count (past m, alias quads, padding cases) carry state 64 in
// their tally byte, so the update needs no branch.
__device__ __forceinline__ void joint_count(uint32_t base, uint32_t state) {
  SG_DCHECK(state < 65u);  // kJointBins
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + state * 4u) : "memory");
}
static constexpr int kJointBins = 65;

// Walk this thread's slots: per latent variable (colour order), QG
// independent Philox blocks (one per quad, sharing the case's first round),
// then per quad 4 table lookups + compares and one byte-SIMD insert.
template <int N, int QG, bool ARMED, int NT = SG_THREADS, bool RED = false>
__device__ __forceinline__ bool small_units(const SmallOrd& o, const QuadSet& qs, const uint32_t* stab,
                                            uint32_t* lanes, const uint8_t* __restrict__ pattern,
                                            const int32_t* __restrict__ case_id, uint32_t hist_a, int cases,
                                            int num_real, int64_t case_base, const FastKey& fk, bool counts,
                                            const uint32_t (&nw0)[QG], uint32_t nP0, int nc0) {
  const int stride = gridDim.x * NT;
  bool zs = false;
  int s = RED ? joint_first_slot() : int(blockIdx.x * NT + threadIdx.x);
  uint32_t nw[QG], nP = nP0;
  int nc = nc0;
#pragma unroll
  for (int g = 0; g < QG; ++g) nw[g] = nw0[g];
  uint32_t* rows = lanes + qs.row0;
  for (; s < cases; s += stride) {
    uint32_t w[QG];
#pragma unroll
    for (int g = 0; g < QG; ++g) w[g] = nw[g];
    const uint32_t P = nP;
    const int c = nc;
    const int sn = s + stride;
    if (sn < cases) {  // prefetch the next slot while this one computes
#pragma unroll
      for (int g = 0; g < QG; ++g) nw[g] = rows[min(g, qs.last) * qs.ld + sn];
      nP = pattern[sn];
      nc = case_id[sn];
    }
    const FastCase fc = fast_case(fk, uint32_t(case_base + c));
#pragma unroll kVarUnroll
    for (int i = 0; i < N; ++i) {
      if (!((P >> o.var[i]) & 1u)) continue;  // warp-uniform: slots are bucketed by pattern
      u32x4 r[QG];
#pragma unroll
      for (int g = 0; g < QG; ++g) r[g] = fast_draw(fc, o.var[i] | (qs.q0w + (uint32_t(min(g, qs.last)) << 16)));
      const uint32_t* tv = stab + o.toff[i];
#pragma unroll
      for (int g = 0; g < QG; ++g) {
        const uint32_t u[4] = {r[g].a >> 1, r[g].b >> 1, r[g].c >> 1, r[g].d >> 1};
        const uint32_t wm = w[g] & o.msk[i];
        const int nl = g < qs.last ? 4 : (g == qs.last ? qs.last_nl : 0);
        uint32_t xs[4];
        if (o.k1[i] == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t t = tv[byte_of(wm, j)];
            if (ARMED && j < nl && t == 0xFFFFFFFFu) zs = true;
            xs[j] = ge(u[j], t);
          }
        } else if (o.k1[i] == 2) {
          const uint2* t2 = reinterpret_cast<const uint2*>(tv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint2 t = t2[byte_of(wm, j)];
            if (ARMED && j < nl && t.x == 0xFFFFFFFFu) zs = true;
            xs[j] = ge(u[j], t.x) + ge(u[j], t.y);
          }
        } else {
          const uint4* t4 = reinterpret_cast<const uint4*>(tv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 t = t4[byte_of(wm, j)];  // card 4: three thresholds + padding
            if (ARMED && j < nl && t.x == 0xFFFFFFFFu) zs = true;
            xs[j] = ge(u[j], t.x) + ge(u[j], t.y) + ge(u[j], t.z);
          }
        }
        const uint32_t x4 = __byte_perm(__byte_perm(xs[0], xs[1], 0x0040), __byte_perm(xs[2], xs[3], 0x0040), 0x5410);
        w[g] = (w[g] & o.clr[i]) | (x4 << o.sh[i]);
      }
    }
    const bool tally = counts && c < num_real;
#pragma unroll
    for (int g = 0; g < QG; ++g) {
      if (g > qs.last) break;  // aliases: nothing to store or count
      const bool full = g < qs.last || qs.last_nl == 4;
      const uint32_t wg = full ? w[g] : (w[g] & qs.last_valid);
      rows[g * qs.ld + s] = wg;
      if (tally) {
        if (full) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (RED) joint_count(hist_a, byte_of(wg, j));
            else hist_inc(hist_a + byte_of(wg, j) * NT);
          }
        } else {
          for (int j = 0; j < qs.last_nl; ++j) {
            if (RED) joint_count(hist_a, byte_of(wg, j));
            else hist_inc(hist_a + byte_of(wg, j) * NT);
          }
        }
      }
    }
  }
  return zs;
}

// The minibatch's range check (sampler.py:429-430) spread over the whole
// grid, one 16-byte load per thread and row at a time (no divisions): int8
// rows (-1 = missing; bytes compared as signed SIMD lanes against card - 1)
// or packed .sgb rows (nib = 4 / 2 bits per case, all-ones = missing).
// Sets SG_ERR_STATE_RANGE.
template <int NT>
__device__ __forceinline__ void obs_range_check(const sg_small& sp, const int8_t* __restrict__ obs, int ld_obs,
                                                int cases, int32_t* err, int nib) {
  obs_range_check_range(sp, obs, ld_obs, cases, err, nib, (blockIdx.y * gridDim.x + blockIdx.x) * NT + threadIdx.x,
                        gridDim.x * gridDim.y * NT);
}

// The common end of both packed sweeps: ZeroSupport word, the minibatch's
// range check (sampler.py:429-430) spread over the whole grid, and the
// joint-state histogram (per-thread byte counters, hist8[J * NT + slot])
// expanded to CPT cells through jcell and flushed with one global atomic per
// touched cell.
template <int N, int NT>
__device__ __forceinline__ void small_epilogue(const sg_small& sp, bool zs, const uint8_t* hist8, uint32_t* cellacc,
                                               const int32_t* __restrict__ jcell, int cells,
                                               unsigned long long* __restrict__ counts,
                                               const int8_t* __restrict__ obs, int ld_obs, int cases,
                                               int32_t* err, int nib = 0) {
  const int tid = threadIdx.x;
  if (zs) atomicOr(err, int(SG_ERR_ZERO_SUPPORT));
  obs_range_check<NT>(sp, obs, ld_obs, cases, err, nib);
  if (!counts) return;
  __syncthreads();
  const int warp = tid >> 5, lane_id = tid & 31;
  for (int J = warp; J < (1 << sp.bits); J += NT / 32) {
    const uint32_t* hrow = reinterpret_cast<const uint32_t*>(hist8 + J * NT);
    int sum = 0;
#pragma unroll
    for (int k = 0; k < NT / 128; ++k) sum = __dp4a(int(hrow[lane_id + 32 * k]), 0x01010101, sum);
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o2);
    if (sum && lane_id < sp.n) atomicAdd(cellacc + __ldg(jcell + J * sp.n + lane_id), uint32_t(sum));
  }
  __syncthreads();
  for (int cell = tid; cell < cells; cell += NT)
    if (cellacc[cell]) atomicAdd(counts + cell, (unsigned long long)cellacc[cell]);
}


// The sweep.  Grid (x: slot blocks, y: quad groups of QG quads).  A thread
// owns the QG lane words of a slot (QG x 4 replicas of one case).
template <int N, int QG>
__global__ void __launch_bounds__(SG_THREADS, SG_SMALL_MINB(QG))
k_small_sweep(const sg_small sp, const SmallOrd o, const uint32_t* stab_g,
              const uint8_t* __restrict__ pattern, const int32_t* __restrict__ case_id, uint32_t* __restrict__ lanes,
              int lane_ld, int cases, int num_real, int m, int64_t case_base, uint64_t key,
              const uint64_t* key_dev, const int32_t* __restrict__ jcell, int cells,
              unsigned long long* __restrict__ counts, const uint32_t* zs_flag,
              const int8_t* __restrict__ obs, int ld_obs, int32_t* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* stab = reinterpret_cast<uint32_t*>(smem);
  uint8_t* hist8 = smem + ((sp.tab_words * 4 + 15) & ~15);
  uint32_t* cellacc = reinterpret_cast<uint32_t*>(hist8 + (SG_THREADS << sp.bits));
  const int tid = threadIdx.x;
  const int Q = (m + 3) >> 2;
  const int q0 = blockIdx.y * QG;
  const int last = min(QG - 1, Q - 1 - q0);
  // PDL prologue: the step tail that follows may start staging its static
  // data now; this kernel's own prologue (counters, first slot's lane words,
  // pattern and case id -- none of them written by the preceding tail) runs
  // before waiting for that tail's tables, key and cleared counts.
  pdl_trigger();
  if (counts) {
    uint32_t* h32 = reinterpret_cast<uint32_t*>(hist8);
    for (int i = tid; i < (SG_THREADS << sp.bits) / 4; i += SG_THREADS) h32[i] = 0;
    for (int i = tid; i < cells; i += SG_THREADS) cellacc[i] = 0;
  }
  uint32_t nw0[QG] = {};
  uint32_t nP0 = 0;
  int nc0 = 0;
  {
    const int s0 = blockIdx.x * SG_THREADS + tid;
    if (s0 < cases) {
      const uint32_t* r0p = lanes + int64_t(q0) * lane_ld;
#pragma unroll
      for (int g = 0; g < QG; ++g) nw0[g] = r0p[int64_t(min(g, last)) * lane_ld + s0];
      nP0 = pattern[s0];
      nc0 = case_id[s0];
    }
  }
  pdl_wait();
  for (int i = tid; i < sp.tab_words; i += SG_THREADS) stab[i] = stab_g[i];
  const bool armed = zs_flag && *zs_flag != 0u;
  QuadSet qs;
  qs.row0 = uint32_t(q0) * uint32_t(lane_ld);
  qs.ld = uint32_t(lane_ld);
  qs.q0w = uint32_t(q0) << 16;
  qs.last = last;
  qs.last_nl = min(4, m - 4 * (q0 + qs.last));
  qs.last_valid = qs.last_nl >= 4 ? 0xFFFFFFFFu : ((1u << (8 * qs.last_nl)) - 1u);
  const int slot = ((tid & 31) << 2) | ((tid >> 5) & 3) | ((tid >> 7) << 7);
  const uint32_t hist_a = uint32_t(__cvta_generic_to_shared(hist8)) + uint32_t(slot);
  const FastKey fk = fast_key(key_dev ? *key_dev : key);
  __syncthreads();
  const bool zs = armed ? small_units<N, QG, true>(o, qs, stab, lanes, pattern, case_id, hist_a, cases, num_real,
                                                   case_base, fk, counts != nullptr, nw0, nP0, nc0)
                        : small_units<N, QG, false>(o, qs, stab, lanes, pattern, case_id, hist_a, cases, num_real,
                                                    case_base, fk, counts != nullptr, nw0, nP0, nc0);
  small_epilogue<N, SG_THREADS>(sp, zs, hist8, cellacc, jcell, cells, counts, obs, ld_obs, cases, err);
}

// Resident CTAs of one sweep instance on the whole device (one full wave).
template <int N, int QG>
static int resident_ctas(size_t smem) {
  static size_t cached_smem = ~size_t(0);
  static int cached = 0;
  if (smem != cached_smem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small_sweep<N, QG>, SG_THREADS, smem);
    cached = sms * std::max(1, per_sm);
    cached_smem = smem;
  }
  return cached;
}

// Quad groups: QG = the quads one thread carries (<= 4, registers), groups =
// ceil(Q / QG) grid rows.
static void quad_groups(int m, int* qg, int* groups) {
  const int Q = (m + 3) / 4;
  *groups = (Q + 3) / 4;
  *qg = (Q + *groups - 1) / *groups;
}

template <int N, int QG>
static void launch_small(const sg_small& sp, const SmallOrd& o, int groups, size_t smem, cudaStream_t st,
                         const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id, uint32_t* lanes,
                         int lane_ld, int cases, int num_real, int m, int64_t case_base, uint64_t key,
                         const uint64_t* key_dev, const int32_t* jcell, int cells, uint64_t* counts,
                         const uint32_t* zs_flag, const int8_t* obs, int ld_obs, int32_t* err) {
  static size_t configured[SG_MAX_DEVICES] = {};  // once per device (keeps graph capture free of attribute calls)
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_small_sweep<N, QG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  // one wave over the quad groups (every CTA strides over the pattern-sorted
  // slots, so unit costs balance), but enough CTAs that no thread's byte
  // counters see more than 255 increments: <= 255 / (4 QG) slots per thread
  const int64_t per_thread = 255 / (4 * QG);
  const int64_t need = (int64_t(cases) + SG_THREADS * per_thread - 1) / (SG_THREADS * per_thread);
  const int64_t fill = (int64_t(cases) + SG_THREADS - 1) / SG_THREADS;
  const int64_t want = std::max<int64_t>(resident_ctas<N, QG>(smem) / groups, need);
  const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>(want, fill))), unsigned(groups));
  // PDL: the sweep's prologue overlaps the preceding step tail (pdl_wait)
  launch_pdl(k_small_sweep<N, QG>, grid, dim3(SG_THREADS), smem, st, sp, o, stab, pattern, case_id, lanes, lane_ld,
             cases, num_real, m, case_base, key, key_dev, jcell, cells, reinterpret_cast<unsigned long long*>(counts),
             zs_flag, obs, ld_obs, err);
}

static size_t small_smem(const sg_small& sp, int cells) {
  return size_t((sp.tab_words * 4 + 15) & ~15) + (size_t(SG_THREADS) << sp.bits) + size_t(cells) * 4 + 16;
}

static SmallOrd small_ord(const sg_small& sp) {
  SmallOrd o{};
  for (int i = sp.n; i < SG_SMALL_MAXV; ++i) o.var[i] = 31u;  // padding: never a latent-pattern bit
  for (int i = 0; i < sp.n; ++i) {
    const int v = sp.order[i];
    o.var[i] = uint32_t(v);
    o.sh[i] = uint32_t(sp.off[v]);
    o.k1[i] = uint32_t(sp.card[v] - 1);
    o.msk[i] = sp.mbmask[v] * 0x01010101u;
    o.clr[i] = ~((((1u << sp.width[v]) - 1u) << sp.off[v]) * 0x01010101u);
    o.toff[i] = uint32_t(sp.toff[v]);
  }
  return o;
}



// ============================================================ joint sweep
//
// rng = "joint" (SG_RNG_JOINT): the whole colour-ordered sweep of one lane
// drawn with ONE uniform.  For a lane word S and latent pattern P the sweep
// (reference gibbs_pass, sampler.py:251-284: colour groups in order, each
// latent variable v drawn from its full conditional given the current
// blanket) is a Markov kernel K_P(S -> S') over the 2^B_P values of the
// latent fields, B_P = sum of the latent variables' field widths:
//
//   K_P(S -> S') = prod_{v latent, colour order} p_v(S'_v | cur_v),
//   cur_v = S with the fields of the variables drawn before v replaced by S'.
//
// k_joint_tables tabulates every row (P, S) of K as an alias table of 2^B_P
// entries (joint_alias_row: integer column masses summing to 2^32); the
// sweep draws one 32-bit uniform per lane and reads ONE entry of its row in
// shared memory (column = top B_P bits, primary-or-alias on the rest) plus
// the column's latent field bits.  Same transition kernel as the
// per-variable sweep up to the 2^-32 quantisation of the row's cumulative
// sums, 1 uniform per lane instead of one per latent variable, 2 dependent
// shared loads instead of 4 table lookups per latent variable (or the
// B_P-level binary search of a cumulative row).  When any conditional has zero
// support (zs_flag armed) the kernel runs the per-variable path instead, so
// ZeroSupport is detected exactly where the reference detects it.
//
// Blob (uint32 words, built on the host once -- netpack.joint_plan -- except
// the rows, which k_joint_tables rewrites after every CPT update):
//   [0, NP)        byte offset of row 0 of pattern P
//   [NP, 2NP)      B_P | keep_P << 8 | (byte offset of dep_P) << 16
//   dep_P[j]       latent field bits of compact column j (pdep(j, latent mask))
//   rows_P[S][j]   alias entries (primary << B_P | alias), 2^bits rows of 2^B_P + 1 words

#ifndef SG_JOINT_THREADS
#define SG_JOINT_THREADS 1024
#endif
#define SG_JOINT_PURPOSE 2u
#define SG_JOINT_MAXB 6

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SG_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> this CTA's shared memory, completion on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Alias draw from a row (joint_alias_row): column i = top B bits of the
// 32-bit uniform; keep it when the low 32 - B bits are below its primary
// mass, else take its alias.  One LDS of the entry, one of the column's
// latent field bits (dep): two dependent shared loads per lane.
template <int B>
__device__ __forceinline__ uint32_t joint_alias_col(uint32_t row, uint32_t u, uint32_t lim) {
  const uint32_t i = u >> (32 - B);
  SG_DCHECK(row + (i << 2) + 4 <= lim);
  uint32_t e;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(row + (i << 2)));
  const uint32_t f = u << B;                 // the low 32 - B bits, left-aligned
  const uint32_t thr = e & ~((1u << B) - 1u);  // primary << B
  return f < thr ? i : (e & ((1u << B) - 1u));
}

// The QG quads of one slot: per lane one 32-bit uniform (word j of the
// quad's Philox block), one alias draw, one dep lookup.  Straight-line over
// all 4 x QG lanes (no per-lane branches) so the compiler interleaves the
// independent chains; lanes past m and alias quads compute garbage that is
// never stored or tallied.  row0 / dep0: shared-window addresses.
template <int B, int QG, int NL>
__device__ __forceinline__ void joint_quads(uint32_t (&w)[QG], const u32x4 (&r)[QG], uint32_t row0, uint32_t dep0,
                                            uint32_t keep, uint32_t lim) {
  constexpr uint32_t kRowBytes = ((1u << B) + 1u) * 4u;  // rows 2^B + 1 words apart (odd: lanes drawing
                                                        // the same column of different rows use different banks)
#pragma unroll
  for (int g = 0; g < QG; ++g) {
    const uint32_t u[4] = {r[g].a, r[g].b, r[g].c, r[g].d};
    uint32_t xs[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (g == QG - 1 && j >= NL) continue;  // compile time: lanes past m in the last quad
      const uint32_t S = byte_of(w[g], j);
#ifdef SG_EXP_NOSEARCH  // timing experiment only: the column straight from the uniform (wrong results)
      const uint32_t col = u[j] >> (32 - B);
#else
      const uint32_t col = joint_alias_col<B>(row0 + S * kRowBytes, u[j], lim);
#endif
      uint32_t lat;
      SG_DCHECK(col < (1u << B) && dep0 + (col << 2) + 4 <= lim);
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lat) : "r"(dep0 + (col << 2)));
      xs[j] = (S & keep) | lat;
    }
    w[g] = __byte_perm(__byte_perm(xs[0], xs[1], 0x0040), __byte_perm(xs[2], xs[3], 0x0040), 0x5410);
  }
}

// NL: lanes of quad QG-1 (m - 4 * (Q - 1) when this CTA row holds the last
// quad, else 4); lanes past it are neither drawn nor tallied.
template <int QG, int NT, int NL>
__device__ __forceinline__ void joint_units(const QuadSet& qs, const unsigned char* blob, int np, uint32_t* lanes,
                                            const uint8_t* __restrict__ pattern, const int32_t* __restrict__ case_id,
                                            uint32_t hist_a, int cases, int num_real,
                                            int64_t case_base, const FastKey& fk, bool counts,
                                            const uint32_t (&nw0)[QG], uint32_t nP0, int nc0, uint32_t blob_bytes) {
  const uint32_t* info = reinterpret_cast<const uint32_t*>(blob);
  const int stride = gridDim.x * NT;
  int s = joint_first_slot();
  uint32_t nw[QG], nP = nP0;
  int nc = nc0;
#pragma unroll
  for (int g = 0; g < QG; ++g) nw[g] = nw0[g];
  // lanes that exist: 4 per quad before the last, last_nl in the last, none in aliases
  // per quad: 0x40 in the bytes of lanes that do not exist (tally -> trash row 64)
  uint32_t trash[QG];
#pragma unroll
  for (int g = 0; g < QG; ++g)
    trash[g] = g < qs.last ? 0u : g == qs.last ? (0x40404040u & ~qs.last_valid) : 0x40404040u;
  // word offset of each quad's row (alias quads read the last real one): 32-bit
  // indices, so every access is one add + one IMAD.WIDE.U32
  uint32_t roff[QG];
#pragma unroll
  for (int g = 0; g < QG; ++g) roff[g] = qs.row0 + uint32_t(min(g, qs.last)) * qs.ld;
  for (; s < cases; s += stride) {
    uint32_t w[QG];
#pragma unroll
    for (int g = 0; g < QG; ++g) w[g] = nw[g];
    const uint32_t P = nP;
    const int c = nc;
    const int sn = s + stride;
    if (sn < cases) {  // prefetch the next slot while this one computes
      const uint32_t usn = uint32_t(sn);
#pragma unroll
      for (int g = 0; g < QG; ++g) nw[g] = lanes[roff[g] + usn];
      nP = pattern[usn];
      nc = case_id[usn];
    }
    SG_DCHECK(P < uint32_t(np) && uint32_t(s) < qs.ld);
    const uint32_t meta = info[np + P];
    const int B = int(meta & 0xFFu);
    if (B) {  // warp-uniform: slots are bucketed by pattern
      const FastCase fc = fast_case(fk, uint32_t(case_base + c));
      u32x4 r[QG];
#pragma unroll
      for (int g = 0; g < QG; ++g) {
#ifdef SG_EXP_NOPHILOX  // timing experiment only: a cheap hash instead of Philox (wrong stream)
        const uint32_t h0 = (fc.x2 ^ (uint32_t(g) * 0x9E3779B9u)) * 0x85EBCA6Bu;
        r[g] = u32x4{h0, h0 * 0xC2B2AE35u, h0 ^ 0x27D4EB2Fu, h0 * 0x165667B1u};
#else
        r[g] = fast_draw(fc, (SG_JOINT_PURPOSE << 28) | (qs.q0w + (uint32_t(min(g, qs.last)) << 16)));
#endif
      }
      const uint32_t row0 = smem_u32(blob) + info[P];
      const uint32_t dep0 = smem_u32(blob) + (meta >> 16);
      const uint32_t keep = (meta >> 8) & 0xFFu;
      [[maybe_unused]] const uint32_t lim = smem_u32(blob) + blob_bytes;
      switch (B) {
        case 1: joint_quads<1, QG, NL>(w, r, row0, dep0, keep, lim); break;
        case 2: joint_quads<2, QG, NL>(w, r, row0, dep0, keep, lim); break;
        case 3: joint_quads<3, QG, NL>(w, r, row0, dep0, keep, lim); break;
        case 4: joint_quads<4, QG, NL>(w, r, row0, dep0, keep, lim); break;
        case 5: joint_quads<5, QG, NL>(w, r, row0, dep0, keep, lim); break;
        default: joint_quads<6, QG, NL>(w, r, row0, dep0, keep, lim); break;
      }
    }
    const bool real_case = c < num_real;
#pragma unroll
    for (int g = 0; g < QG; ++g) {
      const uint32_t wg = w[g] & (g < qs.last ? 0xFFFFFFFFu : qs.last_valid);
      if (g <= qs.last) lanes[roff[g] + uint32_t(s)] = wg;
      if (counts) {
        // padded cases (c >= num_real) and alias quads (g > last): every lane to the trash
        // bin 64 (OR-ing 0x40 into a lane word would index bins 64..127, past this warp's 65)
        const uint32_t wt = (real_case && g <= qs.last) ? (wg | trash[g]) : 0x40404040u;
#ifndef SG_EXP_NOTALLY  // timing experiment only: no tally
#pragma unroll
        for (int j = 0; j < (g == QG - 1 ? NL : 4); ++j) joint_count(hist_a, byte_of(wt, j));
#endif
      }
    }
  }
}

__host__ __device__ inline size_t joint_smem(const sg_small& sp, const sg_joint& jp, int cells) {
  return size_t(jp.words) * 4 + size_t((sp.tab_words * 4 + 15) & ~15) + size_t(SG_JOINT_THREADS / 32) * 65 * 4 +
         size_t((cells * 4 + 15) & ~15) + 16;
}

// One CTA per SM (1024 threads: the register file) with the blob (Koller:
// 109 KB) and per-warp tally bins in shared memory.  NL: lanes of the final
// quad (m - 4 * (Q - 1)).
#ifdef SG_FINISH_TRACE
__device__ unsigned long long g_sweep_trace[8 * 160];
extern "C" int sg_debug_sweep_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_sweep_trace, sizeof(g_sweep_trace)) == cudaSuccess ? 0 : 2;
}
#define SG_SWEEP_STAMP(k)                                                 \
  do {                                                                    \
    if (threadIdx.x == 0 && blockIdx.y == 0) {                            \
      unsigned long long t_;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      g_sweep_trace[blockIdx.x * 8 + (k)] = t_;                           \
    }                                                                     \
  } while (0)
#else
#define SG_SWEEP_STAMP(k) \
  do {                    \
  } while (0)
#endif

template <int QG, int NL>
__global__ void __launch_bounds__(SG_JOINT_THREADS, 1)
k_joint_sweep(const sg_small sp, const SmallOrd o, const sg_joint jp, const uint32_t* stab_g,
              const uint32_t* __restrict__ jblob_g, const uint8_t* __restrict__ pattern,
              const int32_t* __restrict__ case_id, uint32_t* __restrict__ lanes, int lane_ld, int cases, int num_real,
              int m, int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* __restrict__ jcell,
              int cells, unsigned long long* __restrict__ counts, const uint32_t* zs_flag,
              const int8_t* __restrict__ obs, int ld_obs, int obs_nib, int32_t* err) {
  constexpr int NT = SG_JOINT_THREADS;
  SG_SWEEP_STAMP(0);
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* blob = smem;
  const uint32_t jbytes = uint32_t(jp.words) * 4u;
  uint32_t* stab = reinterpret_cast<uint32_t*>(smem + jbytes);
  uint8_t* hist8 = reinterpret_cast<uint8_t*>(stab) + ((sp.tab_words * 4 + 15) & ~15);
  uint32_t* cellacc = reinterpret_cast<uint32_t*>(hist8 + (NT / 32) * kJointBins * 4);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(cellacc) + ((cells * 4 + 15) & ~15));
  const int tid = threadIdx.x;
  const int Q = (m + 3) >> 2;
  const int q0 = blockIdx.y * QG;
  const int last = min(QG - 1, Q - 1 - q0);
  if (tid == 0) mbar_init(bar, 1);
  if (counts) {
    uint32_t* h32 = reinterpret_cast<uint32_t*>(hist8);
    for (int i = tid; i < (NT / 32) * kJointBins; i += NT) h32[i] = 0;
    for (int i = tid; i < cells; i += NT) cellacc[i] = 0;
  }
  uint32_t nw0[QG] = {};
  uint32_t nP0 = 0;
  int nc0 = 0;
  {
    const int s0 = joint_first_slot();
    if (s0 < cases) {
      const uint32_t* r0p = lanes + int64_t(q0) * lane_ld;
#pragma unroll
      for (int g = 0; g < QG; ++g) nw0[g] = r0p[int64_t(min(g, last)) * lane_ld + s0];
      nP0 = pattern[s0];
      nc0 = case_id[s0];
    }
  }
  pdl_wait();  // the blob rows, tables, key and cleared counts of this step
  // Trigger only now: the step tail that follows may then read the previous
  // tail's outputs (running total, key, previous counts) in its prologue.
  pdl_trigger();
  if (tid == 0) {
    mbar_expect_tx(bar, jbytes);
    for (uint32_t o2 = 0; o2 < jbytes; o2 += 32768u)
      bulk_g2s(blob + o2, reinterpret_cast<const unsigned char*>(jblob_g) + o2, min(32768u, jbytes - o2), bar);
  }
  for (int i = tid; i < sp.tab_words; i += NT) stab[i] = stab_g[i];
  const bool armed = zs_flag && *zs_flag != 0u;
  QuadSet qs;
  qs.row0 = uint32_t(q0) * uint32_t(lane_ld);
  qs.ld = uint32_t(lane_ld);
  qs.q0w = uint32_t(q0) << 16;
  qs.last = last;
  qs.last_nl = min(4, m - 4 * (q0 + qs.last));
  qs.last_valid = qs.last_nl >= 4 ? 0xFFFFFFFFu : ((1u << (8 * qs.last_nl)) - 1u);
  const int slot = ((tid & 31) << 2) | ((tid >> 5) & 3) | ((tid >> 7) << 7);
  const uint32_t hist_a = smem_u32(hist8) + uint32_t(tid >> 5) * kJointBins * 4u;  // this warp's bins
  const FastKey fk = fast_key(key_dev ? *key_dev : key);
  // the minibatch's range check while the blob is in flight (no kernel of this
  // step writes the observation block)
  if (obs_nib & SG_OBS_PREFETCH_ONLY) {  // the step tail checks the block: warm L2 for it
    const int nib = obs_nib & 0xFF;
    const int per_byte = nib ? 8 / nib : 1;
    const int lines = ((cases + per_byte - 1) / per_byte + 127) >> 7;
    for (int i = (blockIdx.y * gridDim.x + blockIdx.x) * NT + threadIdx.x; i < lines * sp.n;
         i += gridDim.x * gridDim.y * NT) {
      const int v = i / lines;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(obs + int64_t(v) * ld_obs + (int64_t(i - v * lines) << 7)));
    }
  } else {
    obs_range_check<NT>(sp, obs, ld_obs, cases, err, obs_nib);
  }
  SG_SWEEP_STAMP(2);  // prologue issued (blob copy in flight, range check done)
  __syncthreads();
  mbar_wait(bar, 0);
  SG_SWEEP_STAMP(3);  // blob landed: the draws start
  bool zs = false;
  if (armed) {  // padded SmallOrd entries (variable 31) are never latent: any n <= SG_SMALL_MAXV
    zs = small_units<SG_SMALL_MAXV, QG, true, NT, true>(o, qs, stab, lanes, pattern, case_id, hist_a, cases,
                                                        num_real, case_base, fk, counts != nullptr, nw0, nP0, nc0);
  } else if (NL < 4 && last == QG - 1 && q0 + QG == Q) {  // this row holds the partial final quad
    joint_units<QG, NT, NL>(qs, blob, jp.patterns, lanes, pattern, case_id, hist_a, cases, num_real, case_base, fk,
                            counts != nullptr, nw0, nP0, nc0, jbytes);
  } else {
    joint_units<QG, NT, 4>(qs, blob, jp.patterns, lanes, pattern, case_id, hist_a, cases, num_real, case_base, fk,
                           counts != nullptr, nw0, nP0, nc0, jbytes);
  }
  // per-warp bins -> CPT cells (jcell) -> one global atomic per touched cell
  small_epilogue<SG_SMALL_MAXV, NT>(sp, zs, hist8, cellacc, jcell, cells, nullptr, nullptr, 0, cases, err);
  if (!counts) return;
  __syncthreads();
  const uint32_t* wh = reinterpret_cast<const uint32_t*>(hist8);
  for (int J = tid; J < (1 << sp.bits); J += NT) {
    uint32_t sum = 0;
#pragma unroll 8
    for (int w2 = 0; w2 < NT / 32; ++w2) sum += wh[w2 * kJointBins + J];
    if (sum)
      for (int v = 0; v < sp.n; ++v) atomicAdd(cellacc + __ldg(jcell + J * sp.n + v), sum);
  }
  __syncthreads();
  for (int cell = tid; cell < cells; cell += NT)
    if (cellacc[cell]) atomicAdd(counts + cell, (unsigned long long)cellacc[cell]);
  SG_SWEEP_STAMP(1);
}

// Trace stamps of the step tail's CTAs (debug builds, -DSG_FINISH_TRACE).
#ifdef SG_FINISH_TRACE
__device__ unsigned long long g_tail_trace[16 * 160];
__device__ int g_tail_trace_role[160];
__device__ __forceinline__ void tail_stamp(int k) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tail_trace[blockIdx.x * 16 + k] = t;
  }
}
#else
__device__ __forceinline__ void tail_stamp(int) {}
#endif

#define SG_JOINT_TAB_SLICES 4
// The merged step tail splits a pattern whose rows have 2^B = 64 columns
// (two per lane) into twice as many slices: its per-CTA static preparation
// and rows then cost what a 32-column pattern's do (it was the straggler).
__host__ __device__ __forceinline__ int joint_tail_slices(int B) { return B >= 6 ? 2 * SG_JOINT_TAB_SLICES : SG_JOINT_TAB_SLICES; }
#define SG_JOINT_ROW_WARPS (FINISH_THREADS / 32)

// The row-slice map of the merged tail as a kernel parameter (built on the
// host from the latent field widths): a slice knows its pattern without
// reading the blob header first, so its preparation copy starts at once.
#define SG_TAIL_ROLE_MAX 512
struct TailRoles {
  int count;                            // 0: walk the blob header (tail_slice_of)
  uint16_t r[SG_TAIL_ROLE_MAX];         // P | slice << 7 | slices of P << 11
};

// Row slice k of the merged tail -> (pattern P, slice of P, slices of P):
// patterns from the last down (the all-latent pattern, 64 columns, first:
// the costliest slices take the first tickets, i.e. the earliest CTAs), P =
// -1 past the end.  k_joint_prep lays the static preparation out the same way.
__device__ __forceinline__ void tail_slice_of(const uint32_t* jblob, const sg_joint& jp, int k, int& P, int& slice,
                                              int& nsl) {
  slice = k;
  nsl = SG_JOINT_TAB_SLICES;
  for (P = jp.patterns - 1; P >= 0; --P) {
    nsl = joint_tail_slices(int(jblob[jp.patterns + P] & 0xFFu));
    if (slice < nsl) return;
    slice -= nsl;
  }
}

// One transition row as an alias table (one warp; K = 2^B columns, lane l
// holds column l, or columns 2l, 2l+1 when K = 64).  Input: the inclusive fp64
// cumulative sums of the row's products (c_own at the lane's first column,
// c_hi at its second when `two`) and the row total.  Integer column masses
// w_j = C_j - C_{j-1} with C_j = min(ceil(cum_j * 2^32 / total), 2^32) and
// C_{K-1} = 2^32 sum to exactly 2^32; with T = 2^(32-B):
//   light (w < T): deficit T - w; heavy (w > T): surplus w - T; full (w = T).
// Lights in column order cover [D_{k-1}, D_k) of the deficit line, heavies
// [E_{h-1}, E_h) of the surplus line (both end at the same total).
//   light: primary w, alias = the heavy whose interval holds D_{k-1};
//   heavy: X = first light end >= E_h; overshoot X - E_h > 0 -> primary
//          T - overshoot, alias = the next heavy; else full;
//   full:  primary everything (alias = itself).
// Every column's probability is then exactly w_j / 2^32 (a draw picks column
// u >> (32 - B), keeps it when (u mod T) < primary, else takes the alias).
// Entry = primary << B | alias.  tests/fast_stream.py restates this rule.
__device__ __forceinline__ void joint_alias_row(uint32_t* row, int B, bool two, int lane, double c_own, double c_hi,
                                                double total, uint32_t* sd, uint32_t* se) {
  const int K = 1 << B;
  const uint64_t ONE = 1ull << 32;
  const uint64_t T = ONE >> B;
  const double sc = total > 0.0 ? __ddiv_rn(4294967296.0, total) : 0.0;
  auto quant = [&](double c, int j) -> uint64_t {
    if (j >= K - 1) return ONE;
    return uint64_t(fmin(ceil(__dmul_rn(c, sc)), 4294967296.0));
  };
  const int j0 = two ? 2 * lane : lane;
  const bool act = j0 < K;
  const uint64_t C0 = act ? quant(c_own, j0) : ONE;
  const uint64_t C1 = two ? quant(c_hi, j0 + 1) : C0;
  const uint64_t up = __shfl_up_sync(0xffffffffu, C1, 1);
  const uint64_t prev = lane ? up : 0ull;
  const uint64_t w0 = act ? C0 - prev : T;
  const uint64_t w1 = two ? C1 - C0 : T;
  const uint32_t d0 = w0 < T ? uint32_t(T - w0) : 0u, d1 = w1 < T ? uint32_t(T - w1) : 0u;
  const uint32_t e0 = w0 > T ? uint32_t(w0 - T) : 0u, e1 = w1 > T ? uint32_t(w1 - T) : 0u;
  // inclusive warp scans of the lane sums (every partial sum < 2^32)
  uint32_t dl = d0 + d1, el = e0 + e1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t dy = __shfl_up_sync(0xffffffffu, dl, o), ey = __shfl_up_sync(0xffffffffu, el, o);
    if (lane >= o) {
      dl += dy;
      el += ey;
    }
  }
  const uint32_t D0 = dl - d1, E0 = el - e1;  // inclusive at the lane's first column
  // both scans as 64-entry arrays, padded past K with values above any query
  // (0xFFFFFFFF), so every search below is the same 6-step branch-free loop
  if (two) {
    sd[j0] = D0;
    se[j0] = E0;
    sd[j0 + 1] = dl;
    se[j0 + 1] = el;
  } else {
    sd[lane] = act ? D0 : 0xFFFFFFFFu;
    se[lane] = act ? E0 : 0xFFFFFFFFu;
    sd[lane + 32] = 0xFFFFFFFFu;
    se[lane + 32] = 0xFFFFFFFFu;
  }
  __syncwarp();
  // light: primary w, alias = the heavy holding the light's start D - d on the
  // surplus line; heavy: overshoot = first light end >= E, minus E; primary
  // T - overshoot, alias = the next heavy (the same count-of-E<=q search with
  // q = E).  Both searches run for every lane (no divergence).
  auto entry = [&](int j, uint64_t w, uint32_t d, uint32_t Dinc, uint32_t Einc) -> uint32_t {
    const bool light = w < T, heavy = w > T;
    const uint32_t q = light ? Dinc - d : Einc;
    int al = 0, xi = 0;
#pragma unroll
    for (int step = 32; step; step >>= 1) {
      if (se[al + step - 1] <= q) al += step;    // #{E <= q}: upper bound
      if (sd[xi + step - 1] < Einc) xi += step;  // #{D < E}: lower bound
    }
    const uint32_t ov = sd[min(xi, 63)] - Einc;
    if (light) return (uint32_t(w) << B) | uint32_t(al);
    if (heavy && ov) return (uint32_t(T - ov) << B) | uint32_t(al);
    return uint32_t(j);
  };
  if (act) {
    row[j0] = entry(j0, w0, d0, D0, E0);
    if (two) row[j0 + 1] = entry(j0 + 1, w1, d1, dl, el);
  }
  if (lane == 0) row[K] = 0u;  // stride padding
  __syncwarp();
}
// Slice `slice` (lane words S in [slice * R/4, (slice+1) * R/4)) of pattern
// P's rows.  vprob_g: the step tail's conditionals [n][R][4] (L2-coherent
// loads: written by another CTA of the same grid in the merged tail), or
// NULL to compute them here from cpt.
__device__ __forceinline__ void joint_slice(const sg_net& net, const sg_small& sp, const sg_joint& jp,
                                            const double* cpt, const double* vprob_g, uint32_t* jblob, int P,
                                            int slice, unsigned char* smem, bool wait_pdl,
                                            bool vprob_ready = false, int part = 0, uint16_t* pidx = nullptr,
                                            int slices = SG_JOINT_TAB_SLICES) {
  // part 0: everything; 1: only the static preparation -- the pattern's
  // latent-variable list and, with pidx, every row entry's list of vprob
  // indices (a caller runs it early); 2: everything but that (part 1 ran
  // before).  pidx: [rows_per][K][SG_SMALL_MAXV] u16, 0xFFFF = zero entry.
  __shared__ uint32_t lv[SG_SMALL_MAXV][4];  // latent variables of P in colour order: off|width<<8|card<<16, mbmask, fm, v
  __shared__ uint32_t alias_sd[SG_JOINT_ROW_WARPS][64], alias_se[SG_JOINT_ROW_WARPS][64];  // per-warp alias scans
  __shared__ int nlat;
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint32_t meta = jblob[jp.patterns + P];  // static header
  const int B = int(meta & 0xFFu);
  if (B == 0) {
    if (wait_pdl) pdl_wait();
    return;
  }
  const uint32_t keep = (meta >> 8) & 0xFFu;
  const uint32_t* dep = reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(jblob) + (meta >> 16));
  uint32_t* rows = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(jblob) + jblob[P]);
  const int R = 1 << sp.bits, K = 1 << B;
  const int KS = K + 1;  // row stride (odd: no bank conflicts between lanes of one column)
  const int rows_per = R / slices, r0 = slice * rows_per;
  double* vprob = reinterpret_cast<double*>(smem);  // [n][R][4]
  if (tid == 0 && part != 2) {
    int k = 0;
    for (int i = 0; i < sp.n; ++i) {
      const int v = sp.order[i];
      if (!((P >> v) & 1)) continue;
      lv[k][0] = uint32_t(sp.off[v]) | (uint32_t(sp.width[v]) << 8) | (uint32_t(sp.card[v]) << 16);
      lv[k][1] = sp.mbmask[v];
      lv[k][2] = ((1u << sp.width[v]) - 1u) << sp.off[v];
      lv[k][3] = uint32_t(v);
      ++k;
    }
    nlat = k;
  }
  if (part == 1) {
    if (pidx) {
      __syncthreads();
      const int nl1 = nlat;
      for (int e = tid; e < rows_per * K; e += nt) {
        const int j = e % K;
        const uint32_t S = uint32_t(r0 + e / K);
        const uint32_t Sn = (S & keep) | dep[j];
        uint16_t* out = pidx + size_t(e) * SG_SMALL_MAXV;
        uint32_t cur = S;
        for (int k = 0; k < nl1; ++k) {
          const uint32_t d = lv[k][0];
          const uint32_t x = (Sn >> (d & 0xFFu)) & ((1u << ((d >> 8) & 0xFFu)) - 1u);
          if (x >= (d >> 16)) {
            out[0] = 0xFFFFu;
            break;
          }
          out[k] = uint16_t((int(lv[k][3]) * R + int(cur & lv[k][1])) * 4 + int(x));
          cur = (cur & ~lv[k][2]) | (Sn & lv[k][2]);
        }
      }
    }
    return;
  }
  if (wait_pdl) pdl_wait();  // this step's CPTs (and the tail's conditionals)
  if (vprob_ready) {
    // the caller has filled vprob (joint_cond_apply)
  } else if (vprob_g) {
    for (int i = tid; i < sp.n * R * 4; i += nt) vprob[i] = __ldcg(vprob_g + i);
  } else {
    for (int i = tid; i < sp.n * R; i += nt) {
      const int v = i / R;
      const uint32_t S = uint32_t(i - v * R);
      if (!((P >> v) & 1) || (S & ~sp.mbmask[v])) continue;
      int s[SG_MAX_MB];
      bool valid = true;
      const int m0 = net.mb_start[v], m1 = net.mb_start[v + 1];
      for (int k = m0; k < m1 && valid; ++k) {
        const int u = net.mb_var[k];
        s[k - m0] = small_field(S, sp, u);
        valid = s[k - m0] < sp.card[u];
      }
      double* out = vprob + size_t(i) * 4;
      const int card = sp.card[v];
      if (!valid) {
        for (int t = 0; t < card; ++t) out[t] = 0.0;
        continue;
      }
      with_card(card, [&](auto C) {
        constexpr int KC = decltype(C)::value;
        double w[KC ? KC : SG_MAX_CARD];
        conditional_weights<false, KC>(net, v, s, cpt, w);
        joint_conditional<KC>(w, card, out);
      });
    }
  }
  __syncthreads();
  tail_stamp(3);
  // One warp per row S: lanes hold columns (2l, 2l+1) when K = 64, column l
  // when K <= 32; products in colour order, a Kogge-Stone scan across lanes
  // for the cumulative sums (tests/fast_stream.py restates this order).
  const int nl = nlat;
  const int warp = tid >> 5, lane = tid & 31;
  const bool two = K == 64;
  auto prod = [&](uint32_t S, int j) {
    if (pidx) {  // the indices part 1 resolved: the same products in the same order
      const uint16_t* ix = pidx + size_t((int(S) - r0) * K + j) * SG_SMALL_MAXV;
      if (nl > 0 && ix[0] == 0xFFFFu) return 0.0;
      double p = 1.0;
      for (int k = 0; k < nl; ++k) p = __dmul_rn(p, vprob[ix[k]]);
      return p;
    }
    const uint32_t Sn = (S & keep) | dep[j];
    double p = 1.0;
    uint32_t cur = S;
    for (int k = 0; k < nl; ++k) {
      const uint32_t d = lv[k][0];
      const uint32_t x = (Sn >> (d & 0xFFu)) & ((1u << ((d >> 8) & 0xFFu)) - 1u);
      if (x >= (d >> 16)) return 0.0;
      p = __dmul_rn(p, vprob[(int(lv[k][3]) * R + int(cur & lv[k][1])) * 4 + int(x)]);
      cur = (cur & ~lv[k][2]) | (Sn & lv[k][2]);
    }
    return p;
  };
  tail_stamp(4);
  for (int r = warp; r < rows_per; r += nt >> 5) {
    const uint32_t S = uint32_t(r0 + r);
    const int j0 = two ? 2 * lane : lane;
    const double a = j0 < K ? prod(S, j0) : 0.0;
    const double b2 = two ? prod(S, j0 + 1) : 0.0;
    double x = two ? __dadd_rn(a, b2) : a;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x = __dadd_rn(x, y);
    }
    const double left = __shfl_up_sync(0xffffffffu, x, 1);
    const double total = __shfl_sync(0xffffffffu, x, two ? 31 : K - 1);
    const double c0 = two ? (lane ? __dadd_rn(left, a) : a) : x;
    joint_alias_row(rows + S * KS, B, two, lane, j0 < K ? c0 : 0.0, x, total, alias_sd[warp], alias_se[warp]);
  }
}

// The conditionals p_v(x | lane word S) a slice of pattern P needs, split in
// two: joint_cond_plan (before the new CPTs exist) resolves every CPT index
// of conditional_weights -- the parent row, then each child's factor in
// ascending child order, as (first cell, cell step per state of v) -- and
// joint_cond_apply (once they exist) only gathers, multiplies in that same
// order and normalises (joint_conditional): the same products as the direct
// path, without the dependent index chains on the critical path.
#define SG_JOINT_MAXF (1 + SG_SMALL_MAXV)
__device__ __forceinline__ void joint_cond_plan(const sg_net& net, const sg_small& sp, int P, int2* plan,
                                                int8_t* nf) {
  const int R = 1 << sp.bits;
  for (int i = threadIdx.x; i < sp.n * R; i += blockDim.x) {
    const int v = i / R;
    const uint32_t S = uint32_t(i - v * R);
    if (!((P >> v) & 1) || (S & ~sp.mbmask[v])) {  // never read by this pattern's rows
      nf[i] = -1;
      continue;
    }
    int st[SG_MAX_MB];
    bool valid = true;
    const int m0 = net.mb_start[v], m1 = net.mb_start[v + 1];
    for (int k = m0; k < m1 && valid; ++k) {
      const int u = net.mb_var[k];
      st[k - m0] = small_field(S, sp, u);
      valid = st[k - m0] < sp.card[u];
    }
    if (!valid) {
      nf[i] = 0;
      continue;
    }
    int2* pl = plan + size_t(i) * SG_JOINT_MAXF;
    const int card = net.card[v];
    int64_t cfg = 0;
    for (int j = net.par_start[v], e = net.par_start[v + 1]; j < e; ++j)
      cfg += int64_t(st[net.par_slot[j]]) * net.par_stride[j];
    pl[0] = make_int2(int(net.cpt_off[v] + cfg * card), 1);
    int f = 1;
    for (int k = net.chl_start[v], ke = net.chl_start[v + 1]; k < ke; ++k, ++f) {
      const int c = net.chl_var[k];
      const int cc = net.card[c];
      int64_t cfg0 = 0;
      for (int q = net.chl_pstart[k], qe = net.chl_pstart[k + 1]; q < qe; ++q)
        cfg0 += int64_t(st[net.chl_pslot[q]]) * net.chl_pstride[q];
      pl[f] = make_int2(int(net.cpt_off[c] + st[net.chl_slot[k]] + cfg0 * cc), int(net.chl_vstride[k] * cc));
    }
    nf[i] = int8_t(f);
  }
}

__device__ __forceinline__ void joint_cond_apply(const sg_net& net, const sg_small& sp, const int2* plan,
                                                 const int8_t* nf, const double* cpt, double* vprob) {
  const int R = 1 << sp.bits;
  for (int i = threadIdx.x; i < sp.n * R; i += blockDim.x) {
    const int n_f = nf[i];
    if (n_f < 0) continue;
    const int card = net.card[i / R];
    double* out = vprob + size_t(i) * 4;
    if (n_f == 0) {
      for (int t = 0; t < card; ++t) out[t] = 0.0;
      continue;
    }
    const int2* pl = plan + size_t(i) * SG_JOINT_MAXF;
    with_card(card, [&](auto C) {
      constexpr int KC = decltype(C)::value;
      double w[KC ? KC : SG_MAX_CARD];
      const int2 p0 = pl[0];
#pragma unroll
      for (int t = 0; t < (KC ? KC : card); ++t) w[t] = cpt[p0.x + t];
      if (KC) {  // unrolled over the factor bound: every factor's loads issue together
#pragma unroll
        for (int f = 1; f < SG_JOINT_MAXF; ++f) {
          if (f < n_f) {
            const int2 pf = pl[f];
#pragma unroll
            for (int t = 0; t < (KC ? KC : 1); ++t) w[t] = __dmul_rn(w[t], cpt[pf.x + t * pf.y]);
          }
        }
      } else {
        for (int f = 1; f < n_f; ++f) {
          const int2 pf = pl[f];
          for (int t = 0; t < card; ++t) w[t] = __dmul_rn(w[t], cpt[pf.x + t * pf.y]);
        }
      }
      joint_conditional<KC>(w, card, out);
    });
  }
}

// Rows of pattern P = blockIdx.x, lane words of slice blockIdx.y, from the
// current CPTs (see the blob comment).  fp64 in a fixed order, no FMA:
// p_v = w / norm with the reference's weight product (conditional_weights)
// and sequential norm; products in colour order; warp-scan row sums;
// alias entries from min(ceil(cum * (2^32 / total)), 2^32) (joint_alias_row).
__global__ void __launch_bounds__(256) k_joint_tables(const sg_net net, const sg_small sp, const sg_joint jp,
                                                      const double* cpt, const double* vprob_g, uint32_t* jblob) {
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_trigger();
  joint_slice(net, sp, jp, cpt, vprob_g, jblob, blockIdx.x, blockIdx.y, smem, true);
}

#ifdef SG_FINISH_TRACE
extern "C" int sg_debug_tail_trace(unsigned long long* out) {
  // 8 stamps per CTA (by blockIdx.x), then the CTA -> role map as 160 more words
  if (cudaMemcpyFromSymbol(out, g_tail_trace, sizeof(g_tail_trace)) != cudaSuccess) return 2;
  int roles[160];
  if (cudaMemcpyFromSymbol(roles, g_tail_trace_role, sizeof(roles)) != cudaSuccess) return 2;
  for (int i = 0; i < 160; ++i) out[16 * 160 + i] = (unsigned long long)roles[i];
  return 0;
}
extern "C" int sg_debug_tail_finish_trace(unsigned long long* out) {  // this TU's copy of g_finish_trace
  return cudaMemcpyFromSymbol(out, g_finish_trace, sizeof(unsigned long long) * 12) == cudaSuccess ? 0 : 2;
}
#endif

// The whole step tail of the joint path in ONE grid.  Roles come from a
// ticket (sync[2]): the first CTA to run takes role 0 and runs the single-CTA
// tail (accumulate, CPT update, packed tables, count clearing, key advance),
// releasing sync[0] once the slices can proceed; every later CTA takes the
// next row slice and spins on sync[0].  The spinning CTAs therefore only ever
// wait on a CTA that is already resident, whatever order or subset of CTAs
// the hardware schedules first (no reliance on CTA 0 being dispatched first
// or on co-residency of the whole grid).  The last slice to finish re-arms
// the sync words for the next step.
__global__ void __launch_bounds__(FINISH_THREADS) k_step_tail_joint(const sg_net gnet, const FinishArgs f,
                                                                    const sg_small sp, const sg_joint jp,
                                                                    uint32_t* jblob, uint32_t* sync,
                                                                    const unsigned char* __restrict__ prep,
                                                                    int64_t prep_bytes, const TailRoles roles) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_role;
  // the step's observation block is range-checked by every CTA (a share each, by block
  // index) beside the model update and the slices' preparation -- the sweep only
  // prefetches it then (SG_OBS_PREFETCH_ONLY)
  const int check_t = int(blockIdx.x * blockDim.x + threadIdx.x), check_n = int(gridDim.x * blockDim.x);
#ifdef SG_FINISH_TRACE
  tail_stamp(10);  // entry, before the role ticket
#endif
  if (threadIdx.x == 0) s_role = int(atomicAdd(sync + 2, 1u));
  __syncthreads();
  const int role = s_role;  // 0: the model update; r >= 1: row slice r - 1
  SG_DCHECK(role >= 0 && role < int(gridDim.x));
#ifdef SG_FINISH_TRACE
  if (threadIdx.x == 0) g_tail_trace_role[blockIdx.x] = role;
  auto stamp = [](int k) { tail_stamp(k); };
#else
  auto stamp = [](int) {};
#endif
  stamp(0);
  if (role == 0) {  // releases sync[0] as soon as the new CPTs are written (f.release_sync)
    if (f.check_obs)
      obs_range_check_range(sp, f.check_obs, f.check_ld, f.check_cases, f.check_err, f.check_nib, check_t, check_n);
    step_finish_body(gnet, f, smem, FINISH_THREADS);
    stamp(1);
    return;
  }
  // Slices: stage the network pack while the sweep and CTA 0 run, then wait
  // for the CPTs and build this slice's conditionals and rows.
  const int tid = threadIdx.x;
  const int cells = int(gnet.cells);
  const int64_t cells2 = (gnet.cells + 1) & ~int64_t(1);
  const bool from_lg = f.release_lg != nullptr;  // CTA 0 hands over the gamma draws, not the CPTs
  int64_t* b64 = reinterpret_cast<int64_t*>(smem);
  int32_t* b32 = reinterpret_cast<int32_t*>(b64 + gnet.blob64_words);
  double* cpt_s = reinterpret_cast<double*>(
      reinterpret_cast<unsigned char*>(b32) + ((size_t(gnet.blob32_words) * 4 + 15) & ~size_t(15)));
  double* lg = cpt_s + cells2;
  uint8_t* inlog = reinterpret_cast<uint8_t*>(lg + (from_lg ? cells2 : 0));
  unsigned char* work = inlog + (from_lg ? ((size_t(cells) + 15) & ~size_t(15)) : 0);
  // after the slice's conditionals (work: n * 2^bits * 4 doubles): their gather plan
  const int nr = sp.n << sp.bits;
  int2* plan = reinterpret_cast<int2*>(work + size_t(nr) * 4 * sizeof(double));
  int8_t* plan_nf = reinterpret_cast<int8_t*>(plan + size_t(nr) * SG_JOINT_MAXF);
  uint16_t* pidx = reinterpret_cast<uint16_t*>(plan_nf + ((size_t(nr) + 15) & ~size_t(15)));
  int P, slice, nsl;
  bool live;
  if (roles.count) {
    const uint32_t e = roles.r[role - 1];
    P = int(e & 127u);
    slice = int((e >> 7) & 15u);
    nsl = int(e >> 11);
    live = P != 0;  // every other pattern has latent fields
  } else {
    tail_slice_of(jblob, jp, role - 1, P, slice, nsl);
    live = (jblob[jp.patterns + P] & 0xFFu) != 0;
  }
  pdl_trigger();
  __shared__ __align__(8) uint64_t prep_bar;
  // the static gather plan and row index lists of this slice: precomputed once
  // (sg_joint_prep) and brought in with one TMA bulk copy, or built here
  const bool prepped = prep != nullptr && live;
  if (prepped && tid == 0) {
    mbar_init(&prep_bar, 1);
    mbar_expect_tx(&prep_bar, uint32_t(prep_bytes));
    const unsigned char* src = prep + int64_t(role - 1) * prep_bytes;
    for (int64_t o2 = 0; o2 < prep_bytes; o2 += 32768)
      bulk_g2s(reinterpret_cast<unsigned char*>(plan) + o2, src + o2, uint32_t(prep_bytes - o2 < 32768 ? prep_bytes - o2 : 32768),
               &prep_bar);
  }
  for (int i = tid; i < int(gnet.blob64_words); i += blockDim.x) b64[i] = __ldg(gnet.blob64 + i);
  for (int i = tid; i < int(gnet.blob32_words); i += blockDim.x) b32[i] = __ldg(gnet.blob32 + i);
  // this CTA's share of the observation check (its loads overlap the preparation copy)
  if (f.check_obs)
    obs_range_check_range(sp, f.check_obs, f.check_ld, f.check_cases, f.check_err, f.check_nib, check_t, check_n);
  __syncthreads();
  stamp(8);  // blobs staged, share checked
  const sg_net net = rebase_net(gnet, b32, b64);
  // every CPT index of this pattern's conditionals, while the sweep / CTA 0 still run
  if (live) {
    if (!prepped) joint_cond_plan(net, sp, P, plan, plan_nf);
    joint_slice(net, sp, jp, nullptr, nullptr, jblob, P, slice, work, false, true, 1, prepped ? nullptr : pidx, nsl);
    stamp(9);  // slice part 1 done
    if (prepped) mbar_wait(&prep_bar, 0);
  }
  stamp(7);
  pdl_wait();  // the sweep has finished reading the blob rows this grid overwrites
  if (tid == 0) {
    uint32_t r = 0;
#ifdef SG_CHECKED
    for (long long spin = 0;; ++spin) {  // bounded: a lost release is recorded, not a hang
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(sync) : "memory");
      if (r) break;
      if (spin > (1ll << 27)) {
        SG_DCHECK(false);
        break;
      }
    }
#else
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(sync) : "memory");
      if (r) break;
    }
#endif
  }
  __syncthreads();
  stamp(1);
  if (from_lg) {  // the Dirichlet rows from CTA 0's draws (the same code and rounding as CTA 0's own rows)
    const uint8_t* il_g = reinterpret_cast<const uint8_t*>(f.release_lg + cells);
    for (int i = tid; i < cells; i += blockDim.x) {
      lg[i] = __ldcg(f.release_lg + i);
      inlog[i] = __ldcg(il_g + i);
    }
    __syncthreads();
    stamp(5);
    for (int row = tid; row < int(net.rows); row += blockDim.x) {
      const int v = net.row_var[row];
      const int card = net.card[v];
      const int64_t base = net.cpt_off[v] + (row - net.row_off[v]) * card;
      with_card(card, [&](auto C) {
        constexpr int K = decltype(C)::value;
        if (f.map_estimate) mean_row<K>(lg + base, f.alpha[v], card, cpt_s + base);
        else dirichlet_row<K>(lg + base, inlog + base, card, cpt_s + base);
      });
    }
  } else {
    for (int i = tid; i < cells; i += blockDim.x) cpt_s[i] = __ldcg(f.cpt + i);
  }
  __syncthreads();
  stamp(6);
  if (live) joint_cond_apply(net, sp, plan, plan_nf, cpt_s, reinterpret_cast<double*>(work));
  __syncthreads();
  joint_slice(net, sp, jp, cpt_s, nullptr, jblob, P, slice, work, false, true, 2, pidx, nsl);
  __syncthreads();
  stamp(2);
  if (threadIdx.x == 0 && atomicAdd(sync + 1, 1u) == gridDim.x - 2) {
    sync[1] = 0u;
    sync[0] = 0u;
    sync[2] = 0u;  // every CTA has taken its ticket
  }
}

// Static preparation of every row slice of the merged tail, once per
// network (it depends only on the network and the latent patterns): the
// gather plan of the slice's conditionals and every row entry's vprob index
// list, exactly as the slice would build them, stored per slice (role) so
// that k_step_tail_joint loads them with one bulk copy instead of building
// them on its critical path.
__global__ void __launch_bounds__(FINISH_THREADS) k_joint_prep(const sg_net gnet, const sg_small sp,
                                                               const sg_joint jp, const uint32_t* jblob,
                                                               unsigned char* __restrict__ prep, int64_t prep_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  int64_t* b64 = reinterpret_cast<int64_t*>(smem);
  int32_t* b32 = reinterpret_cast<int32_t*>(b64 + gnet.blob64_words);
  unsigned char* work = reinterpret_cast<unsigned char*>(b32) + ((size_t(gnet.blob32_words) * 4 + 15) & ~size_t(15));
  const int nr = sp.n << sp.bits;
  int2* plan = reinterpret_cast<int2*>(work + size_t(nr) * 4 * sizeof(double));
  int8_t* plan_nf = reinterpret_cast<int8_t*>(plan + size_t(nr) * SG_JOINT_MAXF);
  uint16_t* pidx = reinterpret_cast<uint16_t*>(plan_nf + ((size_t(nr) + 15) & ~size_t(15)));
  int P, slice, nsl;
  tail_slice_of(jblob, jp, int(blockIdx.x), P, slice, nsl);
  if (P < 0 || !(jblob[jp.patterns + P] & 0xFFu)) return;
  for (int i = tid; i < int(gnet.blob64_words); i += blockDim.x) b64[i] = __ldg(gnet.blob64 + i);
  for (int i = tid; i < int(gnet.blob32_words); i += blockDim.x) b32[i] = __ldg(gnet.blob32 + i);
  __syncthreads();
  const sg_net net = rebase_net(gnet, b32, b64);
  joint_cond_plan(net, sp, P, plan, plan_nf);
  joint_slice(net, sp, jp, nullptr, nullptr, const_cast<uint32_t*>(jblob), P, slice, work, false, true, 1, pidx, nsl);
  __syncthreads();
  const unsigned char* src = reinterpret_cast<const unsigned char*>(plan);
  unsigned char* dst = prep + int64_t(blockIdx.x) * prep_bytes;
  for (int64_t i = tid; i < prep_bytes; i += blockDim.x) dst[i] = src[i];
}

// bytes of one slice's prep region (plan, plan_nf, pidx; the slice smem layout)
static int64_t joint_prep_slice_bytes(const sg_small& sp, const sg_joint& jp) {
  const int64_t nr = int64_t(sp.n) << sp.bits;
  const int64_t pidx = (int64_t(1) << sp.bits) / SG_JOINT_TAB_SLICES * (int64_t(1) << jp.max_b) * SG_SMALL_MAXV * 2;
  return (nr * SG_JOINT_MAXF * 8 + ((nr + 15) & ~int64_t(15)) + pidx + 15) & ~int64_t(15);
}

static int joint_tail_slice_count(const sg_small& sp, const sg_joint& jp) {
  int slices = 0;
  for (int P = 0; P < jp.patterns; ++P) {  // B_P = the latent variables' field widths (the blob header's B)
    int B = 0;
    for (int v = 0; v < sp.n; ++v)
      if ((P >> v) & 1) B += sp.width[v];
    slices += joint_tail_slices(B);
  }
  return slices;
}

static size_t joint_tables_smem(const sg_small& sp, int maxb) {
  const size_t R = size_t(1) << sp.bits;
  (void)maxb;
  return size_t(sp.n) * R * 4 * sizeof(double);
}

}  // namespace sg

extern "C" int sg_small_tables(const sg_net* net, const sg_small* sp, const uint32_t* ftab, uint32_t* stab,
                               void* stream) {
  using namespace sg;
  SG_REQUIRE(net && sp && ftab && stab, "sg_small_tables: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV && sp->bits <= SG_SMALL_MAXBITS, "sg_small_tables: bad plan");
  const int total = sp->n << sp->bits;
  k_small_tables<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*net, *sp, ftab, stab);
  return check_launch("sg_small_tables");
}

static bool lane_ld_ok(int lane_ld, int cases) { return lane_ld >= cases && lane_ld % 4 == 0; }

extern "C" int sg_small_prepare(const sg_small* sp, const int8_t* obs, int32_t ld_obs, int32_t cases, int32_t m,
                                int64_t case_base, uint64_t init_key, int32_t init, int32_t* scratch,
                                uint8_t* pattern, int32_t* case_id, uint8_t* lanes, int32_t lane_ld,
                                const uint64_t* init_key_dev, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && obs && scratch && pattern && case_id && lanes, "sg_small_prepare: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV, "sg_small_prepare: bad plan");
  SG_REQUIRE(m >= 1 && m <= 32 && lane_ld_ok(lane_ld, cases), "sg_small_prepare: m %d / lane_ld %d < cases %d", m,
             lane_ld, cases);
  SG_REQUIRE(fast_cases_ok(case_base, cases), "sg_small_prepare: global case index beyond 2^32");
  if (cases == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = std::min((cases + 255) / 256, SMALL_PREP_BLOCKS);
  int* cnt = scratch;                                                                     // [SMALL_PATTERNS][blocks]
  uint8_t* poc = reinterpret_cast<uint8_t*>(scratch + SMALL_PATTERNS * SMALL_PREP_BLOCKS);  // [cases] patterns
  uint8_t* ow = poc + cases;                                                               // [cases] observed fields
  const bool vec4 = ld_obs % 4 == 0 && ld_obs >= (cases + 3) / 4 * 4 && (reinterpret_cast<uintptr_t>(obs) & 3) == 0;
  k_small_count<<<blocks, 1024, 0, s>>>(*sp, obs, ld_obs, cases, poc, ow, cnt, vec4);
  k_small_scatter<<<blocks, 1024, 0, s>>>(cases, poc, cnt, 1 << sp->n, pattern, case_id);
  if (init) {
    const int grid = std::min((cases + 255) / 256, 148 * 8);
#define SG_INIT_LANES(N)                                                                                         \
  case N:                                                                                                      \
    k_small_init_lanes<N><<<grid, 256, 0, s>>>(*sp, ow, cases, m, case_base, init_key, pattern, case_id, lanes, \
                                               lane_ld, init_key_dev);                                           \
    break;
    switch (sp->n) {
      SG_INIT_LANES(1)
      SG_INIT_LANES(2)
      SG_INIT_LANES(3)
      SG_INIT_LANES(4)
      SG_INIT_LANES(5)
      SG_INIT_LANES(6)
      default: SG_INIT_LANES(7)
    }
#undef SG_INIT_LANES
  }
  return check_launch("sg_small_prepare");
}

namespace sg {
static int small_sweep_impl(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                            uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                            int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                            int32_t cells, uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs,
                            int32_t ld_obs, int32_t* err, void* stream) {
  SG_REQUIRE(sp && stab && pattern && case_id && lanes && err, "sg_small_sweep: null argument");
  if (obs)
    SG_REQUIRE(ld_obs % 16 == 0 && (reinterpret_cast<uintptr_t>(obs) & 15) == 0 && ld_obs >= cases,
               "sg_small_sweep: obs rows must be 16-byte aligned");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV && sp->bits <= SG_SMALL_MAXBITS, "sg_small_sweep: bad plan");
  SG_REQUIRE(!counts || jcell, "sg_small_sweep: joint cell map required for the tally");
  SG_REQUIRE(m >= 1 && m <= 32 && lane_ld_ok(lane_ld, cases), "sg_small_sweep: m %d / lane_ld %d < cases %d", m,
             lane_ld, cases);
  SG_REQUIRE(fast_cases_ok(case_base, cases), "sg_small_sweep: global case index beyond 2^32");
  SG_REQUIRE(int64_t((m + 3) / 4) * lane_ld <= (int64_t(1) << 32), "sg_small_sweep: lane block beyond 2^32 words");
  for (int v = 0; v < sp->n; ++v)
    SG_REQUIRE(sp->card[v] >= 2 && sp->card[v] <= 4 && sp->tstride[v] >= sp->card[v] - 1 &&
                   sp->toff[v] % sp->tstride[v] == 0,
               "sg_small_sweep: variable %d needs 2 <= card <= 4 and an aligned table", v);
  if (cases == 0) return SG_OK;
  const size_t smem = small_smem(*sp, cells);
  const SmallOrd o = small_ord(*sp);
  int qg = 1, groups = 1;
  quad_groups(m, &qg, &groups);
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* lw = reinterpret_cast<uint32_t*>(lanes);
#define SG_SMALL_QG(NV, G)                                                                                       \
  case G:                                                                                                        \
    launch_small<NV, G>(*sp, o, groups, smem, st, stab, pattern, case_id, lw, lane_ld, cases, num_real, m,      \
                        case_base, key, key_dev, jcell, cells, counts, zs_flag, obs, ld_obs, err);               \
    break;
#define SG_SMALL_CASE(NV)    \
  case NV:                   \
    switch (qg) {            \
      SG_SMALL_QG(NV, 1)     \
      SG_SMALL_QG(NV, 2)     \
      SG_SMALL_QG(NV, 3)     \
      SG_SMALL_QG(NV, 4)     \
    }                        \
    break;
  switch (sp->n) {
    SG_SMALL_CASE(1)
    SG_SMALL_CASE(2)
    SG_SMALL_CASE(3)
    SG_SMALL_CASE(4)
    SG_SMALL_CASE(5)
    SG_SMALL_CASE(6)
    SG_SMALL_CASE(7)
    default:
      set_error("sg_small_sweep: n=%d", sp->n);
      return SG_EINVAL;
  }
#undef SG_SMALL_CASE
#undef SG_SMALL_QG
  return check_launch("sg_small_sweep");
}
}  // namespace sg

extern "C" int sg_small_sweep(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                              uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                              int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                              int32_t cells, uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs,
                              int32_t ld_obs, int32_t* err, void* stream) {
  return sg::small_sweep_impl(sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real, m, case_base, key, key_dev,
                              jcell, cells, counts, zs_flag, obs, ld_obs, err, stream);
}


extern "C" int sg_small_import(const sg_small* sp, const sg_batch* batch, const int32_t* case_id, uint8_t* lanes,
                               int32_t lane_ld, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && batch && case_id && lanes, "sg_small_import: null argument");
  SG_REQUIRE(lane_ld_ok(lane_ld, batch->cases), "sg_small_import: bad lane_ld");
  const int64_t total = int64_t(batch->m) * batch->cases;
  if (total == 0) return SG_OK;
  k_small_import<<<int(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, (cudaStream_t)stream>>>(
      *sp, *batch, case_id, lanes, lane_ld);
  return check_launch("sg_small_import");
}

extern "C" int sg_small_export(const sg_small* sp, const sg_batch* batch, const int32_t* case_id,
                               const uint8_t* pattern, const uint8_t* lanes, int32_t lane_ld, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && batch && case_id && pattern && lanes, "sg_small_export: null argument");
  SG_REQUIRE(lane_ld_ok(lane_ld, batch->cases), "sg_small_export: bad lane_ld");
  const int64_t total = int64_t(batch->m) * batch->cases;
  if (total == 0) return SG_OK;
  k_small_export<<<int(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, (cudaStream_t)stream>>>(
      *sp, *batch, case_id, pattern, lanes, lane_ld);
  return check_launch("sg_small_export");
}

// Advance the device-side key cursor: current[0..kps) = table[idx*kps ..], idx += 1.
// Lets a captured CUDA graph replay successive minibatch steps with fresh keys.
__global__ void k_keys_advance(const uint64_t* __restrict__ table, int32_t* idx, int kps, uint64_t* current) {
  const int i = *idx;
  for (int k = threadIdx.x; k < kps; k += blockDim.x) current[k] = table[int64_t(i) * kps + k];
  __syncthreads();
  if (threadIdx.x == 0) *idx = i + 1;
}

extern "C" int sg_keys_advance(const uint64_t* table, int32_t* index, int32_t kps, uint64_t* current, void* stream) {
  using namespace sg;
  SG_REQUIRE(table && index && current && kps > 0, "sg_keys_advance: bad argument");
  k_keys_advance<<<1, 32, 0, (cudaStream_t)stream>>>(table, index, kps, current);
  return check_launch("sg_keys_advance");
}

// ------------------------------------------------------------ joint C-ABI
namespace sg {
template <int QG, int NL>
static void launch_joint(const sg_small& sp, const SmallOrd& o, const sg_joint& jp, int groups, size_t smem,
                         cudaStream_t st, const uint32_t* stab, const uint32_t* jblob, const uint8_t* pattern,
                         const int32_t* case_id, uint32_t* lanes, int lane_ld, int cases, int num_real, int m,
                         int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell, int cells,
                         uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs, int ld_obs, int obs_nib,
                         int32_t* err) {
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem)) {
    cudaFuncSetAttribute(k_joint_sweep<QG, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    // the step tail prefers the same carveout: no L1/shared reconfiguration between the two kernels
    cudaFuncSetAttribute(k_joint_sweep<QG, NL>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // one CTA per SM (one wave) but one SM left free, where the step tail's
  // first CTA starts early (PDL) and loads its inputs while the sweep runs;
  // no thread's byte counters past 255 increments
  const int64_t per_thread = 255 / (4 * QG);
  const int64_t need = (int64_t(cases) + SG_JOINT_THREADS * per_thread - 1) / (SG_JOINT_THREADS * per_thread);
  const int64_t fill = (int64_t(cases) + SG_JOINT_THREADS - 1) / SG_JOINT_THREADS;
  const int64_t want = std::max<int64_t>(std::max(1, (sms - 1) / groups), need);
  const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>(want, fill))), unsigned(groups));
  launch_pdl(k_joint_sweep<QG, NL>, grid, dim3(SG_JOINT_THREADS), smem, st, sp, o, jp, stab, jblob, pattern, case_id,
             lanes, lane_ld, cases, num_real, m, case_base, key, key_dev, jcell, cells,
             reinterpret_cast<unsigned long long*>(counts), zs_flag, obs, ld_obs, obs_nib, err);
}

static bool joint_plan_ok(const sg_small& sp, const sg_joint& jp, int cells) {
  return sp.bits >= 2 && sp.bits <= SG_JOINT_MAXB && jp.patterns == (1 << sp.n) && jp.words > 2 * jp.patterns &&
         jp.words % 4 == 0 && jp.max_b >= 1 && jp.max_b <= sp.bits && joint_smem(sp, jp, cells) <= 227 * 1024;
}
}  // namespace sg

extern "C" int sg_joint_smem(const sg_small* sp, const sg_joint* jp, int32_t cells, int64_t* bytes) {
  using namespace sg;
  SG_REQUIRE(sp && jp && bytes, "sg_joint_smem: null argument");
  *bytes = int64_t(joint_smem(*sp, *jp, cells));
  return SG_OK;
}

extern "C" int sg_joint_tables(const sg_net* net, const sg_small* sp, const sg_joint* jp, const double* cpt,
                               const double* vprob, uint32_t* jblob, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && sp && jp && cpt && jblob, "sg_joint_tables: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV && sp->bits >= 2 && sp->bits <= SG_JOINT_MAXB &&
                 jp->patterns == (1 << sp->n) && jp->max_b >= 1 && jp->max_b <= sp->bits,
             "sg_joint_tables: bad plan (bits %d, patterns %d)", sp->bits, jp->patterns);
  SG_REQUIRE(net->max_mb <= SG_MAX_MB, "sg_joint_tables: Markov blanket too large");
  const size_t smem = joint_tables_smem(*sp, jp->max_b);
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_joint_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  launch_pdl(k_joint_tables, dim3(jp->patterns, SG_JOINT_TAB_SLICES), dim3(256), smem, (cudaStream_t)stream, *net, *sp, *jp, cpt, vprob,
             jblob);
  return check_launch("sg_joint_tables");
}

extern "C" int sg_joint_sweep(const sg_small* sp, const sg_joint* jp, const uint32_t* stab, const uint32_t* jblob,
                              const uint8_t* pattern, const int32_t* case_id, uint8_t* lanes, int32_t lane_ld,
                              int32_t cases, int32_t num_real, int32_t m, int64_t case_base, uint64_t key,
                              const uint64_t* key_dev, const int32_t* jcell, int32_t cells, uint64_t* counts,
                              const uint32_t* zs_flag, const int8_t* obs, int32_t ld_obs, int32_t obs_bits,
                              int32_t* err, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && jp && stab && jblob && pattern && case_id && lanes && err, "sg_joint_sweep: null argument");
  SG_REQUIRE((reinterpret_cast<uintptr_t>(jblob) & 15) == 0, "sg_joint_sweep: blob must be 16-byte aligned");
  const int prefetch_only = obs_bits & SG_OBS_PREFETCH_ONLY;
  obs_bits &= ~SG_OBS_PREFETCH_ONLY;
  SG_REQUIRE(obs_bits == 0 || obs_bits == 8 || obs_bits == 4 || obs_bits == 2,
             "sg_joint_sweep: obs_bits must be 0/8 (int8), 4 or 2");
  const int per_byte = (obs_bits == 4 || obs_bits == 2) ? 8 / obs_bits : 1;
  if (obs)
    SG_REQUIRE(ld_obs % 16 == 0 && (reinterpret_cast<uintptr_t>(obs) & 15) == 0 &&
                   int64_t(ld_obs) * per_byte >= cases,
               "sg_joint_sweep: obs rows must be 16-byte aligned");
  if (per_byte > 1)
    for (int v = 0; v < sp->n; ++v)
      SG_REQUIRE(sp->card[v] < (1 << obs_bits), "sg_joint_sweep: %d-bit observations need cards < %d", obs_bits,
                 1 << obs_bits);
  const int obs_nibbles = (per_byte > 1 ? obs_bits : 0) | prefetch_only;
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV, "sg_joint_sweep: bad plan");
  SG_REQUIRE(joint_plan_ok(*sp, *jp, cells), "sg_joint_sweep: joint plan does not fit (bits %d, words %d)", sp->bits,
             jp->words);
  SG_REQUIRE(!counts || jcell, "sg_joint_sweep: joint cell map required for the tally");
  SG_REQUIRE(m >= 1 && m <= 32 && lane_ld_ok(lane_ld, cases), "sg_joint_sweep: m %d / lane_ld %d < cases %d", m,
             lane_ld, cases);
  SG_REQUIRE(fast_cases_ok(case_base, cases), "sg_joint_sweep: global case index beyond 2^32");
  SG_REQUIRE(int64_t((m + 3) / 4) * lane_ld <= (int64_t(1) << 32), "sg_joint_sweep: lane block beyond 2^32 words");
  for (int v = 0; v < sp->n; ++v)
    SG_REQUIRE(sp->card[v] >= 2 && sp->card[v] <= 4 && sp->tstride[v] >= sp->card[v] - 1 &&
                   sp->toff[v] % sp->tstride[v] == 0,
               "sg_joint_sweep: variable %d needs 2 <= card <= 4 and an aligned table", v);
  if (cases == 0) return SG_OK;
  const size_t smem = joint_smem(*sp, *jp, cells);
  const SmallOrd o = small_ord(*sp);
  int qg = 1, groups = 1;
  quad_groups(m, &qg, &groups);
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* lw = reinterpret_cast<uint32_t*>(lanes);
  const int nl = m - 4 * ((m + 3) / 4 - 1);  // lanes of the final quad
#define SG_JOINT_NL(G, L)                                                                                     \
  case L:                                                                                                     \
    launch_joint<G, L>(*sp, o, *jp, groups, smem, st, stab, jblob, pattern, case_id, lw, lane_ld, cases,      \
                       num_real, m, case_base, key, key_dev, jcell, cells, counts, zs_flag, obs, ld_obs,      \
                       obs_nibbles, err);                                                                     \
    break;
#define SG_JOINT_QG(G)   \
  case G:                \
    switch (nl) {        \
      SG_JOINT_NL(G, 1)  \
      SG_JOINT_NL(G, 2)  \
      SG_JOINT_NL(G, 3)  \
      SG_JOINT_NL(G, 4)  \
    }                    \
    break;
  switch (qg) {
    SG_JOINT_QG(1)
    SG_JOINT_QG(2)
    SG_JOINT_QG(3)
    SG_JOINT_QG(4)
    default:
      set_error("sg_joint_sweep: quad group %d", qg);
      return SG_EINVAL;
  }
#undef SG_JOINT_NL
#undef SG_JOINT_QG
  return check_launch("sg_joint_sweep");
}

extern "C" int sg_joint_prep_bytes(const sg_small* sp, const sg_joint* jp, int64_t* bytes) {
  using namespace sg;
  SG_REQUIRE(sp && jp && bytes, "sg_joint_prep_bytes: null argument");
  *bytes = joint_prep_slice_bytes(*sp, *jp) * joint_tail_slice_count(*sp, *jp);
  return SG_OK;
}

extern "C" int sg_joint_prep(const sg_net* net, const sg_small* sp, const sg_joint* jp, const uint32_t* jblob,
                             void* prep, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && sp && jp && jblob && prep, "sg_joint_prep: null argument");
  SG_REQUIRE(sp->bits >= 2 && sp->bits <= SG_JOINT_MAXB && jp->patterns == (1 << sp->n) && jp->max_b >= 1,
             "sg_joint_prep: bad joint plan");
  SG_REQUIRE(net->blob32 && net->blob64 && net->max_mb <= SG_MAX_MB, "sg_joint_prep: network pack not blobbed");
  const int64_t per = joint_prep_slice_bytes(*sp, *jp);
  const int slices = joint_tail_slice_count(*sp, *jp);
  const int64_t nr = int64_t(sp->n) << sp->bits;
  const size_t smem = size_t(net->blob64_words) * 8 + ((size_t(net->blob32_words) * 4 + 15) & ~size_t(15)) +
                      size_t(nr) * 4 * sizeof(double) + size_t(per);
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_joint_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_joint_prep<<<slices, FINISH_THREADS, smem, (cudaStream_t)stream>>>(*net, *sp, *jp, jblob,
                                                                      static_cast<unsigned char*>(prep), per);
  return check_launch("sg_joint_prep");
}

extern "C" int sg_step_tail_joint(const sg_net* net, const sg_small* sp, const sg_finish* f, const sg_joint* jp,
                                  uint32_t* jblob, uint32_t* sync, const void* prep, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && sp && f && jp && jblob && sync && f->stab, "sg_step_tail_joint: null argument");
  SG_REQUIRE(f->acc_mode == SG_ACC_MOVING || f->acc_mode == SG_ACC_EXPONENTIAL, "sg_step_tail_joint: bad mode");
  SG_REQUIRE(net->max_card <= SG_MAX_CARD && net->max_mb <= SG_MAX_MB, "sg_step_tail_joint: capacity exceeded");
  SG_REQUIRE(finish_fits(*net, sp), "sg_step_tail_joint: model too large for the single-CTA tail");
  SG_REQUIRE(sp->bits >= 2 && sp->bits <= SG_JOINT_MAXB && jp->patterns == (1 << sp->n) && jp->max_b >= 1,
             "sg_step_tail_joint: bad joint plan");
  if (net->table_entries > 0) SG_REQUIRE(f->ptab && f->ftab, "sg_step_tail_joint: tables required");
  if (f->key_table) SG_REQUIRE(f->key_index && f->key_current && f->kps > 0, "sg_step_tail_joint: bad key cursor");
  SG_REQUIRE(finish_check_ok(f, sp), "sg_step_tail_joint: bad observation check (aligned rows, err word)");
  FinishArgs a = make_finish_args(f, sp);
  a.early_inputs = 1;    // k_joint_sweep triggers after its own wait
  a.vprob = nullptr;     // the slices derive their conditionals from the CPTs themselves
  a.release_sync = sync;  // ... as soon as CTA 0 has written them
  // With f->vprob as scratch (n * 2^bits * 4 doubles), CTA 0 releases the cells' gamma draws right
  // after drawing them and every slice normalises the rows itself: CTA 0's row phase and its fence
  // leave the critical path.
  const size_t cells2 = size_t((net->cells + 1) & ~int64_t(1));
  const bool from_lg = f->vprob && size_t(sp->n) * (size_t(4) << sp->bits) * 8 >= size_t(net->cells) * 9;
  a.release_lg = from_lg ? f->vprob : nullptr;
  const size_t slice_smem = size_t(net->blob64_words) * 8 + ((size_t(net->blob32_words) * 4 + 15) & ~size_t(15)) +
                            cells2 * 8 + (from_lg ? cells2 * 8 + ((size_t(net->cells) + 15) & ~size_t(15)) : 0) +
                            joint_tables_smem(*sp, jp->max_b) +
                            (size_t(sp->n) << sp->bits) * SG_JOINT_MAXF * sizeof(int2) +
                            (((size_t(sp->n) << sp->bits) + 15) & ~size_t(15)) +
                            (size_t(1) << sp->bits) / SG_JOINT_TAB_SLICES * (size_t(1) << jp->max_b) * SG_SMALL_MAXV * 2;
  const size_t smem = std::max(finish_smem(*net), slice_smem);
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem)) {
    // opted in at any size: dynamic + the static alias scratch may pass 48 KB
    cudaFuncSetAttribute(k_step_tail_joint, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    // same carveout as k_joint_sweep (no L1/shared reconfiguration between sweep and tail)
    cudaFuncSetAttribute(k_step_tail_joint, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
  }
  // one CTA for the model update + the row slices (joint_tail_slices per pattern)
  const dim3 grid(1 + joint_tail_slice_count(*sp, *jp));
  SG_REQUIRE(!prep || (reinterpret_cast<uintptr_t>(prep) & 15) == 0, "sg_step_tail_joint: prep must be 16-byte aligned");
  TailRoles roles{};
  {  // the order of tail_slice_of: patterns from the last down
    int k = 0;
    for (int P = jp->patterns - 1; P >= 0 && k >= 0; --P) {
      int B = 0;
      for (int v = 0; v < sp->n; ++v)
        if ((P >> v) & 1) B += sp->width[v];
      const int nsl = joint_tail_slices(B);
      for (int s = 0; s < nsl; ++s) {
        if (k >= SG_TAIL_ROLE_MAX || P > 127 || nsl > 31) {
          k = -1;
          break;
        }
        roles.r[k++] = uint16_t(P | (s << 7) | (nsl << 11));
      }
    }
    roles.count = k > 0 ? k : 0;
  }
  launch_pdl(k_step_tail_joint, grid, dim3(FINISH_THREADS), smem, (cudaStream_t)stream, *net, a, *sp, *jp, jblob,
             sync, static_cast<const unsigned char*>(prep), joint_prep_slice_bytes(*sp, *jp), roles);
  return check_launch("sg_step_tail_joint");
}

SG_CHECKED_EXPORT(small)
