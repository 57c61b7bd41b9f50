// The chromatic Gibbs sweep + count tally, fused into one kernel.
//
// Reference: gibbs_pass sampler.py:251-284 walks colour groups in order and
// resamples, per variable, all of its latent lanes with numpy vector ops
// (_resample_variable sampler.py:217-248); sweep sampler.py:287-304 then
// tallies the final assignments (tally_counts model.py:148-165).
//
// B200 design.  Lanes never interact: the Markov blanket of (v, lane) lives
// in the same lane.  A CTA therefore owns a tile of TC cases x all m replicas
// x all n variables, stages the tile's int8 lane states in shared memory once
// (one coalesced HBM read), runs every colour group on-chip, tallies the
// final states, and writes the tile back (one HBM write).  Per colour group
// the CTA compacts the latent (variable, case) cells of the group into an
// item list (warp ballots), so threads only spend work on latent cells; an
// item carries all m replicas of one latent case (SAME replicas share the
// observed mask), in quads of 4 replicas = one Philox4x32 call in FAST mode.
// The draw itself is one Markov-blanket index + one conditional-table read
// (sg_tables.cu), or the reference's weight product for variables whose
// blanket is too large to tabulate.
#include "sg_device.cuh"

namespace sg {

enum TallyMode { TALLY_NONE = 0, TALLY_PRIVATE = 1, TALLY_SHARED = 2, TALLY_GLOBAL = 3 };

struct SweepArgs {
  const double* cpt;
  const double* ptab;
  const uint32_t* ftab;
  uint64_t fast_key;
  const uint64_t* keys;
  const double* uniforms;
  const int64_t* inj_off;
  uint64_t* counts;
  int32_t* err;
  int tc;           // cases per tile
  int tally_mode;
  int stage_tables; // 1: tables copied into shared memory
  int64_t tab_bytes;
};

struct SmemLayout {
  size_t st, items, tabs, hist, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout smem_layout(const sg_net& net, int m, int tc, int tally_mode,
                                                  int stage_tables, int64_t tab_bytes) {
  SmemLayout L;
  L.st = 0;
  size_t off = align16(size_t(net.n) * m * tc);
  L.items = off;
  off += align16(size_t(net.max_group) * tc * 4);
  L.tabs = off;
  if (stage_tables) off += align16(size_t(tab_bytes));
  L.hist = off;
  if (tally_mode == TALLY_PRIVATE) off += size_t(net.cells) * SG_THREADS * 4;
  else if (tally_mode == TALLY_SHARED) off += align16(size_t(net.cells) * 4);
  L.total = off;
  return L;
}

template <int MODE>
__device__ __forceinline__ void draw_item(const sg_net& net, const sg_batch& bt, const SweepArgs& a,
                                          const int8_t* __restrict__ st_in, int8_t* st, int tc,
                                          const double* ptab, const uint32_t* ftab, int v, int c,
                                          int rq, int c0, bool& zero_support) {
  const int m = bt.m;
  const int card = __ldg(net.card + v);
  const int64_t nent = __ldg(net.tab_entries + v);
  const int mb0 = __ldg(net.mb_start + v), mb1 = __ldg(net.mb_start + v + 1);
  const int r0 = rq * 4;
  const int r1 = min(r0 + 4, m);
  const int64_t gcase = bt.case_base + c0 + c;

  u32x4 fastw = {0, 0, 0, 0};
  if (MODE == SG_RNG_FAST) fastw = fast_block(a.fast_key, uint64_t(gcase), uint32_t(v), uint32_t(rq), 0u);
  int64_t rank = 0, nmiss = 0;
  uint64_t k0 = 0, k1 = 0;
  if (MODE != SG_RNG_FAST) {
    rank = __ldg(bt.rank + int64_t(v) * bt.ld_rank + c0 + c);
    nmiss = __ldg(bt.nmiss + v);
    if (MODE == SG_RNG_NUMPY) {
      k0 = __ldg(a.keys + 2 * v);
      k1 = __ldg(a.keys + 2 * v + 1);
    }
  }

  for (int r = r0; r < r1; ++r) {
    // ---- uniform
    uint32_t u31 = 0;
    double u = 0.0;
    if (MODE == SG_RNG_FAST) {
      const uint32_t w = pick(fastw, r - r0);
      u31 = w >> 1;
      u = double(w) * 0x1.0p-32;
    } else {
      const int64_t idx = int64_t(r) * nmiss + rank;  // reference lane order
      if (MODE == SG_RNG_NUMPY) u = np_uniform(uint64_t(idx), k0, k1);
      else u = __ldg(a.uniforms + __ldg(a.inj_off + v) + idx);
    }
    // ---- draw
    int x = 0;
    if (nent > 0) {
      int64_t e = 0;
      for (int k = mb0; k < mb1; ++k) {
        const int uvar = __ldg(net.mb_var + k);
        e += int64_t(st[(uvar * m + r) * tc + c] & 0x7F) * __ldg(net.mb_stride + k);
      }
      if (MODE == SG_RNG_FAST) {
        const uint32_t* th = ftab + __ldg(net.ftab_off + v) + e * (card - 1);
        if (th[0] == 0xFFFFFFFFu) zero_support = true;
        for (int s = 0; s < card - 1; ++s) x += (u31 >= th[s]);
      } else {
        const double* p = ptab + __ldg(net.ptab_off + v) + e * card;
        const double norm = p[card - 1];
        if (!(norm > 0.0)) zero_support = true;
        const double au = __dmul_rn(u, norm);
        for (int s = 0; s < card - 1; ++s) x += (au > p[s]);
      }
    } else {
      int s[SG_MAX_MB];
      for (int k = mb0; k < mb1; ++k) {
        const int uvar = __ldg(net.mb_var + k);
        s[k - mb0] = st[(uvar * m + r) * tc + c] & 0x7F;
      }
      double w[SG_MAX_CARD];
      conditional_weights(net, v, s, a.cpt, w);
      const double norm = np_pairwise_sum(w, card);
      if (!(norm > 0.0)) zero_support = true;
      const double au = __dmul_rn(u, norm);
      double cum = 0.0;
      for (int t = 0; t < card - 1; ++t) {
        cum = t ? __dadd_rn(cum, w[t]) : w[0];
        x += (au > cum);
      }
    }
    st[(v * m + r) * tc + c] = int8_t(0x80 | x);
  }
  (void)st_in;
}

template <int MODE>
__global__ void __launch_bounds__(SG_THREADS)
k_sweep(const sg_net net, const sg_batch bt, const SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_nitems;
  __shared__ int s_err;
  const int tc = a.tc;
  const int m = bt.m;
  const int n = net.n;
  const SmemLayout L = smem_layout(net, m, tc, a.tally_mode, a.stage_tables, a.tab_bytes);
  int8_t* st = reinterpret_cast<int8_t*>(smem + L.st);
  uint32_t* items = reinterpret_cast<uint32_t*>(smem + L.items);
  const int c0 = blockIdx.x * tc;
  const int ncase = min(tc, bt.cases - c0);        // sampled cases of this tile
  const int nreal = max(0, min(tc, bt.num_real - c0));  // tallied cases
  const int nload = min(tc, bt.pitch - c0);        // resident cases (multiple of 16)
  const int tid = threadIdx.x;
  if (tid == 0) s_err = 0;

  // ---- stage lane states: rows (v, r) of nload bytes, 16 B per thread-load
  {
    const int chunks = nload >> 4;
    const int per_row = tc >> 4;
    const int total = n * m * chunks;
    for (int i = tid; i < total; i += SG_THREADS) {
      const int row = i / chunks, ch = i - row * chunks;
      const int4 val = *reinterpret_cast<const int4*>(bt.states + int64_t(row) * bt.pitch + c0 + ch * 16);
      reinterpret_cast<int4*>(st)[row * per_row + ch] = val;
    }
  }
  const double* ptab = a.ptab;
  const uint32_t* ftab = a.ftab;
  if (a.stage_tables) {
    const int words = int(a.tab_bytes >> 2);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem + L.tabs);
    const uint32_t* src = MODE == SG_RNG_FAST ? a.ftab : reinterpret_cast<const uint32_t*>(a.ptab);
    for (int i = tid; i < words; i += SG_THREADS) dst[i] = __ldg(src + i);
    if (MODE == SG_RNG_FAST) ftab = dst;
    else ptab = reinterpret_cast<const double*>(dst);
  }
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
  if (a.counts && a.tally_mode == TALLY_PRIVATE) {
    const int words = int(net.cells) * SG_THREADS;
    for (int i = tid; i < words; i += SG_THREADS) hist[i] = 0;
  } else if (a.counts && a.tally_mode == TALLY_SHARED) {
    for (int i = tid; i < int(net.cells); i += SG_THREADS) hist[i] = 0;
  }
  __syncthreads();

  // ---- colour groups, strictly in order
  const int warp = tid >> 5, lane = tid & 31;
  const int nchunk = (ncase + 31) >> 5;
  const int Q = (m + 3) >> 2;
  bool zero_support = false;
  for (int g = 0; g < net.num_groups; ++g) {
    const int gs = __ldg(net.group_start + g), ge = __ldg(net.group_start + g + 1);
    if (tid == 0) s_nitems = 0;
    __syncthreads();
    const int units = (ge - gs) * nchunk;
    for (int uidx = warp; uidx < units; uidx += SG_THREADS / 32) {
      const int vi = gs + uidx / nchunk;
      const int ch = uidx - (uidx / nchunk) * nchunk;
      const int v = __ldg(net.order + vi);
      const int c = ch * 32 + lane;
      const bool lat = c < ncase && (st[(v * m) * tc + c] & 0x80);
      const unsigned mask = __ballot_sync(0xffffffffu, lat);
      int base = 0;
      if (lane == 0 && mask) base = atomicAdd(&s_nitems, __popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (lat) items[base + __popc(mask & lanemask_lt())] = (uint32_t(v) << 16) | uint32_t(c);
    }
    __syncthreads();
    const int work = s_nitems * Q;
    for (int j = tid; j < work; j += SG_THREADS) {
      const int it = j / Q, rq = j - it * Q;
      const uint32_t item = items[it];
      draw_item<MODE>(net, bt, a, nullptr, st, tc, ptab, ftab, int(item >> 16), int(item & 0xFFFFu),
                      rq, c0, zero_support);
    }
    __syncthreads();
  }
  if (zero_support) atomicOr(&s_err, int(SG_ERR_ZERO_SUPPORT));

  // ---- tally of the final assignments over real lanes
  if (a.counts && nreal > 0) {
    const int lanes = m * nreal;
    for (int j = tid; j < lanes; j += SG_THREADS) {
      const int r = j / nreal, c = j - r * nreal;
      for (int v = 0; v < n; ++v) {
        int64_t cfg = 0;
        for (int p = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1); p < pe; ++p)
          cfg += int64_t(st[(__ldg(net.par_var + p) * m + r) * tc + c] & 0x7F) * __ldg(net.par_stride + p);
        const int card = __ldg(net.card + v);
        const int64_t cell = __ldg(net.cpt_off + v) + cfg * card + (st[(v * m + r) * tc + c] & 0x7F);
        if (a.tally_mode == TALLY_PRIVATE) hist[cell * SG_THREADS + tid] += 1u;
        else if (a.tally_mode == TALLY_SHARED) atomicAdd(hist + cell, 1u);
        else atomicAdd(reinterpret_cast<unsigned long long*>(a.counts) + cell, 1ull);
      }
    }
    __syncthreads();
    if (a.tally_mode == TALLY_PRIVATE) {
      for (int cell = tid; cell < int(net.cells); cell += SG_THREADS) {
        uint32_t sum = 0;
        for (int t = 0; t < SG_THREADS; ++t) sum += hist[cell * SG_THREADS + ((t + cell) & (SG_THREADS - 1))];
        if (sum) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts) + cell, (unsigned long long)sum);
      }
    } else if (a.tally_mode == TALLY_SHARED) {
      for (int cell = tid; cell < int(net.cells); cell += SG_THREADS)
        if (hist[cell]) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts) + cell,
                                  (unsigned long long)hist[cell]);
    }
  }

  // ---- write the tile back
  {
    const int chunks = nload >> 4;
    const int per_row = tc >> 4;
    const int total = n * m * chunks;
    for (int i = tid; i < total; i += SG_THREADS) {
      const int row = i / chunks, ch = i - row * chunks;
      *reinterpret_cast<int4*>(bt.states + int64_t(row) * bt.pitch + c0 + ch * 16) =
          reinterpret_cast<const int4*>(st)[row * per_row + ch];
    }
  }
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(a.err, s_err);
}

// Standalone tally over the lanes of a resident batch (no sampling).
__global__ void __launch_bounds__(SG_THREADS)
k_tally(const sg_net net, const sg_batch bt, unsigned long long* counts,
        const double* weights, double* wcounts) {
  const int64_t lanes = int64_t(bt.m) * bt.num_real;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < lanes;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(j / bt.num_real);
    const int c = int(j - int64_t(r) * bt.num_real);
    const int8_t* base = bt.states + int64_t(r) * bt.pitch + c;
    const int64_t vstride = int64_t(bt.m) * bt.pitch;
    const double wt = weights ? weights[int64_t(r) * bt.cases + c] : 1.0;
    for (int v = 0; v < net.n; ++v) {
      int64_t cfg = 0;
      for (int p = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1); p < pe; ++p)
        cfg += int64_t(base[__ldg(net.par_var + p) * vstride] & 0x7F) * __ldg(net.par_stride + p);
      const int64_t cell = __ldg(net.cpt_off + v) + cfg * __ldg(net.card + v) + (base[v * vstride] & 0x7F);
      if (weights) atomicAdd(wcounts + cell, wt);
      else atomicAdd(counts + cell, 1ull);
    }
  }
}

static int choose_tile(const sg_net& net, int m, int cases, int tally_mode, int stage, int64_t tab_bytes,
                       int* tc_out, size_t* smem_out) {
  int best = 0;
  // largest power-of-two tile (<= 512 cases) whose shared memory leaves room
  // for at least two CTAs per SM; fall back to one CTA of up to 200 KB.
  for (int budget : {100 * 1024, 200 * 1024}) {
    for (int tc = 512; tc >= 32; tc >>= 1) {
      const SmemLayout L = smem_layout(net, m, tc, tally_mode, stage, tab_bytes);
      if (L.total <= size_t(budget)) {
        best = tc;
        break;
      }
    }
    if (best) break;
  }
  if (!best) return SG_ECAPACITY;
  // do not make tiles much larger than the minibatch
  while (best > 32 && best / 2 >= cases) best >>= 1;
  *tc_out = best;
  *smem_out = smem_layout(net, m, best, tally_mode, stage, tab_bytes).total;
  return SG_OK;
}

}  // namespace sg

extern "C" int sg_sweep(const sg_net* net, const sg_batch* batch, const double* cpt,
                        const double* ptab, const uint32_t* ftab, int32_t rng_mode,
                        uint64_t fast_key, const uint64_t* keys, const double* uniforms,
                        const int64_t* inj_off, uint64_t* counts, int32_t* err, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && batch && err, "sg_sweep: null argument");
  SG_REQUIRE(batch->states, "sg_sweep: null states");
  SG_REQUIRE(batch->m >= 1 && batch->cases >= 0 && batch->pitch >= batch->cases &&
                 batch->pitch % 16 == 0 && batch->num_real <= batch->cases,
             "sg_sweep: bad batch shape m=%d cases=%d pitch=%d real=%d", batch->m, batch->cases,
             batch->pitch, batch->num_real);
  SG_REQUIRE(net->n < 32768, "sg_sweep: n=%d exceeds 32767", net->n);
  SG_REQUIRE(net->max_card <= SG_MAX_CARD && net->max_mb <= SG_MAX_MB,
             "sg_sweep: card/blanket capacity exceeded");
  SG_REQUIRE(rng_mode >= SG_RNG_FAST && rng_mode <= SG_RNG_INJECTED, "sg_sweep: bad rng mode %d",
             rng_mode);
  if (rng_mode != SG_RNG_FAST)
    SG_REQUIRE(batch->rank && batch->nmiss, "sg_sweep: rank/nmiss required for this rng mode");
  if (rng_mode == SG_RNG_NUMPY) SG_REQUIRE(keys, "sg_sweep: numpy keys required");
  if (rng_mode == SG_RNG_INJECTED) SG_REQUIRE(uniforms && inj_off, "sg_sweep: uniforms required");
  if (net->table_entries > 0) SG_REQUIRE(ptab && ftab, "sg_sweep: tables required");
  if (net->direct_vars > 0) SG_REQUIRE(cpt, "sg_sweep: cpt required for direct variables");
  if (batch->cases == 0) return SG_OK;

  SweepArgs a;
  a.cpt = cpt;
  a.ptab = ptab;
  a.ftab = ftab;
  a.fast_key = fast_key;
  a.keys = keys;
  a.uniforms = uniforms;
  a.inj_off = inj_off;
  a.counts = counts;
  a.err = err;
  a.tab_bytes = rng_mode == SG_RNG_FAST ? net->ftab_size * 4 : net->ptab_size * 8;
  a.stage_tables = (net->table_entries > 0 && a.tab_bytes <= 32 * 1024) ? 1 : 0;
  if (!counts) a.tally_mode = TALLY_NONE;
  else if (net->cells * SG_THREADS * 4 <= 40 * 1024) a.tally_mode = TALLY_PRIVATE;
  else if (net->cells * 4 <= 48 * 1024) a.tally_mode = TALLY_SHARED;
  else a.tally_mode = TALLY_GLOBAL;
  size_t smem = 0;
  int st = choose_tile(*net, batch->m, batch->cases, a.tally_mode, a.stage_tables, a.tab_bytes, &a.tc, &smem);
  if (st != SG_OK) {
    set_error("sg_sweep: tile of n=%d x m=%d does not fit in shared memory", net->n, batch->m);
    return st;
  }
  const int blocks = (batch->cases + a.tc - 1) / a.tc;
  cudaStream_t s = (cudaStream_t)stream;
  switch (rng_mode) {
    case SG_RNG_FAST:
      cudaFuncSetAttribute(k_sweep<SG_RNG_FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      k_sweep<SG_RNG_FAST><<<blocks, SG_THREADS, smem, s>>>(*net, *batch, a);
      break;
    case SG_RNG_NUMPY:
      cudaFuncSetAttribute(k_sweep<SG_RNG_NUMPY>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      k_sweep<SG_RNG_NUMPY><<<blocks, SG_THREADS, smem, s>>>(*net, *batch, a);
      break;
    default:
      cudaFuncSetAttribute(k_sweep<SG_RNG_INJECTED>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      k_sweep<SG_RNG_INJECTED><<<blocks, SG_THREADS, smem, s>>>(*net, *batch, a);
      break;
  }
  return check_launch("sg_sweep");
}

extern "C" int sg_tally(const sg_net* net, const sg_batch* batch, uint64_t* counts, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && batch && counts && batch->states, "sg_tally: null argument");
  const int64_t lanes = int64_t(batch->m) * batch->num_real;
  if (lanes == 0) return SG_OK;
  const int blocks = int((lanes + SG_THREADS - 1) / SG_THREADS < 148 * 32 ? (lanes + SG_THREADS - 1) / SG_THREADS
                                                                          : 148 * 32);
  k_tally<<<blocks, SG_THREADS, 0, (cudaStream_t)stream>>>(
      *net, *batch, reinterpret_cast<unsigned long long*>(counts), nullptr, nullptr);
  return check_launch("sg_tally");
}

extern "C" int sg_tally_weighted(const sg_net* net, const sg_batch* batch, const double* weights,
                                 double* counts, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && batch && counts && weights && batch->states, "sg_tally_weighted: null argument");
  const int64_t lanes = int64_t(batch->m) * batch->num_real;
  if (lanes == 0) return SG_OK;
  const int blocks = int((lanes + SG_THREADS - 1) / SG_THREADS < 148 * 32 ? (lanes + SG_THREADS - 1) / SG_THREADS
                                                                          : 148 * 32);
  k_tally<<<blocks, SG_THREADS, 0, (cudaStream_t)stream>>>(*net, *batch, nullptr, weights, counts);
  return check_launch("sg_tally_weighted");
}
