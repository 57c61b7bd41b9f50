// The chromatic Gibbs sweep + count tally, fused into one kernel.
//
// Reference: gibbs_pass sampler.py:251-284 walks colour groups in order and
// resamples, per variable, all of its latent lanes with numpy vector ops
// (_resample_variable sampler.py:217-248); sweep sampler.py:287-304 then
// tallies the final assignments (tally_counts model.py:148-165).
//
// B200 design.  Lanes never interact: the Markov blanket of (v, lane) lives
// in the same lane.  A CTA owns a tile of TC cases x all m replicas x all n
// variables:
//   1. one coalesced 16-byte-per-thread HBM read stages the tile's lane
//      states in shared memory, splitting the latent flags (bit 7) into one
//      32-case bit mask per variable (SAME replicas share the mask);
//   2. per colour group, the latent (variable, case) cells are compacted,
//      variable-major, into an item list (block scan over mask popcounts), so
//      a warp's 32 consecutive items mostly share one variable (broadcast
//      descriptor loads, little divergence); an item carries all m replicas
//      of its case, handled in quads of 4 independent draws = one Philox4x32
//      call (FAST mode);
//   3. a draw is a Markov-blanket index (one LDS.U8 + IMAD per member, the
//      member count a template parameter) and a conditional-table read
//      (sg_tables.cu) compared with the uniform, or the reference's weight
//      product for variables without a table;
//   4. small models tally the final lanes on-chip -- whole-lane joint states
//      (Koller: 48) or CPT cells (<= 128) in per-thread byte counters -- and
//      flush one atomic per touched cell per CTA; larger models are counted
//      by k_tally_chunked after the sweep (shared-memory histograms per run of
//      variables, one atomic per cell per CTA);
//   5. one coalesced HBM write puts the tile back.
#include "sg_sweep.cuh"

// draw_factored variant of the lane kernel: cards <= SG_LANE_UNIFIED share one path (0 = per card;
// measured on C3: per card 3.40 ms, unified <= 3 3.78 ms, unified <= 4 3.80 ms)
#ifndef SG_LANE_UNIFIED
#define SG_LANE_UNIFIED 0
#endif

namespace sg {

struct SmemLayout {
  size_t st, lat, items, desc, tabs, hist, cellacc, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// SMALL: descriptors and conditional tables live in shared memory.
__host__ __device__ inline SmemLayout smem_layout(const sg_net& net, int m, int tc, int tally_mode, bool small,
                                                  int64_t tab_bytes) {
  SmemLayout L;
  size_t off = 0;
  L.st = off;
  off += align16(size_t(net.n) * m * tc);
  L.lat = off;
  off += align16(size_t(net.n) * (tc / 32) * 4);
  L.items = off;
  off += align16(size_t(net.max_group) * tc * 4);
  L.desc = off;
  if (small) off += align16(size_t(net.n) * SG_DESC_WORDS * 4);
  L.tabs = off;
  if (small) off += align16(size_t(tab_bytes));
  L.hist = off;
  if (tally_mode == TALLY_JOINT) off += align16(size_t(net.joint_size) * SG_THREADS);
  else if (tally_mode == TALLY_CELL8) off += align16(size_t(net.cells) * SG_THREADS);
  L.cellacc = off;
  if (tally_mode == TALLY_JOINT) off += align16(size_t(net.cells) * 4 + 64);
  L.total = off;
  return L;
}

// Byte slot of thread tid in a per-thread byte-counter row of SG_THREADS
// bytes: lane l of every warp lands in bank l, so a warp's increments never
// conflict whatever bins its lanes hit.
static_assert(SG_THREADS == 256, "hist_slot assumes 8 warps per CTA");
__device__ __forceinline__ int hist_slot(int tid) {
  return ((tid & 31) << 2) | ((tid >> 5) & 3) | ((tid >> 7) << 7);
}

// Expand 4 flag bits (bit i -> byte i) into 0x80 markers.
__device__ __forceinline__ uint32_t flags_to_bytes(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) << 7;
}

// Gather bit 7 of each byte of w into bits 0..3.
__device__ __forceinline__ uint32_t byte_flags(uint32_t w) {
  return (((w & 0x80808080u) >> 7) * 0x01020408u) >> 24;
}

// Block-wide exclusive scan of one int per thread; *total gets the sum.
__device__ __forceinline__ int block_scan(int x, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  int base = 0, sum = 0;
#pragma unroll
  for (int w = 0; w < SG_THREADS / 32; ++w) {
    const int t = s_warp[w];
    base += w < warp ? t : 0;
    sum += t;
  }
  __syncthreads();
  *total = sum;
  return base + inc - x;
}

struct ItemCtx {
  int8_t* st;
  int mtc, tc, m;  // m = replicas in this tile (local rows), r0 = global replica of local row 0
  int r0;
  int64_t gcase0;  // global index of the tile's case 0
  int c0;
  uint64_t key;    // FAST key of this sweep
};

// Draw all m replicas of latent cell (v, c); K = Markov-blanket members
// (K < 0: evaluate from the CPTs).  Quads of 4 replicas are independent
// draws, written out so the compiler can overlap their loads.
template <int MODE, int K>
__device__ __forceinline__ void draw_cell(const ItemCtx& x, const sg_net& net, const SweepArgs& a,
                                          const int32_t* dv, const uint32_t* ftab, const double* ptab,
                                          const sg_batch& bt, int v, int c, bool zs_armed, bool& zs) {
  const int card = dv[0];
  const int mtc = x.mtc, tc = x.tc, m = x.m;
  int rows[K > 0 ? K : 1], strd[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    rows[k] = dv[4 + k] * mtc + c;
    strd[k] = dv[4 + SG_DESC_MB + k];
  }
  int8_t* out = x.st + v * mtc + c;
  const uint32_t* tf = ftab + (K >= 0 ? dv[2] : 0);
  const double* tp = ptab + (K >= 0 ? dv[3] : 0);
  int64_t rank = 0, nmiss = 0, ioff = 0;
  uint64_t k0 = 0, k1 = 0;
  if (MODE != SG_RNG_FAST) {
    rank = __ldg(bt.rank + int64_t(v) * bt.ld_rank + x.c0 + c);
    nmiss = __ldg(bt.nmiss + v);
    if (MODE == SG_RNG_NUMPY) {
      k0 = __ldg(a.keys + 2 * v);
      k1 = __ldg(a.keys + 2 * v + 1);
    } else {
      ioff = __ldg(a.inj_off + v);
    }
  }
  // global replica quads overlapping this tile's replicas [r0, r0 + m)
  const int q_lo = x.r0 >> 2, q_hi = (x.r0 + m - 1) >> 2;
  for (int rq = q_lo; rq <= q_hi; ++rq) {
    uint32_t u31[4];
    double u[4];
    int loc[4];  // local replica row of word j (clamped; `ok` tells whether it is ours)
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int l = rq * 4 + j - x.r0;
      ok[j] = l >= 0 && l < m;
      loc[j] = min(max(l, 0), m - 1);
    }
    if (MODE == SG_RNG_FAST) {
      const u32x4 w = fast_block(x.key, uint64_t(x.gcase0 + c), uint32_t(v), uint32_t(rq), 0u);
      u31[0] = w.a >> 1;
      u31[1] = w.b >> 1;
      u31[2] = w.c >> 1;
      u31[3] = w.d >> 1;
      u[0] = double(w.a) * 0x1.0p-32;
      u[1] = double(w.b) * 0x1.0p-32;
      u[2] = double(w.c) * 0x1.0p-32;
      u[3] = double(w.d) * 0x1.0p-32;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = x.r0 + loc[j];
        const int64_t idx = int64_t(r) * nmiss + rank;  // reference lane order (sampler.py:245)
        u[j] = MODE == SG_RNG_NUMPY ? np_uniform(uint64_t(idx), k0, k1) : __ldg(a.uniforms + ioff + idx);
        u31[j] = 0;
      }
    }
    int xs[4];
    if (K >= 0) {
      int e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int roff = loc[j] * tc;
        int acc = 0;
#pragma unroll
        for (int k = 0; k < (K > 0 ? K : 0); ++k) acc += int(x.st[rows[k] + roff]) * strd[k];
        e[j] = acc;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int s = 0;
        if (MODE == SG_RNG_FAST) {
          const uint32_t* th = tf + e[j] * (card - 1);
          const uint32_t t0 = th[0];
          if (zs_armed && ok[j] && t0 == 0xFFFFFFFFu) zs = true;
          s = u31[j] >= t0;
          if (card > 2) {
            s += u31[j] >= th[1];
            if (card > 3) {
              s += u31[j] >= th[2];
              for (int q = 3; q < card - 1; ++q) s += (u31[j] >= th[q]);
            }
          }
        } else {
          const double* p = tp + int64_t(e[j]) * card;
          const double norm = p[card - 1];
          if (ok[j] && !(norm > 0.0)) zs = true;
          const double au = __dmul_rn(u[j], norm);
          for (int q = 0; q < card - 1; ++q) s += (au > p[q]);
        }
        xs[j] = s;
      }
    } else {
      const int32_t* fd = net.fac_desc + __ldg(net.fac_start + v);
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const int8_t* col = x.st + loc[j] * tc + c;
        xs[j] = ok[j] ? draw_factored(fd, a.cpt, [&](int var) { return int(col[var * mtc]); }, u[j], zs) : 0;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ok[j]) out[loc[j] * tc] = int8_t(xs[j]);
  }
}

template <int MODE>
__device__ __forceinline__ void draw_dispatch(int nmb, const ItemCtx& x, const sg_net& net, const SweepArgs& a,
                                              const int32_t* dv, const uint32_t* ftab, const double* ptab,
                                              const sg_batch& bt, int v, int c, bool zs_armed, bool& zs) {
  switch (nmb) {
    case 0: draw_cell<MODE, 0>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 1: draw_cell<MODE, 1>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 2: draw_cell<MODE, 2>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 3: draw_cell<MODE, 3>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 4: draw_cell<MODE, 4>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 5: draw_cell<MODE, 5>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 6: draw_cell<MODE, 6>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 7: draw_cell<MODE, 7>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    case 8: draw_cell<MODE, 8>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
    default: draw_cell<MODE, -1>(x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs); break;
  }
}

// Joint-state tally of N <= 7 variables (prod card <= SG_JOINT_MAX).
template <int N>
__device__ __forceinline__ void tally_joint(const int8_t* st, int mtc, int tc, int m, int nreal,
                                            const int32_t* radix, uint8_t* hist8, int slot) {
  int R[N];
#pragma unroll
  for (int k = 0; k < N; ++k) R[k] = __ldg(radix + k);
  for (int r = 0; r < m; ++r) {
    const int8_t* row = st + r * tc;
    for (int c = threadIdx.x; c < nreal; c += SG_THREADS) {
      int J = 0;
#pragma unroll
      for (int k = 0; k < N; ++k) J += int(row[k * mtc + c]) * R[k];
      hist8[J * SG_THREADS + slot] += 1;
    }
  }
}

template <int MODE, bool SMALL>
#ifndef SG_SWEEP_NP_MINB
#define SG_SWEEP_NP_MINB 3  // CTAs per SM for the NUMPY / INJECTED modes: 80 registers, a few spills, 37.5 % occupancy (2: 128 registers, 6 % slower)
#endif
#ifndef SG_SWEEP_INJ_MINB
#define SG_SWEEP_INJ_MINB 4  // INJECTED (the numpy-parity sweep on pre-generated uniforms): no Philox state
#endif
__global__ void __launch_bounds__(SG_THREADS, MODE == SG_RNG_FAST       ? 4
                                              : MODE == SG_RNG_INJECTED ? SG_SWEEP_INJ_MINB
                                                                        : SG_SWEEP_NP_MINB)
k_sweep(const sg_net net, const sg_batch bt, const SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_warp[SG_THREADS / 32];
  __shared__ int s_err;
  const int tc = a.tc;
  const int rg0 = blockIdx.y * a.mg;              // first replica of this tile
  const int m = min(a.mg, bt.m - rg0);            // replicas of this tile (local rows)
  const int n = net.n;
  const int mtc = m * tc;
  const int words = tc >> 5;  // flag words per variable
  const SmemLayout L = smem_layout(net, a.mg, tc, a.tally_mode, SMALL, a.tab_bytes);
  int8_t* st = reinterpret_cast<int8_t*>(smem + L.st);
  uint32_t* lat = reinterpret_cast<uint32_t*>(smem + L.lat);
  uint16_t* lat16 = reinterpret_cast<uint16_t*>(smem + L.lat);
  uint32_t* items = reinterpret_cast<uint32_t*>(smem + L.items);
  const int c0 = blockIdx.x * tc;
  const int ncase = min(tc, bt.cases - c0);             // sampled cases of this tile
  const int nreal = max(0, min(tc, bt.num_real - c0));  // tallied cases
  const int nload = min(tc, bt.pitch - c0);             // resident cases (multiple of 16)
  const int tid = threadIdx.x;
  if (tid == 0) s_err = 0;

  // ---- 1. stage lane states (flags stripped) + latent masks
  // A thread always handles chunk `ch` of rows row0, row0 + step, ... (tc/16
  // divides the CTA size), so (v, r) advance without divisions.
  const int per_row = tc >> 4;
  const int lg_row = __ffs(per_row) - 1;
  const int my_ch = tid & (per_row - 1);
  const int row_step = SG_THREADS >> lg_row;
  const int row0 = tid >> lg_row;
  const int v0 = row0 / m, r0 = row0 - v0 * m;
  const int step_v = row_step / m, step_r = row_step - step_v * m;  // (v, r) advance per row step
  {
    const int chunks = nload >> 4;
    const int ch = my_ch;
    int v = v0, r = r0;
    for (int row = row0; ch < chunks && row < n * m; row += row_step) {
      int4 val = __ldcs(reinterpret_cast<const int4*>(bt.states + (int64_t(v) * bt.m + rg0 + r) * bt.pitch + c0 +
                                                       ch * 16));
      const bool first = r == 0;  // first replica of the tile (every replica carries the shared mask)
      const int vcur = v;
      r += step_r;
      v += step_v;
      if (r >= m) {
        r -= m;
        ++v;
      }
      if (first) {  // replica 0 carries the mask of all replicas
        const int v = vcur;
        uint32_t bits = byte_flags(val.x) | (byte_flags(val.y) << 4) | (byte_flags(val.z) << 8) |
                        (byte_flags(val.w) << 12);
        const int cc = ch * 16;
        if (cc + 16 > ncase) bits &= cc >= ncase ? 0u : ((1u << (ncase - cc)) - 1u);
        lat16[v * (words * 2) + ch] = uint16_t(bits);
      }
      val.x &= 0x7F7F7F7F;
      val.y &= 0x7F7F7F7F;
      val.z &= 0x7F7F7F7F;
      val.w &= 0x7F7F7F7F;
      reinterpret_cast<int4*>(st)[row * per_row + ch] = val;
    }
    if (nload < tc) {  // tile past the row pitch: clear the masks of unloaded chunks
      const int hw = words * 2;
      for (int i = tid; i < n * hw; i += SG_THREADS)
        if ((i % hw) * 16 >= nload) lat16[i] = 0;
    }
  }
  const int32_t* desc = net.var_desc;
  const double* ptab = a.ptab;
  const uint32_t* ftab = a.ftab;
  const bool zs_armed = a.ftab && net.table_entries > 0 && __ldg(a.ftab + net.ftab_size) != 0u;
  if (SMALL) {
    int32_t* d = reinterpret_cast<int32_t*>(smem + L.desc);
    for (int i = tid; i < n * SG_DESC_WORDS; i += SG_THREADS) d[i] = __ldg(net.var_desc + i);
    desc = d;
    // tables always addressed in shared memory here (empty when no variable has one)
    const int tw = int(a.tab_bytes >> 2);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem + L.tabs);
    const uint32_t* src = MODE == SG_RNG_FAST ? a.ftab : reinterpret_cast<const uint32_t*>(a.ptab);
    for (int i = tid; i < tw; i += SG_THREADS) dst[i] = __ldg(src + i);
    ftab = dst;
    ptab = reinterpret_cast<const double*>(dst);
  }
  uint8_t* hist8 = reinterpret_cast<uint8_t*>(smem + L.hist);
  uint32_t* hist32 = reinterpret_cast<uint32_t*>(smem + L.hist);
  uint32_t* cellacc = reinterpret_cast<uint32_t*>(smem + L.cellacc);
  if (a.counts) {
    if (a.tally_mode == TALLY_JOINT || a.tally_mode == TALLY_CELL8) {
      const int bytes = (a.tally_mode == TALLY_JOINT ? int(net.joint_size) : int(net.cells)) * SG_THREADS;
      for (int i = tid; i < bytes / 4; i += SG_THREADS) hist32[i] = 0;
      if (a.tally_mode == TALLY_JOINT)
        for (int i = tid; i < int(net.cells); i += SG_THREADS) cellacc[i] = 0;
    }
  }
  __syncthreads();

  // ---- 2-3. colour groups, strictly in order
  ItemCtx x;
  x.st = st;
  x.mtc = mtc;
  x.tc = tc;
  x.m = m;
  x.r0 = rg0;
  x.gcase0 = bt.case_base + c0;
  x.key = a.fast_key_dev ? __ldg(a.fast_key_dev) : a.fast_key;
  x.c0 = c0;
  bool zs = false;
  for (int g = 0; g < net.num_groups; ++g) {
    const int gs = __ldg(net.group_start + g), ge = __ldg(net.group_start + g + 1);
    // variable-major compaction of the group's latent cells
    const int units = (ge - gs) * words;
    int nitems = 0;
    for (int u0 = 0; u0 < units; u0 += SG_THREADS) {
      const int uidx = u0 + tid;
      uint32_t mask = 0;
      int v = 0, w = 0;
      if (uidx < units) {
        const int vi = gs + uidx / words;
        w = uidx - (uidx / words) * words;
        v = __ldg(net.order + vi);
        mask = lat[v * words + w];
      }
      int chunk_total;
      int pos = nitems + block_scan(__popc(mask), s_warp, &chunk_total);
      const uint32_t hi = uint32_t(v) << 16;
      while (mask) {
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        items[pos++] = hi | uint32_t(w * 32 + b);
      }
      nitems += chunk_total;
    }
    __syncthreads();
    for (int it = tid; it < nitems; it += SG_THREADS) {
      const uint32_t item = items[it];
      const int v = int(item >> 16), c = int(item & 0xFFFFu);
      const int32_t* dv = desc + v * SG_DESC_WORDS;
      draw_dispatch<MODE>(dv[1], x, net, a, dv, ftab, ptab, bt, v, c, zs_armed, zs);
    }
    __syncthreads();
  }
  if (zs) atomicOr(&s_err, int(SG_ERR_ZERO_SUPPORT));

  // ---- 4. tally of the final assignments over real lanes
  if (a.counts && nreal > 0) {
    const int slot = hist_slot(tid);
    if (a.tally_mode == TALLY_JOINT) {
      switch (n) {
        case 1: tally_joint<1>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        case 2: tally_joint<2>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        case 3: tally_joint<3>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        case 4: tally_joint<4>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        case 5: tally_joint<5>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        case 6: tally_joint<6>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
        default: tally_joint<7>(st, mtc, tc, m, nreal, net.joint_radix, hist8, slot); break;
      }
      __syncthreads();
      // bins -> cells: each warp sums a bin's 256 byte counters with dp4a
      const int warp = tid >> 5, lane_id = tid & 31;
      for (int J = warp; J < int(net.joint_size); J += SG_THREADS / 32) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(hist8 + J * SG_THREADS);
        int sum = __dp4a(int(row[lane_id]), 0x01010101, 0);
        sum = __dp4a(int(row[lane_id + 32]), 0x01010101, sum);
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (sum && lane_id < n) atomicAdd(cellacc + __ldg(net.joint_cell + J * n + lane_id), uint32_t(sum));
      }
      __syncthreads();
      for (int cell = tid; cell < int(net.cells); cell += SG_THREADS)
        if (cellacc[cell])
          atomicAdd(reinterpret_cast<unsigned long long*>(a.counts) + cell, (unsigned long long)cellacc[cell]);
    } else {
      for (int r = 0; r < m; ++r) {
        const int8_t* lane_row = st + r * tc;
        for (int c = tid; c < nreal; c += SG_THREADS) {
          for (int v = 0; v < n; ++v) {
            int cfg = 0;
            for (int p = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1); p < pe; ++p)
              cfg += int(lane_row[__ldg(net.par_var + p) * mtc + c]) * __ldg(net.par_stride + p);
            const int64_t cell =
                __ldg(net.cpt_off + v) + int64_t(cfg) * __ldg(net.card + v) + lane_row[v * mtc + c];
            SG_DCHECK(cell >= __ldg(net.cpt_off + v) && cell < (v + 1 < n ? __ldg(net.cpt_off + v + 1) : net.cells));
            hist8[cell * SG_THREADS + slot] += 1;
          }
        }
      }
      __syncthreads();
      {
        const int warp = tid >> 5, lane_id = tid & 31;
        for (int cell = warp; cell < int(net.cells); cell += SG_THREADS / 32) {
          const uint32_t* row = reinterpret_cast<const uint32_t*>(hist8 + size_t(cell) * SG_THREADS);
          int sum = __dp4a(int(row[lane_id]), 0x01010101, 0);
          sum = __dp4a(int(row[lane_id + 32]), 0x01010101, sum);
#pragma unroll
          for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          if (sum && lane_id == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.counts) + cell, (unsigned long long)sum);
        }
      }
    }
  }

  // ---- 5. write the tile back (flags restored from the masks)
  {
    const int chunks = nload >> 4;
    const int ch = my_ch;
    int v = v0, r = r0;
    for (int row = row0; ch < chunks && row < n * m; row += row_step) {
      const uint32_t bits = lat16[v * (words * 2) + ch];
      const int vcur = v, rcur = r;
      r += step_r;
      v += step_v;
      if (r >= m) {
        r -= m;
        ++v;
      }
      int4 val = reinterpret_cast<const int4*>(st)[row * per_row + ch];
      val.x |= flags_to_bytes(bits & 0xF);
      val.y |= flags_to_bytes((bits >> 4) & 0xF);
      val.z |= flags_to_bytes((bits >> 8) & 0xF);
      val.w |= flags_to_bytes((bits >> 12) & 0xF);
      __stcs(reinterpret_cast<int4*>(bt.states + (int64_t(vcur) * bt.m + rg0 + rcur) * bt.pitch + c0 + ch * 16),
             val);
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
      SG_DCHECK(cell >= __ldg(net.cpt_off + v) && cell < (v + 1 < net.n ? __ldg(net.cpt_off + v + 1) : net.cells));
      if (weights) atomicAdd(wcounts + cell, wt);
      else atomicAdd(counts + cell, 1ull);
    }
  }
}

// ---------------------------------------------------------------- lane sweep
//
// Large networks (n > 32, card <= 16): one thread per lane (case c, replica r)
// walks every variable in colour order, keeping its own column of states
// bit-packed in shared memory (BITS per state) with one latent bit per
// variable.  A single lane's sequential scan in colour order is exactly the
// reference's group-by-group update of that lane (members of a group are
// conditionally independent, lanes never interact), so there are no
// colour-group barriers, no item compaction and no write races; the
// variable is warp-uniform, so its descriptors are broadcast loads and the
// draw kind never diverges.  A warp skips a variable no lane of it has
// latent; otherwise only the latent lanes draw.  HBM traffic: every cell read
// once, every latent cell written once (n * L * (1 + f) bytes).
constexpr int LANE_T = 128;

template <int BITS>
struct LaneColumn {
  uint32_t* st;  // state word w of this thread at st[w * LANE_T]
  uint32_t* fl;  // latent word w at fl[w * LANE_T]
  static constexpr int PER = 32 / BITS;
  static constexpr uint32_t MASK = (1u << BITS) - 1u;
  __device__ __forceinline__ int get(int v) const {
    const uint32_t u = uint32_t(v);
    return int((st[(u / PER) * LANE_T] >> ((u % PER) * BITS)) & MASK);
  }
  __device__ __forceinline__ void set(int v, int x) const {
    const uint32_t u = uint32_t(v);
    uint32_t& w = st[(u / PER) * LANE_T];
    const uint32_t sh = (u % PER) * BITS;
    w = (w & ~(MASK << sh)) | (uint32_t(x) << sh);
  }
  __device__ __forceinline__ bool latent(int v) const {
    const uint32_t u = uint32_t(v);
    return (fl[(u >> 5) * LANE_T] >> (u & 31)) & 1u;
  }
};

template <int BITS>
__host__ __device__ inline size_t lane_smem(int n) {
  return size_t((n + 32 / BITS - 1) / (32 / BITS) + (n + 31) / 32) * LANE_T * 4;
}

template <int MODE, int BITS>
__global__ void __launch_bounds__(LANE_T) k_sweep_lane(const sg_net net, const sg_batch bt, const SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_err;
  const int n = net.n;
  const int tid = threadIdx.x;
  constexpr int PER = 32 / BITS;
  const int sw = (n + PER - 1) / PER;
  LaneColumn<BITS> col{reinterpret_cast<uint32_t*>(smem) + tid, reinterpret_cast<uint32_t*>(smem) + sw * LANE_T + tid};
  // A warp holds G = min(m, 32) replicas of 32 / G consecutive cases (lane =
  // case-in-warp * G + replica), so the replicas of a case -- which share the
  // latent pattern -- sit together and a warp skips every variable none of
  // its cases has latent.  Grid y = replica groups of G.
  const int G = min(bt.m, 32), cpw = 32 / G;
  const int lane = tid & 31, warp = tid >> 5;
  const int c = (blockIdx.x * (LANE_T / 32) + warp) * cpw + lane / G;
  const int r = blockIdx.y * G + lane % G;
  const bool active = lane < cpw * G && c < bt.cases && r < bt.m;
  const int64_t vstride = int64_t(bt.m) * bt.pitch;
  int8_t* base = bt.states + int64_t(active ? r : 0) * bt.pitch + (active ? c : 0);  // cell (v, r, c) at base[v * vstride]
  if (tid == 0) s_err = 0;
  // ---- stage this lane's column: states packed, latent flags as bits
  if (active) {
    for (int w0 = 0; w0 < n; w0 += 32) {
      // 32 variables per step: their latent bits make one flag word and their
      // states BITS packed words (16 or 8 states each)
      uint32_t flags = 0, acc[BITS] = {};
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int v = w0 + k;
        if (v < n) {
          const uint32_t b = uint8_t(base[v * vstride]);
          flags |= (b >> 7) << k;
          acc[k / PER] |= (b & 0x7Fu) << ((k % PER) * BITS);
        }
      }
#pragma unroll
      for (int q = 0; q < BITS; ++q)
        if (w0 + q * PER < n) col.st[(w0 / PER + q) * LANE_T] = acc[q];
      col.fl[(w0 >> 5) * LANE_T] = flags;
    }
  }
  const uint64_t key = a.fast_key_dev ? __ldg(a.fast_key_dev) : a.fast_key;
  const bool zs_armed = a.ftab && net.table_entries > 0 && __ldg(a.ftab + net.ftab_size) != 0u;
  const uint64_t gcase = uint64_t(bt.case_base + c);
  bool zs = false;
  // ---- every variable in colour order
  for (int i = 0; i < n; ++i) {
    const int v = __ldg(net.order + i);
    const bool lat = active && col.latent(v);
    if (!__any_sync(0xffffffffu, lat)) continue;
    if (!lat) continue;
    double u;
    uint32_t u31 = 0;
    if (MODE == SG_RNG_FAST) {
      const uint32_t w = pick(fast_block(key, gcase, uint32_t(v), uint32_t(r >> 2), 0u), r & 3);
      u31 = w >> 1;
      u = double(w) * 0x1.0p-32;
    } else {
      const int64_t idx = int64_t(r) * __ldg(bt.nmiss + v) + __ldg(bt.rank + int64_t(v) * bt.ld_rank + c);
      u = MODE == SG_RNG_NUMPY ? np_uniform(uint64_t(idx), __ldg(a.keys + 2 * v), __ldg(a.keys + 2 * v + 1))
                               : __ldg(a.uniforms + __ldg(a.inj_off + v) + idx);
    }
    const int32_t* dv = net.var_desc + v * SG_DESC_WORDS;
    const int card = dv[0], nmb = dv[1];
    int x = 0;
    if (nmb >= 0) {  // conditional table indexed by the blanket configuration
      int e = 0;
      for (int k = 0; k < nmb; ++k) e += col.get(dv[4 + k]) * dv[4 + SG_DESC_MB + k];
      if (MODE == SG_RNG_FAST) {
        const uint32_t* th = a.ftab + dv[2] + e * (card - 1);
        const uint32_t t0 = __ldg(th);
        if (zs_armed && t0 == 0xFFFFFFFFu) zs = true;
        x = u31 >= t0;
        for (int q = 1; q < card - 1; ++q) x += u31 >= __ldg(th + q);
      } else {
        const double* p = a.ptab + dv[3] + int64_t(e) * card;
        const double norm = __ldg(p + card - 1);
        if (!(norm > 0.0)) zs = true;
        const double au = __dmul_rn(u, norm);
        for (int q = 0; q < card - 1; ++q) x += au > __ldg(p + q);
      }
    } else {
      const int32_t* fd = net.fac_desc + __ldg(net.fac_start + v);
      x = draw_factored<SG_LANE_UNIFIED>(fd, a.cpt, [&](int var) { return col.get(var); }, u, zs);
    }
    col.set(v, x);
  }
  if (zs) atomicOr(&s_err, int(SG_ERR_ZERO_SUPPORT));
  // ---- write back the latent cells (observed cells never change)
  if (active) {
    for (int v = 0; v < n; ++v)
      if (col.latent(v)) base[v * vstride] = int8_t(0x80 | col.get(v));
  }
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(a.err, s_err);
}

template <int MODE, int BITS>
static void launch_lane(const sg_net& net, const sg_batch& bt, const SweepArgs& a, cudaStream_t s) {
  const size_t smem = lane_smem<BITS>(net.n);
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_sweep_lane<MODE, BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int g = std::min(bt.m, 32), cases_per_cta = (LANE_T / 32) * (32 / g);
  const dim3 grid((bt.cases + cases_per_cta - 1) / cases_per_cta, (bt.m + g - 1) / g);
  k_sweep_lane<MODE, BITS><<<grid, LANE_T, smem, s>>>(net, bt, a);
}

// Whether a sweep takes the lane kernel: many variables, small cards, a
// packed column that leaves room for several CTAs per SM, and SAME replicas
// to fill the warps (with m = 1 a warp holds 32 cases and draws only where a
// case is latent; the tile kernel's compaction measured faster there).
static int lane_bits(const sg_net& net, int m) {
  if (net.n <= 32 || net.max_card > 16 || m < 2) return 0;
  const int bits = net.max_card <= 4 ? 2 : 4;
  const size_t smem = bits == 2 ? lane_smem<2>(net.n) : lane_smem<4>(net.n);
  return smem <= 100 * 1024 ? bits : 0;
}

// Chunked tally of a resident batch (large models).  blockIdx.y = a run of
// consecutive variables whose cells fit a shared-memory histogram
// (sg_net.tally_chunk), blockIdx.x = a slice of the cases.  For each variable
// of its run a thread takes 4 consecutive cases of a replica row -- one
// 32-bit load of the variable's row and of each parent's row -- and adds the
// 4 cells to the histogram; the CTA then flushes every non-zero cell with one
// global atomic.  A run holding a single oversized variable counts straight
// into global memory.
//
// V16 (states 16-byte aligned, run histogram local): a thread takes 16
// consecutive cases -- one 16-byte load per row -- and evaluates the cell
// indices two cases per 32-bit word: bytes 0/2 and 1/3 of a state word are
// spread into the 16-bit halves of two words and multiplied by the parent's
// cell stride (stride x card), so each parent costs 5 integer ops per 4 cases
// instead of 4 byte extractions and 4 multiply-adds.  No half can carry into
// its neighbour: every partial sum is <= the variable's last cell index
// < SG_TALLY_CHUNK_CELLS < 2^16.  The ragged last unit of a slice (cases past
// num_real hold padding) takes the per-case path.
__device__ __forceinline__ void tally_add4(uint32_t* hist, int base, uint32_t lo, uint32_t hi) {
  atomicAdd(hist + base + int(lo & 0xFFFFu), 1u);
  atomicAdd(hist + base + int(hi & 0xFFFFu), 1u);
  atomicAdd(hist + base + int(lo >> 16), 1u);
  atomicAdd(hist + base + int(hi >> 16), 1u);
}

__device__ __forceinline__ void tally_spread(uint32_t x, uint32_t& lo, uint32_t& hi) {
  lo = x & 0x007F007Fu;
  hi = (x >> 8) & 0x007F007Fu;
}

__device__ __forceinline__ void tally_run_v16(const sg_net& net, const sg_batch& bt, uint32_t* hist, int v0,
                                              int v1, int64_t cell0) {
  // work items = (replica row, 16-case unit), replica-major so consecutive
  // threads read consecutive 16-byte columns of one row
  const int units = (bt.num_real + 15) >> 4;
  const int full = bt.num_real >> 4;  // units whose 16 cases are all real
  const int items = units * bt.m;
  const int per = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per, i1 = min(items, i0 + per);
  const int64_t vstride = int64_t(bt.m) * bt.pitch;
  for (int v = v0; v < v1; ++v) {
    const int card = __ldg(net.card + v);
    const int ps = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1);
    const int base = int(__ldg(net.cpt_off + v) - cell0);
    const int np4 = min(4, pe - ps);
    int64_t poff[4] = {0, 0, 0, 0};
    uint32_t pst[4] = {0, 0, 0, 0};  // parent cell strides: row stride x card
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < np4) {
        poff[k] = int64_t(__ldg(net.par_var + ps + k)) * vstride;
        pst[k] = uint32_t(__ldg(net.par_stride + ps + k) * card);
      }
    const int64_t voff = int64_t(v) * vstride;
    // two items per thread per iteration: both items' row loads are in flight
    // before either item's cell arithmetic and histogram atomics
    for (int i = i0 + threadIdx.x; i < i1; i += 2 * SG_THREADS) {
      const int8_t* col[2];
      bool vec[2], rag[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ih = i + h * SG_THREADS;
        const int r = ih / units, u = ih - r * units;
        col[h] = bt.states + int64_t(r) * bt.pitch + u * 16;
        vec[h] = ih < i1 && u < full;
        rag[h] = ih < i1 && u >= full;
      }
      uint4 xv[2], xp[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (vec[h]) xv[h] = __ldg(reinterpret_cast<const uint4*>(col[h] + voff));
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (k < np4 && vec[h]) xp[h][k] = __ldg(reinterpret_cast<const uint4*>(col[h] + poff[k]));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (vec[h]) {
          uint32_t lo[4], hi[4];
          tally_spread(xv[h].x, lo[0], hi[0]);
          tally_spread(xv[h].y, lo[1], hi[1]);
          tally_spread(xv[h].z, lo[2], hi[2]);
          tally_spread(xv[h].w, lo[3], hi[3]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < np4) {
              uint32_t a, b;
              tally_spread(xp[h][k].x, a, b); lo[0] += a * pst[k]; hi[0] += b * pst[k];
              tally_spread(xp[h][k].y, a, b); lo[1] += a * pst[k]; hi[1] += b * pst[k];
              tally_spread(xp[h][k].z, a, b); lo[2] += a * pst[k]; hi[2] += b * pst[k];
              tally_spread(xp[h][k].w, a, b); lo[3] += a * pst[k]; hi[3] += b * pst[k];
            }
          for (int p = ps + 4; p < pe; ++p) {  // parents beyond the fourth
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(col[h] + int64_t(__ldg(net.par_var + p)) * vstride));
            const uint32_t st = uint32_t(__ldg(net.par_stride + p) * card);
            uint32_t a, b;
            tally_spread(x.x, a, b); lo[0] += a * st; hi[0] += b * st;
            tally_spread(x.y, a, b); lo[1] += a * st; hi[1] += b * st;
            tally_spread(x.z, a, b); lo[2] += a * st; hi[2] += b * st;
            tally_spread(x.w, a, b); lo[3] += a * st; hi[3] += b * st;
          }
#pragma unroll
          for (int w = 0; w < 4; ++w) tally_add4(hist, base, lo[w], hi[w]);
        } else if (rag[h]) {
          const int c = int(col[h] - bt.states) % bt.pitch;  // ragged last unit: per case
          for (int j = 0; c + j < bt.num_real; ++j) {
            int cell = col[h][voff + j] & 0x7F;
            for (int p = ps; p < pe; ++p)
              cell += (col[h][int64_t(__ldg(net.par_var + p)) * vstride + j] & 0x7F) * __ldg(net.par_stride + p) * card;
            atomicAdd(hist + base + cell, 1u);
          }
        }
      }
    }
  }
}

template <bool V16>
__global__ void __launch_bounds__(SG_THREADS, 4)
k_tally_chunked(const sg_net net, const sg_batch bt, unsigned long long* __restrict__ counts) {
  extern __shared__ uint32_t hist[];
  const int c0v = __ldg(net.tally_chunk + blockIdx.y), c1v = __ldg(net.tally_chunk + blockIdx.y + 1);
  const int64_t cell0 = __ldg(net.cpt_off + c0v);
  const int64_t cell1 = c1v < net.n ? __ldg(net.cpt_off + c1v) : net.cells;
  // grid z splits the run's variables (a few hundred in a run of small tables:
  // one CTA per case slice alone leaves most SMs idle)
  const int v0 = c0v + int(int64_t(c1v - c0v) * blockIdx.z / gridDim.z);
  const int v1 = c0v + int(int64_t(c1v - c0v) * (blockIdx.z + 1) / gridDim.z);
  const bool local = cell1 - cell0 <= SG_TALLY_CHUNK_CELLS;
  const int ncell = int(cell1 - cell0);
  if (local)
    for (int i = threadIdx.x; i < ncell; i += SG_THREADS) hist[i] = 0;
  __syncthreads();
  if (V16 && local) {
    tally_run_v16(net, bt, hist, v0, v1, cell0);
    __syncthreads();
    for (int i = threadIdx.x; i < ncell; i += SG_THREADS)
      if (hist[i]) atomicAdd(counts + cell0 + i, (unsigned long long)hist[i]);
    return;
  }
  const int quads = (bt.num_real + 3) >> 2;
  const int per = (quads + gridDim.x - 1) / gridDim.x;
  const int q0 = blockIdx.x * per, q1 = min(quads, q0 + per);
  const int64_t vstride = int64_t(bt.m) * bt.pitch;
  for (int v = v0; v < v1; ++v) {
    const int card = __ldg(net.card + v);
    const int ps = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1);
    const int64_t base = __ldg(net.cpt_off + v) - cell0;
    // up to 4 parents in registers, so a quad's row loads are issued together
    const int np4 = min(4, pe - ps);
    int64_t poff[4] = {0, 0, 0, 0};
    int pst[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < np4) {
        poff[k] = int64_t(__ldg(net.par_var + ps + k)) * vstride;
        pst[k] = __ldg(net.par_stride + ps + k);
      }
    const int64_t voff = int64_t(v) * vstride;
    for (int q = q0 + threadIdx.x; q < q1; q += SG_THREADS) {
      const int c = q * 4;
      const int nl = min(4, bt.num_real - c);
      for (int r = 0; r < bt.m; ++r) {
        const int8_t* col = bt.states + int64_t(r) * bt.pitch + c;
        const uint32_t xv = __ldg(reinterpret_cast<const uint32_t*>(col + voff)) & 0x7F7F7F7Fu;
        uint32_t xp[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          xp[k] = k < np4 ? __ldg(reinterpret_cast<const uint32_t*>(col + poff[k])) & 0x7F7F7F7Fu : 0u;
        int cfg[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 4; ++j) cfg[j] += int((xp[k] >> (8 * j)) & 0xFF) * pst[k];
        for (int p = ps + 4; p < pe; ++p) {  // parents beyond the fourth
          const uint32_t x =
              __ldg(reinterpret_cast<const uint32_t*>(col + __ldg(net.par_var + p) * vstride)) & 0x7F7F7F7Fu;
          const int st = __ldg(net.par_stride + p);
#pragma unroll
          for (int j = 0; j < 4; ++j) cfg[j] += int((x >> (8 * j)) & 0xFF) * st;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nl) {
            const int64_t cell = base + int64_t(cfg[j]) * card + int((xv >> (8 * j)) & 0xFF);
            if (local) atomicAdd(hist + cell, 1u);
            else atomicAdd(counts + cell0 + cell, 1ull);
          }
        }
      }
    }
  }
  if (!local) return;
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += SG_THREADS)
    if (hist[i]) atomicAdd(counts + cell0 + i, (unsigned long long)hist[i]);
}

static int tally_chunked(const sg_net& net, const sg_batch& bt, uint64_t* counts, cudaStream_t s) {
  const int quads = (bt.num_real + 3) / 4;
  if (quads == 0 || net.tally_chunks == 0) return SG_OK;
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, SG_TALLY_CHUNK_CELLS * 4)) {
    cudaFuncSetAttribute(k_tally_chunked<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SG_TALLY_CHUNK_CELLS * 4);
    cudaFuncSetAttribute(k_tally_chunked<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SG_TALLY_CHUNK_CELLS * 4);
  }
  // 16-case units when every row is 16-byte aligned (pitch % 16 == 0 is part
  // of the sg_batch contract), else 4-case quads
  const bool v16 = (reinterpret_cast<uintptr_t>(bt.states) & 15) == 0 && bt.pitch % 16 == 0;
  const int work = v16 ? (bt.num_real + 15) / 16 * bt.m : quads;
  // ~4 CTAs per SM over all runs, each slice at least one work item per thread
  const int64_t want = std::max<int64_t>(1, (148 * 4 + net.tally_chunks - 1) / net.tally_chunks);
  const int slices = std::max(1, int(std::min<int64_t>(want, (work + SG_THREADS - 1) / SG_THREADS)));
  // and the variables of each run over grid z, to ~8 CTAs per SM in all
  const int64_t ctas = int64_t(slices) * net.tally_chunks;
  const int vsplit = int(std::max<int64_t>(1, std::min<int64_t>((148 * 8 + ctas - 1) / ctas,
                                                               std::max<int64_t>(1, int64_t(net.n) / net.tally_chunks))));
  const dim3 grid(slices, unsigned(net.tally_chunks), unsigned(vsplit));
  auto cp = reinterpret_cast<unsigned long long*>(counts);
  if (v16)
    k_tally_chunked<true><<<grid, SG_THREADS, SG_TALLY_CHUNK_CELLS * 4, s>>>(net, bt, cp);
  else
    k_tally_chunked<false><<<grid, SG_THREADS, SG_TALLY_CHUNK_CELLS * 4, s>>>(net, bt, cp);
  return SG_OK;
}

static int choose_tile(const sg_net& net, int m, int cases, const SweepArgs& a, bool small, int* tc_out,
                       int* mg_out, size_t* smem_out) {
  // Largest power-of-two case tile (<= 512) holding all m replicas whose
  // shared memory leaves room for four CTAs per SM (latency hiding), else
  // two, else one of up to 200 KB.  When even 32 cases x m replicas do not
  // fit (large n x m), the replicas split into groups (grid y): lanes never
  // interact, so any tiling of (cases x replicas) is exact.
#ifndef SG_TILE_BUDGET0
#define SG_TILE_BUDGET0 (56 * 1024)
#endif
  int best = 0, mg = m;
  for (int budget : {SG_TILE_BUDGET0, 100 * 1024, 200 * 1024}) {
    for (int tc = 512; tc >= 32 && !best; tc >>= 1)
      if (smem_layout(net, m, tc, a.tally_mode, small, a.tab_bytes).total <= size_t(budget)) best = tc;
    if (best) break;
  }
  if (!best) {
    // replica groups of 4 (one Philox quad), 2, 1 at the smallest tile
    for (int g : {16, 12, 8, 4, 2, 1}) {
      if (g >= m) continue;
      if (smem_layout(net, g, 32, a.tally_mode, small, a.tab_bytes).total <= size_t(200 * 1024)) {
        best = 32;
        mg = g;
        break;
      }
    }
  }
  if (!best) return SG_ECAPACITY;
  // do not make tiles much larger than the minibatch
  while (best > 32 && best / 2 >= cases) best >>= 1;
  *tc_out = best;
  *mg_out = mg;
  *smem_out = smem_layout(net, mg, best, a.tally_mode, small, a.tab_bytes).total;
  return SG_OK;
}

template <int MODE, bool SMALL>
static void launch_sweep(const sg_net& net, const sg_batch& bt, const SweepArgs& a, dim3 blocks, size_t smem,
                         cudaStream_t s) {
  static size_t configured[SG_MAX_DEVICES] = {};  // once per instantiation and device (graph-capture friendly)
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_sweep<MODE, SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_sweep<MODE, SMALL><<<blocks, SG_THREADS, smem, s>>>(net, bt, a);
}

}  // namespace sg

extern "C" int sg_sweep(const sg_net* net, const sg_batch* batch, const double* cpt,
                        const double* ptab, const uint32_t* ftab, int32_t rng_mode,
                        uint64_t fast_key, const uint64_t* fast_key_dev, const uint64_t* keys,
                        const double* uniforms, const int64_t* inj_off, uint64_t* counts, int32_t* err,
                        void* stream) {
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
  SG_REQUIRE(net->var_desc, "sg_sweep: network pack has no variable descriptors");
  if (net->direct_vars > 0) SG_REQUIRE(net->fac_start && net->fac_desc, "sg_sweep: no factored descriptors");
  SG_REQUIRE(rng_mode >= SG_RNG_FAST && rng_mode <= SG_RNG_INJECTED, "sg_sweep: bad rng mode %d",
             rng_mode);
  if (rng_mode != SG_RNG_FAST)
    SG_REQUIRE(batch->rank && batch->nmiss, "sg_sweep: rank/nmiss required for this rng mode");
  else
    SG_REQUIRE(fast_cases_ok(batch->case_base, batch->cases) && batch->m <= 4 * 4096,
               "sg_sweep: FAST counters need global cases < 2^32 and m <= 16384");
  if (rng_mode == SG_RNG_NUMPY) SG_REQUIRE(keys, "sg_sweep: numpy keys required");
  if (rng_mode == SG_RNG_INJECTED) SG_REQUIRE(uniforms && inj_off, "sg_sweep: uniforms required");
  if (net->table_entries > 0) SG_REQUIRE(ptab && ftab, "sg_sweep: tables required");
  if (net->direct_vars > 0) SG_REQUIRE(cpt, "sg_sweep: cpt required for direct variables");
  if (batch->cases == 0) return SG_OK;

  SweepArgs a;
  a.cpt = cpt;
  a.ptab = ptab;
  a.ftab = net->table_entries > 0 ? ftab : nullptr;
  a.fast_key = fast_key;
  a.fast_key_dev = fast_key_dev;
  a.keys = keys;
  a.uniforms = uniforms;
  a.inj_off = inj_off;
  a.counts = counts;
  a.err = err;
  a.tc = 0;
  a.mg = 0;
  const int64_t tab_bytes = net->table_entries > 0
                                ? (rng_mode == SG_RNG_FAST ? net->ftab_size * 4 : net->ptab_size * 8)
                                : 0;
  const bool small = net->n <= 512 && tab_bytes <= 48 * 1024;
  a.tab_bytes = small ? tab_bytes : 0;
  // tally strategy; byte counters hold at most 255 lanes per thread
  const int max_lanes_per_thread = (batch->m * 512 + SG_THREADS - 1) / SG_THREADS;
  const bool bytes_ok = max_lanes_per_thread <= 255;
  if (!counts) a.tally_mode = TALLY_NONE;
  else if (bytes_ok && net->joint_size > 0 && net->joint_size <= SG_JOINT_MAX && net->n <= 7 &&
           net->joint_radix && net->joint_cell)
    a.tally_mode = TALLY_JOINT;
  else if (bytes_ok && net->cells <= 128) a.tally_mode = TALLY_CELL8;
  else a.tally_mode = TALLY_NONE;  // large models: the chunked tally kernel after the sweep
  const bool chunked = counts && a.tally_mode == TALLY_NONE;
  if (chunked) {
    SG_REQUIRE(net->tally_chunk && net->tally_chunks > 0, "sg_sweep: network pack has no tally runs");
    a.counts = nullptr;  // the sweep itself counts nothing
  }
  cudaStream_t s = (cudaStream_t)stream;
  // Large networks: the lane-per-thread sweep when the latent cells are dense
  // and SAME replicas fill its warps (measured: C3-shaped 2.8 ms vs 6.1 ms),
  // else the big-tile sweep (C4-shaped 17 ms vs 41 ms, C5-shaped 69 vs 115 ms).
  const bool dense_latent = batch->latent_permille >= 800 && batch->m >= 2;
  if (!dense_latent) {
    SweepArgs b = a;
    b.tally_mode = TALLY_NONE;
    b.counts = nullptr;
    if (sweep_big(*net, *batch, b, rng_mode, s)) {
      if (counts) {
        SG_REQUIRE(net->tally_chunk && net->tally_chunks > 0, "sg_sweep: network pack has no tally runs");
        tally_chunked(*net, *batch, counts, s);
      }
      return check_launch("sg_sweep");
    }
  }
  if (const int bits = lane_bits(*net, batch->m)) {
    // large network: lane-per-thread sweep, then the chunked tally
    a.tally_mode = TALLY_NONE;
    a.counts = nullptr;
    switch (rng_mode * 2 + (bits == 2 ? 0 : 1)) {
      case 0: launch_lane<SG_RNG_FAST, 2>(*net, *batch, a, s); break;
      case 1: launch_lane<SG_RNG_FAST, 4>(*net, *batch, a, s); break;
      case 2: launch_lane<SG_RNG_NUMPY, 2>(*net, *batch, a, s); break;
      case 3: launch_lane<SG_RNG_NUMPY, 4>(*net, *batch, a, s); break;
      case 4: launch_lane<SG_RNG_INJECTED, 2>(*net, *batch, a, s); break;
      default: launch_lane<SG_RNG_INJECTED, 4>(*net, *batch, a, s); break;
    }
    if (counts) {
      SG_REQUIRE(net->tally_chunk && net->tally_chunks > 0, "sg_sweep: network pack has no tally runs");
      tally_chunked(*net, *batch, counts, s);
    }
    return check_launch("sg_sweep");
  }
  size_t smem = 0;
  int st = choose_tile(*net, batch->m, batch->cases, a, small, &a.tc, &a.mg, &smem);
  if (st != SG_OK) {
    set_error("sg_sweep: tile of n=%d x m=%d does not fit in shared memory", net->n, batch->m);
    return st;
  }
  const dim3 blocks((batch->cases + a.tc - 1) / a.tc, (batch->m + a.mg - 1) / a.mg);
  switch (rng_mode * 2 + (small ? 1 : 0)) {
    case 0: launch_sweep<SG_RNG_FAST, false>(*net, *batch, a, blocks, smem, s); break;
    case 1: launch_sweep<SG_RNG_FAST, true>(*net, *batch, a, blocks, smem, s); break;
    case 2: launch_sweep<SG_RNG_NUMPY, false>(*net, *batch, a, blocks, smem, s); break;
    case 3: launch_sweep<SG_RNG_NUMPY, true>(*net, *batch, a, blocks, smem, s); break;
    case 4: launch_sweep<SG_RNG_INJECTED, false>(*net, *batch, a, blocks, smem, s); break;
    default: launch_sweep<SG_RNG_INJECTED, true>(*net, *batch, a, blocks, smem, s); break;
  }
  if (chunked) tally_chunked(*net, *batch, counts, s);
  return check_launch("sg_sweep");
}

extern "C" int sg_tally(const sg_net* net, const sg_batch* batch, uint64_t* counts, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && batch && counts && batch->states, "sg_tally: null argument");
  const int64_t lanes = int64_t(batch->m) * batch->num_real;
  if (lanes == 0) return SG_OK;
  SG_REQUIRE(batch->pitch % 16 == 0, "sg_tally: row pitch must be a multiple of 16");
  SG_REQUIRE(net->tally_chunk && net->tally_chunks > 0, "sg_tally: network pack has no tally runs");
  tally_chunked(*net, *batch, counts, (cudaStream_t)stream);
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

SG_CHECKED_EXPORT(sweep)
