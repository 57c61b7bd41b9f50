// Big-tile sweep for large networks (generic FAST / NUMPY / INJECTED modes).
//
// Reference: gibbs_pass sampler.py:251-284 resamples one colour group at a
// time, each variable over all of its latent lanes (_resample_variable
// sampler.py:217-248).  That variable-major order is what keeps a GPU warp
// uniform: here a warp owns one variable of the current colour group at a
// time and draws that variable's latent lanes 32 at a time, so its
// descriptors are broadcast loads and its draw kind (table / factored
// product) and loop trip counts never diverge.
//
// For a warp to find 32 latent lanes of one variable the tile must be wide:
// with n ~ 1000 variables an int8 tile of 512 cases would need 512 KB, so the
// tile keeps the lane states bit-packed (BITS = 2 for cards <= 4, 4 for
// <= 16) and the shared latent mask as one bit per (variable, case):
// C4 (n = 1000, m = 1): ~450 cases in ~170 KB.  One CTA of 32 warps per SM;
// members of a colour group are handed to warps dynamically (their costs
// differ) and the group ends with one CTA barrier.  Writes go to packed
// words shared by 16 (8) cases of one variable row, i.e. by lanes of the
// same warp, so they use shared-memory atomics (and/or).  Draws are the same
// arithmetic as the tile kernel (sg_sweep.cu): bit-exact in NUMPY/INJECTED
// mode, the same FAST counters.  The tally runs afterwards (k_tally_chunked).
#include "sg_sweep.cuh"

namespace sg {

#ifndef SG_BIG_T
#define SG_BIG_T 1024      // threads per CTA
#endif
#ifndef SG_BIG_MINB
#define SG_BIG_MINB 1      // CTAs per SM (register budget)
#endif
#ifndef SG_BIG_SMEM
#define SG_BIG_SMEM (200 * 1024)  // tile budget (shared memory per CTA)
#endif
constexpr int BIG_T = SG_BIG_T;
constexpr int BIG_W = BIG_T / 32;

// states [n][mg][tc / PER] + latent bits [n][tc / 32] + per-warp case lists [BIG_W][tc] (uint16)
template <int BITS>
__host__ __device__ inline size_t big_smem(int n, int mg, int tc) {
  return size_t(n) * mg * (tc / (32 / BITS)) * 4 + size_t(n) * (tc / 32) * 4 + size_t(BIG_W) * tc * 2;
}

// Packed 16-case chunk of an int8 row (flags stripped) -> BITS-bit fields.
template <int BITS>
__device__ __forceinline__ void pack16(const int4 val, uint32_t* out) {
  const uint32_t b[4] = {uint32_t(val.x), uint32_t(val.y), uint32_t(val.z), uint32_t(val.w)};
  if (BITS == 2) {
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) w |= ((b[k >> 2] >> (8 * (k & 3))) & 3u) << (2 * k);
    out[0] = w;
  } else {
    uint32_t w0 = 0, w1 = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) w0 |= ((b[k >> 2] >> (8 * (k & 3))) & 15u) << (4 * k);
#pragma unroll
    for (int k = 8; k < 16; ++k) w1 |= ((b[k >> 2] >> (8 * (k & 3))) & 15u) << (4 * (k - 8));
    out[0] = w0;
    out[1] = w1;
  }
}

__device__ __forceinline__ uint32_t flag_bits16(const int4 val) {
  const uint32_t b[4] = {uint32_t(val.x), uint32_t(val.y), uint32_t(val.z), uint32_t(val.w)};
  uint32_t f = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) f |= ((b[k >> 2] >> (8 * (k & 3) + 7)) & 1u) << k;
  return f;
}

// ---- blanket factor tables (sg_net.bft, cards <= 4)
// Row r = the CPT cells src[2r] + t * step, t < k (zero padded to 4): one
// factor of the weight product as v runs over its states.  Rebuilt from the
// CPTs before every big-tile sweep (3.5 MB on C4: a few microseconds).
__global__ void __launch_bounds__(256) k_build_bft(const sg_net net, const double* __restrict__ cpt) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < net.bft_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int2 s = __ldg(reinterpret_cast<const int2*>(net.bft_src) + r);
    const int step = s.y & ((1 << 26) - 1), k = s.y >> 26;
    double f[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) f[t] = t < k ? __ldg(cpt + s.x + int64_t(t) * step) : 0.0;
    double2* o = reinterpret_cast<double2*>(net.bft) + 2 * r;
    o[0] = make_double2(f[0], f[1]);
    o[1] = make_double2(f[2], f[3]);
  }
}

// K = 4: the whole 32-byte row; K = 2 / 3 (variables of 2 / 3 states): its
// first 16 / 24 bytes only -- the rest is the row's zero padding.
template <int K = 4>
__device__ __forceinline__ void bft_row(const double* __restrict__ bft, int row, double (&f)[K]) {
  const double2* p = reinterpret_cast<const double2*>(bft) + 2 * row;
  const double2 a = __ldg(p);
  f[0] = a.x;
  f[1] = a.y;
  if constexpr (K == 3) {
    f[2] = __ldg(reinterpret_cast<const double*>(p + 1));
  } else if constexpr (K == 4) {
    const double2 b = __ldg(p + 1);
    f[2] = b.x;
    f[3] = b.y;
  }
}

// K = 2: the padded entries are exact zeros, so norm = w0 + w1 exactly and
// the comparisons at w0 + w1 (+ 0) can never hold (u * norm <= norm): the one
// comparison at w0 is the whole draw, bit-identical to K = 4.
template <int K = 4>
__device__ __forceinline__ int bft_finish(const double (&w)[K], double u, bool& zs) {
  if constexpr (K == 2) {
    const double norm = __dadd_rn(w[0], w[1]);
    if (!(norm > 0.0)) zs = true;
    return __dmul_rn(u, norm) > w[0];
  } else if constexpr (K == 3) {  // likewise: norm = (w0 + w1) + w2 exactly, no comparison at it
    const double norm = __dadd_rn(__dadd_rn(w[0], w[1]), w[2]);
    if (!(norm > 0.0)) zs = true;
    const double au = __dmul_rn(u, norm);
    return int(au > w[0]) + int(au > __dadd_rn(w[0], w[1]));
  } else {
    const double norm = __dadd_rn(__dadd_rn(__dadd_rn(w[0], w[1]), w[2]), w[3]);
    if (!(norm > 0.0)) zs = true;
    const double au = __dmul_rn(u, norm);
    double cum = w[0];
    int x = au > cum;
    cum = __dadd_rn(cum, w[1]);
    x += au > cum;
    cum = __dadd_rn(cum, w[2]);
    x += au > cum;
    return x;
  }
}
// Row index of one child factor: base + x_c + sum x_u * stride over the
// child's other parents (records of two; an unused half has stride 0).
template <class Get>
__device__ __forceinline__ int bft_child(const int4*& p, Get get) {
  const int4 c = __ldg(p++);
  int i = c.y + get(c.x);
#pragma unroll 1
  for (int q = 0; q < c.z; ++q, ++p) {
    const int4 r = __ldg(p);
    i += get(r.x) * r.y;
    if (r.w) i += get(r.z) * r.w;
  }
  return i;
}

// The factored draw (draw_factored: sampler.py:226-247) over the blanket
// factor tables: one 32-byte row per factor, products in the reference's
// order (own row, then children in order), numpy's sequential sum, the
// cumulative comparisons.  Zero padding leaves every result bit-identical to
// draw_factored for cards 2..4: padded weights add exact zeros and their
// comparisons are never true (u * norm <= norm).
template <int K, class Get>
__device__ __forceinline__ int draw_bft(const int4* __restrict__ prog, const double* __restrict__ bft, Get get,
                                        double u, bool& zs, int64_t nrows) {
  const int4 h = __ldg(prog);  // card, npar, nchl, own row base
  const int4* p = prog + 1;
  int row = h.w;
#pragma unroll 1
  for (int j = 0; j < h.y; j += 2, ++p) {
    const int4 r = __ldg(p);
    row += get(r.x) * r.y;
    if (r.w) row += get(r.z) * r.w;
  }
  double w[K];
  SG_DCHECK(row >= 0 && row < nrows);
  bft_row<K>(bft, row, w);
  int k = 0;
#pragma unroll 1
  for (; k + 1 < h.z; k += 2) {  // two children per step: both gathers in flight
    const int i0 = bft_child(p, get);
    const int i1 = bft_child(p, get);
    double f0[K], f1[K];
    SG_DCHECK(i0 >= 0 && i1 >= 0 && i0 < nrows && i1 < nrows);
    bft_row<K>(bft, i0, f0);
    bft_row<K>(bft, i1, f1);
#pragma unroll
    for (int t = 0; t < K; ++t) w[t] = __dmul_rn(__dmul_rn(w[t], f0[t]), f1[t]);
  }
  if (k < h.z) {
    const int i0 = bft_child(p, get);
    double f0[K];
    SG_DCHECK(i0 >= 0 && i0 < nrows);
    bft_row<K>(bft, i0, f0);
#pragma unroll
    for (int t = 0; t < K; ++t) w[t] = __dmul_rn(w[t], f0[t]);
  }
  return bft_finish<K>(w, u, zs);
}

// 2-bit tiles: whole-word bit tricks instead of per-case shifts.  A product
// (x & 0x03030303) * 0x01041040 carries no bits (its partial products occupy
// distinct positions) and leaves the four 2-bit fields of x in byte 3;
// (x & 0x80808080) * 0x00204081 leaves the four flag bits in bits 28..31.
__device__ __forceinline__ uint32_t crumb_word(const int4 val) {
  const uint32_t p0 = (uint32_t(val.x) & 0x03030303u) * 0x01041040u;
  const uint32_t p1 = (uint32_t(val.y) & 0x03030303u) * 0x01041040u;
  const uint32_t p2 = (uint32_t(val.z) & 0x03030303u) * 0x01041040u;
  const uint32_t p3 = (uint32_t(val.w) & 0x03030303u) * 0x01041040u;
  return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}
__device__ __forceinline__ uint32_t flag_word16(const int4 val) {
  const uint32_t g0 = (uint32_t(val.x) & 0x80808080u) * 0x00204081u;
  const uint32_t g1 = (uint32_t(val.y) & 0x80808080u) * 0x00204081u;
  const uint32_t g2 = (uint32_t(val.z) & 0x80808080u) * 0x00204081u;
  const uint32_t g3 = (uint32_t(val.w) & 0x80808080u) * 0x00204081u;
  return (g0 >> 28) | ((g1 >> 24) & 0xF0u) | ((g2 >> 20) & 0xF00u) | ((g3 >> 16) & 0xF000u);
}
// Inverse: 4 cases (byte k of the crumb word, flag nibble k) -> 4 int8 states
// (fields spread to bytes with two shifted ORs; flags by a carry-free product).
__device__ __forceinline__ uint32_t state_bytes4(uint32_t crumbs, uint32_t flags, int k) {
  uint32_t x = __byte_perm(crumbs, 0u, 0x4440u | uint32_t(k));
  x |= x << 6;
  x = (x | (x << 12)) & 0x03030303u;
  return x | ((((flags >> (4 * k)) & 0xFu) * 0x10204080u) & 0x80808080u);
}

// Two latent cases of the same variable drawn in lockstep (2-bit tiles): one
// pass over v's program serves both, and both cases' factor rows are in flight
// together.  Tile word offsets ra / rb and field shifts sa / sb locate the
// cases; per case the arithmetic is draw_bft's.
__device__ __forceinline__ int2 get2(const uint32_t* st, int o, int ra, int rb, int sa, int sb, int lim) {
  SG_DCHECK(o >= 0 && ra >= 0 && rb >= 0 && o + ra < lim && o + rb < lim);
  return make_int2(int((st[o + ra] >> sa) & 3u), int((st[o + rb] >> sb) & 3u));
}
template <int K>
__device__ __forceinline__ int2 draw_bft2(const int4* __restrict__ prog, const double* __restrict__ bft,
                                          const uint32_t* st, int rs, int ra, int rb, int sa, int sb, double ua,
                                          double ub, bool& zs, int lim, int64_t nrows) {
  const int4 h = __ldg(prog);  // card, npar, nchl, own row base
  const int4* p = prog + 1;
  int ia = h.w, ib = h.w;
#pragma unroll 1
  for (int j = 0; j < h.y; j += 2, ++p) {
    const int4 r = __ldg(p);
    int2 g = get2(st, r.x * rs, ra, rb, sa, sb, lim);
    ia += g.x * r.y;
    ib += g.y * r.y;
    if (r.w) {
      g = get2(st, r.z * rs, ra, rb, sa, sb, lim);
      ia += g.x * r.w;
      ib += g.y * r.w;
    }
  }
  double wa[K], wb[K];
  SG_DCHECK(ia >= 0 && ib >= 0 && ia < nrows && ib < nrows);
  bft_row<K>(bft, ia, wa);
  bft_row<K>(bft, ib, wb);
#pragma unroll 1
  for (int k = 0; k < h.z; ++k) {
    const int4 c = __ldg(p++);
    int2 g = get2(st, c.x * rs, ra, rb, sa, sb, lim);
    ia = c.y + g.x;
    ib = c.y + g.y;
#pragma unroll 1
    for (int q = 0; q < c.z; ++q, ++p) {
      const int4 r = __ldg(p);
      g = get2(st, r.x * rs, ra, rb, sa, sb, lim);
      ia += g.x * r.y;
      ib += g.y * r.y;
      if (r.w) {
        g = get2(st, r.z * rs, ra, rb, sa, sb, lim);
        ia += g.x * r.w;
        ib += g.y * r.w;
      }
    }
    double fa[K], fb[K];
    SG_DCHECK(ia >= 0 && ib >= 0 && ia < nrows && ib < nrows);
    bft_row<K>(bft, ia, fa);
    bft_row<K>(bft, ib, fb);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      wa[t] = __dmul_rn(wa[t], fa[t]);
      wb[t] = __dmul_rn(wb[t], fb[t]);
    }
  }
  return make_int2(bft_finish<K>(wa, ua, zs), bft_finish<K>(wb, ub, zs));
}

template <int MODE, int BITS>
__global__ void __launch_bounds__(BIG_T, SG_BIG_MINB) k_sweep_big(const sg_net net, const sg_batch bt, const SweepArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ int s_err;
  __shared__ int s_next;  // next colour-group member to hand out
  constexpr int PER = 32 / BITS;
  constexpr uint32_t MASK = (1u << BITS) - 1u;
  const int tc = a.tc, n = net.n;
  const int rg0 = blockIdx.y * a.mg, mg = min(a.mg, bt.m - rg0);  // replicas of this tile
  const int wpr = tc / PER;                                       // state words per (variable, replica) row
  [[maybe_unused]] const int st_words = n * a.mg * wpr;
  uint32_t* st = sm;                                              // [n][a.mg][wpr]
  uint16_t* fl16 = reinterpret_cast<uint16_t*>(sm + size_t(n) * a.mg * wpr);  // [n][tc / 16] latent bits
  const int c0 = blockIdx.x * tc;
  const int ncase = min(tc, bt.cases - c0);
  const int nload = min(tc, bt.pitch - c0);  // multiple of 16
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpr = tc >> 4;  // 16-case chunks per row
  if (tid == 0) s_err = 0;

  // ---- stage the tile: a warp per variable row, one int4 (16 cases) per lane
  // step, the rows of SB variables loaded together (all in flight before any
  // is unpacked)
  auto stage = [&](int v, int r, int ch, int4 val) {
    if (r == 0) {  // every replica carries the shared latent mask
      uint32_t f = BITS == 2 ? flag_word16(val) : flag_bits16(val);
      const int cc = ch * 16;
      if (cc + 16 > ncase) f &= cc >= ncase ? 0u : ((1u << (ncase - cc)) - 1u);
      fl16[v * cpr + ch] = uint16_t(f);
    }
    uint32_t* dst = st + size_t(v * a.mg + r) * wpr + ch * (16 / PER);
    SG_DCHECK(v < n && r < a.mg && ch < cpr && (v * a.mg + r) * wpr + ch * (16 / PER) + (BITS == 2 ? 0 : 1) < st_words);
    if constexpr (BITS == 2) {
      dst[0] = crumb_word(val);
    } else {
      val.x &= 0x7F7F7F7F;
      val.y &= 0x7F7F7F7F;
      val.z &= 0x7F7F7F7F;
      val.w &= 0x7F7F7F7F;
      pack16<BITS>(val, dst);
    }
  };
  constexpr int SB = 4;
  for (int v0 = warp; v0 < n; v0 += SB * BIG_W) {
    for (int r = 0; r < mg; ++r) {
      for (int ch = lane; ch < cpr; ch += 32) {
        int4 val[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
          const int v = v0 + k * BIG_W;
          val[k] = make_int4(0, 0, 0, 0);
          if (v < n && ch * 16 < nload)
            val[k] = __ldcs(reinterpret_cast<const int4*>(bt.states + (int64_t(v) * bt.m + rg0 + r) * bt.pitch +
                                                          c0 + ch * 16));
        }
#pragma unroll
        for (int k = 0; k < SB; ++k)
          if (v0 + k * BIG_W < n) stage(v0 + k * BIG_W, r, ch, val[k]);
      }
    }
  }
  const uint32_t* fl = reinterpret_cast<const uint32_t*>(fl16);  // [n][tc / 32]
  const int fw = tc >> 5;
  uint16_t* wl = reinterpret_cast<uint16_t*>(sm + size_t(n) * a.mg * wpr + size_t(n) * fw) + warp * tc;
  const uint64_t key = a.fast_key_dev ? __ldg(a.fast_key_dev) : a.fast_key;
  const bool zs_armed = a.ftab && net.table_entries > 0 && __ldg(a.ftab + net.ftab_size) != 0u;
  constexpr bool use_bft = BITS == 2;  // 2-bit tiles draw from the blanket factor tables (sweep_big)
  bool zs = false;
  __syncthreads();

  // ---- colour groups; a warp owns one variable at a time
  for (int g = 0; g < net.num_groups; ++g) {
    const int gs = __ldg(net.group_start + g), ge = __ldg(net.group_start + g + 1);
    if (tid == 0) s_next = gs + BIG_W;
    __syncthreads();
    // members are handed out dynamically (costs differ); the first BIG_W go round-robin
    for (int vi = gs + warp; vi < ge;) {
      const int v = __ldg(net.order + vi);
      // the latent cases of v, in order, into this warp's list: each lane
      // expands one 16-bit half of a mask word (one word when the tile has
      // more than 16 words per row), ranks from a warp scan of the counts,
      // highest bit first
      int total;
      {
        const bool half = fw <= 16;
        uint32_t bits = 0;
        if (half) {
          if (lane < 2 * fw) bits = (fl[v * fw + (lane >> 1)] >> ((lane & 1) << 4)) & 0xFFFFu;
        } else if (lane < fw) {
          bits = fl[v * fw + lane];
        }
        int incl = __popc(bits);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        total = __shfl_sync(0xffffffffu, incl, 31);
        const int base = half ? lane << 4 : lane << 5;
        for (int pos = incl; bits; --pos) {
          const int hi = 31 - __clz(bits);
          SG_DCHECK(pos >= 1 && pos <= tc && base + hi < ncase);
          wl[pos - 1] = uint16_t(base + hi);
          bits ^= 1u << hi;
        }
      }
      __syncwarp();
      const int32_t* dv = net.var_desc + v * SG_DESC_WORDS;
      const int card = dv[0], nmb = dv[1];
      const int32_t* fd = !use_bft && nmb < 0 ? net.fac_desc + __ldg(net.fac_start + v) : nullptr;
      const int4* prog = use_bft ? reinterpret_cast<const int4*>(net.bft_desc + __ldg(net.bft_start + v)) : nullptr;
      int64_t nmiss = 0, ioff = 0;
      uint64_t k0 = 0, k1 = 0;
      if (MODE != SG_RNG_FAST) {
        nmiss = __ldg(bt.nmiss + v);
        if (MODE == SG_RNG_NUMPY) {
          k0 = __ldg(a.keys + 2 * v);
          k1 = __ldg(a.keys + 2 * v + 1);
        } else {
          ioff = __ldg(a.inj_off + v);
        }
      }
      const int rs = a.mg * wpr;  // words between variable rows of the tile (32-bit offsets throughout)
      int it1 = lane;             // first list entry of the single-case loop below
      if constexpr (use_bft) {
        if (nmb < 0 && mg == 1) {
          // one replica (m = 1: no Philox block to share across replicas): two cases
          // per lane, it and it + 32 of the warp's 64-entry stride; a final
          // remainder of <= 32 cases takes one single-case round instead
          int& it = it1;
          for (; total - (it - lane) > 32; it += 64) {
            const bool two = it + 32 < total;
            const int ca = wl[it], cb = wl[two ? it + 32 : it];
            const int cwa = ca / PER, sa = (ca % PER) * BITS, cwb = cb / PER, sb = (cb % PER) * BITS;
            int64_t rka = 0, rkb = 0;
            if (MODE != SG_RNG_FAST) {
              rka = __ldg(bt.rank + int64_t(v) * bt.ld_rank + c0 + ca);
              rkb = __ldg(bt.rank + int64_t(v) * bt.ld_rank + c0 + cb);
            }
            const uint64_t ga = uint64_t(bt.case_base + c0 + ca), gb = uint64_t(bt.case_base + c0 + cb);
            for (int l = 0; l < mg; ++l) {
              const int r = rg0 + l;
              double ua, ub;
              if (MODE == SG_RNG_FAST) {
                ua = double(pick(fast_block(key, ga, uint32_t(v), uint32_t(r >> 2), 0u), r & 3)) * 0x1.0p-32;
                ub = double(pick(fast_block(key, gb, uint32_t(v), uint32_t(r >> 2), 0u), r & 3)) * 0x1.0p-32;
              } else if (MODE == SG_RNG_NUMPY) {
                ua = np_uniform(uint64_t(int64_t(r) * nmiss + rka), k0, k1);
                ub = np_uniform(uint64_t(int64_t(r) * nmiss + rkb), k0, k1);
              } else {
                ua = __ldg(a.uniforms + ioff + int64_t(r) * nmiss + rka);
                ub = __ldg(a.uniforms + ioff + int64_t(r) * nmiss + rkb);
              }
              const int2 x =
                  card == 2
                      ? draw_bft2<2>(prog, net.bft, st, rs, l * wpr + cwa, l * wpr + cwb, sa, sb, ua, ub, zs, st_words,
                                     net.bft_rows)
                  : card == 3
                      ? draw_bft2<3>(prog, net.bft, st, rs, l * wpr + cwa, l * wpr + cwb, sa, sb, ua, ub, zs, st_words,
                                     net.bft_rows)
                      : draw_bft2<4>(prog, net.bft, st, rs, l * wpr + cwa, l * wpr + cwb, sa, sb, ua, ub, zs, st_words,
                                     net.bft_rows);
              uint32_t* wa = st + v * rs + l * wpr + cwa;
              const uint32_t da = ((*wa >> sa) ^ uint32_t(x.x)) & MASK;
              if (da) atomicXor(wa, da << sa);
              if (two) {
                uint32_t* wb = st + v * rs + l * wpr + cwb;
                const uint32_t db = ((*wb >> sb) ^ uint32_t(x.y)) & MASK;
                if (db) atomicXor(wb, db << sb);
              }
            }
          }
        }
      }
      for (int it = it1; it < total; it += 32) {
        const int c = wl[it];
        const int cw = c / PER, csh = (c % PER) * BITS;
        int64_t rank = 0;
        if (MODE != SG_RNG_FAST) rank = __ldg(bt.rank + int64_t(v) * bt.ld_rank + c0 + c);
        const uint64_t gcase = uint64_t(bt.case_base + c0 + c);
        u32x4 blk{};
        // the tile's replicas of (v, c): replica r takes word r % 4 of the Philox block of its
        // global quad (FAST counters), one block per quad of the tile's replicas
        for (int l = 0; l < mg; ++l) {
          const int r = rg0 + l;
          const int roff = l * wpr + cw;  // + u * rs selects variable u
          auto get = [&](int u) {
            SG_DCHECK(u >= 0 && u < n && u * rs + roff < st_words);
            return int((st[u * rs + roff] >> csh) & MASK);
          };
          double u01;
          uint32_t u31 = 0;
          if (MODE == SG_RNG_FAST) {
            if (l == 0 || (r & 3) == 0) blk = fast_block(key, gcase, uint32_t(v), uint32_t(r >> 2), 0u);
            const uint32_t wv = pick(blk, r & 3);
            u31 = wv >> 1;
            u01 = double(wv) * 0x1.0p-32;
          } else {
            const int64_t ui = int64_t(r) * nmiss + rank;  // reference lane order (sampler.py:245)
            u01 = MODE == SG_RNG_NUMPY ? np_uniform(uint64_t(ui), k0, k1) : __ldg(a.uniforms + ioff + ui);
          }
          int x = 0;
          if (nmb >= 0) {  // conditional table of the blanket configuration
            int e = 0;
            for (int q = 0; q < nmb; ++q) e += get(dv[4 + q]) * dv[4 + SG_DESC_MB + q];
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
              const double au = __dmul_rn(u01, norm);
              for (int q = 0; q < card - 1; ++q) x += au > __ldg(p + q);
            }
          } else if constexpr (use_bft) {
            x = card == 2   ? draw_bft<2>(prog, net.bft, get, u01, zs, net.bft_rows)
                : card == 3 ? draw_bft<3>(prog, net.bft, get, u01, zs, net.bft_rows)
                            : draw_bft<4>(prog, net.bft, get, u01, zs, net.bft_rows);
          } else {
            x = draw_factored<4>(fd, a.cpt, get, u01, zs);
          }
          // lanes of one state word update disjoint fields: one XOR of (old ^ new) each
          uint32_t* wp = st + v * rs + roff;
          const uint32_t d = ((*wp >> csh) ^ uint32_t(x)) & MASK;
          if (d) atomicXor(wp, d << csh);
        }
      }
      __syncwarp();
      int nx = 0;
      if (lane == 0) nx = atomicAdd(&s_next, 1);
      vi = __shfl_sync(0xffffffffu, nx, 0);
    }
    __syncthreads();
  }
  if (zs) atomicOr(&s_err, int(SG_ERR_ZERO_SUPPORT));

  // ---- write the tile back (flags restored)
  for (int v = warp; v < n; v += BIG_W) {
    for (int r = 0; r < mg; ++r) {
      for (int ch = lane; ch * 16 < nload; ch += 32) {
        const uint32_t f = fl16[v * cpr + ch];
        const uint32_t* src = st + size_t(v * a.mg + r) * wpr + ch * (16 / PER);
        uint32_t o[4] = {0u, 0u, 0u, 0u};
        if constexpr (BITS == 2) {
          const uint32_t w = src[0];
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = state_bytes4(w, f, k);
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const uint32_t x = (src[k >> 3] >> (4 * (k & 7))) & 15u;
            o[k >> 2] |= (x | (((f >> k) & 1u) << 7)) << (8 * (k & 3));
          }
        }
        __stcs(reinterpret_cast<int4*>(bt.states + (int64_t(v) * bt.m + rg0 + r) * bt.pitch + c0 + ch * 16),
               make_int4(int(o[0]), int(o[1]), int(o[2]), int(o[3])));
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(a.err, s_err);
}

template <int MODE, int BITS>
static void launch_big(const sg_net& net, const sg_batch& bt, const SweepArgs& a, size_t smem, cudaStream_t s) {
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, smem))
    cudaFuncSetAttribute(k_sweep_big<MODE, BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const dim3 grid((bt.cases + a.tc - 1) / a.tc, (bt.m + a.mg - 1) / a.mg);
  k_sweep_big<MODE, BITS><<<grid, BIG_T, smem, s>>>(net, bt, a);
}

bool sweep_big(const sg_net& net, const sg_batch& bt, const SweepArgs& a0, int rng_mode, cudaStream_t s) {
  if (net.n <= 32 || net.max_card > 16) return false;
  // 2-bit tiles need the blanket factor tables (built with the pack when cards <= 4)
  const int bits = net.max_card <= 4 && net.bft_rows > 0 && net.bft ? 2 : 4;
  constexpr size_t budget = SG_BIG_SMEM;
  auto smem_of = [&](int mg, int tc) { return bits == 2 ? big_smem<2>(net.n, mg, tc) : big_smem<4>(net.n, mg, tc); };
  // widest tile (<= 1024 cases, multiple of 32) over all replicas; replica
  // groups only when even 64 cases do not fit
  int tc = 0, mg = bt.m;
  for (int t = 1024; t >= 64 && !tc; t -= 32)
    if (smem_of(mg, t) <= budget) tc = t;
  for (int g = bt.m - 1; g >= 1 && !tc; --g)
    for (int t = 512; t >= 64 && !tc; t -= 32)
      if (smem_of(g, t) <= budget) {
        tc = t;
        mg = g;
      }
  if (!tc) return false;
  // do not make tiles much wider than the batch
  while (tc > 64 && tc - 32 >= bt.cases) tc -= 32;
  if (bits == 2) {
    const int64_t blocks = (net.bft_rows + 255) / 256;
    k_build_bft<<<int(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, s>>>(net, a0.cpt);
  }
  SweepArgs a = a0;
  a.tc = tc;
  a.mg = mg;
  const size_t smem = smem_of(mg, tc);
  switch (rng_mode * 2 + (bits == 2 ? 0 : 1)) {
    case 0: launch_big<SG_RNG_FAST, 2>(net, bt, a, smem, s); break;
    case 1: launch_big<SG_RNG_FAST, 4>(net, bt, a, smem, s); break;
    case 2: launch_big<SG_RNG_NUMPY, 2>(net, bt, a, smem, s); break;
    case 3: launch_big<SG_RNG_NUMPY, 4>(net, bt, a, smem, s); break;
    case 4: launch_big<SG_RNG_INJECTED, 2>(net, bt, a, smem, s); break;
    default: launch_big<SG_RNG_INJECTED, 4>(net, bt, a, smem, s); break;
  }
  return true;
}

}  // namespace sg

SG_CHECKED_EXPORT(big)
