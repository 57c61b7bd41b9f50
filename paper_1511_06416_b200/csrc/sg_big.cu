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
  uint32_t* st = sm;                                              // [n][a.mg][wpr]
  uint16_t* fl16 = reinterpret_cast<uint16_t*>(sm + size_t(n) * a.mg * wpr);  // [n][tc / 16] latent bits
  const int c0 = blockIdx.x * tc;
  const int ncase = min(tc, bt.cases - c0);
  const int nload = min(tc, bt.pitch - c0);  // multiple of 16
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpr = tc >> 4;  // 16-case chunks per row
  if (tid == 0) s_err = 0;

  // ---- stage the tile: one int4 (16 cases) per thread step, packed on the fly
  for (int i = tid; i < n * mg * cpr; i += BIG_T) {
    const int row = i / cpr, ch = i - row * cpr;
    const int v = row / mg, r = row - v * mg;
    int4 val = make_int4(0, 0, 0, 0);
    if (ch * 16 < nload)
      val = __ldcs(reinterpret_cast<const int4*>(bt.states + (int64_t(v) * bt.m + rg0 + r) * bt.pitch + c0 + ch * 16));
    if (r == 0) {  // every replica carries the shared latent mask
      uint32_t f = flag_bits16(val);
      const int cc = ch * 16;
      if (cc + 16 > ncase) f &= cc >= ncase ? 0u : ((1u << (ncase - cc)) - 1u);
      fl16[v * cpr + ch] = uint16_t(f);
    }
    val.x &= 0x7F7F7F7F;
    val.y &= 0x7F7F7F7F;
    val.z &= 0x7F7F7F7F;
    val.w &= 0x7F7F7F7F;
    pack16<BITS>(val, st + size_t(v * a.mg + r) * wpr + ch * (16 / PER));
  }
  const uint32_t* fl = reinterpret_cast<const uint32_t*>(fl16);  // [n][tc / 32]
  const int fw = tc >> 5;
  uint16_t* wl = reinterpret_cast<uint16_t*>(sm + size_t(n) * a.mg * wpr + size_t(n) * fw) + warp * tc;
  const uint64_t key = a.fast_key_dev ? __ldg(a.fast_key_dev) : a.fast_key;
  const bool zs_armed = a.ftab && net.table_entries > 0 && __ldg(a.ftab + net.ftab_size) != 0u;
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
      // the latent cases of v, in order, into this warp's list: lane w < fw expands mask word w
      const uint32_t word = lane < fw ? fl[v * fw + lane] : 0u;
      const int cnt = __popc(word);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      {
        int pos = incl - cnt;
        for (uint32_t b = word; b; b &= b - 1) wl[pos++] = uint16_t(lane * 32 + __ffs(b) - 1);
      }
      __syncwarp();
      const int32_t* dv = net.var_desc + v * SG_DESC_WORDS;
      const int card = dv[0], nmb = dv[1];
      const int32_t* fd = nmb < 0 ? net.fac_desc + __ldg(net.fac_start + v) : nullptr;
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
      for (int it = lane; it < total; it += 32) {
        const int c = wl[it];
        const int cw = c / PER, csh = (c % PER) * BITS;
        int64_t rank = 0;
        if (MODE != SG_RNG_FAST) rank = __ldg(bt.rank + int64_t(v) * bt.ld_rank + c0 + c);
        const uint64_t gcase = uint64_t(bt.case_base + c0 + c);
        // the tile's replicas of (v, c): replica r takes word r % 4 of the Philox block of its
        // global quad (FAST counters); the block is recomputed per replica so that no block
        // state stays live across the draw (register pressure: 64 registers at 1024 threads)
        for (int l = 0; l < mg; ++l) {
          const int r = rg0 + l;
          const int roff = l * wpr + cw;  // + u * rs selects variable u
          auto get = [&](int u) { return int((st[u * rs + roff] >> csh) & MASK); };
          double u01;
          uint32_t u31 = 0;
          if (MODE == SG_RNG_FAST) {
            const uint32_t wv = pick(fast_block(key, gcase, uint32_t(v), uint32_t(r >> 2), 0u), r & 3);
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
          } else {
            x = draw_factored<4>(fd, a.cpt, get, u01, zs);
          }
          uint32_t* wp = st + v * rs + roff;
          atomicAnd(wp, ~(MASK << csh));
          atomicOr(wp, uint32_t(x) << csh);
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
  for (int i = tid; i < n * mg * cpr; i += BIG_T) {
    const int row = i / cpr, ch = i - row * cpr;
    if (ch * 16 >= nload) continue;
    const int v = row / mg, r = row - v * mg;
    const uint32_t f = fl16[v * cpr + ch];
    const uint32_t* src = st + size_t(v * a.mg + r) * wpr + ch * (16 / PER);
    uint32_t o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t x = BITS == 2 ? (src[0] >> (2 * k)) & 3u : (src[k >> 3] >> (4 * (k & 7))) & 15u;
      o[k >> 2] |= (x | (((f >> k) & 1u) << 7)) << (8 * (k & 3));
    }
    __stcs(reinterpret_cast<int4*>(bt.states + (int64_t(v) * bt.m + rg0 + r) * bt.pitch + c0 + ch * 16),
           make_int4(int(o[0]), int(o[1]), int(o[2]), int(o[3])));
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
  const int bits = net.max_card <= 4 ? 2 : 4;
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
