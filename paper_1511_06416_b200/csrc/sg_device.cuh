// Device-side building blocks shared by every kernel of the sweep path.
//
//  * Philox4x64-10 exactly as numpy's Philox bit generator consumes it
//    (reference rng.py:23-25 -> numpy Generator.random / integers), and
//    Philox4x32-10 (Random123 constants) for the fast RNG mode.
//  * numpy's pairwise float64 summation, which decides `norm` in
//    _resample_variable (sampler.py:242) and the row sums of mean_cpts
//    (model.py:193) for rows of 8 or more states.
//  * The reference's full-conditional weight product (sampler.py:226-240).
//
// The library is compiled with --fmad=false and every fp64 step uses the
// explicitly rounded intrinsics, so no product/sum is ever contracted into an
// FMA: the reference rounds each numpy operation separately.
#pragma once

#include <cstdlib>
#include <utility>

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/samegibbs_b200.h"

#define SG_THREADS 256
#define SG_MAX_CARD 64      // states per variable (int8 lane state keeps 7 bits)
#define SG_MAX_MB 64        // Markov-blanket members gathered per draw
#define SG_REJ_SLACK 64     // Lemire rejections tolerated per init stream
#define SG_MAX_DEVICES 64   // per-device caches of kernel attribute opt-ins

namespace sg {

// ---------------------------------------------------------------- Philox
struct u64x4 {
  uint64_t a, b, c, d;
};
struct u32x4 {
  uint32_t a, b, c, d;
};

__device__ __forceinline__ u64x4 philox4x64_10(u64x4 x, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t lo0 = M0 * x.a, hi0 = __umul64hi(M0, x.a);
    const uint64_t lo1 = M1 * x.c, hi1 = __umul64hi(M1, x.c);
    x = u64x4{hi1 ^ x.b ^ k0, lo1, hi0 ^ x.d ^ k1, lo0};
  }
  return x;
}

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 x, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint32_t lo0 = M0 * x.a, hi0 = __umulhi(M0, x.a);
    const uint32_t lo1 = M1 * x.c, hi1 = __umulhi(M1, x.c);
    x = u32x4{hi1 ^ x.b ^ k0, lo1, hi0 ^ x.d ^ k1, lo0};
  }
  return x;
}

__device__ __forceinline__ uint64_t pick(const u64x4& w, int i) {
  return i == 0 ? w.a : i == 1 ? w.b : i == 2 ? w.c : w.d;
}
__device__ __forceinline__ uint32_t pick(const u32x4& w, int i) {
  return i == 0 ? w.a : i == 1 ? w.b : i == 2 ? w.c : w.d;
}

// numpy Generator(Philox(key)).random(): draw i of the stream.
__device__ __forceinline__ uint64_t np_raw64(uint64_t i, uint64_t k0, uint64_t k1) {
  const u64x4 w = philox4x64_10(u64x4{(i >> 2) + 1ull, 0ull, 0ull, 0ull}, k0, k1);
  return pick(w, int(i & 3));
}
__device__ __forceinline__ double np_uniform(uint64_t i, uint64_t k0, uint64_t k1) {
  return double(np_raw64(i, k0, k1) >> 11) * 0x1.0p-53;
}
// 32-bit word j of the stream as numpy's next_uint32 hands it out: low half,
// then high half of each 64-bit draw.
__device__ __forceinline__ uint32_t np_word32(uint64_t j, uint64_t k0, uint64_t k1) {
  const uint64_t w = np_raw64(j >> 1, k0, k1);
  return (j & 1) ? uint32_t(w >> 32) : uint32_t(w);
}

// FAST-mode stream: Philox4x32-10 under a FIXED key, counter
//   (global case, v | quad << 16 | purpose << 28, step key lo, step key hi)
// for global case < 2^32, v < 2^16, quad < 2^12, purpose < 16 (checked by
// the entry points).  The step key rides in the counter, so every round key
// is a compile-time immediate, and the first round splits into a per-launch
// part (FastKey, from the key words), a per-case part (FastCase, from the
// case word) and one XOR with the (variable, quad) word -- the packed sweep
// shares the first two across all of a case's draws.
constexpr uint32_t FAST_K0 = 0x243F6A88u, FAST_K1 = 0x85A308D3u;
constexpr uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
constexpr uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

struct FastKey {
  uint32_t hk0, lo1, khi;  // umulhi(M1, key_lo) ^ K0, M1 * key_lo, key_hi ^ K1
};
struct FastCase {
  uint32_t x0, x1, x2, x3;  // state after round 1, without the (v, quad) word
};

__device__ __forceinline__ FastKey fast_key(uint64_t key) {
  const uint32_t lo = uint32_t(key);
  return FastKey{__umulhi(PHILOX_M1, lo) ^ FAST_K0, PHILOX_M1 * lo, uint32_t(key >> 32) ^ FAST_K1};
}
__device__ __forceinline__ FastCase fast_case(const FastKey& k, uint32_t gcase) {
  return FastCase{k.hk0, k.lo1, __umulhi(PHILOX_M0, gcase) ^ k.khi, PHILOX_M0 * gcase};
}
__device__ __forceinline__ uint32_t fast_word(uint32_t v, uint32_t quad, uint32_t purpose) {
  return v | (quad << 16) | (purpose << 28);
}
// Rounds 2..10 after the shared first round.
__device__ __forceinline__ u32x4 fast_draw(const FastCase& c, uint32_t word) {
  u32x4 x{c.x0 ^ word, c.x1, c.x2, c.x3};
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const uint32_t k0 = FAST_K0 + uint32_t(r) * PHILOX_W0, k1 = FAST_K1 + uint32_t(r) * PHILOX_W1;
    const uint32_t lo0 = PHILOX_M0 * x.a, hi0 = __umulhi(PHILOX_M0, x.a);
    const uint32_t lo1 = PHILOX_M1 * x.c, hi1 = __umulhi(PHILOX_M1, x.c);
    x = u32x4{hi1 ^ x.b ^ k0, lo1, hi0 ^ x.d ^ k1, lo0};
  }
  return x;
}
// Host check of the FAST counter's case word: global case ids fit 32 bits.
inline bool fast_cases_ok(int64_t case_base, int64_t cases) {
  return case_base >= 0 && case_base + cases <= (int64_t(1) << 32);
}
// = philox4x32_10({gcase, fast_word(v, quad, purpose), key_lo, key_hi}, FAST_K0, FAST_K1)
__device__ __forceinline__ u32x4 fast_block(uint64_t key, uint64_t gcase, uint32_t v,
                                            uint32_t quad, uint32_t purpose) {
  return fast_draw(fast_case(fast_key(key), uint32_t(gcase)), fast_word(v, quad, purpose));
}

// ---------------------------------------------------------------- fp64
// numpy pairwise_sum (8 accumulators from 8 elements up, halving above 128),
// i.e. ndarray.sum(axis=-1) of a contiguous row of length n.
__device__ __forceinline__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, a[i]);
    return s;
  }
  // n <= SG_MAX_CARD (64) <= 128: single block of 8 accumulators.
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a[i + 0]);
    r1 = __dadd_rn(r1, a[i + 1]);
    r2 = __dadd_rn(r2, a[i + 2]);
    r3 = __dadd_rn(r3, a[i + 3]);
    r4 = __dadd_rn(r4, a[i + 4]);
    r5 = __dadd_rn(r5, a[i + 5]);
    r6 = __dadd_rn(r6, a[i + 6]);
    r7 = __dadd_rn(r7, a[i + 7]);
  }
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                       __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) s = __dadd_rn(s, a[i]);
  return s;
}

// CPT reads: through the read-only path when the CPTs are kernel inputs,
// plain loads when the same kernel just wrote them (sg_step_finish).
template <bool RO, typename T>
__device__ __forceinline__ T ro_load(const T* p) {
  if (RO) return __ldg(p);
  return *p;
}
template <bool RO>
__device__ __forceinline__ double cpt_load(const double* p) {
  return ro_load<RO>(p);
}

// Reference full-conditional weights of v given its Markov-blanket states
// s[slot] (sampler.py:226-240): w = T_v[cfg, :], then for each child c in
// ascending order w[t] *= T_c[cfg0_c + t*stride_vc, x_c].
// K > 0: the caller knows card == K at compile time, so w[] stays in
// registers (K = 0: runtime card, w[] in local memory).
template <bool RO = true, int K = 0>
__device__ __forceinline__ void conditional_weights(const sg_net& net, int v, const int* s,
                                                    const double* cpt, double* w) {
  const int card = K ? K : ro_load<RO>(net.card + v);
  int64_t cfg = 0;
  for (int j = ro_load<RO>(net.par_start + v), e = ro_load<RO>(net.par_start + v + 1); j < e; ++j)
    cfg += int64_t(s[ro_load<RO>(net.par_slot + j)]) * ro_load<RO>(net.par_stride + j);
  const double* row = cpt + ro_load<RO>(net.cpt_off + v) + cfg * card;
#pragma unroll
  for (int t = 0; t < (K ? K : card); ++t) w[t] = cpt_load<RO>(row + t);
  for (int k = ro_load<RO>(net.chl_start + v), ke = ro_load<RO>(net.chl_start + v + 1); k < ke; ++k) {
    const int c = ro_load<RO>(net.chl_var + k);
    const int cc = ro_load<RO>(net.card + c);
    const int xc = s[ro_load<RO>(net.chl_slot + k)];
    int64_t cfg0 = 0;
    for (int q = ro_load<RO>(net.chl_pstart + k), qe = ro_load<RO>(net.chl_pstart + k + 1); q < qe; ++q)
      cfg0 += int64_t(s[ro_load<RO>(net.chl_pslot + q)]) * ro_load<RO>(net.chl_pstride + q);
    const int64_t vs = ro_load<RO>(net.chl_vstride + k);
    const double* tc = cpt + ro_load<RO>(net.cpt_off + c) + xc;
#pragma unroll
    for (int t = 0; t < (K ? K : card); ++t) w[t] = __dmul_rn(w[t], cpt_load<RO>(tc + (cfg0 + t * vs) * cc));
  }
}

// Direct evaluation for variables without a table (blanket too large): the
// reference's weight product for one lane (sampler.py:226-240) from the
// factored descriptor (sg_net.fac_desc) -- parent row, then each child's
// factor in ascending child order, every product rounded as numpy rounds it
// (no FMA).  `get(var)` returns the lane's current state of a variable
// (shared-memory tile or packed column).  Children are taken two at a time
// so their loads overlap.
// KMAX > 0 (K = 0): one code path for every card <= KMAX -- fixed-size arrays,
// the entries t >= card predicated off -- so warps drawing variables of
// different cardinalities share one instruction stream (fewer i-cache misses);
// the arithmetic on the entries t < card is exactly that of K = card.
template <int K, class Get, int KMAX = 0>
__device__ __forceinline__ int draw_factored_k(const int32_t* __restrict__ fd, const double* __restrict__ cpt,
                                               Get get, double u, bool& zs) {
  const int card = K ? K : fd[0];
  const int npar = fd[1], nchl = fd[2];
  int base = fd[3];
  const int32_t* p = fd + 4;
  for (int j = 0; j < npar; ++j, p += 2) {
    const int2 e = *reinterpret_cast<const int2*>(p);
    base += get(e.x) * e.y;
  }
  constexpr int NT = K ? K : (KMAX ? KMAX : SG_MAX_CARD);
  double w[NT];
#pragma unroll
  for (int t = 0; t < (K || KMAX ? NT : card); ++t) w[t] = (K || t < card) ? __ldg(cpt + base + t) : 0.0;
  int k = 0;
  for (; k + 1 < nchl; k += 2) {
    int i0 = p[1] + get(p[0]);
    const int s0 = p[3], n0 = p[4];
    p += 6;
    for (int q = 0; q < n0; ++q, p += 2) {
      const int2 e = *reinterpret_cast<const int2*>(p);
      i0 += get(e.x) * e.y;
    }
    int i1 = p[1] + get(p[0]);
    const int s1 = p[3], n1 = p[4];
    p += 6;
    for (int q = 0; q < n1; ++q, p += 2) {
      const int2 e = *reinterpret_cast<const int2*>(p);
      i1 += get(e.x) * e.y;
    }
    double f0[NT], f1[NT];
#pragma unroll
    for (int t = 0; t < (K || KMAX ? NT : card); ++t) {
      f0[t] = (K || t < card) ? __ldg(cpt + i0 + t * s0) : 0.0;
      f1[t] = (K || t < card) ? __ldg(cpt + i1 + t * s1) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < (K || KMAX ? NT : card); ++t) w[t] = __dmul_rn(__dmul_rn(w[t], f0[t]), f1[t]);
  }
  if (k < nchl) {
    int i0 = p[1] + get(p[0]);
    const int s0 = p[3], n0 = p[4];
    p += 6;
    for (int q = 0; q < n0; ++q, p += 2) {
      const int2 e = *reinterpret_cast<const int2*>(p);
      i0 += get(e.x) * e.y;
    }
#pragma unroll
    for (int t = 0; t < (K || KMAX ? NT : card); ++t)
      if (K || t < card) w[t] = __dmul_rn(w[t], __ldg(cpt + i0 + t * s0));
  }
  double norm;
  if (K && K < 8) {  // numpy's pairwise sum is sequential below 8 terms
    norm = 0.0;
#pragma unroll
    for (int t = 0; t < (K ? K : 1); ++t) norm = __dadd_rn(norm, w[t]);
  } else if (KMAX && KMAX < 8) {
    norm = 0.0;
#pragma unroll
    for (int t = 0; t < (KMAX ? KMAX : 1); ++t)
      if (t < card) norm = __dadd_rn(norm, w[t]);
  } else {
    norm = np_pairwise_sum(w, card);
  }
  if (!(norm > 0.0)) zs = true;
  const double au = __dmul_rn(u, norm);
  double cum = 0.0;
  int x = 0;
#pragma unroll
  for (int t = 0; t < (K ? K - 1 : (KMAX ? KMAX - 1 : card - 1)); ++t) {
    if (K || !KMAX || t < card - 1) {
      cum = t ? __dadd_rn(cum, w[t]) : w[0];
      x += (au > cum);
    }
  }
  return x;
}

// UNIFIED: cards 2..4 share one code path (k_sweep_big: its 32 warps draw
// variables of mixed cardinality side by side, and the unified path cut its
// instruction-fetch stalls -- C4 sweep 15.9 -> 11.4 ms); the lane and tile
// kernels keep one specialisation per card (C3, mostly binary: 3.35 ms vs
// 3.80 ms unified).
template <int UNIFIED = 0, class Get>
__device__ __forceinline__ int draw_factored(const int32_t* fd, const double* cpt, Get get, double u, bool& zs) {
  if (UNIFIED) {
    if (fd[0] <= UNIFIED) return draw_factored_k<0, Get, (UNIFIED ? UNIFIED : 1)>(fd, cpt, get, u, zs);
    if (UNIFIED < 4 && fd[0] == 4) return draw_factored_k<4>(fd, cpt, get, u, zs);
    return draw_factored_k<0>(fd, cpt, get, u, zs);
  }
  switch (fd[0]) {
    case 2: return draw_factored_k<2>(fd, cpt, get, u, zs);
    case 3: return draw_factored_k<3>(fd, cpt, get, u, zs);
    case 4: return draw_factored_k<4>(fd, cpt, get, u, zs);
    default: return draw_factored_k<0>(fd, cpt, get, u, zs);
  }
}

// Call f(std::integral_constant<int, K>) with K = card for the common small
// cardinalities (register-resident weight arrays), K = 0 otherwise.
template <class F>
__device__ __forceinline__ void with_card(int card, F&& f) {
  switch (card) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    default: f(std::integral_constant<int, 0>{}); break;
  }
}

// Sequential draws of one Philox4x32 substream (counter = (cell, call, hi, tag))
// for the Dirichlet CPT update.
struct CellStream {
  uint32_t k0, k1, cell_lo, cell_hi, call;
  u32x4 buf;
  int used;
  __device__ CellStream(uint64_t key, uint64_t cell)
      : k0(uint32_t(key)), k1(uint32_t(key >> 32)), cell_lo(uint32_t(cell)), cell_hi(uint32_t(cell >> 32)),
        call(0), used(4) {}
  __device__ uint32_t next() {
    if (used == 4) {
      buf = philox4x32_10(u32x4{cell_lo, call++, cell_hi, 0x5A4D0001u}, k0, k1);
      used = 0;
    }
    return pick(buf, used++);
  }
  // uniform in (0, 1): 53 bits, never 0
  __device__ double uniform() {
    const uint64_t hi = next() >> 5, lo = next() >> 6;  // 27 + 26 bits
    return (double((hi << 26) | lo) + 0.5) * 0x1.0p-53;
  }
  __device__ double normal() {
    const double u1 = uniform(), u2 = uniform();
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
};

// Gamma(a, 1) draws (Marsaglia & Tsang 2000) from a cell's Philox stream.
// Stream layout: words 0-1 the boost uniform (a < 1: Gamma(a) = Gamma(a + 1)
// * U^(1/a)), words 2-5 the first attempt's normal, 6-7 its acceptance
// uniform; later attempts continue from word 8 (normal, then uniform when
// 1 + c x > 0).  The first attempt's variates do not depend on a, so a
// kernel can draw them before the counts arrive (GammaPre).
struct GammaPre {
  double ub, x, u;
};
__device__ __forceinline__ GammaPre gamma_pre(CellStream& rs) {
  GammaPre g;
  g.ub = rs.uniform();
  g.x = rs.normal();
  g.u = rs.uniform();
  return g;
}

// Returns the draw g itself when a >= 1, or log g when a < 1 (*in_log set):
// tiny shapes are carried in log space so they never underflow (the
// degenerate-row redraw of model.py:168-176 is not needed).
__device__ __forceinline__ double gamma_draw(CellStream& rs, const GammaPre& pre, double a, bool* in_log) {
  double boost = 0.0;
  const bool lg = a < 1.0;
  if (lg) {
    boost = log(pre.ub) / a;
    a += 1.0;
  }
  *in_log = lg;
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (int attempt = 0;; ++attempt) {
    const double x = attempt ? rs.normal() : pre.x;
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    const double u = attempt ? rs.uniform() : pre.u;
    v = v * v * v;
    const double x2 = x * x;
    if (u < 1.0 - 0.0331 * x2 * x2 || log(u) < 0.5 * x2 + d * (1.0 - v + log(v)))
      return lg ? log(d) + log(v) + boost : d * v;
  }
}

// Normalise one row of gamma draws (val[s] = g, or log g where in_log[s])
// into Dirichlet probabilities: linear when no cell is in log space,
// otherwise through exp(log g - max).
template <int K = 0>
__device__ __forceinline__ void dirichlet_row(const double* val, const uint8_t* in_log, int card, double* out) {
  if (K) card = K;
  bool any = false;
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) any |= in_log[s] != 0;
  if (!any) {
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < (K ? K : card); ++s) sum += val[s];
    const double inv = 1.0 / sum;
#pragma unroll
    for (int s = 0; s < (K ? K : card); ++s) out[s] = val[s] * inv;
    return;
  }
  double lv[K ? K : SG_MAX_CARD];
  double mx = -INFINITY;
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) {
    lv[s] = in_log[s] ? val[s] : log(val[s]);
    mx = fmax(mx, lv[s]);
  }
  double sum = 0.0;
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) {
    lv[s] = exp(lv[s] - mx);
    sum += lv[s];
  }
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) out[s] = lv[s] / sum;
}

// One conditional-table entry from the weights w[0..card) of a blanket
// configuration: pe = cum[0..card-2], norm; fe = ceil(cum/norm * 2^31)
// thresholds (0xFFFFFFFF in slot 0 and *zs_flag set when norm <= 0).
// pe may be NULL (thresholds only).
template <int K = 0>
__device__ __forceinline__ void table_entry(const double* w, int card, double* pe, uint32_t* fe,
                                            uint32_t* zs_flag) {
  if (K) card = K;
  double norm;
  if (K && K < 8) {  // numpy's pairwise sum is sequential below 8 terms
    norm = 0.0;
#pragma unroll
    for (int t = 0; t < (K ? K : 1); ++t) norm = __dadd_rn(norm, w[t]);
  } else {
    norm = np_pairwise_sum(w, card);
  }
  const bool ok = norm > 0.0;
  // FAST thresholds only need to be deterministic and monotone: scale by one reciprocal
  const double scale = ok ? __ddiv_rn(2147483648.0, norm) : 0.0;
  double cum = 0.0;
#pragma unroll
  for (int t = 0; t < (K ? K - 1 : card - 1); ++t) {
    cum = t ? __dadd_rn(cum, w[t]) : w[0];
    if (pe) pe[t] = cum;
    const double q = fmin(ceil(__dmul_rn(cum, scale)), 2147483648.0);
    fe[t] = (t == 0 && !ok) ? 0xFFFFFFFFu : uint32_t(q);
  }
  if (pe) pe[card - 1] = norm;
  if (!ok) atomicOr(reinterpret_cast<int*>(zs_flag), 1);
}

// p_v(x | blanket) = w_x * (1 / norm) for the joint sweep's transition tables
// (sequential norm: cards <= 4), 0 where the blanket has no support.
template <int K = 0>
__device__ __forceinline__ void joint_conditional(const double* w, int card, double* out) {
  if (K) card = K;
  double norm = 0.0;
  for (int t = 0; t < card; ++t) norm = __dadd_rn(norm, w[t]);
  const double inv = norm > 0.0 ? __ddiv_rn(1.0, norm) : 0.0;
  for (int t = 0; t < card; ++t) out[t] = __dmul_rn(w[t], inv);
}

// Programmatic dependent launch (PDL).  A kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor in the stream is still running; pdl_wait() blocks until that
// predecessor has completed and its writes are visible (a no-op without
// PDL), pdl_trigger() lets this kernel's own dependent start its prologue.
// Launch with programmatic stream serialization (PDL; see pdl_wait).
template <typename... P, typename... A>
static inline cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const int pdl_off = std::getenv("SG_NO_PDL") != nullptr;  // debugging: plain stream order
  cfg.numAttrs = pdl_off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

// Kernel attribute opt-ins are per device context: each launch site keeps the
// largest shared-memory size it has opted in to, per device, and raises the
// attribute only when a launch needs more (so graph capture sees no
// attribute calls after the first launch on each device).
static inline bool optin_needed(size_t* configured /* [SG_MAX_DEVICES] */, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= SG_MAX_DEVICES) return true;
  if (bytes <= configured[dev]) return false;
  configured[dev] = bytes;
  return true;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int small_field(uint32_t S, const sg_small& sp, int v) {
  return int((S >> sp.off[v]) & ((1u << sp.width[v]) - 1u));
}

// Packed-lane table word(s) i = (v, S): the generic FAST thresholds of the
// blanket configuration that lane word S encodes (0 for unused words).
// Plain loads: ftab may have been written by the same kernel.
template <bool RO = true>
__device__ __forceinline__ void small_table_entry(const sg_net& net, const sg_small& sp, const uint32_t* ftab,
                                                  uint32_t* stab, int i) {
  const int v = i >> sp.bits;
  const uint32_t S = uint32_t(i & ((1 << sp.bits) - 1));
  const int card = sp.card[v];
  uint32_t* out = stab + sp.toff[v] + S * sp.tstride[v];
  bool valid = (S & ~sp.mbmask[v]) == 0u;
  int64_t e = 0;
  for (int k = ro_load<RO>(net.mb_start + v), ke = ro_load<RO>(net.mb_start + v + 1); k < ke && valid; ++k) {
    const int u = ro_load<RO>(net.mb_var + k);
    const int s = small_field(S, sp, u);
    valid = s < sp.card[u];
    e += int64_t(s) * ro_load<RO>(net.mb_stride + k);
  }
  const uint32_t* src = ftab + ro_load<RO>(net.ftab_off + v) + e * (card - 1);
  for (int t = 0; t < card - 1; ++t) out[t] = valid ? src[t] : 0u;
}

// Variable owning CPT cell `cell` (binary search over cpt_off).
template <bool RO = true>
__device__ __forceinline__ int cell_var(const sg_net& net, int64_t cell) {
  int lo = 0, hi = net.n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (ro_load<RO>(net.cpt_off + mid) <= cell) lo = mid; else hi = mid;
  }
  return lo;
}

// Copy of a two-blob network pack whose array pointers point into shared
// memory copies s32 / s64 of the blobs (see sg_net.blob32).
__device__ __forceinline__ sg_net rebase_net(const sg_net& g, const int32_t* s32, const int64_t* s64) {
  sg_net n = g;
#define SG_R32(f) n.f = g.f ? s32 + (g.f - g.blob32) : nullptr
#define SG_R64(f) n.f = g.f ? s64 + (g.f - g.blob64) : nullptr
  SG_R32(card); SG_R32(group_start); SG_R32(order); SG_R32(par_start); SG_R32(par_var); SG_R32(par_stride);
  SG_R32(par_slot); SG_R32(mb_start); SG_R32(mb_var); SG_R32(mb_stride); SG_R32(chl_start); SG_R32(chl_var);
  SG_R32(chl_vstride); SG_R32(chl_slot); SG_R32(chl_pstart); SG_R32(chl_pslot); SG_R32(chl_pstride);
  SG_R32(row_var); SG_R32(joint_radix); SG_R32(joint_cell); SG_R32(var_desc); SG_R32(fac_start); SG_R32(fac_desc); SG_R32(tally_chunk);
  SG_R64(cpt_off); SG_R64(row_off); SG_R64(tab_entries); SG_R64(tab_start); SG_R64(ptab_off); SG_R64(ftab_off);
#undef SG_R32
#undef SG_R64
  return n;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace sg

// ---------------------------------------------------------------- host side
namespace sg {
void set_error(const char* fmt, ...);
int check_launch(const char* what);
}  // namespace sg

// ---------------------------------------------------------------- checked builds
// -DSG_CHECKED (lib_checked.so; compute-sanitizer is closed on this GPU pool):
// SG_DCHECK(cond) asserts an index or protocol invariant on the device and
// records the first failing source line of its translation unit in a device
// word, which sg_debug_checked_<tu>() reads and clears (SG_CHECKED_EXPORT).
// Spin-waits take a bound (SG_SPIN_BOUNDED) and record a failure instead of
// hanging.  In normal builds every check compiles to nothing.
#ifdef SG_CHECKED
static __device__ unsigned int sg_checked_line;
#define SG_DCHECK(cond)                                                          \
  do {                                                                           \
    if (!(cond)) atomicCAS(&::sg_checked_line, 0u, static_cast<unsigned>(__LINE__)); \
  } while (0)
#define SG_CHECKED_EXPORT(tu)                                                        \
  __global__ void sg_checked_probe_##tu() { SG_DCHECK(threadIdx.x != 0); }         \
  extern "C" int sg_debug_checked_##tu(unsigned* line, int probe) {                 \
    if (probe) sg_checked_probe_##tu<<<1, 32>>>();                                  \
    unsigned zero = 0;                                                              \
    if (cudaDeviceSynchronize() != cudaSuccess ||                                   \
        cudaMemcpyFromSymbol(line, ::sg_checked_line, sizeof(unsigned)) != cudaSuccess || \
        cudaMemcpyToSymbol(::sg_checked_line, &zero, sizeof(unsigned)) != cudaSuccess)    \
      return ::sg::check_launch("sg_debug_checked_" #tu);                           \
    return SG_OK;                                                                   \
  }
#else
#define SG_DCHECK(cond) \
  do {                  \
  } while (0)
#define SG_CHECKED_EXPORT(tu)
#endif

#define SG_REQUIRE(cond, ...)        \
  do {                               \
    if (!(cond)) {                   \
      ::sg::set_error(__VA_ARGS__);  \
      return SG_EINVAL;              \
    }                                \
  } while (0)
