// Packed-lane sweep for small networks (FAST RNG mode).
//
// When every variable's state fits in a bit field and the whole lane fits in
// one byte (sum of field widths <= 7; Koller: 1+1+1+2+1 = 6 bits), a lane is
// a single uint8 word S.  Three consequences make the sweep cheap:
//
//  * the full conditional of v is a function of (S & mbmask_v), so the
//    conditional table is indexed by the masked lane word itself -- one LOP
//    and one LDS per draw, no blanket arithmetic;
//  * the latent pattern of a case (which variables are missing) is shared by
//    its m replicas; cases are bucketed by pattern once per minibatch
//    (counting sort, sg_small_prepare) so a warp's threads run the same
//    variable loop -- no divergence, and only latent variables cost work;
//  * the tally histograms S directly (2^bits joint states, per-thread byte
//    counters), expanded to CPT cells once per CTA.
//
// Layout (sg_small_batch): lanes uint8 [m][B] in bucketed slot order;
// pattern uint8 [B]; case_id int32 [B] (slot -> case of the minibatch).
// Counters and draws are identical to the generic kernel's FAST mode
// (Philox4x32 on (case, variable, replica quad)), so both paths produce the
// same states and counts from the same tables (tested).
#include "sg_device.cuh"

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

// Pattern histogram of the minibatch's cases.
__global__ void k_small_count(const sg_small sp, const int8_t* __restrict__ obs, int ld, int cases,
                              uint8_t* __restrict__ pattern_of_case, int* __restrict__ hist) {
  __shared__ int h[SMALL_PATTERNS];
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cases; c += gridDim.x * blockDim.x) {
    uint32_t P = 0;
    for (int v = 0; v < sp.n; ++v) P |= uint32_t(obs[int64_t(v) * ld + c] < 0) << v;
    pattern_of_case[c] = uint8_t(P);
    atomicAdd(&h[P], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

__global__ void k_small_scan(int* hist) {
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < SMALL_PATTERNS; ++i) {
      const int x = hist[i];
      hist[i] = run;
      run += x;
    }
  }
}

// Scatter cases into pattern buckets and build their lanes: observed fields
// from the data, latent fields from the FAST init stream (same draw as
// k_init_states: Philox4x32(key, (case, v, r/4, purpose 1))[r%4] * card >> 32).
// Slots are claimed per block (shared-memory ranks, one global atomic per
// pattern per block); the order inside a bucket is irrelevant to the
// results, which depend on case ids only.
__global__ void __launch_bounds__(256) k_small_scatter(
    const sg_small sp, const int8_t* __restrict__ obs, int ld, int cases, int m, int64_t case_base,
    uint64_t init_key, const uint8_t* __restrict__ pattern_of_case, int* __restrict__ cursor,
    uint8_t* __restrict__ pattern, int32_t* __restrict__ case_id, uint8_t* __restrict__ lanes, int lane_ld, int init) {
  __shared__ int cnt[SMALL_PATTERNS];
  __shared__ int base[SMALL_PATTERNS];
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t P = 0;
  int local = 0;
  if (c < cases) {
    P = pattern_of_case[c];
    local = atomicAdd(&cnt[P], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SMALL_PATTERNS; i += blockDim.x)
    base[i] = cnt[i] ? atomicAdd(cursor + i, cnt[i]) : 0;
  __syncthreads();
  if (c >= cases) return;
  const int s = base[P] + local;
  pattern[s] = uint8_t(P);
  case_id[s] = c;
  if (!init) return;
  uint32_t obsw = 0;
  for (int v = 0; v < sp.n; ++v) {
    const int o = obs[int64_t(v) * ld + c];
    if (o >= 0) obsw |= uint32_t(o) << sp.off[v];
  }
  for (int q = 0; q < (m + 3) / 4; ++q) {
    uint32_t S[4] = {obsw, obsw, obsw, obsw};
    for (int v = 0; v < sp.n; ++v) {
      if (!((P >> v) & 1u)) continue;
      const u32x4 w = fast_block(init_key, uint64_t(case_base + c), uint32_t(v), uint32_t(q), 1u);
      const uint32_t ws[4] = {w.a, w.b, w.c, w.d};
#pragma unroll
      for (int j = 0; j < 4; ++j) S[j] |= uint32_t((uint64_t(ws[j]) * uint32_t(sp.card[v])) >> 32) << sp.off[v];
    }
    for (int j = 0; j < 4 && q * 4 + j < m; ++j) lanes[int64_t(q * 4 + j) * lane_ld + s] = uint8_t(S[j]);
  }
}

// Restore the lane words of already-bucketed slots from generic int8 lane
// states (layout switch), and the reverse export.
__global__ void k_small_import(const sg_small sp, const sg_batch bt, const int32_t* __restrict__ case_id,
                               uint8_t* __restrict__ lanes, int lane_ld) {
  const int64_t total = int64_t(bt.m) * bt.cases;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / bt.cases), s = int(i - int64_t(r) * bt.cases);
    const int c = case_id[s];
    uint32_t S = 0;
    for (int v = 0; v < sp.n; ++v)
      S |= uint32_t(bt.states[(int64_t(v) * bt.m + r) * bt.pitch + c] & 0x7F) << sp.off[v];
    lanes[int64_t(r) * lane_ld + s] = uint8_t(S);
  }
}

__global__ void k_small_export(const sg_small sp, const sg_batch bt, const int32_t* __restrict__ case_id,
                               const uint8_t* __restrict__ pattern, const uint8_t* __restrict__ lanes, int lane_ld) {
  const int64_t total = int64_t(bt.m) * bt.cases;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / bt.cases), s = int(i - int64_t(r) * bt.cases);
    const int c = case_id[s];
    const uint32_t S = lanes[int64_t(r) * lane_ld + s];
    const uint32_t P = pattern[s];
    for (int v = 0; v < sp.n; ++v)
      bt.states[(int64_t(v) * bt.m + r) * bt.pitch + c] =
          int8_t(small_field(S, sp, v) | (((P >> v) & 1u) ? 0x80 : 0));
  }
}

// The sweep.  A thread owns slot s (one case) and walks its replica quads;
// the four lanes of a quad live in registers as lane words.
__global__ void __launch_bounds__(SG_THREADS)
k_small_sweep(const sg_small sp, const uint32_t* __restrict__ stab_g, const uint8_t* __restrict__ pattern,
              const int32_t* __restrict__ case_id, uint8_t* __restrict__ lanes, int lane_ld, int cases, int num_real,
              int m, int64_t case_base, uint64_t key, const uint64_t* __restrict__ key_dev,
              const int32_t* __restrict__ jcell, int cells, unsigned long long* __restrict__ counts,
              const uint32_t* __restrict__ zs_flag, int32_t* err) {
  if (key_dev) key = __ldg(key_dev);
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* stab = reinterpret_cast<uint32_t*>(smem);
  uint8_t* hist8 = smem + ((sp.tab_words * 4 + 15) & ~15);
  uint32_t* cellacc = reinterpret_cast<uint32_t*>(hist8 + (SG_THREADS << sp.bits));
  const int tid = threadIdx.x;
  for (int i = tid; i < sp.tab_words; i += SG_THREADS) stab[i] = __ldg(stab_g + i);
  if (counts) {
    uint32_t* h32 = reinterpret_cast<uint32_t*>(hist8);
    for (int i = tid; i < (SG_THREADS << sp.bits) / 4; i += SG_THREADS) h32[i] = 0;
    for (int i = tid; i < cells; i += SG_THREADS) cellacc[i] = 0;
  }
  const bool armed = zs_flag && __ldg(zs_flag) != 0u;
  __syncthreads();
  const int slot = ((tid & 31) << 2) | ((tid >> 5) & 3) | ((tid >> 7) << 7);
  const int Q = (m + 3) >> 2;
  bool zs = false;
  for (int s = blockIdx.x * SG_THREADS + tid; s < cases; s += gridDim.x * SG_THREADS) {
    const uint32_t P = pattern[s];
    const int c = case_id[s];
    const bool real = counts && c < num_real;
    uint32_t Po = 0;  // latent bits permuted into colour order
    for (int i = 0; i < sp.n; ++i) Po |= ((P >> sp.order[i]) & 1u) << i;
    for (int q = 0; q < Q; ++q) {
      const int nl = min(4, m - q * 4);
      uint8_t* lp = lanes + int64_t(q * 4) * lane_ld + s;
      uint32_t S0 = lp[0];
      uint32_t S1 = nl > 1 ? lp[lane_ld] : 0u;
      uint32_t S2 = nl > 2 ? lp[2 * lane_ld] : 0u;
      uint32_t S3 = nl > 3 ? lp[3 * lane_ld] : 0u;
      for (uint32_t L = Po; L; L &= L - 1u) {  // latent variables, colour order
        const int v = sp.order[__ffs(L) - 1];
        const u32x4 w = fast_block(key, uint64_t(case_base + c), uint32_t(v), uint32_t(q), 0u);
        const uint32_t msk = sp.mbmask[v];
        const uint32_t* tv = stab + sp.toff[v];
        const int sh = sp.off[v];
        const uint32_t clear = ~(((1u << sp.width[v]) - 1u) << sh);
        const int k1 = sp.card[v] - 1;
        if (k1 == 1) {
          const uint32_t t0 = tv[S0 & msk], t1 = tv[S1 & msk], t2 = tv[S2 & msk], t3 = tv[S3 & msk];
          S0 = (S0 & clear) | (uint32_t((w.a >> 1) >= t0) << sh);
          S1 = (S1 & clear) | (uint32_t((w.b >> 1) >= t1) << sh);
          S2 = (S2 & clear) | (uint32_t((w.c >> 1) >= t2) << sh);
          S3 = (S3 & clear) | (uint32_t((w.d >> 1) >= t3) << sh);
          if (armed)
            zs |= t0 == 0xFFFFFFFFu || (nl > 1 && t1 == 0xFFFFFFFFu) || (nl > 2 && t2 == 0xFFFFFFFFu) ||
                  (nl > 3 && t3 == 0xFFFFFFFFu);
        } else {
          uint32_t Sx[4] = {S0, S1, S2, S3};
          const uint32_t ws[4] = {w.a >> 1, w.b >> 1, w.c >> 1, w.d >> 1};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t* th = tv + (Sx[j] & msk) * k1;
            if (armed && j < nl && th[0] == 0xFFFFFFFFu) zs = true;
            uint32_t x = (ws[j] >= th[0]) + (ws[j] >= th[1]);
            for (int t = 2; t < k1; ++t) x += ws[j] >= th[t];
            Sx[j] = (Sx[j] & clear) | (x << sh);
          }
          S0 = Sx[0];
          S1 = Sx[1];
          S2 = Sx[2];
          S3 = Sx[3];
        }
      }
      lp[0] = uint8_t(S0);
      if (nl > 1) lp[lane_ld] = uint8_t(S1);
      if (nl > 2) lp[2 * lane_ld] = uint8_t(S2);
      if (nl > 3) lp[3 * lane_ld] = uint8_t(S3);
      if (real) {
        hist8[(S0 << 8) + slot] += 1;
        if (nl > 1) hist8[(S1 << 8) + slot] += 1;
        if (nl > 2) hist8[(S2 << 8) + slot] += 1;
        if (nl > 3) hist8[(S3 << 8) + slot] += 1;
      }
    }
  }
  if (zs) atomicOr(err, int(SG_ERR_ZERO_SUPPORT));
  if (!counts) return;
  __syncthreads();
  const int warp = tid >> 5, lane_id = tid & 31;
  for (int J = warp; J < (1 << sp.bits); J += SG_THREADS / 32) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(hist8 + (J << 8));
    int sum = __dp4a(int(row[lane_id]), 0x01010101, 0);
    sum = __dp4a(int(row[lane_id + 32]), 0x01010101, sum);
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (sum && lane_id < sp.n) atomicAdd(cellacc + __ldg(jcell + J * sp.n + lane_id), uint32_t(sum));
  }
  __syncthreads();
  for (int cell = tid; cell < cells; cell += SG_THREADS)
    if (cellacc[cell]) atomicAdd(counts + cell, (unsigned long long)cellacc[cell]);
}

static size_t small_smem(const sg_small& sp, int cells) {
  return size_t((sp.tab_words * 4 + 15) & ~15) + (size_t(SG_THREADS) << sp.bits) + size_t(cells) * 4 + 16;
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

extern "C" int sg_small_prepare(const sg_small* sp, const int8_t* obs, int32_t ld_obs, int32_t cases, int32_t m,
                                int64_t case_base, uint64_t init_key, int32_t init, int32_t* scratch,
                                uint8_t* pattern, int32_t* case_id, uint8_t* lanes, int32_t lane_ld, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && obs && scratch && pattern && case_id && lanes, "sg_small_prepare: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV, "sg_small_prepare: bad plan");
  SG_REQUIRE(lane_ld >= cases && m >= 1, "sg_small_prepare: bad lane layout");
  if (cases == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int* hist = scratch;                                                  // [SMALL_PATTERNS]
  uint8_t* poc = reinterpret_cast<uint8_t*>(scratch + SMALL_PATTERNS);  // [cases]
  cudaMemsetAsync(hist, 0, sizeof(int) * SMALL_PATTERNS, s);
  const int blocks = std::min((cases + 255) / 256, 148 * 8);
  k_small_count<<<blocks, 256, 0, s>>>(*sp, obs, ld_obs, cases, poc, hist);
  k_small_scan<<<1, 32, 0, s>>>(hist);
  k_small_scatter<<<(cases + 255) / 256, 256, 0, s>>>(*sp, obs, ld_obs, cases, m, case_base, init_key, poc, hist,
                                                       pattern, case_id, lanes, lane_ld, init);
  return check_launch("sg_small_prepare");
}

extern "C" int sg_small_sweep(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                              uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                              int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                              int32_t cells, uint64_t* counts, const uint32_t* zs_flag, int32_t* err,
                              void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && stab && pattern && case_id && lanes && err, "sg_small_sweep: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV && sp->bits <= SG_SMALL_MAXBITS, "sg_small_sweep: bad plan");
  SG_REQUIRE(!counts || jcell, "sg_small_sweep: joint cell map required for the tally");
  SG_REQUIRE(m <= 252, "sg_small_sweep: m=%d exceeds 252", m);
  if (cases == 0) return SG_OK;
  const size_t smem = small_smem(*sp, cells);
  // byte counters: at most 252 lanes per thread between flushes
  const int64_t per_thread = std::max<int64_t>(1, 252 / m);
  const int64_t need = (int64_t(cases) + int64_t(SG_THREADS) * per_thread - 1) / (int64_t(SG_THREADS) * per_thread);
  const int64_t fill = (int64_t(cases) + SG_THREADS - 1) / SG_THREADS;
  int blocks = int(std::min<int64_t>(std::max<int64_t>(need, 148 * 4), fill));
  if (blocks < 1) blocks = 1;
  static size_t configured = 0;  // raise the opt-in once (keeps graph capture free of attribute calls)
  if (smem > configured) {
    cudaFuncSetAttribute(k_small_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = smem;
  }
  k_small_sweep<<<blocks, SG_THREADS, smem, (cudaStream_t)stream>>>(
      *sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real, m, case_base, key, key_dev, jcell, cells,
      reinterpret_cast<unsigned long long*>(counts), zs_flag, err);
  return check_launch("sg_small_sweep");
}

extern "C" int sg_small_import(const sg_small* sp, const sg_batch* batch, const int32_t* case_id, uint8_t* lanes,
                               int32_t lane_ld, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && batch && case_id && lanes, "sg_small_import: null argument");
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
