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
  uint32_t* out = reinterpret_cast<uint32_t*>(lanes);
  for (int q = 0; q < (m + 3) / 4; ++q) {
    uint32_t S[4] = {obsw, obsw, obsw, obsw};
    for (int v = 0; v < sp.n; ++v) {
      if (!((P >> v) & 1u)) continue;
      const u32x4 w = fast_block(init_key, uint64_t(case_base + c), uint32_t(v), uint32_t(q), 1u);
      const uint32_t ws[4] = {w.a, w.b, w.c, w.d};
#pragma unroll
      for (int j = 0; j < 4; ++j) S[j] |= uint32_t((uint64_t(ws[j]) * uint32_t(sp.card[v])) >> 32) << sp.off[v];
    }
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) word |= (q * 4 + j < m ? (S[j] & 0xFFu) : 0u) << (8 * j);
    out[int64_t(q) * lane_ld + s] = word;
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

// u >= t as 0/1 for 31-bit u and thresholds t <= 2^31 (sentinel 0xFFFFFFFF never passes).
__device__ __forceinline__ uint32_t ge(uint32_t u, uint32_t t) { return u >= t ? 1u : 0u; }

// Per-thread constants of the sweep (the variable loop is unrolled over N
// colour-ordered positions, every per-variable constant in registers).
template <int N>
struct SmallCtx {
  int VAR[N], SH[N], K1[N];
  uint32_t MSK[N], CLR[N];
  const uint32_t* TV[N];
  uint32_t* row;
  const uint8_t* pattern;
  const int32_t* case_id;
  uint8_t* hist8;
  int cases, num_real, q, nl, slot;
  uint32_t valid4;
  int64_t case_base;
  uint64_t key;
  bool counts;
};

// Walk this thread's (slot, quad) units.  ARMED: some table entry has no
// support, so every draw checks for the sentinel (the reference raises
// ZeroSupport only when a lane actually hits such a configuration).
template <int N, bool ARMED>
__device__ __forceinline__ bool small_units(const SmallCtx<N>& x) {
  const int stride = gridDim.x * SG_THREADS;
  bool zs = false;
  int s = blockIdx.x * SG_THREADS + threadIdx.x;
  uint32_t nw = 0, nP = 0;
  int nc = 0;
  if (s < x.cases) {
    nw = x.row[s];
    nP = x.pattern[s];
    nc = x.case_id[s];
  }
  for (; s < x.cases; s += stride) {
    uint32_t w = nw;
    const uint32_t P = nP;
    const int c = nc;
    const int sn = s + stride;
    if (sn < x.cases) {  // prefetch the next unit while this one computes
      nw = x.row[sn];
      nP = x.pattern[sn];
      nc = x.case_id[sn];
    }
    const uint64_t gc = uint64_t(x.case_base + c);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (!((P >> x.VAR[i]) & 1u)) continue;  // warp-uniform: slots are bucketed by pattern
      const u32x4 r = fast_block(x.key, gc, uint32_t(x.VAR[i]), uint32_t(x.q), 0u);
      const uint32_t u[4] = {r.a >> 1, r.b >> 1, r.c >> 1, r.d >> 1};
      const uint32_t wm = w & x.MSK[i];
      uint32_t xs[4];
      if (x.K1[i] == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t t = x.TV[i][byte_of(wm, j)];
          if (ARMED && j < x.nl && t == 0xFFFFFFFFu) zs = true;
          xs[j] = ge(u[j], t);
        }
      } else if (x.K1[i] == 2) {
        const uint2* t2 = reinterpret_cast<const uint2*>(x.TV[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint2 t = t2[byte_of(wm, j)];
          if (ARMED && j < x.nl && t.x == 0xFFFFFFFFu) zs = true;
          xs[j] = ge(u[j], t.x) + ge(u[j], t.y);
        }
      } else {
        const uint4* t4 = reinterpret_cast<const uint4*>(x.TV[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 t = t4[byte_of(wm, j)];  // card 4: three thresholds + padding
          if (ARMED && j < x.nl && t.x == 0xFFFFFFFFu) zs = true;
          xs[j] = ge(u[j], t.x) + ge(u[j], t.y) + ge(u[j], t.z);
        }
      }
      const uint32_t x4 = xs[0] | (xs[1] << 8) | (xs[2] << 16) | (xs[3] << 24);
      w = (w & x.CLR[i]) | (x4 << x.SH[i]);
    }
    w &= x.valid4;
    x.row[s] = w;
    if (x.counts && c < x.num_real) {
      if (x.nl == 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) x.hist8[(byte_of(w, j) << 8) + x.slot] += 1;
      } else {
        for (int j = 0; j < x.nl; ++j) x.hist8[(byte_of(w, j) << 8) + x.slot] += 1;
      }
    }
  }
  return zs;
}

// The sweep.  Grid (x: slots, y: replica quad q).  A thread owns lane word
// (q, s); per latent variable one Philox4x32 call gives the quad's 4
// uniforms, each lane does one table lookup and compare, and the 4 new
// states are inserted with one byte-SIMD mask/or.
template <int N, bool FUSE>
__global__ void __launch_bounds__(SG_THREADS, 4)
k_small_sweep(const sg_small sp, const uint32_t* __restrict__ stab_g, const uint8_t* __restrict__ pattern,
              const int32_t* __restrict__ case_id, uint32_t* __restrict__ lanes, int lane_ld, int cases, int num_real,
              int m, int64_t case_base, uint64_t key, const uint64_t* __restrict__ key_dev,
              const int32_t* __restrict__ jcell, int cells, unsigned long long* __restrict__ counts,
              const uint32_t* __restrict__ zs_flag, const int8_t* __restrict__ obs, int ld_obs, int32_t* err,
              const sg_net fnet, const FinishArgs fin, unsigned int* done) {
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
  SmallCtx<N> x;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const int v = sp.order[i];
    x.VAR[i] = v;
    x.SH[i] = sp.off[v];
    x.K1[i] = sp.card[v] - 1;
    x.MSK[i] = sp.mbmask[v] * 0x01010101u;
    x.CLR[i] = ~((((1u << sp.width[v]) - 1u) << sp.off[v]) * 0x01010101u);
    x.TV[i] = stab + sp.toff[v];
  }
  x.q = blockIdx.y;
  x.nl = min(4, m - 4 * x.q);  // real replicas in this quad
  x.valid4 = x.nl >= 4 ? 0xFFFFFFFFu : ((1u << (8 * x.nl)) - 1u);
  x.row = lanes + int64_t(x.q) * lane_ld;
  x.pattern = pattern;
  x.case_id = case_id;
  x.hist8 = hist8;
  x.cases = cases;
  x.num_real = num_real;
  x.slot = ((tid & 31) << 2) | ((tid >> 5) & 3) | ((tid >> 7) << 7);
  x.case_base = case_base;
  x.key = key_dev ? __ldg(key_dev) : key;
  x.counts = counts != nullptr;
  __syncthreads();
  const bool zs = armed ? small_units<N, true>(x) : small_units<N, false>(x);
  if (zs) atomicOr(err, int(SG_ERR_ZERO_SUPPORT));
  if (obs) {  // the minibatch's range check (sampler.py:429-430), spread over the whole grid
    const int chunks = (cases + 15) >> 4;
    const int gtid = (blockIdx.y * gridDim.x + blockIdx.x) * SG_THREADS + tid;
    const int gthreads = gridDim.x * gridDim.y * SG_THREADS;
    unsigned bad = 0;
    for (int i = gtid; i < N * chunks; i += gthreads) {
      const int v = i / chunks, ch = i - v * chunks;
      const uint32_t lim = 0x01010101u * uint32_t(sp.card[v] - 1);
      const int4 qv = __ldcs(reinterpret_cast<const int4*>(obs + int64_t(v) * ld_obs + ch * 16));
      const uint32_t wv[4] = {uint32_t(qv.x), uint32_t(qv.y), uint32_t(qv.z), uint32_t(qv.w)};
      const int left = cases - ch * 16;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t gt = __vcmpgts4(wv[k], lim);
        const int valid = left - 4 * k;
        if (valid < 4) gt &= valid <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - valid)));
        bad |= gt;
      }
    }
    if (bad) atomicOr(err, int(SG_ERR_STATE_RANGE));
  }
  if (!counts) return;
  __syncthreads();
  const int warp = tid >> 5, lane_id = tid & 31;
  for (int J = warp; J < (1 << sp.bits); J += SG_THREADS / 32) {
    const uint32_t* hrow = reinterpret_cast<const uint32_t*>(hist8 + (J << 8));
    int sum = __dp4a(int(hrow[lane_id]), 0x01010101, 0);
    sum = __dp4a(int(hrow[lane_id + 32]), 0x01010101, sum);
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (sum && lane_id < sp.n) atomicAdd(cellacc + __ldg(jcell + J * sp.n + lane_id), uint32_t(sum));
  }
  __syncthreads();
  for (int cell = tid; cell < cells; cell += SG_THREADS)
    if (cellacc[cell]) atomicAdd(counts + cell, (unsigned long long)cellacc[cell]);
  if (FUSE) {
    // the last CTA to finish runs the step tail on the complete counts
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) *done = 0u;  // re-armed for the next launch
    step_finish_body(fnet, fin, smem, SG_THREADS);
  }
}

// Resident CTAs of one sweep instance on the whole device (one full wave).
template <int N, bool FUSE>
static int resident_ctas(size_t smem) {
  static size_t cached_smem = ~size_t(0);
  static int cached = 0;
  if (smem != cached_smem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small_sweep<N, FUSE>, SG_THREADS, smem);
    cached = sms * std::max(1, per_sm);
    cached_smem = smem;
  }
  return cached;
}

// One wave of CTAs split over the Q replica quads (every CTA strides over the
// pattern-sorted slots, so the units' cost is balanced across CTAs), but at
// least enough CTAs that no thread's byte counters see more than 63 units.
template <int N, bool FUSE>
static dim3 small_grid(int cases, int Q, size_t smem) {
  const int64_t need = (int64_t(cases) + int64_t(SG_THREADS) * 63 - 1) / (int64_t(SG_THREADS) * 63);
  const int64_t fill = (int64_t(cases) + SG_THREADS - 1) / SG_THREADS;
  const int64_t want = std::max<int64_t>(resident_ctas<N, FUSE>(smem) / Q, need);
  return dim3(unsigned(std::max<int64_t>(1, std::min<int64_t>(want, fill))), unsigned(Q));
}

template <int N, bool FUSE>
static void launch_small(const sg_small& sp, int Q, size_t smem, cudaStream_t st, const uint32_t* stab,
                         const uint8_t* pattern, const int32_t* case_id, uint32_t* lanes, int lane_ld, int cases,
                         int num_real, int m, int64_t case_base, uint64_t key, const uint64_t* key_dev,
                         const int32_t* jcell, int cells, uint64_t* counts, const uint32_t* zs_flag,
                         const int8_t* obs, int ld_obs, int32_t* err, const sg_net& fnet, const FinishArgs& fin,
                         unsigned int* done) {
  static size_t configured = 0;  // raise the opt-in once (keeps graph capture free of attribute calls)
  if (smem > configured) {
    cudaFuncSetAttribute(k_small_sweep<N, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = smem;
  }
  const dim3 grid = small_grid<N, FUSE>(cases, Q, smem);
  k_small_sweep<N, FUSE><<<grid, SG_THREADS, smem, st>>>(sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real,
                                                         m, case_base, key, key_dev, jcell, cells,
                                                         reinterpret_cast<unsigned long long*>(counts), zs_flag, obs,
                                                         ld_obs, err, fnet, fin, done);
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

static bool lane_ld_ok(int lane_ld, int cases) { return lane_ld >= cases && lane_ld % 4 == 0; }

extern "C" int sg_small_prepare(const sg_small* sp, const int8_t* obs, int32_t ld_obs, int32_t cases, int32_t m,
                                int64_t case_base, uint64_t init_key, int32_t init, int32_t* scratch,
                                uint8_t* pattern, int32_t* case_id, uint8_t* lanes, int32_t lane_ld, void* stream) {
  using namespace sg;
  SG_REQUIRE(sp && obs && scratch && pattern && case_id && lanes, "sg_small_prepare: null argument");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV, "sg_small_prepare: bad plan");
  SG_REQUIRE(m >= 1 && lane_ld_ok(lane_ld, cases), "sg_small_prepare: lane_ld %d < cases %d", lane_ld, cases);
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

namespace sg {
template <bool FUSE>
static int small_sweep_impl(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                            uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                            int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                            int32_t cells, uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs,
                            int32_t ld_obs, int32_t* err, void* stream, const sg_net* fnet, const sg_finish* f,
                            uint32_t* done) {
  SG_REQUIRE(sp && stab && pattern && case_id && lanes && err, "sg_small_sweep: null argument");
  if (obs)
    SG_REQUIRE(ld_obs % 16 == 0 && (reinterpret_cast<uintptr_t>(obs) & 15) == 0 && ld_obs >= cases,
               "sg_small_sweep: obs rows must be 16-byte aligned");
  SG_REQUIRE(sp->n >= 1 && sp->n <= SG_SMALL_MAXV && sp->bits <= SG_SMALL_MAXBITS, "sg_small_sweep: bad plan");
  SG_REQUIRE(!counts || jcell, "sg_small_sweep: joint cell map required for the tally");
  SG_REQUIRE(m >= 1 && lane_ld_ok(lane_ld, cases), "sg_small_sweep: lane_ld %d < cases %d", lane_ld, cases);
  for (int v = 0; v < sp->n; ++v)
    SG_REQUIRE(sp->card[v] <= 4 && sp->tstride[v] >= sp->card[v] - 1 && sp->toff[v] % sp->tstride[v] == 0,
               "sg_small_sweep: variable %d needs card <= 4 and an aligned table", v);
  if (FUSE) {
    SG_REQUIRE(fnet && f && done && counts, "sg_small_step: network, finish args, counter and counts required");
    if (cases == 0 || !finish_fits(*fnet, sp)) {  // nothing to sweep / model too large to fuse: two launches
      const int st = small_sweep_impl<false>(sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real, m,
                                             case_base, key, key_dev, jcell, cells, counts, zs_flag, obs, ld_obs,
                                             err, stream, nullptr, nullptr, nullptr);
      return st ? st : sg_step_finish(fnet, sp, f, stream);
    }
  }
  if (cases == 0) return SG_OK;
  size_t smem = small_smem(*sp, cells);
  FinishArgs fin{};
  sg_net fn{};
  if (FUSE) {
    fin = make_finish_args(f, sp);
    fn = *fnet;
    smem = std::max(smem, finish_smem(*fnet));
  }
  const int Q = (m + 3) / 4;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* lw = reinterpret_cast<uint32_t*>(lanes);
#define SG_SMALL_CASE(NV)                                                                                     \
  case NV:                                                                                                    \
    launch_small<NV, FUSE>(*sp, Q, smem, st, stab, pattern, case_id, lw, lane_ld, cases, num_real, m, case_base, \
                     key, key_dev, jcell, cells, counts, zs_flag, obs, ld_obs, err, fn, fin, done);           \
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
  return check_launch(FUSE ? "sg_small_step" : "sg_small_sweep");
}
}  // namespace sg

extern "C" int sg_small_sweep(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                              uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                              int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                              int32_t cells, uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs,
                              int32_t ld_obs, int32_t* err, void* stream) {
  return sg::small_sweep_impl<false>(sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real, m, case_base, key,
                                     key_dev, jcell, cells, counts, zs_flag, obs, ld_obs, err, stream, nullptr, nullptr,
                                     nullptr);
}

extern "C" int sg_small_step(const sg_small* sp, const uint32_t* stab, const uint8_t* pattern, const int32_t* case_id,
                             uint8_t* lanes, int32_t lane_ld, int32_t cases, int32_t num_real, int32_t m,
                             int64_t case_base, uint64_t key, const uint64_t* key_dev, const int32_t* jcell,
                             int32_t cells, uint64_t* counts, const uint32_t* zs_flag, const int8_t* obs,
                             int32_t ld_obs, int32_t* err, const sg_net* net, const sg_finish* f, uint32_t* done,
                             void* stream) {
  return sg::small_sweep_impl<true>(sp, stab, pattern, case_id, lanes, lane_ld, cases, num_real, m, case_base, key,
                                    key_dev, jcell, cells, counts, zs_flag, obs, ld_obs, err, stream, net, f, done);
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
