// Minibatch staging on the device: latent ranks, lane replication and the
// initial latent draws.
//
// Reference: replicate_minibatch (sampler.py:174-187) tiles the observed
// block m times and lists, per variable, the latent lanes in ascending lane
// order; init_latent (sampler.py:205-214) fills them with
// substream(seed, "latent_init", pass, mb, v).integers(0, card).  The order of
// that list fixes which uniform each latent cell consumes, so the device keeps
// rank[v][c] = position of case c among v's latent cases; lane (r, c) is then
// draw r * nmiss[v] + rank[v][c] of v's stream.
#include "sg_device.cuh"

namespace sg {

static constexpr int RANK_CASES = 4096;  // cases per rank block (256 threads x 16)

__device__ __forceinline__ int latent_bits16(const int8_t* p) {
  const int4 q = *reinterpret_cast<const int4*>(p);
  const uint32_t w[4] = {uint32_t(q.x), uint32_t(q.y), uint32_t(q.z), uint32_t(q.w)};
  int bits = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int b = 0; b < 4; ++b) bits |= int((w[i] >> (8 * b + 7)) & 1u) << (4 * i + b);
  }
  return bits;
}

// Per (block of 4096 cases, variable): latent count.
__global__ void __launch_bounds__(256) k_rank_count(const int8_t* __restrict__ obs, int ld, int cases,
                                                    int64_t* __restrict__ blk, int nblk) {
  const int v = blockIdx.y, b = blockIdx.x;
  const int c = b * RANK_CASES + threadIdx.x * 16;
  int cnt = 0;
  if (c < cases) {
    int bits = latent_bits16(obs + int64_t(v) * ld + c);
    if (cases - c < 16) bits &= (1 << (cases - c)) - 1;
    cnt = __popc(bits);
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int i = 0; i < 8; ++i) s += ws[i];
    blk[int64_t(v) * nblk + b] = s;
  }
}

// Exclusive scan of block counts per variable (one warp per variable).
__global__ void k_rank_scan(int64_t* __restrict__ blk, int nblk, int64_t* __restrict__ nmiss) {
  const int v = blockIdx.x;
  const int lane = threadIdx.x;
  int64_t carry = 0;
  for (int b0 = 0; b0 < nblk; b0 += 32) {
    const int b = b0 + lane;
    const int64_t x = b < nblk ? blk[int64_t(v) * nblk + b] : 0;
    int64_t inc = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (b < nblk) blk[int64_t(v) * nblk + b] = carry + inc - x;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) nmiss[v] = carry;
}

__global__ void __launch_bounds__(256) k_rank_write(const int8_t* __restrict__ obs, int ld, int cases,
                                                    const int64_t* __restrict__ blk, int nblk,
                                                    int32_t* __restrict__ rank, int ld_rank) {
  const int v = blockIdx.y, b = blockIdx.x;
  const int c = b * RANK_CASES + threadIdx.x * 16;
  int bits = 0;
  if (c < cases) {
    bits = latent_bits16(obs + int64_t(v) * ld + c);
    if (cases - c < 16) bits &= (1 << (cases - c)) - 1;
  }
  const int cnt = __popc(bits);
  // block exclusive scan of cnt
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __shared__ int ws[8];
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  int wbase = 0;
  for (int i = 0; i < warp; ++i) wbase += ws[i];
  int run = int(blk[int64_t(v) * nblk + b]) + wbase + inc - cnt;
  if (c < cases) {
    const int lim = min(16, cases - c);
    int32_t* out = rank + int64_t(v) * ld_rank + c;
    for (int i = 0; i < lim; ++i) {
      out[i] = run;
      run += (bits >> i) & 1;
    }
  }
}

// Lemire rejection scan for numpy's integers(0, card, dtype=int32): word j of
// v's 32-bit stream is skipped iff (w_j * card mod 2^32) < (2^32 - card) % card.
// Records the skipped positions among the first m*nmiss + SLACK words.
__global__ void __launch_bounds__(256) k_lemire_scan(const sg_net net, int m, const int64_t* __restrict__ nmiss,
                                                     const uint64_t* __restrict__ keys,
                                                     int64_t* __restrict__ rej, int32_t* err) {
  const int v = blockIdx.y;
  const uint32_t card = uint32_t(__ldg(net.card + v));
  const uint32_t thr = uint32_t((0x100000000ull - card) % card);
  if (thr == 0) return;
  const int64_t words = int64_t(m) * nmiss[v] + SG_REJ_SLACK;
  const uint64_t k0 = keys[2 * v], k1 = keys[2 * v + 1];
  int64_t* cnt = rej + int64_t(v) * (SG_REJ_SLACK + 2);
  int64_t* pos = cnt + 1;
  // one Philox4x64 block = 8 words
  const int64_t blocks = (words + 7) / 8;
  for (int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b < blocks;
       b += int64_t(gridDim.x) * blockDim.x) {
    const u64x4 w = philox4x64_10(u64x4{uint64_t(b) + 1ull, 0, 0, 0}, k0, k1);
    const uint64_t ws[4] = {w.a, w.b, w.c, w.d};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t j = b * 8 + i;
      const uint32_t x = (i & 1) ? uint32_t(ws[i >> 1] >> 32) : uint32_t(ws[i >> 1]);
      if (j < words && uint32_t(uint64_t(x) * card) < thr) {
        const long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(cnt), 1ull);
        if (slot < SG_REJ_SLACK) pos[slot] = j;
        else atomicOr(err, int(SG_ERR_REJECT_OVERFLOW));
      }
    }
  }
}

__global__ void k_lemire_sort(int n, int64_t* rej) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t* cnt = rej + int64_t(v) * (SG_REJ_SLACK + 2);
  const int k = int(min(cnt[0], int64_t(SG_REJ_SLACK)));
  int64_t* p = cnt + 1;
  for (int i = 1; i < k; ++i) {
    const int64_t x = p[i];
    int j = i - 1;
    while (j >= 0 && p[j] > x) {
      p[j + 1] = p[j];
      --j;
    }
    p[j + 1] = x;
  }
}

// Build lane states for every (v, r, c < pitch): observed state, or latent
// flag | initial draw; cases >= `cases` are inert (state 0, never sampled).
template <int MODE>
__global__ void __launch_bounds__(256) k_init_states(const sg_net net, const sg_batch bt,
                                                     const int8_t* __restrict__ obs, int ld_obs,
                                                     uint64_t fast_key, const uint64_t* __restrict__ keys,
                                                     const int64_t* __restrict__ rej, int32_t* err) {
  const int v = blockIdx.y;
  const int m = bt.m;
  const int card = __ldg(net.card + v);
  const int64_t total = int64_t(m) * bt.pitch;
  uint64_t k0 = 0, k1 = 0;
  int64_t nmiss = 0;
  int nrej = 0;
  const int64_t* rpos = nullptr;
  if (MODE == SG_RNG_NUMPY) {
    k0 = keys[2 * v];
    k1 = keys[2 * v + 1];
    nmiss = bt.nmiss[v];
    const int64_t* cnt = rej + int64_t(v) * (SG_REJ_SLACK + 2);
    nrej = int(min(cnt[0], int64_t(SG_REJ_SLACK)));
    rpos = cnt + 1;
  }
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / bt.pitch);
    const int c = int(i - int64_t(r) * bt.pitch);
    int8_t out = 0;
    if (c < bt.cases) {
      const int o = obs[int64_t(v) * ld_obs + c];
      if (o >= 0) {
        // an out-of-range observation never becomes an index: state 0 + error bit
        out = o < card ? int8_t(o) : int8_t(0);
        bad |= o >= card;
      } else if (MODE == SG_RNG_FAST) {
        const uint32_t w = pick(fast_block(fast_key, uint64_t(bt.case_base + c), uint32_t(v), uint32_t(r >> 2), 1u), r & 3);
        out = int8_t(0x80 | int((uint64_t(w) * uint32_t(card)) >> 32));
      } else {
        const int64_t k = int64_t(r) * nmiss + bt.rank[int64_t(v) * bt.ld_rank + c];
        int j = 0;
        while (j < nrej && rpos[j] <= k + j) ++j;
        const uint32_t x = np_word32(uint64_t(k + j), k0, k1);
        out = int8_t(0x80 | int((uint64_t(x) * uint32_t(card)) >> 32));
      }
    }
    bt.states[(int64_t(v) * m + r) * bt.pitch + c] = out;
  }
  if (bad) atomicOr(err, int(SG_ERR_STATE_RANGE));
}

__global__ void __launch_bounds__(256) k_check_range(const sg_net net, const int8_t* __restrict__ obs, int ld,
                                                     int cases, int32_t* err) {
  // 16 cases per thread-load; bytes compared as signed SIMD lanes against card-1
  const int v = blockIdx.y;
  const uint32_t lim = 0x01010101u * uint32_t(__ldg(net.card + v) - 1);
  const int chunks = (cases + 15) >> 4;
  unsigned bad = 0;
  for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < chunks; ch += gridDim.x * blockDim.x) {
    const int4 q = __ldcs(reinterpret_cast<const int4*>(obs + int64_t(v) * ld + ch * 16));
    uint32_t w[4] = {uint32_t(q.x), uint32_t(q.y), uint32_t(q.z), uint32_t(q.w)};
    const int left = cases - ch * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t gt = __vcmpgts4(w[i], lim);  // 0xFF in every byte holding a state > card-1
      const int valid = left - 4 * i;
      if (valid < 4) gt &= valid <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - valid)));
      bad |= gt;
    }
  }
  if (bad) atomicOr(err, int(SG_ERR_STATE_RANGE));
}

}  // namespace sg

extern "C" int sg_rank_latent(int32_t n, const int8_t* obs, int32_t ld_obs, int32_t cases, int32_t* rank,
                              int32_t ld_rank, int64_t* nmiss, int64_t* scratch, void* stream) {
  using namespace sg;
  SG_REQUIRE(obs && nmiss && scratch, "sg_rank_latent: null argument");
  SG_REQUIRE(ld_obs % 16 == 0 && ld_obs >= cases && (!rank || ld_rank >= cases), "sg_rank_latent: bad pitch");
  SG_REQUIRE(n > 0 && n < 65536, "sg_rank_latent: bad n");
  cudaStream_t s = (cudaStream_t)stream;
  if (cases == 0) {
    cudaMemsetAsync(nmiss, 0, sizeof(int64_t) * n, s);
    return check_launch("sg_rank_latent");
  }
  const int nblk = (cases + RANK_CASES - 1) / RANK_CASES;
  k_rank_count<<<dim3(nblk, n), 256, 0, s>>>(obs, ld_obs, cases, scratch, nblk);
  k_rank_scan<<<n, 32, 0, s>>>(scratch, nblk, nmiss);
  if (rank) k_rank_write<<<dim3(nblk, n), 256, 0, s>>>(obs, ld_obs, cases, scratch, nblk, rank, ld_rank);
  return check_launch("sg_rank_latent");
}

extern "C" int sg_init_states(const sg_net* net, const sg_batch* batch, const int8_t* obs, int32_t ld_obs,
                              int32_t rng_mode, uint64_t fast_key, const uint64_t* keys,
                              int64_t* rej_scratch, int32_t* err, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && batch && obs && err && batch->states, "sg_init_states: null argument");
  SG_REQUIRE(batch->pitch % 16 == 0 && batch->pitch >= batch->cases && ld_obs >= batch->cases,
             "sg_init_states: bad pitch");
  SG_REQUIRE(rng_mode == SG_RNG_FAST || rng_mode == SG_RNG_NUMPY, "sg_init_states: bad rng mode %d",
             rng_mode);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t per_var = int64_t(batch->m) * batch->pitch;
  const int gx = int(std::min<int64_t>((per_var + 255) / 256, 1024));
  if (rng_mode == SG_RNG_FAST) {
    SG_REQUIRE(fast_cases_ok(batch->case_base, batch->cases) && batch->m <= 4 * 4096,
               "sg_init_states: FAST counters need global cases < 2^32 and m <= 16384");
    k_init_states<SG_RNG_FAST><<<dim3(gx, net->n), 256, 0, s>>>(*net, *batch, obs, ld_obs, fast_key, nullptr,
                                                                nullptr, err);
  } else {
    SG_REQUIRE(keys && rej_scratch && batch->rank && batch->nmiss, "sg_init_states: numpy mode needs keys, "
               "rank, nmiss and rej_scratch");
    cudaMemsetAsync(rej_scratch, 0, sizeof(int64_t) * net->n * (SG_REJ_SLACK + 2), s);
    k_lemire_scan<<<dim3(64, net->n), 256, 0, s>>>(*net, batch->m, batch->nmiss, keys, rej_scratch, err);
    k_lemire_sort<<<(net->n + 127) / 128, 128, 0, s>>>(net->n, rej_scratch);
    k_init_states<SG_RNG_NUMPY><<<dim3(gx, net->n), 256, 0, s>>>(*net, *batch, obs, ld_obs, 0, keys,
                                                                 rej_scratch, err);
  }
  return check_launch("sg_init_states");
}

extern "C" int sg_check_range(const sg_net* net, const int8_t* obs, int32_t ld_obs, int32_t cases, int32_t* err,
                              void* stream) {
  using namespace sg;
  SG_REQUIRE(net && obs && err, "sg_check_range: null argument");
  SG_REQUIRE(ld_obs % 16 == 0 && (reinterpret_cast<uintptr_t>(obs) & 15) == 0 && ld_obs >= cases,
             "sg_check_range: obs rows must be 16-byte aligned");
  if (cases == 0) return SG_OK;
  const int chunks = (cases + 15) / 16;
  const int gx = std::min((chunks + 255) / 256, 1024);
  k_check_range<<<dim3(gx, net->n), 256, 0, (cudaStream_t)stream>>>(*net, obs, ld_obs, cases, err);
  return check_launch("sg_check_range");
}
