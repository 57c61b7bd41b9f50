// Site keys on the device and the predict_missing frequency tally.
//
// Site keys.  Every random stream of the reference is keyed by
// blake2b-128("{seed}:{label}:{i0}:...") read as two little-endian uint64
// words (rng.py:16-20).  The numpy-parity sweep needs one such key per
// variable per sweep: stream_key(sweep_seed, "var", v) (sampler.py:245).
// Hashing them in host Python costs microseconds per key (n = 1000: ms per
// sweep) and keeps the numpy path out of CUDA graphs; here one thread per
// variable formats its site text and runs the single-block BLAKE2b
// compression (RFC 7693; every site text is < 128 bytes), with the seed word
// read from device memory when it is itself device-resident (the step
// graphs' key cursor).
//
// predict_missing (metrics.py:89-139) adds 1.0 to freq[t, state] of every
// target after each kept sweep (np.add.at); integer counts divided by
// num_samples give the same fp64 frequencies.
#include "sg_device.cuh"

namespace sg {

__host__ __device__ __forceinline__ uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

#define SG_B2_G(a, b, c, d, x, y) \
  do {                            \
    a = a + b + (x);              \
    d = rotr64(d ^ a, 32);        \
    c = c + d;                    \
    b = rotr64(b ^ c, 24);        \
    a = a + b + (y);              \
    d = rotr64(d ^ a, 16);        \
    c = c + d;                    \
    b = rotr64(b ^ c, 63);        \
  } while (0)

// BLAKE2b-128 of one message of len <= 128 bytes (unkeyed), digest words out[0..1].
__host__ __device__ inline void blake2b128_1block(const unsigned char* msg, int len, uint64_t out[2]) {
  const uint64_t IV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                          0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                          0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
  const unsigned char SIGMA[12][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
  uint64_t m[16];
  for (int i = 0; i < 16; ++i) {
    uint64_t w = 0;
    for (int b = 0; b < 8; ++b) {
      const int k = 8 * i + b;
      w |= uint64_t(k < len ? msg[k] : 0u) << (8 * b);
    }
    m[i] = w;
  }
  uint64_t h[8];
  for (int i = 0; i < 8; ++i) h[i] = IV[i];
  h[0] ^= 0x01010000ull ^ 16ull;  // depth 1, fanout 1, no key, 16-byte digest
  uint64_t v[16];
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = IV[i];
  }
  v[12] ^= uint64_t(len);  // byte counter (t0); t1 = 0
  v[14] = ~v[14];          // final block
#pragma unroll
  for (int r = 0; r < 12; ++r) {
    const unsigned char* s = SIGMA[r];
    SG_B2_G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
    SG_B2_G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
    SG_B2_G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
    SG_B2_G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
    SG_B2_G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
    SG_B2_G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
    SG_B2_G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
    SG_B2_G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
  }
  out[0] = h[0] ^ v[0] ^ v[8];
  out[1] = h[1] ^ v[1] ^ v[9];
}

// Decimal digits of x appended at buf[pos]; returns the new length.
__host__ __device__ inline int put_decimal(unsigned char* buf, int pos, uint64_t x) {
  unsigned char tmp[20];
  int k = 0;
  do {
    tmp[k++] = (unsigned char)('0' + x % 10u);
    x /= 10u;
  } while (x);
  while (k) buf[pos++] = tmp[--k];
  return pos;
}

struct SiteText {
  unsigned char text[SG_SITE_TEXT_MAX];
  int32_t len;
};

// keys[i] = blake2b128( [dec(*seed_dev) ":"-joined with] prefix + dec(first + i) )
__global__ void k_site_keys(const SiteText pre, const uint64_t* __restrict__ seed_dev, int64_t first, int32_t count,
                            uint64_t* __restrict__ keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned char buf[128];
  int len = 0;
  if (seed_dev) len = put_decimal(buf, 0, *seed_dev);
  for (int k = 0; k < pre.len; ++k) buf[len++] = pre.text[k];
  len = put_decimal(buf, len, uint64_t(first + i));
  uint64_t out[2];
  blake2b128_1block(buf, len, out);
  keys[2 * int64_t(i)] = out[0];
  keys[2 * int64_t(i) + 1] = out[1];
}

__global__ void k_predict_tally(const int8_t* __restrict__ states, int64_t var_stride,
                                const int32_t* __restrict__ t_var, const int32_t* __restrict__ t_case, int32_t targets,
                                int32_t max_card, int64_t* __restrict__ freq, int32_t* err) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= targets) return;
  const int s = states[int64_t(t_var[t]) * var_stride + t_case[t]] & 0x7F;
  if (s < max_card) {
    freq[int64_t(t) * max_card + s] += 1;
  } else {
    atomicOr(err, int(SG_ERR_STATE_RANGE));
  }
}

}  // namespace sg

extern "C" int sg_site_keys(const uint64_t* seed_dev, const char* prefix, int32_t prefix_len, int64_t first,
                            int32_t count, uint64_t* keys, void* stream) {
  using namespace sg;
  SG_REQUIRE(keys && prefix_len >= 0 && prefix_len <= SG_SITE_TEXT_MAX && count >= 0 && first >= 0 &&
                 (prefix || prefix_len == 0),
             "sg_site_keys: bad argument");
  // 20 seed digits + prefix + 19 index digits must fit one 128-byte block
  SG_REQUIRE((seed_dev ? 20 : 0) + prefix_len + 19 <= 128, "sg_site_keys: site text longer than one block");
  if (count == 0) return SG_OK;
  SiteText pre;
  for (int k = 0; k < prefix_len; ++k) pre.text[k] = (unsigned char)prefix[k];
  pre.len = prefix_len;
  k_site_keys<<<(count + 127) / 128, 128, 0, (cudaStream_t)stream>>>(pre, seed_dev, first, count, keys);
  return check_launch("sg_site_keys");
}

// Host evaluation of the same code (tests pin it to hashlib.blake2b without a GPU).
// numpy-stream uniforms of one sweep, generated ahead of it (the numpy-parity
// sweep then runs in injected mode).  Variable v's stream is numpy's
// Philox4x64-10 under stream_key(sweep_seed, "var", v) (sampler.py:245,
// rng.py:16-25): its 64-bit word i is word i % 4 of the block at counter
// i / 4 + 1, and random() is (word >> 11) * 2^-53.  The sweep consumes words
// 0 .. m * nmiss[v] - 1 (index r * nmiss[v] + rank, sampler.py:245), i.e.
// every word of every block: one thread per block writes four uniforms,
// where the in-sweep draw computes a whole block per uniform.
namespace sg {
__global__ void __launch_bounds__(256) k_np_uniforms(const int64_t* __restrict__ nmiss,
                                                     const uint64_t* __restrict__ keys, int m, double* __restrict__ out,
                                                     int64_t ld) {
  const int v = blockIdx.y;
  const int64_t want = int64_t(m) * __ldg(nmiss + v);
  SG_DCHECK(want <= ld);
  const int64_t total = want < ld ? want : ld;  // never past the row (the host sizes ld >= m * nmiss)
  const uint64_t k0 = __ldg(keys + 2 * v), k1 = __ldg(keys + 2 * v + 1);
  double* o = out + int64_t(v) * ld;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; 4 * j < total;
       j += int64_t(gridDim.x) * blockDim.x) {
    const u64x4 w = philox4x64_10(u64x4{uint64_t(j) + 1ull, 0ull, 0ull, 0ull}, k0, k1);
    const double u0 = double(w.a >> 11) * 0x1.0p-53, u1 = double(w.b >> 11) * 0x1.0p-53;
    const double u2 = double(w.c >> 11) * 0x1.0p-53, u3 = double(w.d >> 11) * 0x1.0p-53;
    SG_DCHECK(4 * j < ld);
    if (4 * j + 4 <= total) {
      reinterpret_cast<double2*>(o + 4 * j)[0] = make_double2(u0, u1);
      reinterpret_cast<double2*>(o + 4 * j)[1] = make_double2(u2, u3);
    } else {
      o[4 * j] = u0;
      if (4 * j + 1 < total) o[4 * j + 1] = u1;
      if (4 * j + 2 < total) o[4 * j + 2] = u2;
    }
  }
}
}  // namespace sg

extern "C" int sg_np_uniforms(const sg_batch* batch, const uint64_t* keys, int32_t n, double* out, int64_t ld,
                              void* stream) {
  using namespace sg;
  SG_REQUIRE(batch && keys && out && n >= 1 && n <= 65535, "sg_np_uniforms: bad argument");
  SG_REQUIRE(ld % 4 == 0 && ld >= int64_t(batch->m) * batch->cases && (reinterpret_cast<uintptr_t>(out) & 31) == 0,
             "sg_np_uniforms: ld %lld must be a multiple of 4 and >= m * cases, out 32-byte aligned", (long long)ld);
  const int64_t blocks = (int64_t(batch->m) * batch->cases + 3) / 4;
  const int64_t ctas = (blocks + 255) / 256;
  const dim3 grid(unsigned(ctas < 2048 ? (ctas > 0 ? ctas : 1) : 2048), unsigned(n));
  k_np_uniforms<<<grid, 256, 0, (cudaStream_t)stream>>>(batch->nmiss, keys, batch->m, out, ld);
  return check_launch("sg_np_uniforms");
}

extern "C" int sg_site_key_host(const char* text, int32_t len, uint64_t* out) {
  using namespace sg;
  SG_REQUIRE(out && len >= 0 && len <= 128 && (text || len == 0), "sg_site_key_host: bad argument");
  blake2b128_1block(reinterpret_cast<const unsigned char*>(text), len, out);
  return SG_OK;
}

extern "C" int sg_predict_tally(const int8_t* states, int64_t var_stride, const int32_t* t_var,
                                const int32_t* t_case, int32_t targets, int32_t max_card, int64_t* freq, int32_t* err,
                                void* stream) {
  using namespace sg;
  SG_REQUIRE(states && t_var && t_case && freq && err && targets >= 0 && max_card > 0 && var_stride > 0,
             "sg_predict_tally: bad argument");
  if (targets == 0) return SG_OK;
  k_predict_tally<<<(targets + 255) / 256, 256, 0, (cudaStream_t)stream>>>(states, var_stride, t_var, t_case, targets,
                                                                           max_card, freq, err);
  return check_launch("sg_predict_tally");
}

SG_CHECKED_EXPORT(aux)
