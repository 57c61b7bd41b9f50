// Synthetic data on the device (forward_sample datagen.py:91-107 and mask
// datagen.py:110-121), bit-exact with the reference for dense inputs.  The
// reference materialises data as a 20 B/entry coordinate matrix
// (datagen.py:30-32), which cannot hold the 10^7-10^8 case configurations;
// this writes the int8 observation matrix the sweep consumes directly.
#include "sg_device.cuh"

namespace sg {

__global__ void __launch_bounds__(256)
k_forward_sample(const sg_net net, const double* __restrict__ cpt, const int32_t* __restrict__ topo,
                 const uint64_t* __restrict__ keys, int64_t cases, int64_t case_base, int8_t* __restrict__ out,
                 int64_t ld_out, double hide, uint64_t mk0, uint64_t mk1) {
  const int n = net.n;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cases;
       c += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t gc = uint64_t(case_base + c);
    for (int i = 0; i < n; ++i) {
      const int v = __ldg(topo + i);
      const int card = __ldg(net.card + v);
      int64_t cfg = 0;
      for (int p = __ldg(net.par_start + v), pe = __ldg(net.par_start + v + 1); p < pe; ++p)
        cfg += int64_t(out[int64_t(__ldg(net.par_var + p)) * ld_out + c]) * __ldg(net.par_stride + p);
      const double* row = cpt + __ldg(net.cpt_off + v) + cfg * card;
      const double u = np_uniform(gc, __ldg(keys + 2 * v), __ldg(keys + 2 * v + 1));
      double cum = 0.0;
      int x = 0;
      for (int s = 0; s < card; ++s) {
        cum = s ? __dadd_rn(cum, __ldg(row + s)) : __ldg(row);
        x += (u > cum);
      }
      out[int64_t(v) * ld_out + c] = int8_t(min(x, card - 1));
    }
    if (hide > 0.0) {
      // the mask stream runs over present entries in case-major order
      for (int v = 0; v < n; ++v) {
        const double u = np_uniform(gc * uint64_t(n) + uint64_t(v), mk0, mk1);
        if (!(u >= hide)) out[int64_t(v) * ld_out + c] = -1;
      }
    }
  }
}

}  // namespace sg

extern "C" int sg_forward_sample(const sg_net* net, const double* cpt, const int32_t* topo, const uint64_t* keys,
                                 int64_t cases, int64_t case_base, int8_t* out, int64_t ld_out, double hide,
                                 uint64_t mask_key0, uint64_t mask_key1, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && cpt && topo && keys && out, "sg_forward_sample: null argument");
  SG_REQUIRE(ld_out >= cases, "sg_forward_sample: ld_out < cases");
  if (cases == 0) return SG_OK;
  const int64_t b = (cases + 255) / 256;
  const int blocks = int(b < 148 * 16 ? b : 148 * 16);
  k_forward_sample<<<blocks, 256, 0, (cudaStream_t)stream>>>(*net, cpt, topo, keys, cases, case_base, out, ld_out,
                                                             hide, mask_key0, mask_key1);
  return check_launch("sg_forward_sample");
}

// 4-bit observation blocks (the .sgb nibble encoding, io.py): byte j of a
// packed row holds cases 2j (low nibble) and 2j+1 (high nibble); 15 marks a
// missing cell.  Unpacked into the int8 layout the sweep reads (-1 =
// missing).  Each thread expands 16 packed bytes into 32 states.
namespace sg {
__global__ void __launch_bounds__(256)
k_unpack_nibbles(const uint8_t* __restrict__ packed, int64_t ld_packed, int8_t* __restrict__ out, int64_t ld_out,
                 int rows, int64_t cases) {
  const int64_t per_row = (cases + 31) / 32;
  const int64_t total = per_row * rows;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / per_row);
    const int64_t k = i - int64_t(r) * per_row;
    const uint8_t* src = packed + int64_t(r) * ld_packed + k * 16;
    int8_t* dst = out + int64_t(r) * ld_out + k * 32;
    const int64_t left = cases - k * 32;
    if (left >= 32 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(src));
      const uint32_t in[4] = {w.x, w.y, w.z, w.w};
      uint32_t o[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // bytes b0..b3 -> nibbles lo0 hi0 lo1 hi1 | lo2 hi2 lo3 hi3, 15 -> 0xFF
        const uint32_t lo = in[q] & 0x0F0F0F0Fu, hi = (in[q] >> 4) & 0x0F0F0F0Fu;
        const uint32_t a = __byte_perm(lo, hi, 0x5140), b = __byte_perm(lo, hi, 0x7362);
        o[2 * q] = a | __vcmpeq4(a, 0x0F0F0F0Fu);
        o[2 * q + 1] = b | __vcmpeq4(b, 0x0F0F0F0Fu);
      }
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
      for (int64_t j = 0; j < left && j < 32; ++j) {
        const uint32_t nib = (src[j >> 1] >> (4 * (j & 1))) & 0xF;
        dst[j] = nib == 15 ? int8_t(-1) : int8_t(nib);
      }
    }
  }
}
}  // namespace sg

extern "C" int sg_unpack_nibbles(const uint8_t* packed, int64_t ld_packed, int8_t* out, int64_t ld_out,
                                 int32_t rows, int64_t cases, void* stream) {
  using namespace sg;
  SG_REQUIRE(packed && out, "sg_unpack_nibbles: null argument");
  SG_REQUIRE(rows >= 0 && cases >= 0 && ld_packed * 2 >= cases && ld_out >= cases, "sg_unpack_nibbles: bad shape");
  const int64_t work = int64_t(rows) * ((cases + 31) / 32);
  if (work == 0) return SG_OK;
  const int blocks = int(std::min<int64_t>((work + 255) / 256, 148 * 16));
  k_unpack_nibbles<<<blocks, 256, 0, (cudaStream_t)stream>>>(packed, ld_packed, out, ld_out, rows, cases);
  return check_launch("sg_unpack_nibbles");
}

// 2-bit blocks: one thread per output byte group of 4 cases (simple; the
// file-streaming path decodes one minibatch per visit).
__global__ void k_unpack_crumbs(const uint8_t* __restrict__ packed, int64_t ld_packed, int8_t* __restrict__ out,
                                int64_t ld_out, int rows, int64_t cases) {
  const int64_t per_row = (cases + 3) / 4;
  const int64_t total = per_row * rows;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / per_row);
    const int64_t k = i - int64_t(r) * per_row;
    const uint32_t b = packed[int64_t(r) * ld_packed + k];
    for (int h = 0; h < 4 && k * 4 + h < cases; ++h) {
      const uint32_t x = (b >> (2 * h)) & 3u;
      out[int64_t(r) * ld_out + k * 4 + h] = x == 3u ? int8_t(-1) : int8_t(x);
    }
  }
}

extern "C" int sg_unpack_crumbs(const uint8_t* packed, int64_t ld_packed, int8_t* out, int64_t ld_out, int32_t rows,
                                int64_t cases, void* stream) {
  using namespace sg;
  SG_REQUIRE(packed && out, "sg_unpack_crumbs: null argument");
  SG_REQUIRE(rows >= 0 && cases >= 0 && ld_packed * 4 >= cases && ld_out >= cases, "sg_unpack_crumbs: bad shape");
  const int64_t work = int64_t(rows) * ((cases + 3) / 4);
  if (work == 0) return SG_OK;
  const int blocks = int(std::min<int64_t>((work + 255) / 256, 148 * 16));
  k_unpack_crumbs<<<blocks, 256, 0, (cudaStream_t)stream>>>(packed, ld_packed, out, ld_out, rows, cases);
  return check_launch("sg_unpack_crumbs");
}
