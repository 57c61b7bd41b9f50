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
