// Conditional tables: the full conditional of v is a deterministic function
// of its Markov-blanket configuration, so instead of re-gathering CPT rows for
// every latent lane (what _resample_variable does, sampler.py:226-242) we
// evaluate the reference's weight product once per blanket configuration per
// CPT update.  For Koller the five tables hold 31 configurations in total; a
// sweep then costs one blanket index + one table read per latent cell.
//
// Table entry layout (entry e of variable v, card k):
//   ptab[ptab_off[v] + e*k + s]  = cum_s   (s = 0..k-2, sequential cumsum)
//   ptab[ptab_off[v] + e*k + k-1] = norm   (numpy pairwise sum of the k weights)
//   ftab[ftab_off[v] + e*(k-1) + s] = ceil(cum_s / norm * 2^31)
//                                     (0xFFFFFFFF in slot 0 when norm <= 0)
#include "sg_device.cuh"

namespace sg {

__global__ void __launch_bounds__(SG_THREADS)
k_build_tables(const sg_net net, const double* __restrict__ cpt, double* __restrict__ ptab,
               uint32_t* __restrict__ ftab) {
  const int64_t total = net.table_entries;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    // variable owning global entry g: tab_start is a prefix over variables
    int lo = 0, hi = net.n;  // find v with tab_start[v] <= g < tab_start[v+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(net.tab_start + mid) <= g) lo = mid; else hi = mid;
    }
    const int v = lo;
    const int64_t e = g - __ldg(net.tab_start + v);
    const int card = __ldg(net.card + v);
    int s[SG_MAX_MB];
    const int m0 = __ldg(net.mb_start + v), m1 = __ldg(net.mb_start + v + 1);
    for (int k = m0; k < m1; ++k) {
      const int u = __ldg(net.mb_var + k);
      s[k - m0] = int((e / __ldg(net.mb_stride + k)) % __ldg(net.card + u));
    }
    double* pe = ptab + __ldg(net.ptab_off + v) + e * card;
    uint32_t* fe = ftab + __ldg(net.ftab_off + v) + e * (card - 1);
    with_card(card, [&](auto C) {
      constexpr int K = decltype(C)::value;
      double w[K ? K : SG_MAX_CARD];
      conditional_weights<true, K>(net, v, s, cpt, w);
      table_entry<K>(w, card, pe, fe, ftab + net.ftab_size);
    });
  }
}

}  // namespace sg

extern "C" int sg_build_tables(const sg_net* net, const double* cpt, double* ptab,
                               uint32_t* ftab, void* stream) {
  SG_REQUIRE(net && cpt, "sg_build_tables: null argument");
  if (net->table_entries == 0) return SG_OK;
  SG_REQUIRE(ptab && ftab, "sg_build_tables: null table");
  SG_REQUIRE(net->max_card <= SG_MAX_CARD, "sg_build_tables: card %d > %d", net->max_card,
             SG_MAX_CARD);
  SG_REQUIRE(net->max_mb <= SG_MAX_MB, "sg_build_tables: blanket %d > %d", net->max_mb,
             SG_MAX_MB);
  const int64_t blocks64 = (net->table_entries + SG_THREADS - 1) / SG_THREADS;
  const int blocks = int(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
  cudaMemsetAsync(ftab + net->ftab_size, 0, sizeof(uint32_t), (cudaStream_t)stream);
  sg::k_build_tables<<<blocks, SG_THREADS, 0, (cudaStream_t)stream>>>(*net, cpt, ptab, ftab);
  return sg::check_launch("sg_build_tables");
}
