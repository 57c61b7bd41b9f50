// Count accumulators and CPT updates (model-sized work after each minibatch).
//
//  * sg_accumulate: update_moving_sum / update_exponential (sampler.py:337-351)
//    through CountSet.add / scale (model.py:56-62), rounding exactly where
//    numpy rounds: `mine += scale * theirs` is one product and one sum.
//  * sg_mean_cpts: mean_cpts (model.py:188-194), (c + alpha) / pairwise row sum.
//  * sg_sample_cpts: sample_cpts (model.py:179-185) draws each row from
//    Dirichlet(c + alpha).  numpy's standard_gamma (ziggurat normals) is not
//    reproduced; this is a Marsaglia-Tsang sampler carried in log space, so
//    rows whose parameters are tiny (the degenerate-row redraw of
//    _draw_dirichlet_rows, model.py:168-176) normalise without underflow.
#include "sg_device.cuh"

namespace sg {

__global__ void k_accumulate(int mode, double* __restrict__ total, const unsigned long long* __restrict__ nw,
                             const unsigned long long* __restrict__ prev, const double* __restrict__ nwf,
                             const double* __restrict__ prevf, double decay, int64_t cells) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cells;
       i += int64_t(gridDim.x) * blockDim.x) {
    double t = total[i];
    const double add = nw ? double(nw[i]) : nwf[i];
    if (mode == SG_ACC_MOVING) {
      if (prev) t = __dadd_rn(t, -double(prev[i]));
      else if (prevf) t = __dadd_rn(t, __dmul_rn(-1.0, prevf[i]));
      t = __dadd_rn(t, add);
    } else {
      t = __dmul_rn(t, decay);
      t = __dadd_rn(t, add);
    }
    total[i] = t;
  }
}

__global__ void k_mean_cpts(const sg_net net, const double* __restrict__ total, const double* __restrict__ alpha,
                            double* __restrict__ out) {
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < net.rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int v = __ldg(net.row_var + row);
    const int card = __ldg(net.card + v);
    const int64_t base = __ldg(net.cpt_off + v) + (row - __ldg(net.row_off + v)) * card;
    const double a = alpha[v];
    double sh[SG_MAX_CARD];
    for (int s = 0; s < card; ++s) sh[s] = __dadd_rn(total[base + s], a);
    const double sum = np_pairwise_sum(sh, card);
    for (int s = 0; s < card; ++s) out[base + s] = __ddiv_rn(sh[s], sum);
  }
}

// Sequential draws of one Philox4x32 substream (counter = (cell, call, 0, tag)).
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

// log of a Gamma(a, 1) draw, a > 0 (Marsaglia & Tsang 2000; a < 1 via
// Gamma(a) = Gamma(a + 1) * U^(1/a), kept in log space).
__device__ double log_gamma_draw(CellStream& rs, double a) {
  double boost = 0.0;
  if (a < 1.0) {
    boost = log(rs.uniform()) / a;
    a += 1.0;
  }
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = rs.normal();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rs.uniform();
    const double x2 = x * x;
    if (u < 1.0 - 0.0331 * x2 * x2 || log(u) < 0.5 * x2 + d * (1.0 - v + log(v)))
      return log(d) + log(v) + boost;
  }
}

__global__ void k_sample_cpts(const sg_net net, const double* __restrict__ total, const double* __restrict__ alpha,
                              uint64_t key, const uint64_t* __restrict__ key_dev, double* __restrict__ out) {
  if (key_dev) key = __ldg(key_dev);
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < net.rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int v = __ldg(net.row_var + row);
    const int card = __ldg(net.card + v);
    const int64_t base = __ldg(net.cpt_off + v) + (row - __ldg(net.row_off + v)) * card;
    const double a = alpha[v];
    double lg[SG_MAX_CARD];
    double mx = -INFINITY;
    for (int s = 0; s < card; ++s) {
      CellStream rs(key, uint64_t(base + s));
      lg[s] = log_gamma_draw(rs, total[base + s] + a);
      mx = fmax(mx, lg[s]);
    }
    double sum = 0.0;
    for (int s = 0; s < card; ++s) {
      lg[s] = exp(lg[s] - mx);
      sum += lg[s];
    }
    for (int s = 0; s < card; ++s) out[base + s] = lg[s] / sum;
  }
}

static int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return int(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

}  // namespace sg

extern "C" int sg_accumulate(int32_t mode, double* total, const uint64_t* new_counts, const uint64_t* prev_counts,
                             double decay, int64_t cells, void* stream) {
  using namespace sg;
  SG_REQUIRE(total && new_counts, "sg_accumulate: null argument");
  SG_REQUIRE(mode == SG_ACC_MOVING || mode == SG_ACC_EXPONENTIAL, "sg_accumulate: bad mode %d", mode);
  if (cells == 0) return SG_OK;
  k_accumulate<<<grid_for(cells), 256, 0, (cudaStream_t)stream>>>(
      mode, total, reinterpret_cast<const unsigned long long*>(new_counts),
      reinterpret_cast<const unsigned long long*>(prev_counts), nullptr, nullptr, decay, cells);
  return check_launch("sg_accumulate");
}

extern "C" int sg_accumulate_f64(int32_t mode, double* total, const double* new_counts, const double* prev_counts,
                                 double decay, int64_t cells, void* stream) {
  using namespace sg;
  SG_REQUIRE(total && new_counts, "sg_accumulate_f64: null argument");
  SG_REQUIRE(mode == SG_ACC_MOVING || mode == SG_ACC_EXPONENTIAL, "sg_accumulate_f64: bad mode %d", mode);
  if (cells == 0) return SG_OK;
  k_accumulate<<<grid_for(cells), 256, 0, (cudaStream_t)stream>>>(mode, total, nullptr, nullptr, new_counts,
                                                                   prev_counts, decay, cells);
  return check_launch("sg_accumulate_f64");
}

extern "C" int sg_mean_cpts(const sg_net* net, const double* total, const double* alpha, double* cpt_out,
                            void* stream) {
  using namespace sg;
  SG_REQUIRE(net && total && alpha && cpt_out, "sg_mean_cpts: null argument");
  SG_REQUIRE(net->max_card <= SG_MAX_CARD, "sg_mean_cpts: card capacity exceeded");
  k_mean_cpts<<<grid_for(net->rows), 256, 0, (cudaStream_t)stream>>>(*net, total, alpha, cpt_out);
  return check_launch("sg_mean_cpts");
}

extern "C" int sg_sample_cpts(const sg_net* net, const double* total, const double* alpha, uint64_t key,
                              const uint64_t* key_dev, double* cpt_out, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && total && alpha && cpt_out, "sg_sample_cpts: null argument");
  SG_REQUIRE(net->max_card <= SG_MAX_CARD, "sg_sample_cpts: card capacity exceeded");
  k_sample_cpts<<<grid_for(net->rows), 256, 0, (cudaStream_t)stream>>>(*net, total, alpha, key, key_dev, cpt_out);
  return check_launch("sg_sample_cpts");
}
