// Count accumulators and CPT updates (model-sized work after each minibatch).
//
//  * sg_accumulate: update_moving_sum / update_exponential (sampler.py:337-351)
//    through CountSet.add / scale (model.py:56-62), rounding exactly where
//    numpy rounds: `mine += scale * theirs` is one product and one sum.
//  * sg_mean_cpts: mean_cpts (model.py:188-194), (c + alpha) / pairwise row sum.
//  * sg_sample_cpts: sample_cpts (model.py:179-185) draws each row from
//    Dirichlet(c + alpha).  numpy's standard_gamma (ziggurat normals) is not
//    reproduced; each cell draws a Marsaglia-Tsang gamma from its own Philox
//    substream (sg_device.cuh), shapes below 1 carried in log space so they never
//    underflow (the reference's degenerate-row redraw, model.py:168-176).
//  * sg_step_finish: accumulate + CPT update + conditional tables (+ packed
//    tables, next-count clearing, key advance) fused into ONE single-CTA
//    kernel for model-sized networks -- a minibatch step is then check +
//    sweep + finish.  Same arithmetic, same results as the separate calls.
#include "sg_finish.cuh"

namespace sg {

__global__ void k_accumulate(int mode, double* __restrict__ total, const unsigned long long* __restrict__ nw,
                             const unsigned long long* __restrict__ prev, const double* __restrict__ nwf,
                             const double* __restrict__ prevf, double decay, int64_t cells) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cells;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double add = nw ? double(nw[i]) : nwf[i];
    const bool hp = prev || prevf;
    const double pv = prev ? double(prev[i]) : (prevf ? prevf[i] : 0.0);
    total[i] = acc_cell(mode, total[i], add, hp, pv, decay);
  }
}

__global__ void k_mean_cpts(const sg_net net, const double* __restrict__ total, const double* __restrict__ alpha,
                            double* __restrict__ out) {
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < net.rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int v = __ldg(net.row_var + row);
    const int card = __ldg(net.card + v);
    const int64_t base = __ldg(net.cpt_off + v) + (row - __ldg(net.row_off + v)) * card;
    mean_row(total + base, alpha[v], card, out + base);
  }
}

// One warp per row: lanes draw the row's cells in parallel, lane 0 normalises.
__global__ void k_sample_cpts(const sg_net net, const double* __restrict__ total, const double* __restrict__ alpha,
                              uint64_t key, const uint64_t* __restrict__ key_dev, double* __restrict__ out) {
  __shared__ double lg[8][SG_MAX_CARD];
  __shared__ uint8_t inlog[8][SG_MAX_CARD];
  if (key_dev) key = __ldg(key_dev);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * int64_t(blockDim.x >> 5) + warp; row < net.rows; row += wstride) {
    const int v = __ldg(net.row_var + row);
    const int card = __ldg(net.card + v);
    const int64_t base = __ldg(net.cpt_off + v) + (row - __ldg(net.row_off + v)) * card;
    const double a = alpha[v];
    for (int s = lane; s < card; s += 32) {
      CellStream rs(key, uint64_t(base + s));
      const GammaPre pre = gamma_pre(rs);
      bool il;
      lg[warp][s] = gamma_draw(rs, pre, total[base + s] + a, &il);
      inlog[warp][s] = il;
    }
    __syncwarp();
    if (lane == 0) dirichlet_row(lg[warp], inlog[warp], card, out + base);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(FINISH_THREADS) k_step_finish(const sg_net gnet, const FinishArgs f) {
  extern __shared__ __align__(16) unsigned char smem[];
  step_finish_body(gnet, f, smem, FINISH_THREADS);
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
  k_sample_cpts<<<grid_for(net->rows * 32), 256, 0, (cudaStream_t)stream>>>(*net, total, alpha, key, key_dev,
                                                                           cpt_out);
  return check_launch("sg_sample_cpts");
}

extern "C" int sg_step_finish(const sg_net* net, const sg_small* sp, const sg_finish* f, void* stream) {
  using namespace sg;
  SG_REQUIRE(net && f && f->total && f->new_counts && f->alpha && f->cpt, "sg_step_finish: null argument");
  SG_REQUIRE(f->acc_mode == SG_ACC_MOVING || f->acc_mode == SG_ACC_EXPONENTIAL, "sg_step_finish: bad mode");
  SG_REQUIRE(net->max_card <= SG_MAX_CARD && net->max_mb <= SG_MAX_MB, "sg_step_finish: capacity exceeded");
  if (net->table_entries > 0) SG_REQUIRE(f->ptab && f->ftab, "sg_step_finish: tables required");
  if (sp) SG_REQUIRE(f->stab, "sg_step_finish: packed table required");
  SG_REQUIRE(!f->check_obs, "sg_step_finish: the observation check is sg_step_tail_joint's");
  if (f->key_table) SG_REQUIRE(f->key_index && f->key_current && f->kps > 0, "sg_step_finish: bad key cursor");
  cudaStream_t s = (cudaStream_t)stream;
  if (finish_fits(*net, sp)) {
    const FinishArgs a = make_finish_args(f, sp);
    const size_t smem = finish_smem(*net);
    static size_t configured[SG_MAX_DEVICES] = {};  // raise the opt-in once per device (graph-capture friendly)
    if (optin_needed(configured, smem))
      cudaFuncSetAttribute(k_step_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    launch_pdl(k_step_finish, dim3(1), dim3(FINISH_THREADS), smem, s, *net, a);  // staging overlaps the sweep
    return check_launch("sg_step_finish");
  }
  // large models: the same steps as separate grid-wide launches
  int st = sg_accumulate(f->acc_mode, f->total, f->new_counts, f->prev_counts, f->decay, net->cells, stream);
  if (st) return st;
  st = f->map_estimate ? sg_mean_cpts(net, f->total, f->alpha, f->cpt, stream)
                       : sg_sample_cpts(net, f->total, f->alpha, f->key, f->key_dev, f->cpt, stream);
  if (st) return st;
  st = sg_build_tables(net, f->cpt, f->ptab, f->ftab, stream);
  if (st) return st;
  if (sp) {
    st = sg_small_tables(net, sp, f->ftab, f->stab, stream);
    if (st) return st;
  }
  if (f->cpt_host) {
    st = sg_copy_small(f->cpt_host, f->cpt, net->cells * int64_t(sizeof(double)), stream);
    if (st) return st;
  }
  if (f->clear_counts) cudaMemsetAsync(f->clear_counts, 0, sizeof(uint64_t) * net->cells, s);
  if (f->key_table) return sg_keys_advance(f->key_table, f->key_index, f->kps, f->key_current, stream);
  return check_launch("sg_step_finish");
}

#ifdef SG_FINISH_TRACE
extern "C" int sg_debug_finish_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, sg::g_finish_trace, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 2;
}
#endif
