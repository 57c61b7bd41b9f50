// Count accumulators and CPT updates (model-sized work after each minibatch).
//
//  * sg_accumulate: update_moving_sum / update_exponential (sampler.py:337-351)
//    through CountSet.add / scale (model.py:56-62), rounding exactly where
//    numpy rounds: `mine += scale * theirs` is one product and one sum.
//  * sg_mean_cpts: mean_cpts (model.py:188-194), (c + alpha) / pairwise row sum.
//  * sg_sample_cpts: sample_cpts (model.py:179-185) draws each row from
//    Dirichlet(c + alpha).  numpy's standard_gamma (ziggurat normals) is not
//    reproduced; each cell draws a Marsaglia-Tsang gamma from its own Philox
//    substream (sg_device.cuh), carried in log space so tiny shapes never
//    underflow (the reference's degenerate-row redraw, model.py:168-176).
//  * sg_step_finish: accumulate + CPT update + conditional tables (+ packed
//    tables, next-count clearing, key advance) fused into ONE single-CTA
//    kernel for model-sized networks -- a minibatch step is then check +
//    sweep + finish.  Same arithmetic, same results as the separate calls.
#include "sg_device.cuh"

namespace sg {

__device__ __forceinline__ double acc_cell(int mode, double t, double add, bool has_prev, double prev, double decay) {
  if (mode == SG_ACC_MOVING) {
    if (has_prev) t = __dadd_rn(t, __dmul_rn(-1.0, prev));
    return __dadd_rn(t, add);
  }
  t = __dmul_rn(t, decay);
  return __dadd_rn(t, add);
}

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

__device__ __forceinline__ void mean_row(const double* total, double a, int card, double* out) {
  double sh[SG_MAX_CARD];
  for (int s = 0; s < card; ++s) sh[s] = __dadd_rn(total[s], a);
  const double sum = np_pairwise_sum(sh, card);
  for (int s = 0; s < card; ++s) out[s] = __ddiv_rn(sh[s], sum);
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
      lg[warp][s] = log_gamma_draw(rs, total[base + s] + a);
    }
    __syncwarp();
    if (lane == 0) dirichlet_normalise(lg[warp], card, out + base);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- fused finish

struct FinishArgs {
  int acc_mode, map_estimate;
  double decay;
  double* total;
  const unsigned long long* new_counts;
  const unsigned long long* prev_counts;
  const double* alpha;
  uint64_t key;
  const uint64_t* key_dev;
  double* cpt;
  double* ptab;
  uint32_t* ftab;
  uint32_t* stab;
  unsigned long long* clear_counts;
  const uint64_t* key_table;
  int32_t* key_index;
  int kps;
  uint64_t* key_current;
  int has_small;
  sg_small sp;
};

static constexpr int FINISH_THREADS = 512;
static constexpr int FINISH_MAX_CELLS = 4096;

__global__ void __launch_bounds__(FINISH_THREADS) k_step_finish(const sg_net net, const FinishArgs f) {
  __shared__ double lg[FINISH_MAX_CELLS];
  const int tid = threadIdx.x;
  const int cells = int(net.cells);
  const uint64_t key = f.key_dev ? __ldg(f.key_dev) : f.key;
  if (tid == 0 && net.table_entries > 0) f.ftab[net.ftab_size] = 0u;
  // 1. accumulator
  for (int i = tid; i < cells; i += FINISH_THREADS) {
    const double t = acc_cell(f.acc_mode, f.total[i], double(f.new_counts[i]), f.prev_counts != nullptr,
                              f.prev_counts ? double(f.prev_counts[i]) : 0.0, f.decay);
    f.total[i] = t;
    if (!f.map_estimate) {
      const int v = cell_var(net, i);
      CellStream rs(key, uint64_t(i));
      lg[i] = log_gamma_draw(rs, t + f.alpha[v]);
    }
  }
  __syncthreads();
  // 2. CPT update, one row per thread
  for (int row = tid; row < int(net.rows); row += FINISH_THREADS) {
    const int v = __ldg(net.row_var + row);
    const int card = __ldg(net.card + v);
    const int64_t base = __ldg(net.cpt_off + v) + (row - __ldg(net.row_off + v)) * card;
    if (f.map_estimate) mean_row(f.total + base, f.alpha[v], card, f.cpt + base);
    else dirichlet_normalise(lg + base, card, f.cpt + base);
  }
  __syncthreads();
  // 3. conditional tables from the new CPTs (plain loads: written above)
  for (int g = tid; g < int(net.table_entries); g += FINISH_THREADS) {
    int lo = 0, hi = net.n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(net.tab_start + mid) <= g) lo = mid; else hi = mid;
    }
    const int v = lo;
    const int64_t e = g - __ldg(net.tab_start + v);
    const int card = __ldg(net.card + v);
    int s[SG_MAX_MB];
    const int m0 = __ldg(net.mb_start + v), m1 = __ldg(net.mb_start + v + 1);
    for (int k = m0; k < m1; ++k) s[k - m0] = int((e / __ldg(net.mb_stride + k)) % __ldg(net.card + __ldg(net.mb_var + k)));
    double w[SG_MAX_CARD];
    conditional_weights<false>(net, v, s, f.cpt, w);
    table_entry(w, card, f.ptab + __ldg(net.ptab_off + v) + e * card, f.ftab + __ldg(net.ftab_off + v) + e * (card - 1),
                f.ftab + net.ftab_size);
  }
  __syncthreads();
  // 4. packed-lane tables
  if (f.has_small) {
    const sg_small& sp = f.sp;
    for (int i = tid; i < (sp.n << sp.bits); i += FINISH_THREADS) small_table_entry(net, sp, f.ftab, f.stab, i);
  }
  // 5. clear the next visit's count buffer, advance the key cursor
  if (f.clear_counts)
    for (int i = tid; i < cells; i += FINISH_THREADS) f.clear_counts[i] = 0ull;
  if (f.key_table) {
    __syncthreads();  // every thread has read this step's keys
    const int idx = *f.key_index;
    for (int k = tid; k < f.kps; k += FINISH_THREADS) f.key_current[k] = f.key_table[int64_t(idx) * f.kps + k];
    __syncthreads();
    if (tid == 0) *f.key_index = idx + 1;
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
  if (f->key_table) SG_REQUIRE(f->key_index && f->key_current && f->kps > 0, "sg_step_finish: bad key cursor");
  cudaStream_t s = (cudaStream_t)stream;
  if (net->cells <= FINISH_MAX_CELLS && net->table_entries <= 65536 && (!sp || (sp->n << sp->bits) <= 65536)) {
    FinishArgs a;
    a.acc_mode = f->acc_mode;
    a.map_estimate = f->map_estimate;
    a.decay = f->decay;
    a.total = f->total;
    a.new_counts = reinterpret_cast<const unsigned long long*>(f->new_counts);
    a.prev_counts = reinterpret_cast<const unsigned long long*>(f->prev_counts);
    a.alpha = f->alpha;
    a.key = f->key;
    a.key_dev = f->key_dev;
    a.cpt = f->cpt;
    a.ptab = f->ptab;
    a.ftab = f->ftab;
    a.stab = f->stab;
    a.clear_counts = reinterpret_cast<unsigned long long*>(f->clear_counts);
    a.key_table = f->key_table;
    a.key_index = f->key_index;
    a.kps = f->kps;
    a.key_current = f->key_current;
    a.has_small = sp ? 1 : 0;
    if (sp) a.sp = *sp;
    k_step_finish<<<1, FINISH_THREADS, 0, s>>>(*net, a);
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
  if (f->clear_counts) cudaMemsetAsync(f->clear_counts, 0, sizeof(uint64_t) * net->cells, s);
  if (f->key_table) return sg_keys_advance(f->key_table, f->key_index, f->kps, f->key_current, stream);
  return check_launch("sg_step_finish");
}
