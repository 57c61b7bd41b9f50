// The model-sized tail of a minibatch step (accumulate -> CPT update ->
// conditional tables -> packed tables -> clear next counts -> advance keys),
// as a device function that one CTA runs (k_step_finish, sg_model.cu).
#pragma once

#include "sg_device.cuh"

namespace sg {

// Debug build only (-DSG_FINISH_TRACE): %globaltimer at the phase boundaries
// of the step tail, read back with sg_debug_finish_trace (tools/trace_finish.py).
#ifdef SG_FINISH_TRACE
__device__ unsigned long long g_finish_trace[12];
#define SG_TRACE(i)                                                                             \
  do {                                                                                          \
    if (threadIdx.x == 0) {                                                                     \
      unsigned long long t;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                                     \
      g_finish_trace[i] = t;                                                                    \
    }                                                                                           \
  } while (0)
#else
#define SG_TRACE(i) \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ double acc_cell(int mode, double t, double add, bool has_prev, double prev, double decay) {
  if (mode == SG_ACC_MOVING) {
    if (has_prev) t = __dadd_rn(t, __dmul_rn(-1.0, prev));
    return __dadd_rn(t, add);
  }
  t = __dmul_rn(t, decay);
  return __dadd_rn(t, add);
}

template <int K = 0>
__device__ __forceinline__ void mean_row(const double* total, double a, int card, double* out) {
  if (K) card = K;
  double sh[K ? K : SG_MAX_CARD];
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) sh[s] = __dadd_rn(total[s], a);
  double sum;
  if (K && K < 8) {  // numpy's pairwise sum is sequential below 8 terms
    sum = 0.0;
#pragma unroll
    for (int s = 0; s < (K ? K : 1); ++s) sum = __dadd_rn(sum, sh[s]);
  } else {
    sum = np_pairwise_sum(sh, card);
  }
#pragma unroll
  for (int s = 0; s < (K ? K : card); ++s) out[s] = __ddiv_rn(sh[s], sum);
}

__device__ __forceinline__ uint32_t packed_invalid(uint32_t w, int card, int nib) {
  if (nib == 2) {  // crumbs: 3 = missing; only 2 can be out of range (binary variables)
    return card >= 3 ? 0u : ((w >> 1) & ~w & 0x55555555u);
  }
  const uint32_t lim = 0x01010101u * uint32_t(card - 1);  // nibbles: 15 = missing
  const uint32_t xe = w & 0x0F0F0F0Fu, xo = (w >> 4) & 0x0F0F0F0Fu;
  return (__vcmpgtu4(xe, lim) & ~__vcmpeq4(xe, 0x0F0F0F0Fu)) | (__vcmpgtu4(xo, lim) & ~__vcmpeq4(xo, 0x0F0F0F0Fu));
}

// Range check of an observation block (int8, or packed .sgb rows with nib 4 /
// 2) by threads gtid = 0 .. gthreads - 1 of the caller's choosing: a whole grid
// (the sweeps) or one CTA (the step tail's model update, while the sweep runs).
__device__ __forceinline__ void obs_range_check_range(const sg_small& sp, const int8_t* __restrict__ obs, int ld_obs,
                                                      int cases, int32_t* err, int nib, int gtid, int gthreads) {
  if (!obs || cases <= 0) return;
  const bool packed = nib == 4 || nib == 2;
  const int per_word = packed ? 32 / nib : 4;  // cases per 32-bit word
  const int words = (cases + per_word - 1) / per_word;
  const int vecs = (words + 3) >> 2;
  unsigned bad = 0;
  for (int i = gtid; i < sp.n * vecs; i += gthreads) {
    int v = 0, q = i;  // (row, vector): n <= 7 subtractions instead of a division
    while (q >= vecs) {
      q -= vecs;
      ++v;
    }
    const int card = sp.card[v];
    const uint4* row = reinterpret_cast<const uint4*>(obs + int64_t(v) * ld_obs);
    const uint32_t lim = 0x01010101u * uint32_t(card - 1);
    {
      const uint4 x = __ldcs(row + q);
      const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int first = (4 * q + k) * per_word;  // first case of this word
        if (first >= cases) break;
        uint32_t b = packed ? packed_invalid(wv[k], card, nib) : __vcmpgts4(wv[k], lim);
        const int valid = cases - first;
        if (valid < per_word) {  // the row's last word: cases past the minibatch do not count
          const int field_bits = packed ? nib : 8;
          if (packed && nib == 4) {  // planes: byte b of the even plane is case 2b, of the odd plane 2b + 1
            uint32_t keep = 0;
            for (int j = 0; j < valid; ++j) keep |= 0xFu << (4 * j);
            const uint32_t we = wv[k] | ~keep;  // cases past `valid` read as missing (15)
            b = packed_invalid(we, card, nib);
          } else {
            b &= valid * field_bits >= 32 ? 0xFFFFFFFFu : ((1u << (valid * field_bits)) - 1u);
          }
        }
        bad |= b;
      }
    }
  }
  if (bad) atomicOr(err, int(SG_ERR_STATE_RANGE));
}

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
  double* vprob;
  uint32_t* release_sync;  // != NULL: release this word (st.release.gpu) once the new CPTs are in f.cpt
  // != NULL (with release_sync): release right after phase 1 instead, with the
  // cells' gamma draws (MAP: totals) in release_lg[0..cells) and their in-log
  // flags in the bytes after them; the readers normalise the rows themselves
  double* release_lg;
  double* cpt_host;  // != NULL: mapped pinned host copy of the new CPTs
  const int8_t* check_obs;  // != NULL: the merged tail's row slices range-check this block
  int check_ld, check_nib, check_cases;
  int32_t* check_err;
  int has_small;
  int early_inputs;  // the preceding sweep triggers only after its own wait: read total/prev/key before ours
  int packed_only;  // SG_FINISH_PACKED_ONLY: skip ptab/ftab, build stab from the CPTs
  sg_small sp;
};

// Packed word(s) i = (v, S) straight from the CPTs: the weights and
// thresholds table_entry computes for the blanket configuration S encodes,
// i.e. exactly the words small_table_entry copies out of ftab.
__device__ __forceinline__ void small_table_direct(const sg_net& net, const sg_small& sp, const double* cpt,
                                                   uint32_t* stab, uint32_t* zs_flag, int i, double* vprob) {
  const int v = i >> sp.bits;
  const uint32_t S = uint32_t(i & ((1 << sp.bits) - 1));
  const int card = sp.card[v];
  uint32_t* out = stab + sp.toff[v] + S * sp.tstride[v];
  bool valid = (S & ~sp.mbmask[v]) == 0u;
  int s[SG_MAX_MB];
  const int m0 = net.mb_start[v], m1 = net.mb_start[v + 1];
  for (int k = m0; k < m1 && valid; ++k) {
    const int u = net.mb_var[k];
    s[k - m0] = small_field(S, sp, u);
    valid = s[k - m0] < sp.card[u];
  }
  if (!valid) {
    for (int t = 0; t < card - 1; ++t) out[t] = 0u;
    if (vprob)
      for (int t = 0; t < card; ++t) vprob[size_t(i) * 4 + t] = 0.0;
    return;
  }
  with_card(card, [&](auto C) {
    constexpr int K = decltype(C)::value;
    double w[K ? K : SG_MAX_CARD];
    conditional_weights<false, K>(net, v, s, cpt, w);
    table_entry<K>(w, card, nullptr, out, zs_flag);
    if (vprob) joint_conditional<K>(w, card, vprob + size_t(i) * 4);
  });
}

static constexpr int FINISH_THREADS = 512;
static constexpr int FINISH_MAX_CELLS = 4096;
static constexpr size_t FINISH_MAX_SMEM = 160 * 1024;

__host__ __device__ inline size_t finish_smem(const sg_net& net) {
  return size_t(net.cells) * 16 + size_t(net.blob64_words) * 8 + ((size_t(net.blob32_words) * 4 + 15) & ~size_t(15)) +
         ((size_t(net.cells) + 15) & ~size_t(15));
}

// The step tail, run by ONE CTA of `nt` threads (tid = threadIdx.x).  The
// network pack (two blobs) and the CPTs are staged in shared memory `smem`
// (finish_smem bytes) so the dependent index chains of the table build hit
// on-chip memory instead of L2.
__device__ __forceinline__ void step_finish_body(const sg_net& gnet, const FinishArgs& f, unsigned char* smem,
                                                 const int nt) {
  double* lg = reinterpret_cast<double*>(smem);
  double* cpt_s = lg + gnet.cells;
  int64_t* b64 = reinterpret_cast<int64_t*>(cpt_s + gnet.cells);
  int32_t* b32 = reinterpret_cast<int32_t*>(b64 + gnet.blob64_words);
  const int tid = threadIdx.x;
  const int cells = int(gnet.cells);
  uint8_t* inlog = reinterpret_cast<uint8_t*>(b32) + ((size_t(gnet.blob32_words) * 4 + 15) & ~size_t(15));
  SG_TRACE(7);
  for (int i = tid; i < int(gnet.blob64_words); i += nt) b64[i] = __ldg(gnet.blob64 + i);
  for (int i = tid; i < int(gnet.blob32_words); i += nt) b32[i] = __ldg(gnet.blob32 + i);
  // With early_inputs the preceding sweep has waited for the previous tail
  // before letting this grid start, so the running total, this minibatch's
  // previous counts and the Dirichlet key are final already: load them and
  // draw each cell's first gamma attempt (independent of the counts) while
  // the sweep is still running.
  const bool early = f.early_inputs != 0;
  double t_old = 0.0, t_prev = 0.0, a_cell = 0.0;
  GammaPre pre{};
  int my_cell = -1;  // early path: one cell per thread
  uint64_t key = 0;
  // early path: the next visit's keys (static table) and the cursor, stored right after the wait
  const bool early_keys = early && f.key_table && f.kps <= nt;
  uint64_t next_key = 0;
  int key_idx = 0;
  if (early_keys) {
    key_idx = *f.key_index;
    if (tid < f.kps) next_key = f.key_table[int64_t(key_idx) * f.kps + tid];
  }
  if (early && cells <= nt) {
    key = f.key_dev ? *f.key_dev : f.key;
    if (tid < cells) {
      my_cell = tid;
      t_old = f.total[tid];
      t_prev = f.prev_counts ? double(f.prev_counts[tid]) : 0.0;
      if (!f.map_estimate) {
        int lo = 0, hi = gnet.n;  // cell_var on the global pack (blobs not yet synchronised)
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(gnet.cpt_off + mid) <= tid) lo = mid; else hi = mid;
        }
        a_cell = f.alpha[lo];
        CellStream rs(key, uint64_t(tid));
        pre = gamma_pre(rs);
      }
    }
  }
  // Everything above reads data no kernel in flight writes; from here on the
  // inputs are the sweep's counts (and, without early_inputs, the previous
  // tail's key cursor).  Once they are complete the next sweep may start its
  // own prologue.
  SG_TRACE(0);
  pdl_wait();
  pdl_trigger();
  if (!(early && cells <= nt)) key = f.key_dev ? *f.key_dev : f.key;
  if (tid == 0 && gnet.table_entries > 0) f.ftab[gnet.ftab_size] = 0u;
  const bool early_clear = early && cells <= nt && f.clear_counts;  // prev counts already in registers
  if (early_clear && tid < cells) f.clear_counts[tid] = 0ull;
  if (early_keys) {  // every reader of this step's keys has them (the sweep finished, ours are in registers)
    if (tid < f.kps) f.key_current[tid] = next_key;
    if (tid == 0) *f.key_index = key_idx + 1;
  }
  __syncthreads();
  SG_TRACE(1);
  const sg_net net = rebase_net(gnet, b32, b64);
  // 1. accumulator (+ the cell's gamma draw)
  if (my_cell >= 0) {
    const int i = my_cell;
    const double nc = double(f.new_counts[i]);
    SG_TRACE(8);
    const double t = acc_cell(f.acc_mode, t_old, nc, f.prev_counts != nullptr, t_prev, f.decay);
    f.total[i] = t;
    if (f.map_estimate) {
      lg[i] = t;
    } else {
      CellStream rs(key, uint64_t(i));
      rs.call = 2;  // the first attempt's words (gamma_pre) are consumed
      bool il;
      lg[i] = gamma_draw(rs, pre, t + a_cell, &il);
      inlog[i] = il;
    }
    SG_TRACE(9);
  } else if (!(early && cells <= nt)) {
    for (int i = tid; i < cells; i += nt) {
      const double t = acc_cell(f.acc_mode, f.total[i], double(f.new_counts[i]), f.prev_counts != nullptr,
                                f.prev_counts ? double(f.prev_counts[i]) : 0.0, f.decay);
      f.total[i] = t;
      if (f.map_estimate) {
        lg[i] = t;
      } else {
        const int v = cell_var<false>(net, i);
        CellStream rs(key, uint64_t(i));
        const GammaPre p0 = gamma_pre(rs);
        bool il;
        lg[i] = gamma_draw(rs, p0, t + f.alpha[v], &il);
        inlog[i] = il;
      }
    }
  }
  if (f.release_sync && f.release_lg) {  // hand the draws over now: the slices build their rows from them
    // Publication without a per-thread fence: every thread's stores happen
    // before the CTA barrier, the barrier before tid 0's st.release.gpu, and
    // a release is cumulative over what happens before it -- a slice that
    // reads the flag with ld.acquire.gpu sees all of them.
    uint8_t* il_out = reinterpret_cast<uint8_t*>(f.release_lg + cells);
    if (my_cell >= 0) {
      f.release_lg[my_cell] = lg[my_cell];
      il_out[my_cell] = f.map_estimate ? 0 : inlog[my_cell];
    } else if (!(early && cells <= nt)) {
      for (int i = tid; i < cells; i += nt) {
        f.release_lg[i] = lg[i];
        il_out[i] = f.map_estimate ? 0 : inlog[i];
      }
    }
    __syncthreads();
    if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f.release_sync), "r"(1u) : "memory");
  } else {
    __syncthreads();
  }
  SG_TRACE(2);
  // 2. CPT update, one row per thread
  for (int row = tid; row < int(net.rows); row += nt) {
    const int v = net.row_var[row];
    const int card = net.card[v];
    const int64_t base = net.cpt_off[v] + (row - net.row_off[v]) * card;
    with_card(card, [&](auto C) {
      constexpr int K = decltype(C)::value;
      if (f.map_estimate) mean_row<K>(lg + base, f.alpha[v], card, cpt_s + base);
      else dirichlet_row<K>(lg + base, inlog + base, card, cpt_s + base);
    });
    for (int s2 = 0; s2 < card; ++s2) f.cpt[base + s2] = cpt_s[base + s2];
    if (f.cpt_host)
      for (int s2 = 0; s2 < card; ++s2) f.cpt_host[base + s2] = cpt_s[base + s2];
  }
  const bool release_cpts = f.release_sync && !f.release_lg;
  if (release_cpts && tid < int(net.rows)) __threadfence();  // this thread's CPT rows are visible device-wide ...
  __syncthreads();                      // ... for every thread before the release
  if (release_cpts && tid == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f.release_sync), "r"(1u) : "memory");
  SG_TRACE(3);
  // 3. conditional tables from the new CPTs (packed-only: the packed words directly)
  if (f.packed_only) {
    const sg_small& sp = f.sp;
    for (int i = tid; i < (sp.n << sp.bits); i += nt)
      small_table_direct(net, sp, cpt_s, f.stab, f.ftab + net.ftab_size, i, f.vprob);
  }
  for (int g = f.packed_only ? int(net.table_entries) : tid; g < int(net.table_entries); g += nt) {
    int lo = 0, hi = net.n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (net.tab_start[mid] <= g) lo = mid; else hi = mid;
    }
    const int v = lo;
    const int64_t e = g - net.tab_start[v];
    const int card = net.card[v];
    int s[SG_MAX_MB];
    const int m0 = net.mb_start[v], m1 = net.mb_start[v + 1];
    for (int k = m0; k < m1; ++k) s[k - m0] = int((e / net.mb_stride[k]) % net.card[net.mb_var[k]]);
    double* pe = f.ptab + net.ptab_off[v] + e * card;
    uint32_t* fe = f.ftab + net.ftab_off[v] + e * (card - 1);
    with_card(card, [&](auto C) {
      constexpr int K = decltype(C)::value;
      double w[K ? K : SG_MAX_CARD];
      conditional_weights<false, K>(net, v, s, cpt_s, w);
      table_entry<K>(w, card, pe, fe, f.ftab + net.ftab_size);
    });
  }
  __syncthreads();
  SG_TRACE(4);
  // 4. packed-lane tables
  if (f.has_small && !f.packed_only) {
    const sg_small& sp = f.sp;
    for (int i = tid; i < (sp.n << sp.bits); i += nt) small_table_entry<false>(net, sp, f.ftab, f.stab, i);
  }
  SG_TRACE(5);
  // 5. clear the next visit's count buffer, advance the key cursor
  if (f.clear_counts && !early_clear)
    for (int i = tid; i < cells; i += nt) f.clear_counts[i] = 0ull;
  if (f.key_table && !early_keys) {
    __syncthreads();  // every thread has read this step's keys
    const int idx = *f.key_index;
    for (int k = tid; k < f.kps; k += nt) f.key_current[k] = f.key_table[int64_t(idx) * f.kps + k];
    __syncthreads();
    if (tid == 0) *f.key_index = idx + 1;
  }
  SG_TRACE(6);
}


// Kernel-side copy of an sg_finish (+ optional packed plan).
// The optional observation-block check of sg_finish is well formed.
inline bool finish_check_ok(const sg_finish* f, const sg_small* sp) {
  if (!f->check_obs) return true;
  const int b = f->check_bits;
  const int per_byte = b == 4 || b == 2 ? 8 / b : 1;
  return sp && f->check_err && (b == 8 || b == 4 || b == 2 || b == 0) && f->check_ld % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(f->check_obs) & 15) == 0 && f->check_cases >= 0 &&
         int64_t(f->check_ld) * per_byte >= f->check_cases;
}

inline FinishArgs make_finish_args(const sg_finish* f, const sg_small* sp) {
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
  a.vprob = sp ? f->vprob : nullptr;
  a.cpt_host = f->cpt_host;
  a.check_obs = sp ? static_cast<const int8_t*>(f->check_obs) : nullptr;
  a.check_ld = f->check_ld;
  a.check_nib = f->check_bits == 4 || f->check_bits == 2 ? f->check_bits : 0;
  a.check_cases = f->check_cases;
  a.check_err = f->check_err;
  a.early_inputs = 0;
  a.release_sync = nullptr;
  a.release_lg = nullptr;
  a.has_small = sp ? 1 : 0;
  a.packed_only = (sp && (f->flags & SG_FINISH_PACKED_ONLY)) ? 1 : 0;
  if (sp) a.sp = *sp;
  return a;
}

// Whether the single-CTA tail can handle this model.
inline bool finish_fits(const sg_net& net, const sg_small* sp) {
  return net.blob32 && net.blob64 && net.cells <= FINISH_MAX_CELLS && finish_smem(net) <= FINISH_MAX_SMEM &&
         net.table_entries <= 65536 && (!sp || (sp->n << sp->bits) <= 65536);
}

}  // namespace sg
