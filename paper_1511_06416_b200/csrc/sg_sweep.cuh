// Shared declarations of the generic sweep kernels (sg_sweep.cu, sg_big.cu).
#pragma once

#include "sg_device.cuh"

namespace sg {

// In-sweep tallies of small models; larger ones run k_tally_chunked after the sweep.
enum TallyMode { TALLY_NONE = 0, TALLY_JOINT = 1, TALLY_CELL8 = 2 };

struct SweepArgs {
  const double* cpt;
  const double* ptab;
  const uint32_t* ftab;
  uint64_t fast_key;
  const uint64_t* fast_key_dev;  // when set, the FAST key is read from device memory (graph replay)
  const uint64_t* keys;
  const double* uniforms;
  const int64_t* inj_off;
  uint64_t* counts;
  int32_t* err;
  int tc;            // cases per tile (multiple of 32)
  int mg;            // replicas per tile (replica groups: blockIdx.y)
  int tally_mode;
  int64_t tab_bytes; // bytes of the table this mode reads (staged when SMALL)
};

// Big-tile sweep of large networks (sg_big.cu): returns false when the
// network or batch does not fit its layout (the caller then takes another kernel).
bool sweep_big(const sg_net& net, const sg_batch& bt, const SweepArgs& a, int rng_mode, cudaStream_t s);

}  // namespace sg
