// vt_sim.h — launch parameters of the simulate kernel (K4), shared by host and device code.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voltana.h"
#include "vt_device.cuh"

namespace vt {

constexpr int SIM_THREADS = 128;      // 4 warps per CTA, one scenario per warp
constexpr int MAX_SLOS = 64, MAX_LAYOUTS = 16, MAX_GRIDS = 16, MAX_PROFILES = 8;
constexpr uint32_t WHEEL_BUCKETS = 1024;  // per decode instance (power of two)

struct SimParams {
  // traces (device)
  const double *arrival;
  const uint32_t *in_len, *out_len;
  const uint64_t *offset;
  const double *duration;
  // scenarios (device)
  const uint32_t *trace_id, *slo_id, *layout_id, *grid_id, *profile_id;
  const uint64_t *hash_seed;
  uint32_t n;
  uint32_t nb;                 // wheel buckets per decode instance
  uint32_t n_slots;            // workspace slots = warps that may run scenarios
  uint32_t n_slos, n_layouts, n_grids, n_profiles;
  uint64_t n_traces;
  voltana_result *out;
  // workspace
  uint32_t *counter;
  char *slots;
  size_t slot_bytes, node_bytes, xd_bytes;
  uint64_t max_requests;
  // host tables copied into the kernel parameter bank
  voltana_slo slo[MAX_SLOS];
  voltana_layout lay[MAX_LAYOUTS];
  voltana_grid grid[MAX_GRIDS];
  DevProfile prof[MAX_PROFILES];
};

template <int MAXP, int MAXD> const void *sim_kernel_ptr();
template <int MAXP, int MAXD> cudaError_t launch_sim(const SimParams &P, int grid, cudaStream_t st);

}  // namespace vt
