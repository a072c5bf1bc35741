// vt_series.h — launch parameters of K5 (voltana_series_to_samples).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voltana.h"

namespace vt {

constexpr int SERIES_THREADS = 256;
constexpr int SERIES_MAX_GRIDS = 16, SERIES_MAX_LAYOUTS = 16;

struct SeriesParams {
  const voltana_iteration *iters;
  const uint32_t *iter_count;
  const uint64_t *iter_offset;   // [n] ascending, multiples of cap
  uint32_t cap, profile_id;
  const uint32_t *layout_id, *grid_id, *scen_profile_id;
  size_t n, n_slots;
  uint8_t *phase;
  uint16_t *level;
  uint32_t *n_bt, *n_req, *n_kv;
  double *lat;
  int32_t n_p[SERIES_MAX_LAYOUTS];
  voltana_grid grid[SERIES_MAX_GRIDS];
};

cudaError_t launch_series(const SeriesParams &P, int grid, cudaStream_t st);

}  // namespace vt
