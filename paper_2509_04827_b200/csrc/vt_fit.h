// vt_fit.h — launch parameters of K1 (voltana_fit_profile).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vt {

constexpr int FIT_MAX_WARPS = 8;

struct FitParams {
  const uint8_t *phase;
  const uint16_t *level;
  const uint32_t *n_bt, *n_req, *n_kv;
  const double *lat;
  size_t n, chunk;            // samples, samples per warp
  int32_t k, n_tiles, tile_w, cells;
  int32_t n_ptiles, kp;       // prefill tiles T_p (>= 1) and TTFT cells kp = T_p * k [F1]
  uint32_t pcut, pad;         // prefill cutoff (N_bt above it: the last prefill tile); pad: log2 W + 1 when W is a power of two, else 0
  double tile_step;
  double *a1, *c1, *a2, *b2, *c2, *mae;
  uint8_t *status;
  uint64_t *invalid_count;
  // workspace
  double *part;               // [blocks][cells][<=5] CTA partials
  double *red;                // [cells][<=5] grid sums
  double *means;              // [cells][3]
  uint64_t *cnt;              // [cells]
  uint32_t *ticket;           // [3] CTAs finished per pass (zeroed by the call; reset by the last CTA)
};

int fit_warps_per_block(int cells);
cudaError_t launch_fit(const FitParams &P, int blocks, int wpb, cudaStream_t st, int *launches);

}  // namespace vt
