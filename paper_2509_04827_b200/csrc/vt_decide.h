// vt_decide.h — launch parameters of K2 (control_step) and K3 (route_batch).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voltana.h"
#include "vt_device.cuh"

namespace vt {

constexpr int DECIDE_THREADS = 256;
#ifndef VT_DECIDE_UNROLL
#define VT_DECIDE_UNROLL 2
#endif
constexpr int DECIDE_UNROLL = VT_DECIDE_UNROLL;  // items per thread per tile (independent loads in flight)

struct LadderParam {
  int32_t k;
  uint16_t level[VOLTANA_MAX_LEVELS];
};

struct ControlParams {
  DevProfile prof;
  LadderParam lad;
  const uint32_t *load, *n_kv, *queue_len;
  const double *wait, *target;
  size_t n;
  uint16_t *out_level;
  uint8_t *out_status;
  int32_t mode;        // 0 EcoFreq lowest feasible, 1 energy argmin [B4]
};

struct RouteParams {
  DevProfile prof;
  LadderParam lad;
  int32_t n_d, policy, delta, pad;   // pad: 1 = n_req / n_kv are 8-byte aligned (vector loads)
  const uint32_t *n_req, *n_kv, *req_in;
  const double *target;
  uint32_t *cursor;
  size_t n;
  uint16_t *out_instance;
  uint8_t *out_case, *out_status;
};

size_t decide_smem_bytes(int k, int n_tiles, int n_ptiles);
cudaError_t launch_control(const ControlParams &P, int phase, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_route(const RouteParams &P, int grid, size_t smem, cudaStream_t st);

}  // namespace vt
