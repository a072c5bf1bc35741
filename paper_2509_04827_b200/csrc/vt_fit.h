// vt_fit.h — launch parameters of K1 (voltana_fit_profile).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vt {

constexpr int FIT_MAX_WARPS = 8; 
constexpr int FIT_CTAS_PER_SM = 2;   // co-resident CTAs per SM (<= 128 registers); the workspace is sized for it   // warps per CTA (the per-warp rows usually allow fewer)

struct FitParams {
  const uint8_t *phase;
  const uint16_t *level;
  const uint32_t *n_bt, *n_req, *n_kv;
  const double *lat;
  size_t n, chunk;            // samples, samples per warp (a multiple of 128)
  int32_t vec;                // 1: vector loads (phase 4-B, level 8-B, counts and latencies 16-B aligned)
  int32_t k, n_tiles, tile_w, cells;
  int32_t n_ptiles, kp;       // prefill tiles T_p (>= 1) and TTFT cells kp = T_p * k [F1]
  uint32_t pcut, pad;         // prefill cutoff (N_bt above it: the last prefill tile); pad: log2 W + 1 when W is a power of two, else 0
  double tile_step;
  double *a1, *c1, *a2, *b2, *c2, *mae;
  uint8_t *status;
  uint64_t *invalid_count;
  // workspace
  double *rows;               // [blocks * warps][cells][5] per-warp accumulator rows (zeroed in the kernel)
  int32_t bmw;                // words of a warp's touched-cell bitmap = ceil(cells / 32)
  double *part;               // [blocks][cells][<=5] CTA partials
  double *red;                // [cells][<=5] grid sums
  double *means;              // [cells][3]
  uint64_t *cnt;              // [cells]
  uint32_t *ticket;           // [4] grid-barrier counter (zeroed by the call before the launch)
};

int fit_warps_per_block(int cells);               // warps per CTA whose rows fit the shared memory
size_t fit_smem_bytes(int cells, int wpb);        // dynamic shared memory of one CTA
int fit_max_blocks(int cells, int wpb);           // co-resident CTAs on this device (0: unknown / no GPU)
// one cooperative launch (every CTA resident: grid barriers between the passes)
cudaError_t launch_fit(const FitParams &P, int blocks, int wpb, cudaStream_t st, int *launches);

}  // namespace vt
