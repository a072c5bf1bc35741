// vt_device.cuh — device building blocks shared by the sm_100a kernels of libvoltana.
// (Product code only: nothing here is shared with oracle/.)
//
// Canonical arithmetic (A33): IEEE fp64, each operation rounded
// separately. The library is compiled with -fmad=false and every predictor /
// energy expression below uses the explicit _rn intrinsics, so no FMA can be formed.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Bounds checks of a checked build (-DVT_CHECKS, tools/variants.py checks=VT_CHECKS=1): a failed
// check prints its site and traps the kernel. Compiled out of the product build.
#ifdef VT_CHECKS
#define VT_CHECK(c)                                                                               \
  do {                                                                                            \
    if (!(c)) {                                                                                   \
      printf("VT_CHECK failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__,       \
             (int)blockIdx.x, (int)threadIdx.x);                                                  \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define VT_CHECK(c) do { } while (0)
#endif

#include "../../include/voltana.h"

namespace vt {

constexpr uint32_t NIL = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }

// Device-side copy of one profile (kernel parameter / constant bank).
struct DevProfile {
  int32_t k, n_tiles, tile_w, n_ptiles;  // n_ptiles >= 1 (prefill tiles, F1)
  const int32_t *mhz;
  const double *a1, *c1, *a2, *b2, *c2, *dyn;
  double p_idle, tdp, uh[2];
  uint32_t pcut, pad;                    // prefill cutoff (N_bt above it: the last prefill tile)
};

__host__ __device__ inline DevProfile to_dev(const voltana_profile &p) {
  DevProfile d;
  d.k = p.k; d.n_tiles = p.n_tiles; d.tile_w = p.tile_w; d.n_ptiles = p.n_ptiles < 1 ? 1 : p.n_ptiles;
  d.pcut = p.prefill_cutoff < 0 ? 0u : (uint32_t)p.prefill_cutoff; d.pad = 0;
  d.mhz = p.mhz; d.a1 = p.a1; d.c1 = p.c1; d.a2 = p.a2; d.b2 = p.b2; d.c2 = p.c2; d.dyn = p.dyn;
  d.p_idle = p.p_idle; d.tdp = p.tdp; d.uh[0] = p.u_half_prefill; d.uh[1] = p.u_half_decode;
  return d;
}

// tile j = min(T-1, (n_req-1)/W): batch-size boundaries at multiples of W (A21)
__device__ __forceinline__ uint32_t tile_of(uint32_t n_req, uint32_t tile_w, uint32_t n_tiles) {
  uint32_t j = (n_req - 1u) / tile_w;
  return j < n_tiles - 1u ? j : n_tiles - 1u;
}

// prefill tile (Appendix B; F1): one tile, or N_bt above the cutoff -> the last,
// else min(T_p - 1, (N_bt - 1) / W)
__device__ __forceinline__ uint32_t ptile_of(uint32_t n_bt, uint32_t tile_w, uint32_t n_ptiles, uint32_t pcut) {
  if (n_ptiles <= 1u) return 0u;
  if (n_bt > pcut) return n_ptiles - 1u;
  const uint32_t j = (n_bt - 1u) / tile_w;
  return j < n_ptiles - 1u ? j : n_ptiles - 1u;
}

// eq:pred-ttft: (a1 * N_bt) + c1
__device__ __forceinline__ double ttft_pred(double a1, double c1, uint32_t n_bt) {
  return add(mul(a1, (double)n_bt), c1);
}

// eq:pred-itl: ((a2 * N_req) + (b2 * N_kv)) + c2
__device__ __forceinline__ double itl_pred(double a2, double b2, double c2, uint32_t n_req,
                                           uint32_t n_kv) {
  return add(add(mul(a2, (double)n_req), mul(b2, (double)n_kv)), c2);
}

// busy power (eq:P-f P:187 as per-level tables, A22): min(TDP, P_idle + u * DYN)
__device__ __forceinline__ double busy_power(double p_idle, double tdp, double uh, double dyn,
                                             uint32_t load) {
  double u = div((double)load, add((double)load, uh));
  double w = add(p_idle, mul(u, dyn));
  return w < tdp ? w : tdp;
}

// energy = time x power: J from W and ms
__device__ __forceinline__ double energy_j(double w, double dur_ms) { return div(mul(w, dur_ms), 1000.0); }

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// decision hash fold (A36)
__device__ __forceinline__ uint64_t fold(uint64_t h, uint64_t kind, uint64_t inst, uint64_t level,
                                         uint64_t cse) {
  return (h ^ ((kind << 48) ^ (inst << 32) ^ (level << 16) ^ cse)) * 0x9E3779B97F4A7C15ull;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// lowest set bit index of a non-zero mask
__device__ __forceinline__ int ffs0(unsigned m) { return __ffs(m) - 1; }

}  // namespace vt
