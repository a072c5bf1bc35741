// k_series.cu — K5 (voltana_series_to_samples): the fit -> simulate loop.
//
// Maps every slot of voltana_simulate_ex's per-instance iteration series to one EcoPred
// calibration sample ("offline profiling", here from simulated — optionally noisy —
// executions): prefill iteration -> (phase 0, profile level, N_bt, latency); decode
// iteration -> (phase 1, profile level, N_req, N_kv, latency). Empty slots (j >= count)
// and scenarios of other profiles become phase 0xFF, which voltana_fit_profile skips and
// counts as invalid. One thread per slot, grid-stride, coalesced SoA stores; the slot's
// scenario is found by binary search over the ascending iter_offset.
#include <cstdint>

#include "vt_series.h"

namespace vt {

__global__ void __launch_bounds__(SERIES_THREADS) series_kernel(const __grid_constant__ SeriesParams P) {
  for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < P.n_slots; x += (size_t)gridDim.x * blockDim.x) {
    // scenario s: the last with iter_offset[s] <= x
    size_t lo = 0, hi = P.n;
    while (hi - lo > 1) {
      const size_t mid = (lo + hi) >> 1;
      if (P.iter_offset[mid] <= x) lo = mid; else hi = mid;
    }
    const size_t s = lo;
    const uint64_t rel = x - P.iter_offset[s];
    const uint32_t u = (uint32_t)(rel / P.cap), j = (uint32_t)(rel % P.cap);
    const uint32_t li = P.layout_id[s], gi = P.grid_id[s];
    const uint32_t np = (uint32_t)P.n_p[li];
    const uint64_t inst = P.iter_offset[s] / P.cap + u;
    bool ok = P.scen_profile_id[s] == P.profile_id && j < P.iter_count[inst];
    uint8_t ph = 0xFF;
    uint16_t lv = 0;
    uint32_t bt = 0, nr = 0, kv = 0;
    double y = 0.0;
    if (ok) {
      const voltana_iteration r = P.iters[x];
      ph = u < np ? 0 : 1;
      lv = P.grid[gi].level[r.level];
      if (ph == 0) bt = r.load;
      else { nr = r.load; kv = r.n_kv; }
      y = r.dur_ms;
    }
    P.phase[x] = ph; P.level[x] = lv; P.n_bt[x] = bt; P.n_req[x] = nr; P.n_kv[x] = kv; P.lat[x] = y;
  }
}

cudaError_t launch_series(const SeriesParams &P, int grid, cudaStream_t st) {
  series_kernel<<<grid, SERIES_THREADS, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace vt
