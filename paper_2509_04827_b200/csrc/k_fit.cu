// k_fit.cu — K1 (voltana_fit_profile): EcoPred least squares per cell.
//
// Three streaming passes over the sample SoA (HBM-bound, 23 B/sample/pass):
//   pass 1: per-cell count and sums of x1, x2 (exact u64) and y       -> means
//   pass 2: per-cell centred S11, S12, S22, S1y, S2y                  -> OLS solve
//   pass 3: per-cell sum |y - y_hat|                                   -> MAE
// Determinism without fp64 atomics: every warp owns a contiguous sample range and a
// private shared-memory accumulator row per cell. Consecutive 32-sample chunks of one cell (the
// usual case: calibration samples come run by run) accumulate in registers, each lane
// summing its own samples in order, and at the end of the run a fixed binary tree over the
// lanes adds them to the row; otherwise lanes of equal cell are ranked with __match_any_sync and
// add in ascending lane order (one round per rank; lanes of one round touch distinct cells). Warp partials are combined in warp order per
// CTA, CTA partials in CTA order per cell: a fixed tree, independent of timing.
#include <cstdint>

#include "vt_device.cuh"
#include "vt_fit.h"

#ifndef VT_FIT_PF
#define VT_FIT_PF 8
#endif

namespace vt {

struct Sample {
  int cell;          // -1 = invalid / out of range
  uint32_t x1, x2;
  double y;
};

// A sample's raw fields: every load is unconditional, so the loads of the chunks ahead issue
// back to back (a load predicated on another load's value would stall the warp at issue).
struct Raw {
  uint8_t ph;
  uint16_t lv;
  uint32_t nb, nr, kv;
  double y;
  bool in;
};

__device__ __forceinline__ Raw load_raw(const FitParams &P, size_t i, bool in_range) {
  Raw r;
  r.in = in_range;
  r.ph = 0; r.lv = 0; r.nb = 0; r.nr = 0; r.kv = 0; r.y = 0.0;
  if (in_range) {  // predicate from the index only: the six loads issue together
    r.ph = P.phase[i]; r.lv = P.level[i];
    r.nb = P.n_bt[i]; r.nr = P.n_req[i]; r.kv = P.n_kv[i];
    r.y = P.lat[i];
  }
  return r;
}

__device__ __forceinline__ Sample decode_sample(const FitParams &P, const Raw &r) {
  Sample s;
  s.cell = -1; s.x1 = 0; s.x2 = 0; s.y = 0.0;
  if (!r.in) return s;
  const uint32_t ph = r.ph, lv = r.lv, nr = r.nr;
  const uint32_t nb = ph == 0u ? r.nb : 1u;
  if (ph > 1u || lv >= (uint32_t)P.k || (ph == 1u && nr == 0u) || nb == 0u) { s.cell = -2; return s; }
  s.y = r.y;
  if (ph == 0u) {
    // prefill tile (F1): T_p <= 1 one tile; N_bt above the cutoff the last; else (N_bt-1)/W
    uint32_t jp = 0;
    if (P.n_ptiles > 1) jp = nb > P.pcut ? (uint32_t)P.n_ptiles - 1u : tile_of(nb, (uint32_t)P.tile_w, (uint32_t)P.n_ptiles);
    s.cell = (int)jp * P.k + (int)lv;
    s.x1 = nb;
  } else {
    uint32_t j = P.pad ? (nr - 1u) >> (P.pad - 1u) : (nr - 1u) / (uint32_t)P.tile_w;  // pad = log2 W + 1
    j = j < (uint32_t)P.n_tiles - 1u ? j : (uint32_t)P.n_tiles - 1u;
    s.cell = P.kp + (int)j * P.k + (int)lv;
    s.x1 = nr;
    s.x2 = r.kv;
  }
  return s;
}

// grid reduction of CTA partials in CTA order, one thread per (cell, stat): red[c][q]
template <int NS>
__device__ void grid_reduce(const FitParams &P, int nblocks) {
  const size_t stride = (size_t)P.cells * NS;
  for (int x = threadIdx.x; x < P.cells * NS; x += blockDim.x) {
    if (NS == 4 && (x % NS) < 3) {
      uint64_t s = 0;
      for (int b = 0; b < nblocks; ++b) s += __ldcg((const unsigned long long *)P.part + (size_t)b * stride + x);
      ((uint64_t *)P.red)[x] = s;
    } else {
      double s = 0.0;
      for (int b = 0; b < nblocks; ++b) s = add(s, __ldcg(P.part + (size_t)b * stride + x));
      P.red[x] = s;
    }
  }
}

__device__ void fit_means(const FitParams &P) {
  for (int c = threadIdx.x; c < P.cells; c += blockDim.x) {
  const uint64_t *u = (const uint64_t *)(P.red + 4 * (size_t)c);
  const uint64_t cnt = u[0];
  P.cnt[c] = cnt;
  double *m = P.means + 3 * (size_t)c;
  if (cnt > 0) {
    const double dc = (double)cnt;
    m[0] = div((double)u[1], dc);
    m[1] = div((double)u[2], dc);
    m[2] = div(P.red[4 * (size_t)c + 3], dc);
  } else {
    m[0] = m[1] = m[2] = 0.0;
  }
  }
}

__device__ void fit_solve(const FitParams &P) {
  // thread k < K: TTFT level k; thread K + k: ITL level k over tiles j = 0..T-1 (F4 chains)
  const int K = P.k, T = P.n_tiles;
  for (int t = threadIdx.x; t < 2 * K; t += blockDim.x) {
  if (t < K) {  // TTFT level t over prefill tiles jp = 0..T_p-1 (empty jp > 0 inherits jp-1, F2)
    for (int jp = 0; jp < P.n_ptiles; ++jp) {
      const int c = jp * K + t;
      const double *m = P.means + 3 * (size_t)c;
      const double *r = P.red + 5 * (size_t)c;
      double a = 0.0, cc = 0.0;
      uint8_t st;
      const double s11 = r[0], s1y = r[4];
      if (P.cnt[c] == 0) {
        if (jp == 0) st = 2;
        else { a = P.a1[c - K]; cc = add(P.c1[c - K], P.tile_step); st = 1; }
      } else if (P.cnt[c] < 2 || !(s11 > 0.0)) st = 3;   // A31
      else {
        a = div(s1y, s11);
        cc = sub(m[2], mul(a, m[0]));
        st = 0;
      }
      P.a1[c] = a; P.c1[c] = cc; P.status[c] = st;
    }
    continue;
  }
  const int k = t - K;
  for (int j = 0; j < T; ++j) {
    const int c = P.kp + j * K + k, o = j * K + k;
    const double *m = P.means + 3 * (size_t)c;
    const double *r = P.red + 5 * (size_t)c;
    double a = 0.0, b = 0.0, cc = 0.0;
    uint8_t st;
    if (P.cnt[c] == 0) {
      if (j == 0) st = 2;
      else {                                 // inherit tile j-1 plus the step (F4)
        a = P.a2[o - K]; b = P.b2[o - K]; cc = add(P.c2[o - K], P.tile_step);
        st = 1;
      }
    } else {
      const double s11 = r[0], s12 = r[1], s22 = r[2], s2y = r[3], s1y = r[4];
      const double pr = mul(s11, s22);
      const double det = sub(mul(s11, s22), mul(s12, s12));
      if (P.cnt[c] < 3 || !(pr > 0.0) || !(det > mul(1e-10, pr))) {
        st = 3;
      } else {
        a = div(sub(mul(s22, s1y), mul(s12, s2y)), det);
        b = div(sub(mul(s11, s2y), mul(s12, s1y)), det);
        cc = sub(sub(m[2], mul(a, m[0])), mul(b, m[1]));
        st = 0;
      }
    }
    P.a2[o] = a; P.b2[o] = b; P.c2[o] = cc; P.status[c] = st;
  }
  }
}

__device__ void fit_mae(const FitParams &P) {
  for (int c = threadIdx.x; c < P.cells; c += blockDim.x)
    P.mae[c] = P.status[c] == 0 ? div(P.red[c], (double)P.cnt[c]) : 0.0;
}

// Ordered per-warp accumulation of NS doubles (pass 2/3) or the pass-1 record.
template <int PASS>
__global__ void __launch_bounds__(FIT_MAX_WARPS * 32) fit_pass_kernel(const __grid_constant__ FitParams P) {
  extern __shared__ double sm[];
  constexpr int NS = PASS == 1 ? 4 : (PASS == 2 ? 5 : 1);
  const int C = P.cells;
  const int lane = lane_id(), wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  double *acc = sm + (size_t)wib * C * NS;   // pass 1 stores u64 bit patterns in slots 0..2
  for (int x = lane; x < C * NS; x += 32) acc[x] = 0.0;
  __syncwarp();

  const size_t gw = (size_t)blockIdx.x * wpb + wib;
  const size_t lo = gw * P.chunk, hi = lo + P.chunk < P.n ? lo + P.chunk : P.n;
  uint64_t invalid = 0;
  constexpr int PF = VT_FIT_PF;  // 32-sample chunks loaded ahead (processed strictly in order)
  Raw buf[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) buf[u] = load_raw(P, lo + (size_t)u * 32 + lane, lo + (size_t)u * 32 + lane < hi);
  // a run of one-cell chunks accumulates in registers (lane l sums its own samples in order);
  // flush: a fixed tree over the lanes, added to the warp's row once per run
  int run_cell = -1;
  double racc[NS];
  uint64_t rx1 = 0, rx2 = 0, rcnt = 0;
#pragma unroll
  for (int q = 0; q < NS; ++q) racc[q] = 0.0;
  auto flush = [&]() {
    if (run_cell < 0) return;
    double t[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) t[q] = racc[q];
    uint64_t x1 = rx1, x2 = rx2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        if (PASS == 1 && q < 3) continue;
        const double y = __shfl_down_sync(FULL, t[q], o);
        if (lane < o) t[q] = add(t[q], y);
      }
      if (PASS == 1) {
        const uint64_t y1 = __shfl_down_sync(FULL, x1, o), y2 = __shfl_down_sync(FULL, x2, o);
        if (lane < o) { x1 += y1; x2 += y2; }
      }
    }
    if (lane == 0) {
      double *a = acc + (size_t)run_cell * NS;
      if (PASS == 1) {
        uint64_t *u = (uint64_t *)a;
        u[0] += rcnt * 32u;
        u[1] += x1;
        u[2] += x2;
        a[3] = add(a[3], t[3]);
      } else {
#pragma unroll
        for (int q = 0; q < NS; ++q) a[q] = add(a[q], t[q]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NS; ++q) racc[q] = 0.0;
    rx1 = rx2 = rcnt = 0;
    run_cell = -1;
  };
  // chunk processing (in sample order); the PF chunks ahead sit in a ring of registers, refilled
  // slot by slot in a loop unrolled by PF (no register shifting)
  auto process = [&](const Sample &s) {
    if (s.cell == -2) invalid++;
    double v[NS];
    if (PASS == 1) {
      v[0] = 0; v[1] = 0; v[2] = 0; v[3] = s.y;
    } else if (PASS == 2) {
      if (s.cell >= 0) {
        const double *m = P.means + 3 * (size_t)s.cell;
        double dx1 = sub((double)s.x1, m[0]);
        double dy = sub(s.y, m[2]);
        v[0] = mul(dx1, dx1);
        v[4] = mul(dx1, dy);   // S1y
        if (s.cell >= P.kp) {
          double dx2 = sub((double)s.x2, m[1]);
          v[1] = mul(dx1, dx2);
          v[2] = mul(dx2, dx2);
          v[3] = mul(dx2, dy);
        } else {
          v[1] = v[2] = v[3] = 0.0;
        }
      }
    } else {
      if (s.cell >= 0 && P.status[s.cell] == 0) {
        double yh;
        if (s.cell < P.kp) {
          yh = ttft_pred(P.a1[s.cell], P.c1[s.cell], s.x1);
        } else {
          int o = s.cell - P.kp;
          yh = itl_pred(P.a2[o], P.b2[o], P.c2[o], s.x1, s.x2);
        }
        v[0] = fabs(sub(s.y, yh));
      } else {
        v[0] = 0.0;
      }
    }
    const bool act = s.cell >= 0 && (PASS != 3 || P.status[s.cell] == 0);
    const int key = act ? s.cell : -1 - lane;
    const unsigned peers = __match_any_sync(FULL, key);
    if (peers == FULL) {   // the whole chunk is one cell: extend (or start) the register run
      if (s.cell != run_cell) { flush(); run_cell = s.cell; }
      if (PASS == 1) {
        rx1 += s.x1;
        rx2 += s.x2;
        rcnt += 1u;
        racc[3] = add(racc[3], v[3]);
      } else {
#pragma unroll
        for (int q = 0; q < NS; ++q) racc[q] = add(racc[q], v[q]);
      }
      return;
    }
    flush();
    const unsigned rank = __popc(peers & ((1u << lane) - 1u));
    const unsigned maxr = __reduce_max_sync(FULL, act ? rank : 0u);
    for (unsigned r = 0; r <= maxr; ++r) {
      if (act && rank == r) {
        double *a = acc + (size_t)s.cell * NS;
        if (PASS == 1) {
          uint64_t *u = (uint64_t *)a;
          u[0] += 1u;
          u[1] += s.x1;
          u[2] += s.x2;
          a[3] = add(a[3], v[3]);
        } else {
#pragma unroll
          for (int q = 0; q < NS; ++q) a[q] = add(a[q], v[q]);
        }
      }
      __syncwarp();
    }
    };
  for (size_t base = lo; base < hi; base += (size_t)PF * 32) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const size_t cb = base + (size_t)u * 32;
      if (cb >= hi) break;
      const Sample s = decode_sample(P, buf[u]);
      const size_t ni = cb + (size_t)PF * 32 + lane;
      buf[u] = load_raw(P, ni, ni < hi);
      process(s);
    }
  }
  flush();
  if (PASS == 1) {
    for (int o = 16; o > 0; o >>= 1) invalid += __shfl_xor_sync(FULL, invalid, o);
    if (lane == 0 && invalid && P.invalid_count) atomicAdd((unsigned long long *)P.invalid_count, invalid);
  }
  __syncthreads();
  // CTA partial: warps combined in warp order, one thread per (cell, stat)
  double *out = P.part + (size_t)blockIdx.x * C * NS;
  for (int x = threadIdx.x; x < C * NS; x += blockDim.x) {
    const int stat = x % NS;
    if (PASS == 1 && stat < 3) {
      uint64_t s = 0;
      for (int w = 0; w < wpb; ++w) s += ((const uint64_t *)(sm + (size_t)w * C * NS))[x];
      ((uint64_t *)out)[x] = s;
    } else {
      double s = 0.0;
      for (int w = 0; w < wpb; ++w) s = add(s, sm[(size_t)w * C * NS + x]);
      out[x] = s;
    }
  }
  // the last CTA to finish reduces the partials in CTA order and runs this pass's epilogue
  // (one launch per pass; the order of the sums does not depend on which CTA is last)
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(P.ticket + (PASS - 1), 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  grid_reduce<NS>(P, (int)gridDim.x);
  __syncthreads();
  if (PASS == 1) fit_means(P);
  else if (PASS == 2) fit_solve(P);
  else fit_mae(P);
  if (threadIdx.x == 0) P.ticket[PASS - 1] = 0u;   // ready for the next call
}

int fit_warps_per_block(int cells) {
  // pass 2 needs 40 B per cell per warp; keep <= 200 KB of shared memory per CTA
  int w = (int)(200 * 1024 / ((size_t)cells * 40));
  if (w > FIT_MAX_WARPS) w = FIT_MAX_WARPS;
  return w < 1 ? 1 : w;
}

template <int PASS>
static cudaError_t launch_pass(const FitParams &P, int blocks, int wpb, cudaStream_t st) {
  constexpr int NS = PASS == 1 ? 4 : (PASS == 2 ? 5 : 1);
  size_t smem = (size_t)wpb * P.cells * NS * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(fit_pass_kernel<PASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fit_pass_kernel<PASS><<<blocks, wpb * 32, smem, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_fit(const FitParams &P, int blocks, int wpb, cudaStream_t st, int *launches) {
  cudaError_t e;
  if ((e = launch_pass<1>(P, blocks, wpb, st)) != cudaSuccess) return e;   // + means
  if ((e = launch_pass<2>(P, blocks, wpb, st)) != cudaSuccess) return e;   // + OLS solve
  if ((e = launch_pass<3>(P, blocks, wpb, st)) != cudaSuccess) return e;   // + MAE
  *launches = 3;
  return cudaGetLastError();
}

}  // namespace vt
