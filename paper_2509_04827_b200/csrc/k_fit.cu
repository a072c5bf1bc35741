// k_fit.cu — K1 (voltana_fit_profile): EcoPred least squares per cell.
//
// One cooperative launch, three streaming passes over the sample SoA (HBM-bound, 23 B/sample/pass):
//   pass 1: per-cell count and sums of x1, x2 (exact u64) and y       -> means
//   pass 2: per-cell centred S11, S12, S22, S1y, S2y                  -> OLS solve
//   pass 3: per-cell sum |y - y_hat|                                   -> MAE
// Each warp owns a contiguous sample range (a multiple of 128 samples) and streams it in chunks
// of 128: lane l loads samples 4l..4l+3 of the chunk with one vector load per field (a u32 of
// four phases, a u64 of four levels, a uint4 per count array, two double2 of latencies), a
// few chunks ahead. A chunk whose 128 samples are one cell (the usual case: calibration samples
// come run by run) is added into registers (each lane sums its own samples in order); at
// the end of the run a fixed binary tree over the lanes adds it to the warp's row of that cell.
// Any other chunk goes sample slot by sample slot (j = 0..3): runs of consecutive lanes of one
// cell are summed by a segmented scan over the lanes (a fixed tree) and added to the row by the
// run's last lane; runs of one cell that are not contiguous (shuffled input) are ranked with
// __match_any_sync and add in lane order. A row is written, not added, at its cell's first touch
// in a pass: no zeroing. The rows (cells x 5 doubles per warp) live in global memory, private to the warp
// (L1/L2-resident, touched only at run ends and mixed chunks), with a touched-cell bitmap per
// warp in shared memory; so the per-warp state does not limit the occupancy (16 warps per SM).
// Every warp partial is a fixed sum, independent of timing (no fp64 atomics). Between passes the grid synchronises
// (the launch is cooperative, every CTA resident): each CTA writes its partial (warps combined
// in warp order), every warp of the grid then reduces some (cell, stat) pairs over the CTA
// partials in CTA order (lane-strided sums and a fixed xor tree), and after a second barrier
// every CTA computes the pass's epilogue (means; the OLS solve of F2-F4) into its own
// shared-memory tables for the next pass — the same arithmetic in every CTA, so no third
// barrier; CTA 0 writes the outputs. Result within 1e-12 of the sequential oracle and
// bit-identical run to run.
#include <cstdint>
#include <mutex>

#include "vt_device.cuh"
#include "vt_fit.h"

#ifndef VT_FIT_PF
#define VT_FIT_PF 1
#endif

namespace vt {

constexpr int FIT_CH = 128;  // samples per chunk (32 lanes x 4)

struct Sample {
  int cell;          // -1 = padding (beyond the range), -2 = invalid sample
  uint32_t x1, x2;
  double y;
};

// four consecutive samples of one lane (raw fields)
struct Raw4 {
  uint32_t ph;       // 4 x u8
  uint2 lv;          // 4 x u16
  uint4 nb, nr, kv;
  double y[4];
  uint32_t nvalid;   // samples of the four below the range end
};

__device__ __forceinline__ uint32_t comp(const uint4 &v, int j) { return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w)); }

// Load samples i0..i0+3 (i0 = chunk base + 4 lane). Vector loads when the whole chunk lies
// below n and the arrays are aligned (host-checked, P.vec); else element by element.
__device__ __forceinline__ Raw4 load_raw4(const FitParams &P, size_t cb, size_t hi) {
  Raw4 r;
  const size_t i0 = cb + 4u * (size_t)lane_id();
  r.nvalid = i0 >= hi ? 0u : (hi - i0 >= 4 ? 4u : (uint32_t)(hi - i0));
  if (P.vec && cb + FIT_CH <= P.n) {
    r.ph = __ldcs((const unsigned int *)(P.phase + i0));
    const uint64_t l = __ldcs((const unsigned long long *)(P.level + i0));
    r.lv = make_uint2((uint32_t)l, (uint32_t)(l >> 32));
    r.nb = __ldcs((const uint4 *)(P.n_bt + i0));
    r.nr = __ldcs((const uint4 *)(P.n_req + i0));
    r.kv = __ldcs((const uint4 *)(P.n_kv + i0));
    const double2 a = __ldcs((const double2 *)(P.lat + i0)), b = __ldcs((const double2 *)(P.lat + i0 + 2));
    r.y[0] = a.x; r.y[1] = a.y; r.y[2] = b.x; r.y[3] = b.y;
    return r;
  }
  r.ph = 0; r.lv = make_uint2(0, 0); r.nb = r.nr = r.kv = make_uint4(0, 0, 0, 0);
  uint32_t nb[4] = {0, 0, 0, 0}, nr[4] = {0, 0, 0, 0}, kv[4] = {0, 0, 0, 0}, lv[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    r.y[j] = 0.0;
    if ((uint32_t)j < r.nvalid) {
      r.ph |= (uint32_t)P.phase[i0 + j] << (8 * j);
      lv[j] = P.level[i0 + j];
      nb[j] = P.n_bt[i0 + j]; nr[j] = P.n_req[i0 + j]; kv[j] = P.n_kv[i0 + j];
      r.y[j] = P.lat[i0 + j];
    }
  }
  r.lv = make_uint2(lv[0] | lv[1] << 16, lv[2] | lv[3] << 16);
  r.nb = make_uint4(nb[0], nb[1], nb[2], nb[3]);
  r.nr = make_uint4(nr[0], nr[1], nr[2], nr[3]);
  r.kv = make_uint4(kv[0], kv[1], kv[2], kv[3]);
  return r;
}

// sample j of a lane's four: cell key (F1 prefill tiles, tile of N_req for ITL cells), x, y
__device__ __forceinline__ Sample decode_j(const FitParams &P, const Raw4 &r, int j) {
  Sample s;
  s.cell = -1; s.x1 = 0; s.x2 = 0; s.y = 0.0;
  if ((uint32_t)j >= r.nvalid) return s;
  const uint32_t ph = (r.ph >> (8 * j)) & 0xffu;
  const uint32_t lv = ((j < 2 ? r.lv.x : r.lv.y) >> (16 * (j & 1))) & 0xffffu;
  const uint32_t nr = comp(r.nr, j);
  const uint32_t nb = ph == 0u ? comp(r.nb, j) : 1u;
  if (ph > 1u || lv >= (uint32_t)P.k || (ph == 1u && nr == 0u) || nb == 0u) { s.cell = -2; return s; }
  s.y = r.y[j];
  if (ph == 0u) {
    // prefill tile (F1): T_p <= 1 one tile; N_bt above the cutoff the last; else (N_bt-1)/W
    uint32_t jp = 0;
    if (P.n_ptiles > 1) jp = nb > P.pcut ? (uint32_t)P.n_ptiles - 1u : tile_of(nb, (uint32_t)P.tile_w, (uint32_t)P.n_ptiles);
    s.cell = (int)jp * P.k + (int)lv;
    s.x1 = nb;
  } else {
    uint32_t t = P.pad ? (nr - 1u) >> (P.pad - 1u) : (nr - 1u) / (uint32_t)P.tile_w;  // pad = log2 W + 1
    t = t < (uint32_t)P.n_tiles - 1u ? t : (uint32_t)P.n_tiles - 1u;
    s.cell = P.kp + (int)t * P.k + (int)lv;
    s.x1 = nr;
    s.x2 = comp(r.kv, j);
  }
  return s;
}

// per-CTA tables of the epilogues (shared memory), read by the next pass
struct FitTabs {
  double *means;    // [cells][3]   pass 1 -> pass 2
  double *coef;     // [cells][3]   a, b, c (TTFT cells: a1, c1, 0): pass 2 -> pass 3
  uint64_t *cnt;    // [cells]
  uint8_t *status;  // [cells]
};

// the pass's per-sample values: pass 1 {y} (x sums are integers), pass 2 the centred products,
// pass 3 |y - y_hat|
template <int PASS, int NS>
__device__ __forceinline__ void sample_values(const FitParams &P, const FitTabs &T, const Sample &s, double *v) {
#pragma unroll
  for (int q = 0; q < NS; ++q) v[q] = 0.0;
  if (s.cell < 0) return;
  if (PASS == 1) {
    v[3] = s.y;
  } else if (PASS == 2) {
    const double *m = T.means + 3 * s.cell;
    const double dx1 = sub((double)s.x1, m[0]);
    const double dy = sub(s.y, m[2]);
    v[0] = mul(dx1, dx1);
    v[4] = mul(dx1, dy);   // S1y
    if (s.cell >= P.kp) {
      const double dx2 = sub((double)s.x2, m[1]);
      v[1] = mul(dx1, dx2);
      v[2] = mul(dx2, dx2);
      v[3] = mul(dx2, dy);
    }
  } else {
    const double *c = T.coef + 3 * s.cell;
    const double yh = s.cell < P.kp ? ttft_pred(c[0], c[1], s.x1) : itl_pred(c[0], c[1], c[2], s.x1, s.x2);
    v[0] = fabs(sub(s.y, yh));
  }
}

// one streaming pass of this warp over [lo, hi) into its rows acc[cells][NS] (global memory,
// private to the warp; bm marks the cells it touched)
template <int PASS>
__device__ void stream_pass(const FitParams &P, const FitTabs &T, double *acc, uint32_t *bm, size_t lo, size_t hi,
                            uint64_t &invalid) {
  constexpr int NS = PASS == 1 ? 4 : (PASS == 2 ? 5 : 1);
  const int lane = lane_id();
  constexpr int PF = VT_FIT_PF;  // chunks loaded ahead (processed strictly in order)
  Raw4 buf[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) buf[u] = load_raw4(P, lo + (size_t)u * FIT_CH, hi);
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
      const bool first = !((bm[run_cell >> 5] >> (run_cell & 31)) & 1u);   // the row is written, not added
      atomicOr(bm + (run_cell >> 5), 1u << (run_cell & 31));
      VT_CHECK(run_cell >= 0 && run_cell < P.cells);
      double *a = acc + (size_t)run_cell * NS;
      if (PASS == 1) {
        uint64_t *u = (uint64_t *)a;
        u[0] = (first ? 0u : u[0]) + rcnt * (uint64_t)FIT_CH;
        u[1] = (first ? 0u : u[1]) + x1;
        u[2] = (first ? 0u : u[2]) + x2;
        a[3] = first ? t[3] : add(a[3], t[3]);
      } else {
#pragma unroll
        for (int q = 0; q < NS; ++q) a[q] = first ? t[q] : add(a[q], t[q]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NS; ++q) racc[q] = 0.0;
    rx1 = rx2 = rcnt = 0;
    run_cell = -1;
  };
  auto process = [&](const Raw4 &r) {
    Sample s[4];
    bool act[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      s[j] = decode_j(P, r, j);
      invalid += s[j].cell == -2 ? 1u : 0u;
      act[j] = s[j].cell >= 0 && (PASS != 3 || T.status[s[j].cell] == 0);
    }
    const int c0 = s[0].cell;
    const bool mine = act[0] && act[1] && act[2] && act[3] && s[1].cell == c0 && s[2].cell == c0 && s[3].cell == c0;
    const int c_l0 = __shfl_sync(FULL, c0, 0);   // every lane (not inside a short-circuit)
    if (__all_sync(FULL, mine && c0 == c_l0)) {
      // the whole chunk is one cell: extend (or start) the register run
      if (c0 != run_cell) { flush(); run_cell = c0; }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (PASS == 1) {
          rx1 += s[j].x1;
          rx2 += s[j].x2;
          racc[3] = add(racc[3], s[j].y);
        } else {
          double v[NS];
          sample_values<PASS, NS>(P, T, s[j], v);
#pragma unroll
          for (int q = 0; q < NS; ++q) racc[q] = add(racc[q], v[q]);
        }
      }
      rcnt += 1u;   // chunks of the run (FIT_CH samples each)
      return;
    }
    flush();
    // slot by slot (j = 0..3): runs of consecutive lanes of one cell (recording order: the few
    // cell boundaries of a chunk) are summed by a segmented inclusive scan over the lanes (five
    // shuffle steps, a fixed tree), and the run's last lane adds the run to the row; runs of
    // one cell that are not contiguous (shuffled input) are ranked with __match_any_sync and
    // add one at a time in lane order. The row is written, not added, at the cell's first touch.
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int key = act[j] ? s[j].cell : -1 - lane;
      double t[NS];
      sample_values<PASS, NS>(P, T, s[j], t);
      uint64_t x1 = s[j].x1, x2 = s[j].x2;
      const int pkey = __shfl_up_sync(FULL, key, 1);
      const unsigned heads = __ballot_sync(FULL, lane == 0 || pkey != key);
      const int start = 31 - __clz(heads & (0xFFFFFFFFu >> (31 - lane)));   // this run's first lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if (PASS == 1 && q < 3) continue;
          const double y = __shfl_up_sync(FULL, t[q], o);
          if (lane - o >= start) t[q] = add(y, t[q]);
        }
        if (PASS == 1) {
          const uint64_t y1 = __shfl_up_sync(FULL, x1, o), y2 = __shfl_up_sync(FULL, x2, o);
          if (lane - o >= start) { x1 += y1; x2 += y2; }
        }
      }
      const bool item = act[j] && (lane == 31 || ((heads >> (lane + 1)) & 1u));   // a run's last lane
      const unsigned peers = __match_any_sync(FULL, item ? key : -1 - lane);
      const unsigned rank = __popc(peers & ((1u << lane) - 1u));
      const unsigned maxr = __reduce_max_sync(FULL, item ? rank : 0u);
      for (unsigned rr = 0; rr <= maxr; ++rr) {
        if (item && rank == rr) {
          const int c = s[j].cell;
          const bool first = !((bm[c >> 5] >> (c & 31)) & 1u);   // the row is written, not added
          atomicOr(bm + (c >> 5), 1u << (c & 31));
          VT_CHECK(c >= 0 && c < P.cells && lane - start + 1 >= 1);
          double *a = acc + (size_t)c * NS;
          if (PASS == 1) {
            uint64_t *u = (uint64_t *)a;
            u[0] = (first ? 0u : u[0]) + (uint64_t)(lane - start + 1);
            u[1] = (first ? 0u : u[1]) + x1;
            u[2] = (first ? 0u : u[2]) + x2;
            a[3] = first ? t[3] : add(a[3], t[3]);
          } else {
#pragma unroll
            for (int q = 0; q < NS; ++q) a[q] = first ? t[q] : add(a[q], t[q]);
          }
        }
        __syncwarp();
      }
    }
  };
  for (size_t base = lo; base < hi; base += (size_t)PF * FIT_CH) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const size_t cb = base + (size_t)u * FIT_CH;
      if (cb >= hi) break;
      const Raw4 r = buf[u];
      buf[u] = load_raw4(P, cb + (size_t)PF * FIT_CH, hi);
      process(r);
    }
  }
  flush();
}

// grid-wide barrier of a cooperative launch: every CTA is resident; the counter is zeroed by
// the host before the launch and counts CTA arrivals monotonically (epoch = barriers x grid)
__device__ __forceinline__ void grid_sync(uint32_t *bar, uint32_t &epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= epoch) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// pass epilogues, computed by every CTA into its tables (CTA 0 also writes the outputs)
__device__ void fit_means(const FitParams &P, const FitTabs &T, const double *red) {
  for (int c = threadIdx.x; c < P.cells; c += blockDim.x) {
    const uint64_t cnt = ((const uint64_t *)red)[4 * (size_t)c];
    T.cnt[c] = cnt;
    double *m = T.means + 3 * (size_t)c;
    if (cnt > 0) {
      const double dc = (double)cnt;
      m[0] = div((double)((const uint64_t *)red)[4 * (size_t)c + 1], dc);
      m[1] = div((double)((const uint64_t *)red)[4 * (size_t)c + 2], dc);
      m[2] = div(red[4 * (size_t)c + 3], dc);
    } else {
      m[0] = m[1] = m[2] = 0.0;
    }
  }
}

__device__ void fit_solve(const FitParams &P, const FitTabs &T, const double *red, bool out) {
  // thread k < K: TTFT level k over prefill tiles; thread K + k: ITL level k over tiles j = 0..T-1 (F4 chains)
  const int K = P.k, NT = P.n_tiles;
  for (int t = threadIdx.x; t < 2 * K; t += blockDim.x) {
    if (t < K) {  // TTFT level t over prefill tiles jp = 0..T_p-1 (empty jp > 0 inherits jp-1, F2)
      for (int jp = 0; jp < P.n_ptiles; ++jp) {
        const int c = jp * K + t;
        const double *m = T.means + 3 * (size_t)c;
        double a = 0.0, cc = 0.0;
        uint8_t st;
        const double s11 = red[5 * (size_t)c], s1y = red[5 * (size_t)c + 4];
        if (T.cnt[c] == 0) {
          if (jp == 0) st = 2;
          else { a = T.coef[3 * (c - K)]; cc = add(T.coef[3 * (c - K) + 1], P.tile_step); st = 1; }
        } else if (T.cnt[c] < 2 || !(s11 > 0.0)) st = 3;   // A31
        else {
          a = div(s1y, s11);
          cc = sub(m[2], mul(a, m[0]));
          st = 0;
        }
        T.coef[3 * c] = a; T.coef[3 * c + 1] = cc; T.coef[3 * c + 2] = 0.0; T.status[c] = st;
        if (out) { P.a1[c] = a; P.c1[c] = cc; P.status[c] = st; }
      }
      continue;
    }
    const int k = t - K;
    for (int j = 0; j < NT; ++j) {
      const int c = P.kp + j * K + k, o = j * K + k;
      const double *m = T.means + 3 * (size_t)c;
      const double *r = red + 5 * (size_t)c;
      double a = 0.0, b = 0.0, cc = 0.0;
      uint8_t st;
      if (T.cnt[c] == 0) {
        if (j == 0) st = 2;
        else {                                 // inherit tile j-1 plus the step (F4)
          a = T.coef[3 * (c - K)]; b = T.coef[3 * (c - K) + 1]; cc = add(T.coef[3 * (c - K) + 2], P.tile_step);
          st = 1;
        }
      } else {
        const double s11 = r[0], s12 = r[1], s22 = r[2], s2y = r[3], s1y = r[4];
        const double pr = mul(s11, s22);
        const double det = sub(mul(s11, s22), mul(s12, s12));
        if (T.cnt[c] < 3 || !(pr > 0.0) || !(det > mul(1e-10, pr))) {
          st = 3;
        } else {
          a = div(sub(mul(s22, s1y), mul(s12, s2y)), det);
          b = div(sub(mul(s11, s2y), mul(s12, s1y)), det);
          cc = sub(sub(m[2], mul(a, m[0])), mul(b, m[1]));
          st = 0;
        }
      }
      T.coef[3 * c] = a; T.coef[3 * c + 1] = b; T.coef[3 * c + 2] = cc; T.status[c] = st;
      if (out) { P.a2[o] = a; P.b2[o] = b; P.c2[o] = cc; P.status[c] = st; }
    }
  }
}

// CTA partial of one pass (warps combined in warp order), then — after the grid barrier —
// every warp of the grid reduces its (cell, stat) pairs over the CTA partials in CTA order
template <int NS>
__device__ void cta_partial(const FitParams &P, uint32_t *bms, int wpb) {
  const int C = P.cells;
  double *out = P.part + (size_t)blockIdx.x * C * NS;
  double *rows = P.rows + (size_t)blockIdx.x * wpb * C * 5;   // this CTA's warps' rows, [w][cells][5]
  for (int x = threadIdx.x; x < C * NS; x += blockDim.x) {
    const int cell = x / NS;
    uint64_t su = 0;
    double sd = 0.0;
    for (int w = 0; w < wpb; ++w) {
      if (!((bms[w * P.bmw + (cell >> 5)] >> (cell & 31)) & 1u)) continue;   // untouched: zero
      double *r = rows + ((size_t)w * C * 5 + x);
      if (NS == 4 && (x % NS) < 3) su += *(const uint64_t *)r;
      else sd = add(sd, *r);
    }
    if (NS == 4 && (x % NS) < 3) ((uint64_t *)out)[x] = su;
    else out[x] = sd;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < wpb * P.bmw; x += blockDim.x) bms[x] = 0u;
}

template <int NS>
__device__ void grid_reduce(const FitParams &P, int wpb) {
  const int lane = lane_id();
  const size_t stride = (size_t)P.cells * NS;
  const int nb = (int)gridDim.x;
  const size_t tw = (size_t)gridDim.x * wpb, gw = (size_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  constexpr int RB = 16;   // CTA partials per lane loaded before any add (nb <= 32 RB)
  if (nb <= 32) {          // a small grid: one thread per (cell, stat), the CTA partials in CTA order
    for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < stride; x += (size_t)gridDim.x * blockDim.x) {
      uint64_t vb[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) vb[b] = b < nb ? __ldcg((const unsigned long long *)P.part + (size_t)b * stride + x) : 0ull;
      if (NS == 4 && (x % NS) < 3) {
        uint64_t s = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) s += vb[b];
        ((uint64_t *)P.red)[x] = s;
      } else {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 32; ++b)
          if (b < nb) s = add(s, __longlong_as_double((long long)vb[b]));
        P.red[x] = s;
      }
    }
    return;
  }
  for (size_t x = gw; x < stride; x += tw) {
    const bool isu = NS == 4 && (x % NS) < 3;
    uint64_t vb[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int b = lane + 32 * q;
      vb[q] = b < nb ? __ldcg((const unsigned long long *)P.part + (size_t)b * stride + x) : 0ull;
    }
    if (isu) {
      uint64_t s = 0;
#pragma unroll
      for (int q = 0; q < RB; ++q) s += vb[q];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
      if (lane == 0) ((uint64_t *)P.red)[x] = s;
    } else {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < RB; ++q)
        if (lane + 32 * q < nb) s = add(s, __longlong_as_double((long long)vb[q]));
      for (int o = 16; o > 0; o >>= 1) s = add(s, __shfl_xor_sync(FULL, s, o));   // same value in every lane
      if (lane == 0) P.red[x] = s;
    }
  }
}

// the grid sums of one pass into this CTA's shared memory (the epilogue reads them there)
__device__ void stage_red(const FitParams &P, double *red_s, int n) {
  for (int x = threadIdx.x; x < n; x += blockDim.x) red_s[x] = __ldcg(P.red + x);
  __syncthreads();
}

__global__ void __launch_bounds__(FIT_MAX_WARPS * 32, FIT_CTAS_PER_SM) fit_kernel(const __grid_constant__ FitParams P) {
  extern __shared__ double sm[];
  const int C = P.cells;
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int lane = lane_id();
  // shared memory: red [cells][5] | means [cells][3] | coef [cells][3] | cnt [cells] | touched bitmaps [wpb][bmw] |
  // status [cells]
  double *red_s = sm;
  FitTabs T;
  T.means = sm + (size_t)C * 5;
  T.coef = T.means + (size_t)C * 3;
  T.cnt = (uint64_t *)(T.coef + (size_t)C * 3);
  uint32_t *bms = (uint32_t *)(T.cnt + C);
  T.status = (uint8_t *)(bms + wpb * P.bmw);
  uint32_t *bm = bms + wib * P.bmw;
  const size_t gw = (size_t)blockIdx.x * wpb + wib;
  VT_CHECK(P.bmw == (C + 31) / 32 && P.chunk % FIT_CH == 0);
  // this warp's rows (global, private to the warp): a cell's row is written at its first touch
  // in a pass (touched bitmap), so no zeroing; cta_partial reads only touched rows
  double *acc = P.rows + gw * C * 5;
  for (int x = threadIdx.x; x < wpb * P.bmw; x += blockDim.x) bms[x] = 0u;
  __syncthreads();
  const size_t lo0 = gw * P.chunk;
  const size_t lo = lo0 < P.n ? lo0 : P.n, hi = lo0 + P.chunk < P.n ? lo0 + P.chunk : P.n;
  uint32_t epoch = 0;
  uint64_t invalid = 0;
  // ---------------------------------------------------------------- pass 1: counts, sums -> means
  stream_pass<1>(P, T, acc, bm, lo, hi, invalid);
  for (int o = 16; o > 0; o >>= 1) invalid += __shfl_xor_sync(FULL, invalid, o);
  if (lane == 0 && invalid && P.invalid_count) atomicAdd((unsigned long long *)P.invalid_count, invalid);
  __syncthreads();
  cta_partial<4>(P, bms, wpb);
  grid_sync(P.ticket, epoch);
  grid_reduce<4>(P, wpb);
  grid_sync(P.ticket, epoch);
  stage_red(P, red_s, 4 * C);
  fit_means(P, T, red_s);
  __syncthreads();
  // ---------------------------------------------------------------- pass 2: centred sums -> OLS
  stream_pass<2>(P, T, acc, bm, lo, hi, invalid);
  __syncthreads();
  cta_partial<5>(P, bms, wpb);
  grid_sync(P.ticket, epoch);
  grid_reduce<5>(P, wpb);
  grid_sync(P.ticket, epoch);
  stage_red(P, red_s, 5 * C);
  fit_solve(P, T, red_s, blockIdx.x == 0);
  __syncthreads();
  // ---------------------------------------------------------------- pass 3: |residual| -> MAE
  stream_pass<3>(P, T, acc, bm, lo, hi, invalid);
  __syncthreads();
  cta_partial<1>(P, bms, wpb);
  grid_sync(P.ticket, epoch);
  grid_reduce<1>(P, wpb);
  grid_sync(P.ticket, epoch);
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < C; c += blockDim.x)
      P.mae[c] = T.status[c] == 0 ? div(__ldcg(P.red + c), (double)T.cnt[c]) : 0.0;
}

size_t fit_smem_bytes(int cells, int wpb) {
  return (size_t)cells * (11 * sizeof(double) + sizeof(uint64_t)) + (size_t)wpb * ((cells + 31) / 32) * 4 +
         ((size_t)cells + 15) / 16 * 16;
}

int fit_warps_per_block(int cells) {
  (void)cells;
  return FIT_MAX_WARPS;
}

// cudaFuncSetAttribute for the dynamic shared memory, once per (device, size): host-side cost
static cudaError_t set_fit_smem(size_t smem) {
  static std::mutex mu;
  static size_t done[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (dev >= 0 && dev < 64 && smem <= done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = smem;
  return e;
}

int fit_max_blocks(int cells, int wpb) {
  static std::mutex mu;
  static int c_cells = -1, c_wpb = -1, c_dev = -1, c_val = 0;
  const size_t smem = fit_smem_bytes(cells, wpb);
  if (smem > 227 * 1024) return 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  {
    std::lock_guard<std::mutex> g(mu);
    if (cells == c_cells && wpb == c_wpb && dev == c_dev) return c_val;
  }
  if (set_fit_smem(smem) != cudaSuccess) { cudaGetLastError(); return 0; }
  int nb = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fit_kernel, wpb * 32, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  std::lock_guard<std::mutex> g(mu);
  c_cells = cells; c_wpb = wpb; c_dev = dev; c_val = nb * sms;
  return c_val;
}

cudaError_t launch_fit(const FitParams &P, int blocks, int wpb, cudaStream_t st, int *launches) {
  const size_t smem = fit_smem_bytes(P.cells, wpb);
  cudaError_t e = set_fit_smem(smem);
  if (e != cudaSuccess) return e;
  FitParams Pc = P;
  void *args[] = {&Pc};
  e = cudaLaunchCooperativeKernel((const void *)fit_kernel, dim3(blocks), dim3(wpb * 32), args, smem, st);
  *launches = 1;
  return e;
}

}  // namespace vt
