// k_decide.cu — K2 (voltana_control_step) and K3 (voltana_route_batch): streaming
// single-decision kernels over caller-provided SoA snapshots (HBM-bound).
//
// One thread per item, grid-stride, a few CTAs per SM. The scenario's ladder-resolved
// EcoPred tables are staged once per CTA in shared memory ([tile][level] rows of
// {a2,b2,c2}, or {a1,c1} for prefill), so the only HBM traffic is the snapshot
// stream itself: coalesced 4/8-byte SoA loads in, 2/1-byte SoA stores out.
// The level scan is the paper's ascending scan with early exit.
#include <cstdint>

#include "vt_decide.h"
#include "vt_device.cuh"

constexpr int ITS = 3;       // ITL rows {a2, b2, c2} per (tile, level)

namespace vt {

// ---------------------------------------------------------------- shared-memory tables
struct SmemTables {
  const double *tt;   // [K][2]: a1, c1
  const double *it;   // [T][K][3]: a2, b2, c2
  const int *mhz;     // [K]
};

// Layout (doubles): [T_p][K][2] a1,c1 | [T][K][3] a2,b2,c2 | [K] DYN row of `dyn_phase`;
// then int [K] MHz. T_p = prefill tiles (F1).
__device__ __forceinline__ int tt_len(int K, const DevProfile &PR) { return 2 * PR.n_ptiles * K; }
__device__ __forceinline__ double *itl_smem(double *sm, int K, const DevProfile &PR) { return sm + tt_len(K, PR); }
__device__ __forceinline__ double *dyn_smem(double *sm, int K, const DevProfile &PR) {
  return sm + tt_len(K, PR) + ITS * PR.n_tiles * K;
}
__device__ __forceinline__ int *mhz_smem(double *sm, int K, const DevProfile &PR) {
  return (int *)(sm + tt_len(K, PR) + ITS * PR.n_tiles * K + K);
}
// TTFT row {a1, c1}[K] of the batch's prefill tile
__device__ __forceinline__ const double *tt_row(const double *sm, int K, const DevProfile &PR, uint32_t nbt) {
  return sm + 2 * K * (int)ptile_of(nbt, (uint32_t)PR.tile_w, (uint32_t)PR.n_ptiles, PR.pcut);
}

__device__ void stage_tables(const DevProfile &PR, const LadderParam &LP, bool need_tt, bool need_it,
                             int dyn_phase, double *sm, int *smi) {
  const int K = LP.k, T = PR.n_tiles;
  double *dy = dyn_smem(sm, K, PR);
  for (int x = threadIdx.x; x < K; x += blockDim.x) {
    int lv = LP.level[x];
    if (dyn_phase >= 0) dy[x] = PR.dyn[dyn_phase * PR.k + lv];
    smi[x] = PR.mhz[lv];
  }
  if (need_tt) {
    for (int x = threadIdx.x; x < PR.n_ptiles * K; x += blockDim.x) {
      const int jp = x / K, k = x - jp * K;
      const size_t o = (size_t)jp * PR.k + LP.level[k];
      sm[2 * x] = PR.a1[o]; sm[2 * x + 1] = PR.c1[o];
    }
  }
  if (need_it) {
    double *it = itl_smem(sm, K, PR);
    for (int x = threadIdx.x; x < T * K; x += blockDim.x) {
      int j = x / K, k = x - j * K;
      size_t o = (size_t)j * PR.k + LP.level[k];
      it[ITS * x] = PR.a2[o]; it[ITS * x + 1] = PR.b2[o]; it[ITS * x + 2] = PR.c2[o];
    }
  }
  __syncthreads();
}

template <int KK>
__device__ __forceinline__ int scan_ttft_ilp(const double *tt, uint32_t nbt, double budget);

template <int KK = 0>
__device__ __forceinline__ int scan_ttft(const double *tt, int K, uint32_t nbt, double budget) {
  if (KK == 1) return 0;
  if (KK > 1) return scan_ttft_ilp<(KK > 1 ? KK : 2)>(tt, nbt, budget);
  switch (K) {
    case 1: return 0;
    case 2: return scan_ttft_ilp<2>(tt, nbt, budget);
    case 3: return scan_ttft_ilp<3>(tt, nbt, budget);
    case 4: return scan_ttft_ilp<4>(tt, nbt, budget);
    case 5: return scan_ttft_ilp<5>(tt, nbt, budget);
    case 6: return scan_ttft_ilp<6>(tt, nbt, budget);
    case 7: return scan_ttft_ilp<7>(tt, nbt, budget);
    case 8: return scan_ttft_ilp<8>(tt, nbt, budget);
    default: break;
  }
  for (int k = 0; k < K; ++k)
    if (ttft_pred(tt[2 * k], tt[2 * k + 1], nbt) <= budget) return k;
  return K - 1;
}

// 64-bit state: the what-if state (n+1, kv+in+1) may exceed 32 bits for caller data.
// Tile index by shift when the tile width is a power of two (wshift >= 0).
__device__ __forceinline__ const double *itl_row(const double *it, const DevProfile &PR, int K, uint64_t n,
                                                 int wshift) {
  uint64_t j = wshift >= 0 ? (n - 1u) >> wshift : (n - 1u) / (uint64_t)PR.tile_w;
  if (j > (uint64_t)(PR.n_tiles - 1)) j = (uint64_t)(PR.n_tiles - 1);
  return it + ITS * (size_t)j * K;
}
// Row of the tile holding N_req = m + 1 for a 32-bit m (the tile of n is row32(n - 1), of n + 1
// is row32(n): no 64-bit arithmetic and no overflow), power-of-two tile width.
__device__ __forceinline__ const double *itl_row32(const double *it, uint32_t m, int wshift, uint32_t tmax,
                                                   uint32_t row_len) {
  uint32_t j = m >> wshift;
  j = j < tmax ? j : tmax;
  return it + j * row_len;
}

__device__ __forceinline__ double itl_eval(const double *row, int k, double dn, double dkv) {
  return add(add(mul(row[3 * k], dn), mul(row[3 * k + 1], dkv)), row[3 * k + 2]);
}

__device__ __forceinline__ uint32_t itl_tile(const DevProfile &PR, uint64_t n, int wshift) {
  uint64_t j = wshift >= 0 ? (n - 1u) >> wshift : (n - 1u) / (uint64_t)PR.tile_w;
  return j > (uint64_t)(PR.n_tiles - 1) ? (uint32_t)(PR.n_tiles - 1) : (uint32_t)j;
}

// K <= 8: levels 0..K-2 evaluated without branches (independent, predicated selects from the
// top down = the lowest feasible level), else K-1 — the ascending scan's answer (A2).
// The threads of a warp no longer wait for the longest early-exit chain among them.
template <int KK>
__device__ __forceinline__ int scan_itl_ilp(const double *row, double dn, double dkv, double target) {
  int kk = KK - 1;
#pragma unroll
  for (int k = KK - 2; k >= 0; --k)
    if (itl_eval(row, k, dn, dkv) <= target) kk = k;
  return kk;
}
template <int KK>
__device__ __forceinline__ int scan_ttft_ilp(const double *tt, uint32_t nbt, double budget) {
  int kk = KK - 1;
#pragma unroll
  for (int k = KK - 2; k >= 0; --k)
    if (ttft_pred(tt[2 * k], tt[2 * k + 1], nbt) <= budget) kk = k;
  return kk;
}

template <int KK = 0>
__device__ __forceinline__ int scan_itl(const double *it, const DevProfile &PR, int K, uint64_t n,
                                        uint64_t kv, double target, int wshift) {
  const double *row = itl_row(it, PR, K, n, wshift);
  const double dn = (double)n, dkv = (double)kv;
  if (KK == 1) return 0;
  if (KK > 1) return scan_itl_ilp<(KK > 1 ? KK : 2)>(row, dn, dkv, target);
  switch (K) {
    case 1: return 0;
    case 2: return scan_itl_ilp<2>(row, dn, dkv, target);
    case 3: return scan_itl_ilp<3>(row, dn, dkv, target);
    case 4: return scan_itl_ilp<4>(row, dn, dkv, target);
    case 5: return scan_itl_ilp<5>(row, dn, dkv, target);
    case 6: return scan_itl_ilp<6>(row, dn, dkv, target);
    case 7: return scan_itl_ilp<7>(row, dn, dkv, target);
    case 8: return scan_itl_ilp<8>(row, dn, dkv, target);
    default: break;
  }
  for (int k = 0; k < K; ++k)
    if (itl_eval(row, k, dn, dkv) <= target) return k;
  return K - 1;
}

// EcoRoute's what-if pair of one instance (A10-A12): the lowest feasible level now (n, kv) and
// after the hypothetical addition (n + 1, kv + in + 1). Both states usually fall in the same
// batch-size tile, so each level's {a2, b2, c2} is loaded once and evaluated twice (the
// shared-memory loads, not the FP64 work, bound this kernel). Same values as two scans.
template <int KK>
__device__ __forceinline__ void scan_pair_ilp(const double *r0, const double *r1, double n0, double k0d, double n1,
                                              double k1d, double target, int &kn, int &ka) {
  kn = KK - 1;
  ka = KK - 1;
  if (r0 == r1) {
#pragma unroll
    for (int k = KK - 2; k >= 0; --k) {
      const double a = r0[3 * k], b = r0[3 * k + 1], c = r0[3 * k + 2];
      if (add(add(mul(a, n0), mul(b, k0d)), c) <= target) kn = k;
      if (add(add(mul(a, n1), mul(b, k1d)), c) <= target) ka = k;
    }
  } else {
#pragma unroll
    for (int k = KK - 2; k >= 0; --k) {
      if (itl_eval(r0, k, n0, k0d) <= target) kn = k;
      if (itl_eval(r1, k, n1, k1d) <= target) ka = k;
    }
  }
}

template <int KK = 0>
__device__ __forceinline__ void scan_pair(const double *it, const DevProfile &PR, int K, uint64_t n, uint64_t kv,
                                          uint64_t in, double target, int wshift, int &kn, int &ka) {
  const uint64_t n1 = n + 1u, kv1 = kv + in + 1u;  // A12
  const double *r0, *r1;
  if (KK > 0 && wshift >= 0) {   // 32-bit tile rows (n < 2^32 by type)
    const uint32_t tmax = (uint32_t)PR.n_tiles - 1u, rl = (uint32_t)(ITS * K);
    r1 = itl_row32(it, (uint32_t)n, wshift, tmax, rl);
    r0 = n == 0u ? r1 : itl_row32(it, (uint32_t)n - 1u, wshift, tmax, rl);
  } else {
    r1 = itl_row(it, PR, K, n1, wshift);
    r0 = n == 0u ? r1 : itl_row(it, PR, K, n, wshift);
  }
  // (n + 1, kv + in + 1) < 2^34: exact as doubles, so the successor is formed in fp64 (no 64-bit
  // integer adds and conversions); the values equal (double)n1 and (double)kv1
  const double dn0 = (double)n, dk0 = (double)kv, dn1 = add(dn0, 1.0), dk1 = add(dk0, (double)(in + 1u));
  if (KK == 1) { kn = 0; ka = 0; return; }
  if (KK > 1) {
    // both states with the row of n (the successor's tile differs only when n is a multiple of
    // the tile width: then f' is re-scanned on its own row, a rare, per-lane fix-up instead of
    // a second path the whole warp would execute)
    constexpr int KQ = KK > 1 ? KK : 2;
    const double *r = n == 0u ? r1 : r0;
    kn = KQ - 1;
    ka = KQ - 1;
#pragma unroll
    for (int k = KQ - 2; k >= 0; --k) {
      const double a = r[3 * k], b = r[3 * k + 1], c = r[3 * k + 2];
      if (add(add(mul(a, dn0), mul(b, dk0)), c) <= target) kn = k;
      if (add(add(mul(a, dn1), mul(b, dk1)), c) <= target) ka = k;
    }
    if (n == 0u) kn = 0;
    if (r1 != r) ka = scan_itl_ilp<KQ>(r1, dn1, dk1, target);
    return;
  }
  switch (K) {
    case 1: kn = 0; ka = 0; return;
    case 2: scan_pair_ilp<2>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 3: scan_pair_ilp<3>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 4: scan_pair_ilp<4>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 5: scan_pair_ilp<5>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 6: scan_pair_ilp<6>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 7: scan_pair_ilp<7>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    case 8: scan_pair_ilp<8>(r0, r1, dn0, dk0, dn1, dk1, target, kn, ka); break;
    default:
      kn = scan_itl<>(it, PR, K, n, kv, target, wshift);
      ka = scan_itl<>(it, PR, K, n1, kv1, target, wshift);
      break;
  }
  if (n == 0u) kn = 0;  // an idle instance: level 0 (A11)
}

// busy power (eq:P-f P:187, A22) for a 64-bit load
__device__ __forceinline__ double power_at(const DevProfile &PR, int phase, double dyn, uint64_t load) {
  const double u = div((double)load, add((double)load, PR.uh[phase]));
  const double w = add(PR.p_idle, mul(u, dyn));
  return w < PR.tdp ? w : PR.tdp;
}

// Energy-argmin controller [B4]: lowest P*T among feasible levels, ties -> lower; else K-1.
__device__ __forceinline__ int energy_ttft(const double *tt, const double *dy, const DevProfile &PR, int K,
                                           uint32_t nbt, double budget) {
  int best = -1;
  double be = 0.0;
  for (int k = 0; k < K; ++k) {
    const double t = ttft_pred(tt[2 * k], tt[2 * k + 1], nbt);
    if (!(t <= budget)) continue;
    const double e = mul(power_at(PR, 0, dy[k], nbt), t);
    if (best < 0 || e < be) { best = k; be = e; }
  }
  return best < 0 ? K - 1 : best;
}

__device__ __forceinline__ int energy_itl(const double *it, const double *dy, const DevProfile &PR, int K,
                                          uint64_t n, uint64_t kv, double target, int wshift) {
  const double *row = itl_row(it, PR, K, n, wshift);
  const double dn = (double)n, dkv = (double)kv;
  int best = -1;
  double be = 0.0;
  for (int k = 0; k < K; ++k) {
    const double t = itl_eval(row, k, dn, dkv);
    if (!(t <= target)) continue;
    const double e = mul(power_at(PR, 1, dy[k], n), t);
    if (best < 0 || e < be) { best = k; be = e; }
  }
  return best < 0 ? K - 1 : best;
}

// ---------------------------------------------------------------- K2 control_step
constexpr int CTL_MINB = 8;       // 8 CTAs x 8 warps per SM with 2 items per thread: measured best
template <int PHASE, int KK>   // KK: the ladder length when known at compile time (0: runtime)
__global__ void __launch_bounds__(DECIDE_THREADS, CTL_MINB)
control_kernel(const __grid_constant__ ControlParams P) {
  extern __shared__ double sm[];
  int *smi = mhz_smem(sm, P.lad.k, P.prof);
  stage_tables(P.prof, P.lad, PHASE == 0, PHASE == 1, P.mode == 1 ? PHASE : -1, sm, smi);
  const int K = KK > 0 ? KK : P.lad.k;
  const double *dy = dyn_smem(sm, K, P.prof);
  const double *its = itl_smem(sm, K, P.prof);
  const bool emode = P.mode == 1;
  const int wshift = (P.prof.tile_w & (P.prof.tile_w - 1)) == 0 ? __ffs(P.prof.tile_w) - 1 : -1;
  // DECIDE_UNROLL items per thread per tile, block-strided: every load instruction is
  // coalesced and each thread keeps DECIDE_UNROLL independent loads of each array in flight.
  const size_t tile = (size_t)blockDim.x * DECIDE_UNROLL;
  for (size_t base = (size_t)blockIdx.x * tile; base < P.n; base += (size_t)gridDim.x * tile) {
    uint32_t load[DECIDE_UNROLL], kv[DECIDE_UNROLL], q[DECIDE_UNROLL];
    double tgt[DECIDE_UNROLL], wait[DECIDE_UNROLL];
#pragma unroll
    for (int u = 0; u < DECIDE_UNROLL; ++u) {
      const size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
      const bool in = i < P.n;
      load[u] = in ? P.load[i] : 1u;
      q[u] = in ? P.queue_len[i] : 1u;
      tgt[u] = in ? P.target[i] : 0.0;
      if (PHASE == 0) wait[u] = in ? P.wait[i] : 0.0;
      else kv[u] = in ? P.n_kv[i] : 1u;
    }
#pragma unroll
    for (int u = 0; u < DECIDE_UNROLL; ++u) {
      const size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
      if (i >= P.n) continue;
      uint16_t lvl;
      uint8_t st = VOLTANA_ITEM_OK;
      if (PHASE == 0) {
        if (load[u] == 0u) {
          lvl = 0xFFFF; st = VOLTANA_ITEM_E_CONTRACT;
        } else if (q[u] > 0u) {
          lvl = (uint16_t)(K - 1);                      // backlog
        } else {
          double b = sub(tgt[u], wait[u]);
          b = b > 0.0 ? b : 0.0;
          const double *ttr = tt_row(sm, K, P.prof, load[u]);   // prefill tile (F1)
          lvl = (uint16_t)(emode ? energy_ttft(ttr, dy, P.prof, K, load[u], b) : scan_ttft<KK>(ttr, K, load[u], b));
        }
      } else {
        if (load[u] == 0u || kv[u] < load[u]) {
          lvl = 0xFFFF; st = VOLTANA_ITEM_E_CONTRACT;
        } else if (q[u] > 0u) {
          lvl = (uint16_t)(K - 1);
        } else {
          lvl = (uint16_t)(emode ? energy_itl(its, dy, P.prof, K, load[u], kv[u], tgt[u], wshift)
                                 : scan_itl<KK>(its, P.prof, K, load[u], kv[u], tgt[u], wshift));
        }
      }
      P.out_level[i] = lvl;
      P.out_status[i] = st;
    }
  }
}

// ---------------------------------------------------------------- K3 route_batch
// EcoRoute's case analysis (A13-A17) from each instance's lowest feasible level now
// (kn) and after the hypothetical addition (ka): the candidate set (bit d) and the case 1-5.
template <int NI>
__device__ __forceinline__ unsigned eco_levels(const int *kn, const int *ka, const int *smi, int ND, int32_t delta,
                                               int &cse) {
  unsigned inset = 0;
  int fnow[NI], faft[NI];
  int ncross = 0, mu = 0x7fffffff, mr = 0x7fffffff, mn = 0x7fffffff, ma = 0x7fffffff;
#pragma unroll
  for (int d = 0; d < NI; ++d) {
    fnow[d] = faft[d] = 0;
    if (d < ND) {
      fnow[d] = smi[kn[d]];
      faft[d] = smi[ka[d]];
      const bool cr = faft[d] > fnow[d];                                                 // A13
      ncross += cr;
      if (!cr && fnow[d] < mu) mu = fnow[d];
      if (cr && faft[d] < mr) mr = faft[d];
      if (fnow[d] < mn) mn = fnow[d];
      if (faft[d] < ma) ma = faft[d];
    }
  }
  if (ncross == 0) {
#pragma unroll
    for (int d = 0; d < NI; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
    cse = __popc(inset) == 1 ? 1 : 2;
  } else if (ncross < ND) {
    const long long g = (long long)mu - (long long)mr;                                  // A14, A15
    if (g <= (long long)delta) {
#pragma unroll
      for (int d = 0; d < NI; ++d)
        if (d < ND && !(faft[d] > fnow[d]) && fnow[d] == mu) inset |= 1u << d;
      cse = 3;
    } else {
#pragma unroll
      for (int d = 0; d < NI; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
      cse = 4;
    }
  } else {
#pragma unroll
    for (int d = 0; d < NI; ++d) if (d < ND && faft[d] == ma) inset |= 1u << d;
    cse = 5;
  }
  return inset;
}

// round robin among the candidate set from the cursor (A17)
__device__ __forceinline__ uint32_t rr_pick(unsigned inset, int ND, uint32_t &cursor) {
  const unsigned rot = ((inset >> cursor) | (inset << (ND - cursor))) & ((1u << ND) - 1u);
  uint32_t d = cursor + (uint32_t)ffs0(rot);   // < 2 N_D: wrap without a division
  d = d >= (uint32_t)ND ? d - (uint32_t)ND : d;
  if (__popc(inset) >= 2) cursor = d + 1u >= (uint32_t)ND ? 0u : d + 1u;
  return d;
}

// N_D = 2 decision table over (kn0, ka0, kn1, ka1, cursor): dsel | case << 1 | new cursor << 4,
// filled by the CTA from eco_levels (so it is the same decision); 2 K^4 bytes
__device__ void build_route_lut(uint8_t *lut, int K, const int *smi, int32_t delta) {
  const int n = 2 * K * K * K * K;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    int r = e >> 1;
    const int ka1 = r % K; r /= K;
    const int kn1 = r % K; r /= K;
    const int ka0 = r % K; r /= K;
    const int kn0 = r;
    const int kn[2] = {kn0, kn1}, ka[2] = {ka0, ka1};
    int cse;
    const unsigned inset = eco_levels<2>(kn, ka, smi, 2, delta, cse);
    uint32_t cur = (uint32_t)(e & 1);
    const uint32_t d = rr_pick(inset, 2, cur);
    lut[e] = (uint8_t)(d | (uint32_t)cse << 1 | cur << 4);
  }
}

// One EcoRoute decision on caller-given effective states; NI = the kernel's
// instance bound (2, 4 or 8), so the per-instance arrays stay in registers at that size.
template <int NI, int KK>
__device__ __forceinline__ void route_item(const RouteParams &P, const double *it, const double *dy, const int *smi,
                                           int K, int ND, int wshift, uint32_t in, double tgt, uint32_t &cursor,
                                           const uint32_t *n, const uint32_t *kv, uint16_t &dsel, uint8_t &cse,
                                           uint8_t &st, const uint8_t *lut) {
  bool bad = cursor >= (uint32_t)ND || in == 0u;
#pragma unroll
  for (int d = 0; d < NI; ++d)
    if (d < ND) bad = bad || kv[d] < n[d];
  dsel = 0xFFFF; cse = 0xFF; st = VOLTANA_ITEM_E_CONTRACT;
  if (bad) return;
  st = VOLTANA_ITEM_OK;
  if (P.policy == 1 || ND == 1) {
    dsel = (uint16_t)cursor;
    cursor = cursor + 1u >= (uint32_t)ND ? 0u : cursor + 1u;
    cse = 0;
    return;
  }
  unsigned inset = 0;
  if (P.policy == 2) {  // energy-scored router [B1-B3]
    double score[NI], tmax[NI];
    bool feas[NI];
    bool any = false;
#pragma unroll
    for (int d = 0; d < NI; ++d) {
      score[d] = tmax[d] = 0.0;
      feas[d] = false;
      if (d >= ND) continue;
      double enow = 0.0;
      if (n[d] != 0u) {
        const double *r0 = itl_row(it, P.prof, K, n[d], wshift);
        const int k0 = scan_itl<KK>(it, P.prof, K, n[d], kv[d], tgt, wshift);        // A10, A11
        enow = mul(power_at(P.prof, 1, dy[k0], n[d]), itl_eval(r0, k0, (double)n[d], (double)kv[d]));
      }
      const uint64_t n1 = (uint64_t)n[d] + 1u, kv1 = (uint64_t)kv[d] + in + 1u;   // A12
      const double *row = itl_row(it, P.prof, K, n1, wshift);
      const double dn = (double)n1, dkv = (double)kv1;
      double best = 0.0, t = 0.0;
      for (int k = 0; k < K; ++k) {
        t = itl_eval(row, k, dn, dkv);
        if (!(t <= tgt)) continue;
        const double e = mul(power_at(P.prof, 1, dy[k], n1), t);
        if (!feas[d] || e < best) best = e;
        feas[d] = true;
      }
      tmax[d] = t;
      score[d] = sub(best, enow);
      any = any || feas[d];
    }
    double m = 0.0;
    bool first = true;
#pragma unroll
    for (int d = 0; d < NI; ++d) {
      if (d >= ND || (any && !feas[d])) continue;
      const double v = any ? score[d] : tmax[d];
      if (first || v < m) { m = v; first = false; }
    }
#pragma unroll
    for (int d = 0; d < NI; ++d)
      if (d < ND && (any ? (feas[d] && score[d] == m) : tmax[d] == m)) inset |= 1u << d;
    cse = any ? 6 : 7;
  } else {
    int kn[NI], ka[NI];
#pragma unroll
    for (int d = 0; d < NI; ++d) {
      kn[d] = ka[d] = 0;
      if (d < ND) scan_pair<KK>(it, P.prof, K, n[d], kv[d], in, tgt, wshift, kn[d], ka[d]);   // A10-A12
    }
    if (NI == 2 && lut) {   // N_D = 2, K <= 8: the case analysis as a table (built by eco_levels)
      VT_CHECK(kn[0] < K && ka[0] < K && kn[NI - 1] < K && ka[NI - 1] < K && cursor < 2u);
      const uint32_t v = lut[((((uint32_t)(kn[0] * K + ka[0]) * K + kn[NI - 1]) * K + ka[NI - 1]) << 1) | cursor];
      dsel = (uint16_t)(v & 1u);
      cse = (uint8_t)((v >> 1) & 7u);
      cursor = v >> 4;
      return;
    }
    int c;
    inset = eco_levels<NI>(kn, ka, smi, ND, P.delta, c);
    cse = (uint8_t)c;
  }
  dsel = (uint16_t)rr_pick(inset, ND, cursor);                                         // A17
}

constexpr int ROUTE_MINB = 4;     // CTAs of 8 warps per SM (<= 64 registers); 5 CTAs or 3-4 items: slower
constexpr int ROUTE_U2 = 2;       // items per thread per tile when N_D <= 2
template <int ND_MAX, int KK>   // KK: the ladder length when known at compile time (0: runtime)
__global__ void __launch_bounds__(DECIDE_THREADS, ROUTE_MINB)
route_kernel(const __grid_constant__ RouteParams P) {
  extern __shared__ double sm[];
  int *smi = mhz_smem(sm, P.lad.k, P.prof);
  stage_tables(P.prof, P.lad, false, true, P.policy == 2 ? 1 : -1, sm, smi);
  // <2, KK > 0> instantiations run only for N_D == 2 (host dispatch): N_D is a constant there
  const int K = KK > 0 ? KK : P.lad.k, ND = (ND_MAX == 2 && KK > 0) ? 2 : P.n_d;
  const double *it = itl_smem(sm, K, P.prof);
  const double *dy = dyn_smem(sm, K, P.prof);
  const int wshift = (P.prof.tile_w & (P.prof.tile_w - 1)) == 0 ? __ffs(P.prof.tile_w) - 1 : -1;
  // N_D = 2 EcoRoute with a known ladder length: the case analysis as a shared-memory table
  uint8_t *lut = nullptr;
  if (ND_MAX == 2 && KK > 0 && P.policy == 0) {
    lut = (uint8_t *)(smi + K);
    build_route_lut(lut, K, smi, P.delta);
    __syncthreads();
  }
  constexpr int U = ND_MAX <= 2 ? ROUTE_U2 : 2;
  const size_t tile = (size_t)blockDim.x * U;
  for (size_t base = (size_t)blockIdx.x * tile; base < P.n; base += (size_t)gridDim.x * tile) {
    uint32_t inv[U], cur[U], n[U][ND_MAX], kv[U][ND_MAX];
    double tg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // every load of the tile issued before any decision
      const size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
      const bool in = i < P.n;
      inv[u] = in ? P.req_in[i] : 1u;
      tg[u] = in ? P.target[i] : 0.0;
      cur[u] = in ? P.cursor[i] : 0u;
      if (ND_MAX == 2 && ND == 2 && P.pad) {   // one 8-byte load per array (8-B aligned, host-checked)
        const uint2 a = in ? reinterpret_cast<const uint2 *>(P.n_req)[i] : make_uint2(0u, 0u);
        const uint2 b = in ? reinterpret_cast<const uint2 *>(P.n_kv)[i] : make_uint2(0u, 0u);
        n[u][0] = a.x; n[u][ND_MAX > 1 ? 1 : 0] = a.y;
        kv[u][0] = b.x; kv[u][ND_MAX > 1 ? 1 : 0] = b.y;
      } else {
#pragma unroll
        for (int d = 0; d < ND_MAX; ++d) {
          n[u][d] = in && d < ND ? P.n_req[i * ND + d] : 0u;
          kv[u][d] = in && d < ND ? P.n_kv[i * ND + d] : 0u;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
      if (i >= P.n) continue;
      uint16_t dsel;
      uint8_t cse, st;
      route_item<ND_MAX, KK>(P, it, dy, smi, K, ND, wshift, inv[u], tg[u], cur[u], n[u], kv[u], dsel, cse, st, lut);
      P.out_instance[i] = dsel;
      P.out_case[i] = cse;
      P.out_status[i] = st;
      P.cursor[i] = cur[u];
    }
  }
}

size_t decide_smem_bytes(int k, int n_tiles, int n_ptiles) {
  const int tp = n_ptiles < 1 ? 1 : n_ptiles;
  return (size_t)(2 * tp * k + ITS * n_tiles * k + k) * sizeof(double) + (size_t)k * sizeof(int);
}

template <int PHASE, int KK>
static cudaError_t launch_control_t(const ControlParams &P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(control_kernel<PHASE, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  control_kernel<PHASE, KK><<<grid, DECIDE_THREADS, smem, st>>>(P);
  return cudaGetLastError();
}

template <int PHASE>
static cudaError_t launch_control_p(const ControlParams &P, int grid, size_t smem, cudaStream_t st) {
  switch (P.lad.k) {
    case 2: return launch_control_t<PHASE, 2>(P, grid, smem, st);
    case 5: return launch_control_t<PHASE, 5>(P, grid, smem, st);
    default: return launch_control_t<PHASE, 0>(P, grid, smem, st);
  }
}

cudaError_t launch_control(const ControlParams &P, int phase, int grid, size_t smem, cudaStream_t st) {
  return phase == 0 ? launch_control_p<0>(P, grid, smem, st) : launch_control_p<1>(P, grid, smem, st);
}

template <int NDM, int KK>
static cudaError_t launch_route_t(const RouteParams &P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(route_kernel<NDM, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  route_kernel<NDM, KK><<<grid, DECIDE_THREADS, smem, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_route(const RouteParams &P, int grid, size_t smem, cudaStream_t st) {
  if (P.n_d == 2) {
    if (P.policy == 0 && P.lad.k <= 8) smem += 2 * (size_t)P.lad.k * P.lad.k * P.lad.k * P.lad.k;   // decision table
    switch (P.lad.k) {  // ladder length (and N_D = 2) as template arguments: straight-line code
      case 1: return launch_route_t<2, 1>(P, grid, smem, st);
      case 2: return launch_route_t<2, 2>(P, grid, smem, st);
      case 3: return launch_route_t<2, 3>(P, grid, smem, st);
      case 4: return launch_route_t<2, 4>(P, grid, smem, st);
      case 5: return launch_route_t<2, 5>(P, grid, smem, st);
      case 6: return launch_route_t<2, 6>(P, grid, smem, st);
      case 7: return launch_route_t<2, 7>(P, grid, smem, st);
      case 8: return launch_route_t<2, 8>(P, grid, smem, st);
      default: return launch_route_t<2, 0>(P, grid, smem, st);
    }
  }
  if (P.n_d <= 2) return launch_route_t<2, 0>(P, grid, smem, st);
  if (P.n_d <= 4) return launch_route_t<4, 0>(P, grid, smem, st);
  return launch_route_t<8, 0>(P, grid, smem, st);
}

}  // namespace vt
