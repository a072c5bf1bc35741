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

namespace vt {

// ---------------------------------------------------------------- shared-memory tables
struct SmemTables {
  const double *tt;   // [K][2]: a1, c1
  const double *it;   // [T][K][3]: a2, b2, c2
  const int *mhz;     // [K]
};

__device__ void stage_tables(const DevProfile &PR, const LadderParam &LP, bool need_tt, bool need_it,
                             double *sm, int *smi) {
  const int K = LP.k, T = PR.n_tiles;
  for (int x = threadIdx.x; x < K; x += blockDim.x) {
    int lv = LP.level[x];
    if (need_tt) { sm[2 * x] = PR.a1[lv]; sm[2 * x + 1] = PR.c1[lv]; }
    smi[x] = PR.mhz[lv];
  }
  if (need_it) {
    double *it = sm + 2 * K;
    for (int x = threadIdx.x; x < T * K; x += blockDim.x) {
      int j = x / K, k = x - j * K;
      size_t o = (size_t)j * PR.k + LP.level[k];
      it[3 * x] = PR.a2[o]; it[3 * x + 1] = PR.b2[o]; it[3 * x + 2] = PR.c2[o];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int scan_ttft(const double *tt, int K, uint32_t nbt, double budget) {
  for (int k = 0; k < K; ++k)
    if (ttft_pred(tt[2 * k], tt[2 * k + 1], nbt) <= budget) return k;
  return K - 1;
}

// 64-bit state: the what-if state (n+1, kv+in+1) may exceed 32 bits for caller data.
// Tile index by shift when the tile width is a power of two (wshift >= 0).
__device__ __forceinline__ int scan_itl(const double *it, const DevProfile &PR, int K, uint64_t n,
                                        uint64_t kv, double target, int wshift) {
  uint64_t j = wshift >= 0 ? (n - 1u) >> wshift : (n - 1u) / (uint64_t)PR.tile_w;
  if (j > (uint64_t)(PR.n_tiles - 1)) j = (uint64_t)(PR.n_tiles - 1);
  const double *row = it + 3 * (size_t)j * K;
  const double dn = (double)n, dkv = (double)kv;
  for (int k = 0; k < K; ++k)
    if (add(add(mul(row[3 * k], dn), mul(row[3 * k + 1], dkv)), row[3 * k + 2]) <= target) return k;
  return K - 1;
}

// ---------------------------------------------------------------- K2 control_step
template <int PHASE>
__global__ void __launch_bounds__(DECIDE_THREADS)
control_kernel(const __grid_constant__ ControlParams P) {
  extern __shared__ double sm[];
  int *smi = (int *)(sm + 2 * P.lad.k + 3 * P.prof.n_tiles * P.lad.k);
  stage_tables(P.prof, P.lad, PHASE == 0, PHASE == 1, sm, smi);
  const int K = P.lad.k;
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
          lvl = (uint16_t)scan_ttft(sm, K, load[u], b);
        }
      } else {
        if (load[u] == 0u || kv[u] < load[u]) {
          lvl = 0xFFFF; st = VOLTANA_ITEM_E_CONTRACT;
        } else if (q[u] > 0u) {
          lvl = (uint16_t)(K - 1);
        } else {
          lvl = (uint16_t)scan_itl(sm + 2 * K, P.prof, K, load[u], kv[u], tgt[u], wshift);
        }
      }
      P.out_level[i] = lvl;
      P.out_status[i] = st;
    }
  }
}

// ---------------------------------------------------------------- K3 route_batch
// One EcoRoute decision on caller-given effective states.
__device__ __forceinline__ void route_item(const RouteParams &P, const double *it, const int *smi, int K, int ND,
                                           int wshift, uint32_t in, double tgt, uint32_t &cursor,
                                           const uint32_t *n, const uint32_t *kv, uint16_t &dsel, uint8_t &cse,
                                           uint8_t &st) {
  bool bad = cursor >= (uint32_t)ND || in == 0u;
#pragma unroll
  for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d)
    if (d < ND) bad = bad || kv[d] < n[d];
  dsel = 0xFFFF; cse = 0xFF; st = VOLTANA_ITEM_E_CONTRACT;
  if (bad) return;
  st = VOLTANA_ITEM_OK;
  if (P.policy == 1 || ND == 1) {
    dsel = (uint16_t)cursor;
    cursor = (cursor + 1u) % (uint32_t)ND;
    cse = 0;
    return;
  }
  int fnow[VOLTANA_MAX_INSTANCES], faft[VOLTANA_MAX_INSTANCES];
  int ncross = 0, mu = 0x7fffffff, mr = 0x7fffffff, mn = 0x7fffffff, ma = 0x7fffffff;
#pragma unroll
  for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) {
    fnow[d] = faft[d] = 0;
    if (d < ND) {
      const int kn = n[d] == 0u ? 0 : scan_itl(it, P.prof, K, n[d], kv[d], tgt, wshift);   // A10, A11
      const int ka = scan_itl(it, P.prof, K, (uint64_t)n[d] + 1u, (uint64_t)kv[d] + in + 1u, tgt, wshift);  // A12
      fnow[d] = smi[kn];
      faft[d] = smi[ka];
      const bool cr = faft[d] > fnow[d];                                                 // A13
      ncross += cr;
      if (!cr && fnow[d] < mu) mu = fnow[d];
      if (cr && faft[d] < mr) mr = faft[d];
      if (fnow[d] < mn) mn = fnow[d];
      if (faft[d] < ma) ma = faft[d];
    }
  }
  unsigned inset = 0;
  if (ncross == 0) {
#pragma unroll
    for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
    cse = __popc(inset) == 1 ? 1 : 2;
  } else if (ncross < ND) {
    const long long g = (long long)mu - (long long)mr;                                  // A14, A15
    if (g <= (long long)P.delta) {
#pragma unroll
      for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d)
        if (d < ND && !(faft[d] > fnow[d]) && fnow[d] == mu) inset |= 1u << d;
      cse = 3;
    } else {
#pragma unroll
      for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
      cse = 4;
    }
  } else {
#pragma unroll
    for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) if (d < ND && faft[d] == ma) inset |= 1u << d;
    cse = 5;
  }
  const unsigned rot = ((inset >> cursor) | (inset << (ND - cursor))) & ((1u << ND) - 1u);
  const uint32_t d = (cursor + (uint32_t)ffs0(rot)) % (uint32_t)ND;
  dsel = (uint16_t)d;
  if (__popc(inset) >= 2) cursor = (d + 1u) % (uint32_t)ND;                             // A17
}

template <int ND_MAX>
__global__ void __launch_bounds__(DECIDE_THREADS)
route_kernel(const __grid_constant__ RouteParams P) {
  extern __shared__ double sm[];
  int *smi = (int *)(sm + 2 * P.lad.k + 3 * P.prof.n_tiles * P.lad.k);
  stage_tables(P.prof, P.lad, false, true, sm, smi);
  const int K = P.lad.k, ND = P.n_d;
  const double *it = sm + 2 * K;
  const int wshift = (P.prof.tile_w & (P.prof.tile_w - 1)) == 0 ? __ffs(P.prof.tile_w) - 1 : -1;
  constexpr int U = ND_MAX <= 2 ? DECIDE_UNROLL : 2;
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
#pragma unroll
      for (int d = 0; d < ND_MAX; ++d) {
        n[u][d] = in && d < ND ? P.n_req[i * ND + d] : 0u;
        kv[u][d] = in && d < ND ? P.n_kv[i * ND + d] : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
      if (i >= P.n) continue;
      uint32_t nn[VOLTANA_MAX_INSTANCES], kk[VOLTANA_MAX_INSTANCES];
#pragma unroll
      for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) {
        nn[d] = d < ND_MAX ? n[u][d < ND_MAX ? d : 0] : 0u;
        kk[d] = d < ND_MAX ? kv[u][d < ND_MAX ? d : 0] : 0u;
      }
      uint16_t dsel;
      uint8_t cse, st;
      route_item(P, it, smi, K, ND, wshift, inv[u], tg[u], cur[u], nn, kk, dsel, cse, st);
      P.out_instance[i] = dsel;
      P.out_case[i] = cse;
      P.out_status[i] = st;
      P.cursor[i] = cur[u];
    }
  }
}

size_t decide_smem_bytes(int k, int n_tiles) {
  return (size_t)(2 * k + 3 * n_tiles * k) * sizeof(double) + (size_t)k * sizeof(int);
}

cudaError_t launch_control(const ControlParams &P, int phase, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e;
  if (phase == 0) {
    e = cudaFuncSetAttribute(control_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    control_kernel<0><<<grid, DECIDE_THREADS, smem, st>>>(P);
  } else {
    e = cudaFuncSetAttribute(control_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    control_kernel<1><<<grid, DECIDE_THREADS, smem, st>>>(P);
  }
  return cudaGetLastError();
}

template <int NDM>
static cudaError_t launch_route_t(const RouteParams &P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(route_kernel<NDM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  route_kernel<NDM><<<grid, DECIDE_THREADS, smem, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_route(const RouteParams &P, int grid, size_t smem, cudaStream_t st) {
  if (P.n_d <= 2) return launch_route_t<2>(P, grid, smem, st);
  if (P.n_d <= 4) return launch_route_t<4>(P, grid, smem, st);
  return launch_route_t<8>(P, grid, smem, st);
}

}  // namespace vt
