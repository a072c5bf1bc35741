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

// 64-bit loads: the what-if state (n+1, kv+in+1) may exceed 32 bits for caller data
__device__ __forceinline__ int scan_itl(const double *it, const DevProfile &PR, int K, uint64_t n,
                                        uint64_t kv, double target) {
  uint64_t j = (n - 1u) / (uint64_t)PR.tile_w;
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
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    const uint32_t load = P.load[i];
    const uint32_t q = P.queue_len[i];
    const double tgt = P.target[i];
    uint16_t lvl;
    uint8_t st = VOLTANA_ITEM_OK;
    if (PHASE == 0) {
      const double wait = P.wait[i];
      if (load == 0u) {
        lvl = 0xFFFF; st = VOLTANA_ITEM_E_CONTRACT;
      } else if (q > 0u) {
        lvl = (uint16_t)(K - 1);                      // backlog
      } else {
        double b = sub(tgt, wait);
        b = b > 0.0 ? b : 0.0;
        lvl = (uint16_t)scan_ttft(sm, K, load, b);
      }
    } else {
      const uint32_t kv = P.n_kv[i];
      if (load == 0u || kv < load) {
        lvl = 0xFFFF; st = VOLTANA_ITEM_E_CONTRACT;
      } else if (q > 0u) {
        lvl = (uint16_t)(K - 1);
      } else {
        lvl = (uint16_t)scan_itl(sm + 2 * K, P.prof, K, load, kv, tgt);
      }
    }
    P.out_level[i] = lvl;
    P.out_status[i] = st;
  }
}

// ---------------------------------------------------------------- K3 route_batch
__global__ void __launch_bounds__(DECIDE_THREADS)
route_kernel(const __grid_constant__ RouteParams P) {
  extern __shared__ double sm[];
  int *smi = (int *)(sm + 2 * P.lad.k + 3 * P.prof.n_tiles * P.lad.k);
  stage_tables(P.prof, P.lad, false, true, sm, smi);
  const int K = P.lad.k, ND = P.n_d;
  const double *it = sm + 2 * K;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    const uint32_t in = P.req_in[i];
    const double tgt = P.target[i];
    uint32_t cursor = P.cursor[i];
    uint32_t n[VOLTANA_MAX_INSTANCES], kv[VOLTANA_MAX_INSTANCES];
    bool bad = cursor >= (uint32_t)ND || in == 0u;
#pragma unroll
    for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) {
      n[d] = 0; kv[d] = 0;
      if (d < ND) {
        n[d] = P.n_req[i * ND + d];
        kv[d] = P.n_kv[i * ND + d];
        bad = bad || kv[d] < n[d];
      }
    }
    uint16_t dsel = 0xFFFF;
    uint8_t cse = 0xFF, st = VOLTANA_ITEM_E_CONTRACT;
    if (!bad) {
      st = VOLTANA_ITEM_OK;
      if (P.policy == 1 || ND == 1) {
        dsel = (uint16_t)cursor;
        cursor = (cursor + 1u) % (uint32_t)ND;
        cse = 0;
      } else {
        int fnow[VOLTANA_MAX_INSTANCES], faft[VOLTANA_MAX_INSTANCES];
        int ncross = 0, mu = 0x7fffffff, mr = 0x7fffffff, mn = 0x7fffffff, ma = 0x7fffffff;
#pragma unroll
        for (int d = 0; d < VOLTANA_MAX_INSTANCES; ++d) {
          fnow[d] = faft[d] = 0;
          if (d < ND) {
            int kn = n[d] == 0u ? 0 : scan_itl(it, P.prof, K, n[d], kv[d], tgt);   // A10, A11
            int ka = scan_itl(it, P.prof, K, (uint64_t)n[d] + 1u, (uint64_t)kv[d] + in + 1u, tgt);  // A12
            fnow[d] = smi[kn];
            faft[d] = smi[ka];
            bool cr = faft[d] > fnow[d];                                           // A13
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
          long long g = (long long)mu - (long long)mr;
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
        unsigned rot = ((inset >> cursor) | (inset << (ND - cursor))) & ((1u << ND) - 1u);
        uint32_t d = (cursor + (uint32_t)ffs0(rot)) % (uint32_t)ND;
        dsel = (uint16_t)d;
        if (__popc(inset) >= 2) cursor = (d + 1u) % (uint32_t)ND;   // A17
      }
    }
    P.out_instance[i] = dsel;
    P.out_case[i] = cse;
    P.out_status[i] = st;
    P.cursor[i] = cursor;
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

cudaError_t launch_route(const RouteParams &P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  route_kernel<<<grid, DECIDE_THREADS, smem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace vt
