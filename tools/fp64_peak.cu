// FP64 throughput and dependent-latency microbenchmark for the roofline denominators of the
// K4 / K2 / K3 kernels ("measure the FP64 peak"; SURVEY §6 "FP64 is not measured").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp64_peak tools/fp64_peak.cu
//   ./tools/fp64_peak            -> one JSON object on stdout
//
// Throughput: every SM runs 16 CTAs x 256 threads; each thread keeps 8 independent chains of
// DADD (x += a), DMUL (x *= b) or DFMA (x = fma(x, b, a)) for `iters` rounds. ops = threads x
// iters x 8 (DFMA counted as 2 flops, reported separately). Best of 5 launches, CUDA events.
// Latency: one warp, one dependent chain of 4096 operations timed with clock64 (cycles/op) for
// DADD, DMUL, SHFL, REDUX (__reduce_min_sync), VOTE (ballot), LDS (smem pointer chase) and
// LDG (L1-resident pointer chase).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int OP>
__global__ void thr_kernel(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) x[j] = __dadd_rn(x[j], a);
      else if (OP == 1) x[j] = __dmul_rn(x[j], b);
      else x[j] = __fma_rn(x[j], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;   // practically never; keeps the chains alive
}

template <int OP>
__global__ void lat_kernel(long long *cyc, double *out, const unsigned *chase, int n) {
  __shared__ unsigned sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = chase[i];
  __syncwarp();
  double x = 1.0 + threadIdx.x * 1e-9;
  unsigned u = threadIdx.x, p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = __dadd_rn(x, 1e-7);
    else if (OP == 1) x = __dmul_rn(x, 1.0000001);
    else if (OP == 2) u = __shfl_sync(0xffffffffu, u, (threadIdx.x + 1) & 31) + 1;
    else if (OP == 3) u = __reduce_min_sync(0xffffffffu, u + threadIdx.x) + 1;
    else if (OP == 4) u = __ballot_sync(0xffffffffu, ((u >> (i & 7)) & 1) != 0) + threadIdx.x;
    else if (OP == 5) p = sm[p];
    else p = __ldg(chase + p);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (x == 3.0 || u == 0xdeadbeefu || p == 0xdeadbeefu) out[0] = x + u + p;
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  int sm = pr.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double *out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, thr = 256, blocks = sm * 16;
  double best[3] = {0, 0, 0};
  for (int op = 0; op < 3; ++op) {
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(a);
      if (op == 0) thr_kernel<0><<<blocks, thr>>>(out, iters, 1e-9, 1.0000001);
      else if (op == 1) thr_kernel<1><<<blocks, thr>>>(out, iters, 1e-9, 1.0000001);
      else thr_kernel<2><<<blocks, thr>>>(out, iters, 1e-9, 1.0000001);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * thr * iters * 8;
      double g = ops / (ms * 1e-3) / 1e9;
      if (r > 0 && g > best[op]) best[op] = g;
    }
  }
  // latency: a random cyclic permutation (pointer chase) of 1024 entries
  unsigned h[1024], perm[1024];
  for (int i = 0; i < 1024; ++i) perm[i] = i;
  unsigned s = 12345;
  for (int i = 1023; i > 0; --i) { s = s * 1103515245u + 12345u; int j = (s >> 8) % (i + 1); unsigned t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
  for (int i = 0; i < 1024; ++i) h[perm[i]] = perm[(i + 1) % 1024];
  unsigned *chase;
  long long *cyc, hc;
  CK(cudaMalloc(&chase, sizeof(h)));
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMemcpy(chase, h, sizeof(h), cudaMemcpyHostToDevice));
  const char *names[7] = {"dadd", "dmul", "shfl", "redux_min", "ballot", "lds_chase", "ldg_l1_chase"};
  double lat[7];
  const int n = 4096;
  for (int op = 0; op < 7; ++op) {
    for (int r = 0; r < 3; ++r) {
      switch (op) {
        case 0: lat_kernel<0><<<1, 32>>>(cyc, out, chase, n); break;
        case 1: lat_kernel<1><<<1, 32>>>(cyc, out, chase, n); break;
        case 2: lat_kernel<2><<<1, 32>>>(cyc, out, chase, n); break;
        case 3: lat_kernel<3><<<1, 32>>>(cyc, out, chase, n); break;
        case 4: lat_kernel<4><<<1, 32>>>(cyc, out, chase, n); break;
        case 5: lat_kernel<5><<<1, 32>>>(cyc, out, chase, n); break;
        default: lat_kernel<6><<<1, 32>>>(cyc, out, chase, n); break;
      }
      CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
    lat[op] = (double)hc / n;
  }
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"fp64_gops\": {\"dadd\": %.1f, \"dmul\": %.1f, "
         "\"dfma_instr\": %.1f, \"dfma_flops\": %.1f}, \"fp64_lanes_per_sm_per_clk_at_attr_clock\": {\"dadd\": %.2f, "
         "\"dmul\": %.2f, \"dfma\": %.2f}, \"latency_cycles\": {",
         pr.name, sm, clk_khz / 1e3, best[0], best[1], best[2], 2 * best[2],
         best[0] * 1e9 / (sm * clk_khz * 1e3), best[1] * 1e9 / (sm * clk_khz * 1e3), best[2] * 1e9 / (sm * clk_khz * 1e3));
  for (int op = 0; op < 7; ++op) printf("%s\"%s\": %.1f", op ? ", " : "", names[op], lat[op]);
  printf("}, \"how\": \"%d CTAs x %d threads x 8 independent chains x %d rounds, best of 5, CUDA events; latency: "
         "1 warp, dependent chain of %d ops, clock64\"}\n", blocks, thr, iters, n);
  return 0;
}
