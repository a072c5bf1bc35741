// vt_sim.h — launch parameters of the simulate kernel (K4), shared by host and device code.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voltana.h"
#include "vt_device.cuh"

namespace vt {

#ifndef VT_SIM_THREADS
#define VT_SIM_THREADS 128
#endif
constexpr int SIM_THREADS = VT_SIM_THREADS;  // 4 warps per CTA, one scenario per warp
#ifndef VT_SIM_MIN_BLOCKS
#define VT_SIM_MIN_BLOCKS 4
#endif
constexpr int SIM_MIN_BLOCKS = VT_SIM_MIN_BLOCKS;  // 4: <= 128 registers, 16 warps per SM
#ifndef VT_SPW
#define VT_SPW 1
#endif
constexpr int SPW = VT_SPW;           // scenarios per warp (lane groups of 32 / SPW; N_P, N_D <= 8)
constexpr int MAX_SLOS = 64, MAX_LAYOUTS = 16, MAX_GRIDS = 16, MAX_PROFILES = 8;
size_t sim_smem_fixed(bool fast);  // per-warp shared-memory block without the staged ITL table
constexpr size_t SIM_ITL_SMEM_MAX = 4096;   // stage the ladder's ITL table in smem up to this size
#ifndef VT_NBMAX
#define VT_NBMAX 2048
#endif
#ifndef VT_UTAB
#define VT_UTAB 1  // utilisation table for busy power (one 1-MB setup launch; measured -0.5 %)
#endif
constexpr uint32_t SIM_UTAB = 8192;         // loads with a tabulated utilisation (VT_UTAB)
constexpr uint32_t SIM_WHEEL_MAX = VT_NBMAX; // decode wheel buckets (L2-resident); longer requests use the far list

#ifndef VT_SPLIT_A
#define VT_SPLIT_A 1  // phase A (prefill lanes) as its own launch (K4a) ahead of the decode kernel
#endif
#ifndef VT_PA_WARP
#define VT_PA_WARP 1  // K4a: one warp per (scenario, prefill instance) (0: one thread each)
#endif
constexpr bool PA_WARP = VT_PA_WARP;
#ifndef VT_PA_G
#define VT_PA_G 32    // K4a: lanes per prefill instance (a power of two <= 32): 32 / G instances per warp
#endif
constexpr int PA_G = VT_PA_G;
constexpr int PA_THREADS = VT_PA_WARP ? 128 : 32;
#ifndef VT_PA_MIN_BLOCKS
#define VT_PA_MIN_BLOCKS 6
#endif
constexpr int PA_MIN_BLOCKS = VT_PA_WARP ? VT_PA_MIN_BLOCKS : 1;
constexpr int RT_STRIDE = 3 * VOLTANA_MAX_LEVELS;  // resolved ladder row: [K][a1, c1] then prefill DYN [K]

struct PaRes {     // phase-A result of one prefill instance (K4a -> K4b; the record's prefill part)
  double ebusy, bms, top, sttft, tlast, errt;  // W*ms, ms, ms, ms, last event, first error time (+inf none)
  uint64_t h;                                  // decision-hash chain (A36)
  uint32_t iters, ttft_ok, itl_ok, both, errc, ndec, head, pad;  // head: first routed request (NIL none)
};

#ifndef VT_DEFER_ITL
#define VT_DEFER_ITL VT_SPLIT_A  // paper's-policy kernels: per-request ITL accounting deferred (K4c; needs the split)
#endif
#ifndef VT_ITL_INWARP
#define VT_ITL_INWARP 1  // the deferred ITL pass runs in K4b's warp right after its scenario (else K4c launch)
#endif
#ifndef VT_ITL_CAP
#define VT_ITL_CAP 4     // ITL pass: values of one list gathered by its lane (the rest: walked in order)
#endif
#ifndef VT_ITL_UW
#define VT_ITL_UW 1      // in-warp ITL pass: log entries per lane per round
#endif
constexpr uint32_t ITL_CAP = VT_ITL_CAP;
constexpr int ITL_UW = VT_ITL_UW;
template <int U> struct ItlScratch {  // per-warp scratch of the ITL pass (shared memory)
  double v[32 * U][ITL_CAP];          // gathered values of a round's entries
  double seq[32 * U * (ITL_CAP + 1)]; // the round's values regrouped instance by instance, log order
  double td[32 * U];
  uint32_t id[32 * U];                // where a list longer than ITL_CAP continues
};
constexpr uint32_t ITL_SCRATCH = (uint32_t)((sizeof(ItlScratch<ITL_UW>) + 15) & ~(size_t)15);
constexpr uint32_t CLOG_CHUNK = 32;  // completion-log slots handed to a decode lane at a time
struct CEnt {      // K4b -> K4c: one decode iteration end with completions (16 B)
  double td;       // the iteration's end time
  uint32_t head;   // first request of its completion list (admission order, linked by node.next)
  uint32_t d;      // decode instance
};

struct SimParams {
  // traces (device)
  const double *arrival;
  const uint32_t *in_len, *out_len;
  const uint64_t *offset;
  const double *duration;
  // scenarios (device)
  const uint32_t *trace_id, *slo_id, *layout_id, *grid_id, *profile_id;
  const uint64_t *hash_seed;
  uint32_t n;
  uint32_t nb;                 // wheel buckets per decode instance (power of two >= max_out)
  uint32_t max_out;
  uint32_t n_slots;            // workspace slots = warps that may run scenarios
  uint32_t n_slos, n_layouts, n_grids, n_profiles;
  uint64_t n_traces;
  uint64_t max_requests;
  voltana_result *out;
  // workspace
  uint32_t *counter;
  char *slots;                 // [n_slots][slot_bytes]: request nodes
  size_t slot_bytes, node_bytes;  // slot = [N] 16-B nodes, then [N] u32 far-list finishing iterations
  uint4 *wheels;               // [n_slots][wheel_per_slot]: decode timing wheels (16-B buckets, 0 = empty)
  size_t wheel_per_slot;       // max N_D * nb buckets
  uint32_t itl_smem;           // stage the ladder's ITL table in shared memory
  uint32_t smem_per_warp;
  uint32_t sw_off;             // VT_SWHEEL: byte offset of the near wheel in the per-warp block
  uint64_t *timing;            // debug: [n][2] globaltimer ns at scenario start/end | smid<<56 (NULL: off)
  voltana_outputs o;           // optional per-request / per-instance outputs (variant kernel only)
  const double *utab;          // VT_UTAB: [MAX_PROFILES][2][SIM_UTAB] utilisation u = l / (l + u_half)
  double *ring_e;              // ITL modes (E3): [n_slots][max N_D][ring_r] iteration end times
  uint32_t *ring_c;            //   ... and cumulative counts of gaps above the ITL SLO
  uint32_t ring_r, ring_nd;    //   ring length (power of two >= max_out), instances per slot
  char *nodes;                 // VT_SPLIT_A: [n][max_requests] 16-B request nodes (scenario in kernel order)
  PaRes *pares;                // VT_SPLIT_A: [n][VOLTANA_MAX_INSTANCES] phase-A results
  double *rtab;                // VT_SPLIT_A: [MAX_GRIDS][MAX_PROFILES][RT_STRIDE] ladder-resolved prefill tables
  uint32_t np_max;             // VT_SPLIT_A: max N_P over the launch's layouts (K4a threads per scenario)
  CEnt *clog;                  // VT_DEFER_ITL: [n][max_requests] completion log per scenario (log order)
  uint32_t *clog_n;            // VT_DEFER_ITL: [n] log slots used by each scenario (empty ones: head NIL)
  size_t clog_stride;          // VT_DEFER_ITL: log slots per scenario (max_requests + 2 * 8 * CLOG_CHUNK)
  uint32_t ks_off;             // VT_ITL_INWARP: byte offset of the ITL scratch in the per-warp block
  // host tables copied into the kernel parameter bank
  voltana_slo slo[MAX_SLOS];
  voltana_layout lay[MAX_LAYOUTS];
  voltana_grid grid[MAX_GRIDS];
  DevProfile prof[MAX_PROFILES];
};

// v: variant bits (1 energy scoring B1-B4; 2 window/overhead/noise/ITL modes/outputs C-E);
// fast: every ladder has K <= 8, every tile width is a power of two and the ITL tables are
// staged in shared memory, so the general table paths are compiled out.
const void *sim_kernel_ptr(int v, bool fast);
cudaError_t launch_sim(const SimParams &P, int v, bool fast, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_utab(const SimParams &P, cudaStream_t st);  // VT_UTAB: fill P.utab
cudaError_t launch_prefill(const SimParams &P, int v, bool fast, cudaStream_t st);  // K4a (VT_SPLIT_A)
cudaError_t launch_itl(const SimParams &P, cudaStream_t st);  // K4c (VT_DEFER_ITL)

}  // namespace vt
