// vt_sim.h — launch parameters of the simulate kernels (K4a prefill, K4b routing + decode),
// shared by host and device code.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voltana.h"
#include "vt_device.cuh"

namespace vt {

constexpr int SIM_THREADS = 128;      // K4b: 4 warps per CTA, one scenario per warp
constexpr int SIM_MIN_BLOCKS = 4;     // <= 128 registers, 16 warps per SM (5: 96 registers, spills: 87 vs 80 ms)
constexpr int MAX_SLOS = 64, MAX_LAYOUTS = 16, MAX_GRIDS = 16, MAX_PROFILES = 8;
size_t sim_smem_fixed(bool fast);     // per-warp shared-memory block without the staged ITL table
constexpr size_t SIM_ITL_SMEM_MAX = 4096;   // stage the ladder's ITL table in smem up to this size ...
constexpr size_t SIM_ITL_SMEM_BIG = 24576;  // ... or up to this size when the occupancy is not needed
constexpr uint32_t SIM_WHEEL_MAX = 2048;    // decode wheel buckets; longer requests use the far list
                                            // (512 / 1024 / 4096: 80.2 / 78.0 / 77.7 vs 77.8 ms on C4)
constexpr uint32_t SIM_UTAB = 8192;         // loads with a tabulated utilisation u = l / (l + u_half)

constexpr int PA_G = 32;              // K4a: one warp per (scenario, prefill instance)
constexpr int PA_THREADS = 128;
constexpr int PA_MIN_BLOCKS = 6;
constexpr int RT_STRIDE = 3 * VOLTANA_MAX_LEVELS;  // resolved ladder row: [K][a1, c1] then prefill DYN [K]

struct PaRes {     // phase-A result of one prefill instance (K4a -> K4b; the record's prefill part)
  double ebusy, bms, top, sttft, tlast, errt;  // W*ms, ms, ms, ms, last event, first error time (+inf none)
  uint64_t h;                                  // decision-hash chain (A36)
  uint32_t iters, ttft_ok, itl_ok, both, errc, ndec;
  uint32_t send;   // stream end: the first request id of this instance whose node was not written
  uint32_t valid;  // every request of this instance's stream passed the input checks (A40)
  uint64_t tok;    // sum of in + out over the stream (A40: the scenario total must be < 2^31)
};

// Completion log (K4b -> its in-warp ITL pass): one 16-B entry per decode iteration end with
// completions, CLOG_CHUNK-entry chunks handed to the decode lanes in lane order; CLOG_CAP
// entries per resident warp, flushed through the ITL pass when full.
constexpr uint32_t CLOG_CHUNK = 32;
constexpr uint32_t CLOG_CAP = 64 * CLOG_CHUNK;
constexpr uint32_t ITL_CAP = 4;       // ITL pass: values of one list gathered by its lane (the rest: walked in order)
struct ItlScratch {                   // per-warp scratch of the ITL pass (shared memory)
  double v[32][ITL_CAP];              // gathered values of a round's entries
  double seq[32 * (ITL_CAP + 1)];     // the round's values regrouped instance by instance, log order
  double td[32];
  uint32_t id[32];                    // where a list longer than ITL_CAP continues
};
struct CEnt {      // one decode iteration end with completions (16 B)
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
  const uint64_t *node_offset; // [n + 1] request-node base of each scenario (NULL: s * max_requests)
  uint32_t n;
  uint32_t nb;                 // wheel buckets per decode instance (power of two >= max_out, <= SIM_WHEEL_MAX)
  uint32_t max_out;
  uint32_t n_slots;            // workspace slots = warps that may run scenarios
  uint32_t n_slos, n_layouts, n_grids, n_profiles;
  uint64_t n_traces;
  uint64_t max_requests;
  voltana_result *out;
  // workspace
  uint32_t *counter;
  char *slots;                 // [n_slots][slot_bytes]: the completion log [CLOG_CAP] CEnt
  size_t slot_bytes;
  uint4 *wheels;               // [n_slots][wheel_per_slot]: decode timing wheels (16-B buckets, 0 = empty)
  size_t wheel_per_slot;       // max N_D * nb buckets
  uint32_t itl_smem;           // stage the ladder's ITL table in shared memory
  uint32_t smem_per_warp;
  uint32_t ks_off;             // byte offset of the ITL-pass scratch in the per-warp block
  uint32_t np_max;             // max N_P over the launch's layouts (K4a warps per scenario)
  uint64_t *timing;            // debug: [n][2] globaltimer ns at scenario start/end | smid<<56 (NULL: off)
  voltana_outputs o;           // optional per-request / per-instance outputs (variant kernel only)
  const double *utab;          // [MAX_PROFILES][2][SIM_UTAB] utilisation u = l / (l + u_half)
  double *ring_e;              // ITL modes (E3): [n_slots][max N_D][ring_r] iteration end times
  uint32_t *ring_c;            //   ... and cumulative counts of gaps above the ITL SLO
  uint32_t ring_r, ring_nd;    //   ring length (power of two >= max_out), instances per slot
  char *nodes;                 // request nodes (16 B each), per scenario in kernel order (node_offset)
  PaRes *pares;                // [n][VOLTANA_MAX_INSTANCES] phase-A results
  double *rtab;                // [MAX_GRIDS][MAX_PROFILES][RT_STRIDE] ladder-resolved prefill tables
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
const void *pa_kernel_ptr(int v, bool fast);
cudaError_t launch_sim(const SimParams &P, int v, bool fast, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_utab(const SimParams &P, cudaStream_t st);  // setup: utilisation and ladder rows
cudaError_t launch_prefill(const SimParams &P, int v, bool fast, cudaStream_t st);  // K4a

}  // namespace vt
