/* voltana.h — C ABI of the B200 evaluator of VoltanaLLM's policies (arXiv 2509.04827).
 *
 * Four calls mirror the paper's problem statement: offline EcoPred
 * calibration, EcoFreq frequency control, EcoRoute request routing, and the batched
 * trace-driven evaluation of both policies over many serving scenarios.
 * Citations: P:NNN = PAPER.md line; readings [Axx] are listed in DESIGN.md §2.
 *
 * Conventions (all calls)
 *  - Pointers documented "device" must be CUDA device memory of the current device;
 *    "host" structs/tables are read during the call only. The caller owns every buffer;
 *    the library never allocates device memory; scratch comes from a caller workspace.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). All device work is
 *    enqueued asynchronously on it; pointers must stay valid until it completes.
 *  - Host-side validation is synchronous: a non-OK return other than VOLTANA_E_CUDA means
 *    NOTHING was enqueued; voltana_last_error_detail() names the offending argument.
 *    VOLTANA_E_CUDA is a launch/runtime failure and may follow a partial enqueue (earlier
 *    memsets or kernels of the same call); kernel attributes are set before any enqueue.
 *  - Problems found on the device are reported per item (status bytes / result.status),
 *    never by aborting the batch.
 *  - Arithmetic: IEEE fp64, every operation rounded separately, no FMA contraction
 *    (reading A33). Outputs are byte-deterministic for given inputs, independent of the
 *    launch configuration, stream and GPU count.
 *  - Thread-safe: no global mutable state except a per-thread error string.
 */
#ifndef VOLTANA_H
#define VOLTANA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VOLTANA_OK = 0,
  VOLTANA_E_INVALID_ARG = 1, /* null pointer, bad enum, size out of range            */
  VOLTANA_E_LADDER = 2,      /* empty / unsorted / duplicate frequency list    */
  VOLTANA_E_COVERAGE = 3,    /* ladder level not on its profile grid          */
  VOLTANA_E_CALIBRATION = 4, /* fit: empty or degenerate cell, see cell_status        */
  VOLTANA_E_CONFIG = 5,      /* N_P/N_D outside 1..8, B or C == 0 or >= 2^31, tau     */
  VOLTANA_E_WORKSPACE = 6,   /* workspace smaller than *_workspace_bytes()            */
  VOLTANA_E_CUDA = 7         /* launch/runtime error (detail has cudaGetErrorString)  */
} voltana_status;

/* per-item status bytes / result.status */
#define VOLTANA_ITEM_OK 0u
#define VOLTANA_ITEM_E_KV 1u       /* a request can never fit an empty decode instance [A20] */
#define VOLTANA_ITEM_E_CONTRACT 2u /* non-positive predicted duration, n_kv < n_req, ...   */
#define VOLTANA_ITEM_E_INPUT 3u    /* trace invalid (unsorted, lengths outside [1,65535]...) */
#define VOLTANA_ITEM_E_INTERNAL 4u /* watchdog: a scenario exceeded its step bound (library bug) */

#define VOLTANA_MAX_LEVELS 64      /* K <= 64 levels per ladder                            */
#define VOLTANA_MAX_INSTANCES 8    /* N_P, N_D <= 8                                        */
#define VOLTANA_DELTA_INF 2147483647 /* Delta "set to a large value"               */

/* One calibrated profile (the output of the offline profiling pass).
 * Host struct holding DEVICE table pointers. Level l of the profile grid runs at
 * mhz[l]; tables are indexed by level, ITL tables are [n_tiles][k] and TTFT tables
 * [n_ptiles][k] (row = tile). Prefill tile of a batch (Appendix B) [F1]:
 * n_ptiles <= 1 -> 0; N_bt > prefill_cutoff -> n_ptiles-1; else min(n_ptiles-1, (N_bt-1)/W). */
typedef struct {
  int32_t k;          /* levels on the grid, 1..1024                                   */
  int32_t n_tiles;    /* ITL tiles T >= 1 (batch-size boundaries)               */
  int32_t tile_w;     /* tile width W >= 1 (128)                                */
  int32_t n_ptiles;   /* prefill tiles T_p, 0 or 1 = a single TTFT tile, <= 64 [F1]     */
  const int32_t *mhz; /* device [k] strictly increasing MHz                            */
  const double *a1;   /* device [max(1,n_ptiles)*k] eq:pred-ttft T = a1*N_bt + c1 */
  const double *c1;   /* device [max(1,n_ptiles)*k] ms                                 */
  const double *a2;   /* device [n_tiles*k] eq:pred-itl, ms per request         */
  const double *b2;   /* device [n_tiles*k] ms per KV token                            */
  const double *c2;   /* device [n_tiles*k] ms                                         */
  const double *dyn;  /* device [2*k] busy dynamic power at full utilisation, W:
                         [0,k) prefill, [k,2k) decode (eq:P-f P:187, [A22])            */
  double p_idle;      /* W, idle draw at any frequency                                 */
  double tdp;         /* W, power clip                                         */
  double u_half_prefill, u_half_decode; /* utilisation u = load / (load + u_half)      */
  int32_t prefill_cutoff; /* N_bt above which prefill uses the last tile (2000) [F1] */
  int32_t reserved;
} voltana_profile;

/* ------------------------------------------------------------------------------------
 * voltana_control_step — EcoFreq (fig:governor-arch P:400-410), one decision
 * per snapshot i (SoA, device arrays of length n):
 *   queue_len[i] > 0                     -> top level (K-1)           backlog
 *   else prefill: lowest k with a1*load + c1 <= max(0, target - wait)
 *   else decode : lowest k with a2*load + b2*n_kv + c2 (tile of load) <= target
 *   nothing feasible -> K-1 [A2]
 * mode: 0 = EcoFreq as above; 1 = energy argmin [DESIGN B4]: among the feasible levels the
 *   one minimising P(k, load) * T(k) (busy power eq:P-f P:187 times the prediction; energy =
 *   time x power P:74), ties -> lower level; backlog / nothing feasible as above.
 * phase: 0 prefill (load = N_bt; n_kv unused, may be NULL), 1 decode (load = N_req;
 * wait_ms unused, may be NULL). ladder_h: host [k] ascending profile-level indices.
 * out_level[i] = ladder index (0..k-1), 0xFFFF on a contract error; out_status[i] per
 * the VOLTANA_ITEM_* codes (load == 0, decode n_kv < load -> E_CONTRACT).
 * Errors: INVALID_ARG (null/phase/mode/n), LADDER, COVERAGE.                            */
voltana_status voltana_control_step(const voltana_profile *prof_h, int phase, int mode,
                                    const uint16_t *ladder_h, int k, const uint32_t *load,
                                    const uint32_t *n_kv, const uint32_t *queue_len,
                                    const double *wait_ms, const double *target_ms, size_t n,
                                    uint16_t *out_level, uint8_t *out_status, void *stream);

/* ------------------------------------------------------------------------------------
 * voltana_route_batch — EcoRoute, one decision per item i:
 *   for every decode instance d: f(d) = EcoFreq level on (n_req, n_kv) (n_req = 0 -> level
 *   0), f'(d) = EcoFreq level on (n_req + 1, n_kv + req_in + 1) [A10-A12]; crossed iff
 *   MHz(f') > MHz(f) [A13]; cases (1)-(5) with Delta (inclusive g <= Delta) [A14-A16];
 *   ties go round robin from cursor[i] [A17]. policy 1 = plain round robin.
 *   policy 2 = energy-scored [DESIGN B1-B3] (the north_star's argmin-energy successor
 *   state): score(d) = min over feasible k of P(k,n+1)*T(k,n+1,kv+in+1) - P(k_now,n)*T(k_now,n,kv)
 *   (0 if n = 0), argmin over instances with a feasible k (case 6); none feasible: the
 *   lowest top-level T after adding (case 7); ties round robin.
 * n_req, n_kv: device [n * n_d] row-major (item, instance) effective states (running +
 * pending). req_in, itl_target_ms: device [n]. cursor: device [n] in/out.
 * out_instance[i] in 0..n_d-1 (0xFFFF on error), out_case[i] 0 = RR, 1..5 = cases, 6/7 energy.
 * Errors: INVALID_ARG (policy outside 0..2), LADDER, COVERAGE, CONFIG (n_d outside 1..8).                     */
voltana_status voltana_route_batch(const voltana_profile *prof_h, const uint16_t *ladder_h,
                                   int k, int n_d, const uint32_t *n_req, const uint32_t *n_kv,
                                   const uint32_t *req_in, const double *itl_target_ms,
                                   int32_t delta_mhz, int policy, uint32_t *cursor, size_t n,
                                   uint16_t *out_instance, uint8_t *out_case,
                                   uint8_t *out_status, void *stream);

/* ------------------------------------------------------------------------------------
 * voltana_fit_profile — EcoPred calibration: ordinary least squares
 * per cell. TTFT cell = (prefill, level l, prefill tile jp as in voltana_profile [F1]):
 * lat ~ a1*N_bt + c1. ITL cell = (decode, level l, tile j = min(T-1, (N_req-1)/W)):
 * lat ~ a2*N_req + b2*N_kv + c2. An empty tile j > 0 (prefill: jp > 0) inherits tile j-1
 * plus tile_step on c2 (c1) [F2]; MAE per fitted cell.
 * Samples (device SoA, length n): phase u8 (0/1), level u16 (< k), n_bt/n_req/n_kv u32,
 * lat_ms f64. Outputs (device), Tp = n_ptiles >= 1: a1,c1 [Tp*k]; a2,b2,c2 [T*k];
 * mae [Tp*k + T*k]; cell_status [Tp*k + T*k] (0 fitted, 1 inherited, 2 empty,
 * 3 degenerate) — cell index: TTFT (jp, l) -> jp*k + l, ITL (j, l) -> Tp*k + j*k + l.
 * Returns OK after enqueueing; cell errors are reported in cell_status (read it back:
 * any 2 or 3 is the E_CALIBRATION condition). Sums use a fixed reduction order, so the
 * result is deterministic and within 1e-12 relative of the sequential oracle.
 * Samples with phase > 1, level >= k, (decode and n_req == 0) or (prefill and n_bt == 0)
 * are ignored and counted in invalid_count (device u64, may be NULL).
 * Launch: one cooperative kernel (every CTA resident, grid barriers between the three
 * passes: means, centred sums + solve, MAE); a device that cannot co-schedule the grid makes
 * the launch fail with VOLTANA_E_CUDA. The workspace (voltana_fit_workspace_bytes) holds
 * warp-private accumulator rows (40 B per cell per resident warp), the CTA partials and the
 * grid sums; it needs no initialisation (rows are written at their first touch).          */
size_t voltana_fit_workspace_bytes(size_t n_samples, int k, int n_tiles, int n_ptiles);
voltana_status voltana_fit_profile(const uint8_t *phase, const uint16_t *level,
                                   const uint32_t *n_bt, const uint32_t *n_req,
                                   const uint32_t *n_kv, const double *lat_ms, size_t n,
                                   int k, int n_tiles, int tile_w, double tile_step,
                                   int n_ptiles, uint32_t prefill_cutoff,
                                   double *a1, double *c1, double *a2, double *b2, double *c2,
                                   double *mae, uint8_t *cell_status, uint64_t *invalid_count,
                                   void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * voltana_simulate — the north_star call: evaluate both policies over n independent
 * scenarios (trace x SLO x layout x frequency ladder x profile).
 * Per scenario, the discrete-event loop of DESIGN.md §2 (A4-A23): Poisson-driven
 * arrivals, prefill round robin + FCFS token-budget batching, EcoFreq before every
 * prefill batch and decode iteration, EcoRoute for every request leaving prefill,
 * continuous decode batching with KV capacity, energy = time x power(f).
 * Host tables: slos[n_slos] (<= 64), layouts[n_layouts] (<= 16), grids[n_grids] (<= 16),
 * profiles[n_profiles] (<= 8). Device: traces, scenario table, out[n] records.
 * Scenarios are claimed in array order by persistent warps: put expensive scenarios
 * first for load balance (the Python layer does LPT ordering).
 * Enqueues three kernels on `stream`: a setup launch (utilisation and ladder tables), the
 * prefill timelines of every scenario (K4a, one warp per prefill instance), then routing +
 * decode (K4b, one warp per scenario; the per-request ITL accounting runs in the same warp
 * after each scenario for the paper's-policy kernels).
 * Workspace (voltana_simulate_workspace_bytes[_ex]): a 16-B node per request of every
 * scenario (K4a -> K4b) plus fixed per-warp scratch (see below).
 * A non-OK return means nothing was enqueued (kernel attributes are set before any enqueue).
 * Errors: INVALID_ARG, LADDER, COVERAGE, CONFIG, WORKSPACE, CUDA. Per-scenario problems
 * go to out[i].status (then only status and n_requests are set).                        */
typedef struct {
  double ttft_ms, itl_ms; /* SLO thresholds (attainment)                          */
  double scale;           /* controller target = scale * SLO, (0,1] typical [A3]         */
} voltana_slo;

typedef struct {
  int32_t n_p, n_d;        /* prefill / decode instances, 1..8 (2P2D in P:593)          */
  int32_t policy;          /* 0 EcoRoute, 1 round robin (SGLang baseline),
                              2 energy-scored router [DESIGN B1-B3]                      */
  int32_t delta_mhz;       /* EcoRoute threshold Delta; VOLTANA_DELTA_INF         */
  uint32_t max_batch_tokens; /* prefill batch token budget B (8192) [A6]                 */
  uint32_t kv_capacity;    /* decode KV tokens C (400000) [A20]                          */
  double kv_transfer_ms;   /* tau: 0, or >= 1e-3 [A18]                                    */
  int32_t ctrl_mode;       /* 0 EcoFreq lowest feasible, 1 energy argmin [B4] */
  int32_t itl_mode;        /* per-request ITL for the attainment counts: 0 mean
                              (A30), 1 max inter-token gap, 2 nearest-rank P99 of the gaps;
                              sum_itl_mean_ms stays the mean [E3]                         */
  double ctrl_interval_ms; /* window control: an instance decides at
                              an iteration START only when >= this has elapsed since its
                              previous decision (inclusive); 0 = every iteration [C1]      */
  double freq_overhead_ms; /* blocking frequency set: an iteration whose
                              level differs from the running one starts this much later;
                              0 = non-blocking. Instances start at the top level [C2, C3]  */
  const double *exec_noise; /* device [noise_len] execution-noise factors or NULL (S:401,
                              S:469): iteration j of instance i (prefill p: i = p, decode
                              d: i = n_p + d) runs prediction x exec_noise[splitmix64(
                              hash_seed ^ 0xD1B54A32D192ED03 ^ i<<40 ^ j) & (noise_len-1)];
                              a factor outside (0, 1e6] sets status E_INPUT [D1, D2]      */
  uint32_t noise_len;      /* power of two when exec_noise != NULL                        */
  uint32_t reserved2;      /* 0                                                           */
} voltana_layout;

typedef struct {
  int32_t k;                            /* 1..64 levels                                  */
  uint16_t level[VOLTANA_MAX_LEVELS];   /* ascending profile-level indices               */
} voltana_grid;

typedef struct {
  const double *arrival;    /* device, concatenated [R] ms, non-decreasing per trace    */
  const uint32_t *in_len;   /* device [R] 1..65535                                      */
  const uint32_t *out_len;  /* device [R] 1..65535                                      */
  const uint64_t *offset;   /* device [n_traces + 1]                                    */
  const double *duration_ms;/* device [n_traces] nominal trace duration [A39]           */
  uint64_t n_traces;
  uint64_t max_requests;    /* host bound on any trace's request count (workspace size) */
  uint32_t max_out;         /* host bound on out_len, 1..65535 (decode timing-wheel size);
                               a scenario with a longer request gets status E_INPUT      */
  uint32_t reserved;
} voltana_traces;

typedef struct {            /* device arrays [n]                                        */
  const uint32_t *trace_id, *slo_id, *layout_id, *grid_id, *profile_id;
  const uint64_t *hash_seed;/* h0 of the decision hash = global scenario index [A36]    */
  const uint64_t *node_offset; /* device [n + 1] or NULL: exclusive prefix sum of the
                               scenarios' request counts (array order), so the request
                               nodes take total_requests x 16 B instead of n x
                               max_requests x 16 B; a scenario whose range differs from
                               its trace's length gets status E_INPUT                    */
  uint64_t total_requests;  /* host: node_offset[n] (ignored when node_offset is NULL)  */
} voltana_scenarios;

typedef struct {            /* 128-byte per-scenario record                             */
  uint32_t status, n_requests, n_ttft_ok, n_itl_ok, n_both_ok;
  uint32_t prefill_iters;   /* prefill batches started                                  */
  uint64_t steps_ctrl, steps_route, decision_hash;
  double sum_ttft_ms, sum_itl_mean_ms, e_prefill_busy_j, e_prefill_idle_j, e_decode_busy_j,
      e_decode_idle_j, busy_ms_prefill, busy_ms_decode, top_level_ms, horizon_ms;
} voltana_result;

/* Workspace of voltana_simulate for n_scenarios scenarios: the request nodes (16 B per
 * request of every scenario: n_scenarios x max_requests, or total_requests when the scenario
 * table carries node_offset — pass that total to the _ex form), plus per resident warp a
 * completion log (32 KB) and decode timing wheels (16 B x max N_D x 2048).               */
size_t voltana_simulate_workspace_bytes(const voltana_traces *traces_h,
                                        const voltana_layout *layouts_h, int n_layouts,
                                        size_t n_scenarios);
size_t voltana_simulate_workspace_bytes_ex(const voltana_traces *traces_h,
                                           const voltana_layout *layouts_h, int n_layouts,
                                           size_t n_scenarios, uint64_t total_requests);
voltana_status voltana_simulate(const voltana_traces *traces_h, const voltana_slo *slos_h,
                                int n_slos, const voltana_layout *layouts_h, int n_layouts,
                                const voltana_grid *grids_h, int n_grids,
                                const voltana_profile *profiles_h, int n_profiles,
                                const voltana_scenarios *scen_h, size_t n, voltana_result *out,
                                void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * voltana_simulate_ex — voltana_simulate plus optional per-request records and per-instance
 * iteration time series ("time series (frequency, n_req, n_kv per
 * instance at event granularity)"; DESIGN E1-E3). outputs_h == NULL: same as
 * voltana_simulate. All output pointers are device pointers; a group is off when its
 * offset array is NULL. Contents for a scenario with status != 0 are unspecified.
 *
 * Per-request group (req_offset != NULL): scenario i writes request r of its trace (trace
 * order) at index req_offset[i] + r; an empty range [req_offset[i], req_offset[i+1]) skips
 * the scenario, any other length than the trace's request count sets status E_INPUT.
 *   req_tfirst  first-token time = prefill end (ms); req_tdone last-token time (= tfirst
 *   when out == 1); req_itl mean inter-token latency (0 when out == 1, A30);
 *   req_decode decode instance, req_case routing case 0..7 (0xFF when out == 1).
 * Iteration group (iter_offset != NULL): instance u of scenario i (prefill p: u = p, decode
 * d: u = n_p + d) writes its j-th started iteration at iters[iter_offset[i] + u*iter_cap + j]
 * for j < iter_cap and its total iteration count at iter_count[iter_offset[i]/iter_cap + u];
 * iter_offset[i] must be a multiple of iter_cap with room for n_p + n_d instances.        */
typedef struct {           /* 32-byte iteration record                                   */
  double t_start;          /* START time t, ms (the iteration runs from t + overhead, C3) */
  double dur_ms;           /* true duration = prediction x noise factor (D1)              */
  uint32_t load;           /* N_bt (prefill) or N_req (decode) at START                   */
  uint32_t n_kv;           /* N_kv at START (decode), 0 (prefill)                         */
  uint16_t level;          /* ladder index                                                */
  uint8_t flags;           /* bit0 controller decision taken (C1), bit1 overhead paid (C3),
                              bit2 backlog (A5)                                            */
  uint8_t reserved[5];
} voltana_iteration;

typedef struct {
  const uint64_t *req_offset;  /* [n + 1] or NULL                                         */
  double *req_tfirst, *req_tdone, *req_itl;
  uint8_t *req_decode, *req_case;
  const uint64_t *iter_offset; /* [n] or NULL                                             */
  voltana_iteration *iters;
  uint32_t *iter_count;
  uint32_t iter_cap;           /* >= 1                                                    */
  uint32_t reserved;
} voltana_outputs;

voltana_status voltana_simulate_ex(const voltana_traces *traces_h, const voltana_slo *slos_h,
                                   int n_slos, const voltana_layout *layouts_h, int n_layouts,
                                   const voltana_grid *grids_h, int n_grids,
                                   const voltana_profile *profiles_h, int n_profiles,
                                   const voltana_scenarios *scen_h, size_t n, voltana_result *out,
                                   const voltana_outputs *outputs_h, void *workspace,
                                   size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * voltana_series_to_samples — the fit -> simulate loop (DESIGN E4): map
 * the iteration series written by voltana_simulate_ex (outputs_h: iters, iter_count,
 * iter_offset ascending, iter_cap) into EcoPred calibration samples for
 * voltana_fit_profile: slot x = iter_offset[s] + u*iter_cap + j becomes
 * sample x — prefill instance (u < n_p): phase 0, level = grids[grid_id[s]].level[rec.level],
 * n_bt = load; decode: phase 1, n_req = load, n_kv; lat_ms = true duration (noise included,
 * overhead excluded). Slots with j >= count, and scenarios whose profile_id differs from
 * `profile_id`, get phase 0xFF (skipped by the fit, counted invalid).
 * scen_h, layouts_h, grids_h: as passed to voltana_simulate_ex (same kernel order).
 * n_slots = total slots (iter_offset[n-1] + (n_p + n_d) * iter_cap of the last scenario).
 * Outputs: device SoA [n_slots]. Errors: INVALID_ARG.                                   */
voltana_status voltana_series_to_samples(const voltana_outputs *outputs_h,
                                         const voltana_layout *layouts_h, int n_layouts,
                                         const voltana_grid *grids_h, int n_grids,
                                         const voltana_scenarios *scen_h, size_t n, size_t n_slots,
                                         uint32_t profile_id, uint8_t *phase, uint16_t *level,
                                         uint32_t *n_bt, uint32_t *n_req, uint32_t *n_kv,
                                         double *lat_ms, void *stream);

/* Kernel-launch statistics of the last voltana_simulate on this thread (for the bench):
 * number of kernels launched. */
int voltana_last_launch_count(void);

/* Debug/profiling hook (this thread's next voltana_simulate calls): when buf != NULL,
 * buf[2i] (device u64, [2n]) receives the %globaltimer ns at which scenario i started and
 * buf[2i+1] its duration in ns with the SM id in bits 56..63. NULL turns it off. */
void voltana_debug_set_timing(uint64_t *buf);

/* Profiling hook (this thread's next voltana_simulate calls): when ev != NULL (a cudaEvent_t
 * created by the caller), it is recorded on the call's stream between the phase-A launch
 * (prefill_kernel, K4a) and the decode launch (simulate_kernel, K4b), so the caller can time
 * the two kernels with its own start/end events. NULL turns it off. */
void voltana_set_split_event(void *ev);

const char *voltana_status_string(voltana_status s);
const char *voltana_last_error_detail(void); /* thread-local, names the argument        */

#ifdef __cplusplus
}
#endif
#endif /* VOLTANA_H */
