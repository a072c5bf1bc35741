// voltana_api.cu — host side of the C ABI declared in include/voltana.h:
// synchronous argument validation, workspace sizing, launch configuration.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/voltana.h"
#include "vt_decide.h"
#include "vt_device.cuh"
#include "vt_fit.h"
#include "vt_series.h"
#include "vt_sim.h"

using namespace vt;

namespace {

thread_local char g_detail[512] = "";
thread_local int g_launches = 0;
thread_local uint64_t *g_debug_timing = nullptr;
thread_local void *g_split_event = nullptr;

voltana_status fail(voltana_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
  return s;
}

voltana_status ok() {
  g_detail[0] = 0;
  return VOLTANA_OK;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

voltana_status check_profile(const voltana_profile *p, const char *what) {
  if (!p) return fail(VOLTANA_E_INVALID_ARG, "%s: null profile", what);
  if (p->k < 1 || p->k > 1024) return fail(VOLTANA_E_INVALID_ARG, "%s: profile.k=%d outside 1..1024", what, p->k);
  if (p->n_tiles < 1 || p->n_tiles > 64)
    return fail(VOLTANA_E_INVALID_ARG, "%s: profile.n_tiles=%d outside 1..64", what, p->n_tiles);
  if (p->tile_w < 1) return fail(VOLTANA_E_INVALID_ARG, "%s: profile.tile_w=%d < 1", what, p->tile_w);
  if (p->n_ptiles < 0 || p->n_ptiles > 64)
    return fail(VOLTANA_E_INVALID_ARG, "%s: profile.n_ptiles=%d outside 0..64", what, p->n_ptiles);
  if (p->n_ptiles > 1 && p->prefill_cutoff < p->tile_w)
    return fail(VOLTANA_E_INVALID_ARG, "%s: profile.prefill_cutoff=%d < tile_w (S:100)", what, p->prefill_cutoff);
  if (!p->mhz || !p->a1 || !p->c1 || !p->a2 || !p->b2 || !p->c2 || !p->dyn)
    return fail(VOLTANA_E_INVALID_ARG, "%s: profile table pointer is null", what);
  if (!std::isfinite(p->p_idle) || !std::isfinite(p->tdp) || !(p->u_half_prefill > 0) || !(p->u_half_decode > 0))
    return fail(VOLTANA_E_INVALID_ARG, "%s: profile power scalars invalid", what);
  return VOLTANA_OK;
}

voltana_status check_ladder(const uint16_t *lad, int k, int prof_k, const char *what) {
  if (!lad) return fail(VOLTANA_E_INVALID_ARG, "%s: null ladder", what);
  if (k < 1 || k > VOLTANA_MAX_LEVELS) return fail(VOLTANA_E_LADDER, "%s: ladder has %d levels (1..64)", what, k);
  for (int i = 0; i < k; ++i) {
    if (lad[i] >= prof_k)
      return fail(VOLTANA_E_COVERAGE, "%s: ladder[%d]=%u not on the profile grid (k=%d)", what, i, lad[i], prof_k);
    if (i > 0 && lad[i] <= lad[i - 1])
      return fail(VOLTANA_E_LADDER, "%s: ladder not strictly increasing at index %d", what, i);
  }
  return VOLTANA_OK;
}

voltana_status cuda_fail(cudaError_t e, const char *what) {
  return fail(VOLTANA_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int decide_grid(size_t n) {
  size_t want = (n + DECIDE_THREADS - 1) / DECIDE_THREADS;
  size_t cap = (size_t)sm_count() * 8;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

}  // namespace

extern "C" {

const char *voltana_status_string(voltana_status s) {
  switch (s) {
    case VOLTANA_OK: return "ok";
    case VOLTANA_E_INVALID_ARG: return "invalid argument";
    case VOLTANA_E_LADDER: return "invalid frequency ladder";
    case VOLTANA_E_COVERAGE: return "ladder level not on the profile grid";
    case VOLTANA_E_CALIBRATION: return "calibration error";
    case VOLTANA_E_CONFIG: return "invalid layout configuration";
    case VOLTANA_E_WORKSPACE: return "workspace too small";
    case VOLTANA_E_CUDA: return "CUDA error";
  }
  return "unknown status";
}

const char *voltana_last_error_detail(void) { return g_detail; }
int voltana_last_launch_count(void) { return g_launches; }
void voltana_debug_set_timing(uint64_t *buf) { g_debug_timing = buf; }
void voltana_set_split_event(void *ev) { g_split_event = ev; }

// ------------------------------------------------------------------ K2
voltana_status voltana_control_step(const voltana_profile *prof_h, int phase, int mode, const uint16_t *ladder_h, int k,
                                    const uint32_t *load, const uint32_t *n_kv, const uint32_t *queue_len,
                                    const double *wait_ms, const double *target_ms, size_t n,
                                    uint16_t *out_level, uint8_t *out_status, void *stream) {
  g_launches = 0;
  voltana_status s;
  if ((s = check_profile(prof_h, "control_step")) != VOLTANA_OK) return s;
  if (phase != 0 && phase != 1) return fail(VOLTANA_E_INVALID_ARG, "control_step: phase=%d", phase);
  if (mode != 0 && mode != 1) return fail(VOLTANA_E_INVALID_ARG, "control_step: mode=%d", mode);
  if ((s = check_ladder(ladder_h, k, prof_h->k, "control_step")) != VOLTANA_OK) return s;
  if (n == 0) return ok();
  if (!load || !queue_len || !target_ms || !out_level || !out_status || (phase == 0 && !wait_ms) ||
      (phase == 1 && !n_kv))
    return fail(VOLTANA_E_INVALID_ARG, "control_step: null array pointer");
  ControlParams P;
  memset(&P, 0, sizeof(P));
  P.prof = to_dev(*prof_h);
  P.lad.k = k;
  for (int i = 0; i < k; ++i) P.lad.level[i] = ladder_h[i];
  P.load = load; P.n_kv = n_kv; P.queue_len = queue_len; P.wait = wait_ms; P.target = target_ms;
  P.n = n; P.out_level = out_level; P.out_status = out_status;
  P.mode = mode;
  cudaError_t e = launch_control(P, phase, decide_grid(n), decide_smem_bytes(k, prof_h->n_tiles, prof_h->n_ptiles),
                                 (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "control_step launch");
  g_launches = 1;
  return ok();
}

// ------------------------------------------------------------------ K3
voltana_status voltana_route_batch(const voltana_profile *prof_h, const uint16_t *ladder_h, int k, int n_d,
                                   const uint32_t *n_req, const uint32_t *n_kv, const uint32_t *req_in,
                                   const double *itl_target_ms, int32_t delta_mhz, int policy,
                                   uint32_t *cursor, size_t n, uint16_t *out_instance, uint8_t *out_case,
                                   uint8_t *out_status, void *stream) {
  g_launches = 0;
  voltana_status s;
  if ((s = check_profile(prof_h, "route_batch")) != VOLTANA_OK) return s;
  if ((s = check_ladder(ladder_h, k, prof_h->k, "route_batch")) != VOLTANA_OK) return s;
  if (n_d < 1 || n_d > VOLTANA_MAX_INSTANCES) return fail(VOLTANA_E_CONFIG, "route_batch: n_d=%d outside 1..8", n_d);
  if (policy < 0 || policy > 2) return fail(VOLTANA_E_INVALID_ARG, "route_batch: policy=%d", policy);
  if (n == 0) return ok();
  if (!n_req || !n_kv || !req_in || !itl_target_ms || !cursor || !out_instance || !out_case || !out_status)
    return fail(VOLTANA_E_INVALID_ARG, "route_batch: null array pointer");
  RouteParams P;
  memset(&P, 0, sizeof(P));
  P.prof = to_dev(*prof_h);
  P.lad.k = k;
  for (int i = 0; i < k; ++i) P.lad.level[i] = ladder_h[i];
  P.n_d = n_d; P.policy = policy; P.delta = delta_mhz;
  P.n_req = n_req; P.n_kv = n_kv; P.req_in = req_in; P.target = itl_target_ms; P.cursor = cursor;
  P.n = n; P.out_instance = out_instance; P.out_case = out_case; P.out_status = out_status;
  P.pad = (((uintptr_t)n_req | (uintptr_t)n_kv) & 7u) == 0 ? 1 : 0;  // 8-B vector loads of the N_D = 2 states
  cudaError_t e = launch_route(P, decide_grid(n), decide_smem_bytes(k, prof_h->n_tiles, prof_h->n_ptiles), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "route_batch launch");
  g_launches = 1;
  return ok();
}

// ------------------------------------------------------------------ K1
namespace {
struct FitLayout { int cells, wpb, blocks; size_t chunk, rows, part, red, means, cnt, ticket, total; };

FitLayout fit_layout(size_t n, int k, int n_tiles, int n_ptiles) {
  FitLayout L;
  L.cells = (n_ptiles < 1 ? 1 : n_ptiles) * k + n_tiles * k;
  L.wpb = fit_warps_per_block(L.cells);
#ifndef VT_FIT_SPW
#define VT_FIT_SPW 256
#endif
  // co-resident CTAs (cooperative launch): the occupancy of this device, else an upper bound
  // from the shared-memory and thread limits (the workspace is sized by the bound)
  const int bound = sm_count() * FIT_CTAS_PER_SM;
  const int occ = fit_max_blocks(L.cells, L.wpb);
  const int cap = occ > 0 && occ < bound ? occ : bound;
  size_t warps_want = (n + VT_FIT_SPW - 1) / VT_FIT_SPW;  // >= VT_FIT_SPW samples per warp (small n: more CTAs)
  size_t want_b = (warps_want + L.wpb - 1) / L.wpb;
  L.blocks = (int)(want_b < 1 ? 1 : (want_b < (size_t)cap ? want_b : (size_t)cap));
  size_t tw = (size_t)L.blocks * L.wpb;
  L.chunk = (n + tw - 1) / tw;
  L.chunk = (L.chunk + 127) & ~(size_t)127;
  if (L.chunk == 0) L.chunk = 128;
  const int pb = bound > L.blocks ? bound : L.blocks;   // partials and rows for any grid up to the bound
  L.rows = 0;
  L.part = align256(L.rows + (size_t)pb * L.wpb * L.cells * 5 * sizeof(double));
  L.red = align256(L.part + (size_t)pb * L.cells * 5 * sizeof(double));
  L.means = align256(L.red + (size_t)L.cells * 5 * sizeof(double));
  L.cnt = align256(L.means + (size_t)L.cells * 3 * sizeof(double));
  L.ticket = align256(L.cnt + (size_t)L.cells * sizeof(uint64_t));
  L.total = align256(L.ticket + 4 * sizeof(uint32_t));
  return L;
}
}  // namespace

size_t voltana_fit_workspace_bytes(size_t n_samples, int k, int n_tiles, int n_ptiles) {
  if (k < 1 || n_tiles < 1 || n_ptiles < 1) return 0;
  return fit_layout(n_samples, k, n_tiles, n_ptiles).total;
}

voltana_status voltana_fit_profile(const uint8_t *phase, const uint16_t *level, const uint32_t *n_bt,
                                   const uint32_t *n_req, const uint32_t *n_kv, const double *lat_ms, size_t n,
                                   int k, int n_tiles, int tile_w, double tile_step, int n_ptiles,
                                   uint32_t prefill_cutoff, double *a1, double *c1,
                                   double *a2, double *b2, double *c2, double *mae, uint8_t *cell_status,
                                   uint64_t *invalid_count, void *workspace, size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (k < 1 || k > 1024 || n_tiles < 1 || n_tiles > 64 || tile_w < 1)
    return fail(VOLTANA_E_INVALID_ARG, "fit_profile: k=%d n_tiles=%d tile_w=%d", k, n_tiles, tile_w);
  if (n_ptiles < 1 || n_ptiles > 64) return fail(VOLTANA_E_INVALID_ARG, "fit_profile: n_ptiles=%d (1..64)", n_ptiles);
  if (!a1 || !c1 || !a2 || !b2 || !c2 || !mae || !cell_status)
    return fail(VOLTANA_E_INVALID_ARG, "fit_profile: null output pointer");
  if (n > 0 && (!phase || !level || !n_bt || !n_req || !n_kv || !lat_ms))
    return fail(VOLTANA_E_INVALID_ARG, "fit_profile: null sample pointer");
  if (!std::isfinite(tile_step)) return fail(VOLTANA_E_INVALID_ARG, "fit_profile: tile_step not finite");
  FitLayout L = fit_layout(n, k, n_tiles, n_ptiles);
  if (fit_smem_bytes(L.cells, L.wpb) > 227 * 1024)
    return fail(VOLTANA_E_INVALID_ARG, "fit_profile: %d cells exceed shared memory", L.cells);
  if (!workspace || ws_bytes < L.total)
    return fail(VOLTANA_E_WORKSPACE, "fit_profile: workspace %zu < %zu bytes", ws_bytes, L.total);
  FitParams P;
  memset(&P, 0, sizeof(P));
  P.phase = phase; P.level = level; P.n_bt = n_bt; P.n_req = n_req; P.n_kv = n_kv; P.lat = lat_ms;
  const uintptr_t al = (uintptr_t)n_bt | (uintptr_t)n_req | (uintptr_t)n_kv | (uintptr_t)lat_ms;
  P.vec = ((uintptr_t)phase & 3u) == 0 && ((uintptr_t)level & 7u) == 0 && (al & 15u) == 0 ? 1 : 0;
  P.n = n; P.chunk = L.chunk; P.k = k; P.n_tiles = n_tiles; P.tile_w = tile_w; P.cells = L.cells;
  P.tile_step = tile_step;
  P.n_ptiles = n_ptiles; P.kp = n_ptiles * k; P.pcut = prefill_cutoff;
  P.pad = (tile_w & (tile_w - 1)) == 0 ? (uint32_t)__builtin_ctz((unsigned)tile_w) + 1u : 0u;  // log2 W + 1 (pow2 W)
  P.a1 = a1; P.c1 = c1; P.a2 = a2; P.b2 = b2; P.c2 = c2; P.mae = mae; P.status = cell_status;
  P.invalid_count = invalid_count;
  char *ws = (char *)workspace;
  P.rows = (double *)(ws + L.rows);
  P.bmw = (L.cells + 31) / 32;
  P.part = (double *)(ws + L.part);
  P.red = (double *)(ws + L.red);
  P.means = (double *)(ws + L.means);
  P.cnt = (uint64_t *)(ws + L.cnt);
  P.ticket = (uint32_t *)(ws + L.ticket);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e0 = cudaMemsetAsync(P.ticket, 0, 4 * sizeof(uint32_t), st);
  if (e0 == cudaSuccess && invalid_count) e0 = cudaMemsetAsync(invalid_count, 0, sizeof(uint64_t), st);
  if (e0 != cudaSuccess) return cuda_fail(e0, "fit_profile memset");
  int launches = 0;
  cudaError_t e = launch_fit(P, L.blocks, L.wpb, st, &launches);
  if (e != cudaSuccess) return cuda_fail(e, "fit_profile launch");
  g_launches = launches;
  return ok();
}

// ------------------------------------------------------------------ K4
namespace {

int max_nd(const voltana_layout *lays, int n_layouts) {
  int md = 1;
  for (int i = 0; i < n_layouts; ++i) md = lays[i].n_d > md ? lays[i].n_d : md;
  return md;
}

uint32_t wheel_buckets(uint32_t max_out) {
  uint32_t nb = 2;
  while (nb < max_out && nb < SIM_WHEEL_MAX) nb <<= 1;
  return nb;
}

struct SimLayout {
  size_t slot, wheel_per_slot, slots_off, wheels_off, total, smem_per_warp, smem, utab_off;
  uint32_t n_slots, nb, itl_smem, ring_r = 0, ring_nd = 0, ks_off = 0;
  size_t ring_e_off = 0, ring_c_off = 0;
  size_t nodes_off = 0, pares_off = 0, rtab_off = 0;
};

int resident_warps(size_t smem_per_block) {
  static std::mutex mu;
  static size_t cached_smem = (size_t)-1;
  static int cached = 0;
  std::lock_guard<std::mutex> g(mu);
  if (smem_per_block != cached_smem) {
    int nb = 0;
    // both instantiations are built for the same bound (128 registers, 4 CTAs per SM)
    cudaFuncSetAttribute(sim_kernel_ptr(0, false), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_per_block);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sim_kernel_ptr(0, false), SIM_THREADS,
                                                      smem_per_block) !=
            cudaSuccess || nb < 1) {
      cudaGetLastError();
      nb = 1;
    }
    cached = nb * sm_count() * (SIM_THREADS / 32);  // scenario slots
    cached_smem = smem_per_block;
  }
  return cached;
}

// fast: the fast-table instantiation (K <= 8 staged tables) will run [DESIGN §5 item 7]
// total_requests: sum of the scenarios' request counts (0: n x max_requests)
SimLayout sim_layout(const voltana_traces *tr, const voltana_layout *lays, int n_layouts, int kmax, int tmax,
                     size_t n, uint64_t total_requests, bool fast = false) {
  SimLayout L;
  L.nb = wheel_buckets(tr->max_out);
  size_t itl_bytes = (size_t)kmax * tmax * 24;
  // the ladder's ITL table is staged in shared memory when it is small, or when the launch has
  // fewer scenarios than the warps that stay resident with the larger block (C2: 28 levels x
  // 16 tiles = 10.7 KB per warp, 1024 scenarios): then staging costs no occupancy that is used
  auto block = [&](bool stage) {
    size_t w = (sim_smem_fixed(fast) + (stage ? itl_bytes : 0) + 15) & ~(size_t)15;
    return w + ((sizeof(ItlScratch) + 15) & ~(size_t)15);
  };
  L.itl_smem = itl_bytes <= SIM_ITL_SMEM_MAX ? 1u : 0u;
  if (!L.itl_smem && itl_bytes <= SIM_ITL_SMEM_BIG && block(true) * (SIM_THREADS / 32) <= 200 * 1024 &&
      (size_t)resident_warps(block(true) * (SIM_THREADS / 32)) >= n)
    L.itl_smem = 1u;
  L.smem_per_warp = block(L.itl_smem != 0u);
  L.ks_off = (uint32_t)(L.smem_per_warp - ((sizeof(ItlScratch) + 15) & ~(size_t)15));  // ITL-pass scratch
  L.smem = L.smem_per_warp * (SIM_THREADS / 32);
  // per resident warp: the completion log
  L.slot = (size_t)CLOG_CAP * sizeof(CEnt);
  L.wheel_per_slot = (size_t)max_nd(lays, n_layouts) * L.nb;
  size_t rw = (size_t)resident_warps(L.smem);
  L.n_slots = (uint32_t)(n < rw ? (n < 1 ? 1 : n) : rw);
  L.slots_off = 256;
  L.wheels_off = align256(L.slots_off + (size_t)L.n_slots * L.slot);
  L.total = L.wheels_off + (size_t)L.n_slots * L.wheel_per_slot * sizeof(uint4);
  // ITL Max / P99 (E3): per decode instance, the end time and the running count of gaps above
  // the SLO of its last ring_r iterations (ring_r >= max_out covers every request's window)
  L.ring_r = 0;
  for (int i = 0; i < n_layouts; ++i)
    if (lays[i].itl_mode != 0) L.ring_r = 2;
  if (L.ring_r) {
    while (L.ring_r < tr->max_out) L.ring_r <<= 1;
    L.ring_nd = (uint32_t)max_nd(lays, n_layouts);
    L.ring_e_off = align256(L.total);
    L.ring_c_off = align256(L.ring_e_off + (size_t)L.n_slots * L.ring_nd * L.ring_r * sizeof(double));
    L.total = L.ring_c_off + (size_t)L.n_slots * L.ring_nd * L.ring_r * sizeof(uint32_t);
  }
  L.utab_off = align256(L.total);
  L.total = L.utab_off + (size_t)MAX_PROFILES * 2 * SIM_UTAB * sizeof(double);
  // request nodes, written by K4a and read by K4b: one 16-B node per request per scenario
  const uint64_t nodes = total_requests ? total_requests : (uint64_t)(n < 1 ? 1 : n) * tr->max_requests;
  L.nodes_off = align256(L.total);
  L.total = L.nodes_off + align256((size_t)(nodes < 1 ? 1 : nodes) * 16);
  L.pares_off = L.total;
  L.total = L.pares_off + align256((size_t)(n < 1 ? 1 : n) * VOLTANA_MAX_INSTANCES * sizeof(PaRes));
  L.rtab_off = L.total;
  L.total = L.rtab_off + (size_t)MAX_GRIDS * MAX_PROFILES * RT_STRIDE * sizeof(double);
  return L;
}

void table_extent(const voltana_grid *grids, int n_grids, const voltana_profile *profs, int n_profiles, int *kmax,
                  int *tmax) {
  *kmax = 1;
  *tmax = 1;
  for (int i = 0; i < n_grids; ++i) *kmax = grids[i].k > *kmax ? grids[i].k : *kmax;
  for (int i = 0; i < n_profiles; ++i) *tmax = profs[i].n_tiles > *tmax ? profs[i].n_tiles : *tmax;
}

}  // namespace

size_t voltana_simulate_workspace_bytes_ex(const voltana_traces *traces_h, const voltana_layout *layouts_h,
                                           int n_layouts, size_t n_scenarios, uint64_t total_requests) {
  if (!traces_h || !layouts_h || n_layouts < 1) return 0;
  // conservative table extent (ITL table staged in shared memory or not does not change the size)
  return sim_layout(traces_h, layouts_h, n_layouts, VOLTANA_MAX_LEVELS, 64, n_scenarios, total_requests).total;
}

size_t voltana_simulate_workspace_bytes(const voltana_traces *traces_h, const voltana_layout *layouts_h,
                                        int n_layouts, size_t n_scenarios) {
  return voltana_simulate_workspace_bytes_ex(traces_h, layouts_h, n_layouts, n_scenarios, 0);
}

voltana_status voltana_simulate(const voltana_traces *traces_h, const voltana_slo *slos_h, int n_slos,
                                const voltana_layout *layouts_h, int n_layouts, const voltana_grid *grids_h,
                                int n_grids, const voltana_profile *profiles_h, int n_profiles,
                                const voltana_scenarios *scen_h, size_t n, voltana_result *out, void *workspace,
                                size_t ws_bytes, void *stream) {
  return voltana_simulate_ex(traces_h, slos_h, n_slos, layouts_h, n_layouts, grids_h, n_grids, profiles_h,
                             n_profiles, scen_h, n, out, nullptr, workspace, ws_bytes, stream);
}

voltana_status voltana_simulate_ex(const voltana_traces *traces_h, const voltana_slo *slos_h, int n_slos,
                                   const voltana_layout *layouts_h, int n_layouts, const voltana_grid *grids_h,
                                   int n_grids, const voltana_profile *profiles_h, int n_profiles,
                                   const voltana_scenarios *scen_h, size_t n, voltana_result *out,
                                   const voltana_outputs *outputs_h, void *workspace, size_t ws_bytes,
                                   void *stream) {
  g_launches = 0;
  if (outputs_h) {
    const voltana_outputs &o = *outputs_h;
    if (o.req_offset && (!o.req_tfirst || !o.req_tdone || !o.req_itl || !o.req_decode || !o.req_case))
      return fail(VOLTANA_E_INVALID_ARG, "simulate: outputs.req_* null with req_offset set");
    if (o.iter_offset && (!o.iters || !o.iter_count || o.iter_cap < 1))
      return fail(VOLTANA_E_INVALID_ARG, "simulate: outputs.iters/iter_count null or iter_cap == 0");
  }
  if (!traces_h || !slos_h || !layouts_h || !grids_h || !profiles_h || !scen_h)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: null table pointer");
  if (n_slos < 1 || n_slos > MAX_SLOS) return fail(VOLTANA_E_INVALID_ARG, "simulate: n_slos=%d (1..64)", n_slos);
  if (n_layouts < 1 || n_layouts > MAX_LAYOUTS)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: n_layouts=%d (1..16)", n_layouts);
  if (n_grids < 1 || n_grids > MAX_GRIDS) return fail(VOLTANA_E_INVALID_ARG, "simulate: n_grids=%d (1..16)", n_grids);
  if (n_profiles < 1 || n_profiles > MAX_PROFILES)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: n_profiles=%d (1..8)", n_profiles);
  if (n > 0x7fffffffull) return fail(VOLTANA_E_INVALID_ARG, "simulate: n=%zu too large", n);
  if (traces_h->max_requests > 0x7ffffffeull)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: traces.max_requests too large");
  if (traces_h->max_out < 1 || traces_h->max_out > 65535)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: traces.max_out=%u outside 1..65535", traces_h->max_out);
  voltana_status s;
  for (int i = 0; i < n_slos; ++i) {
    const voltana_slo &x = slos_h[i];
    if (!(x.ttft_ms > 0) || !(x.itl_ms > 0) || !(x.scale > 0) || !std::isfinite(x.ttft_ms) ||
        !std::isfinite(x.itl_ms) || !std::isfinite(x.scale))
      return fail(VOLTANA_E_INVALID_ARG, "simulate: slos[%d] must be positive and finite", i);
  }
  for (int i = 0; i < n_layouts; ++i) {
    const voltana_layout &x = layouts_h[i];
    if (x.n_p < 1 || x.n_p > VOLTANA_MAX_INSTANCES || x.n_d < 1 || x.n_d > VOLTANA_MAX_INSTANCES)
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d] n_p=%d n_d=%d (1..8)", i, x.n_p, x.n_d);
    if (x.policy < 0 || x.policy > 2) return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].policy=%d", i, x.policy);
    if (x.ctrl_mode != 0 && x.ctrl_mode != 1)
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].ctrl_mode=%d", i, x.ctrl_mode);
    if (x.itl_mode < 0 || x.itl_mode > 2)
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].itl_mode=%d (0 mean, 1 max, 2 P99)", i, x.itl_mode);
    if (!(x.ctrl_interval_ms >= 0.0 && x.ctrl_interval_ms < 1e12))
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].ctrl_interval_ms must be in [0, 1e12)", i);
    if (!(x.freq_overhead_ms >= 0.0 && x.freq_overhead_ms < 1e9))
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].freq_overhead_ms must be in [0, 1e9)", i);
    if (x.exec_noise && (x.noise_len == 0 || (x.noise_len & (x.noise_len - 1)) != 0))
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].noise_len=%u must be a power of two", i, x.noise_len);
    if (x.max_batch_tokens == 0 || x.max_batch_tokens > 0x7fffffffu || x.kv_capacity == 0 ||
        x.kv_capacity > 0x7fffffffu)
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d] B or C outside 1..2^31-1", i);
    if (!(x.kv_transfer_ms == 0.0 || x.kv_transfer_ms >= 1e-3) || !std::isfinite(x.kv_transfer_ms))
      return fail(VOLTANA_E_CONFIG, "simulate: layouts[%d].kv_transfer_ms must be 0 or >= 1e-3", i);
  }
  for (int i = 0; i < n_profiles; ++i) {
    char what[64];
    snprintf(what, sizeof(what), "simulate: profiles[%d]", i);
    if ((s = check_profile(&profiles_h[i], what)) != VOLTANA_OK) return s;
  }
  int kmin = profiles_h[0].k;
  for (int j = 1; j < n_profiles; ++j) kmin = profiles_h[j].k < kmin ? profiles_h[j].k : kmin;
  for (int i = 0; i < n_grids; ++i) {
    char what[64];
    snprintf(what, sizeof(what), "simulate: grids[%d]", i);
    // every grid must be valid on every profile it may be paired with
    if ((s = check_ladder(grids_h[i].level, grids_h[i].k, kmin, what)) != VOLTANA_OK) return s;
  }
  if (n == 0) return ok();
  if (!out || !traces_h->arrival || !traces_h->in_len || !traces_h->out_len || !traces_h->offset ||
      !traces_h->duration_ms || !scen_h->trace_id || !scen_h->slo_id || !scen_h->layout_id || !scen_h->grid_id ||
      !scen_h->profile_id || !scen_h->hash_seed)
    return fail(VOLTANA_E_INVALID_ARG, "simulate: null device array");
  int kmax, tmax;
  table_extent(grids_h, n_grids, profiles_h, n_profiles, &kmax, &tmax);
  // fast tables: every ladder K <= 8, ITL tables staged, pow2 tiles, no prefill tiles
  bool fast = (size_t)kmax * tmax * 24 <= SIM_ITL_SMEM_MAX && kmax <= 8;
  for (int i = 0; i < n_profiles; ++i)
    fast = fast && (profiles_h[i].tile_w & (profiles_h[i].tile_w - 1)) == 0 && profiles_h[i].n_ptiles <= 1;
  const uint64_t total_req = scen_h->node_offset ? scen_h->total_requests : 0;
  SimLayout L = sim_layout(traces_h, layouts_h, n_layouts, kmax, tmax, n, total_req, fast);
  const size_t need = voltana_simulate_workspace_bytes_ex(traces_h, layouts_h, n_layouts, n, total_req);
  if (!workspace || ws_bytes < need || ws_bytes < L.total)
    return fail(VOLTANA_E_WORKSPACE, "simulate: workspace %zu < %zu bytes", ws_bytes, need);
  int v = 0;  // variant bits of the instantiation: 1 energy scoring, 2 light variants / outputs
  for (int i = 0; i < n_layouts; ++i) {
    const voltana_layout &x = layouts_h[i];
    if (x.policy == 2 || x.ctrl_mode != 0) v |= 1;
    if (x.ctrl_interval_ms > 0.0 || x.freq_overhead_ms > 0.0 || x.exec_noise != nullptr || x.itl_mode != 0) v |= 2;
  }
  if (outputs_h && (outputs_h->req_offset != nullptr || outputs_h->iter_offset != nullptr)) v |= 2;  // E1-E2
  if (v == 0 && fast && kmax <= 5) {  // the N_D = 2 EcoRoute instantiation (decision table, fewer registers)
    bool nd2 = true;
    for (int i = 0; i < n_layouts; ++i) nd2 = nd2 && layouts_h[i].n_d == 2 && layouts_h[i].policy == 0;
    if (nd2) v = 4;
  }
  // every kernel attribute is set before anything of this call is enqueued: a non-OK return
  // below this point is a launch failure (VOLTANA_E_CUDA), the only partial-enqueue case
  cudaError_t e = cudaFuncSetAttribute(sim_kernel_ptr(v, fast), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L.smem);
  if (e != cudaSuccess) return cuda_fail(e, "simulate kernel attribute");

  static_assert(sizeof(SimParams) < 32000, "kernel parameter block too large");
  SimParams *P = new SimParams;
  memset(P, 0, sizeof(SimParams));
  P->arrival = traces_h->arrival; P->in_len = traces_h->in_len; P->out_len = traces_h->out_len;
  P->offset = traces_h->offset; P->duration = traces_h->duration_ms;
  P->trace_id = scen_h->trace_id; P->slo_id = scen_h->slo_id; P->layout_id = scen_h->layout_id;
  P->grid_id = scen_h->grid_id; P->profile_id = scen_h->profile_id; P->hash_seed = scen_h->hash_seed;
  P->node_offset = scen_h->node_offset;
  P->n = (uint32_t)n; P->nb = L.nb; P->max_out = traces_h->max_out; P->out = out;
  P->n_slots = L.n_slots;
  P->n_slos = (uint32_t)n_slos; P->n_layouts = (uint32_t)n_layouts; P->n_grids = (uint32_t)n_grids;
  P->n_profiles = (uint32_t)n_profiles; P->n_traces = traces_h->n_traces;
  P->max_requests = traces_h->max_requests;
  if (outputs_h) P->o = *outputs_h;  // zeroed (off) otherwise
  char *ws = (char *)workspace;
  P->counter = (uint32_t *)ws;
  P->slots = ws + L.slots_off;
  P->slot_bytes = L.slot;
  P->wheels = (uint4 *)(ws + L.wheels_off);
  if (L.ring_r) {
    P->ring_e = (double *)(ws + L.ring_e_off);
    P->ring_c = (uint32_t *)(ws + L.ring_c_off);
    P->ring_r = L.ring_r;
    P->ring_nd = L.ring_nd;
  }
  P->utab = (const double *)(ws + L.utab_off);
  P->nodes = ws + L.nodes_off;
  P->pares = (PaRes *)(ws + L.pares_off);
  P->rtab = (double *)(ws + L.rtab_off);
  P->ks_off = L.ks_off;
  P->np_max = 1;
  for (int i = 0; i < n_layouts; ++i) P->np_max = (uint32_t)layouts_h[i].n_p > P->np_max ? layouts_h[i].n_p : P->np_max;
  P->wheel_per_slot = L.wheel_per_slot;
  P->itl_smem = L.itl_smem;
  P->smem_per_warp = (uint32_t)L.smem_per_warp;
  P->timing = g_debug_timing;
  for (int i = 0; i < n_slos; ++i) P->slo[i] = slos_h[i];
  for (int i = 0; i < n_layouts; ++i) P->lay[i] = layouts_h[i];
  for (int i = 0; i < n_grids; ++i) P->grid[i] = grids_h[i];
  for (int i = 0; i < n_profiles; ++i) P->prof[i] = to_dev(profiles_h[i]);
  cudaStream_t st = (cudaStream_t)stream;
  // scenario counter = 0; every wheel bucket empty (buckets are left clean after use)
  e = cudaMemsetAsync(P->counter, 0, 4 * sizeof(uint32_t), st);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(P->wheels, 0, (size_t)L.n_slots * L.wheel_per_slot * sizeof(uint4), st);
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "simulate memset"); }
  const int per_cta = SIM_THREADS / 32;
  const int grid = (int)((L.n_slots + per_cta - 1) / per_cta);
  e = launch_utab(*P, st);  // setup: utilisation table and ladder-resolved prefill rows
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "simulate setup launch"); }
  e = launch_prefill(*P, v, fast, st);  // K4a: every prefill timeline of every scenario
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "simulate prefill launch"); }
  if (g_split_event) {
    e = cudaEventRecord((cudaEvent_t)g_split_event, st);
    if (e != cudaSuccess) { delete P; return cuda_fail(e, "simulate split event"); }
  }
  e = launch_sim(*P, v, fast, grid, L.smem, st);  // K4b: routing + decode, ITL pass in-warp
  delete P;
  if (e != cudaSuccess) return cuda_fail(e, "simulate launch");
  g_launches = 3;
  return ok();
}

// ------------------------------------------------------------------ K5
voltana_status voltana_series_to_samples(const voltana_outputs *o, const voltana_layout *layouts_h, int n_layouts,
                                         const voltana_grid *grids_h, int n_grids, const voltana_scenarios *scen_h,
                                         size_t n, size_t n_slots, uint32_t profile_id, uint8_t *phase,
                                         uint16_t *level, uint32_t *n_bt, uint32_t *n_req, uint32_t *n_kv,
                                         double *lat_ms, void *stream) {
  g_launches = 0;
  if (!o || !layouts_h || !grids_h || !scen_h)
    return fail(VOLTANA_E_INVALID_ARG, "series_to_samples: null table pointer");
  if (!o->iters || !o->iter_count || !o->iter_offset || o->iter_cap < 1)
    return fail(VOLTANA_E_INVALID_ARG, "series_to_samples: outputs hold no iteration series");
  if (n_layouts < 1 || n_layouts > SERIES_MAX_LAYOUTS || n_grids < 1 || n_grids > SERIES_MAX_GRIDS)
    return fail(VOLTANA_E_INVALID_ARG, "series_to_samples: n_layouts=%d n_grids=%d (1..16)", n_layouts, n_grids);
  if (n == 0 || n_slots == 0) return ok();
  if (!scen_h->layout_id || !scen_h->grid_id || !scen_h->profile_id || !phase || !level || !n_bt || !n_req ||
      !n_kv || !lat_ms)
    return fail(VOLTANA_E_INVALID_ARG, "series_to_samples: null array pointer");
  SeriesParams P;
  memset(&P, 0, sizeof(P));
  P.iters = o->iters; P.iter_count = o->iter_count; P.iter_offset = o->iter_offset; P.cap = o->iter_cap;
  P.profile_id = profile_id;
  P.layout_id = scen_h->layout_id; P.grid_id = scen_h->grid_id; P.scen_profile_id = scen_h->profile_id;
  P.n = n; P.n_slots = n_slots;
  P.phase = phase; P.level = level; P.n_bt = n_bt; P.n_req = n_req; P.n_kv = n_kv; P.lat = lat_ms;
  for (int i = 0; i < n_layouts; ++i) P.n_p[i] = layouts_h[i].n_p;
  for (int i = 0; i < n_grids; ++i) P.grid[i] = grids_h[i];
  const size_t want = (n_slots + SERIES_THREADS - 1) / SERIES_THREADS;
  const int grid = (int)(want < (size_t)sm_count() * 8 ? want : (size_t)sm_count() * 8);
  cudaError_t e = launch_series(P, grid, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "series_to_samples launch");
  g_launches = 1;
  return ok();
}

}  // extern "C"
