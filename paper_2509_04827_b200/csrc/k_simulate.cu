// k_simulate.cu — K4: batched trace-driven evaluation of EcoFreq + EcoRoute (north_star).
//
// One warp per scenario (persistent warps claim scenarios in array order). The scenario
// is evaluated through its exact causal decomposition:
//
//  Phase A  Prefill instances never read decode state: requests go round robin by id
//            and batches are FCFS (A6). Each prefill instance p is simulated
//           by lane p, independently: batch formation, EcoFreq with the waiting-time budget
//           (P:377-388), TTFT accounting, energy. Output: every request's first-token time,
//           and per instance the chain of routed requests (out > 1) in completion order.
//  Phase B  Routing happens at prefill completions, in (time, instance, id)
//           order: a warp-wide min over the N_P stream heads picks the next request. Before
//           routing at time t, decode lane d advances its own instance through every event
//           strictly before t (iteration END/START, admission, EcoFreq, energy) — decode
//           instances interact only through routing, and at equal times a PrefillDone drains
//           before a DecodeIterDone and before every START (A18), so this order is exact.
//           The what-if (f, f') of instance d is evaluated by lane d on its own state; the
//           case analysis is a handful of warp reductions (ballot / reduce_min).
// Decisions therefore match the sequential oracle bit for bit; the record's report-only
// accumulators are per instance (A36/A37), so they match bit for bit too.
//
// Decode running sets: a per-instance timing wheel of NB (<= 1024, L2-resident) buckets keyed
// by the iteration at which a request finishes (admission iteration + out - 2). All running
// requests advance together (+1 token per iteration), so a bucket's request count and
// KV total retire the whole iteration's completions in O(1); the rare request finishing NB or
// more iterations ahead waits on a sorted far list until its bucket enters the window. Bucket
// lists keep admission order; the per-request ITL accounting (A30) walks them later, in
// completion order, off the decision chain.
//
// Register budget: per-lane instance state lives in registers; everything cold (scenario
// constants, staged tables, phase-A results) lives in a per-warp shared-memory block.
#include <cstdint>

#include "vt_device.cuh"
#include "vt_sim.h"

#ifndef VT_QCACHE
#define VT_QCACHE 1    // keep the admission-queue head node in registers
#endif
#ifndef VT_BHPF
#define VT_BHPF 0      // prefetch the bucket the queue head will join at the next START
#endif
#ifndef VT_TWO_ENDED
#define VT_TWO_ENDED 0 // heavy scenarios claimed by the last warp of each CTA (arbiter priority)
#endif
#ifndef VT_DACC_SMEM
#define VT_DACC_SMEM 0 // decode-lane accumulators in shared memory instead of registers
#endif
#if VT_DACC_SMEM
#define ACC(f) W.da_##f[d]
#else
#define ACC(f) D.f
#endif
#ifndef VT_ITL_FIFO
#define VT_ITL_FIFO 1  // completion lists deferred before their ITL accounting runs (1..8; 1 measured best)
#endif

#ifndef VT_L2HINT
#define VT_L2HINT 0    // wheel buckets loaded/stored with an L2 evict_last cache policy
#endif
#ifndef VT_PIPE_ARGMIN
#define VT_PIPE_ARGMIN 0  // select the next request right after advancing the stream (overlap)
#endif
#ifndef VT_PF
#define VT_PF 2        // software prefetch: 1 next stream line, 2 + the queue head admission bucket (3, 4: measured no gain)
#endif
#ifndef VT_SWHEEL
#define VT_SWHEEL 0    // near timing-wheel window in shared memory (buckets; power of two, 0 = off)
#endif
#ifndef VT_PFA
#define VT_PFA 0       // prefill lanes: prefetch the trace this many requests ahead (0 = off)
#endif
#ifndef VT_ADM_DEFER
#define VT_ADM_DEFER 0  // K4b: wheel appends applied at the next START, line prefetched now (measured +5 %: off)
#endif
constexpr uint32_t ADM_PQ = 8;  // pending appends per decode lane (shared memory)
#ifndef VT_SCAN_ILP
#define VT_SCAN_ILP 0  // K4b fast tables: all K evaluations issued together (heaviest alone -4 %, full sweep +24 %: off)
#endif
#ifndef VT_NODE_PF_L1
#define VT_NODE_PF_L1 8  // K4b: L1 prefetch of the prefill stream this many request ids ahead
#endif
#ifndef VT_NODE_PF_L2
#define VT_NODE_PF_L2 0  // K4b: bulk L2 prefetch of the node array this many requests ahead (1024/4096: no gain)
#endif
#ifndef VT_EDEFER
#define VT_EDEFER 0    // decode busy energy: table loads issued at START, added at END (measured: no gain)
#endif
#ifndef VT_ITL_SMEM_ONLY
#define VT_ITL_SMEM_ONLY 0  // experiment: assume the ITL table is staged (no global fallback)
#endif

namespace vt {

// ---- wheel bucket access (optionally pinned in L2 against the streaming node traffic)
__device__ __forceinline__ uint4 wld(const uint4 *a) {
#if VT_L2HINT
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint4 r;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(a), "l"(pol) : "memory");
  return r;
#else
  return *a;
#endif
}
__device__ __forceinline__ void wst(uint4 *a, uint4 v) {
#if VT_L2HINT
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
#else
  *a = v;
#endif
}

__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" :: "l"(p)); }

// ---- scenario groups: SPW scenarios per warp, GS lanes each; every collective is group-masked
constexpr int GS = 32 / SPW;
__device__ __forceinline__ int glane() { return (int)(threadIdx.x & (GS - 1)); }
__device__ __forceinline__ unsigned gbase() { return (threadIdx.x & 31u) & ~(unsigned)(GS - 1); }
__device__ __forceinline__ unsigned gmask() { return GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << gbase()); }
__device__ __forceinline__ unsigned gballot(bool p) { return __ballot_sync(gmask(), p) >> gbase(); }
template <class T> __device__ __forceinline__ T gshfl(T v, int src) { return __shfl_sync(gmask(), v, src, GS); }

struct Node {       // 16 B per request (workspace)
  double tf;        // +t_first if the TTFT SLO was met, -t_first otherwise (t_first > 0)
  uint32_t next;    // phase A: next routed request of the same prefill stream; later: queue/wheel link
  uint16_t in, out;
};

constexpr int ITL_FIFO = VT_ITL_FIFO;  // deferred completion lists per decode lane
constexpr int NI = VOLTANA_MAX_INSTANCES;

// Per-warp shared-memory block (one scenario at a time). Sized by SIM_SMEM_FIXED.
template <int KC>  // KC: level capacity of the staged tables (8 in the fast-table kernel, else 64)
struct WarpSmemT {
  // ---- deferred ITL accounting: completion-list heads and times, per decode lane
  uint32_t fid[NI][ITL_FIFO];
  double ft[NI][ITL_FIFO];
  // ---- phase-A results per prefill lane (read back for the record)
  PaRes pa[NI];
#if VT_DACC_SMEM
  // ---- decode-lane accumulators (VT_DACC_SMEM)
  double da_ebusy[NI], da_bms[NI], da_top[NI], da_sitl[NI], da_tlast[NI];
  uint64_t da_h[NI];
  uint32_t da_n_itl_ok[NI], da_n_both[NI];
#endif
  // ---- scenario constants
  double tau, slo_itl, tgt_itl, slo_ttft, tgt_ttft, p_idle, tdp, uh_p, uh_d;
  const double *a2g, *b2g, *c2g;   // profile ITL tables (when not staged)
  const double *a1g, *c1g;         // profile TTFT tables [T_p][kp] (read when T_p > 1, F1)
  uint32_t ptiles, pcut;           // prefill tiles T_p (>= 1), cutoff
  const double *ut;                // VT_UTAB: this profile's utilisation tables [2][SIM_UTAB]
  uint32_t kvcap, max_steps, B, K, T, W, kp, nb;
  int32_t wshift;
  uint32_t itl_smem, mono_tt, mono_it;
  uint32_t ctrl;                   // layout ctrl_mode: 0 EcoFreq, 1 energy argmin [B4]
  double ctrl_iv, fs_ov;           // window interval, blocking frequency-set overhead [C1-C3]
  const double *noise;             // execution-noise factor table or NULL [D1, D2]
  uint32_t noise_mask, np;         // np: N_P (decode instance d is noise instance N_P + d)
  uint64_t seed;                   // scenario hash seed (noise index)
  double *re;                      // ITL modes (E3): this slot's rings [N_D][ring_r] of iteration end times
  uint32_t *rc;                    //   ... and of cumulative counts of gaps above the ITL SLO
  uint32_t itlm, rmask;            //   layout itl_mode, ring_r - 1
  uint32_t clog_m;                 // VT_DEFER_ITL: log slots handed out (chunks of CLOG_CHUNK)
#if VT_ADM_DEFER
  uint32_t pq_i[NI][ADM_PQ], pq_fin[NI][ADM_PQ], pq_io[NI][ADM_PQ];  // decode lane: pending wheel appends
#endif
  uint32_t wo;                     // window control or blocking overhead active (C1-C3)
  uint32_t dl_vc[VOLTANA_MAX_INSTANCES];  // decode lane: gaps above the ITL SLO so far
  uint64_t rq_base, it_base;       // outputs (E1-E3): request / iteration-slot base of the scenario
  uint32_t rq_on, it_on;
  // ---- variant-kernel per-instance controller state [C1-C3]
  double dl_last[NI];              // decode lane: time of the last decision (-inf: none)
  uint32_t dl_cur[NI], dl_ndec[NI];  // decode lane: running level, decisions taken
  // ---- staged ladder tables
  uint16_t lad[KC];
  int32_t mhz[KC];
  double tt[2 * KC];   // [K][2]: a1, c1
  double dyn[2 * KC];  // [2][K]: prefill, decode
  double it[1];                        // [T][K][3]: a2, b2, c2 (flexible; itl_smem)
};

// ------------------------------------------------------------------ EcoPred on staged tables
// F ("fast tables"): the ITL table is staged, K <= 8 and the tile width is a power of two for
// every scenario of the launch (host-checked): the dead general paths are compiled out.
template <bool F, class WS>
__device__ __forceinline__ uint32_t tile_j(const WS &W, uint32_t n) {
  const uint32_t j = (F || W.wshift >= 0) ? (n - 1u) >> W.wshift : (n - 1u) / W.W;
  return j < W.T - 1u ? j : W.T - 1u;
}

// eq:pred-itl at ladder index k, tile j; dn = (double)N_req, dkv = (double)N_kv (exact)
template <bool F, class WS>
__device__ __forceinline__ double itl_at(const WS &W, uint32_t j, int k, double dn, double dkv) {
  if (F || VT_ITL_SMEM_ONLY || W.itl_smem) {
    const double *r = W.it + 3 * ((size_t)j * W.K + k);
    return add(add(mul(r[0], dn), mul(r[1], dkv)), r[2]);
  }
  const size_t o = (size_t)j * W.kp + W.lad[k];
  return add(add(mul(__ldg(W.a2g + o), dn), mul(__ldg(W.b2g + o), dkv)), __ldg(W.c2g + o));
}

template <bool F, class WS>
__device__ __forceinline__ double ttft_at(const WS &W, int k, uint32_t nbt) {
  if (F || W.ptiles <= 1u) return ttft_pred(W.tt[2 * k], W.tt[2 * k + 1], nbt);
  // prefill tiles (F1): the batch's tile row of the profile tables
  const size_t o = (size_t)ptile_of(nbt, W.W, W.ptiles, W.pcut) * W.kp + W.lad[k];
  return ttft_pred(__ldg(W.a1g + o), __ldg(W.c1g + o), nbt);
}

// Lowest ladder index whose prediction meets `target` (A1), else K-1 (A2);
// *pred = the prediction there. Ascending scan with early exit, or an exact binary search
// when the tables are coefficient-monotone in f (A32).
// All KK levels evaluated independently (no early-exit chain: the evaluations overlap), then
// the lowest feasible one selected from the top down — the same values as the ascending scan.
template <int KK, class WS>
__device__ __forceinline__ int lowest_itl_ilp(const WS &W, uint32_t j, double dn, double dkv, double target,
                                              double *pred) {
  double p[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) {
    const double *r = W.it + 3 * ((size_t)j * KK + k);
    p[k] = add(add(mul(r[0], dn), mul(r[1], dkv)), r[2]);
  }
  int kk = KK - 1;
  double pp = p[KK - 1];
#pragma unroll
  for (int k = KK - 2; k >= 0; --k)
    if (p[k] <= target) { kk = k; pp = p[k]; }
  *pred = pp;
  return kk;
}

template <bool F, class WS>
__device__ int lowest_itl(const WS &W, uint32_t n, uint32_t kv, double target, double *pred) {
  const uint32_t j = tile_j<F>(W, n);
  const int K = (int)W.K;
  const double dn = (double)n, dkv = (double)kv;
#if VT_SCAN_ILP
  if (F) {
    switch (K) {
      case 1: return lowest_itl_ilp<1>(W, j, dn, dkv, target, pred);
      case 2: return lowest_itl_ilp<2>(W, j, dn, dkv, target, pred);
      case 3: return lowest_itl_ilp<3>(W, j, dn, dkv, target, pred);
      case 4: return lowest_itl_ilp<4>(W, j, dn, dkv, target, pred);
      case 5: return lowest_itl_ilp<5>(W, j, dn, dkv, target, pred);
      case 6: return lowest_itl_ilp<6>(W, j, dn, dkv, target, pred);
      case 7: return lowest_itl_ilp<7>(W, j, dn, dkv, target, pred);
      default: return lowest_itl_ilp<8>(W, j, dn, dkv, target, pred);
    }
  }
#endif
  if (!F && W.mono_it && K > 8) {
    int lo = 0, hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (itl_at<F>(W, j, mid, dn, dkv) <= target) hi = mid; else lo = mid + 1;
    }
    const int k = lo < K ? lo : K - 1;
    *pred = itl_at<F>(W, j, k, dn, dkv);
    return k;
  }
  for (int k = 0; k < K - 1; ++k) {
    const double p = itl_at<F>(W, j, k, dn, dkv);
    if (p <= target) { *pred = p; return k; }
  }
  *pred = itl_at<F>(W, j, K - 1, dn, dkv);
  return K - 1;
}

template <bool F, class WS>
__device__ int lowest_ttft(const WS &W, uint32_t nbt, double budget, double *pred) {
  const int K = (int)W.K;
  if (!F && W.mono_tt && K > 8) {
    int lo = 0, hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ttft_at<F>(W, mid, nbt) <= budget) hi = mid; else lo = mid + 1;
    }
    const int k = lo < K ? lo : K - 1;
    *pred = ttft_at<F>(W, k, nbt);
    return k;
  }
  for (int k = 0; k < K - 1; ++k) {
    const double p = ttft_at<F>(W, k, nbt);
    if (p <= budget) { *pred = p; return k; }
  }
  *pred = ttft_at<F>(W, K - 1, nbt);
  return K - 1;
}

// busy power (eq:P-f P:187, A22) with the utilisation from the launch's table when tabulated
// (VT_UTAB; the entries are the same division, so the value is identical)
template <class WS>
__device__ __forceinline__ double bpow(const WS &W, int phase, double dyn, uint32_t load) {
#if VT_UTAB
  const double uh = phase ? W.uh_d : W.uh_p;
  const double u = load < SIM_UTAB ? __ldg(W.ut + phase * SIM_UTAB + load) : div((double)load, add((double)load, uh));
  const double w = add(W.p_idle, mul(u, dyn));
  return w < W.tdp ? w : W.tdp;
#else
  return busy_power(W.p_idle, W.tdp, phase ? W.uh_d : W.uh_p, dyn, load);
#endif
}

// Energy-argmin controller [B4]: among the levels meeting the target, the lowest busy
// energy P(k, load) * T(k) (eq:P-f P:187, energy = time x power P:74); ties -> lower level;
// none feasible -> K-1 (A2). Full scan (the energy curve is not monotone).
template <bool F, class WS>
__device__ int energy_itl(const WS &W, uint32_t n, uint32_t kv, double target, double *pred) {
  const uint32_t j = tile_j<F>(W, n);
  const int K = (int)W.K;
  const double dn = (double)n, dkv = (double)kv;
  int best = -1;
  double be = 0.0, bt = 0.0;
  for (int k = 0; k < K; ++k) {
    const double t = itl_at<F>(W, j, k, dn, dkv);
    if (!(t <= target)) continue;
    const double e = mul(bpow(W, 1, W.dyn[K + k], n), t);
    if (best < 0 || e < be) { best = k; be = e; bt = t; }
  }
  if (best < 0) { best = K - 1; bt = itl_at<F>(W, j, K - 1, dn, dkv); }
  *pred = bt;
  return best;
}

template <bool F, class WS>
__device__ int energy_ttft(const WS &W, uint32_t nbt, double budget, double *pred) {
  const int K = (int)W.K;
  int best = -1;
  double be = 0.0, bt = 0.0;
  for (int k = 0; k < K; ++k) {
    const double t = ttft_at<F>(W, k, nbt);
    if (!(t <= budget)) continue;
    const double e = mul(bpow(W, 0, W.dyn[k], nbt), t);
    if (best < 0 || e < be) { best = k; be = e; bt = t; }
  }
  if (best < 0) { best = K - 1; bt = ttft_at<F>(W, K - 1, nbt); }
  *pred = bt;
  return best;
}

// [D2] execution-noise factor of iteration j of instance inst: counter-based index into the
// host-drawn table (no transcendental on either side).
template <class WS>
__device__ __forceinline__ double noise_at(const WS &W, uint64_t inst, uint64_t j) {
  const uint64_t x = W.seed ^ 0xD1B54A32D192ED03ull ^ (inst << 40) ^ j;
  return __ldg(W.noise + (splitmix64(x) & W.noise_mask));
}

// ------------------------------------------------------------------ decode lanes
// Timing-wheel bucket (16 B; all-zero = empty): x = first request + 1, y = last request + 1
// (list in admission order), z = requests finishing in this iteration, w = their in + out.
struct Err {               // first error of one lane in its own event order
  double t;                // +inf = none
  uint32_t code;
};

struct Dec {               // decode instance d, owned by lane d
  uint32_t nreq, nkv, pn, pkv, iters, cur, qh, qt, n_itl_ok, n_both, nfifo, far_h, far_hfin;
  bool busy, dead;
#if VT_ADM_DEFER
  uint32_t npq;            // pending wheel appends (admitted at the last START, applied at the next)
#endif
  double end, ebusy, bms, top, sitl, tlast;
#if VT_EDEFER
  double e_u, e_dyn, e_dur;  // running iteration's utilisation, DYN entry and duration (energy added at END)
#endif
  uint64_t h;
  uint4 bcur;              // bucket of the running iteration, read at its START (final by then)
#if VT_DEFER_ITL
  uint32_t lpos, lend;     // this lane's chunk [lpos, lend) of the scenario's completion log
  bool lneed;              // the chunk is full: dec_advance stopped before an END
#endif
#if VT_QCACHE
  Node qhn;                // register copy of the admission-queue head node
#endif
#if VT_BHPF
  uint32_t bh_fin;
  uint4 bh;
#endif
#if VT_PF == 4
  uint32_t nxh;            // head (+1) of the next iteration's bucket as read one START early (prefetch only)
#endif
};

struct Lane {              // per-lane pointers
#if VT_SWHEEL
  uint4 *sw;               // near wheel in shared memory: buckets [iters, iters + VT_SWHEEL)
#endif
  Node *node;
  uint32_t *farfin;        // [N] finishing iteration of requests on the far list
  uint4 *wheel;            // this lane's decode instance: [NB] buckets
  uint32_t *fid;
  double *ft;
  CEnt *clog;              // VT_DEFER_ITL: the scenario's completion log
};

__device__ __forceinline__ Node queue_head(const Dec &D, const Lane &L) {
#if VT_QCACHE
  return D.qhn;
#else
  return L.node[D.qh];
#endif
}

// ITL accounting of deferred completion lists, in completion order (A30, A37); the head
// nodes of up to four lists are loaded together.
template <int V, bool F, class WS>
__device__ void itl_drain(Dec &D, const Lane &L, WS &W, int d, const voltana_outputs &O) {
#ifdef VT_ITL_SKIP
  D.nfifo = 0;  // experiment only (wrong records): the cost of the ITL walk
  return;
#endif
  const double slo = W.slo_itl;
  for (uint32_t e0 = 0; e0 < D.nfifo; e0 += 4) {
    Node h4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u < D.nfifo) h4[u] = L.node[L.fid[e0 + u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (e0 + u >= D.nfifo) continue;
      const double td = L.ft[e0 + u];
      Node nd = h4[u];
      uint32_t id = L.fid[e0 + u];
      for (uint32_t hop = 0; hop < W.max_steps; ++hop) {
        const double itl = div(sub(td, fabs(nd.tf)), (double)(nd.out - 1u));
        ACC(sitl) = add(ACC(sitl), itl);
        bool ok = itl <= slo;
        if ((V & 2) && W.itlm) {
          // ITL Max / P99 (E3): the request's gaps are e_a - t_first and the iteration gaps of
          // (a, f], f = this iteration, a = f - (out - 2); count those above the SLO from the
          // instance's rings and compare with the nearest-rank allowance (0 for Max)
          static_assert(VT_ITL_FIFO == 1, "ITL modes read the completing iteration from D.cur");
          const uint32_t n = (uint32_t)nd.out - 1u;
          const uint32_t a = D.cur - (n - 1u);
          const double ea = W.re[(size_t)d * (W.rmask + 1u) + (a & W.rmask)];
          const uint32_t ca = W.rc[(size_t)d * (W.rmask + 1u) + (a & W.rmask)];
          const uint32_t viol = (W.dl_vc[d] - ca) + (sub(ea, fabs(nd.tf)) > slo ? 1u : 0u);
          const uint32_t allow = W.itlm == 1u ? 0u : n - (99u * n + 99u) / 100u;
          ok = viol <= allow;
        }
        ACC(n_itl_ok) += ok;
        ACC(n_both) += ok && nd.tf > 0.0;
        if ((V & 2) && W.rq_on) {  // per-request record (E1)
          O.req_tdone[W.rq_base + id] = td;
          O.req_itl[W.rq_base + id] = itl;
        }
        if (nd.next == NIL) break;
        id = nd.next;
        nd = L.node[id];
      }
    }
  }
  D.nfifo = 0;
}

// iteration record of the per-instance time series (E2)
template <class WS>
__device__ __forceinline__ void log_iter(const voltana_outputs &O, const WS &W, uint32_t u, uint32_t j,
                                         double t, double dur, uint32_t load, uint32_t kv, int k, uint32_t flags) {
  if (!W.it_on || j >= O.iter_cap) return;
  voltana_iteration r;
  r.t_start = t; r.dur_ms = dur; r.load = load; r.n_kv = kv; r.level = (uint16_t)k; r.flags = (uint8_t)flags;
#pragma unroll
  for (int x = 0; x < 5; ++x) r.reserved[x] = 0;
  O.iters[W.it_base + (uint64_t)u * O.iter_cap + j] = r;
}

// Bucket of finishing iteration fin >= D.iters during a START (before the iteration counter
// advances): the near window [iters, iters + VT_SWHEEL) lives in shared memory.
__device__ __forceinline__ uint4 bkt_ld(const Dec &D, const Lane &L, uint32_t nbm, uint32_t fin) {
#if VT_SWHEEL
  if (fin - D.iters < (uint32_t)VT_SWHEEL) return L.sw[fin & (VT_SWHEEL - 1)];
#endif
  return wld(L.wheel + (fin & nbm));
}
__device__ __forceinline__ void bkt_st(const Dec &D, const Lane &L, uint32_t nbm, uint32_t fin, uint4 b) {
#if VT_SWHEEL
  if (fin - D.iters < (uint32_t)VT_SWHEEL) { L.sw[fin & (VT_SWHEEL - 1)] = b; return; }
#endif
  wst(L.wheel + (fin & nbm), b);
}

// Append request i (finishing at iteration fin) to its bucket; (lfin, lb) = the bucket
// written last during this START, kept coherent with the prefetched copy.
__device__ __forceinline__ void bucket_append(Dec &D, const Lane &L, uint32_t nbm, uint32_t i, uint32_t fin,
                                              uint32_t inout, uint32_t &lfin, uint4 &lb) {
#if VT_BHPF
  uint4 b = fin == lfin ? lb : (fin == D.bh_fin ? D.bh : bkt_ld(D, L, nbm, fin));
#else
  uint4 b = fin == lfin ? lb : bkt_ld(D, L, nbm, fin);
#endif
  L.node[i].next = NIL;
  if (b.y == 0u) b.x = i + 1u; else L.node[b.y - 1u].next = i;
  b.y = i + 1u;
  b.z += 1u;
  b.w += inout;
  bkt_st(D, L, nbm, fin, b);
  lfin = fin;
  lb = b;
#if VT_BHPF
  if (fin == D.bh_fin) D.bh = b;
#endif
}

// A request finishing NB or more iterations ahead waits on the far list, sorted by
// (finishing iteration, admission order); rare (out > NB + 1).
__device__ void far_insert(Dec &D, const Lane &L, uint32_t max_steps, uint32_t i, uint32_t fin) {
  L.farfin[i] = fin;
  if (D.far_h == NIL || fin < D.far_hfin) {
    L.node[i].next = D.far_h;
    D.far_h = i;
    D.far_hfin = fin;
    return;
  }
  uint32_t prev = D.far_h;
  for (uint32_t hop = 0; hop < max_steps; ++hop) {
    const uint32_t nx = L.node[prev].next;
    if (nx == NIL || L.farfin[nx] > fin) break;
    prev = nx;
  }
  L.node[i].next = L.node[prev].next;
  L.node[prev].next = i;
}

// Advance decode instance `d` through every event with time < t_lim (END, START).
template <int V, bool F, class WS>  // V: variant bits, 1 energy scoring (B1-B4), 2 window/overhead/noise/ITL modes/outputs (C-E)
__device__ void dec_advance(Dec &D, int d, const Lane &L, WS &W, double t_lim, Err &E,
                            const voltana_outputs &O) {
  if (D.dead) return;
  const uint32_t nbm = W.nb - 1u;
  for (;;) {
    double tnow;
    bool cont = false;  // this START follows an END at the same time (the instance stays busy)
    if (D.busy) {
      if (!(D.end < t_lim)) return;
#if VT_DEFER_ITL
      if (!(V & 2) && D.lpos == D.lend) { D.lneed = true; return; }  // a new chunk first (dec_advance_all)
#endif
      tnow = D.end;
      cont = true;
      // ---- O6 DecodeIterDone: +1 KV token per running request; this iteration's completions
      D.nkv += D.nreq;
      const uint4 b = D.bcur;
      D.nreq -= b.z;
      D.nkv -= b.w;
      if (b.x != 0u) {
#if VT_SWHEEL
        L.sw[D.cur & (VT_SWHEEL - 1)] = make_uint4(0u, 0u, 0u, 0u);
#else
        wst(L.wheel + (D.cur & nbm), make_uint4(0u, 0u, 0u, 0u));
#endif
#if VT_DEFER_ITL
        if (!(V & 2)) {  // log (td, list head, instance); K4c does the ITL accounting (A30, A37)
          CEnt ce;
          ce.td = tnow; ce.head = b.x - 1u; ce.d = (uint32_t)d;
          L.clog[D.lpos++] = ce;
        } else
#endif
        {
          L.fid[D.nfifo] = b.x - 1u;
          L.ft[D.nfifo] = tnow;
          if (++D.nfifo == VT_ITL_FIFO) itl_drain<V, F>(D, L, W, d, O);
        }
      }
      D.busy = false;
      ACC(tlast) = tnow;
#if VT_EDEFER
      {  // busy energy of the iteration that just ended, in iteration order (W*ms, A23)
        const double w = add(W.p_idle, mul(D.e_u, D.e_dyn));
        ACC(ebusy) = add(ACC(ebusy), mul(w < W.tdp ? w : W.tdp, D.e_dur));
      }
#endif
    } else {
      // idle: the next START happens when the head of the admission queue becomes available
      if (D.qh == NIL) return;
      const double av = add(fabs(queue_head(D, L).tf), W.tau);  // KvTransferDone (A18)
      if (!(av < t_lim)) return;
      tnow = av;
    }
    // ---- O7 START_DECODE at tnow
    uint32_t lfin = NIL;
    uint4 lb = make_uint4(0u, 0u, 0u, 0u);
#if VT_SWHEEL
    {  // bucket iters + VT_SWHEEL - 1 enters the near window: global -> shared (its slot held
       // bucket iters - 1, completed and cleared at the previous END)
      const uint32_t m = D.iters + (uint32_t)VT_SWHEEL - 1u;
      const uint4 g = wld(L.wheel + (m & nbm));
      L.sw[m & (VT_SWHEEL - 1)] = g;
      if (g.z != 0u) wst(L.wheel + (m & nbm), make_uint4(0u, 0u, 0u, 0u));
      prefetch_l1(L.wheel + ((m + 1u) & nbm));   // the next START's migration
    }
#endif
    // far requests whose finishing iteration entered the window join their bucket now,
    // before any direct admission can reach that bucket (admission order, A37)
    while (D.far_h != NIL && D.far_hfin - D.iters < W.nb) {
      const uint32_t i = D.far_h;
      const Node fn = L.node[i];
      const uint32_t fin = D.far_hfin;
      D.far_h = fn.next;
      D.far_hfin = fn.next != NIL ? L.farfin[fn.next] : NIL;
      bucket_append(D, L, nbm, i, fin, (uint32_t)fn.in + fn.out, lfin, lb);
    }
#if VT_ADM_DEFER && !VT_SWHEEL
    // the previous START's admissions join their buckets now, in admission order (their lines
    // were prefetched then; none of them finishes before this iteration ends)
    for (uint32_t q = 0; q < D.npq; ++q) bucket_append(D, L, nbm, W.pq_i[d][q], W.pq_fin[d][q], W.pq_io[d][q], lfin, lb);
    D.npq = 0u;
#endif
    // FCFS admission while KV fits (A20)
    const double tau = W.tau;
    const uint32_t kvcap = W.kvcap;
    while (D.qh != NIL) {
      const Node hn = queue_head(D, L);
      if (!(add(fabs(hn.tf), tau) <= tnow)) break;  // still in KV transfer
      const uint32_t need = (uint32_t)hn.in + 1u;
      if (D.nkv + need > kvcap) break;
      const uint32_t i = D.qh;
      D.qh = hn.next;
      if (D.qh == NIL) D.qt = NIL;
#if VT_QCACHE
      else D.qhn = L.node[D.qh];
#endif
      const uint32_t fin = D.iters + (uint32_t)hn.out - 2u;  // its last iteration
      const uint32_t o2 = (uint32_t)hn.out - 2u;
      if (o2 < W.nb) {
#if VT_ADM_DEFER && !VT_SWHEEL
        if (o2 != 0u) {  // finishes after this iteration: append at the next START
          if (D.npq == ADM_PQ) {  // full: apply the pending ones first (admission order)
            for (uint32_t q = 0; q < ADM_PQ; ++q)
              bucket_append(D, L, nbm, W.pq_i[d][q], W.pq_fin[d][q], W.pq_io[d][q], lfin, lb);
            D.npq = 0u;
          }
          W.pq_i[d][D.npq] = i; W.pq_fin[d][D.npq] = fin; W.pq_io[d][D.npq] = (uint32_t)hn.in + hn.out;
          D.npq += 1u;
          prefetch_l1(L.wheel + (fin & nbm));
        } else
#endif
        bucket_append(D, L, nbm, i, fin, (uint32_t)hn.in + hn.out, lfin, lb);
      } else {
        far_insert(D, L, W.max_steps, i, fin);
      }
      D.nreq += 1u;
      D.nkv += need;
      D.pn -= 1u;
      D.pkv -= need;
    }
    const bool backlog = D.qh != NIL && add(fabs(queue_head(D, L).tf), tau) <= tnow;  // A5
    if (D.iters >= W.max_steps) { E.t = tnow; E.code = VOLTANA_ITEM_E_INTERNAL; D.dead = true; return; }
    if (D.nreq == 0u) {
      if (backlog) { E.t = tnow; E.code = VOLTANA_ITEM_E_KV; D.dead = true; return; }
      continue;  // stays idle
    }
    double dur;
    int k;
    uint32_t fl = backlog ? 4u : 0u;
    if ((V & 2) && W.wo && !(sub(tnow, W.dl_last[d]) >= W.ctrl_iv)) {  // window gating: keep the running level [C1]
      k = (int)W.dl_cur[d];
      dur = itl_at<F>(W, tile_j<F>(W, D.nreq), k, (double)D.nreq, (double)D.nkv);
    } else {
      fl |= 1u;
      if (backlog) { k = (int)W.K - 1; dur = itl_at<F>(W, tile_j<F>(W, D.nreq), k, (double)D.nreq, (double)D.nkv); }
      else if ((V & 1) && W.ctrl) k = energy_itl<F>(W, D.nreq, D.nkv, W.tgt_itl, &dur);  // B4
      else k = lowest_itl<F>(W, D.nreq, D.nkv, W.tgt_itl, &dur);
      ACC(h) = fold(ACC(h), 2, (uint64_t)d, (uint64_t)k, 0);
      if ((V & 2) && W.wo) { W.dl_last[d] = tnow; W.dl_ndec[d] += 1u; }
    }
    if (!(dur > 0.0)) { E.t = tnow; E.code = VOLTANA_ITEM_E_CONTRACT; D.dead = true; return; }
    if ((V & 2) && W.noise) {  // [D1]
      const double e = noise_at(W, (uint64_t)W.np + d, D.iters);
      if (!(e > 0.0 && e <= 1e6)) { E.t = tnow; E.code = VOLTANA_ITEM_E_INPUT; D.dead = true; return; }
      dur = mul(dur, e);
    }
    double t0 = tnow;
    if ((V & 2) && W.wo) {  // blocking frequency set on a level change [C3]
      if (k != (int)W.dl_cur[d] && W.fs_ov > 0.0) { t0 = add(tnow, W.fs_ov); fl |= 2u; }
      W.dl_cur[d] = (uint32_t)k;
    }
    if ((V & 2)) log_iter(O, W, W.np + (uint32_t)d, D.iters, tnow, dur, D.nreq, D.nkv, k, fl);
    D.end = add(t0, dur);
    D.busy = true;
    if ((V & 2) && W.itlm) {  // ITL modes (E3): gap e_i - e_{i-1} of this iteration, if continuous
      W.dl_vc[d] += (cont && sub(D.end, tnow) > W.slo_itl) ? 1u : 0u;
      const size_t ro = (size_t)d * (W.rmask + 1u) + (D.iters & W.rmask);
      W.re[ro] = D.end;
      W.rc[ro] = W.dl_vc[d];
    }
#if VT_EDEFER
    // the table loads are consumed at this iteration's END (off the in-order path of the START)
    D.e_u = D.nreq < SIM_UTAB && VT_UTAB ? __ldg(W.ut + SIM_UTAB + D.nreq)
                                          : div((double)D.nreq, add((double)D.nreq, W.uh_d));
    D.e_dyn = W.dyn[W.K + k];
    D.e_dur = dur;
#else
    ACC(ebusy) = add(ACC(ebusy), mul(bpow(W, 1, W.dyn[W.K + k], D.nreq), dur));  // W*ms, A23
#endif
    ACC(bms) = add(ACC(bms), dur);
    if (k == (int)W.K - 1) ACC(top) = add(ACC(top), dur);
    D.cur = D.iters;
    D.iters += 1u;
#if VT_SWHEEL
    D.bcur = L.sw[D.cur & (VT_SWHEEL - 1)];  // final now: read at the END of this iteration
#else
    D.bcur = wld(L.wheel + (D.cur & nbm));  // final now: read at the END of this iteration
#endif
#if VT_PF == 4
    // the completion list of this iteration was (most likely) known one START ago: pull its
    // head node towards L1 for the ITL walk at END; then peek at the next iteration's bucket
    if (D.nxh != 0u) prefetch_l1(L.node + (D.nxh - 1u));
    D.nxh = L.wheel[(D.cur + 1u) & nbm].x;
#endif
#if VT_PF == 3 || VT_PF == 4
    if (D.qh != NIL) prefetch_l1(L.wheel + ((D.iters + (uint32_t)queue_head(D, L).out - 2u) & nbm));
#endif
#if VT_BHPF
    if (D.qh != NIL) {
      D.bh_fin = D.iters + (uint32_t)queue_head(D, L).out - 2u;
      D.bh = wld(L.wheel + (D.bh_fin & nbm));
    } else {
      D.bh_fin = NIL;
    }
#endif
  }
}

// dec_advance for every lane of the warp (converged call site). VT_DEFER_ITL: a lane whose log
// chunk is full stops before its next END; the warp then hands out new chunks in lane order
// (one ballot, no atomics: shared-memory atomics inside the divergent advance cost 75 % of K4b)
// and those lanes continue.
template <int V, bool F, class WS>
__device__ __forceinline__ void dec_advance_all(Dec &D, int d, const Lane &L, WS &W, double t_lim, Err &E,
                                                const voltana_outputs &O) {
  dec_advance<V, F>(D, d, L, W, t_lim, E, O);
#if VT_DEFER_ITL
  if (!(V & 2)) {
    for (;;) {
      const unsigned nm = gballot(D.lneed);
      if (nm == 0u) break;
      const uint32_t top = W.clog_m;
      if (D.lneed) {
        D.lpos = top + CLOG_CHUNK * (uint32_t)__popc(nm & ((1u << glane()) - 1u));
        D.lend = D.lpos + CLOG_CHUNK;
        D.lneed = false;
        dec_advance<V, F>(D, d, L, W, t_lim, E, O);
      }
      __syncwarp(gmask());
      if (glane() == 0) W.clog_m = top + CLOG_CHUNK * (uint32_t)__popc(nm);
      __syncwarp(gmask());
    }
  }
#endif
}

// Append request i (routed at its first-token time) to instance d's admission queue.
__device__ __forceinline__ void dec_push(Dec &D, const Lane &L, uint32_t i, double tf, uint32_t in,
                                         uint32_t out, uint32_t nbm) {
  D.pn += 1u;
  D.pkv += in + 1u;
  L.node[i].next = NIL;
#if VT_PF == 5
  prefetch_l1(L.wheel + ((D.iters + out - 2u) & nbm));  // every pushed request's bucket at the next START
#endif
  if (D.qt == NIL) {
    D.qh = i;
#if VT_PF >= 2 && VT_PF != 5
    if (!VT_SWHEEL || out - 2u >= (uint32_t)VT_SWHEEL)
      prefetch_l1(L.wheel + ((D.iters + out - 2u) & nbm));  // its bucket at the next START
#endif
#if VT_QCACHE
    D.qhn.tf = tf; D.qhn.next = NIL; D.qhn.in = (uint16_t)in; D.qhn.out = (uint16_t)out;
#endif
  } else {
    L.node[D.qt].next = i;
#if VT_QCACHE
    if (D.qt == D.qh) D.qhn.next = i;  // keep the register copy coherent
#endif
  }
  D.qt = i;
}

// x mod nd for x < 2 nd (cursor arithmetic without an integer division)
__device__ __forceinline__ uint32_t wrap_nd(uint32_t x, uint32_t nd) { return x >= nd ? x - nd : x; }

// warp-wide min of a non-negative double held by lanes with `valid`; returns the lowest lane
// attaining it, or -1 if no lane is valid. Bit patterns of non-negative doubles order as u64.
__device__ __forceinline__ int argmin_time(double t, bool valid) {
  const uint64_t b = __double_as_longlong(t);
  const uint32_t hi = valid ? (uint32_t)(b >> 32) : 0xffffffffu;
  const uint32_t mhi = __reduce_min_sync(gmask(), hi);
  const bool c1 = valid && hi == mhi;
  const uint32_t lo = c1 ? (uint32_t)b : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(gmask(), lo);
  const unsigned m = gballot(c1 && lo == mlo);
  return m ? ffs0(m) : -1;
}

// Lanes holding the minimum of a signed double among lanes with `valid` (bitmask, group
// relative). -0 is folded into +0 first so the set equals the `==` set of the oracle.
__device__ __forceinline__ unsigned min_set(double v, bool valid) {
  if (v == 0.0) v = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint64_t key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // total order as unsigned
  const uint32_t hi = valid ? (uint32_t)(key >> 32) : 0xffffffffu;
  const uint32_t mhi = __reduce_min_sync(gmask(), hi);
  const bool c1 = valid && hi == mhi;
  const uint32_t lo = c1 ? (uint32_t)key : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(gmask(), lo);
  return gballot(c1 && lo == mlo);
}

__device__ __forceinline__ void write_status(const SimParams &P, uint32_t s, uint32_t n_req, uint32_t status) {
  if (glane() == 0) {
    voltana_result R = voltana_result{};
    R.status = status;
    R.n_requests = n_req;
    P.out[s] = R;
  }
}

// ------------------------------------------------------------------ phase A: prefill lane p
// K4a stream prefetch: each thread walks its own trace stream (32 independent streams per
// warp), so without prefetching almost every step waits on some lane's DRAM miss. Bulk L2
// prefetches run PA_PF_L2 entries ahead in PA_PF_CHUNK-entry chunks, L1 line prefetches
// PA_PF_L1 entries ahead.
#ifndef VT_PA_PF_L2
#define VT_PA_PF_L2 1024
#endif
#ifndef VT_PA_PF_L1
#define VT_PA_PF_L1 64
#endif
constexpr uint32_t PA_PF_CHUNK = 256;
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
// prefetch entries [from, from + cnt) of an array of `esz`-byte elements (16-B aligned bulk)
__device__ __forceinline__ void prefetch_l2_range(const void *base, uint32_t from, uint32_t cnt, uint32_t esz) {
  uintptr_t a = (uintptr_t)base + (uintptr_t)from * esz;
  uintptr_t e = a + (uintptr_t)cnt * esz;
  a &= ~(uintptr_t)15;
  e &= ~(uintptr_t)15;
  if (e > a) prefetch_l2_bulk((const void *)a, (uint32_t)(e - a));
}

template <int V, bool F, bool PFK, class WS>
__device__ void prefill_lane(const SimParams &P, WS &W, Node *node, const double *arr, const uint32_t *inl,
                             const uint32_t *outl, uint32_t N, uint32_t p, uint32_t NP, uint64_t h0, PaRes &R) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double ebusy = 0.0, bms = 0.0, top = 0.0, sttft = 0.0, tlast = 0.0, errt = INF;
  uint64_t h = h0;
  uint32_t iters = 0, ttft_ok = 0, itl_ok = 0, both = 0, errc = 0, head = NIL;
  const double tgt_ttft = W.tgt_ttft, slo_ttft = W.slo_ttft;
  const uint32_t B = W.B, K = W.K;
  double tfree = 0.0;
  double last = -INF;             // [C1] time of the last decision
  uint32_t cur = K - 1u, ndec = 0;  // [C2] running level (starts at the top), decisions
  uint32_t nxt = p, prev = NIL;
  Node pend;
  pend.tf = 0.0; pend.next = NIL; pend.in = 0; pend.out = 0;
  uint32_t pf1 = p, pf2 = p;  // PFK: next entry to prefetch into L1 / L2
  while (nxt < N) {
    if (PFK) {
      while (pf2 < N && pf2 < nxt + (uint32_t)VT_PA_PF_L2) {
        const uint32_t c = N - pf2 < PA_PF_CHUNK ? N - pf2 : PA_PF_CHUNK;
        prefetch_l2_range(arr, pf2, c, 8u);
        prefetch_l2_range(inl, pf2, c, 4u);
        prefetch_l2_range(outl, pf2, c, 4u);
        pf2 += PA_PF_CHUNK;
      }
      while (pf1 < N && pf1 < nxt + (uint32_t)VT_PA_PF_L1) {
        prefetch_l1(arr + pf1);
        prefetch_l1(inl + pf1);
        prefetch_l1(outl + pf1);
        pf1 += 16u;
      }
    }
#if VT_PFA
    if (nxt + VT_PFA < N) {  // the trace stream ahead of the batch being formed
      prefetch_l1(arr + nxt + VT_PFA);
      prefetch_l1(inl + nxt + VT_PFA);
      prefetch_l1(outl + nxt + VT_PFA);
    }
#endif
    const double a0 = arr[nxt];
    const double ts = tfree > a0 ? tfree : a0;  // START: instance idle and queue non-empty
    // FCFS prefix of the arrived queue with sum(in) <= B, at least one request (A6)
    uint32_t nbt = inl[nxt], cnt = 1, id = nxt + NP;
    bool backlog = false;  // (A5) requests still queued after the batch
    for (bool stop = false; !stop;) {  // 4 candidates per round, loads issued together
      double av[4];
      uint32_t xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = id + (uint32_t)u * NP;
        av[u] = j < N ? arr[j] : INF;  // past the trace end: "not arrived"
        xv[u] = j < N ? inl[j] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (stop) continue;
        if (!(av[u] <= ts)) stop = true;                                // not arrived yet
        else if (nbt + xv[u] > B) { backlog = true; stop = true; }      // does not fit
        else { nbt += xv[u]; cnt++; id += NP; }
      }
    }
    double budget = sub(tgt_ttft, sub(ts, a0));  // A4: SLO minus the oldest request's wait
    budget = budget > 0.0 ? budget : 0.0;
    double dur;
    int k;
    uint32_t fl = backlog ? 4u : 0u;
    if ((V & 2) && W.wo && !(sub(ts, last) >= W.ctrl_iv)) {  // window gating: keep the running level [C1]
      k = (int)cur;
      dur = ttft_at<F>(W, k, nbt);
    } else {
      fl |= 1u;
      if (backlog) { k = (int)K - 1; dur = ttft_at<F>(W, k, nbt); }
      else if ((V & 1) && W.ctrl) k = energy_ttft<F>(W, nbt, budget, &dur);  // B4
      else k = lowest_ttft<F>(W, nbt, budget, &dur);
      h = fold(h, 1, (uint64_t)p, (uint64_t)k, 0);
      if ((V & 2) && W.wo) { last = ts; ndec++; }
    }
    const uint32_t jit = iters++;
    if (!(dur > 0.0)) { errt = ts; errc = VOLTANA_ITEM_E_CONTRACT; break; }
    if ((V & 2) && W.noise) {  // true time = prediction x lognormal factor [D1]
      const double e = noise_at(W, p, jit);
      if (!(e > 0.0 && e <= 1e6)) { errt = ts; errc = VOLTANA_ITEM_E_INPUT; break; }
      dur = mul(dur, e);
    }
    double t0 = ts;
    if ((V & 2) && W.wo) {  // blocking frequency set on a level change [C3]
      if (k != (int)cur && W.fs_ov > 0.0) { t0 = add(ts, W.fs_ov); fl |= 2u; }
      cur = (uint32_t)k;
    }
    if ((V & 2)) log_iter(P.o, W, p, jit, ts, dur, nbt, 0u, k, fl);
    const double end = add(t0, dur);
    ebusy = add(ebusy, mul(bpow(W, 0, W.dyn[k], nbt), dur));  // W*ms (A23)
    bms = add(bms, dur);
    if (k == (int)K - 1) top = add(top, dur);
    // ---- O5 PrefillDone at `end`, batch in FCFS order
    for (uint32_t q = 0, i = nxt; q < cnt; ++q, i += NP) {
      const double ttft = sub(end, arr[i]);  // A26
      sttft = add(sttft, ttft);
      const bool ok = ttft <= slo_ttft;
      ttft_ok += ok;
      const uint32_t o = outl[i];
      if ((V & 2) && W.rq_on) {  // per-request record (E1)
        P.o.req_tfirst[W.rq_base + i] = end;
        if (o == 1u) {
          P.o.req_tdone[W.rq_base + i] = end; P.o.req_itl[W.rq_base + i] = 0.0;
          P.o.req_decode[W.rq_base + i] = 0xFF; P.o.req_case[W.rq_base + i] = 0xFF;
        }
      }
      if (o == 1u) {  // first token came from prefill: done (A8, A30)
        itl_ok++;
        both += ok;
        continue;
      }
      if (prev != NIL) { pend.next = i; node[prev] = pend; } else head = i;
      prev = i;
      pend.tf = ok ? end : -end;
      pend.next = NIL;
      pend.in = (uint16_t)inl[i];
      pend.out = (uint16_t)o;
    }
    tfree = end;
    tlast = end;
    nxt = id;
  }
  if (prev != NIL) { pend.next = NIL; node[prev] = pend; }
  R.ebusy = ebusy; R.bms = bms; R.top = top; R.sttft = sttft; R.tlast = tlast; R.errt = errt; R.h = h;
  R.iters = iters; R.ttft_ok = ttft_ok; R.itl_ok = itl_ok; R.both = both; R.errc = errc; R.ndec = ndec;
  R.head = head; R.pad = 0;
  if ((V & 2) && W.it_on) P.o.iter_count[W.it_base / P.o.iter_cap + p] = iters;
}

// ------------------------------------------------------------------ phase A, warp-cooperative (K4a)
// Prefill instance p of one scenario on a whole warp. The instance's decisions are a serial
// chain over batches (O7 START_PREFILL): everything on that chain is computed redundantly by
// all lanes, so control flow stays uniform. The lanes hold a window of the instance's next 32
// queued requests (arrival, in, out, and the inclusive prefix sum of in):
//  - batch formation at time ts from head lane h is one ballot: candidate j > h joins iff it
//    and every candidate before it has arrived by ts and the tokens from h through j fit in B;
//    the first failing lane ends the batch and says whether it is a backlog (A5, A6);
//  - the per-request TTFT accounting of O5 runs once per window for all its batches: each lane
//    holds its batch's end time, the report sum is added in FCFS order (A37), the counts are
//    ballots, and each routed request links to the next routed one.
// A batch longer than the window (> 32 requests) takes the general path (rounds of 32).

// K4a lane groups: G lanes per prefill instance (32 / G instances per warp); every collective
// is masked to the group, lane indices and window positions are group-relative.
template <int G> struct Grp {
  uint32_t gl, base;
  unsigned m;
  __device__ __forceinline__ Grp() {
    gl = threadIdx.x & (G - 1);
    base = (threadIdx.x & 31u) & ~(uint32_t)(G - 1);
    m = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << base);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const { return __ballot_sync(m, p) >> base; }
  template <class T> __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(m, v, src, G); }
  template <class T> __device__ __forceinline__ T shfl_up(T v, int d) const { return __shfl_up_sync(m, v, d, G); }
  static constexpr unsigned all = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
};

// Window element access: from the group's shared copy (PCtxS) or by shuffle (register context).
struct PCtxS;
struct PCtx;
template <int G> __device__ __forceinline__ void win_put(PCtx &, uint32_t, double, uint32_t) {}
template <int G> __device__ __forceinline__ double win_a(const PCtx &, const Grp<G> &g, double a, uint32_t i) {
  return g.shfl(a, (int)i);
}
template <int G> __device__ __forceinline__ uint32_t win_ps(const PCtx &, const Grp<G> &g, uint32_t ps, uint32_t i) {
  return g.shfl(ps, (int)i);
}
template <int G> __device__ __forceinline__ void win_tput(PCtx &, uint32_t, double) {}
template <int G> __device__ __forceinline__ double win_t(const PCtx &, const Grp<G> &g, double t, uint32_t i) {
  return g.shfl(t, (int)i);
}

struct PState {   // uniform state of one prefill instance (every lane holds the same values)
  double ebusy, bms, top, sttft, tlast, errt, tfree, last;
  uint64_t h;
  uint32_t iters, ttft_ok, itl_ok, both, errc, head, cur, ndec, prev;
  Node pend;      // node of request `prev` (last routed so far), written when its successor is known
};

// O7 decision for a batch of nbt tokens starting at ts, head arrival a0: EcoFreq,
// duration, energy (A23). false: per-item error recorded in S.
template <int V, bool F, int G, class WS>
__device__ __forceinline__ bool pa_decide(const SimParams &P, const WS &W, PState &S, uint32_t p, double ts,
                                          double a0, uint32_t nbt, bool backlog, double &end) {
  double budget = sub(W.tgt_ttft, sub(ts, a0));  // A4: SLO minus the oldest request's wait
  budget = budget > 0.0 ? budget : 0.0;
  const uint32_t K = W.K;
  double dur;
  int k;
  uint32_t fl = backlog ? 4u : 0u;
  if ((V & 2) && W.wo && !(sub(ts, S.last) >= W.ctrl_iv)) {  // window gating: keep the running level [C1]
    k = (int)S.cur;
    dur = ttft_at<F>(W, k, nbt);
  } else {
    fl |= 1u;
    if (backlog) { k = (int)K - 1; dur = ttft_at<F>(W, k, nbt); }
    else if ((V & 1) && W.ctrl) k = energy_ttft<F>(W, nbt, budget, &dur);  // B4
    else k = lowest_ttft<F>(W, nbt, budget, &dur);
    S.h = fold(S.h, 1, (uint64_t)p, (uint64_t)k, 0);
    if ((V & 2) && W.wo) { S.last = ts; S.ndec++; }
  }
  const uint32_t jit = S.iters++;
  if (!(dur > 0.0)) { S.errt = ts; S.errc = VOLTANA_ITEM_E_CONTRACT; return false; }
  if ((V & 2) && W.noise) {  // true time = prediction x lognormal factor [D1]
    const double e = noise_at(W, p, jit);
    if (!(e > 0.0 && e <= 1e6)) { S.errt = ts; S.errc = VOLTANA_ITEM_E_INPUT; return false; }
    dur = mul(dur, e);
  }
  double t0 = ts;
  if ((V & 2) && W.wo) {  // blocking frequency set on a level change [C3]
    if (k != (int)S.cur && W.fs_ov > 0.0) { t0 = add(ts, W.fs_ov); fl |= 2u; }
    S.cur = (uint32_t)k;
  }
  if ((V & 2) && (threadIdx.x & (G - 1)) == 0) log_iter(P.o, W, p, jit, ts, dur, nbt, 0u, k, fl);
  end = add(t0, dur);
  S.ebusy = add(S.ebusy, mul(bpow(W, 0, W.dyn[k], nbt), dur));  // W*ms (A23)
  S.bms = add(S.bms, dur);
  if (k == (int)K - 1) S.top = add(S.top, dur);
  S.tfree = end;
  S.tlast = end;
  return true;
}

// O5 for lanes [0, n): request base + lane*NP (arrival a, in x, out o) finished prefill at e.
template <int V, int G, class WS>
__device__ __forceinline__ void pa_account(const SimParams &P, WS &W, PState &S, Node *node, uint32_t base,
                                           uint32_t NP, uint32_t n, double e, double a, uint32_t x, uint32_t o) {
  if (n == 0u) return;
  const Grp<G> g;
  const uint32_t lane = g.gl;
  const bool valid = lane < n;
  const uint32_t i = base + lane * NP;
  const double ttft = valid ? sub(e, a) : 0.0;  // A26
  const bool ok = valid && ttft <= W.slo_ttft;
  __syncwarp(g.m);
  win_tput<G>(W, lane, ttft);
  __syncwarp(g.m);
  for (uint32_t b = 0; b < n; b += 8u) {  // the report sum in FCFS order (A37)
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = win_t<G>(W, g, ttft, (b + u) & (G - 1));
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b + u < n) S.sttft = add(S.sttft, v[u]);
  }
  S.ttft_ok += __popc(g.ballot(ok));
  const bool one = valid && o == 1u;  // first token came from prefill: done (A8, A30)
  S.itl_ok += __popc(g.ballot(one));
  S.both += __popc(g.ballot(one && ok));
  if ((V & 2) && W.rq_on && valid) {  // per-request record (E1)
    P.o.req_tfirst[W.rq_base + i] = e;
    if (o == 1u) {
      P.o.req_tdone[W.rq_base + i] = e; P.o.req_itl[W.rq_base + i] = 0.0;
      P.o.req_decode[W.rq_base + i] = 0xFF; P.o.req_case[W.rq_base + i] = 0xFF;
    }
  }
  const unsigned rm = g.ballot(valid && o != 1u);  // routed requests, FCFS = lane order
  if (rm == 0u) return;
  const int f0 = ffs0(rm), ll = 31 - __clz(rm);
  const uint32_t i_first = base + (uint32_t)f0 * NP;
  if (S.prev != NIL) {
    if (lane == 0) { S.pend.next = i_first; node[S.prev] = S.pend; }
  } else {
    S.head = i_first;
  }
  Node me;
  me.tf = ok ? e : -e;
  me.in = (uint16_t)x;
  me.out = (uint16_t)o;
  if (((rm >> lane) & 1u) && (int)lane != ll) {  // the next routed request is in this set
    const unsigned above = rm & ~((2u << lane) - 1u);
    me.next = base + (uint32_t)ffs0(above) * NP;
    node[i] = me;
  }
  S.prev = base + (uint32_t)ll * NP;  // the last routed request: pending until its successor
  S.pend.tf = g.shfl(me.tf, ll);
  S.pend.in = (uint16_t)g.shfl((uint32_t)me.in, ll);
  S.pend.out = (uint16_t)g.shfl((uint32_t)me.out, ll);
  S.pend.next = NIL;
}

// General path for one batch starting at request nxt (any length): candidates in rounds of 32,
// accounting in chunks of 32. Returns the next unbatched request, or NIL on an error.
template <int V, bool F, int G, class WS>
__device__ uint32_t pa_batch_general(const SimParams &P, WS &W, PState &S, Node *node, const double *arr,
                                     const uint32_t *inl, const uint32_t *outl, uint32_t N, uint32_t p,
                                     uint32_t NP, uint32_t nxt) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const Grp<G> g;
  const uint32_t lane = g.gl, B = W.B;
  const double a0 = arr[nxt];
  const double ts = S.tfree > a0 ? S.tfree : a0;
  uint32_t nbt = inl[nxt], cnt = 1, id = nxt + NP;
  bool backlog = false;
  for (;;) {
    const uint32_t j = id + lane * NP;
    const bool in_tr = j < N && j >= id;
    const double av = in_tr ? arr[j] : INF;  // past the trace end: "not arrived"
    const uint32_t xv = in_tr ? inl[j] : 0u;
    uint32_t ps = xv;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const uint32_t y = g.shfl_up(ps, o);
      if (lane >= (uint32_t)o) ps += y;
    }
    const bool arrived = av <= ts;
    const unsigned m = g.ballot(arrived && !(nbt + ps > B));
    const uint32_t f = m == Grp<G>::all ? (uint32_t)G : (uint32_t)ffs0(~m);
    if (f > 0u) {
      nbt += g.shfl(ps, (int)f - 1);
      cnt += f;
      id += f * NP;
    }
    if (f < (uint32_t)G) {
      backlog = g.shfl(arrived, (int)f);
      break;
    }
  }
  double end;
  if (!pa_decide<V, F, G>(P, W, S, p, ts, a0, nbt, backlog, end)) return NIL;
  for (uint32_t q0 = 0; q0 < cnt; q0 += (uint32_t)G) {
    const uint32_t nv = cnt - q0 < (uint32_t)G ? cnt - q0 : (uint32_t)G;
    const uint32_t i = nxt + (q0 + lane) * NP;
    double a = 0.0;
    uint32_t x = 0u, o = 0u;
    if (lane < nv) { a = arr[i]; x = inl[i]; o = outl[i]; }
    pa_account<V, G>(P, W, S, node, nxt + q0 * NP, NP, nv, end, a, x, o);
  }
  return id;
}

template <int V, bool F, int G, class WS>
__device__ void prefill_warp(const SimParams &P, WS &W, Node *node, const double *arr, const uint32_t *inl,
                             const uint32_t *outl, uint32_t N, uint32_t p, uint32_t NP, uint64_t h0, PaRes &R) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const Grp<G> g;
  const uint32_t lane = g.gl, B = W.B;
  PState S;
  S.ebusy = S.bms = S.top = S.sttft = S.tlast = S.tfree = 0.0;
  S.errt = INF;
  S.last = -INF;             // [C1] time of the last decision
  S.h = h0;
  S.iters = S.ttft_ok = S.itl_ok = S.both = S.errc = S.ndec = 0;
  S.cur = W.K - 1u;          // [C2] running level (starts at the top)
  S.head = S.prev = NIL;
  S.pend.tf = 0.0; S.pend.next = NIL; S.pend.in = 0; S.pend.out = 0;
  uint32_t wbase = p;        // request of lane 0 in the window (the instance's next unbatched request)
  uint32_t pf2 = p;          // next entry to prefetch into L2
  while (wbase < N) {
    if (lane == 0)
      while (pf2 < N && pf2 < wbase + (uint32_t)VT_PA_PF_L2) {
        const uint32_t c = N - pf2 < PA_PF_CHUNK ? N - pf2 : PA_PF_CHUNK;
        prefetch_l2_range(arr, pf2, c, 8u);
        prefetch_l2_range(inl, pf2, c, 4u);
        prefetch_l2_range(outl, pf2, c, 4u);
        pf2 += PA_PF_CHUNK;
      }
    const uint32_t rem = (N - wbase + NP - 1u) / NP;  // requests left on this instance
    const uint32_t nwin = rem < (uint32_t)G ? rem : (uint32_t)G;
    const uint32_t idx = wbase + lane * NP;
    const bool v = lane < nwin;
    const double a = v ? arr[idx] : INF;  // past the trace end: "not arrived"
    const uint32_t x = v ? inl[idx] : 0u;
    const uint32_t o = v ? outl[idx] : 0u;
    uint32_t ps = x;
#pragma unroll
    for (int s = 1; s < G; s <<= 1) {
      const uint32_t y = g.shfl_up(ps, s);
      if (lane >= (uint32_t)s) ps += y;
    }
    __syncwarp(g.m);           // the previous window's reads are done
    win_put<G>(W, lane, a, ps);
    __syncwarp(g.m);
    double e = 0.0;            // this lane's batch end, once its batch has started
    uint32_t hl = 0;           // head lane of the next batch
    bool err = false, general = false;
    while (hl < nwin) {
      const double a0 = win_a<G>(W, g, a, hl);
      const double ts = S.tfree > a0 ? S.tfree : a0;  // START: instance idle and queue non-empty
      const uint32_t psb = hl ? win_ps<G>(W, g, ps, hl - 1u) : 0u;  // tokens before the head
      const bool arrived = a <= ts;
      const bool take = lane > hl && arrived && !(ps - psb > B);
      const unsigned fails = g.ballot(lane > hl && !take);
      if (fails == 0u) {       // a full window of arrivals that all fit: the batch may run on
        general = hl == 0u;    // more than 32 requests: the general path; else re-window at the head
        break;
      }
      const uint32_t f = (uint32_t)ffs0(fails);  // first candidate not taken
      const bool backlog = win_a<G>(W, g, a, f) <= ts;  // arrived but does not fit (A5)
      const uint32_t nbt = win_ps<G>(W, g, ps, f - 1u) - psb;
      double end;
      if (!pa_decide<V, F, G>(P, W, S, p, ts, a0, nbt, backlog, end)) { err = true; break; }
      if (lane >= hl && lane < f) e = end;
      hl = f;
    }
    pa_account<V, G>(P, W, S, node, wbase, NP, hl, e, a, x, o);  // O5 for the window's batches
    wbase += hl * NP;
    if (err) break;
    if (general) {
      wbase = pa_batch_general<V, F, G>(P, W, S, node, arr, inl, outl, N, p, NP, wbase);
      if (wbase == NIL) break;
    }
  }
  if (S.prev != NIL && lane == 0) { S.pend.next = NIL; node[S.prev] = S.pend; }
  R.ebusy = S.ebusy; R.bms = S.bms; R.top = S.top; R.sttft = S.sttft; R.tlast = S.tlast; R.errt = S.errt;
  R.h = S.h; R.iters = S.iters; R.ttft_ok = S.ttft_ok; R.itl_ok = S.itl_ok; R.both = S.both; R.errc = S.errc;
  R.ndec = S.ndec; R.head = S.head; R.pad = 0;
  if ((V & 2) && W.it_on && lane == 0) P.o.iter_count[W.it_base / P.o.iter_cap + p] = S.iters;
}

// ------------------------------------------------------------------ deferred ITL accounting (K4c)
__device__ __forceinline__ double itl_marker(uint32_t slot) {  // "list continues": NaN with the slot
  return __longlong_as_double((long long)(0xFFF8000000000000ull | slot));
}
// The ITL accounting of one scenario's completion log E[0, m) on the calling warp (all 32
// lanes): c_ok / c_both summed over the warp, sitl = the decode instances' sums in instance
// order, each the sequential sum in completion order (A30, A37).
template <int U>
__device__ void itl_scenario(const SimParams &P, uint32_t m, int ND, double slo, const CEnt *E, const Node *node,
                             ItlScratch<U> &S, uint32_t &c_ok_out, uint32_t &c_both_out, double &sitl_out) {
  constexpr uint32_t RN = 32u * U;  // entries per round
  const uint32_t lane = threadIdx.x & 31u;
  double sd = 0.0;                // lane d: instance d's running sum
  uint32_t c_ok = 0, c_both = 0;  // this lane's counts
  for (uint32_t c0 = 0; c0 < m; c0 += RN) {
    double td[U];
    uint32_t id[U], cnt[U], dd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = c0 + (uint32_t)u * 32u + lane;
      CEnt e;
      e.td = 0.0; e.head = NIL; e.d = 0u;
      if (q < m) e = E[q];
      td[u] = e.td; id[u] = e.head; dd[u] = e.d; cnt[u] = 0u;
    }
#pragma unroll
    for (uint32_t jj = 0; jj < ITL_CAP; ++jj) {  // step jj of every walk: U independent loads in flight
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (id[u] != NIL) {
          const Node nd = node[id[u]];
          const double x = div(sub(td[u], fabs(nd.tf)), (double)(nd.out - 1u));
          const bool ok = x <= slo;
          c_ok += ok;
          c_both += ok && nd.tf > 0.0;
          S.v[u * 32 + lane][jj] = x;
          cnt[u]++;
          id[u] = nd.next;
        }
      }
    }
    // regroup: the values of instance d, in log order, go to seq[base_d ...] (exclusive scans)
    uint32_t pos[U], tot[NI];
#pragma unroll
    for (int d = 0; d < NI; ++d) tot[d] = 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t cp = cnt[u] + (id[u] != NIL ? 1u : 0u);  // values + a continuation marker
      pos[u] = 0u;
#pragma unroll
      for (int d = 0; d < NI; ++d) {
        if (d >= ND) break;
        const uint32_t c = dd[u] == (uint32_t)d ? cp : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (dd[u] == (uint32_t)d) pos[u] = tot[d] + incl - c;
        tot[d] += __shfl_sync(FULL, incl, 31);
      }
    }
    uint32_t base = 0u, my_base = 0u, my_tot = 0u;  // lane d: its sequence [my_base, my_base + my_tot)
#pragma unroll
    for (int d = 0; d < NI; ++d) {
      if (d >= ND) break;
      if (lane == (uint32_t)d) { my_base = base; my_tot = tot[d]; }
      base += tot[d];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t b = 0u;
#pragma unroll
      for (int d = 0; d < NI; ++d) {
        if (d >= ND) break;
        const uint32_t bd = __shfl_sync(FULL, my_base, d);
        if (dd[u] == (uint32_t)d) b = bd;
      }
      double *o = &S.seq[b + pos[u]];
      for (uint32_t jj = 0; jj < cnt[u]; ++jj) o[jj] = S.v[u * 32 + lane][jj];
      if (id[u] != NIL) {
        o[cnt[u]] = itl_marker((uint32_t)u * 32u + lane);
        S.td[u * 32 + lane] = td[u];
        S.id[u * 32 + lane] = id[u];
      }
    }
    __syncwarp();
    if (lane < (uint32_t)ND) {  // instance `lane` adds its values in log order (A37)
      for (uint32_t q = 0; q < my_tot; ++q) {
        const double v = S.seq[my_base + q];
        if (v == v) {
          sd = add(sd, v);
        } else {  // a list longer than ITL_CAP: its rest, in order
          const uint32_t slot = (uint32_t)(__double_as_longlong(v) & 0xFFFFu);
          const double t = S.td[slot];
          uint32_t r = S.id[slot];
          for (uint32_t hop = 0; r != NIL && hop < P.max_requests; ++hop) {
            const Node nd = node[r];
            const double itl = div(sub(t, fabs(nd.tf)), (double)(nd.out - 1u));
            sd = add(sd, itl);
            const bool ok = itl <= slo;
            c_ok += ok;
            c_both += ok && nd.tf > 0.0;
            r = nd.next;
          }
        }
      }
    }
    __syncwarp();
  }
  c_ok_out = __reduce_add_sync(FULL, c_ok);
  c_both_out = __reduce_add_sync(FULL, c_both);
  double sitl = 0.0;  // decode instances in instance order (A37)
  for (int d = 0; d < ND; ++d) sitl = add(sitl, __shfl_sync(FULL, sd, d));
  sitl_out = sitl;
}

template <int V, bool F, class WS>
__device__ void run_scenario(const SimParams &P, uint32_t s, char *slot, uint4 *wheels, WS &W, uint32_t sid) {
  const int lane = glane();
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  // ---------------------------------------------------------------- ids and table rows
  if (!(P.trace_id[s] < P.n_traces && P.slo_id[s] < P.n_slos && P.layout_id[s] < P.n_layouts &&
        P.grid_id[s] < P.n_grids && P.profile_id[s] < P.n_profiles)) {
    write_status(P, s, 0, VOLTANA_ITEM_E_INPUT);
    return;
  }
  const uint32_t tr = P.trace_id[s];
  const voltana_slo &SL = P.slo[P.slo_id[s]];
  const voltana_layout &LY = P.lay[P.layout_id[s]];
  const voltana_grid &GR = P.grid[P.grid_id[s]];
  const DevProfile &PR = P.prof[P.profile_id[s]];
  const uint64_t off = P.offset[tr];
  const uint64_t N64 = P.offset[tr + 1] - off;
  const double Dur = P.duration[tr];
  const double *arr = P.arrival + off;
  const uint32_t *inl = P.in_len + off;
  const uint32_t *outl = P.out_len + off;

  // ---------------------------------------------------------------- device validation (A40)
  uint32_t tok_total;
  {
    bool ok = N64 <= P.max_requests && Dur >= 0.0;
    uint64_t tok = 0;
    if (ok) {
      for (uint64_t i = lane; i < N64; i += GS) {
        const uint32_t a = inl[i], b = outl[i];
        const double x = arr[i];
        ok = ok && a >= 1u && a <= 65535u && b >= 1u && b <= P.max_out && x >= 0.0 && x < 1e9;
        if (i > 0) ok = ok && !(x < arr[i - 1]);
        tok += (uint64_t)a + b;
      }
    }
    for (int o = GS / 2; o > 0; o >>= 1) tok += __shfl_xor_sync(gmask(), tok, o, GS);
    ok = __all_sync(gmask(), ok) && tok <= 0x7fffffffull;
    if (!ok) {
      write_status(P, s, (uint32_t)N64, VOLTANA_ITEM_E_INPUT);
      return;
    }
    tok_total = (uint32_t)tok + 2u;
  }
  const uint32_t N = (uint32_t)N64;
  const int NP = LY.n_p, ND = LY.n_d;
  uint64_t rq_base = 0, it_base = 0;
  bool rq_on = false;
  if ((V & 2) && P.o.req_offset) {  // per-request range: empty (skip) or exactly the trace (E1)
    rq_base = P.o.req_offset[s];
    const uint64_t len = P.o.req_offset[s + 1] - rq_base;
    if (len != 0 && len != N64) {
      write_status(P, s, N, VOLTANA_ITEM_E_INPUT);
      return;
    }
    rq_on = len != 0;
  }
  if ((V & 2) && P.o.iter_offset) it_base = P.o.iter_offset[s];

  // ---------------------------------------------------------------- stage constants and tables
  const uint32_t K = (uint32_t)GR.k, T = (uint32_t)PR.n_tiles;
  if (lane == 0) {
    W.tau = LY.kv_transfer_ms; W.slo_itl = SL.itl_ms; W.slo_ttft = SL.ttft_ms;
    W.tgt_itl = mul(SL.scale, SL.itl_ms);   // A3
    W.tgt_ttft = mul(SL.scale, SL.ttft_ms);
    W.p_idle = PR.p_idle; W.tdp = PR.tdp; W.uh_p = PR.uh[0]; W.uh_d = PR.uh[1];
    W.a2g = PR.a2; W.b2g = PR.b2; W.c2g = PR.c2;
    W.a1g = PR.a1; W.c1g = PR.c1; W.ptiles = (uint32_t)PR.n_ptiles; W.pcut = PR.pcut;
    W.ut = VT_UTAB ? P.utab + (size_t)P.profile_id[s] * 2 * SIM_UTAB : nullptr;
    W.kvcap = LY.kv_capacity; W.max_steps = tok_total; W.B = LY.max_batch_tokens;
    W.K = K; W.T = T; W.W = (uint32_t)PR.tile_w; W.kp = (uint32_t)PR.k; W.nb = P.nb;
    W.wshift = (PR.tile_w & (PR.tile_w - 1)) == 0 ? __ffs(PR.tile_w) - 1 : -1;
    W.itl_smem = P.itl_smem;
    W.ctrl = (uint32_t)LY.ctrl_mode;
    W.ctrl_iv = LY.ctrl_interval_ms;
    W.fs_ov = LY.freq_overhead_ms;
    W.noise = LY.exec_noise;
    W.noise_mask = LY.noise_len - 1u;
    W.seed = P.hash_seed[s];
    W.np = (uint32_t)NP;
    W.itlm = (V & 2) ? (uint32_t)LY.itl_mode : 0u;
    W.wo = (V & 2) && (LY.ctrl_interval_ms > 0.0 || LY.freq_overhead_ms > 0.0) ? 1u : 0u;
    W.rmask = P.ring_r - 1u;
    W.re = P.ring_e ? P.ring_e + (size_t)sid * P.ring_nd * P.ring_r : nullptr;
    W.rc = P.ring_c ? P.ring_c + (size_t)sid * P.ring_nd * P.ring_r : nullptr;
    W.rq_on = rq_on; W.rq_base = rq_base;
    W.it_on = (V & 2) && P.o.iter_offset != nullptr; W.it_base = it_base;
  }
  if ((V & 2) && lane < NI) {
    W.dl_vc[lane] = 0u;
    W.dl_last[lane] = -INF;
    W.dl_cur[lane] = (uint32_t)GR.k - 1u;  // the GPU starts at the top of the ladder [C2]
    W.dl_ndec[lane] = 0u;
  }
  for (uint32_t k = lane; k < K; k += GS) {
    const int lv = GR.level[k];
    W.lad[k] = (uint16_t)lv;
    W.tt[2 * k] = PR.a1[lv];
    W.tt[2 * k + 1] = PR.c1[lv];
    W.dyn[k] = PR.dyn[lv];
    W.dyn[K + k] = PR.dyn[PR.k + lv];
    W.mhz[k] = PR.mhz[lv];
  }
  if (P.itl_smem) {
    for (uint32_t x = lane; x < T * K; x += GS) {
      const uint32_t j = x / K, k = x - j * K;
      const size_t o = (size_t)j * PR.k + GR.level[k];
      W.it[3 * x] = PR.a2[o]; W.it[3 * x + 1] = PR.b2[o]; W.it[3 * x + 2] = PR.c2[o];
    }
  }
  {  // coefficient-monotone (non-increasing in f) tables allow the exact binary search (A32)
    bool mt = true, mi = true;
    for (uint32_t k = lane; k + 1 < K; k += GS)
      mt = mt && PR.a1[GR.level[k + 1]] <= PR.a1[GR.level[k]] && PR.c1[GR.level[k + 1]] <= PR.c1[GR.level[k]];
    for (uint32_t x = lane; x < T * (K - 1); x += GS) {
      const uint32_t j = x / (K - 1), k = x - j * (K - 1);
      const size_t o0 = (size_t)j * PR.k + GR.level[k], o1 = (size_t)j * PR.k + GR.level[k + 1];
      mi = mi && PR.a2[o1] <= PR.a2[o0] && PR.b2[o1] <= PR.b2[o0] && PR.c2[o1] <= PR.c2[o0];
    }
    mt = __all_sync(gmask(), mt) && PR.n_ptiles <= 1;  // tiled TTFT: the ascending scan (F1)
    mi = __all_sync(gmask(), mi);
    if (lane == 0) { W.mono_tt = mt; W.mono_it = mi; }
  }
  __syncwarp(gmask());
#if VT_SPLIT_A
  Node *node = (Node *)(P.nodes + (size_t)s * P.max_requests * sizeof(Node));
#else
  Node *node = (Node *)slot;
#endif
  const uint64_t h0 = P.hash_seed[s];

  // ================================================================ PHASE A: prefill lanes
#if VT_SPLIT_A
  // computed by K4a (prefill_kernel) before this launch: read back lane p's result
  if (lane < NP) W.pa[lane] = P.pares[(size_t)s * NI + lane];
#else
  if (lane < NP) prefill_lane<V, F, false>(P, W, node, arr, inl, outl, N, (uint32_t)lane, (uint32_t)NP, h0, W.pa[lane]);
#endif
  __syncwarp(gmask());
  const uint32_t p_head = lane < NP ? W.pa[lane].head : NIL;
#ifdef VT_PHASE_TIMING
  if (P.timing && glane() == 0) {  // experiment: phase-A end time replaces the start stamp
    uint64_t ta;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
    P.timing[2 * s] = ta;
  }
#endif

  // ================================================================ PHASE B: routing + decode lanes
  const int dl = lane < ND ? lane : 0;
  Lane L;
#if VT_SWHEEL
  L.sw = (uint4 *)((char *)&W + P.sw_off) + (size_t)dl * VT_SWHEEL;
  if (lane < ND)
    for (uint32_t b = 0; b < (uint32_t)VT_SWHEEL; ++b) L.sw[b] = make_uint4(0u, 0u, 0u, 0u);
#endif
  L.node = node;
  L.farfin = (uint32_t *)(slot + P.node_bytes);
  L.wheel = wheels + (size_t)dl * P.nb;
  L.fid = W.fid[dl];
  L.ft = W.ft[dl];
#if VT_DEFER_ITL
  L.clog = P.clog + (size_t)s * P.clog_stride;
  if (lane == 0) W.clog_m = (uint32_t)ND * CLOG_CHUNK;  // the first chunk of every decode lane
  __syncwarp(gmask());
#endif
  Dec D;
  D.nreq = D.nkv = D.pn = D.pkv = D.iters = D.cur = 0;
  D.qh = D.qt = NIL;
  D.nfifo = 0;
  D.far_h = D.far_hfin = NIL;
  D.busy = false;
  D.dead = !(lane < ND);
  D.end = 0.0;
#if VT_ADM_DEFER
  D.npq = 0u;
#endif
#if VT_DEFER_ITL
  D.lpos = (uint32_t)lane * CLOG_CHUNK;  // first chunks: one per lane, allocated in lane order
  D.lend = D.lpos + CLOG_CHUNK;
  D.lneed = false;
#endif
#if VT_EDEFER
  D.e_u = D.e_dyn = D.e_dur = 0.0;
#endif
  {
    const int d = lane < ND ? lane : 0;
    if (lane < ND || !VT_DACC_SMEM) {
      ACC(ebusy) = 0.0; ACC(bms) = 0.0; ACC(top) = 0.0; ACC(sitl) = 0.0; ACC(tlast) = 0.0;
      ACC(h) = h0; ACC(n_itl_ok) = 0; ACC(n_both) = 0;
    }
  }
  D.bcur = make_uint4(0u, 0u, 0u, 0u);
#if VT_PF == 4
  D.nxh = 0u;
#endif
#if VT_QCACHE
  D.qhn.tf = 0.0; D.qhn.next = NIL; D.qhn.in = 0; D.qhn.out = 0;
#endif
#if VT_BHPF
  D.bh_fin = NIL;
  D.bh = D.bcur;
#endif
  Err dE = {INF, 0};

  // stream head of prefill lane p (head node hn and, loaded one step ahead, its successor nn)
  uint32_t hd = lane < NP ? p_head : NIL;
#if VT_SPLIT_A && VT_NODE_PF_L2
  uint32_t npf = 0;  // nodes [0, npf) of the scenario already prefetched into L2 (shared by the streams)
  if (lane < NP)
    for (; npf < (uint32_t)VT_NODE_PF_L2 && npf < N; npf += 256u)
      prefetch_l2_range(node, npf, N - npf < 256u ? N - npf : 256u, 16u);
#endif
  Node hn, nn;
  hn.tf = 0.0; hn.next = NIL; hn.in = 0; hn.out = 0;
  nn = hn;
  if (hd != NIL) {
    hn = node[hd];
    if (hn.next != NIL) nn = node[hn.next];
  }
  uint64_t h_r = h0;
  uint32_t cursor = 0, steps_route = 0;
  double t_adv = -1.0;                              // decode lanes are caught up to events < t_adv
  uint32_t c_n = NIL, c_kv = 0;                     // what-if cache: EcoFreq level of the lane's
  int c_lvl = 0;                                    // effective state (c_n, c_kv)
  int ka_last = 0;
  double c_en = 0.0, en_new = 0.0;                  // energy router: P*T of the cached state / successor
  const bool eco = LY.policy == 0 && ND > 1;
  const bool ens = (V & 1) && LY.policy == 2 && ND > 1;
  const int32_t delta = LY.delta_mhz;
  int w = argmin_time(fabs(hn.tf), hd != NIL);  // next PrefillDone request in (t, p, id) order
#ifdef VT_LAT_PROBE
  // experiment: clock64 cycles per phase of the route loop, summed over the scenario
  // [0] select + stream advance, [1] decode advance, [2] EcoRoute + push, [3] drain + ITL pass
  long long lp_acc[4] = {0, 0, 0, 0}, lp_t = clock64();
#define LP_MARK(q) do { const long long _n = clock64(); lp_acc[q] += _n - lp_t; lp_t = _n; } while (0)
#else
#define LP_MARK(q) do { } while (0)
#endif
  for (;;) {
    if (w < 0) break;
    if (steps_route > N) { dE.t = 0.0; dE.code = VOLTANA_ITEM_E_INTERNAL; break; }  // watchdog
    const double t = gshfl(fabs(hn.tf), w);
    const uint32_t i = gshfl(hd, w);
    const uint32_t io = gshfl((uint32_t)hn.in | ((uint32_t)hn.out << 16), w);
    const double tf_i = gshfl(hn.tf, w);  // signed: carries the TTFT verdict
    const uint32_t in_i = io & 0xffffu;
    if (lane == w) {                                  // advance that stream; prefetch one further
      hd = hn.next;
      hn = nn;
      if (hd != NIL && hn.next != NIL) {
        nn = node[hn.next];
#if VT_PF >= 1
        prefetch_l1(node + hn.next + (uint32_t)VT_NODE_PF_L1);  // the stream's next line (ids advance by N_P)
#endif
      }
#if VT_SPLIT_A && VT_NODE_PF_L2
      // K4a wrote the node array long before (DRAM): keep the stream's next nodes coming into L2
      if (hd != NIL && hd + (uint32_t)VT_NODE_PF_L2 > npf && npf < N) {
        prefetch_l2_range(node, npf, N - npf < 256u ? N - npf : 256u, 16u);
        npf += 256u;
      }
#endif
    }
#if VT_PIPE_ARGMIN
    // the next request depends only on the stream heads: its selection overlaps this route
    const int w_next = argmin_time(fabs(hn.tf), hd != NIL);
#endif
    // decode instances catch up to t: events strictly before t (PrefillDone drains first)
    LP_MARK(0);
    if (t != t_adv) {  // routes of one batch share t: nothing new happens between them
      dec_advance_all<V, F>(D, lane, L, W, t, dE, P.o);
      t_adv = t;
    }
    LP_MARK(1);
    // ---- O8 EcoRoute
    int dsel, cse;
    if (ens) {  // ---- energy-scored router [B1-B3]
      const bool act = lane < ND;
      bool feas = false;
      double score = 0.0, tmax = 0.0;
      if (act) {
        const uint32_t n = D.nreq + D.pn, kv = D.nkv + D.pkv;  // A9 effective state
        double enow = 0.0;
        if (n != 0u) {
          if (n != c_n || kv != c_kv) {
            double pr;
            const int k0 = lowest_itl<F>(W, n, kv, W.tgt_itl, &pr);  // EcoFreq level now (A10/A11)
            c_en = mul(bpow(W, 1, W.dyn[W.K + k0], n), pr);
            c_n = n; c_kv = kv;
          }
          enow = c_en;
        }
        const uint32_t n1 = n + 1u, kv1 = kv + in_i + 1u;  // A12
        const uint32_t j = tile_j<F>(W, n1);
        const double dn = (double)n1, dkv = (double)kv1;
        double best = 0.0, t = 0.0;
        for (int k = 0; k < (int)W.K; ++k) {
          t = itl_at<F>(W, j, k, dn, dkv);
          if (!(t <= W.tgt_itl)) continue;
          const double e = mul(bpow(W, 1, W.dyn[W.K + k], n1), t);
          if (!feas) en_new = e;                    // the successor's own EcoFreq-level P*T
          if (!feas || e < best) best = e;
          feas = true;
        }
        tmax = t;                                   // T at K-1
        if (!feas) en_new = mul(bpow(W, 1, W.dyn[W.K + W.K - 1], n1), tmax);
        score = sub(best, enow);
      }
      const bool any = gballot(feas) != 0u;
      const unsigned inset = any ? min_set(score, feas) : min_set(tmax, act);
      cse = any ? 6 : 7;
      const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & ((1u << ND) - 1u);
      dsel = (int)wrap_nd(cursor + (uint32_t)ffs0(rot), (uint32_t)ND);
      if (__popc(inset) >= 2) cursor = wrap_nd((uint32_t)dsel + 1u, (uint32_t)ND);
    } else if (!eco) {
      dsel = (int)cursor;
      cursor = wrap_nd(cursor + 1u, (uint32_t)ND);
      cse = 0;
    } else {
      int fnow = 0x7fffffff, faft = 0x7fffffff;
      if (lane < ND) {
        const uint32_t n = D.nreq + D.pn, kv = D.nkv + D.pkv;  // A9 effective state
        double pr;
        int kn = 0;                                                            // A10, A11
        if (n != 0u) {
          if (n != c_n || kv != c_kv) { c_lvl = lowest_itl<F>(W, n, kv, W.tgt_itl, &pr); c_n = n; c_kv = kv; }
          kn = c_lvl;
        }
        const int ka = lowest_itl<F>(W, n + 1u, kv + in_i + 1u, W.tgt_itl, &pr);  // A12
        ka_last = ka;
        fnow = W.mhz[kn];
        faft = W.mhz[ka];
      }
      const bool act = lane < ND;
      const bool cr = act && faft > fnow;  // A13
      const int nc = __popc(gballot(cr));
      const int mn = (int)__reduce_min_sync(gmask(), (unsigned)fnow);
      unsigned inset;
      if (nc == 0) {
        inset = gballot(act && fnow == mn);
        cse = __popc(inset) == 1 ? 1 : 2;
      } else if (nc < ND) {
        const int mu = (int)__reduce_min_sync(gmask(), (unsigned)(act && !cr ? fnow : 0x7fffffff));
        const int mr = (int)__reduce_min_sync(gmask(), (unsigned)(cr ? faft : 0x7fffffff));
        const long long g = (long long)mu - (long long)mr;  // A14, A15
        if (g <= (long long)delta) { inset = gballot(act && !cr && fnow == mu); cse = 3; }
        else { inset = gballot(act && fnow == mn); cse = 4; }
      } else {
        const int ma = (int)__reduce_min_sync(gmask(), (unsigned)faft);
        inset = gballot(act && faft == ma);
        cse = 5;
      }
      // round robin among the candidate set from the cursor (A17)
      const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & ((1u << ND) - 1u);
      dsel = (int)wrap_nd(cursor + (uint32_t)ffs0(rot), (uint32_t)ND);
      if (__popc(inset) >= 2) cursor = wrap_nd((uint32_t)dsel + 1u, (uint32_t)ND);
    }
    steps_route++;
    LP_MARK(2);
    h_r = fold(h_r, 3, (uint64_t)dsel, 0, (uint64_t)cse);
    if (lane == dsel) {
      if (eco) { c_n = D.nreq + D.pn + 1u; c_kv = D.nkv + D.pkv + in_i + 1u; c_lvl = ka_last; }  // its new state
      if (ens) { c_n = D.nreq + D.pn + 1u; c_kv = D.nkv + D.pkv + in_i + 1u; c_en = en_new; }
      dec_push(D, L, i, tf_i, in_i, io >> 16, W.nb - 1u);
      if ((V & 2) && W.rq_on) { P.o.req_decode[W.rq_base + i] = (uint8_t)dsel; P.o.req_case[W.rq_base + i] = (uint8_t)cse; }
    }
#if VT_PIPE_ARGMIN
    w = w_next;
#else
    w = argmin_time(fabs(hn.tf), hd != NIL);
#endif
  }
  // drain: every decode instance runs to completion, then its deferred ITL accounting
  dec_advance_all<V, F>(D, lane, L, W, INF, dE, P.o);
  if (lane < ND && !D.dead) itl_drain<V, F>(D, L, W, lane, P.o);
#if VT_DEFER_ITL
  uint32_t k_ok = 0u, k_both = 0u;  // the decode ITL accounting of the completion log (in-warp K4c)
  double k_sitl = 0.0;
  if (!(V & 2)) {
    if (lane < ND)  // the unused rest of this lane's chunk: empty entries
      for (uint32_t q = D.lpos; q < D.lend; ++q) { CEnt ce; ce.td = 0.0; ce.head = NIL; ce.d = 0u; L.clog[q] = ce; }
    __syncwarp(gmask());
#if VT_ITL_INWARP
    // the scenario's log and nodes are still warm in L2: all 32 lanes gather, then sum in order
    itl_scenario<ITL_UW>(P, W.clog_m, ND, W.slo_itl, L.clog, node, *(ItlScratch<ITL_UW> *)((char *)&W + P.ks_off), k_ok,
                    k_both, k_sitl);
#else
    if (lane == 0) P.clog_n[s] = W.clog_m;
#endif
  }
#endif
  if ((V & 2) && W.it_on && lane < ND) P.o.iter_count[W.it_base / P.o.iter_cap + NP + lane] = D.iters;
  __syncwarp(gmask());

#ifdef VT_LAT_PROBE
  LP_MARK(3);
  if (P.timing && lane == 0)
    for (int q = 0; q < 4; ++q) P.timing[2 * (size_t)P.n + 4 * (size_t)s + q] = (uint64_t)lp_acc[q];
#endif
  // ================================================================ O9: record
  // first error in (time, prefill before decode, instance) order = the oracle's stop point
  const double pet = lane < NP ? W.pa[lane].errt : INF;
  const int wp = argmin_time(pet, lane < NP && pet < INF);
  const int wd = argmin_time(dE.t, lane < ND && dE.t < INF);
  if (wp >= 0 || wd >= 0) {
    const double tp = wp >= 0 ? W.pa[wp].errt : INF;
    const double td = wd >= 0 ? gshfl(dE.t, wd) : INF;
    const uint32_t cd = gshfl(dE.code, wd >= 0 ? wd : 0);
    write_status(P, s, N, (wp >= 0 && tp <= td) ? W.pa[wp].errc : cd);
    if (lane < ND)  // leave the wheel clean for the next scenario of this warp
      for (uint32_t b = 0; b < P.nb; ++b) wst(wheels + (size_t)lane * P.nb + b, make_uint4(0u, 0u, 0u, 0u));
    return;
  }
  const int dd = lane < ND ? lane : 0;
#if VT_DACC_SMEM
#define LACC(f) W.da_##f[dd]
#else
#define LACC(f) D.f
#endif
  double tl = lane < ND ? LACC(tlast) : 0.0;
  if (lane < NP) tl = tl > W.pa[lane].tlast ? tl : W.pa[lane].tlast;
  for (int o = GS / 2; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(gmask(), tl, o, GS);
    tl = x > tl ? x : tl;
  }
  const double horizon = Dur > tl ? Dur : tl;  // A23
  // decode instances: lane d's totals gathered in instance order (A36/A37)
  uint64_t hd_[NI];
  double topd_[NI];
  double sitl = 0.0, edb = 0.0, edi = 0.0, bd = 0.0;
#pragma unroll
  for (int d = 0; d < NI; ++d) {
    hd_[d] = gshfl(LACC(h), d);
    if (d < ND) {
      sitl = add(sitl, gshfl(LACC(sitl), d));
      topd_[d] = gshfl(LACC(top), d);
      edb = add(edb, div(gshfl(LACC(ebusy), d), 1000.0));
      const double b = gshfl(LACC(bms), d);
      edi = add(edi, energy_j(W.p_idle, sub(horizon, b)));
      bd = add(bd, b);
    }
  }
  uint32_t c_itl = __reduce_add_sync(gmask(), lane < ND ? LACC(n_itl_ok) : 0u);
  uint32_t c_both = __reduce_add_sync(gmask(), lane < ND ? LACC(n_both) : 0u);
#if VT_DEFER_ITL && VT_ITL_INWARP
  if (!(V & 2)) { c_itl += k_ok; c_both += k_both; sitl = k_sitl; }
#endif
  const uint32_t c_di = __reduce_add_sync(gmask(), lane < ND ? D.iters : 0u);
  if (lane == 0) {
    voltana_result R = voltana_result{};
    uint64_t hh = splitmix64(h_r);  // A36: route chain, then prefill chains, then decode chains
    double sttft = 0.0, top = 0.0, epb = 0.0, epi = 0.0, bp = 0.0;
    uint32_t c_ttft = 0, c_itl_p = 0, c_both_p = 0, c_pi = 0;
    for (int q = 0; q < NP; ++q) {
      hh = splitmix64(hh ^ W.pa[q].h);
      sttft = add(sttft, W.pa[q].sttft);
      top = add(top, W.pa[q].top);
      epb = add(epb, div(W.pa[q].ebusy, 1000.0));
      epi = add(epi, energy_j(W.p_idle, sub(horizon, W.pa[q].bms)));
      bp = add(bp, W.pa[q].bms);
      c_ttft += W.pa[q].ttft_ok; c_itl_p += W.pa[q].itl_ok; c_both_p += W.pa[q].both; c_pi += W.pa[q].iters;
    }
#pragma unroll
    for (int d = 0; d < NI; ++d)
      if (d < ND) {
        hh = splitmix64(hh ^ hd_[d]);
        top = add(top, topd_[d]);  // one running sum: prefill instances, then decode (A37)
      }
    R.status = 0; R.n_requests = N;
    R.n_ttft_ok = c_ttft; R.n_itl_ok = c_itl_p + c_itl; R.n_both_ok = c_both_p + c_both; R.prefill_iters = c_pi;
    uint64_t sc = (uint64_t)c_pi + c_di;  // one decision per iteration ...
    if ((V & 2) && W.wo) {                   // ... unless window control skipped some [C1]
      sc = 0;
      for (int q = 0; q < NP; ++q) sc += W.pa[q].ndec;
      for (int d = 0; d < ND; ++d) sc += W.dl_ndec[d];
    }
    R.steps_ctrl = sc; R.steps_route = steps_route; R.decision_hash = hh;
    R.sum_ttft_ms = sttft; R.sum_itl_mean_ms = sitl;
    R.e_prefill_busy_j = epb; R.e_prefill_idle_j = epi; R.e_decode_busy_j = edb; R.e_decode_idle_j = edi;
    R.busy_ms_prefill = bp; R.busy_ms_decode = bd; R.top_level_ms = top; R.horizon_ms = horizon;
    P.out[s] = R;
  }
}

// V = 0: the paper's EcoFreq/EcoRoute/RR only (the default kernel); V & 1 adds the energy-scored
// router and controller [B1-B4]; V & 2 adds window control, blocking overhead, execution noise,
// ITL modes and the optional outputs [C-E]. The host launches the smallest V that covers the
// launch's layouts, so each variant pays only for its own registers.
template <int V, bool F>
__global__ void __launch_bounds__(SIM_THREADS, SIM_MIN_BLOCKS) simulate_kernel(const __grid_constant__ SimParams P) {
  extern __shared__ __align__(16) char smem[];
  const int lane = glane();
  const uint32_t grp = (threadIdx.x & 31u) / GS;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t sid = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * SPW + grp;  // scenario slot
  if (sid >= P.n_slots) return;
  char *slot = P.slots + (size_t)sid * P.slot_bytes;
  uint4 *wheels = P.wheels + (size_t)sid * P.wheel_per_slot;
  using WS = WarpSmemT<F ? 8 : VOLTANA_MAX_LEVELS>;
  WS &W = *(WS *)(smem + (size_t)(wib * SPW + grp) * P.smem_per_warp);
  for (;;) {
    uint32_t s = 0;
#if VT_TWO_ENDED
    // the last warp of each CTA takes the expensive end of the (LPT-ordered) list, the
    // others the cheap end; counter[0] bounds the total so the two ends never overlap
    if (lane == 0) {
      s = atomicAdd(P.counter, 1u);
      if (s < P.n)
        s = wib == SIM_THREADS / 32 - 1 ? atomicAdd(P.counter + 1, 1u) : P.n - 1u - atomicAdd(P.counter + 2, 1u);
    }
#else
    if (lane == 0) s = atomicAdd(P.counter, 1u);
#endif
    s = gshfl(s, 0);
    if (s >= P.n) break;
    uint64_t t0 = 0;
    if (P.timing) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    run_scenario<V, F>(P, s, slot, wheels, W, sid);
    __syncwarp(gmask());
    if (P.timing && lane == 0) {
      uint64_t t1;
      uint32_t sm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
#ifdef VT_PHASE_TIMING
      P.timing[2 * s] -= t0;       // phase-A duration (ns)
#else
      P.timing[2 * s] = t0;
#endif
      P.timing[2 * s + 1] = (t1 - t0) | ((uint64_t)sm << 56);
    }
  }
}

// ------------------------------------------------------------------ K4a: phase A as its own launch
// One thread per (scenario, prefill instance p): prefill instances never read decode state
// (A6, A7), so every prefill timeline of every scenario is independent work.
// The per-thread context names its members as the per-warp block does, so prefill_lane is
// the same code in both arrangements; the ladder-resolved TTFT / prefill-power rows come
// from P.rtab (filled by the setup launch), read through L1.
struct PCtx {
  double tgt_ttft, slo_ttft, p_idle, tdp, uh_p, uh_d, ctrl_iv, fs_ov;
  const double *tt, *dyn, *a1g, *c1g, *ut, *noise;
  const uint16_t *lad;
  uint32_t B, K, W, kp, ptiles, pcut, mono_tt, ctrl, wo, noise_mask, rq_on, it_on;
  uint64_t seed, rq_base, it_base;
};
// The same context in shared memory, one per lane group (VT_PA_SMEM): the fields are uniform
// over the group, so they cost no registers, and the ladder rows are read with LDS.
struct PCtxS {
  double tgt_ttft, slo_ttft, p_idle, tdp, uh_p, uh_d, ctrl_iv, fs_ov;
  const double *a1g, *c1g, *ut, *noise;
  const uint16_t *lad;
  uint32_t B, K, W, kp, ptiles, pcut, mono_tt, ctrl, wo, noise_mask, rq_on, it_on;
  uint64_t seed, rq_base, it_base;
  double tt[2 * VOLTANA_MAX_LEVELS];  // [K][a1, c1]
  double dyn[VOLTANA_MAX_LEVELS];     // prefill DYN
  double wa[32];                      // the window's arrivals and inclusive token prefix sums
  uint32_t wps[32];
  double wt[32];                      // the TTFTs being added to the report sum (O5, A37)
};
template <int G> __device__ __forceinline__ void win_put(PCtxS &W, uint32_t lane, double a, uint32_t ps) {
  W.wa[lane] = a;
  W.wps[lane] = ps;
}
template <int G> __device__ __forceinline__ double win_a(const PCtxS &W, const Grp<G> &, double, uint32_t i) {
  return W.wa[i];
}
template <int G> __device__ __forceinline__ uint32_t win_ps(const PCtxS &W, const Grp<G> &, uint32_t, uint32_t i) {
  return W.wps[i];
}
template <int G> __device__ __forceinline__ void win_tput(PCtxS &W, uint32_t lane, double t) { W.wt[lane] = t; }
template <int G> __device__ __forceinline__ double win_t(const PCtxS &W, const Grp<G> &, double, uint32_t i) {
  return W.wt[i];
}
__device__ __forceinline__ void pctx_scalars(PCtxS &S, const PCtx &C) {
  S.tgt_ttft = C.tgt_ttft; S.slo_ttft = C.slo_ttft; S.p_idle = C.p_idle; S.tdp = C.tdp; S.uh_p = C.uh_p;
  S.uh_d = C.uh_d; S.ctrl_iv = C.ctrl_iv; S.fs_ov = C.fs_ov; S.a1g = C.a1g; S.c1g = C.c1g; S.ut = C.ut;
  S.noise = C.noise; S.lad = C.lad; S.B = C.B; S.K = C.K; S.W = C.W; S.kp = C.kp; S.ptiles = C.ptiles;
  S.pcut = C.pcut; S.mono_tt = C.mono_tt; S.ctrl = C.ctrl; S.wo = C.wo; S.noise_mask = C.noise_mask;
  S.rq_on = C.rq_on; S.it_on = C.it_on; S.seed = C.seed; S.rq_base = C.rq_base; S.it_base = C.it_base;
}
#ifndef VT_PA_SMEM
#define VT_PA_SMEM 1
#endif

template <int V, bool F>
__global__ void __launch_bounds__(PA_THREADS, PA_MIN_BLOCKS) prefill_kernel(const __grid_constant__ SimParams P) {
  const uint32_t total = P.n * P.np_max;
  const uint32_t wpb = PA_WARP ? blockDim.x / PA_G : blockDim.x;
  const uint32_t x0 = blockIdx.x * wpb + (PA_WARP ? threadIdx.x / PA_G : threadIdx.x);
  for (uint32_t x = x0; x < total; x += gridDim.x * wpb) {
    const uint32_t s = x / P.np_max, p = x - s * P.np_max;
    if (!(P.trace_id[s] < P.n_traces && P.slo_id[s] < P.n_slos && P.layout_id[s] < P.n_layouts &&
          P.grid_id[s] < P.n_grids && P.profile_id[s] < P.n_profiles))
      continue;  // K4b writes E_INPUT
    const voltana_layout &LY = P.lay[P.layout_id[s]];
    const uint32_t NP = (uint32_t)LY.n_p;
    if (p >= NP) continue;
    const uint32_t tr = P.trace_id[s];
    const uint64_t off = P.offset[tr];
    const uint64_t N64 = P.offset[tr + 1] - off;
    if (!(N64 <= P.max_requests)) continue;  // K4b writes E_INPUT (its other checks follow there)
    const voltana_slo &SL = P.slo[P.slo_id[s]];
    const uint32_t g = P.grid_id[s], pr = P.profile_id[s];
    const voltana_grid &GR = P.grid[g];
    const DevProfile &PR = P.prof[pr];
    PCtx C;
    C.rq_on = 0u; C.rq_base = 0; C.it_on = 0u; C.it_base = 0;
    if ((V & 2) && P.o.req_offset) {
      C.rq_base = P.o.req_offset[s];
      const uint64_t len = P.o.req_offset[s + 1] - C.rq_base;
      if (len != 0 && len != N64) continue;  // K4b writes E_INPUT
      C.rq_on = len != 0;
    }
    if ((V & 2) && P.o.iter_offset) { C.it_on = 1u; C.it_base = P.o.iter_offset[s]; }
    C.tgt_ttft = mul(SL.scale, SL.ttft_ms);  // A3
    C.slo_ttft = SL.ttft_ms;
    C.p_idle = PR.p_idle; C.tdp = PR.tdp; C.uh_p = PR.uh[0]; C.uh_d = PR.uh[1];
    C.ctrl_iv = LY.ctrl_interval_ms; C.fs_ov = LY.freq_overhead_ms;
    const double *rt = P.rtab + ((size_t)g * MAX_PROFILES + pr) * RT_STRIDE;
    C.tt = rt; C.dyn = rt + 2 * VOLTANA_MAX_LEVELS;
    C.a1g = PR.a1; C.c1g = PR.c1;
    C.ut = VT_UTAB ? P.utab + (size_t)pr * 2 * SIM_UTAB : nullptr;
    C.noise = LY.exec_noise; C.noise_mask = LY.noise_len - 1u;
    C.lad = GR.level;
    C.B = LY.max_batch_tokens; C.K = (uint32_t)GR.k; C.W = (uint32_t)PR.tile_w; C.kp = (uint32_t)PR.k;
    C.ptiles = (uint32_t)PR.n_ptiles; C.pcut = PR.pcut;
    C.ctrl = (uint32_t)LY.ctrl_mode;
    C.wo = (V & 2) && (LY.ctrl_interval_ms > 0.0 || LY.freq_overhead_ms > 0.0) ? 1u : 0u;
    C.seed = P.hash_seed[s];
    {  // coefficient-monotone TTFT rows allow the exact binary search (A32); tiled TTFT: scan (F1)
      bool mt = PR.n_ptiles <= 1;
      for (uint32_t k = 0; mt && k + 1 < C.K; ++k)
        mt = rt[2 * k + 2] <= rt[2 * k] && rt[2 * k + 3] <= rt[2 * k + 1];
      C.mono_tt = mt;
    }
    Node *node = (Node *)(P.nodes + (size_t)s * P.max_requests * sizeof(Node));
    PaRes R;
#ifdef VT_PA_TIMING
    uint64_t tq0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq0));
#endif
    if (PA_WARP) {
#if VT_PA_SMEM
      __shared__ PCtxS cs[PA_THREADS / PA_G];
      PCtxS &S = cs[threadIdx.x / PA_G];
      const Grp<PA_G> g;
      if (g.gl == 0) pctx_scalars(S, C);
      for (uint32_t k = g.gl; k < C.K; k += PA_G) {
        S.tt[2 * k] = C.tt[2 * k];
        S.tt[2 * k + 1] = C.tt[2 * k + 1];
        S.dyn[k] = C.dyn[k];
      }
      __syncwarp(g.m);
      prefill_warp<V, F, PA_G>(P, S, node, P.arrival + off, P.in_len + off, P.out_len + off, (uint32_t)N64, p, NP,
                               P.hash_seed[s], R);
      __syncwarp(g.m);  // the next item of this group rewrites S
#else
      prefill_warp<V, F, PA_G>(P, C, node, P.arrival + off, P.in_len + off, P.out_len + off, (uint32_t)N64, p, NP,
                               P.hash_seed[s], R);
#endif
      if ((threadIdx.x & (PA_G - 1)) == 0) P.pares[(size_t)s * NI + p] = R;
#ifdef VT_PA_TIMING
      if (P.timing && (threadIdx.x & (PA_G - 1)) == 0) {  // experiment: [x][2] chain start, duration
        uint64_t tq1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq1));
        P.timing[2 * (size_t)P.n + 2 * x] = tq0;   // after K4b's [n][2]
        P.timing[2 * (size_t)P.n + 2 * x + 1] = tq1 - tq0;
      }
#endif
    } else {
      prefill_lane<V, F, true>(P, C, node, P.arrival + off, P.in_len + off, P.out_len + off, (uint32_t)N64, p,
                               NP, P.hash_seed[s], R);
      P.pares[(size_t)s * NI + p] = R;
    }
  }
}

template <int V>
static void launch_pa_v(const SimParams &P, bool fast, int grid, cudaStream_t st) {
  if (fast) prefill_kernel<V, true><<<grid, PA_THREADS, 0, st>>>(P);
  else prefill_kernel<V, false><<<grid, PA_THREADS, 0, st>>>(P);
}

cudaError_t launch_prefill(const SimParams &P, int v, bool fast, cudaStream_t st) {
  const uint64_t total = (uint64_t)P.n * P.np_max;
  const uint64_t per_cta = PA_WARP ? PA_THREADS / PA_G : PA_THREADS;
  const int grid = (int)((total + per_cta - 1) / per_cta);
  if (grid < 1) return cudaSuccess;
  switch (v & 3) {
    case 1: launch_pa_v<1>(P, fast, grid, st); break;
    case 2: launch_pa_v<2>(P, fast, grid, st); break;
    case 3: launch_pa_v<3>(P, fast, grid, st); break;
    default: launch_pa_v<0>(P, fast, grid, st); break;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K4c: deferred ITL accounting
// The per-request mean-ITL accounting of O6 (A30) for the paper's-policy kernels, taken off
// K4b's in-order path: K4b logs every iteration end with completions (end time, head of the
// completion list, instance) in its own order; here one warp per scenario walks the lists.
// Lanes gather 32 log entries at a time (each walks its list, up to 4 values in registers),
// then the values are added to their instance's running sum one by one in log order, so each
// instance's sum is the oracle's sequential sum in completion order (A37); the counts are
// order-free. The record's decode ITL fields are completed here (K4b wrote the prefill part).
// K4c as its own launch (VT_ITL_INWARP = 0): one warp per scenario after K4b.
constexpr int ITL_U = 2;
__global__ void __launch_bounds__(128) itl_kernel(const __grid_constant__ SimParams P) {
  __shared__ ItlScratch<ITL_U> scr[4];
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < P.n; s += nw) {
    voltana_result *R = P.out + s;
    if (R->status != 0u) continue;
    uint32_t c_ok, c_both;
    double sitl;
    itl_scenario<ITL_U>(P, P.clog_n[s], P.lay[P.layout_id[s]].n_d, P.slo[P.slo_id[s]].itl_ms,
                        P.clog + (size_t)s * P.clog_stride,
                        (const Node *)(P.nodes + (size_t)s * P.max_requests * sizeof(Node)), scr[wib], c_ok, c_both,
                        sitl);
    if (lane == 0) {
      R->n_itl_ok += c_ok;
      R->n_both_ok += c_both;
      R->sum_itl_mean_ms = sitl;
    }
  }
}

cudaError_t launch_itl(const SimParams &P, cudaStream_t st) {
  int grid = (int)((P.n + 3u) / 4u);
  grid = grid < 1 ? 1 : grid;
  itl_kernel<<<grid, 128, 0, st>>>(P);
  return cudaGetLastError();
}

size_t sim_smem_fixed(bool fast) {
  const size_t b = fast ? sizeof(WarpSmemT<8>) : sizeof(WarpSmemT<VOLTANA_MAX_LEVELS>);
  return (b - sizeof(double) + 15) & ~(size_t)15;
}

__global__ void utab_kernel(const __grid_constant__ SimParams P) {
  const uint32_t stride = gridDim.x * blockDim.x, x0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (P.utab) {
    const uint32_t total = P.n_profiles * 2u * SIM_UTAB;
    for (uint32_t x = x0; x < total; x += stride) {
      const uint32_t pr = x / (2u * SIM_UTAB), ph = (x / SIM_UTAB) & 1u, l = x % SIM_UTAB;
      const double uh = P.prof[pr].uh[ph];
      ((double *)P.utab)[x] = div((double)l, add((double)l, uh));
    }
  }
  if (P.rtab) {  // VT_SPLIT_A: ladder-resolved prefill rows per (grid, profile): [K][a1, c1], DYN_prefill[K]
    const uint32_t total = P.n_grids * P.n_profiles * VOLTANA_MAX_LEVELS;
    for (uint32_t x = x0; x < total; x += stride) {
      const uint32_t g = x / (P.n_profiles * VOLTANA_MAX_LEVELS), r = x % (P.n_profiles * VOLTANA_MAX_LEVELS);
      const uint32_t pr = r / VOLTANA_MAX_LEVELS, k = r % VOLTANA_MAX_LEVELS;
      if (k >= (uint32_t)P.grid[g].k) continue;
      const DevProfile &PR = P.prof[pr];
      const uint32_t lv = P.grid[g].level[k];
      if (lv >= (uint32_t)PR.k) continue;  // grid not paired with this profile (host-validated when used)
      double *rt = P.rtab + ((size_t)g * MAX_PROFILES + pr) * RT_STRIDE;
      rt[2 * k] = PR.a1[lv];
      rt[2 * k + 1] = PR.c1[lv];
      rt[2 * VOLTANA_MAX_LEVELS + k] = PR.dyn[lv];
    }
  }
}

cudaError_t launch_utab(const SimParams &P, cudaStream_t st) {
  utab_kernel<<<64, 256, 0, st>>>(P);
  return cudaGetLastError();
}

template <int V>
static const void *kptr(bool fast) {
  return fast ? (const void *)simulate_kernel<V, true> : (const void *)simulate_kernel<V, false>;
}

const void *sim_kernel_ptr(int v, bool fast) {
  switch (v & 3) {
    case 1: return kptr<1>(fast);
    case 2: return kptr<2>(fast);
    case 3: return kptr<3>(fast);
    default: return kptr<0>(fast);
  }
}

template <int V>
static void launch_v(const SimParams &P, bool fast, int grid, size_t smem, cudaStream_t st) {
  if (fast) simulate_kernel<V, true><<<grid, SIM_THREADS, smem, st>>>(P);
  else simulate_kernel<V, false><<<grid, SIM_THREADS, smem, st>>>(P);
}

cudaError_t launch_sim(const SimParams &P, int v, bool fast, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(sim_kernel_ptr(v, fast), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  switch (v & 3) {
    case 1: launch_v<1>(P, fast, grid, smem, st); break;
    case 2: launch_v<2>(P, fast, grid, smem, st); break;
    case 3: launch_v<3>(P, fast, grid, smem, st); break;
    default: launch_v<0>(P, fast, grid, smem, st); break;
  }
  return cudaGetLastError();
}

}  // namespace vt
