// k_simulate.cu — K4: batched trace-driven evaluation of EcoFreq + EcoRoute (north_star).
//
// The scenario is evaluated through its exact causal decomposition, in two
// launches after a small setup launch:
//
//  K4a (prefill_kernel)  Prefill instances never read decode state: requests go round robin by
//           id and batches are FCFS (A6). One warp per (scenario, prefill
//           instance p) runs p's batch formation, EcoFreq with the waiting-time budget
//           (P:377-388), TTFT accounting and energy, and writes one 16-B node per request
//           (first-token time with the TTFT verdict in its sign, in, out).
//  K4b (simulate_kernel) One warp per scenario (persistent warps). Routing happens
//           at prefill completions in (time, instance, id) order: the warp merges the N_P
//           prefill streams 32 requests at a time (merge path by warp shuffles) into a
//           shared-memory window and routes from it. Before routing at time t, decode lane d
//           advances its own instance through every event strictly before t (iteration
//           END/START, admission, EcoFreq, energy) — decode instances interact only through
//           routing, and at equal times a PrefillDone drains before a DecodeIterDone and
//           before every START (A18), so this order is exact. EcoRoute's what-if (f, f') of
//           every (instance, level) is one lane each and one ballot; the case analysis
//            then runs redundantly in every lane with no further collective.
// Decisions therefore match the sequential oracle bit for bit; the record's report-only
// accumulators are per instance (A36/A37), so they match bit for bit too.
//
// Decode running sets: a per-instance timing wheel of NB (<= 2048, L2-resident) buckets keyed
// by the iteration at which a request finishes (admission iteration + out - 2). All running
// requests advance together (+1 token per iteration), so a bucket's request count and
// KV total retire the whole iteration's completions in O(1); the rare request finishing NB or
// more iterations ahead waits on a sorted far list until its bucket enters the window. Bucket
// lists keep admission order; the per-request ITL accounting (A30) walks them later, in
// completion order, off the decision chain (a per-warp completion log and an in-warp pass).
//
// Register budget: per-lane instance state lives in registers; everything cold (scenario
// constants, staged tables, phase-A results, the route window) lives in a per-warp
// shared-memory block.
#include <cstdint>

#include "vt_device.cuh"
#include "vt_sim.h"

namespace vt {

__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" :: "l"(p)); }
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); }

__device__ __forceinline__ unsigned wballot(bool p) { return __ballot_sync(FULL, p); }
template <class T> __device__ __forceinline__ T wshfl(T v, int src) { return __shfl_sync(FULL, v, src); }

struct Node {       // 16 B per request (workspace, written by K4a)
  double tf;        // +t_first if the TTFT SLO was met, -t_first otherwise (t_first > 0)
  uint32_t next;    // K4b: admission-queue / wheel-bucket / far-list link
  uint32_t io;      // in | out << 16; on the far list: the finishing iteration (see far_insert)
};
__device__ __forceinline__ uint32_t node_in(const Node &n) { return n.io & 0xffffu; }
__device__ __forceinline__ uint32_t node_out(const Node &n) { return n.io >> 16; }

struct RouteEnt {   // one request of the merged route stream (16 B)
  double tf;        // as Node.tf
  uint32_t id;      // request id (trace order)
  uint32_t io;      // in | out << 16
};

constexpr int NI = VOLTANA_MAX_INSTANCES;
constexpr int ECO_LUT_K = 5;   // the N_D = 2 EcoRoute decision table covers ladders up to 5 levels
constexpr int ECO_LUT_N = ECO_LUT_K * ECO_LUT_K * ECO_LUT_K * ECO_LUT_K * 2;

struct RouteWin {   // the merged window of the prefill streams (per warp, shared memory)
  RouteEnt ring[32];
  uint32_t sbase[NI];  // next unconsumed request id of prefill stream p (ids p, p + N_P, ...)
  uint32_t send[NI];   // stream end: ids >= send[p] were not written (K4a stopped on an error)
};

// Cold per-instance state of decode lane d (shared memory: fewer live registers on the route
// chain; touched once per iteration START, or rarely)
struct DecCold {
  double ebusy, bms, top, sitl;    // busy energy (W*ms), busy time, top-level time, ITL sum (V & 2)
  uint64_t h;                      // decision-hash chain (A36)
  uint32_t far_h, far_hfin;        // far list head and its finishing iteration (NIL: empty)
  uint32_t n_itl_ok, n_both;       // in-line ITL accounting counts (V & 2)
};

// Per-warp shared-memory block (one scenario at a time). Sized by sim_smem_fixed.
template <int KC>  // KC: level capacity of the staged tables (8 in the fast-table kernel, else 64)
struct WarpSmemT {
  RouteWin rw;
  PaRes pa[NI];                    // phase-A results per prefill lane (read back for the record)
  // ---- scenario constants
  double tau, slo_itl, tgt_itl, slo_ttft, tgt_ttft, p_idle, tdp, uh_p, uh_d;
  const double *a2g, *b2g, *c2g;   // profile ITL tables (when not staged)
  const double *ut;                // this profile's utilisation tables [2][SIM_UTAB]
  uint32_t kvcap, max_steps, K, T, W, kp, nb;
  int32_t wshift;
  uint32_t itl_smem, mono_it;
  uint32_t ctrl;                   // layout ctrl_mode: 0 EcoFreq, 1 energy argmin [B4]
  double ctrl_iv, fs_ov;           // window interval, blocking frequency-set overhead [C1-C3]
  const uint32_t *tin, *tout;      // this scenario's trace lengths (far-list requests, see far_insert)
  const double *noise;             // execution-noise factor table or NULL [D1, D2]
  uint32_t noise_mask, np;         // np: N_P (decode instance d is noise instance N_P + d)
  uint64_t seed;                   // scenario hash seed (noise index)
  double *re;                      // ITL modes (E3): this slot's rings [N_D][ring_r] of iteration end times
  uint32_t *rc;                    //   ... and of cumulative counts of gaps above the ITL SLO
  uint32_t itlm, rmask;            //   layout itl_mode, ring_r - 1
  uint32_t clog_m;                 // completion-log slots handed out (chunks of CLOG_CHUNK)
  uint32_t wo;                     // window control or blocking overhead active (C1-C3)
  uint32_t dl_vc[NI];              // decode lane: gaps above the ITL SLO so far
  DecCold dc[NI];                  // decode lane d's cold state
  uint64_t rq_base, it_base;       // outputs (E1-E3): request / iteration-slot base of the scenario
  uint32_t rq_on, it_on;
  // ---- variant-kernel per-instance controller state [C1-C3]
  double dl_last[NI];              // decode lane: time of the last decision (-inf: none)
  uint32_t dl_cur[NI], dl_ndec[NI];  // decode lane: running level, decisions taken
  uint8_t lut[KC == 8 ? ECO_LUT_N : 1];  // N_D = 2 EcoRoute decision table (fast kernel)
  // ---- staged ladder tables
  uint16_t lad[KC];
  int32_t mhz[KC];
  double dyn[2 * KC];  // [2][K]: prefill, decode
  double it[1];        // [T][K][3]: a2, b2, c2 (flexible; itl_smem)
};

__device__ __forceinline__ char *node_base(const SimParams &P, uint32_t s) {
  const uint64_t o = P.node_offset ? P.node_offset[s] : (uint64_t)s * P.max_requests;
  return P.nodes + o * sizeof(Node);
}

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
  if (F || W.itl_smem) {
    const double *r = W.it + 3 * ((size_t)j * W.K + k);
    return add(add(mul(r[0], dn), mul(r[1], dkv)), r[2]);
  }
  const size_t o = (size_t)j * W.kp + W.lad[k];
  return add(add(mul(__ldg(W.a2g + o), dn), mul(__ldg(W.b2g + o), dkv)), __ldg(W.c2g + o));
}

// Lowest ladder index whose prediction meets `target` (A1), else K-1 (A2);
// *pred = the prediction there. Ascending scan with early exit, or an exact binary search
// when the tables are coefficient-monotone in f (A32).
template <bool F, class WS>
__device__ int lowest_itl(const WS &W, uint32_t n, uint32_t kv, double target, double *pred) {
  const uint32_t j = tile_j<F>(W, n);
  const int K = (int)W.K;
  const double dn = (double)n, dkv = (double)kv;
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

// The same lowest feasible level, searched from a start level k0 (the instance's previous
// decision): on coefficient-monotone tables (A32) the feasible levels are upward closed, so
// galloping from k0 (steps 1, 2, 4, ... towards the boundary, then a binary search between
// the last infeasible and the first feasible probe) ends at the ascending scan's answer —
// usually after two or three evaluations instead of up to K (or log2 K for a long ladder).
// Level K-1 counts as feasible (A2: nothing feasible below it selects it).
template <bool F, class WS>
__device__ __forceinline__ int lowest_itl_from(const WS &W, uint32_t n, uint32_t kv, double target, int k0,
                                               double *pred) {
  const int K = (int)W.K;
  if (!W.mono_it || K < 3) return lowest_itl<F>(W, n, kv, target, pred);
  const uint32_t j = tile_j<F>(W, n);
  const double dn = (double)n, dkv = (double)kv;
  int k = k0 < K - 2 ? k0 : K - 2;
  double p = itl_at<F>(W, j, k, dn, dkv);
  if (F) {   // short ladders: a plain walk (fewer instructions than galloping; 77.7 vs 80.4 ms on C4)
    if (p <= target) {
      while (k > 0) {
        const double q = itl_at<F>(W, j, k - 1, dn, dkv);
        if (!(q <= target)) break;
        --k;
        p = q;
      }
    } else {
      do {
        ++k;
        p = itl_at<F>(W, j, k, dn, dkv);
      } while (k < K - 1 && !(p <= target));
    }
    *pred = p;
    return k;
  }
  int bad, ok;            // bad: infeasible (or -1), ok: feasible (or K-1); answer in (bad, ok]
  double pok;
  if (p <= target) {
    ok = k; pok = p; bad = -1;
    for (int step = 1; ok > 0; step <<= 1) {
      const int q = ok - step >= 0 ? ok - step : 0;
      const double pq = itl_at<F>(W, j, q, dn, dkv);
      if (!(pq <= target)) { bad = q; break; }
      ok = q; pok = pq;
      if (q == 0) break;
    }
  } else {
    bad = k; ok = K - 1; pok = 0.0;
    bool have = false;
    for (int step = 1; bad < K - 2; step <<= 1) {
      const int q = bad + step <= K - 2 ? bad + step : K - 2;
      const double pq = itl_at<F>(W, j, q, dn, dkv);
      if (pq <= target) { ok = q; pok = pq; have = true; break; }
      bad = q;
    }
    if (!have) {          // nothing feasible below K-1 (A2)
      *pred = itl_at<F>(W, j, K - 1, dn, dkv);
      return K - 1;
    }
  }
  while (ok - bad > 1) {  // (bad, ok]: bad infeasible, ok feasible
    const int mid = (bad + ok) >> 1;
    const double pm = itl_at<F>(W, j, mid, dn, dkv);
    if (pm <= target) { ok = mid; pok = pm; } else bad = mid;
  }
  *pred = pok;
  return ok;
}

// The lowest feasible level (A1, A2) of the state (n >= 1, kv) held by this lane's group of
// eight lanes (lanes 8g..8g+7, `on` uniform in the group), on coefficient-monotone tables where
// the feasible levels are upward closed (A32): round 1 probes levels S-1, 2S-1, ... (S =
// ceil(K/8), the last probe is K-1, feasible by A2); round 2 probes the < 8 levels below the first
// feasible probe. The ascending scan's answer, in two parallel evaluations per lane. K <= 64.
template <bool F, class WS>
__device__ __forceinline__ int lowest_itl_g8(const WS &W, uint32_t n, uint32_t kv, double target, bool on) {
  const uint32_t lane = threadIdx.x & 31u, r = lane & 7u, gsh = lane & ~7u;
  const int K = (int)W.K;
  const int S = (K + 7) >> 3;
  const uint32_t j = tile_j<F>(W, n);
  const double dn = (double)n, dkv = (double)kv;
  const int p = min((int)(r + 1u) * S - 1, K - 1);
  bool f = !on || p == K - 1 || itl_at<F>(W, j, p, dn, dkv) <= target;
  unsigned m = (__ballot_sync(FULL, f) >> gsh) & 0xFFu;
  const int fi = ffs0(m);                        // the first feasible probe (the last one is K-1)
  const int hi = min((fi + 1) * S - 1, K - 1);   // feasible
  const int lo = fi * S;                         // levels lo..hi-1: not probed yet
  const int q = lo + (int)r;
  f = !on || q >= hi || itl_at<F>(W, j, q, dn, dkv) <= target;
  m = (__ballot_sync(FULL, f) >> gsh) & 0xFFu;
  const int k = lo + ffs0(m);
  VT_CHECK(m != 0u && hi >= 0 && hi < K && lo >= 0);
  return k < hi ? k : hi;
}

// busy power (eq:P-f P:187, A22) with the utilisation from the launch's table (the entries
// are the same division, so the value is identical)
__device__ __forceinline__ double bpow_u(const double *ut, double p_idle, double tdp, double uh, int phase, double dyn,
                                         uint32_t load) {
  const double u = load < SIM_UTAB ? __ldg(ut + phase * SIM_UTAB + load) : div((double)load, add((double)load, uh));
  const double w = add(p_idle, mul(u, dyn));
  return w < tdp ? w : tdp;
}
template <class WS>
__device__ __forceinline__ double bpow(const WS &W, int phase, double dyn, uint32_t load) {
  return bpow_u(W.ut, W.p_idle, W.tdp, phase ? W.uh_d : W.uh_p, phase, dyn, load);
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

// [D2] execution-noise factor of iteration j of instance inst: counter-based index into the
// host-drawn table (no transcendental on either side).
__device__ __forceinline__ double noise_at(const double *noise, uint32_t mask, uint64_t seed, uint64_t inst,
                                           uint64_t j) {
  const uint64_t x = seed ^ 0xD1B54A32D192ED03ull ^ (inst << 40) ^ j;
  return __ldg(noise + (splitmix64(x) & mask));
}

// iteration record of the per-instance time series (E2)
__device__ __forceinline__ void log_iter(const voltana_outputs &O, bool on, uint64_t base, uint32_t u, uint32_t j,
                                         double t, double dur, uint32_t load, uint32_t kv, int k, uint32_t flags) {
  if (!on || j >= O.iter_cap) return;
  voltana_iteration r;
  r.t_start = t; r.dur_ms = dur; r.load = load; r.n_kv = kv; r.level = (uint16_t)k; r.flags = (uint8_t)flags;
#pragma unroll
  for (int x = 0; x < 5; ++x) r.reserved[x] = 0;
  O.iters[base + (uint64_t)u * O.iter_cap + j] = r;
}

// ------------------------------------------------------------------ decode lanes
// Timing-wheel bucket (16 B; all-zero = empty): x = first request + 1, y = last request + 1
// (list in admission order), z = requests finishing in this iteration, w = their in + out.
struct Err {               // first error of one lane in its own event order
  double t;                // +inf = none
  uint32_t code;
};

struct Dec {               // decode instance d, owned by lane d (hot state; the cold rest in WarpSmemT::dc)
  uint32_t nreq, nkv, pn, pkv, iters, cur, qh, qt;
  int klast;               // the last EcoFreq level found by the search (start of the next one)
  uint32_t lpos, lend;     // this lane's chunk [lpos, lend) of the completion log
  bool busy, dead, lneed;  // lneed: the chunk is full, dec_advance stopped before an END
  double end;
  uint4 bcur;              // bucket of the running iteration, read at its START (final by then)
  Node qhn;                // register copy of the admission-queue head node
};

struct Lane {              // per-lane pointers
  Node *node;
  uint4 *wheel;            // this lane's decode instance: [NB] buckets
  CEnt *clog;              // the warp's completion log [CLOG_CAP]
};

// ITL accounting of one completion list at its iteration end td (variant kernels with ITL
// modes or per-request outputs: in line, in completion order, A30, A37).
template <int V, bool F, class WS>
__device__ void itl_walk(Dec &D, const Lane &L, WS &W, int d, const voltana_outputs &O, uint32_t id, double td) {
  const double slo = W.slo_itl;
  Node nd = L.node[id];
  for (uint32_t hop = 0; hop < W.max_steps; ++hop) {
    const double itl = div(sub(td, fabs(nd.tf)), (double)(node_out(nd) - 1u));
    W.dc[d].sitl = add(W.dc[d].sitl, itl);
    bool ok = itl <= slo;
    if ((V & 2) && W.itlm) {
      // ITL Max / P99 (E3): the request's gaps are e_a - t_first and the iteration gaps of
      // (a, f], f = this iteration, a = f - (out - 2); count those above the SLO from the
      // instance's rings and compare with the nearest-rank allowance (0 for Max)
      const uint32_t n = node_out(nd) - 1u;
      const uint32_t a = D.cur - (n - 1u);
      const double ea = W.re[(size_t)d * (W.rmask + 1u) + (a & W.rmask)];
      const uint32_t ca = W.rc[(size_t)d * (W.rmask + 1u) + (a & W.rmask)];
      const uint32_t viol = (W.dl_vc[d] - ca) + (sub(ea, fabs(nd.tf)) > slo ? 1u : 0u);
      const uint32_t allow = W.itlm == 1u ? 0u : n - (99u * n + 99u) / 100u;
      ok = viol <= allow;
    }
    W.dc[d].n_itl_ok += ok;
    W.dc[d].n_both += ok && nd.tf > 0.0;
    if ((V & 2) && W.rq_on) {  // per-request record (E1)
      O.req_tdone[W.rq_base + id] = td;
      O.req_itl[W.rq_base + id] = itl;
    }
    if (nd.next == NIL) break;
    id = nd.next;
    nd = L.node[id];
  }
}

// Append request i (finishing at iteration fin) to its bucket; (lfin, lb) = the bucket
// written last during this START, kept coherent with the loaded copy.
__device__ __forceinline__ void bucket_append(const Lane &L, uint32_t nbm, uint32_t i, uint32_t fin, uint32_t inout,
                                              uint32_t &lfin, uint4 &lb) {
  uint4 b = fin == lfin ? lb : L.wheel[fin & nbm];
  L.node[i].next = NIL;
  if (b.y == 0u) b.x = i + 1u; else L.node[b.y - 1u].next = i;
  b.y = i + 1u;
  b.z += 1u;
  b.w += inout;
  L.wheel[fin & nbm] = b;
  lfin = fin;
  lb = b;
}

// A request finishing NB or more iterations ahead waits on the far list, sorted by
// (finishing iteration, admission order); rare (out > NB + 1). While it waits, its node's io
// field holds the finishing iteration (no per-request side array in the workspace); in and out
// are restored from the trace when it joins its bucket.
__device__ void far_insert(DecCold &C, const Lane &L, uint32_t max_steps, uint32_t i, uint32_t fin) {
  L.node[i].io = fin;
  if (C.far_h == NIL || fin < C.far_hfin) {
    L.node[i].next = C.far_h;
    C.far_h = i;
    C.far_hfin = fin;
    return;
  }
  uint32_t prev = C.far_h;
  for (uint32_t hop = 0; hop < max_steps; ++hop) {
    const uint32_t nx = L.node[prev].next;
    if (nx == NIL || L.node[nx].io > fin) break;
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
      if (!(V & 2) && D.lpos == D.lend) { D.lneed = true; return; }  // a new log chunk first (dec_advance_all)
      tnow = D.end;
      cont = true;
      // ---- O6 DecodeIterDone: +1 KV token per running request; this iteration's completions
      D.nkv += D.nreq;
      const uint4 b = D.bcur;
      D.nreq -= b.z;
      D.nkv -= b.w;
      if (b.x != 0u) {
        L.wheel[D.cur & nbm] = make_uint4(0u, 0u, 0u, 0u);
        if (!(V & 2)) {  // log (td, list head, instance); the in-warp ITL pass does the accounting (A30, A37)
          CEnt ce;
          ce.td = tnow; ce.head = b.x - 1u; ce.d = (uint32_t)d;
          L.clog[D.lpos++] = ce;
        } else {
          itl_walk<V, F>(D, L, W, d, O, b.x - 1u, tnow);
        }
      }
      D.busy = false;
    } else {
      // idle: the next START happens when the head of the admission queue becomes available
      if (D.qh == NIL) return;
      const double av = add(fabs(D.qhn.tf), W.tau);  // KvTransferDone (A18)
      if (!(av < t_lim)) return;
      tnow = av;
    }
    // ---- O7 START_DECODE at tnow
    uint32_t lfin = NIL;
    uint4 lb = make_uint4(0u, 0u, 0u, 0u);
    // far requests whose finishing iteration entered the window join their bucket now,
    // before any direct admission can reach that bucket (admission order, A37)
    DecCold &C = W.dc[d];
    while (C.far_hfin - D.iters < W.nb) {   // (an empty far list has far_hfin = NIL)
      const uint32_t i = C.far_h;
      const Node fn = L.node[i];
      const uint32_t fin = C.far_hfin;
      C.far_h = fn.next;
      C.far_hfin = fn.next != NIL ? L.node[fn.next].io : NIL;
      const uint32_t io = (uint32_t)(uint16_t)W.tin[i] | (uint32_t)(uint16_t)W.tout[i] << 16;  // as K4a wrote it
      L.node[i].io = io;
      bucket_append(L, nbm, i, fin, (io & 0xffffu) + (io >> 16), lfin, lb);
    }
    // FCFS admission while KV fits (A20)
    const double tau = W.tau;
    const uint32_t kvcap = W.kvcap;
    while (D.qh != NIL) {
      const Node hn = D.qhn;
      if (!(add(fabs(hn.tf), tau) <= tnow)) break;  // still in KV transfer
      const uint32_t need = node_in(hn) + 1u;
      if (D.nkv + need > kvcap) break;
      const uint32_t i = D.qh;
      D.qh = hn.next;
      if (D.qh == NIL) D.qt = NIL;
      else D.qhn = L.node[D.qh];
      const uint32_t fin = D.iters + node_out(hn) - 2u;  // its last iteration
      if (node_out(hn) - 2u < W.nb) bucket_append(L, nbm, i, fin, node_in(hn) + node_out(hn), lfin, lb);
      else far_insert(W.dc[d], L, W.max_steps, i, fin);
      VT_CHECK(D.nreq < 0x7fffffffu);
      D.nreq += 1u;
      D.nkv += need;
      D.pn -= 1u;
      D.pkv -= need;
    }
    const bool backlog = D.qh != NIL && add(fabs(D.qhn.tf), tau) <= tnow;  // A5
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
      else { k = lowest_itl_from<F>(W, D.nreq, D.nkv, W.tgt_itl, D.klast, &dur); D.klast = k; }
      C.h = fold(C.h, 2, (uint64_t)d, (uint64_t)k, 0);
      if ((V & 2) && W.wo) { W.dl_last[d] = tnow; W.dl_ndec[d] += 1u; }
    }
    if (!(dur > 0.0)) { E.t = tnow; E.code = VOLTANA_ITEM_E_CONTRACT; D.dead = true; return; }
    if ((V & 2) && W.noise) {  // [D1]
      const double e = noise_at(W.noise, W.noise_mask, W.seed, (uint64_t)W.np + d, D.iters);
      if (!(e > 0.0 && e <= 1e6)) { E.t = tnow; E.code = VOLTANA_ITEM_E_INPUT; D.dead = true; return; }
      dur = mul(dur, e);
    }
    double t0 = tnow;
    if ((V & 2) && W.wo) {  // blocking frequency set on a level change [C3]
      if (k != (int)W.dl_cur[d] && W.fs_ov > 0.0) { t0 = add(tnow, W.fs_ov); fl |= 2u; }
      W.dl_cur[d] = (uint32_t)k;
    }
    if ((V & 2)) log_iter(O, W.it_on, W.it_base, W.np + (uint32_t)d, D.iters, tnow, dur, D.nreq, D.nkv, k, fl);
    D.end = add(t0, dur);
    D.busy = true;
    if ((V & 2) && W.itlm) {  // ITL modes (E3): gap e_i - e_{i-1} of this iteration, if continuous
      W.dl_vc[d] += (cont && sub(D.end, tnow) > W.slo_itl) ? 1u : 0u;
      const size_t ro = (size_t)d * (W.rmask + 1u) + (D.iters & W.rmask);
      W.re[ro] = D.end;
      W.rc[ro] = W.dl_vc[d];
    }
    C.ebusy = add(C.ebusy, mul(bpow(W, 1, W.dyn[W.K + k], D.nreq), dur));  // W*ms, A23
    C.bms = add(C.bms, dur);
    if (k == (int)W.K - 1) C.top = add(C.top, dur);
    D.cur = D.iters;
    D.iters += 1u;
    D.bcur = L.wheel[D.cur & nbm];  // final now: read at the END of this iteration
  }
}

// ------------------------------------------------------------------ deferred ITL accounting
__device__ __forceinline__ double itl_marker(uint32_t slot) {  // "list continues": NaN with the slot
  return __longlong_as_double((long long)(0xFFF8000000000000ull | slot));
}
// The ITL accounting of completion-log entries E[0, m) on the calling warp (all 32 lanes):
// c_ok / c_both are this lane's counts, sd is lane d's running sum for decode instance d —
// the sequential sum in completion order (A30, A37), continued across calls.
__device__ __noinline__ void itl_pass(uint32_t m, int ND, double slo, uint32_t max_hops, const CEnt *E, const Node *node,
                         ItlScratch &S, double &sd, uint32_t &c_ok, uint32_t &c_both) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t c0 = 0; c0 < m; c0 += 32u) {
    const uint32_t q = c0 + lane;
    CEnt e;
    e.td = 0.0; e.head = NIL; e.d = 0u;
    if (q < m) e = E[q];
    const double td = e.td;
    uint32_t id = e.head, cnt = 0u;
    const uint32_t dd = e.d;
#pragma unroll
    for (uint32_t jj = 0; jj < ITL_CAP; ++jj) {
      if (id != NIL) {
        const Node nd = node[id];
        const double x = div(sub(td, fabs(nd.tf)), (double)(node_out(nd) - 1u));
        const bool ok = x <= slo;
        c_ok += ok;
        c_both += ok && nd.tf > 0.0;
        S.v[lane][jj] = x;
        cnt++;
        id = nd.next;
      }
    }
    // regroup: the values of instance d, in log order, go to seq[base_d ...] (exclusive scans)
    const uint32_t cp = cnt + (id != NIL ? 1u : 0u);  // values + a continuation marker
    uint32_t pos = 0u, base = 0u, my_base = 0u, my_tot = 0u, b = 0u;
#pragma unroll
    for (int d = 0; d < NI; ++d) {
      if (d >= ND) break;
      const uint32_t c = dd == (uint32_t)d ? cp : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      const uint32_t tot = __shfl_sync(FULL, incl, 31);
      if (dd == (uint32_t)d) { pos = incl - c; b = base; }
      if (lane == (uint32_t)d) { my_base = base; my_tot = tot; }
      base += tot;
    }
    double *o = &S.seq[b + pos];
    for (uint32_t jj = 0; jj < cnt; ++jj) o[jj] = S.v[lane][jj];
    if (id != NIL) {
      o[cnt] = itl_marker(lane);
      S.td[lane] = td;
      S.id[lane] = id;
    }
    __syncwarp();
    if (lane < (uint32_t)ND) {  // instance `lane` adds its values in log order (A37)
      for (uint32_t r = 0; r < my_tot; ++r) {
        const double v = S.seq[my_base + r];
        if (v == v) {
          sd = add(sd, v);
        } else {  // a list longer than ITL_CAP: its rest, in order
          const uint32_t slot = (uint32_t)(__double_as_longlong(v) & 0xFFFFu);
          const double t = S.td[slot];
          uint32_t rr = S.id[slot];
          for (uint32_t hop = 0; rr != NIL && hop < max_hops; ++hop) {
            const Node nd = node[rr];
            const double itl = div(sub(t, fabs(nd.tf)), (double)(node_out(nd) - 1u));
            sd = add(sd, itl);
            const bool ok = itl <= slo;
            c_ok += ok;
            c_both += ok && nd.tf > 0.0;
            rr = nd.next;
          }
        }
      }
    }
    __syncwarp();
  }
}

// dec_advance for every lane of the warp (converged call site). A lane whose completion-log
// chunk is full stops before its next END; the warp then hands out new chunks in lane order
// (one ballot, no atomics) and those lanes continue. When the warp's log is full it is first
// run through the ITL pass (every entry logged so far precedes every later one of the same
// instance, so the per-instance sums stay in completion order).
template <int V, bool F, class WS>
__device__ __forceinline__ void dec_advance_all(Dec &D, int d, const Lane &L, WS &W, double t_lim, Err &E,
                                                const voltana_outputs &O, int ND, ItlScratch &S, double &sd,
                                                uint32_t &c_ok, uint32_t &c_both) {
  const uint32_t lane = threadIdx.x & 31u;
  bool go = true;
  for (;;) {
    if (go) dec_advance<V, F>(D, d, L, W, t_lim, E, O);  // the one call site (code size)
    if (V & 2) break;
    const unsigned nm = wballot(D.lneed);
    if (nm == 0u) break;
    const uint32_t top = W.clog_m;
    go = D.lneed;
    if (top + CLOG_CHUNK * (uint32_t)__popc(nm) > CLOG_CAP) {  // flush through the ITL pass
      if (lane < (uint32_t)ND)
        for (uint32_t q = D.lpos; q < D.lend; ++q) { CEnt ce; ce.td = 0.0; ce.head = NIL; ce.d = 0u; L.clog[q] = ce; }
      __syncwarp();
      itl_pass(top, ND, W.slo_itl, W.max_steps, L.clog, L.node, S, sd, c_ok, c_both);
      if (lane < (uint32_t)ND) { D.lpos = lane * CLOG_CHUNK; D.lend = D.lpos + CLOG_CHUNK; }
      __syncwarp();
      if (lane == 0) W.clog_m = (uint32_t)ND * CLOG_CHUNK;
    } else {
      if (D.lneed) {
        D.lpos = top + CLOG_CHUNK * (uint32_t)__popc(nm & ((1u << lane) - 1u));
        D.lend = D.lpos + CLOG_CHUNK;
      }
      __syncwarp();
      if (lane == 0) W.clog_m = top + CLOG_CHUNK * (uint32_t)__popc(nm);
    }
    __syncwarp();
    D.lneed = false;
  }
}

// Append request i (routed at its first-token time) to instance d's admission queue.
__device__ __forceinline__ void dec_push(Dec &D, const Lane &L, uint32_t i, double tf, uint32_t in,
                                         uint32_t out, uint32_t nbm) {
  D.pn += 1u;
  D.pkv += in + 1u;
  if (D.qt == NIL) {  // (K4a wrote node i with next = NIL)
    D.qh = i;
    prefetch_l1(L.wheel + ((D.iters + out - 2u) & nbm));  // its bucket at the next START
    D.qhn.tf = tf; D.qhn.next = NIL; D.qhn.io = (uint32_t)(uint16_t)in | (uint32_t)(uint16_t)out << 16;
  } else {
    L.node[D.qt].next = i;
    if (D.qt == D.qh) D.qhn.next = i;  // keep the register copy coherent
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
  const uint32_t mhi = __reduce_min_sync(FULL, hi);
  const bool c1 = valid && hi == mhi;
  const uint32_t lo = c1 ? (uint32_t)b : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(FULL, lo);
  const unsigned m = wballot(c1 && lo == mlo);
  return m ? ffs0(m) : -1;
}

// Lanes holding the minimum of a signed double among lanes with `valid` (bitmask). -0 is
// folded into +0 first so the set equals the `==` set of the oracle.
__device__ __forceinline__ unsigned min_set(double v, bool valid) {
  if (v == 0.0) v = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint64_t key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // total order as unsigned
  const uint32_t hi = valid ? (uint32_t)(key >> 32) : 0xffffffffu;
  const uint32_t mhi = __reduce_min_sync(FULL, hi);
  const bool c1 = valid && hi == mhi;
  const uint32_t lo = c1 ? (uint32_t)key : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(FULL, lo);
  return wballot(c1 && lo == mlo);
}

__device__ __forceinline__ void write_status(const SimParams &P, uint32_t s, uint32_t n_req, uint32_t status) {
  if ((threadIdx.x & 31u) == 0) {
    voltana_result R = voltana_result{};
    R.status = status;
    R.n_requests = n_req;
    P.out[s] = R;
  }
}

// ------------------------------------------------------------------ the merged route stream
// Number of entries of window q (one key per lane, ascending by lane) that precede key x in
// the (time, prefill instance, id) drain order (A18): keys below x, and equal keys when
// stream q comes first (q < p). Binary search by shuffles: 6 probes.
__device__ __forceinline__ uint32_t cnt_before(double kq, double x, bool q_first) {
  uint32_t c = 0u;
#pragma unroll
  for (uint32_t s = 16u; s >= 1u; s >>= 1) {
    const double y = __shfl_sync(FULL, kq, (int)(c + s - 1u));
    if (y < x || (q_first && y == x)) c += s;
  }
  const double y = __shfl_sync(FULL, kq, 31);
  if (c == 31u && (y < x || (q_first && y == x))) c = 32u;
  return c;
}

// Refill the route window: the next (up to) 32 requests of the merge of the N_P prefill
// streams in (time, instance, id) order (A18; within a stream FCFS = id order). Lane l
// loads entry l of every stream's next 32; its merged rank is l plus, for every other stream,
// the count of that window's entries before it. The first 32 merged entries all lie in the
// streams' first 32 (merge path), so ranks < 32 are exact. Returns the entries written.
__device__ __noinline__ uint32_t route_refill(RouteWin &R, const Node *node, uint32_t NP) {
  const uint32_t lane = threadIdx.x & 31u;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double key[NI], tf[NI];
  uint32_t io[NI], id[NI];
  __syncwarp();  // every lane has read the old window before any lane overwrites it
#pragma unroll
  for (int q = 0; q < NI; ++q) {
    key[q] = INF; tf[q] = 0.0; io[q] = 0u; id[q] = NIL;
    if ((uint32_t)q < NP) {
      const uint32_t x = R.sbase[q] + lane * NP;
      if (x < R.send[q]) {
        const Node nd = node[x];
        tf[q] = nd.tf; io[q] = nd.io; key[q] = fabs(nd.tf); id[q] = x;
      }
    }
  }
  uint32_t total = 0u, used[NI];
#pragma unroll
  for (int p = 0; p < NI; ++p) {
    used[p] = 0u;
    if ((uint32_t)p >= NP) continue;
    uint32_t r = lane;
#pragma unroll
    for (int q = 0; q < NI; ++q) {
      if ((uint32_t)q >= NP || q == p) continue;
      r += cnt_before(key[q], key[p], q < p);
    }
    const bool take = id[p] != NIL && r < 32u;
    if (take) { RouteEnt e; e.tf = tf[p]; e.id = id[p]; e.io = io[p]; R.ring[r] = e; }
    used[p] = (uint32_t)__popc(wballot(take));
    total += used[p];
  }
  __syncwarp();
  uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
  for (int p = 0; p < NI; ++p) {
    if ((uint32_t)p >= NP) continue;
    const uint32_t b = R.sbase[p] + used[p] * NP;
    lo = b < lo ? b : lo;
    const uint32_t e = b + 32u * NP < R.send[p] ? b + 32u * NP : R.send[p];
    hi = e > hi ? e : hi;
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < NI; ++p)
    if ((uint32_t)p < NP && lane == (uint32_t)p) R.sbase[p] += used[p] * NP;
  // the next window's nodes towards L2 (one 128-B line = 8 nodes per lane)
  if (hi > lo)
    for (uint32_t x = lo + lane * 8u; x < hi && x < lo + 64u * 8u; x += 256u) prefetch_l2(node + x);
  __syncwarp();
  return total;
}

// EcoRoute's case analysis (A13-A17) from the feasibility ballot of the what-if
// lanes (bit 2Kd + k: level k feasible for instance d now; bit 2Kd + K + k: after adding the
// request). Every lane computes the same decision; MHz from the staged ladder. ND is a
// template parameter so the per-instance loops are straight-line code.
template <int ND>
__device__ __forceinline__ void eco_from_levels(const int *kn, const int *ka, const int32_t *mhz, int32_t delta,
                                                uint32_t &cursor, int &dsel, int &cse) {
  int fn[ND], fa[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    fn[d] = mhz[kn[d]];   // f: lowest feasible level now (A10, A11)
    fa[d] = mhz[ka[d]];   // f': after the hypothetical addition (A12)
  }
  int mnAll = fn[0], maAll = fa[0], mnU = 0x7fffffff, maR = 0x7fffffff;
  unsigned Rm = 0u;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    if (fa[d] > fn[d]) { Rm |= 1u << d; maR = fa[d] < maR ? fa[d] : maR; }   // crossed (A13)
    else mnU = fn[d] < mnU ? fn[d] : mnU;
    mnAll = fn[d] < mnAll ? fn[d] : mnAll;
    maAll = fa[d] < maAll ? fa[d] : maAll;
  }
  constexpr unsigned all = (1u << ND) - 1u;
  // candidate set: argmin of f over U (3), over everybody (1, 2, 4), or of f' (5)
  int key = mnAll;
  bool use_fa = false, only_u = false;
  if (Rm == 0u) {
    cse = 1;                 // nobody crosses: the lowest current frequency (1 unique, 2 tied)
  } else if (Rm != all) {    // some cross: the gap decides (A14, A15)
    if ((long long)mnU - (long long)maR <= (long long)delta) { key = mnU; only_u = true; cse = 3; }
    else cse = 4;
  } else {                   // everybody crosses: the lowest new frequency
    key = maAll; use_fa = true; cse = 5;
  }
  unsigned inset = 0u;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const int v = use_fa ? fa[d] : fn[d];
    if (v == key && !(only_u && ((Rm >> d) & 1u))) inset |= 1u << d;
  }
  if (cse == 1 && __popc(inset) > 1) cse = 2;
  // round robin among the candidate set from the cursor (A17)
  const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & all;
  dsel = (int)wrap_nd(cursor + (uint32_t)ffs0(rot), (uint32_t)ND);
  if (__popc(inset) >= 2) cursor = wrap_nd((uint32_t)dsel + 1u, (uint32_t)ND);
}

// lowest feasible level of a K-bit feasibility mask, else K-1 (A2)
__device__ __forceinline__ int lowest_of(unsigned m, int K) { return ffs0(m | (1u << (K - 1))); }

template <int ND>
__device__ __forceinline__ void eco_cases_nd(unsigned fm, int K, const int32_t *mhz, int32_t delta,
                                             uint32_t &cursor, int &dsel, int &cse) {
  const unsigned km = (1u << K) - 1u;
  int kn[ND], ka[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    kn[d] = lowest_of((fm >> (2 * K * d)) & km, K);
    ka[d] = lowest_of((fm >> (2 * K * d + K)) & km, K);
  }
  eco_from_levels<ND>(kn, ka, mhz, delta, cursor, dsel, cse);
}

// N_D = 2, K <= ECO_LUT_K: the whole case analysis as a table over (f, f' of both instances,
// cursor), built per scenario by the same function (so it is the same decision), read with one
// shared-memory byte load per route: dsel | cse << 1 | new cursor << 4.
__device__ __forceinline__ void eco_lut_build(uint8_t *lut, int K, const int32_t *mhz, int32_t delta) {
  const int K2 = K * K, n = K2 * K2 * 2;
  for (int e = (int)(threadIdx.x & 31u); e < n; e += 32) {
    const int c0 = e / (2 * K2), c1 = (e / 2) % K2;
    int kn[2] = {c0 / K, c1 / K}, ka[2] = {c0 % K, c1 % K};
    uint32_t cur = (uint32_t)(e & 1);
    int dsel, cse;
    eco_from_levels<2>(kn, ka, mhz, delta, cur, dsel, cse);
    lut[e] = (uint8_t)(dsel | cse << 1 | cur << 4);
  }
}

__device__ __forceinline__ void eco_cases(unsigned fm, int ND, int K, const int32_t *mhz, int32_t delta,
                                          uint32_t &cursor, int &dsel, int &cse) {
  switch (ND) {
    case 2: eco_cases_nd<2>(fm, K, mhz, delta, cursor, dsel, cse); break;
    case 3: eco_cases_nd<3>(fm, K, mhz, delta, cursor, dsel, cse); break;
    case 4: eco_cases_nd<4>(fm, K, mhz, delta, cursor, dsel, cse); break;
    case 5: eco_cases_nd<5>(fm, K, mhz, delta, cursor, dsel, cse); break;
    case 6: eco_cases_nd<6>(fm, K, mhz, delta, cursor, dsel, cse); break;
    case 7: eco_cases_nd<7>(fm, K, mhz, delta, cursor, dsel, cse); break;
    default: eco_cases_nd<8>(fm, K, mhz, delta, cursor, dsel, cse); break;
  }
}

// ------------------------------------------------------------------ K4a: prefill instance p
// Prefill instance p of one scenario on a whole warp. The instance's decisions are a serial
// chain over batches (O7 START_PREFILL): everything on that chain is computed redundantly by
// all lanes, so control flow stays uniform. The lanes hold a window of the instance's next 32
// queued requests (arrival, in, out, and the inclusive prefix sum of in):
//  - batch formation at time ts from head lane h is one ballot: candidate j > h joins iff it
//    and every candidate before it has arrived by ts and the tokens from h through j fit in B;
//    the first failing lane ends the batch and says whether it is a backlog (A5, A6);
//  - the per-request TTFT accounting of O5 runs once per window for all its batches: each lane
//    holds its batch's end time, the report sum is added in FCFS order (A37), the counts are
//    ballots, and each lane writes its request's node.
// A batch longer than the window (> 32 requests) takes the general path (rounds of 32).
struct PCtxS {   // per-warp context in shared memory (uniform over the warp)
  double tgt_ttft, slo_ttft, p_idle, tdp, uh_p, ctrl_iv, fs_ov;
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

template <bool F>
__device__ __forceinline__ double ttft_at(const PCtxS &C, int k, uint32_t nbt) {
  if (F || C.ptiles <= 1u) return ttft_pred(C.tt[2 * k], C.tt[2 * k + 1], nbt);
  // prefill tiles (F1): the batch's tile row of the profile tables
  const size_t o = (size_t)ptile_of(nbt, C.W, C.ptiles, C.pcut) * C.kp + C.lad[k];
  return ttft_pred(__ldg(C.a1g + o), __ldg(C.c1g + o), nbt);
}

template <bool F>
__device__ int lowest_ttft(const PCtxS &C, uint32_t nbt, double budget, double *pred) {
  const int K = (int)C.K;
  if (!F && C.mono_tt && K > 8) {
    int lo = 0, hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ttft_at<F>(C, mid, nbt) <= budget) hi = mid; else lo = mid + 1;
    }
    const int k = lo < K ? lo : K - 1;
    *pred = ttft_at<F>(C, k, nbt);
    return k;
  }
  for (int k = 0; k < K - 1; ++k) {
    const double p = ttft_at<F>(C, k, nbt);
    if (p <= budget) { *pred = p; return k; }
  }
  *pred = ttft_at<F>(C, K - 1, nbt);
  return K - 1;
}

template <bool F>
__device__ int energy_ttft(const PCtxS &C, uint32_t nbt, double budget, double *pred) {
  const int K = (int)C.K;
  int best = -1;
  double be = 0.0, bt = 0.0;
  for (int k = 0; k < K; ++k) {
    const double t = ttft_at<F>(C, k, nbt);
    if (!(t <= budget)) continue;
    const double e = mul(bpow_u(C.ut, C.p_idle, C.tdp, C.uh_p, 0, C.dyn[k], nbt), t);
    if (best < 0 || e < be) { best = k; be = e; bt = t; }
  }
  if (best < 0) { best = K - 1; bt = ttft_at<F>(C, K - 1, nbt); }
  *pred = bt;
  return best;
}

struct PState {   // uniform state of one prefill instance (every lane holds the same values) ...
  double ebusy, bms, top, sttft, tlast, errt, tfree, last;
  uint64_t h;
  uint32_t iters, ttft_ok, itl_ok, both, errc, cur, ndec;
  uint64_t tok;   // ... except the input checks of the requests this lane accounted (A40)
  bool vok;
};

// Input checks of request i (A40): 1 <= in <= 65535, 1 <= out <= max_out, 0 <= arrival < 1e9,
// arrivals non-decreasing (prev = arrival of request i - 1).
__device__ __forceinline__ bool req_ok(double a, uint32_t x, uint32_t o, uint32_t max_out, uint32_t i, double prev) {
  return x >= 1u && x <= 65535u && o >= 1u && o <= max_out && a >= 0.0 && a < 1e9 && !(i > 0u && a < prev);
}

// O7 decision for a batch of nbt tokens starting at ts, head arrival a0: EcoFreq,
// duration, energy (A23). false: per-item error recorded in S.
template <int V, bool F>
__device__ __forceinline__ bool pa_decide(const SimParams &P, const PCtxS &C, PState &S, uint32_t p, double ts,
                                          double a0, uint32_t nbt, bool backlog, double &end) {
  double budget = sub(C.tgt_ttft, sub(ts, a0));  // A4: SLO minus the oldest request's wait
  budget = budget > 0.0 ? budget : 0.0;
  const uint32_t K = C.K;
  double dur;
  int k;
  uint32_t fl = backlog ? 4u : 0u;
  if ((V & 2) && C.wo && !(sub(ts, S.last) >= C.ctrl_iv)) {  // window gating: keep the running level [C1]
    k = (int)S.cur;
    dur = ttft_at<F>(C, k, nbt);
  } else {
    fl |= 1u;
    if (backlog) { k = (int)K - 1; dur = ttft_at<F>(C, k, nbt); }
    else if ((V & 1) && C.ctrl) k = energy_ttft<F>(C, nbt, budget, &dur);  // B4
    else k = lowest_ttft<F>(C, nbt, budget, &dur);
    S.h = fold(S.h, 1, (uint64_t)p, (uint64_t)k, 0);
    if ((V & 2) && C.wo) { S.last = ts; S.ndec++; }
  }
  const uint32_t jit = S.iters++;
  if (!(dur > 0.0)) { S.errt = ts; S.errc = VOLTANA_ITEM_E_CONTRACT; return false; }
  if ((V & 2) && C.noise) {  // true time = prediction x lognormal factor [D1]
    const double e = noise_at(C.noise, C.noise_mask, C.seed, p, jit);
    if (!(e > 0.0 && e <= 1e6)) { S.errt = ts; S.errc = VOLTANA_ITEM_E_INPUT; return false; }
    dur = mul(dur, e);
  }
  double t0 = ts;
  if ((V & 2) && C.wo) {  // blocking frequency set on a level change [C3]
    if (k != (int)S.cur && C.fs_ov > 0.0) { t0 = add(ts, C.fs_ov); fl |= 2u; }
    S.cur = (uint32_t)k;
  }
  if ((V & 2) && (threadIdx.x & 31u) == 0) log_iter(P.o, C.it_on, C.it_base, p, jit, ts, dur, nbt, 0u, k, fl);
  end = add(t0, dur);
  S.ebusy = add(S.ebusy, mul(bpow_u(C.ut, C.p_idle, C.tdp, C.uh_p, 0, C.dyn[k], nbt), dur));  // W*ms (A23)
  S.bms = add(S.bms, dur);
  if (k == (int)K - 1) S.top = add(S.top, dur);
  S.tfree = end;
  S.tlast = end;
  return true;
}

// O5 for lanes [0, n): request base + lane*NP (arrival a, in x, out o) finished prefill at e.
template <int V>
__device__ __forceinline__ void pa_account(const SimParams &P, PCtxS &C, PState &S, Node *node, const double *arr,
                                           uint32_t base, uint32_t NP, uint32_t n, double e, double a, uint32_t x,
                                           uint32_t o) {
  if (n == 0u) return;
  const uint32_t lane = threadIdx.x & 31u;
  const bool valid = lane < n;
  const uint32_t i = base + lane * NP;
  if (valid) {  // every request is accounted exactly once: its input checks (A40)
    const double prev = i > 0u ? arr[i - 1u] : 0.0;
    S.vok = S.vok && req_ok(a, x, o, P.max_out, i, prev);
    S.tok += (uint64_t)x + o;
  }
  const double ttft = valid ? sub(e, a) : 0.0;  // A26
  const bool ok = valid && ttft <= C.slo_ttft;
  __syncwarp();
  C.wt[lane] = ttft;
  __syncwarp();
  for (uint32_t b = 0; b < n; b += 8u) {  // the report sum in FCFS order (A37)
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = C.wt[(b + u) & 31u];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b + u < n) S.sttft = add(S.sttft, v[u]);
  }
  S.ttft_ok += __popc(wballot(ok));
  const bool one = valid && o == 1u;  // first token came from prefill: done (A8, A30)
  S.itl_ok += __popc(wballot(one));
  S.both += __popc(wballot(one && ok));
  if ((V & 2) && C.rq_on && valid) {  // per-request record (E1)
    P.o.req_tfirst[C.rq_base + i] = e;
    if (o == 1u) {
      P.o.req_tdone[C.rq_base + i] = e; P.o.req_itl[C.rq_base + i] = 0.0;
      P.o.req_decode[C.rq_base + i] = 0xFF; P.o.req_case[C.rq_base + i] = 0xFF;
    }
  }
  if (valid) {  // the request's node: first-token time with the TTFT verdict in its sign
    Node me;
    me.tf = ok ? e : -e;
    me.next = NIL;
    me.io = (uint32_t)(uint16_t)x | (uint32_t)(uint16_t)o << 16;
    node[i] = me;
  }
}

// General path for one batch starting at request nxt (any length): candidates in rounds of 32,
// accounting in chunks of 32. Returns the next unbatched request, or NIL on an error.
template <int V, bool F>
__device__ uint32_t pa_batch_general(const SimParams &P, PCtxS &C, PState &S, Node *node, const double *arr,
                                     const uint32_t *inl, const uint32_t *outl, uint32_t N, uint32_t p,
                                     uint32_t NP, uint32_t nxt) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t lane = threadIdx.x & 31u, B = C.B;
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
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, ps, o);
      if (lane >= (uint32_t)o) ps += y;
    }
    const bool arrived = av <= ts;
    const unsigned m = wballot(arrived && !(nbt + ps > B));
    const uint32_t f = m == FULL ? 32u : (uint32_t)ffs0(~m);
    if (f > 0u) {
      nbt += wshfl(ps, (int)f - 1);
      cnt += f;
      id += f * NP;
    }
    if (f < 32u) {
      backlog = wshfl(arrived, (int)f);
      break;
    }
  }
  double end;
  if (!pa_decide<V, F>(P, C, S, p, ts, a0, nbt, backlog, end)) return NIL;
  for (uint32_t q0 = 0; q0 < cnt; q0 += 32u) {
    const uint32_t nv = cnt - q0 < 32u ? cnt - q0 : 32u;
    const uint32_t i = nxt + (q0 + lane) * NP;
    double a = 0.0;
    uint32_t x = 0u, o = 0u;
    if (lane < nv) { a = arr[i]; x = inl[i]; o = outl[i]; }
    pa_account<V>(P, C, S, node, arr, nxt + q0 * NP, NP, nv, end, a, x, o);
  }
  return id;
}

constexpr uint32_t PA_PF_L2 = 1024;   // bulk L2 prefetch of the trace this many entries ahead
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

template <int V, bool F>
__device__ void prefill_warp(const SimParams &P, PCtxS &C, Node *node, const double *arr, const uint32_t *inl,
                             const uint32_t *outl, uint32_t N, uint32_t p, uint32_t NP, uint64_t h0, PaRes &R) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t lane = threadIdx.x & 31u, B = C.B;
  PState S;
  S.ebusy = S.bms = S.top = S.sttft = S.tlast = S.tfree = 0.0;
  S.errt = INF;
  S.last = -INF;             // [C1] time of the last decision
  S.h = h0;
  S.iters = S.ttft_ok = S.itl_ok = S.both = S.errc = S.ndec = 0;
  S.cur = C.K - 1u;          // [C2] running level (starts at the top)
  S.tok = 0;
  S.vok = true;
  uint32_t wbase = p;        // request of lane 0 in the window (the instance's next unbatched request)
  uint32_t pf2 = p;          // next entry to prefetch into L2
  while (wbase < N) {
    if (lane == 0)
      while (pf2 < N && pf2 < wbase + PA_PF_L2) {
        const uint32_t c = N - pf2 < PA_PF_CHUNK ? N - pf2 : PA_PF_CHUNK;
        prefetch_l2_range(arr, pf2, c, 8u);
        prefetch_l2_range(inl, pf2, c, 4u);
        prefetch_l2_range(outl, pf2, c, 4u);
        pf2 += PA_PF_CHUNK;
      }
    const uint32_t rem = (N - wbase + NP - 1u) / NP;  // requests left on this instance
    const uint32_t nwin = rem < 32u ? rem : 32u;
    const uint32_t idx = wbase + lane * NP;
    const bool v = lane < nwin;
    const double a = v ? arr[idx] : INF;  // past the trace end: "not arrived"
    const uint32_t x = v ? inl[idx] : 0u;
    const uint32_t o = v ? outl[idx] : 0u;
    uint32_t ps = x;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, ps, s);
      if (lane >= (uint32_t)s) ps += y;
    }
    __syncwarp();           // the previous window's reads are done
    C.wa[lane] = a;
    C.wps[lane] = ps;
    __syncwarp();
    double e = 0.0;         // this lane's batch end, once its batch has started
    uint32_t hl = 0;        // head lane of the next batch
    bool err = false, general = false;
    while (hl < nwin) {
      const double a0 = C.wa[hl];
      const double ts = S.tfree > a0 ? S.tfree : a0;  // START: instance idle and queue non-empty
      const uint32_t psb = hl ? C.wps[hl - 1u] : 0u;  // tokens before the head
      const bool arrived = a <= ts;
      const bool take = lane > hl && arrived && !(ps - psb > B);
      const unsigned fails = wballot(lane > hl && !take);
      if (fails == 0u) {    // a full window of arrivals that all fit: the batch may run on
        general = hl == 0u; // more than 32 requests: the general path; else re-window at the head
        break;
      }
      const uint32_t f = (uint32_t)ffs0(fails);  // first candidate not taken
      const bool backlog = C.wa[f] <= ts;         // arrived but does not fit (A5)
      const uint32_t nbt = C.wps[f - 1u] - psb;
      double end;
      if (!pa_decide<V, F>(P, C, S, p, ts, a0, nbt, backlog, end)) { err = true; break; }
      if (lane >= hl && lane < f) e = end;
      hl = f;
    }
    pa_account<V>(P, C, S, node, arr, wbase, NP, hl, e, a, x, o);  // O5 for the window's batches
    wbase += hl * NP;
    if (err) break;
    if (general) {
      const uint32_t nx = pa_batch_general<V, F>(P, C, S, node, arr, inl, outl, N, p, NP, wbase);
      if (nx == NIL) break;
      wbase = nx;
    }
  }
  // the requests after an error were not accounted: their input checks (A40)
  for (uint32_t i = wbase + lane * NP; i < N; i += 32u * NP) {
    const uint32_t x = inl[i], o = outl[i];
    S.vok = S.vok && req_ok(arr[i], x, o, P.max_out, i, i > 0u ? arr[i - 1u] : 0.0);
    S.tok += (uint64_t)x + o;
  }
  uint64_t tok = S.tok;
  for (int o = 16; o > 0; o >>= 1) tok += __shfl_xor_sync(FULL, tok, o);
  R.ebusy = S.ebusy; R.bms = S.bms; R.top = S.top; R.sttft = S.sttft; R.tlast = S.tlast; R.errt = S.errt;
  R.h = S.h; R.iters = S.iters; R.ttft_ok = S.ttft_ok; R.itl_ok = S.itl_ok; R.both = S.both; R.errc = S.errc;
  R.ndec = S.ndec; R.send = wbase < N ? wbase : N;
  R.valid = __all_sync(FULL, S.vok) ? 1u : 0u;
  R.tok = tok;
  if ((V & 2) && C.it_on && lane == 0) P.o.iter_count[C.it_base / P.o.iter_cap + p] = S.iters;
}

// The node range of scenario s must hold exactly its trace when the caller gave offsets.
__device__ __forceinline__ bool node_range_ok(const SimParams &P, uint32_t s, uint64_t N) {
  return !P.node_offset || P.node_offset[s + 1] - P.node_offset[s] == N;
}

template <int V, bool F>
__global__ void __launch_bounds__(PA_THREADS, PA_MIN_BLOCKS) prefill_kernel(const __grid_constant__ SimParams P) {
  __shared__ PCtxS cs[PA_THREADS / 32];
  const uint64_t total = (uint64_t)P.n * P.np_max;
  const uint64_t wpb = blockDim.x / 32u;
  const uint64_t x0 = blockIdx.x * wpb + threadIdx.x / 32u;
  const uint32_t lane = threadIdx.x & 31u;
  PCtxS &C = cs[threadIdx.x / 32u];
  for (uint64_t x = x0; x < total; x += (uint64_t)gridDim.x * wpb) {
    const uint32_t s = (uint32_t)(x / P.np_max), p = (uint32_t)(x - (uint64_t)s * P.np_max);
    if (!(P.trace_id[s] < P.n_traces && P.slo_id[s] < P.n_slos && P.layout_id[s] < P.n_layouts &&
          P.grid_id[s] < P.n_grids && P.profile_id[s] < P.n_profiles))
      continue;  // K4b writes E_INPUT
    const voltana_layout &LY = P.lay[P.layout_id[s]];
    const uint32_t NP = (uint32_t)LY.n_p;
    if (p >= NP) continue;
    const uint32_t tr = P.trace_id[s];
    const uint64_t off = P.offset[tr];
    const uint64_t N64 = P.offset[tr + 1] - off;
    if (!(N64 <= P.max_requests) || !node_range_ok(P, s, N64)) continue;  // K4b writes E_INPUT
    const voltana_slo &SL = P.slo[P.slo_id[s]];
    const uint32_t g = P.grid_id[s], pr = P.profile_id[s];
    const voltana_grid &GR = P.grid[g];
    const DevProfile &PR = P.prof[pr];
    uint32_t rq_on = 0u;
    uint64_t rq_base = 0;
    if ((V & 2) && P.o.req_offset) {
      rq_base = P.o.req_offset[s];
      const uint64_t len = P.o.req_offset[s + 1] - rq_base;
      if (len != 0 && len != N64) continue;  // K4b writes E_INPUT
      rq_on = len != 0;
    }
    const double *rt = P.rtab + ((size_t)g * MAX_PROFILES + pr) * RT_STRIDE;
    if (lane == 0) {
      C.rq_on = rq_on; C.rq_base = rq_base;
      C.it_on = (V & 2) && P.o.iter_offset ? 1u : 0u;
      C.it_base = C.it_on ? P.o.iter_offset[s] : 0;
      C.tgt_ttft = mul(SL.scale, SL.ttft_ms);  // A3
      C.slo_ttft = SL.ttft_ms;
      C.p_idle = PR.p_idle; C.tdp = PR.tdp; C.uh_p = PR.uh[0];
      C.ctrl_iv = LY.ctrl_interval_ms; C.fs_ov = LY.freq_overhead_ms;
      C.a1g = PR.a1; C.c1g = PR.c1;
      C.ut = P.utab + (size_t)pr * 2 * SIM_UTAB;
      C.noise = LY.exec_noise; C.noise_mask = LY.noise_len - 1u;
      C.lad = GR.level;
      C.B = LY.max_batch_tokens; C.K = (uint32_t)GR.k; C.W = (uint32_t)PR.tile_w; C.kp = (uint32_t)PR.k;
      C.ptiles = (uint32_t)PR.n_ptiles; C.pcut = PR.pcut;
      C.ctrl = (uint32_t)LY.ctrl_mode;
      C.wo = (V & 2) && (LY.ctrl_interval_ms > 0.0 || LY.freq_overhead_ms > 0.0) ? 1u : 0u;
      C.seed = P.hash_seed[s];
      // coefficient-monotone TTFT rows allow the exact binary search (A32); tiled TTFT: scan (F1)
      bool mt = PR.n_ptiles <= 1;
      for (uint32_t k = 0; mt && k + 1 < (uint32_t)GR.k; ++k)
        mt = rt[2 * k + 2] <= rt[2 * k] && rt[2 * k + 3] <= rt[2 * k + 1];
      C.mono_tt = mt;
    }
    for (uint32_t k = lane; k < (uint32_t)GR.k; k += 32u) {
      C.tt[2 * k] = rt[2 * k];
      C.tt[2 * k + 1] = rt[2 * k + 1];
      C.dyn[k] = rt[2 * VOLTANA_MAX_LEVELS + k];
    }
    __syncwarp();
    Node *node = (Node *)node_base(P, s);
    PaRes R;
    prefill_warp<V, F>(P, C, node, P.arrival + off, P.in_len + off, P.out_len + off, (uint32_t)N64, p, NP,
                       P.hash_seed[s], R);
    __syncwarp();  // the next item of this warp rewrites C
    if (lane == 0) P.pares[(size_t)s * NI + p] = R;
  }
}

// ------------------------------------------------------------------ K4b: routing + decode lanes
template <int V, bool F, class WS>
__device__ void run_scenario(const SimParams &P, uint32_t s, char *slot, uint4 *wheels, WS &W, ItlScratch &S,
                             uint32_t sid) {
  const int lane = (int)(threadIdx.x & 31u);
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

  // ---------------------------------------------------------------- device validation (A40)
  // the per-request checks ran in K4a (each prefill warp over its stream); here their results
  // V & 4: every layout of the launch is N_D = 2 EcoRoute on a ladder of <= 5 levels (host-checked):
  // the route loop keeps only the what-if lanes and the decision table (fewer live registers)
  const int NP = LY.n_p, ND = (V & 4) ? 2 : LY.n_d;
  uint32_t tok_total;
  {
    bool ok = N64 <= P.max_requests && Dur >= 0.0 && node_range_ok(P, s, N64);
    uint64_t tok = 0;
    if (ok && lane < NP) {
      W.pa[lane] = P.pares[(size_t)s * NI + lane];
      ok = W.pa[lane].valid != 0u;
      tok = W.pa[lane].tok;
    }
    for (int o = 16; o > 0; o >>= 1) tok += __shfl_xor_sync(FULL, tok, o);
    ok = __all_sync(FULL, ok) && tok <= 0x7fffffffull;
    if (!ok) {
      write_status(P, s, (uint32_t)N64, VOLTANA_ITEM_E_INPUT);
      return;
    }
    tok_total = (uint32_t)tok + 2u;
  }
  const uint32_t N = (uint32_t)N64;
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
    W.tin = P.in_len + off; W.tout = P.out_len + off;
    W.tau = LY.kv_transfer_ms; W.slo_itl = SL.itl_ms; W.slo_ttft = SL.ttft_ms;
    W.tgt_itl = mul(SL.scale, SL.itl_ms);   // A3
    W.tgt_ttft = mul(SL.scale, SL.ttft_ms);
    W.p_idle = PR.p_idle; W.tdp = PR.tdp; W.uh_p = PR.uh[0]; W.uh_d = PR.uh[1];
    W.a2g = PR.a2; W.b2g = PR.b2; W.c2g = PR.c2;
    W.ut = P.utab + (size_t)P.profile_id[s] * 2 * SIM_UTAB;
    W.kvcap = LY.kv_capacity; W.max_steps = tok_total;
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
  for (uint32_t k = lane; k < K; k += 32u) {
    const int lv = GR.level[k];
    W.lad[k] = (uint16_t)lv;
    W.dyn[k] = PR.dyn[lv];
    W.dyn[K + k] = PR.dyn[PR.k + lv];
    W.mhz[k] = PR.mhz[lv];
  }
  if (P.itl_smem) {
    for (uint32_t x = lane; x < T * K; x += 32u) {
      const uint32_t j = x / K, k = x - j * K;
      const size_t o = (size_t)j * PR.k + GR.level[k];
      W.it[3 * x] = PR.a2[o]; W.it[3 * x + 1] = PR.b2[o]; W.it[3 * x + 2] = PR.c2[o];
    }
  }
  {  // coefficient-monotone (non-increasing in f) tables allow the exact binary search (A32)
    bool mi = true;
    for (uint32_t x = lane; x < T * (K - 1); x += 32u) {
      const uint32_t j = x / (K - 1), k = x - j * (K - 1);
      const size_t o0 = (size_t)j * PR.k + GR.level[k], o1 = (size_t)j * PR.k + GR.level[k + 1];
      mi = mi && PR.a2[o1] <= PR.a2[o0] && PR.b2[o1] <= PR.b2[o0] && PR.c2[o1] <= PR.c2[o0];
    }
    mi = __all_sync(FULL, mi);
    if (lane == 0) W.mono_it = mi;
  }
  // N_D = 2 EcoRoute decision table (fast kernel, K <= 5)
  const bool lut_on = (V & 4) || (F && LY.policy == 0 && ND == 2 && K <= (uint32_t)ECO_LUT_K);
  __syncwarp();  // the staged ladder (W.mhz) is complete before any lane reads it
  if (lut_on) eco_lut_build(W.lut, (int)K, W.mhz, LY.delta_mhz);
  Node *node = (Node *)node_base(P, s);
  const uint64_t h0 = P.hash_seed[s];
  // ================================================================ PHASE A results (K4a)
  if (lane < NP) {
    W.rw.sbase[lane] = (uint32_t)lane;
    W.rw.send[lane] = W.pa[lane].send;
  }
  __syncwarp();

  // ================================================================ PHASE B: routing + decode lanes
  const int dl = lane < ND ? lane : 0;
  Lane L;
  L.node = node;
  L.clog = (CEnt *)slot;
  L.wheel = wheels + (size_t)dl * P.nb;
  if (lane == 0) W.clog_m = (uint32_t)ND * CLOG_CHUNK;  // the first chunk of every decode lane
  Dec D;
  D.nreq = D.nkv = D.pn = D.pkv = D.iters = D.cur = 0;
  D.klast = 0;
  D.qh = D.qt = NIL;
  D.busy = false;
  D.dead = !(lane < ND);
  D.end = 0.0;
  D.lpos = (uint32_t)lane * CLOG_CHUNK;  // first chunks: one per lane, allocated in lane order
  D.lend = D.lpos + CLOG_CHUNK;
  D.lneed = false;
  if (lane < NI) {
    DecCold &C = W.dc[lane];
    C.ebusy = C.bms = C.top = C.sitl = 0.0;
    C.h = h0; C.n_itl_ok = C.n_both = 0;
    C.far_h = C.far_hfin = NIL;
  }
  D.bcur = make_uint4(0u, 0u, 0u, 0u);
  D.qhn.tf = 0.0; D.qhn.next = NIL; D.qhn.io = 0u;
  Err dE = {INF, 0};
  double k_sd = 0.0;                                // deferred ITL pass: lane d's instance sum
  uint32_t k_ok = 0u, k_both = 0u;                  // ... and this lane's counts
  __syncwarp();

  uint64_t h_r = h0;
  uint32_t cursor = 0, steps_route = 0;
  double t_adv = -1.0;                              // decode lanes are caught up to events < t_adv
  uint32_t c_n = NIL, c_kv = 0;                     // what-if cache (general path): EcoFreq level of
  int c_lvl = 0;                                    // the lane's effective state (c_n, c_kv)
  int ka_last = 0;
  double c_en = 0.0, en_new = 0.0;                  // energy router: P*T of the cached state / successor
  const bool eco = (V & 4) || (LY.policy == 0 && ND > 1);
  const bool ens = (V & 1) && LY.policy == 2 && ND > 1;
  const bool wif = (V & 4) || (F && eco && (uint32_t)ND * 2u * K <= 32u);   // the lane-parallel what-if
  const int32_t delta = LY.delta_mhz;
  // what-if lane (fast path): instance wd, state ws (0 now, 1 after), level wk, packed
  // wk | ws << 8 | wd << 16 (NIL: an idle lane)
  uint32_t wpk = NIL;
  {
    const uint32_t wd = (uint32_t)lane / (2u * K), wr = (uint32_t)lane - wd * 2u * K;
    const uint32_t ws = wr >= K ? 1u : 0u, wk = ws ? wr - K : wr;
    if (wif && wd < (uint32_t)ND) wpk = wk | ws << 8 | wd << 16;
  }
#ifdef VT_LAT_PROBE
  // experiment: clock64 cycles per phase of the route loop, summed over the scenario
  // [0] window read / refill, [1] decode advance, [2] EcoRoute + push, [3] drain + ITL pass
  long long lp_acc[4] = {0, 0, 0, 0}, lp_t = clock64();
#define LP_MARK(q) do { const long long _n = clock64(); lp_acc[q] += _n - lp_t; lp_t = _n; } while (0)
#else
#define LP_MARK(q) do { } while (0)
#endif
  uint32_t e_n0 = 0u, e_k0 = 0u, e_n1 = 0u, e_k1 = 0u;   // V & 4: both instances' effective states
  uint32_t rcnt = route_refill(W.rw, node, (uint32_t)NP), rpos = 0;
  for (;;) {
    // the next request of the merged stream; none left: the drain marker (t = +inf, io = 0)
    RouteEnt e;
    if (rpos < rcnt) {
      e = W.rw.ring[rpos++];
    } else {
      if (rcnt == 32u) {  // a full window was consumed: the streams may hold more
        rcnt = route_refill(W.rw, node, (uint32_t)NP);
        rpos = 0;
      }
      if (rpos < rcnt) {
        e = W.rw.ring[rpos++];
      } else {
        e.tf = INF; e.id = NIL; e.io = 0u;
      }
    }
    const uint32_t out_i = e.io >> 16;
    if (out_i == 1u) continue;                      // first token from prefill: not routed (A8)
    const double t = fabs(e.tf);
    LP_MARK(0);
    // decode instances catch up to t: events strictly before t (PrefillDone drains first);
    // the drain marker (t = +inf) runs every instance to completion
    if (t != t_adv) {  // routes of one batch share t: nothing new happens between them
      dec_advance_all<V, F>(D, lane, L, W, t, dE, P.o, ND, S, k_sd, k_ok, k_both);
      t_adv = t;
      if (e.io == 0u) break;
      if (V & 4) {
        const uint32_t en = D.nreq + D.pn, ek = D.nkv + D.pkv;
        e_n0 = wshfl(en, 0); e_k0 = wshfl(ek, 0); e_n1 = wshfl(en, 1); e_k1 = wshfl(ek, 1);
      }
    }
    const uint32_t i = e.id;
    const uint32_t in_i = e.io & 0xffffu;
    LP_MARK(1);
    // ---- O8 EcoRoute
    int dsel, cse;
    if (wif) {   // one lane per (instance, state, level): the whole what-if in one ballot
      uint32_t n0, kv0;   // A9 effective state (running + pending) of the lane's instance
      if (V & 4) {        // kept in every lane (re-read after a catch-up, bumped by each push)
        const bool one = ((wpk >> 16) & 0xffu) != 0u;
        n0 = one ? e_n1 : e_n0;
        kv0 = one ? e_k1 : e_k0;
      } else {
        const uint32_t en = D.nreq + D.pn, ek = D.nkv + D.pkv;
        const int src = (int)((wpk >> 16) & 0xffu);
        n0 = wshfl(en, src & 31);
        kv0 = wshfl(ek, src & 31);
      }
      bool feas = false;
      if (wpk != NIL) {
        const uint32_t ws = (wpk >> 8) & 1u, wk = wpk & 0xffu;
        const uint32_t n = n0 + ws, kv = kv0 + (ws ? in_i + 1u : 0u);   // A12
        if (n == 0u) feas = wk == 0u;                                   // n = 0 -> level 0 (A11)
        else feas = itl_at<F>(W, tile_j<F>(W, n), (int)wk, (double)n, (double)kv) <= W.tgt_itl;
      }
      const unsigned fm = wballot(feas);
      if (F && lut_on) {   // N_D = 2: one table read (built by eco_from_levels at scenario start)
        const unsigned km = (1u << K) - 1u;
        const uint32_t c0 = (uint32_t)lowest_of(fm & km, (int)K) * K + (uint32_t)lowest_of((fm >> K) & km, (int)K);
        const uint32_t c1 = (uint32_t)lowest_of((fm >> (2 * K)) & km, (int)K) * K +
                            (uint32_t)lowest_of((fm >> (3 * K)) & km, (int)K);
        VT_CHECK(c0 < K * K && c1 < K * K && cursor < 2u && K <= (uint32_t)ECO_LUT_K);
        const uint32_t v = W.lut[((c0 * K * K + c1) << 1) | cursor];
        dsel = (int)(v & 1u);
        cse = (int)((v >> 1) & 7u);
        cursor = v >> 4;
      } else {
        eco_cases(fm, ND, (int)K, W.mhz, delta, cursor, dsel, cse);
      }
    } else if (ens) {  // ---- energy-scored router [B1-B3]
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
        double best = 0.0, tt = 0.0;
        for (int k = 0; k < (int)W.K; ++k) {
          tt = itl_at<F>(W, j, k, dn, dkv);
          if (!(tt <= W.tgt_itl)) continue;
          const double en1 = mul(bpow(W, 1, W.dyn[W.K + k], n1), tt);
          if (!feas) en_new = en1;                   // the successor's own EcoFreq-level P*T
          if (!feas || en1 < best) best = en1;
          feas = true;
        }
        tmax = tt;                                   // T at K-1
        if (!feas) en_new = mul(bpow(W, 1, W.dyn[W.K + W.K - 1], n1), tmax);
        score = sub(best, enow);
      }
      const bool any = wballot(feas) != 0u;
      const unsigned inset = any ? min_set(score, feas) : min_set(tmax, act);
      cse = any ? 6 : 7;
      const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & ((1u << ND) - 1u);
      dsel = (int)wrap_nd(cursor + (uint32_t)ffs0(rot), (uint32_t)ND);
      if (__popc(inset) >= 2) cursor = wrap_nd((uint32_t)dsel + 1u, (uint32_t)ND);
    } else if (!eco) {
      dsel = (int)cursor;
      cursor = wrap_nd(cursor + 1u, (uint32_t)ND);
      cse = 0;
    } else {     // general tables: per-lane what-if with a cached current level
      int fnow = 0x7fffffff, faft = 0x7fffffff;
      if (!F && W.mono_it && W.K > 8u && ND <= 4) {
        // long ladder, coefficient-monotone tables (A32): eight lanes per instance search its
        // levels in two rounds of parallel probes (lowest_itl_g8) instead of one lane's binary
        // search — for the cached current level when the state changed, and for the successor
        const uint32_t g = lane >> 3;
        const bool gon = g < (uint32_t)ND;
        const uint32_t en = D.nreq + D.pn, ek = D.nkv + D.pkv;  // A9 effective state (lane d < N_D)
        const bool mine_need = lane < (uint32_t)ND && en != 0u && (en != c_n || ek != c_kv);
        const uint32_t n_g = wshfl(en, (int)(g & 3u)), kv_g = wshfl(ek, (int)(g & 3u));
        const bool need_g = __shfl_sync(FULL, mine_need, (int)(g & 3u));   // every lane (no short-circuit)
        const bool need = gon && need_g;
        int kn_g = 0;
        if (__any_sync(FULL, need)) kn_g = lowest_itl_g8<F>(W, need ? n_g : 1u, kv_g, W.tgt_itl, need);
        const int ka_g = lowest_itl_g8<F>(W, n_g + 1u, kv_g + in_i + 1u, W.tgt_itl, gon);   // A12
        const int src = lane < (uint32_t)ND ? 8 * lane : 0;
        const int kn_s = __shfl_sync(FULL, kn_g, src), ka = __shfl_sync(FULL, ka_g, src);
        if (lane < (uint32_t)ND) {
          if (mine_need) { c_lvl = kn_s; c_n = en; c_kv = ek; }
          const int kn = en == 0u ? 0 : c_lvl;                                   // A10, A11
          ka_last = ka;
          fnow = W.mhz[kn];
          faft = W.mhz[ka];
        }
      } else if (lane < ND) {
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
      const int nc = __popc(wballot(cr));
      const int mn = (int)__reduce_min_sync(FULL, (unsigned)fnow);
      unsigned inset;
      if (nc == 0) {
        inset = wballot(act && fnow == mn);
        cse = __popc(inset) == 1 ? 1 : 2;
      } else if (nc < ND) {
        const int mu = (int)__reduce_min_sync(FULL, (unsigned)(act && !cr ? fnow : 0x7fffffff));
        const int mr = (int)__reduce_min_sync(FULL, (unsigned)(cr ? faft : 0x7fffffff));
        const long long g = (long long)mu - (long long)mr;  // A14, A15
        if (g <= (long long)delta) { inset = wballot(act && !cr && fnow == mu); cse = 3; }
        else { inset = wballot(act && fnow == mn); cse = 4; }
      } else {
        const int ma = (int)__reduce_min_sync(FULL, (unsigned)faft);
        inset = wballot(act && faft == ma);
        cse = 5;
      }
      // round robin among the candidate set from the cursor (A17)
      const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & ((1u << ND) - 1u);
      dsel = (int)wrap_nd(cursor + (uint32_t)ffs0(rot), (uint32_t)ND);
      if (__popc(inset) >= 2) cursor = wrap_nd((uint32_t)dsel + 1u, (uint32_t)ND);
    }
    steps_route++;
    h_r = fold(h_r, 3, (uint64_t)dsel, 0, (uint64_t)cse);
    if (V & 4) {   // the pending request joins instance dsel's effective state (A9, A12)
      if (dsel == 0) { e_n0 += 1u; e_k0 += in_i + 1u; } else { e_n1 += 1u; e_k1 += in_i + 1u; }
    }
    if (lane == dsel) {
      if (eco && !wif) { c_n = D.nreq + D.pn + 1u; c_kv = D.nkv + D.pkv + in_i + 1u; c_lvl = ka_last; }  // its new state
      if (ens) { c_n = D.nreq + D.pn + 1u; c_kv = D.nkv + D.pkv + in_i + 1u; c_en = en_new; }
      dec_push(D, L, i, e.tf, in_i, out_i, W.nb - 1u);
      if ((V & 2) && W.rq_on) { P.o.req_decode[W.rq_base + i] = (uint8_t)dsel; P.o.req_case[W.rq_base + i] = (uint8_t)cse; }
    }
    LP_MARK(2);
  }
  // every decode instance ran to completion: the deferred ITL accounting of the rest of the log
  if (!(V & 2)) {
    if (lane < ND)  // the unused rest of this lane's chunk: empty entries
      for (uint32_t q = D.lpos; q < D.lend; ++q) { CEnt ce; ce.td = 0.0; ce.head = NIL; ce.d = 0u; L.clog[q] = ce; }
    __syncwarp();
    // the scenario's log and nodes are still warm in L2: all 32 lanes gather, then sum in order
    itl_pass(W.clog_m, ND, W.slo_itl, W.max_steps, L.clog, node, S, k_sd, k_ok, k_both);
  }
  if ((V & 2) && W.it_on && lane < ND) P.o.iter_count[W.it_base / P.o.iter_cap + NP + lane] = D.iters;
  __syncwarp();

#ifdef VT_LAT_PROBE
  LP_MARK(3);
  if (P.timing && lane == 0)
    for (int q = 0; q < 4; ++q) P.timing[2 * (size_t)P.n + 4 * (size_t)s + q] = (uint64_t)lp_acc[q];
#endif
  // ================================================================ O9: record
  // first error in (time, prefill before decode, instance) order = the oracle's stop point
  const double pet = lane < NP ? W.pa[lane].errt : INF;
  const int wp = argmin_time(pet, lane < NP && pet < INF);
  const int wdd = argmin_time(dE.t, lane < ND && dE.t < INF);
  if (wp >= 0 || wdd >= 0) {
    const double tp = wp >= 0 ? W.pa[wp].errt : INF;
    const double td = wdd >= 0 ? wshfl(dE.t, wdd) : INF;
    const uint32_t cd = wshfl(dE.code, wdd >= 0 ? wdd : 0);
    write_status(P, s, N, (wp >= 0 && tp <= td) ? W.pa[wp].errc : cd);
    if (lane < ND)  // leave the wheel clean for the next scenario of this warp
      for (uint32_t b = 0; b < P.nb; ++b) wheels[(size_t)lane * P.nb + b] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  // the last decode event of instance d is the END of its last iteration (the drain ran them all)
  double tl = lane < ND && D.iters > 0u ? D.end : 0.0;
  if (lane < NP) tl = tl > W.pa[lane].tlast ? tl : W.pa[lane].tlast;
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(FULL, tl, o);
    tl = x > tl ? x : tl;
  }
  const double horizon = Dur > tl ? Dur : tl;  // A23
  // decode instances: lane d's totals gathered in instance order (A36/A37)
  double sitl = 0.0, edb = 0.0, edi = 0.0, bd = 0.0;
  const double my_sitl = (V & 2) ? 0.0 : k_sd;
#pragma unroll
  for (int d = 0; d < NI; ++d) {
    if (d < ND) {
      sitl = add(sitl, (V & 2) ? W.dc[d].sitl : wshfl(my_sitl, d));
      edb = add(edb, div(W.dc[d].ebusy, 1000.0));
      const double b = W.dc[d].bms;
      edi = add(edi, energy_j(W.p_idle, sub(horizon, b)));
      bd = add(bd, b);
    }
  }
  uint32_t c_itl = __reduce_add_sync(FULL, (lane < ND ? W.dc[lane].n_itl_ok : 0u) + k_ok);
  uint32_t c_both = __reduce_add_sync(FULL, (lane < ND ? W.dc[lane].n_both : 0u) + k_both);
  const uint32_t c_di = __reduce_add_sync(FULL, lane < ND ? D.iters : 0u);
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
        hh = splitmix64(hh ^ W.dc[d].h);
        top = add(top, W.dc[d].top);  // one running sum: prefill instances, then decode (A37)
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
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t sid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // scenario slot
  if (sid >= P.n_slots) return;
  char *slot = P.slots + (size_t)sid * P.slot_bytes;
  uint4 *wheels = P.wheels + (size_t)sid * P.wheel_per_slot;
  using WS = WarpSmemT<F ? 8 : VOLTANA_MAX_LEVELS>;
  WS &W = *(WS *)(smem + (size_t)wib * P.smem_per_warp);
  ItlScratch &S = *(ItlScratch *)((char *)&W + P.ks_off);
  for (;;) {
    uint32_t s = 0;
    if (lane == 0) s = atomicAdd(P.counter, 1u);
    s = wshfl(s, 0);
    if (s >= P.n) break;
    uint64_t t0 = 0;
    if (P.timing) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    run_scenario<V, F>(P, s, slot, wheels, W, S, sid);
    __syncwarp();
    if (P.timing && lane == 0) {
      uint64_t t1;
      uint32_t sm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      P.timing[2 * s] = t0;
      P.timing[2 * s + 1] = (t1 - t0) | ((uint64_t)sm << 56);
    }
  }
}

size_t sim_smem_fixed(bool fast) {
  const size_t b = fast ? sizeof(WarpSmemT<8>) : sizeof(WarpSmemT<VOLTANA_MAX_LEVELS>);
  return (b - sizeof(double) + 15) & ~(size_t)15;
}

__global__ void utab_kernel(const __grid_constant__ SimParams P) {
  const uint32_t stride = gridDim.x * blockDim.x, x0 = blockIdx.x * blockDim.x + threadIdx.x;
  {  // utilisation table u = l / (l + u_half) per profile and phase (eq:P-f, A22)
    const uint32_t total = P.n_profiles * 2u * SIM_UTAB;
    for (uint32_t x = x0; x < total; x += stride) {
      const uint32_t pr = x / (2u * SIM_UTAB), ph = (x / SIM_UTAB) & 1u, l = x % SIM_UTAB;
      const double uh = P.prof[pr].uh[ph];
      ((double *)P.utab)[x] = div((double)l, add((double)l, uh));
    }
  }
  {  // ladder-resolved prefill rows per (grid, profile): [K][a1, c1], DYN_prefill[K]
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
static const void *pa_ptr(bool fast) {
  return fast ? (const void *)prefill_kernel<V, true> : (const void *)prefill_kernel<V, false>;
}
const void *pa_kernel_ptr(int v, bool fast) {
  switch (v & 3) {
    case 1: return pa_ptr<1>(fast);
    case 2: return pa_ptr<2>(fast);
    case 3: return pa_ptr<3>(fast);
    default: return pa_ptr<0>(fast);
  }
}

template <int V>
static void launch_pa_v(const SimParams &P, bool fast, int grid, cudaStream_t st) {
  if (fast) prefill_kernel<V, true><<<grid, PA_THREADS, 0, st>>>(P);
  else prefill_kernel<V, false><<<grid, PA_THREADS, 0, st>>>(P);
}

cudaError_t launch_prefill(const SimParams &P, int v, bool fast, cudaStream_t st) {
  const uint64_t total = (uint64_t)P.n * P.np_max;
  const uint64_t per_cta = PA_THREADS / 32;
  const uint64_t want = (total + per_cta - 1) / per_cta;
  const int grid = (int)(want < (1ull << 30) ? want : (1ull << 30));
  if (grid < 1) return cudaSuccess;
  switch (v & 3) {
    case 1: launch_pa_v<1>(P, fast, grid, st); break;
    case 2: launch_pa_v<2>(P, fast, grid, st); break;
    case 3: launch_pa_v<3>(P, fast, grid, st); break;
    default: launch_pa_v<0>(P, fast, grid, st); break;
  }
  return cudaGetLastError();
}

template <int V>
static const void *kptr(bool fast) {
  return fast ? (const void *)simulate_kernel<V, true> : (const void *)simulate_kernel<V, false>;
}

const void *sim_kernel_ptr(int v, bool fast) {
  if (v == 4 && fast) return (const void *)simulate_kernel<4, true>;
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

// The dynamic shared-memory attribute of the instantiation is set by the host before anything
// of the call is enqueued (voltana_simulate_ex), so a failure here is a launch error only.
cudaError_t launch_sim(const SimParams &P, int v, bool fast, int grid, size_t smem, cudaStream_t st) {
  if (v == 4 && fast) {
    simulate_kernel<4, true><<<grid, SIM_THREADS, smem, st>>>(P);
    return cudaGetLastError();
  }
  switch (v & 3) {
    case 1: launch_v<1>(P, fast, grid, smem, st); break;
    case 2: launch_v<2>(P, fast, grid, smem, st); break;
    case 3: launch_v<3>(P, fast, grid, smem, st); break;
    default: launch_v<0>(P, fast, grid, smem, st); break;
  }
  return cudaGetLastError();
}

}  // namespace vt
