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
// Decode running sets: a per-instance timing wheel of NB >= max(out) buckets keyed by the
// iteration index at which a request finishes (admission iteration + out - 2). All running
// requests advance together (+1 token per iteration), so completions are O(1) per
// request; buckets are lists appended in admission order (oracle order, A37).
#include <cstdint>

#include "vt_device.cuh"
#include "vt_sim.h"

namespace vt {

struct Node {       // 16 B per request (workspace)
  double tf;        // +t_first if the TTFT SLO was met, -t_first otherwise (t_first > 0)
  uint32_t next;    // phase A: next routed request of the same prefill stream; later: queue/wheel link
  uint16_t in, out;
};

// ------------------------------------------------------------------ per-warp tables (smem)
struct Tables {
  int K, T, W, kp, wshift;  // wshift >= 0: W is a power of two (tile index by shift)
  bool itl_smem, mono_tt, mono_it;
  const uint16_t *lad;     // [K] profile levels
  const double *tt;        // [K][2] a1, c1
  const double *dyn;       // [2][K] prefill, decode
  const int *mhz;          // [K]
  const double *it;        // [T][K][3] (itl_smem)
  const double *a2g, *b2g, *c2g;
};

__device__ __forceinline__ uint32_t tile_j(const Tables &S, uint32_t n) {
  uint32_t j = S.wshift >= 0 ? (n - 1u) >> S.wshift : (n - 1u) / (uint32_t)S.W;
  return j < (uint32_t)(S.T - 1) ? j : (uint32_t)(S.T - 1);
}

__device__ __forceinline__ double itl_at(const Tables &S, uint32_t j, int k, uint32_t n, uint32_t kv) {
  if (S.itl_smem) {
    const double *r = S.it + 3 * ((size_t)j * S.K + k);
    return itl_pred(r[0], r[1], r[2], n, kv);
  }
  const size_t o = (size_t)j * S.kp + S.lad[k];
  return itl_pred(__ldg(S.a2g + o), __ldg(S.b2g + o), __ldg(S.c2g + o), n, kv);
}

__device__ __forceinline__ double ttft_at(const Tables &S, int k, uint32_t nbt) {
  return ttft_pred(S.tt[2 * k], S.tt[2 * k + 1], nbt);
}

// Lowest ladder index whose prediction meets `target` (A1), else K-1 (A2);
// *pred = the prediction at the returned index. Ascending scan with early exit, or an
// exact binary search when the tables are coefficient-monotone in f (A32).
__device__ int lowest_itl(const Tables &S, uint32_t n, uint32_t kv, double target, double *pred) {
  const uint32_t j = tile_j(S, n);
  if (S.mono_it && S.K > 8) {
    int lo = 0, hi = S.K;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (itl_at(S, j, mid, n, kv) <= target) hi = mid; else lo = mid + 1;
    }
    int k = lo < S.K ? lo : S.K - 1;
    *pred = itl_at(S, j, k, n, kv);
    return k;
  }
  for (int k = 0; k < S.K - 1; ++k) {
    double p = itl_at(S, j, k, n, kv);
    if (p <= target) { *pred = p; return k; }
  }
  *pred = itl_at(S, j, S.K - 1, n, kv);
  return S.K - 1;
}

__device__ int lowest_ttft(const Tables &S, uint32_t nbt, double budget, double *pred) {
  if (S.mono_tt && S.K > 8) {
    int lo = 0, hi = S.K;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (ttft_at(S, mid, nbt) <= budget) hi = mid; else lo = mid + 1;
    }
    int k = lo < S.K ? lo : S.K - 1;
    *pred = ttft_at(S, k, nbt);
    return k;
  }
  for (int k = 0; k < S.K - 1; ++k) {
    double p = ttft_at(S, k, nbt);
    if (p <= budget) { *pred = p; return k; }
  }
  *pred = ttft_at(S, S.K - 1, nbt);
  return S.K - 1;
}

// ------------------------------------------------------------------ scenario context
struct Ctx {
  Node *node;
  uint2 *wheel;            // this lane's decode instance: [NB] {head, tail}
  uint32_t nbm;
  double tau, slo_itl, tgt_itl, p_idle, tdp, uh_d;
  uint32_t kvcap;
};

struct Err {               // first error of one lane in its own event order
  double t;                // +inf = none
  uint32_t code;
};

// Decode instance state: owned by lane d.
struct Dec {
  uint32_t nreq, nkv, pn, pkv, iters, cur, qh, qt, n_itl_ok, n_both;
  bool busy, dead;
  double end, ebusy, bms, top, sitl, tlast;
  uint64_t h;
};

__device__ __forceinline__ double avail_time(const Ctx &C, uint32_t i) {
  return add(fabs(C.node[i].tf), C.tau);  // KvTransferDone time = t_first + tau (A18); tau = 0: routing time
}

// Advance decode instance `d` through every event with time < t_lim (END, START).
__device__ void dec_advance(Dec &D, int d, const Ctx &C, const Tables &S, double t_lim, Err &E) {
  if (D.dead) return;
  for (;;) {
    double tnow;
    if (D.busy) {
      if (!(D.end < t_lim)) return;
      tnow = D.end;
      // ---- O6 DecodeIterDone: +1 KV token per running request, completions of this iteration
      D.nkv += D.nreq;
      uint2 *bk = C.wheel + (D.cur & C.nbm);
      const uint2 b = *bk;
      uint32_t r = b.x;
      while (r != NIL) {
        const Node nd = C.node[r];
        const double itl = div(sub(tnow, fabs(nd.tf)), (double)(nd.out - 1u));  // A30
        D.sitl = add(D.sitl, itl);
        const bool ok = itl <= C.slo_itl;
        D.n_itl_ok += ok;
        D.n_both += ok && nd.tf > 0.0;
        D.nreq -= 1u;
        D.nkv -= (uint32_t)nd.in + (uint32_t)nd.out;
        r = nd.next;
      }
      if (b.x != NIL) *bk = make_uint2(NIL, NIL);
      D.busy = false;
      D.tlast = tnow;
    } else {
      // idle: the next START happens when the head of the admission queue becomes available
      if (D.qh == NIL) return;
      const double av = avail_time(C, D.qh);
      if (!(av < t_lim)) return;
      tnow = av;
    }
    // ---- O7 START_DECODE at tnow: FCFS admission while KV fits (A20)
    while (D.qh != NIL) {
      const uint32_t i = D.qh;
      const Node hn = C.node[i];
      if (!(add(fabs(hn.tf), C.tau) <= tnow)) break;  // still in KV transfer
      const uint32_t need = (uint32_t)hn.in + 1u;
      if (D.nkv + need > C.kvcap) break;
      D.qh = hn.next;
      if (D.qh == NIL) D.qt = NIL;
      const uint32_t fin = D.iters + (uint32_t)hn.out - 2u;  // its last iteration
      uint2 *bk = C.wheel + (fin & C.nbm);
      uint2 b = *bk;
      C.node[i].next = NIL;
      if (b.y == NIL) b.x = i; else C.node[b.y].next = i;
      b.y = i;
      *bk = b;
      D.nreq += 1u;
      D.nkv += need;
      D.pn -= 1u;
      D.pkv -= need;
    }
    const bool backlog = D.qh != NIL && avail_time(C, D.qh) <= tnow;  // A5
    if (D.nreq == 0u) {
      if (backlog) { E.t = tnow; E.code = VOLTANA_ITEM_E_KV; D.dead = true; return; }
      continue;  // stays idle
    }
    double dur;
    int k;
    if (backlog) { k = S.K - 1; dur = itl_at(S, tile_j(S, D.nreq), k, D.nreq, D.nkv); }
    else k = lowest_itl(S, D.nreq, D.nkv, C.tgt_itl, &dur);
    D.h = fold(D.h, 2, (uint64_t)d, (uint64_t)k, 0);
    if (!(dur > 0.0)) { E.t = tnow; E.code = VOLTANA_ITEM_E_CONTRACT; D.dead = true; return; }
    D.end = add(tnow, dur);
    D.busy = true;
    D.ebusy = add(D.ebusy, mul(busy_power(C.p_idle, C.tdp, C.uh_d, S.dyn[S.K + k], D.nreq), dur));  // W*ms (A23)
    D.bms = add(D.bms, dur);
    if (k == S.K - 1) D.top = add(D.top, dur);
    D.cur = D.iters;
    D.iters += 1u;
  }
}

// warp-wide min of a non-negative double held by lanes with `valid`; returns the lowest lane
// attaining it, or -1 if no lane is valid. Bit patterns of non-negative doubles order as u64.
__device__ __forceinline__ int argmin_time(double t, bool valid) {
  const uint64_t b = __double_as_longlong(t);
  const uint32_t hi = valid ? (uint32_t)(b >> 32) : 0xffffffffu;
  const uint32_t mhi = __reduce_min_sync(FULL, hi);
  const bool c1 = valid && hi == mhi;
  const uint32_t lo = c1 ? (uint32_t)b : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(FULL, lo);
  const unsigned m = __ballot_sync(FULL, c1 && lo == mlo);
  return m ? ffs0(m) : -1;
}

__device__ void run_scenario(const SimParams &P, uint32_t s, char *slot, uint2 *wheels, char *wsm) {
  const int lane = lane_id();
  voltana_result R = voltana_result{};
  // ---------------------------------------------------------------- ids and table rows
  if (!(P.trace_id[s] < P.n_traces && P.slo_id[s] < P.n_slos && P.layout_id[s] < P.n_layouts &&
        P.grid_id[s] < P.n_grids && P.profile_id[s] < P.n_profiles)) {
    R.status = VOLTANA_ITEM_E_INPUT;
    if (lane == 0) P.out[s] = R;
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
  R.n_requests = (uint32_t)N64;

  // ---------------------------------------------------------------- device validation (A40)
  {
    bool ok = N64 <= P.max_requests && Dur >= 0.0;
    uint64_t tok = 0;
    if (ok) {
      for (uint64_t i = lane; i < N64; i += 32) {
        const uint32_t a = inl[i], b = outl[i];
        const double x = arr[i];
        ok = ok && a >= 1u && a <= 65535u && b >= 1u && b <= P.max_out && x >= 0.0 && x < 1e9;
        if (i > 0) ok = ok && !(x < arr[i - 1]);
        tok += (uint64_t)a + b;
      }
    }
    for (int o = 16; o > 0; o >>= 1) tok += __shfl_xor_sync(FULL, tok, o);
    ok = __all_sync(FULL, ok) && tok <= 0x7fffffffull;
    if (!ok) {
      R.status = VOLTANA_ITEM_E_INPUT;
      if (lane == 0) P.out[s] = R;
      return;
    }
  }
  const uint32_t N = (uint32_t)N64;
  const int NP = LY.n_p, ND = LY.n_d;

  // ---------------------------------------------------------------- stage the ladder's tables
  Tables S;
  S.K = GR.k; S.T = PR.n_tiles; S.W = PR.tile_w; S.kp = PR.k;
  S.wshift = (PR.tile_w & (PR.tile_w - 1)) == 0 ? __ffs(PR.tile_w) - 1 : -1;
  S.itl_smem = P.itl_smem != 0;
  {
    char *p = wsm;
    uint16_t *lad = (uint16_t *)p; p += 128;
    double *tt = (double *)p; p += 16 * VOLTANA_MAX_LEVELS;
    double *dyn = (double *)p; p += 16 * VOLTANA_MAX_LEVELS;
    int *mhz = (int *)p; p += 4 * VOLTANA_MAX_LEVELS;
    double *it = (double *)p;
    for (int k = lane; k < S.K; k += 32) {
      const int lv = GR.level[k];
      lad[k] = (uint16_t)lv;
      tt[2 * k] = PR.a1[lv]; tt[2 * k + 1] = PR.c1[lv];
      dyn[k] = PR.dyn[lv]; dyn[S.K + k] = PR.dyn[PR.k + lv];
      mhz[k] = PR.mhz[lv];
    }
    if (S.itl_smem) {
      for (int x = lane; x < S.T * S.K; x += 32) {
        const int j = x / S.K, k = x - j * S.K;
        const size_t o = (size_t)j * PR.k + GR.level[k];
        it[3 * x] = PR.a2[o]; it[3 * x + 1] = PR.b2[o]; it[3 * x + 2] = PR.c2[o];
      }
    }
    __syncwarp();
    S.lad = lad; S.tt = tt; S.dyn = dyn; S.mhz = mhz; S.it = it;
    S.a2g = PR.a2; S.b2g = PR.b2; S.c2g = PR.c2;
    // coefficient-monotone (non-increasing in f) tables allow the exact binary search (A32)
    bool mt = true, mi = true;
    for (int k = lane; k + 1 < S.K; k += 32)
      mt = mt && tt[2 * k + 2] <= tt[2 * k] && tt[2 * k + 3] <= tt[2 * k + 1];
    for (int x = lane; x < S.T * (S.K - 1); x += 32) {
      const int j = x / (S.K - 1), k = x - j * (S.K - 1);
      const size_t o0 = (size_t)j * PR.k + GR.level[k], o1 = (size_t)j * PR.k + GR.level[k + 1];
      mi = mi && PR.a2[o1] <= PR.a2[o0] && PR.b2[o1] <= PR.b2[o0] && PR.c2[o1] <= PR.c2[o0];
    }
    S.mono_tt = __all_sync(FULL, mt);
    S.mono_it = __all_sync(FULL, mi);
  }
  Node *node = (Node *)slot;
  const double tgt_ttft = mul(SL.scale, SL.ttft_ms);  // A3
  const double tgt_itl = mul(SL.scale, SL.itl_ms);
  const double INF = __longlong_as_double(0x7ff0000000000000ll);

  // ================================================================ PHASE A: prefill lanes
  double p_ebusy = 0.0, p_bms = 0.0, p_top = 0.0, p_sttft = 0.0, p_tlast = 0.0;
  uint64_t p_h = P.hash_seed[s];
  uint32_t p_iters = 0, p_ttft_ok = 0, p_itl_ok = 0, p_both = 0, p_head = NIL;
  Err pE = {INF, 0};
  if (lane < NP) {
    const uint32_t p = (uint32_t)lane, NPu = (uint32_t)NP;
    double tfree = 0.0;
    uint32_t nxt = p, prev = NIL;
    Node pend;
    pend.tf = 0.0; pend.next = NIL; pend.in = 0; pend.out = 0;
    while (nxt < N) {
      const double a0 = arr[nxt];
      const double ts = tfree > a0 ? tfree : a0;  // START: instance idle and queue non-empty
      // FCFS prefix of the arrived queue with sum(in) <= B, at least one request (A6)
      uint32_t nbt = inl[nxt], cnt = 1, id = nxt + NPu;
      bool backlog = false;
      for (bool stop = false; !stop;) {  // 4 candidates per round, loads issued together
        double av[4];
        uint32_t xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t j = id + (uint32_t)u * NPu;
          av[u] = j < N ? arr[j] : INF;     // past the trace end: "not arrived"
          xv[u] = j < N ? inl[j] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (stop) continue;
          if (!(av[u] <= ts)) stop = true;                                             // not arrived yet
          else if (nbt + xv[u] > LY.max_batch_tokens) { backlog = true; stop = true; }  // does not fit
          else { nbt += xv[u]; cnt++; id += NPu; }
        }
      }
      // (A5) backlog: requests still queued after the batch
      double budget = sub(tgt_ttft, sub(ts, a0));  // A4: SLO minus the oldest request's wait
      budget = budget > 0.0 ? budget : 0.0;
      double dur;
      int k;
      if (backlog) { k = S.K - 1; dur = ttft_at(S, k, nbt); }
      else k = lowest_ttft(S, nbt, budget, &dur);
      p_h = fold(p_h, 1, (uint64_t)p, (uint64_t)k, 0);
      p_iters++;
      if (!(dur > 0.0)) { pE.t = ts; pE.code = VOLTANA_ITEM_E_CONTRACT; break; }
      const double end = add(ts, dur);
      p_ebusy = add(p_ebusy, mul(busy_power(PR.p_idle, PR.tdp, PR.uh[0], S.dyn[k], nbt), dur));  // W*ms (A23)
      p_bms = add(p_bms, dur);
      if (k == S.K - 1) p_top = add(p_top, dur);
      // ---- O5 PrefillDone at `end`, batch in FCFS order
      for (uint32_t q = 0, i = nxt; q < cnt; ++q, i += NPu) {
        const double ttft = sub(end, arr[i]);  // A26
        p_sttft = add(p_sttft, ttft);
        const bool ok = ttft <= SL.ttft_ms;
        p_ttft_ok += ok;
        const uint32_t o = outl[i];
        if (o == 1u) {  // first token came from prefill: done (A8, A30)
          p_itl_ok++;
          p_both += ok;
          continue;
        }
        if (prev != NIL) { pend.next = i; node[prev] = pend; } else p_head = i;
        prev = i;
        pend.tf = ok ? end : -end;
        pend.next = NIL;
        pend.in = (uint16_t)inl[i];
        pend.out = (uint16_t)o;
      }
      tfree = end;
      p_tlast = end;
      nxt = id;
    }
    if (prev != NIL) { pend.next = NIL; node[prev] = pend; }
  }
  __syncwarp();

  // ================================================================ PHASE B: routing + decode lanes
  Ctx C;
  C.node = node;
  C.wheel = wheels + (size_t)(lane < ND ? lane : 0) * P.nb;
  C.nbm = P.nb - 1u;
  C.tau = LY.kv_transfer_ms; C.slo_itl = SL.itl_ms; C.tgt_itl = tgt_itl;
  C.p_idle = PR.p_idle; C.tdp = PR.tdp; C.uh_d = PR.uh[1]; C.kvcap = LY.kv_capacity;
  Dec D;
  D.nreq = D.nkv = D.pn = D.pkv = D.iters = D.cur = 0;
  D.qh = D.qt = NIL;
  D.n_itl_ok = D.n_both = 0;
  D.busy = false; D.dead = !(lane < ND);
  D.end = D.ebusy = D.bms = D.top = D.sitl = D.tlast = 0.0;
  D.h = P.hash_seed[s];
  Err dE = {INF, 0};

  // stream head of prefill lane p: next routed request in its completion order
  // (head node hn and, loaded one step ahead, its successor nn)
  uint32_t hd = lane < NP ? p_head : NIL;
  Node hn, nn;
  hn.tf = 0.0; hn.next = NIL; hn.in = 0; hn.out = 0;
  nn = hn;
  if (hd != NIL) {
    hn = node[hd];
    if (hn.next != NIL) nn = node[hn.next];
  }
  uint64_t h_r = P.hash_seed[s];
  uint32_t cursor = 0, steps_route = 0;
  const bool eco = LY.policy == 0 && ND > 1;
  for (;;) {
    const double ht = fabs(hn.tf);
    const int w = argmin_time(ht, hd != NIL);  // next PrefillDone request in (t, p, id) order
    if (w < 0) break;
    const double t = __shfl_sync(FULL, ht, w);
    const uint32_t i = __shfl_sync(FULL, hd, w);
    const uint32_t in_i = __shfl_sync(FULL, (uint32_t)hn.in, w);
    if (lane == w) {                           // advance that stream; prefetch one further
      hd = hn.next;
      hn = nn;
      if (hd != NIL && hn.next != NIL) nn = node[hn.next];
    }
    // decode instances catch up to t: events strictly before t (PrefillDone drains first)
    dec_advance(D, lane, C, S, t, dE);
    // ---- O8 EcoRoute
    int dsel, cse;
    if (!eco) {
      dsel = (int)cursor;
      cursor = (cursor + 1u) % (uint32_t)ND;
      cse = 0;
    } else {
      int fnow = 0x7fffffff, faft = 0x7fffffff;
      if (lane < ND) {
        const uint32_t n = D.nreq + D.pn, kv = D.nkv + D.pkv;  // A9 effective state
        double pr;
        const int kn = n == 0u ? 0 : lowest_itl(S, n, kv, tgt_itl, &pr);  // A10, A11
        const int ka = lowest_itl(S, n + 1u, kv + in_i + 1u, tgt_itl, &pr);  // A12
        fnow = S.mhz[kn];
        faft = S.mhz[ka];
      }
      const bool act = lane < ND;
      const bool cr = act && faft > fnow;  // A13
      const unsigned Rm = __ballot_sync(FULL, cr);
      const int nc = __popc(Rm);
      const int mn = (int)__reduce_min_sync(FULL, (unsigned)fnow);
      unsigned inset;
      if (nc == 0) {
        inset = __ballot_sync(FULL, act && fnow == mn);
        cse = __popc(inset) == 1 ? 1 : 2;
      } else if (nc < ND) {
        const int mu = (int)__reduce_min_sync(FULL, (unsigned)(act && !cr ? fnow : 0x7fffffff));
        const int mr = (int)__reduce_min_sync(FULL, (unsigned)(cr ? faft : 0x7fffffff));
        const long long g = (long long)mu - (long long)mr;  // A14, A15
        if (g <= (long long)LY.delta_mhz) { inset = __ballot_sync(FULL, act && !cr && fnow == mu); cse = 3; }
        else { inset = __ballot_sync(FULL, act && fnow == mn); cse = 4; }
      } else {
        const int ma = (int)__reduce_min_sync(FULL, (unsigned)faft);
        inset = __ballot_sync(FULL, act && faft == ma);
        cse = 5;
      }
      // round robin among the candidate set from the cursor (A17)
      const unsigned rot = ((inset >> cursor) | (inset << (ND - (int)cursor))) & ((1u << ND) - 1u);
      dsel = (int)((cursor + (uint32_t)ffs0(rot)) % (uint32_t)ND);
      if (__popc(inset) >= 2) cursor = (uint32_t)(dsel + 1) % (uint32_t)ND;
    }
    steps_route++;
    h_r = fold(h_r, 3, (uint64_t)dsel, 0, (uint64_t)cse);
    if (lane == dsel) {
      D.pn += 1u;
      D.pkv += in_i + 1u;
      node[i].next = NIL;
      if (D.qt == NIL) D.qh = i; else node[D.qt].next = i;
      D.qt = i;
    }
  }
  // drain: every decode instance runs to completion
  dec_advance(D, lane, C, S, INF, dE);
  __syncwarp();

  // ================================================================ O9: record
  // first error in (time, prefill before decode, instance) order = the oracle's stop point
  const int wp = argmin_time(pE.t, lane < NP && pE.t < INF);
  const int wd = argmin_time(dE.t, lane < ND && dE.t < INF);
  if (wp >= 0 || wd >= 0) {
    const double tp = wp >= 0 ? __shfl_sync(FULL, pE.t, wp) : INF;
    const double td = wd >= 0 ? __shfl_sync(FULL, dE.t, wd) : INF;
    const uint32_t cp = __shfl_sync(FULL, pE.code, wp >= 0 ? wp : 0);
    const uint32_t cd = __shfl_sync(FULL, dE.code, wd >= 0 ? wd : 0);
    R.status = (wp >= 0 && tp <= td) ? cp : cd;
    // leave the wheels clean for the next scenario of this warp
    if (lane < ND)
      for (uint32_t b = 0; b < P.nb; ++b) wheels[(size_t)lane * P.nb + b] = make_uint2(NIL, NIL);
    if (lane == 0) P.out[s] = R;
    return;
  }
  double tl = p_tlast > D.tlast ? p_tlast : D.tlast;
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(FULL, tl, o);
    tl = x > tl ? x : tl;
  }
  const double horizon = Dur > tl ? Dur : tl;  // A23
  uint64_t hh = splitmix64(h_r);                // A36: route chain, prefill chains, decode chains
  double sttft = 0.0, sitl = 0.0, top = 0.0, epb = 0.0, epi = 0.0, edb = 0.0, edi = 0.0, bp = 0.0, bd = 0.0;
  for (int q = 0; q < NP; ++q) {
    hh = splitmix64(hh ^ __shfl_sync(FULL, p_h, q));
    sttft = add(sttft, __shfl_sync(FULL, p_sttft, q));
    top = add(top, __shfl_sync(FULL, p_top, q));
    epb = add(epb, div(__shfl_sync(FULL, p_ebusy, q), 1000.0));
    const double b = __shfl_sync(FULL, p_bms, q);
    epi = add(epi, energy_j(PR.p_idle, sub(horizon, b)));
    bp = add(bp, b);
  }
  for (int d = 0; d < ND; ++d) {
    hh = splitmix64(hh ^ __shfl_sync(FULL, D.h, d));
    sitl = add(sitl, __shfl_sync(FULL, D.sitl, d));
    top = add(top, __shfl_sync(FULL, D.top, d));
    edb = add(edb, div(__shfl_sync(FULL, D.ebusy, d), 1000.0));
    const double b = __shfl_sync(FULL, D.bms, d);
    edi = add(edi, energy_j(PR.p_idle, sub(horizon, b)));
    bd = add(bd, b);
  }
  uint32_t c_ttft = p_ttft_ok, c_itl = p_itl_ok + (lane < ND ? D.n_itl_ok : 0u);
  uint32_t c_both = p_both + (lane < ND ? D.n_both : 0u), c_pi = lane < NP ? p_iters : 0u;
  uint32_t c_di = lane < ND ? D.iters : 0u;
  c_ttft = __reduce_add_sync(FULL, c_ttft);
  c_itl = __reduce_add_sync(FULL, c_itl);
  c_both = __reduce_add_sync(FULL, c_both);
  c_pi = __reduce_add_sync(FULL, c_pi);
  c_di = __reduce_add_sync(FULL, c_di);
  R.n_ttft_ok = c_ttft; R.n_itl_ok = c_itl; R.n_both_ok = c_both; R.prefill_iters = c_pi;
  R.steps_ctrl = (uint64_t)c_pi + c_di; R.steps_route = steps_route; R.decision_hash = hh;
  R.sum_ttft_ms = sttft; R.sum_itl_mean_ms = sitl;
  R.e_prefill_busy_j = epb; R.e_prefill_idle_j = epi; R.e_decode_busy_j = edb; R.e_decode_idle_j = edi;
  R.busy_ms_prefill = bp; R.busy_ms_decode = bd; R.top_level_ms = top; R.horizon_ms = horizon;
  if (lane == 0) P.out[s] = R;
}

__global__ void __launch_bounds__(SIM_THREADS, SIM_MIN_BLOCKS) simulate_kernel(const __grid_constant__ SimParams P) {
  extern __shared__ __align__(16) char smem[];
  const int lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= P.n_slots) return;
  char *slot = P.slots + (size_t)warp * P.slot_bytes;
  uint2 *wheels = P.wheels + (size_t)warp * P.wheel_per_slot;
  char *wsm = smem + (size_t)wib * P.smem_per_warp;
  for (;;) {
    uint32_t s = 0;
    if (lane == 0) s = atomicAdd(P.counter, 1u);
    s = __shfl_sync(FULL, s, 0);
    if (s >= P.n) break;
    run_scenario(P, s, slot, wheels, wsm);
    __syncwarp();
  }
}

const void *sim_kernel_ptr() { return (const void *)simulate_kernel; }

cudaError_t launch_sim(const SimParams &P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(simulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  simulate_kernel<<<grid, SIM_THREADS, smem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace vt
