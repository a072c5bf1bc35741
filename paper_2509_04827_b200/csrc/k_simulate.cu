// k_simulate.cu — K4: batched trace-driven evaluation of EcoFreq + EcoRoute (north_star).
//
// One warp per scenario, persistent warps claiming scenarios in array order.
// The event loop (A4-A23) runs warp-uniformly: every lane holds the
// same scenario state in registers, so control flow never diverges; the lanes split
// only the EcoPred evaluations across frequency levels (lane l evaluates ladder
// levels l and l+32) and reduce "lowest feasible level" with one __ballot_sync —
// an exact integer reduction, so decisions are bit-identical to the sequential scan.
//
// Decode running sets use a per-instance timing wheel of NB buckets keyed by the
// iteration index at which a request finishes (admission iteration + out - 2); all
// running requests advance together (+1 token per iteration), so a
// completion is O(1) instead of a scan of the running set. Buckets are singly
// linked lists through per-request 16-byte nodes, appended in admission order, so
// completions are processed in the oracle's order (A37) and sums are bit-exact.
#include <cstdint>

#include "vt_device.cuh"
#include "vt_sim.h"

namespace vt {

struct Node {       // 16 B per request of the scenario (workspace)
  double tfirst;    // first-token time (prefill end)
  uint32_t next;    // FIFO / wheel link
  uint32_t tag;     // bit 31: TTFT met; bits 0..30: finishing iteration index
};

// Lowest feasible ladder index given per-lane predictions for levels lane and lane+32.
__device__ __forceinline__ int lowest_from(bool f0, bool f1, int K) {
  unsigned m0 = __ballot_sync(FULL, f0);
  if (m0) return ffs0(m0);
  if (K > 32) {
    unsigned m1 = __ballot_sync(FULL, f1);
    if (m1) return 32 + ffs0(m1);
  }
  return K - 1;  // nothing feasible -> top level (A2)
}

// value held by the lane owning ladder index k (v0: levels 0..31, v1: 32..63)
__device__ __forceinline__ double pick(double v0, double v1, int k) {
  double x0 = __shfl_sync(FULL, v0, k & 31);
  double x1 = __shfl_sync(FULL, v1, k & 31);
  return k < 32 ? x0 : x1;
}
__device__ __forceinline__ int pick_i(int v0, int v1, int k) {
  int x0 = __shfl_sync(FULL, v0, k & 31);
  int x1 = __shfl_sync(FULL, v1, k & 31);
  return k < 32 ? x0 : x1;
}

// Per-lane view of the scenario's ladder: lane l owns levels l and l+32.
struct LaneLevels {
  int K;
  int lv0, lv1;          // profile-level index (0 if lane beyond K)
  bool ok0, ok1;         // lane owns a level
  double a1_0, c1_0, a1_1, c1_1;
  double dp0, dp1, dd0, dd1;  // busy dynamic power prefill / decode
  int mhz0, mhz1;
};

// eq:pred-itl for ladder index (lane, lane+32) at (n, kv): predictions and feasibility.
struct ItlEval { double p0, p1; bool f0, f1; };

__device__ __forceinline__ ItlEval itl_eval(const DevProfile &PR, const LaneLevels &L, uint32_t n,
                                            uint32_t kv, double target) {
  uint32_t j = tile_of(n, (uint32_t)PR.tile_w, (uint32_t)PR.n_tiles);
  size_t row = (size_t)j * (size_t)PR.k;
  ItlEval e;
  e.p0 = 0.0; e.p1 = 0.0;
  if (L.ok0) {
    size_t o = row + (size_t)L.lv0;
    e.p0 = itl_pred(__ldg(PR.a2 + o), __ldg(PR.b2 + o), __ldg(PR.c2 + o), n, kv);
  }
  if (L.ok1) {
    size_t o = row + (size_t)L.lv1;
    e.p1 = itl_pred(__ldg(PR.a2 + o), __ldg(PR.b2 + o), __ldg(PR.c2 + o), n, kv);
  }
  e.f0 = L.ok0 && e.p0 <= target;
  e.f1 = L.ok1 && e.p1 <= target;
  return e;
}

template <int MAXP, int MAXD>
__device__ void run_scenario(const SimParams &P, uint32_t s, char *slot) {
  const int lane = lane_id();
  voltana_result R;
  R = voltana_result{};
  // ---------------------------------------------------------------- scenario tables
  {
    const bool ids_ok = P.trace_id[s] < P.n_traces && P.slo_id[s] < P.n_slos && P.layout_id[s] < P.n_layouts &&
                        P.grid_id[s] < P.n_grids && P.profile_id[s] < P.n_profiles;
    if (!ids_ok) {
      R.status = VOLTANA_ITEM_E_INPUT;
      if (lane == 0) P.out[s] = R;
      return;
    }
  }
  const uint32_t tr = P.trace_id[s];
  const voltana_slo &SL = P.slo[P.slo_id[s]];
  const voltana_layout &LY = P.lay[P.layout_id[s]];
  const voltana_grid &GR = P.grid[P.grid_id[s]];
  const DevProfile &PR = P.prof[P.profile_id[s]];
  const uint64_t h0 = P.hash_seed[s];
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
        uint32_t a = inl[i], b = outl[i];
        double x = arr[i];
        ok = ok && a >= 1u && a <= 65535u && b >= 1u && b <= 65535u && x >= 0.0 && x < 1e9;
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
  const int K = GR.k;
  const int NP = LY.n_p, ND = LY.n_d;
  const uint32_t B = LY.max_batch_tokens, C = LY.kv_capacity;
  const double tau = LY.kv_transfer_ms;
  const double tgt_ttft = mul(SL.scale, SL.ttft_ms);  // A3
  const double tgt_itl = mul(SL.scale, SL.itl_ms);

  LaneLevels L;
  L.K = K;
  L.ok0 = lane < K;
  L.ok1 = lane + 32 < K;
  L.lv0 = L.ok0 ? GR.level[lane] : 0;
  L.lv1 = L.ok1 ? GR.level[lane + 32] : 0;
  L.a1_0 = __ldg(PR.a1 + L.lv0); L.c1_0 = __ldg(PR.c1 + L.lv0);
  L.a1_1 = __ldg(PR.a1 + L.lv1); L.c1_1 = __ldg(PR.c1 + L.lv1);
  L.dp0 = __ldg(PR.dyn + L.lv0); L.dp1 = __ldg(PR.dyn + L.lv1);
  L.dd0 = __ldg(PR.dyn + PR.k + L.lv0); L.dd1 = __ldg(PR.dyn + PR.k + L.lv1);
  L.mhz0 = __ldg(PR.mhz + L.lv0); L.mhz1 = __ldg(PR.mhz + L.lv1);

  // ---------------------------------------------------------------- workspace views
  Node *node = (Node *)slot;
  uint8_t *xd = (uint8_t *)(slot + P.node_bytes);
  uint2 *wheel = (uint2 *)(slot + P.node_bytes + P.xd_bytes);
  const uint32_t NB = P.nb, NBM = P.nb - 1;
  for (uint32_t i = lane; i < (uint32_t)ND * NB; i += 32) wheel[i] = make_uint2(NIL, NIL);
  __syncwarp();

  // ---------------------------------------------------------------- state (warp-uniform)
  uint32_t p_qhead[MAXP], p_bstart[MAXP], p_bcnt[MAXP];
  bool p_busy[MAXP];
  double p_end[MAXP], p_ebusy[MAXP], p_bms[MAXP];
#pragma unroll
  for (int q = 0; q < MAXP; ++q) {
    p_qhead[q] = q; p_bstart[q] = 0; p_bcnt[q] = 0; p_busy[q] = false;
    p_end[q] = 0.0; p_ebusy[q] = 0.0; p_bms[q] = 0.0;
  }
  uint32_t d_nreq[MAXD], d_nkv[MAXD], d_pn[MAXD], d_pkv[MAXD], d_iters[MAXD], d_cur[MAXD];
  uint32_t d_qh[MAXD], d_qt[MAXD];
  bool d_busy[MAXD];
  double d_end[MAXD], d_ebusy[MAXD], d_bms[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    d_nreq[d] = 0; d_nkv[d] = 0; d_pn[d] = 0; d_pkv[d] = 0; d_iters[d] = 0; d_cur[d] = 0;
    d_qh[d] = NIL; d_qt[d] = NIL; d_busy[d] = false;
    d_end[d] = 0.0; d_ebusy[d] = 0.0; d_bms[d] = 0.0;
  }
  uint32_t a = 0, cursor = 0, xh = NIL, xt = NIL, status = 0;
  uint64_t h = h0, steps_ctrl = 0, steps_route = 0;
  uint32_t n_ttft_ok = 0, n_itl_ok = 0, n_both = 0, prefill_iters = 0;
  double sum_ttft = 0.0, sum_itl = 0.0, top_ms = 0.0, t = 0.0, t_last = 0.0;
  double next_arr = N > 0 ? arr[0] : 0.0;

  for (;;) {
    // ------------------------------------------------------------ O1: next event time
    bool have = false;
    double tn = 0.0;
    if (a < N) { tn = next_arr; have = true; }
    if (xh != NIL) {
      double tx = add(node[xh].tfirst, tau);
      if (!have || tx < tn) { tn = tx; have = true; }
    }
#pragma unroll
    for (int q = 0; q < MAXP; ++q)
      if (q < NP && p_busy[q] && (!have || p_end[q] < tn)) { tn = p_end[q]; have = true; }
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < ND && d_busy[d] && (!have || d_end[d] < tn)) { tn = d_end[d]; have = true; }
    if (!have) break;
    t = tn;
    t_last = t;

    // ------------------------------------------------------------ O2/O3: arrivals at t
    while (a < N && next_arr == t) {
      ++a;
      next_arr = a < N ? arr[a] : 0.0;
    }
    // ------------------------------------------------------------ O4: KV transfers done
    while (xh != NIL) {
      Node nd = node[xh];
      if (!(add(nd.tfirst, tau) == t)) break;
      uint32_t i = xh, dd = xd[i];
      xh = nd.next;
      if (xh == NIL) xt = NIL;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (d == (int)dd) {
          if (d_qt[d] == NIL) d_qh[d] = i; else node[d_qt[d]].next = i;
          d_qt[d] = i;
        }
      }
      node[i].next = NIL;
    }
    // ------------------------------------------------------------ O5: PrefillDone
#pragma unroll
    for (int q = 0; q < MAXP; ++q) {
      if (!(q < NP && p_busy[q] && p_end[q] == t)) continue;
      for (uint32_t jj = 0; jj < p_bcnt[q]; ++jj) {
        uint32_t i = p_bstart[q] + jj * (uint32_t)NP;
        double ttft = sub(t, arr[i]);  // A26
        sum_ttft = add(sum_ttft, ttft);
        bool tok = ttft <= SL.ttft_ms;
        n_ttft_ok += tok;
        uint32_t oi = outl[i], ii = inl[i];
        if (oi == 1u) {  // finished at prefill (A8, A30)
          n_itl_ok += 1;
          n_both += tok;
          continue;
        }
        // ---------------------------------------------------- O8: EcoRoute
        int dsel, cse;
        if (LY.policy == 1 || ND == 1) {
          dsel = (int)cursor;
          cursor = (cursor + 1u) % (uint32_t)ND;
          cse = 0;
        } else {
          int fnow[MAXD], faft[MAXD];
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            fnow[d] = 0; faft[d] = 0;
            if (d < ND) {
              uint32_t n = d_nreq[d] + d_pn[d];  // effective state (A9)
              uint32_t kv = d_nkv[d] + d_pkv[d];
              int kn = 0;
              if (n > 0) {
                ItlEval e = itl_eval(PR, L, n, kv, tgt_itl);
                kn = lowest_from(e.f0, e.f1, K);
              }
              ItlEval e2 = itl_eval(PR, L, n + 1u, kv + ii + 1u, tgt_itl);  // A12
              int ka = lowest_from(e2.f0, e2.f1, K);
              fnow[d] = pick_i(L.mhz0, L.mhz1, kn);
              faft[d] = pick_i(L.mhz0, L.mhz1, ka);
            }
          }
          // U/R partition and cases (1)-(5) (A13-A16), integer MHz
          int ncross = 0, mu = 0x7fffffff, mr = 0x7fffffff, mn = 0x7fffffff, ma = 0x7fffffff;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d < ND) {
              bool cr = faft[d] > fnow[d];
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
            for (int d = 0; d < MAXD; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
            cse = __popc(inset) == 1 ? 1 : 2;
          } else if (ncross < ND) {
            long long g = (long long)mu - (long long)mr;
            if (g <= (long long)LY.delta_mhz) {
#pragma unroll
              for (int d = 0; d < MAXD; ++d)
                if (d < ND && !(faft[d] > fnow[d]) && fnow[d] == mu) inset |= 1u << d;
              cse = 3;
            } else {
#pragma unroll
              for (int d = 0; d < MAXD; ++d) if (d < ND && fnow[d] == mn) inset |= 1u << d;
              cse = 4;
            }
          } else {
#pragma unroll
            for (int d = 0; d < MAXD; ++d) if (d < ND && faft[d] == ma) inset |= 1u << d;
            cse = 5;
          }
          // round robin among the candidate set from the cursor (A17)
          unsigned rot = ((inset >> cursor) | (inset << (ND - cursor))) & ((1u << ND) - 1u);
          dsel = (int)((cursor + (uint32_t)ffs0(rot)) % (uint32_t)ND);
          if (__popc(inset) >= 2) cursor = (uint32_t)(dsel + 1) % (uint32_t)ND;
        }
        steps_route++;
        h = fold(h, 3, (uint64_t)dsel, 0, (uint64_t)cse);
        Node nw;
        nw.tfirst = t;
        nw.next = NIL;
        nw.tag = tok ? 0x80000000u : 0u;
        node[i] = nw;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          if (d == dsel) {
            d_pn[d] += 1u;
            d_pkv[d] += ii + 1u;
            if (tau == 0.0) {
              if (d_qt[d] == NIL) d_qh[d] = i; else node[d_qt[d]].next = i;
              d_qt[d] = i;
            }
          }
        }
        if (tau != 0.0) {
          xd[i] = (uint8_t)dsel;
          if (xt == NIL) xh = i; else node[xt].next = i;
          xt = i;
        }
      }
      p_busy[q] = false;
    }
    // ------------------------------------------------------------ O6: DecodeIterDone
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      if (!(d < ND && d_busy[d] && d_end[d] == t)) continue;
      d_nkv[d] += d_nreq[d];  // +1 KV token per running request (A19)
      const uint32_t cur = d_cur[d];
      uint2 *bk = wheel + (size_t)d * NB + (cur & NBM);
      uint2 hb = *bk;
      uint32_t r = hb.x, prev = NIL, nh = NIL;
      while (r != NIL) {
        Node nd = node[r];
        uint32_t nxt = nd.next;
        if ((nd.tag & 0x7fffffffu) == cur) {
          uint32_t oi = outl[r], ii = inl[r];
          double itl = div(sub(t, nd.tfirst), (double)(oi - 1u));  // A30
          sum_itl = add(sum_itl, itl);
          bool ok = itl <= SL.itl_ms;
          n_itl_ok += ok;
          n_both += ok && (nd.tag >> 31);
          d_nreq[d] -= 1u;
          d_nkv[d] -= ii + oi;
          if (prev != NIL) node[prev].next = nxt;
        } else {
          if (nh == NIL) nh = r;
          prev = r;
        }
        r = nxt;
      }
      *bk = make_uint2(nh, prev);
      d_busy[d] = false;
    }

    // ------------------------------------------------------------ O7: START prefill
#pragma unroll
    for (int q = 0; q < MAXP; ++q) {
      if (!(q < NP && !p_busy[q] && p_qhead[q] < a)) continue;
      // FCFS prefix with sum(in) <= B, at least one request (A6), 32 candidates per step
      uint32_t id = p_qhead[q], nbt = 0, cnt = 0;
      for (;;) {
        uint32_t idj = id + (uint32_t)lane * (uint32_t)NP;
        bool valid = idj < a;
        uint32_t v = valid ? inl[idj] : 0u;
        uint32_t pre = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t y = __shfl_up_sync(FULL, pre, o);
          if (lane >= o) pre += y;
        }
        bool fits = valid && (nbt + pre <= B || (cnt == 0u && lane == 0));
        unsigned m = __ballot_sync(FULL, fits);
        uint32_t nfit = (uint32_t)__popc(m);
        uint32_t add_tok = __shfl_sync(FULL, pre, (int)(nfit > 0 ? nfit - 1 : 0));
        if (nfit > 0) nbt += add_tok;
        cnt += nfit;
        id += nfit * (uint32_t)NP;
        if (nfit < 32u || id >= a) break;
      }
      const bool backlog = id < a;  // A5
      const double wait = sub(t, arr[p_qhead[q]]);
      double budget = sub(tgt_ttft, wait);
      budget = budget > 0.0 ? budget : 0.0;  // A4
      double p0 = ttft_pred(L.a1_0, L.c1_0, nbt), p1 = ttft_pred(L.a1_1, L.c1_1, nbt);
      int k = lowest_from(L.ok0 && p0 <= budget, L.ok1 && p1 <= budget, K);
      if (backlog) k = K - 1;
      steps_ctrl++;
      h = fold(h, 1, (uint64_t)q, (uint64_t)k, 0);
      const double dur = pick(p0, p1, k);
      if (!(dur > 0.0)) { status = VOLTANA_ITEM_E_CONTRACT; break; }
      const double dyn = pick(L.dp0, L.dp1, k);
      p_end[q] = add(t, dur);
      p_busy[q] = true;
      p_bstart[q] = p_qhead[q];
      p_bcnt[q] = cnt;
      p_qhead[q] = id;
      p_ebusy[q] = add(p_ebusy[q], energy_j(busy_power(PR.p_idle, PR.tdp, PR.uh[0], dyn, nbt), dur));
      p_bms[q] = add(p_bms[q], dur);
      prefill_iters++;
      if (k == K - 1) top_ms = add(top_ms, dur);
    }
    if (status) break;
    // ------------------------------------------------------------ O7: START decode
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      if (!(d < ND && !d_busy[d])) continue;
      // admission at the iteration boundary, FCFS while KV fits (A20)
      while (d_qh[d] != NIL) {
        const uint32_t hd = d_qh[d];
        const uint32_t ii = inl[hd];
        const uint32_t need = ii + 1u;
        if (d_nkv[d] + need > C) break;
        Node nd = node[hd];
        d_qh[d] = nd.next;
        if (d_qh[d] == NIL) d_qt[d] = NIL;
        const uint32_t fin = d_iters[d] + outl[hd] - 2u;  // last iteration of this request
        nd.next = NIL;
        nd.tag = (nd.tag & 0x80000000u) | fin;
        node[hd] = nd;
        uint2 *bk = wheel + (size_t)d * NB + (fin & NBM);
        uint2 w = *bk;
        if (w.y == NIL) { w.x = hd; } else { node[w.y].next = hd; }
        w.y = hd;
        *bk = w;
        d_nreq[d] += 1u;
        d_nkv[d] += need;
        d_pn[d] -= 1u;
        d_pkv[d] -= need;
      }
      if (d_nreq[d] == 0u) {
        if (d_qh[d] != NIL) { status = VOLTANA_ITEM_E_KV; break; }
        continue;
      }
      const bool backlog = d_qh[d] != NIL;
      ItlEval e = itl_eval(PR, L, d_nreq[d], d_nkv[d], tgt_itl);
      int k = lowest_from(e.f0, e.f1, K);
      if (backlog) k = K - 1;
      steps_ctrl++;
      h = fold(h, 2, (uint64_t)d, (uint64_t)k, 0);
      const double dur = pick(e.p0, e.p1, k);
      if (!(dur > 0.0)) { status = VOLTANA_ITEM_E_CONTRACT; break; }
      const double dyn = pick(L.dd0, L.dd1, k);
      d_end[d] = add(t, dur);
      d_busy[d] = true;
      d_ebusy[d] = add(d_ebusy[d], energy_j(busy_power(PR.p_idle, PR.tdp, PR.uh[1], dyn, d_nreq[d]), dur));
      d_bms[d] = add(d_bms[d], dur);
      d_cur[d] = d_iters[d];
      d_iters[d] += 1u;
      if (k == K - 1) top_ms = add(top_ms, dur);
    }
    if (status) break;
  }

  if (status) {
    R.status = status;
  } else {
    // ------------------------------------------------------------ O9: totals (A23)
    const double horizon = Dur > t_last ? Dur : t_last;
    double epb = 0.0, epi = 0.0, edb = 0.0, edi = 0.0, bp = 0.0, bd = 0.0;
#pragma unroll
    for (int q = 0; q < MAXP; ++q) {
      if (q < NP) {
        epb = add(epb, p_ebusy[q]);
        epi = add(epi, energy_j(PR.p_idle, sub(horizon, p_bms[q])));
        bp = add(bp, p_bms[q]);
      }
    }
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      if (d < ND) {
        edb = add(edb, d_ebusy[d]);
        edi = add(edi, energy_j(PR.p_idle, sub(horizon, d_bms[d])));
        bd = add(bd, d_bms[d]);
      }
    }
    R.n_ttft_ok = n_ttft_ok; R.n_itl_ok = n_itl_ok; R.n_both_ok = n_both; R.prefill_iters = prefill_iters;
    R.steps_ctrl = steps_ctrl; R.steps_route = steps_route; R.decision_hash = h;
    R.sum_ttft_ms = sum_ttft; R.sum_itl_mean_ms = sum_itl;
    R.e_prefill_busy_j = epb; R.e_prefill_idle_j = epi;
    R.e_decode_busy_j = edb; R.e_decode_idle_j = edi;
    R.busy_ms_prefill = bp; R.busy_ms_decode = bd;
    R.top_level_ms = top_ms; R.horizon_ms = horizon;
  }
  if (lane == 0) P.out[s] = R;
}

template <int MAXP, int MAXD>
__global__ void __launch_bounds__(SIM_THREADS) simulate_kernel(const __grid_constant__ SimParams P) {
  const int lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= P.n_slots) return;
  char *slot = P.slots + (size_t)warp * P.slot_bytes;
  for (;;) {
    uint32_t s = 0;
    if (lane == 0) s = atomicAdd(P.counter, 1u);
    s = __shfl_sync(FULL, s, 0);
    if (s >= P.n) break;
    run_scenario<MAXP, MAXD>(P, s, slot);
    __syncwarp();
  }
}

template <int MAXP, int MAXD>
const void *sim_kernel_ptr() { return (const void *)simulate_kernel<MAXP, MAXD>; }

template <int MAXP, int MAXD>
cudaError_t launch_sim(const SimParams &P, int grid, cudaStream_t st) {
  simulate_kernel<MAXP, MAXD><<<grid, SIM_THREADS, 0, st>>>(P);
  return cudaGetLastError();
}

#define VT_INST(p, d)                                                          \
  template const void *sim_kernel_ptr<p, d>();                                  \
  template cudaError_t launch_sim<p, d>(const SimParams &, int, cudaStream_t);
VT_INST(1, 1)
VT_INST(2, 2)
VT_INST(4, 4)
VT_INST(8, 8)
#undef VT_INST

}  // namespace vt
