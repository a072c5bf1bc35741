/* oracle.c — TEST INFRASTRUCTURE ONLY: the plain CPU oracle of the VoltanaLLM
 * hot path (arXiv 2509.04827). See oracle.h for who may use it.
 *
 * What it computes, in the paper's order and notation:
 *   EcoPred   eq:pred-ttft  T_ttft(f, N_bt) = a1_f N_bt + c1_f
 *             eq:pred-itl   T_itl(f, N_req, N_kv) = a2_f N_req + b2_f N_kv + c2_f,
 *                           per batch-size tile
 *   EcoFreq   backlog -> max frequency; else the lowest frequency of the list
 *             whose predicted latency meets the SLO target; prefill target =
 *             SLO - waiting time, decode target = SLO
 *   EcoRoute  what-if f/f' per decode instance, cases (1)-(5) with Delta
 *   prefill routing: round robin
 *   energy    time x power(f)                                               (eq:P-f P:187)
 *   fit       per-frequency (and per tile) least squares
 * The discrete-event semantics the paper leaves open are the readings A1-A39
 * listed in DESIGN.md ("Readings of the paper"); each is marked [Axx] below.
 *
 * Plain data structures on purpose: the running set of a decode instance is
 * an admission-ordered array scanned in full every iteration; queues are
 * arrays. Nothing here is tuned.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- EcoPred */

static int tile_index(const orc_profile *p, uint64_t n_req) {
  /* j = min(T-1, floor((N_req-1)/W)): tile boundaries at multiples of W = 128,
   * "increasing the batch size from 128 to 129 (crossing a boundary)" [A21] */
  uint64_t j = (n_req - 1) / (uint64_t)p->tile_w;
  if (j > (uint64_t)(p->n_tiles - 1)) j = (uint64_t)(p->n_tiles - 1);
  return (int)j;
}

/* prefill tile (Appendix B: a staircase below ~2000 batched tokens that "gradually
 * becomes less significant" above): T_p <= 1 -> one tile; else N_bt above the
 * cutoff -> the last tile T_p - 1, otherwise min(T_p - 1, floor((N_bt - 1) / W)) [F1] */
static int ptile_index(const orc_profile *p, uint64_t n_bt) {
  if (p->n_ptiles <= 1) return 0;
  if (n_bt > (uint64_t)p->prefill_cutoff) return p->n_ptiles - 1;
  uint64_t j = (n_bt - 1) / (uint64_t)p->tile_w;
  if (j > (uint64_t)(p->n_ptiles - 1)) j = (uint64_t)(p->n_ptiles - 1);
  return (int)j;
}

static double predict_ttft(const orc_profile *p, int lvl, uint64_t n_bt) {
  /* eq:pred-ttft, evaluated as (a1 * N_bt) + c1 [A33], on the batch's prefill tile */
  size_t idx = (size_t)ptile_index(p, n_bt) * (size_t)p->k + (size_t)lvl;
  return (p->a1[idx] * (double)n_bt) + p->c1[idx];
}

static double predict_itl(const orc_profile *p, int lvl, uint64_t n_req, uint64_t n_kv) {
  /* eq:pred-itl "(each tile)": ((a2 * N_req) + (b2 * N_kv)) + c2 [A33] */
  int j = tile_index(p, n_req);
  size_t idx = (size_t)j * (size_t)p->k + (size_t)lvl;
  return ((p->a2[idx] * (double)n_req) + (p->b2[idx] * (double)n_kv)) + p->c2[idx];
}

/* ---------------------------------------------------------------- EcoFreq */

/* "for all candidates in the list of frequencies, it queries EcoPred ... Finally,
 * it selects the lowest frequency in the list whose corresponding predicted
 * latency satisfies the SLO target". Feasible means pred <= target
 * [A1]; if none is feasible the maximum level is used [A2]. */
static int lowest_feasible_ttft(const orc_profile *p, const uint16_t *L, int K, uint64_t n_bt,
                                double target) {
  for (int k = 0; k < K; ++k)
    if (predict_ttft(p, L[k], n_bt) <= target) return k;
  return K - 1;
}

static int lowest_feasible_itl(const orc_profile *p, const uint16_t *L, int K, uint64_t n_req,
                               uint64_t n_kv, double target) {
  for (int k = 0; k < K; ++k)
    if (predict_itl(p, L[k], n_req, n_kv) <= target) return k;
  return K - 1;
}

/* prefill target: "subtracts the waiting time from total SLO budget" [A4] */
static double prefill_budget(double target, double wait) {
  double b = target - wait;
  return b > 0.0 ? b : 0.0;
}

/* ------------------------------------------------------------ power/energy */

/* busy power, eq:P-f as per-level tables with TDP clip [A22]:
 *   P = min(TDP, P_idle + u(load) * DYN[phase][level]),  u = load / (load + u_half) */
static double busy_power(const orc_profile *p, int phase, int lvl, uint64_t load) {
  double uh = phase == 0 ? p->uh_prefill : p->uh_decode;
  double u = (double)load / ((double)load + uh);
  double w = p->p_idle + (u * p->dyn[(size_t)phase * (size_t)p->k + (size_t)lvl]);
  return w < p->tdp ? w : p->tdp;
}

/* energy = time x power: joules from watts and milliseconds */
static double interval_energy(double power_w, double dur_ms) { return (power_w * dur_ms) / 1000.0; }

/* ------------------------------------------------------------ ITL aggregation [E3] */

static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x > y) - (x < y);
}

/* nearest-rank P99 of n gaps: the ceil(0.99 n)-th smallest ("itl_mode P99") [E3] */
static double p99_nearest_rank(double *g, uint64_t n) {
  qsort(g, (size_t)n, sizeof(double), cmp_double);
  uint64_t rank = (99 * n + 99) / 100; /* ceil(0.99 n), exact in integers */
  return g[rank - 1];
}

/* ------------------------------------------------------------ decision hash */

static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* h <- (h ^ (kind<<48 ^ instance<<32 ^ level<<16 ^ case)) * phi64 [A36]: for a fixed
 * decision word the step is a bijection of h, so two decision sequences that differ in
 * one decision keep differing; the chains are mixed with splitmix64 at the end. */
/* [D2] execution-noise factor of iteration j of instance `inst` (prefill q, decode N_P + d):
 * a counter-based index into the host-drawn factor table, so both sides read the same
 * factor without evaluating a transcendental. */
static double noise_factor(const orc_scenario *s, uint64_t inst, uint64_t j) {
  uint64_t x = s->hash_seed ^ 0xD1B54A32D192ED03ull ^ (inst << 40) ^ j;
  return s->noise[splitmix64(x) & (s->noise_len - 1)];
}

static uint64_t fold(uint64_t h, uint64_t kind, uint64_t inst, uint64_t level, uint64_t cse) {
  return (h ^ ((kind << 48) ^ (inst << 32) ^ (level << 16) ^ cse)) * 0x9E3779B97F4A7C15ull;
}

/* ---------------------------------------------------------------- EcoRoute */

/* One EcoRoute decision for a request of input length `in`.
 * n[d], kv[d]: effective state of decode instance d (running + routed-but-not-
 * admitted, [A9]). Returns the instance, writes the case (0 = round robin). */
/* Round robin among a candidate set, starting at the cursor [A17]. */
static int rr_pick(const int *in_set, int n_d, uint32_t *cursor) {
  int cnt = 0, best = -1;
  uint32_t best_dist = UINT32_MAX;
  for (int d = 0; d < n_d; ++d) {
    if (!in_set[d]) continue;
    cnt++;
    uint32_t dist = (uint32_t)((d - (int)*cursor + n_d) % n_d);
    if (dist < best_dist) { best_dist = dist; best = d; }
  }
  if (cnt >= 2) *cursor = (uint32_t)((best + 1) % n_d);
  return best;
}

/* [f1, B1-B3] Energy-scored routing, the north_star's reading of the state-space router:
 * "scores every (candidate instance, frequency) successor state with the latency and
 * power(f) models, masks SLO violators and takes the argmin-energy decision". Routing to d
 * changes only d's per-iteration energy P*T, so the system's energy rate changes by
 *   score(d) = min over SLO-feasible k of P(k, n+1) * T_itl(k, n+1, kv+in+1)
 *              - P(k_now, n) * T_itl(k_now, n, kv)        (0 for an empty instance),
 * k_now = EcoFreq's level of the current effective state [A9-A11]. argmin score over
 * instances with a feasible k (case 6); none feasible: the fastest top-level successor
 * (case 7); ties round robin [A17]. */
static int energy_route(const orc_profile *p, const uint16_t *L, int K, int n_d, const uint64_t *n,
                        const uint64_t *kv, uint64_t in, double target, uint32_t *cursor, int *case_out) {
  double score[64], tmax[64];
  int feas[64], in_set[64], any = 0;
  for (int d = 0; d < n_d; ++d) {
    double enow = 0.0;
    if (n[d] > 0) {
      int k0 = lowest_feasible_itl(p, L, K, n[d], kv[d], target);
      enow = busy_power(p, 1, L[k0], n[d]) * predict_itl(p, L[k0], n[d], kv[d]);
    }
    double best = 0.0;
    int found = 0;
    for (int k = 0; k < K; ++k) {
      double t = predict_itl(p, L[k], n[d] + 1, kv[d] + in + 1);
      if (t <= target) {
        double e = busy_power(p, 1, L[k], n[d] + 1) * t;
        if (!found || e < best) { best = e; found = 1; }
      }
    }
    feas[d] = found;
    any |= found;
    score[d] = best - enow;
    tmax[d] = predict_itl(p, L[K - 1], n[d] + 1, kv[d] + in + 1);
  }
  double m = 0.0;
  int first = 1;
  for (int d = 0; d < n_d; ++d) {
    if (any && !feas[d]) continue;
    double v = any ? score[d] : tmax[d];
    if (first || v < m) { m = v; first = 0; }
  }
  for (int d = 0; d < n_d; ++d) in_set[d] = any ? (feas[d] && score[d] == m) : (tmax[d] == m);
  *case_out = any ? 6 : 7;
  return rr_pick(in_set, n_d, cursor);
}

/* [f1, B4] Energy-argmin controller: among the levels whose prediction meets the target,
 * the one with the lowest iteration energy P(k, load) * T(k); ties -> lower level; none
 * feasible -> top level (A2). Differs from the paper's lowest feasible level only when the
 * grid spans the bottom of the U-shaped energy curve. */
static int energy_level_itl(const orc_profile *p, const uint16_t *L, int K, uint64_t n, uint64_t kv,
                            double target) {
  int best = -1;
  double be = 0.0;
  for (int k = 0; k < K; ++k) {
    double t = predict_itl(p, L[k], n, kv);
    if (!(t <= target)) continue;
    double e = busy_power(p, 1, L[k], n) * t;
    if (best < 0 || e < be) { best = k; be = e; }
  }
  return best < 0 ? K - 1 : best;
}

static int energy_level_ttft(const orc_profile *p, const uint16_t *L, int K, uint64_t nbt, double budget) {
  int best = -1;
  double be = 0.0;
  for (int k = 0; k < K; ++k) {
    double t = predict_ttft(p, L[k], nbt);
    if (!(t <= budget)) continue;
    double e = busy_power(p, 0, L[k], nbt) * t;
    if (best < 0 || e < be) { best = k; be = e; }
  }
  return best < 0 ? K - 1 : best;
}

static int ecoroute(const orc_profile *p, const uint16_t *L, int K, int n_d, const uint64_t *n,
                    const uint64_t *kv, uint64_t in, double target, int32_t delta, int policy,
                    uint32_t *cursor, int *case_out) {
  if (policy == 2 && n_d > 1) return energy_route(p, L, K, n_d, n, kv, in, target, cursor, case_out);
  if (policy == 1 || n_d == 1) { /* SGLang round robin / single instance [A17] */
    int d = (int)*cursor;
    *cursor = (uint32_t)((d + 1) % n_d);
    *case_out = 0;
    return d;
  }
  int64_t fnow[64], faft[64];
  int crossed[64];
  for (int d = 0; d < n_d; ++d) {
    /* "what-if": frequency now and after hypothetically adding the request.
     * EcoFreq's predictor rule without the backlog override [A10, A11];
     * an empty instance sits at the lowest level; the request adds in+1 KV [A12]. */
    int k_now = n[d] == 0 ? 0 : lowest_feasible_itl(p, L, K, n[d], kv[d], target);
    int k_aft = lowest_feasible_itl(p, L, K, n[d] + 1, kv[d] + in + 1, target);
    fnow[d] = p->mhz[L[k_now]];
    faft[d] = p->mhz[L[k_aft]];
    crossed[d] = faft[d] > fnow[d]; /* "cross the boundaries" [A13] */
  }
  int n_cross = 0;
  for (int d = 0; d < n_d; ++d) n_cross += crossed[d];
  int in_set[64];
  int cse;
  if (n_cross == 0) {
    /* (1)/(2): no instance crosses -> lowest current frequency; ties round robin [A16] */
    int64_t m = INT64_MAX;
    for (int d = 0; d < n_d; ++d) if (fnow[d] < m) m = fnow[d];
    int cnt = 0;
    for (int d = 0; d < n_d; ++d) { in_set[d] = fnow[d] == m; cnt += in_set[d]; }
    cse = cnt == 1 ? 1 : 2;
  } else if (n_cross < n_d) {
    /* (3)/(4): g = (lowest unchanged f) - (lowest crossed f') compared with Delta [A14, A15] */
    int64_t mu = INT64_MAX, mr = INT64_MAX;
    for (int d = 0; d < n_d; ++d) {
      if (!crossed[d] && fnow[d] < mu) mu = fnow[d];
      if (crossed[d] && faft[d] < mr) mr = faft[d];
    }
    int64_t g = mu - mr;
    if (g <= (int64_t)delta) {
      /* (3): dispatch to the instance whose frequency would remain unchanged */
      for (int d = 0; d < n_d; ++d) in_set[d] = !crossed[d] && fnow[d] == mu;
      cse = 3;
    } else {
      /* (4): the instance with the lowest current frequency */
      int64_t m = INT64_MAX;
      for (int d = 0; d < n_d; ++d) if (fnow[d] < m) m = fnow[d];
      for (int d = 0; d < n_d; ++d) in_set[d] = fnow[d] == m;
      cse = 4;
    }
  } else {
    /* (5): all cross -> the lowest resulting frequency */
    int64_t m = INT64_MAX;
    for (int d = 0; d < n_d; ++d) if (faft[d] < m) m = faft[d];
    for (int d = 0; d < n_d; ++d) in_set[d] = faft[d] == m;
    cse = 5;
  }
  /* ties: round robin among the candidate set, starting at the cursor [A17] */
  *case_out = cse;
  return rr_pick(in_set, n_d, cursor);
}

/* --------------------------------------------------------------- simulator */

typedef struct { uint32_t id; uint32_t rem; } run_entry;

typedef struct {
  /* decode instance state */
  run_entry *run; uint64_t n_run, cap_run;   /* admission-ordered running set */
  uint32_t *admq; uint64_t q_head, q_tail;   /* FIFO admission queue (capacity n) */
  uint64_t nreq, nkv, pend_n, pend_kv;
  int busy; double end, ebusy /* W*ms */, bms; uint64_t iters;
  uint64_t h;       /* decision-hash chain of this instance's controller decisions [A36] */
  double sum_itl;   /* ITL-mean sum of this instance's completions, completion order [A37] */
  double top;       /* ms at the top level [A37] */
  int cur;          /* ladder index the GPU runs at [C2] */
  double last_dec;  /* time of the last controller decision (-inf: none) [C1] */
} dec_inst;

typedef struct {
  uint64_t qhead;          /* first id (== p mod N_P) not yet batched [A7] */
  uint64_t bstart, bcnt;   /* ids of the batch in flight: bstart + j*N_P */
  int busy; double end, ebusy /* W*ms */, bms; uint64_t iters;
  uint64_t h;       /* decision-hash chain of this instance's controller decisions [A36] */
  double sum_ttft;  /* TTFT sum of this instance's completions, completion order [A37] */
  double top;       /* ms at the top level [A37] */
  int cur;          /* ladder index the GPU runs at [C2] */
  double last_dec;  /* time of the last controller decision (-inf: none) [C1] */
} pre_inst;

static int validate(const orc_scenario *s) {
  if (!s->prof || !s->ladder || s->K < 1 || s->K > 64) return 0;
  const orc_profile *p = s->prof;
  if (p->k < 1 || p->n_tiles < 1 || p->tile_w < 1) return 0;
  for (int k = 0; k < s->K; ++k) {
    if (s->ladder[k] >= p->k) return 0;
    if (k > 0 && s->ladder[k] <= s->ladder[k - 1]) return 0;
  }
  if (s->n_p < 1 || s->n_d < 1 || s->n_p > 64 || s->n_d > 64) return 0;
  if (s->policy < 0 || s->policy > 2 || s->ctrl_mode < 0 || s->ctrl_mode > 1) return 0;
  if (!(s->ctrl_interval_ms >= 0.0 && s->ctrl_interval_ms < 1e12)) return 0;
  if (!(s->freq_overhead_ms >= 0.0 && s->freq_overhead_ms < 1e9)) return 0;
  if (s->noise && (s->noise_len == 0 || (s->noise_len & (s->noise_len - 1)) != 0)) return 0;
  if (s->itl_mode < 0 || s->itl_mode > 2) return 0;
  if (s->max_batch_tokens == 0 || s->kv_capacity == 0) return 0;
  if (s->max_batch_tokens > 0x7fffffffu || s->kv_capacity > 0x7fffffffu) return 0;
  if (!(s->slo_ttft > 0.0) || !(s->slo_itl > 0.0) || !(s->slo_scale > 0.0)) return 0;
  if (!(s->kv_transfer_ms == 0.0 || s->kv_transfer_ms >= 1e-3)) return 0;
  if (!(s->duration_ms >= 0.0)) return 0;
  uint64_t tok = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    if (s->in_len[i] < 1 || s->out_len[i] < 1 || s->in_len[i] > 65535u || s->out_len[i] > 65535u)
      return 0;
    if (!(s->arrival[i] >= 0.0) || !(s->arrival[i] < 1e9)) return 0;
    if (i > 0 && s->arrival[i] < s->arrival[i - 1]) return 0;
    tok += (uint64_t)s->in_len[i] + s->out_len[i];
  }
  if (tok > 0x7fffffffull) return 0;
  return 1;
}

int oracle_simulate(const orc_scenario *s, orc_result *res, orc_diag *diag) {
  memset(res, 0, sizeof(*res));
  res->n_requests = (uint32_t)s->n;
  if (!validate(s)) { res->status = ORC_E_INPUT; return 0; }

  const orc_profile *p = s->prof;
  const uint16_t *L = s->ladder;
  const int K = s->K, NP = s->n_p, ND = s->n_d;
  const uint64_t N = s->n;
  const double *arr = s->arrival;
  const uint32_t *in = s->in_len, *out = s->out_len;
  const double tau = s->kv_transfer_ms;
  /* controller targets: SLO with margin s (default 1.0) [A3] */
  const double tgt_ttft = s->slo_scale * s->slo_ttft;
  const double tgt_itl = s->slo_scale * s->slo_itl;

  pre_inst *P = calloc((size_t)NP, sizeof(pre_inst));
  dec_inst *D = calloc((size_t)ND, sizeof(dec_inst));
  double *tfirst = calloc(N ? N : 1, sizeof(double));
  uint8_t *ttft_ok = calloc(N ? N : 1, 1);
  uint32_t *xq_id = malloc((N ? N : 1) * sizeof(uint32_t)); /* KV-transfer FIFO [A18] */
  uint32_t *xq_d = malloc((N ? N : 1) * sizeof(uint32_t));
  uint64_t xq_head = 0, xq_tail = 0;
  /* ITL Max / P99 [E3]: every request's token times (last token, running max, all gaps) */
  double *last_tok = NULL, *maxgap = NULL, *gapbuf = NULL;
  uint64_t *gap_off = NULL, *gap_n = NULL;
  if (s->itl_mode != 0) {
    last_tok = calloc(N ? N : 1, sizeof(double));
    maxgap = calloc(N ? N : 1, sizeof(double));
    if (s->itl_mode == 2) {
      gap_off = calloc(N + 1, sizeof(uint64_t));
      gap_n = calloc(N ? N : 1, sizeof(uint64_t));
      for (uint64_t i = 0; i < N; ++i) gap_off[i + 1] = gap_off[i] + (out[i] > 1 ? out[i] - 1 : 0);
      gapbuf = malloc((gap_off[N] ? gap_off[N] : 1) * sizeof(double));
    }
  }
  uint64_t *eff_n = malloc((size_t)ND * sizeof(uint64_t));
  uint64_t *eff_kv = malloc((size_t)ND * sizeof(uint64_t));
  for (int q = 0; q < NP; ++q) {
    P[q].qhead = (uint64_t)q;
    P[q].h = s->hash_seed;
    P[q].cur = K - 1; /* the GPU starts at the top of the ladder [C2] */
    P[q].last_dec = -INFINITY;
  }
  for (int d = 0; d < ND; ++d) {
    D[d].cur = K - 1;
    D[d].last_dec = -INFINITY;
    D[d].h = s->hash_seed;
    D[d].cap_run = 16;
    D[d].run = malloc(D[d].cap_run * sizeof(run_entry));
    D[d].admq = malloc((N ? N : 1) * sizeof(uint32_t));
  }

  uint64_t a = 0;           /* next arrival */
  uint32_t cursor = 0;      /* EcoRoute / round-robin cursor [A17] */
  uint64_t h = s->hash_seed; /* routing-decision chain [A36] */
  uint64_t steps_ctrl = 0, steps_route = 0, n_ttft_ok = 0, n_itl_ok = 0, n_both = 0;
  double t = 0.0, t_last = 0.0;
  uint64_t force_pos = 0;
  uint32_t status = ORC_OK;

  for (;;) {
    /* O1: next event time = min over pending events */
    int have = 0;
    double tn = 0.0;
    if (a < N) { tn = arr[a]; have = 1; }
    if (xq_head < xq_tail) {
      double tx = tfirst[xq_id[xq_head]] + tau;
      if (!have || tx < tn) { tn = tx; have = 1; }
    }
    for (int q = 0; q < NP; ++q)
      if (P[q].busy && (!have || P[q].end < tn)) { tn = P[q].end; have = 1; }
    for (int d = 0; d < ND; ++d)
      if (D[d].busy && (!have || D[d].end < tn)) { tn = D[d].end; have = 1; }
    if (!have) break;
    t = tn;
    t_last = t;

    /* O2: drain every event at time t in (kind, id) order:
     * Arrival < KvTransferDone < PrefillDone < DecodeIterDone [A18] */
    while (a < N && arr[a] == t) a++; /* O3: request a joins prefill queue a mod N_P [A7] */

    while (xq_head < xq_tail && tfirst[xq_id[xq_head]] + tau == t) { /* O4 [A12] */
      uint32_t i = xq_id[xq_head], d = xq_d[xq_head];
      xq_head++;
      D[d].admq[D[d].q_tail++] = i;
      if (diag && diag->req_tqueue) diag->req_tqueue[i] = t;
    }

    for (int q = 0; q < NP; ++q) { /* O5: PrefillDone(q) */
      if (!(P[q].busy && P[q].end == t)) continue;
      for (uint64_t j = 0; j < P[q].bcnt; ++j) {
        uint64_t i = P[q].bstart + j * (uint64_t)NP;
        double ttft = t - arr[i]; /* TTFT = waiting + execution [A26] */
        P[q].sum_ttft += ttft;
        int ok = ttft <= s->slo_ttft;
        n_ttft_ok += (uint64_t)ok;
        ttft_ok[i] = (uint8_t)ok;
        tfirst[i] = t;
        if (last_tok) last_tok[i] = t; /* the first token [E3] */
        if (diag && diag->req_tfirst) diag->req_tfirst[i] = t;
        if (out[i] == 1) { /* first token came from prefill; nothing to decode [A8, A30] */
          n_itl_ok++;
          n_both += (uint64_t)ok;
          if (diag && diag->req_tdone) diag->req_tdone[i] = t;
          if (diag && diag->req_decode) diag->req_decode[i] = -1;
          if (diag && diag->req_itl) diag->req_itl[i] = 0.0;
          continue;
        }
        int cse, d;
        if (diag && diag->force_decode) {
          d = diag->force_decode[i];
          cse = 15; /* forced (test hook), not a routing case */
        } else {
          for (int e = 0; e < ND; ++e) { /* effective state = running + pending [A9] */
            eff_n[e] = D[e].nreq + D[e].pend_n;
            eff_kv[e] = D[e].nkv + D[e].pend_kv;
          }
          d = ecoroute(p, L, K, ND, eff_n, eff_kv, in[i], tgt_itl, s->delta_mhz, s->policy,
                       &cursor, &cse);
        }
        steps_route++;
        h = fold(h, 3, (uint64_t)d, 0, (uint64_t)cse);
        if (diag && diag->req_decode) diag->req_decode[i] = d;
        if (diag && diag->req_case) diag->req_case[i] = (uint8_t)cse;
        D[d].pend_n += 1;
        D[d].pend_kv += (uint64_t)in[i] + 1;
        if (tau == 0.0) {
          D[d].admq[D[d].q_tail++] = (uint32_t)i;
          if (diag && diag->req_tqueue) diag->req_tqueue[i] = t;
        } else {
          xq_id[xq_tail] = (uint32_t)i;
          xq_d[xq_tail] = (uint32_t)d;
          xq_tail++;
        }
      }
      P[q].busy = 0;
    }

    for (int d = 0; d < ND; ++d) { /* O6: DecodeIterDone(d) [A19] */
      dec_inst *I = &D[d];
      if (!(I->busy && I->end == t)) continue;
      I->nkv += I->nreq; /* every running request stored one more token */
      uint64_t w = 0;
      for (uint64_t r = 0; r < I->n_run; ++r) {
        run_entry e = I->run[r];
        e.rem -= 1;
        if (last_tok) { /* this iteration produced one token for every running request [E3] */
          double gap = t - last_tok[e.id];
          last_tok[e.id] = t;
          if (gap > maxgap[e.id]) maxgap[e.id] = gap;
          if (gapbuf) gapbuf[gap_off[e.id] + gap_n[e.id]++] = gap;
        }
        if (e.rem == 0) {
          uint32_t id = e.id;
          /* per-request ITL = mean inter-token latency [A30] */
          double itl = (t - tfirst[id]) / (double)(out[id] - 1);
          I->sum_itl += itl;
          int ok = itl <= s->slo_itl;
          if (s->itl_mode == 1) ok = maxgap[id] <= s->slo_itl; /* ITL Max [E3] */
          if (s->itl_mode == 2) ok = p99_nearest_rank(gapbuf + gap_off[id], gap_n[id]) <= s->slo_itl;
          n_itl_ok += (uint64_t)ok;
          n_both += (uint64_t)(ok && ttft_ok[id]);
          I->nreq -= 1;
          I->nkv -= (uint64_t)in[id] + out[id];
          if (diag && diag->req_tdone) diag->req_tdone[id] = t;
          if (diag && diag->req_itl) diag->req_itl[id] = itl;
        } else {
          I->run[w++] = e;
        }
      }
      I->n_run = w;
      I->busy = 0;
    }

    /* O7: START phase, prefill 0..N_P-1 then decode 0..N_D-1 [A18] */
    for (int q = 0; q < NP && status == ORC_OK; ++q) {
      pre_inst *I = &P[q];
      if (I->busy || I->qhead >= a) continue;
      /* FCFS prefix with sum(in) <= B, at least one request [A6] */
      uint64_t id = I->qhead, nbt = 0, cnt = 0;
      while (id < a) {
        if (cnt > 0 && nbt + in[id] > s->max_batch_tokens) break;
        nbt += in[id];
        cnt++;
        id += (uint64_t)NP;
      }
      int backlog = id < a; /* requests still waiting after the batch [A5] */
      double wait = t - arr[I->qhead];
      int k = I->cur;
      int decided = 0;
      /* window gating: decide only when the interval has elapsed since
       * the last decision, boundary inclusive; interval 0 = every iteration [C1] */
      if (t - I->last_dec >= s->ctrl_interval_ms) {
        decided = 1;
        if (diag && diag->force_level && force_pos < diag->n_force_level) {
          k = diag->force_level[force_pos++];
        } else {
          /* EcoFreq: backlog -> max frequency; else lowest feasible */
          double bud = prefill_budget(tgt_ttft, wait);
          k = backlog ? K - 1
                      : (s->ctrl_mode == 1 ? energy_level_ttft(p, L, K, nbt, bud)
                                           : lowest_feasible_ttft(p, L, K, nbt, bud));
        }
        steps_ctrl++;
        I->h = fold(I->h, 1, (uint64_t)q, (uint64_t)k, 0);
        I->last_dec = t;
      }
      /* blocking frequency set: the iteration starts after the overhead when the level
       * changes [C3] */
      int paid = k != I->cur && s->freq_overhead_ms > 0.0;
      double t0 = paid ? t + s->freq_overhead_ms : t;
      I->cur = k;
      double dur = predict_ttft(p, L[k], nbt); /* execution time = prediction (noise 0) [A25] */
      if (!(dur > 0.0)) { status = ORC_E_CONTRACT; break; }
      if (s->noise) { /* true time = prediction x lognormal factor [D1] */
        double e = noise_factor(s, (uint64_t)q, I->iters);
        if (!(e > 0.0 && e <= 1e6)) { status = ORC_E_INPUT; break; }
        dur = dur * e;
      }
      if (diag && diag->iter_n < diag->iter_cap) {
        diag->iter_inst[diag->iter_n] = q;
        diag->iter_level[diag->iter_n] = (uint16_t)k;
        diag->iter_dur[diag->iter_n] = dur;
        diag->iter_target[diag->iter_n] = prefill_budget(tgt_ttft, wait);
        if (diag->iter_start) diag->iter_start[diag->iter_n] = t;
        if (diag->iter_load) diag->iter_load[diag->iter_n] = (uint32_t)nbt;
        if (diag->iter_kv) diag->iter_kv[diag->iter_n] = 0;
        if (diag->iter_flags) diag->iter_flags[diag->iter_n] = (uint8_t)(decided | paid << 1 | backlog << 2);
        diag->iter_n++;
      }
      I->end = t0 + dur;
      I->busy = 1;
      I->bstart = I->qhead;
      I->bcnt = cnt;
      I->qhead = id;
      I->ebusy += busy_power(p, 0, L[k], nbt) * dur; /* W*ms; converted to J once [A23] */
      I->bms += dur;
      I->iters++;
      if (k == K - 1) I->top += dur;
    }
    for (int d = 0; d < ND && status == ORC_OK; ++d) {
      dec_inst *I = &D[d];
      if (I->busy) continue;
      /* admission at the iteration boundary, FCFS while KV fits [A20] */
      while (I->q_head < I->q_tail) {
        uint32_t hd = I->admq[I->q_head];
        uint64_t need = (uint64_t)in[hd] + 1;
        if (I->nkv + need > s->kv_capacity) break;
        I->q_head++;
        if (I->n_run == I->cap_run) {
          I->cap_run *= 2;
          I->run = realloc(I->run, I->cap_run * sizeof(run_entry));
        }
        if (diag && diag->req_tadmit) diag->req_tadmit[hd] = t;
        I->run[I->n_run].id = hd;
        I->run[I->n_run].rem = out[hd] - 1;
        I->n_run++;
        I->nreq += 1;
        I->nkv += need;
        I->pend_n -= 1;
        I->pend_kv -= need;
      }
      if (I->nreq == 0) {
        if (I->q_head < I->q_tail) { status = ORC_E_SCENARIO_KV; break; }
        continue;
      }
      int backlog = I->q_head < I->q_tail; /* KV-blocked admission queue [A5] */
      int k = I->cur;
      int decided = 0;
      if (t - I->last_dec >= s->ctrl_interval_ms) { /* window gating [C1] */
        decided = 1;
        if (diag && diag->force_level && force_pos < diag->n_force_level) {
          k = diag->force_level[force_pos++];
        } else {
          k = backlog ? K - 1
                      : (s->ctrl_mode == 1 ? energy_level_itl(p, L, K, I->nreq, I->nkv, tgt_itl)
                                           : lowest_feasible_itl(p, L, K, I->nreq, I->nkv, tgt_itl));
        }
        steps_ctrl++;
        I->h = fold(I->h, 2, (uint64_t)d, (uint64_t)k, 0);
        I->last_dec = t;
      }
      int paid = k != I->cur && s->freq_overhead_ms > 0.0; /* [C3] */
      double t0 = paid ? t + s->freq_overhead_ms : t;
      I->cur = k;
      double dur = predict_itl(p, L[k], I->nreq, I->nkv);
      if (!(dur > 0.0)) { status = ORC_E_CONTRACT; break; }
      if (s->noise) { /* [D1] */
        double e = noise_factor(s, (uint64_t)(NP + d), I->iters);
        if (!(e > 0.0 && e <= 1e6)) { status = ORC_E_INPUT; break; }
        dur = dur * e;
      }
      if (diag && diag->time_busy) diag->time_busy[d] += dur;
      if (diag && diag->time_le_boundary && I->nreq <= diag->boundary) diag->time_le_boundary[d] += dur;
      if (diag && diag->max_nreq && I->nreq > diag->max_nreq[d]) diag->max_nreq[d] = (uint32_t)I->nreq;
      if (diag && diag->tokens) diag->tokens[d] += I->nreq;
      if (diag && diag->kv_peak && I->nkv > diag->kv_peak[d]) diag->kv_peak[d] = I->nkv;
      if (diag && diag->iter_n < diag->iter_cap) {
        diag->iter_inst[diag->iter_n] = NP + d;
        diag->iter_level[diag->iter_n] = (uint16_t)k;
        diag->iter_dur[diag->iter_n] = dur;
        diag->iter_target[diag->iter_n] = tgt_itl;
        if (diag->iter_start) diag->iter_start[diag->iter_n] = t;
        if (diag->iter_load) diag->iter_load[diag->iter_n] = (uint32_t)I->nreq;
        if (diag->iter_kv) diag->iter_kv[diag->iter_n] = (uint32_t)I->nkv;
        if (diag->iter_flags) diag->iter_flags[diag->iter_n] = (uint8_t)(decided | paid << 1 | backlog << 2);
        diag->iter_n++;
      }
      I->end = t0 + dur;
      I->busy = 1;
      I->ebusy += busy_power(p, 1, L[k], I->nreq) * dur; /* W*ms [A23] */
      I->bms += dur;
      I->iters++;
      if (k == K - 1) I->top += dur;
    }
    if (status != ORC_OK) break;
  }

  if (status == ORC_OK) {
    /* O9: horizon and idle energy [A23, A39] */
    double horizon = s->duration_ms > t_last ? s->duration_ms : t_last;
    double epb = 0.0, epi = 0.0, edb = 0.0, edi = 0.0, bp = 0.0, bd = 0.0;
    double sum_ttft = 0.0, sum_itl = 0.0, top_ms = 0.0;
    /* decision identity: route chain, then every prefill chain, then every decode chain [A36] */
    uint64_t hh = splitmix64(h);
    for (int q = 0; q < NP; ++q) hh = splitmix64(hh ^ P[q].h);
    for (int d = 0; d < ND; ++d) hh = splitmix64(hh ^ D[d].h);
    /* report-only totals: per-instance sums added in instance order [A37] */
    for (int q = 0; q < NP; ++q) { sum_ttft += P[q].sum_ttft; top_ms += P[q].top; }
    for (int d = 0; d < ND; ++d) { sum_itl += D[d].sum_itl; top_ms += D[d].top; }
    for (int q = 0; q < NP; ++q) {
      epb += P[q].ebusy / 1000.0; /* J = (sum of P*dur in W*ms) / 1000 per instance [A23] */
      epi += interval_energy(p->p_idle, horizon - P[q].bms);
      bp += P[q].bms;
    }
    for (int d = 0; d < ND; ++d) {
      edb += D[d].ebusy / 1000.0;
      edi += interval_energy(p->p_idle, horizon - D[d].bms);
      bd += D[d].bms;
    }
    res->status = ORC_OK;
    res->n_ttft_ok = (uint32_t)n_ttft_ok;
    res->n_itl_ok = (uint32_t)n_itl_ok;
    res->n_both_ok = (uint32_t)n_both;
    {
      uint64_t pi = 0;
      for (int q = 0; q < NP; ++q) pi += P[q].iters;
      res->prefill_iters = (uint32_t)pi;
    }
    res->steps_ctrl = steps_ctrl;
    res->steps_route = steps_route;
    res->decision_hash = hh;
    res->sum_ttft_ms = sum_ttft;
    res->sum_itl_mean_ms = sum_itl;
    res->e_prefill_busy_j = epb;
    res->e_prefill_idle_j = epi;
    res->e_decode_busy_j = edb;
    res->e_decode_idle_j = edi;
    res->busy_ms_prefill = bp;
    res->busy_ms_decode = bd;
    res->top_level_ms = top_ms;
    res->horizon_ms = horizon;
    if (diag && diag->iters) {
      for (int q = 0; q < NP; ++q) diag->iters[q] = P[q].iters;
      for (int d = 0; d < ND; ++d) diag->iters[NP + d] = D[d].iters;
    }
  } else {
    res->status = status; /* per-scenario error: status and n_requests only */
  }

  for (int d = 0; d < ND; ++d) { free(D[d].run); free(D[d].admq); }
  free(P); free(D); free(tfirst); free(ttft_ok); free(xq_id); free(xq_d); free(eff_n); free(eff_kv);
  free(last_tok); free(maxgap); free(gapbuf); free(gap_off); free(gap_n);
  return 0;
}

/* ------------------------------------------------ single-decision oracles */

int oracle_control_step(const orc_profile *p, int phase, int mode, const uint16_t *L, int K,
                        const uint32_t *load, const uint32_t *n_kv, const uint32_t *queue_len,
                        const double *wait_ms, const double *target_ms, size_t n,
                        uint16_t *out_level, uint8_t *out_status) {
  for (size_t i = 0; i < n; ++i) {
    int bad = load[i] == 0 || (phase == 1 && n_kv[i] < load[i]);
    if (bad) { out_level[i] = 0xFFFF; out_status[i] = (uint8_t)ORC_E_CONTRACT; continue; }
    int k;
    if (queue_len[i] > 0) {
      k = K - 1; /* backlog -> max frequency */
    } else if (phase == 0) {
      double bud = prefill_budget(target_ms[i], wait_ms[i]);
      k = mode == 1 ? energy_level_ttft(p, L, K, load[i], bud) : lowest_feasible_ttft(p, L, K, load[i], bud);
    } else { /* no wait subtraction */
      k = mode == 1 ? energy_level_itl(p, L, K, load[i], n_kv[i], target_ms[i])
                    : lowest_feasible_itl(p, L, K, load[i], n_kv[i], target_ms[i]);
    }
    out_level[i] = (uint16_t)k;
    out_status[i] = (uint8_t)ORC_OK;
  }
  return 0;
}

int oracle_route_batch(const orc_profile *p, const uint16_t *L, int K, int n_d,
                       const uint32_t *n_req, const uint32_t *n_kv, const uint32_t *req_in,
                       const double *itl_target, int32_t delta_mhz, int policy,
                       uint32_t *cursor, size_t n, uint16_t *out_instance,
                       uint8_t *out_case, uint8_t *out_status) {
  uint64_t nn[64], kk[64];
  for (size_t i = 0; i < n; ++i) {
    int bad = cursor[i] >= (uint32_t)n_d || req_in[i] == 0;
    for (int d = 0; d < n_d; ++d) {
      nn[d] = n_req[i * (size_t)n_d + (size_t)d];
      kk[d] = n_kv[i * (size_t)n_d + (size_t)d];
      if (kk[d] < nn[d]) bad = 1;
    }
    if (bad) { out_instance[i] = 0xFFFF; out_case[i] = 0xFF; out_status[i] = (uint8_t)ORC_E_CONTRACT; continue; }
    int cse;
    int d = ecoroute(p, L, K, n_d, nn, kk, req_in[i], itl_target[i], delta_mhz, policy, &cursor[i], &cse);
    out_instance[i] = (uint16_t)d;
    out_case[i] = (uint8_t)cse;
    out_status[i] = (uint8_t)ORC_OK;
  }
  return 0;
}

/* ------------------------------------------------------------------ fitter */

/* cell_status codes */
#define FIT_OK 0
#define FIT_INHERITED 1
#define FIT_EMPTY 2
#define FIT_DEGENERATE 3

/* prefill tile of a sample, as ptile_index [F1] */
static size_t fit_ptile(uint32_t nbt, int Tp, uint32_t cutoff, int W) {
  if (Tp <= 1) return 0;
  if (nbt > cutoff) return (size_t)(Tp - 1);
  uint32_t j = (nbt - 1) / (uint32_t)W;
  return j < (uint32_t)(Tp - 1) ? (size_t)j : (size_t)(Tp - 1);
}

int oracle_fit_profile(const uint8_t *phase, const uint16_t *level, const uint32_t *n_bt,
                       const uint32_t *n_req, const uint32_t *n_kv, const double *lat_ms,
                       size_t n, int K, int T, int W, double tile_step, int Tp, uint32_t cutoff,
                       double *a1, double *c1, double *a2, double *b2, double *c2,
                       double *mae, uint8_t *cell_status) {
  /* F1: cells. TTFT cell (prefill, level k, prefill tile jp) = index jp*K + k; ITL cell
   * (decode, level k, tile j) = index Tp*K + j*K + k, tile j = min(T-1, (N_req-1)/W)
   * (prefill tiles P:880-885). Tp <= 1: one prefill tile. */
  if (Tp < 1) Tp = 1;
  const size_t KP = (size_t)Tp * (size_t)K;
  const size_t C = KP + (size_t)T * (size_t)K;
  for (size_t i = 0; i < n; ++i) {
    if (phase[i] > 1 || level[i] >= K) return 1;
    if (phase[i] == 1 && n_req[i] == 0) return 1;
    if (phase[i] == 0 && n_bt[i] == 0) return 1;
  }
  #define CELL(i) (phase[i] == 0 ? fit_ptile(n_bt[i], Tp, cutoff, W) * (size_t)K + level[i] : \
      KP + (size_t)((n_req[i] - 1) / (uint32_t)W < (uint32_t)(T - 1) ? (n_req[i] - 1) / (uint32_t)W : (uint32_t)(T - 1)) * (size_t)K + level[i])
  double *cnt = calloc(C, sizeof(double));
  double *s1 = calloc(C, sizeof(double)), *s2 = calloc(C, sizeof(double)), *sy = calloc(C, sizeof(double));
  /* pass 1: means, sequential sums in sample order */
  for (size_t i = 0; i < n; ++i) {
    size_t c = CELL(i);
    cnt[c] += 1.0;
    if (phase[i] == 0) { s1[c] += (double)n_bt[i]; }
    else { s1[c] += (double)n_req[i]; s2[c] += (double)n_kv[i]; }
    sy[c] += lat_ms[i];
  }
  double *m1 = calloc(C, sizeof(double)), *m2 = calloc(C, sizeof(double)), *my = calloc(C, sizeof(double));
  for (size_t c = 0; c < C; ++c) {
    if (cnt[c] > 0.0) { m1[c] = s1[c] / cnt[c]; m2[c] = s2[c] / cnt[c]; my[c] = sy[c] / cnt[c]; }
  }
  /* pass 2: centred sums of squares and cross products */
  double *S11 = calloc(C, sizeof(double)), *S12 = calloc(C, sizeof(double)), *S22 = calloc(C, sizeof(double));
  double *S1y = calloc(C, sizeof(double)), *S2y = calloc(C, sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    size_t c = CELL(i);
    double dx1 = (phase[i] == 0 ? (double)n_bt[i] : (double)n_req[i]) - m1[c];
    double dy = lat_ms[i] - my[c];
    S11[c] += dx1 * dx1;
    S1y[c] += dx1 * dy;
    if (phase[i] == 1) {
      double dx2 = (double)n_kv[i] - m2[c];
      S12[c] += dx1 * dx2;
      S22[c] += dx2 * dx2;
      S2y[c] += dx2 * dy;
    }
  }
  int err = 0;
  /* F2: TTFT per (prefill tile, level): a = Sxy / Sxx, c = ybar - a xbar; needs >= 2 distinct
   * N_bt [A31]; an empty prefill tile jp > 0 inherits jp - 1 with the step on c1 [F2] */
  for (int jp = 0; jp < Tp; ++jp) {
    for (int k = 0; k < K; ++k) {
      size_t c = (size_t)jp * (size_t)K + (size_t)k;
      if (cnt[c] == 0.0) {
        if (jp == 0) { cell_status[c] = FIT_EMPTY; a1[c] = c1[c] = 0.0; err = 1; }
        else { a1[c] = a1[c - (size_t)K]; c1[c] = c1[c - (size_t)K] + tile_step; cell_status[c] = FIT_INHERITED; }
        continue;
      }
      if (cnt[c] < 2.0 || !(S11[c] > 0.0)) { cell_status[c] = FIT_DEGENERATE; a1[c] = c1[c] = 0.0; err = 1; continue; }
      a1[c] = S1y[c] / S11[c];
      c1[c] = my[c] - (a1[c] * m1[c]);
      cell_status[c] = FIT_OK;
    }
  }
  /* F3/F4: ITL per (tile, level), two regressors; empty tile j>0 inherits j-1 + step */
  for (int j = 0; j < T; ++j) {
    for (int k = 0; k < K; ++k) {
      size_t c = KP + (size_t)j * (size_t)K + (size_t)k;
      size_t o = (size_t)j * (size_t)K + (size_t)k;
      if (cnt[c] == 0.0) {
        if (j == 0) { cell_status[c] = FIT_EMPTY; a2[o] = b2[o] = c2[o] = 0.0; err = 1; }
        else {
          size_t pv = o - (size_t)K;
          a2[o] = a2[pv]; b2[o] = b2[pv]; c2[o] = c2[pv] + tile_step;
          cell_status[c] = FIT_INHERITED;
        }
        continue;
      }
      double pr = S11[c] * S22[c];
      double det = (S11[c] * S22[c]) - (S12[c] * S12[c]);
      if (cnt[c] < 3.0 || !(pr > 0.0) || !(det > 1e-10 * pr)) {
        cell_status[c] = FIT_DEGENERATE; a2[o] = b2[o] = c2[o] = 0.0; err = 1; continue;
      }
      a2[o] = ((S22[c] * S1y[c]) - (S12[c] * S2y[c])) / det;
      b2[o] = ((S11[c] * S2y[c]) - (S12[c] * S1y[c])) / det;
      c2[o] = (my[c] - (a2[o] * m1[c])) - (b2[o] * m2[c]);
      cell_status[c] = FIT_OK;
    }
  }
  /* F5: mean absolute error per cell, same evaluation order as EcoPred */
  double *ae = calloc(C, sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    size_t c = CELL(i);
    if (cell_status[c] != FIT_OK) continue;
    double yh;
    if (phase[i] == 0) {
      yh = (a1[c] * (double)n_bt[i]) + c1[c];
    } else {
      size_t o = c - KP;
      yh = ((a2[o] * (double)n_req[i]) + (b2[o] * (double)n_kv[i])) + c2[o];
    }
    ae[c] += fabs(lat_ms[i] - yh);
  }
  for (size_t c = 0; c < C; ++c) mae[c] = (cell_status[c] == FIT_OK) ? ae[c] / cnt[c] : 0.0;
  #undef CELL
  free(cnt); free(s1); free(s2); free(sy); free(m1); free(m2); free(my);
  free(S11); free(S12); free(S22); free(S1y); free(S2y); free(ae);
  return err ? 4 : 0;
}

/* ------------------------------------------------------------- pin helpers */

double oracle_predict_ttft(const orc_profile *p, int level, uint32_t n_bt) { return predict_ttft(p, level, n_bt); }
double oracle_predict_itl(const orc_profile *p, int level, uint32_t n_req, uint32_t n_kv) {
  return predict_itl(p, level, n_req, n_kv);
}
int oracle_tile_index(const orc_profile *p, uint32_t n_req) { return tile_index(p, n_req); }
int oracle_ptile_index(const orc_profile *p, uint32_t n_bt) { return ptile_index(p, n_bt); }
double oracle_busy_power(const orc_profile *p, int phase, int level, uint32_t load) {
  return busy_power(p, phase, level, load);
}
double oracle_interval_energy(double power_w, double dur_ms) { return interval_energy(power_w, dur_ms); }
