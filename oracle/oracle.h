/* oracle.h — TEST INFRASTRUCTURE ONLY (parity oracle for the VoltanaLLM hot path).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load liboracle.so. The product path
 * (paper_2509_04827_b200/) never includes, links or calls anything here, and
 * this directory shares no code, header, table or constant with csrc/.
 *
 * Citations: P:NNN = PAPER.md line, S:NNN = SPEC.md line.
 * Every function follows the paper's algorithm step by step in plain
 * sequential C: IEEE fp64, each operation rounded separately (built with
 * -ffp-contract=off, no -ffast-math).
 */
#ifndef VOLTANA_ORACLE_H
#define VOLTANA_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A calibrated profile: EcoPred tables per frequency level (eq:pred-ttft P:514,
 * eq:pred-itl P:516) and busy dynamic power per level and phase. */
typedef struct {
  int32_t k;             /* levels on the profile grid                       */
  int32_t n_tiles;       /* ITL tiles T                                      */
  int32_t tile_w;        /* tile width W (128)                        */
  int32_t n_ptiles;      /* prefill tiles T_p (<= 1: single tile) [F1]       */
  const int32_t *mhz;    /* [k] frequency of each level                      */
  const double *a1, *c1; /* [n_ptiles*k], row = prefill tile                 */
  const double *a2, *b2, *c2; /* [n_tiles*k], row = tile                     */
  const double *dyn;     /* [2*k] prefill row then decode row (W)            */
  double p_idle, tdp, uh_prefill, uh_decode;
  int32_t prefill_cutoff; /* N_bt above which prefill is the last tile [F1]  */
  int32_t pad2_;
} orc_profile;

/* One scenario: trace x SLO x layout x frequency ladder (BASELINE north_star). */
typedef struct {
  const double *arrival;  /* [n] ms, non-decreasing */
  const uint32_t *in_len; /* [n] >= 1 */
  const uint32_t *out_len;/* [n] >= 1 */
  uint64_t n;
  double duration_ms;
  double slo_ttft, slo_itl, slo_scale;
  int32_t n_p, n_d, policy;          /* policy 0 EcoRoute, 1 round-robin, 2 energy-scored [B1] */
  uint32_t max_batch_tokens, kv_capacity;
  double kv_transfer_ms;
  int32_t delta_mhz;                 /* INT32_MAX = "large value" */
  const uint16_t *ladder;            /* [K] ascending profile-level indices */
  int32_t K;
  const orc_profile *prof;
  uint64_t hash_seed;
  int32_t ctrl_mode;                 /* 0 EcoFreq lowest feasible, 1 energy argmin [B4] */
  double ctrl_interval_ms;           /* window control: decide when >= this elapsed (0 = every iteration) [C1] */
  double freq_overhead_ms;           /* blocking frequency-set delay on a level change (0 = non-blocking) [C3] */
  const double *noise;               /* [noise_len] execution-noise factors, NULL = none [D1, D2] */
  uint64_t noise_len;                /* power of two */
  int32_t itl_mode;                  /* per-request ITL for attainment: 0 mean, 1 max, 2 P99 [E3] */
  int32_t pad3_;
} orc_scenario;

/* 128-byte per-scenario result record. */
typedef struct {
  uint32_t status, n_requests, n_ttft_ok, n_itl_ok, n_both_ok, prefill_iters;
  uint64_t steps_ctrl, steps_route, decision_hash;
  double sum_ttft_ms, sum_itl_mean_ms, e_prefill_busy_j, e_prefill_idle_j,
         e_decode_busy_j, e_decode_idle_j, busy_ms_prefill, busy_ms_decode,
         top_level_ms, horizon_ms;
} orc_result;

/* Optional diagnostics and test hooks (all pointers may be NULL). */
typedef struct {
  double *req_tfirst;      /* [n] prefill end (first token) time            */
  double *req_tdone;       /* [n] last token time                           */
  double *req_itl;         /* [n] mean ITL (0 for out == 1)                 */
  int32_t *req_decode;     /* [n] decode instance, -1 if out == 1           */
  uint8_t *req_case;       /* [n] routing case 0..7 (15 = forced)           */
  uint64_t *iters;         /* [n_p + n_d] iterations started per instance  */
  double *time_le_boundary;/* [n_d] busy ms with n_req <= boundary          */
  double *time_busy;       /* [n_d] busy ms                                 */
  uint32_t *max_nreq;      /* [n_d]                                         */
  uint32_t boundary;
  const int32_t *force_decode; /* [n] forced decode instance per request (brute force) */
  const uint16_t *force_level; /* forced ladder index per controller decision, consumed in order */
  uint64_t n_force_level;
  uint64_t *tokens;        /* [n_d] sum of N_req over decode iterations (tokens generated) */
  uint64_t *kv_peak;       /* [n_d] max N_kv at an iteration start          */
  uint64_t iter_cap;       /* capacity of the iteration log (0 = no log)    */
  uint64_t iter_n;         /* out: iterations logged                        */
  int32_t *iter_inst;      /* [iter_cap] instance (prefill p, decode N_P+d) */
  uint16_t *iter_level;    /* [iter_cap] ladder index                       */
  double *iter_dur;        /* [iter_cap] duration ms                        */
  double *iter_target;     /* [iter_cap] controller target (budget) ms      */
  double *iter_start;      /* [iter_cap] START time t (the iteration runs from t + overhead) */
  uint32_t *iter_load;     /* [iter_cap] N_bt (prefill) / N_req (decode)     */
  uint32_t *iter_kv;       /* [iter_cap] N_kv (decode), 0 (prefill)          */
  uint8_t *iter_flags;     /* [iter_cap] bit0 decision, bit1 overhead, bit2 backlog */
  double *req_tadmit;      /* [n] time the request joined its decode running set (NaN: never) */
  double *req_tqueue;      /* [n] time it joined its decode admission queue (NaN: never)       */
} orc_diag;

/* status codes (result.status / per-item status) */
#define ORC_OK 0u
#define ORC_E_SCENARIO_KV 1u
#define ORC_E_CONTRACT 2u
#define ORC_E_INPUT 3u

int oracle_simulate(const orc_scenario *s, orc_result *res, orc_diag *diag);

/* mode 0 EcoFreq (lowest feasible), 1 energy argmin [B4] */
int oracle_control_step(const orc_profile *p, int phase, int mode, const uint16_t *ladder, int K,
                        const uint32_t *load, const uint32_t *n_kv, const uint32_t *queue_len,
                        const double *wait_ms, const double *target_ms, size_t n,
                        uint16_t *out_level, uint8_t *out_status);

int oracle_route_batch(const orc_profile *p, const uint16_t *ladder, int K, int n_d,
                       const uint32_t *n_req, const uint32_t *n_kv, const uint32_t *req_in,
                       const double *itl_target, int32_t delta_mhz, int policy,
                       uint32_t *cursor, size_t n, uint16_t *out_instance,
                       uint8_t *out_case, uint8_t *out_status);

int oracle_fit_profile(const uint8_t *phase, const uint16_t *level, const uint32_t *n_bt,
                       const uint32_t *n_req, const uint32_t *n_kv, const double *lat_ms,
                       size_t n, int K, int T, int W, double tile_step, int Tp, uint32_t cutoff,
                       double *a1, double *c1, double *a2, double *b2, double *c2,
                       double *mae, uint8_t *cell_status);

/* single predictor / energy evaluations (pins) */
double oracle_predict_ttft(const orc_profile *p, int level, uint32_t n_bt);
double oracle_predict_itl(const orc_profile *p, int level, uint32_t n_req, uint32_t n_kv);
int oracle_tile_index(const orc_profile *p, uint32_t n_req);
int oracle_ptile_index(const orc_profile *p, uint32_t n_bt);
double oracle_busy_power(const orc_profile *p, int phase, int level, uint32_t load);
double oracle_interval_energy(double power_w, double dur_ms);

#ifdef __cplusplus
}
#endif
#endif
