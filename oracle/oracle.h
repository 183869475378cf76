/*
 * oracle/oracle.h -- records shared by the oracle's own translation units.
 * TEST INFRASTRUCTURE ONLY; never included by the product (include/, paper_2502_03796_b200/).
 * oracle/oracle.py mirrors these layouts with ctypes.
 */
#ifndef MAGUS_ORACLE_H
#define MAGUS_ORACLE_H
#include <cstdint>
extern "C" {
/* ---- the oracle's own parameter / result records (ctypes mirrors them in oracle/oracle.py) ---- */

enum { O_MAGUS = 0, O_STATIC_MAX = 1, O_STATIC_MIN = 2, O_TDP_DEFAULT = 3 };
enum { O_LO = 0, O_HI = 1 };

typedef struct {
    int32_t kind;                 /* O_MAGUS / O_STATIC_MAX / O_STATIC_MIN / O_TDP_DEFAULT */
    int32_t deriv_ticks;          /* k: direv_length = k * sample_period  ([A2]) */
    double  inc_threshold;        /* GB/s per s  ([A3]) */
    double  dec_threshold;        /* GB/s per s */
    int32_t tune_log_capacity;    /* C = len(uncore_tune_ls) when full  ([A6]) */
    int32_t _pad;
    double  high_freq_threshold;  /* 0.6 in the paper */
    double  tdp_w;                /* TDP_DEFAULT only ([A24]) */
    double  tdp_margin;
} OPolicy;

typedef struct {
    double  sample_period_s;      /* Delta [A1] */
    double  f_min_ghz, f_max_ghz; /* 0.8 / 2.2 GHz */
    double  bw_max_gbps;          /* bandwidth at f_max */
    int32_t bw_shape;             /* 0 Linear, 1 Saturating */
    int32_t observe;              /* 0 closed loop: A = min(D, B[f]) [A14]; 1 open loop: the recorded
                                     throughput is observed as is, A = D [A30] */
    double  bw_knee;
    double  p_pkg_idle_w, p_core_active_w, p_uncore_min_w, p_uncore_max_w, p_exponent;
    double  p_gpu_active_w;       /* GPU power while the trace runs */
    double  dram_w_per_gbps;      /* DRAM power proxy, TDP predicate only ([A20]) */
} OModel;

typedef struct {
    int64_t  n_hi;          /* ticks spent at f_max */
    int64_t  n_thr;         /* throttled ticks (achieved < demand) */
    int64_t  transitions;   /* ticks with cmd != level in effect [A25] */
    int64_t  tune_events;   /* 1-flags pushed into uncore_tune_ls */
    int64_t  lock_ticks;    /* ticks where Alg. 2 returned True */
    double   T;             /* execution time, s */
    double   E_pkg;         /* CPU package energy, J */
    double   E;             /* package + GPU energy, J */
    double   EDP;           /* E * T */
    double   T_base, E_base;                 /* static-max baseline on the same trace [A21] */
    double   slowdown;                       /* perf loss as a fraction */
    double   energy_saving, edp_saving, pkg_power_saving;   /* fractions */
    uint64_t digest;        /* sum over 32-tick blocks of mix64(words ^ b*PHI) */
    int32_t  status;        /* 0 ok, 2 = bad sample (err_tick set) */
    int32_t  _pad;
    int64_t  err_tick;
} OResult;


typedef struct {
    uint64_t seed;
    int32_t  n_traces;          /* local traces written */
    int32_t  class_mix;         /* 0 cfg2, 1 cfg3/4, 2 cfg5 adversarial, 3 cfg1 concatenated */
    int64_t  n_samples;
    int64_t  trace_stride;      /* floats between time rows (>= n_traces) */
    int64_t  global_trace_offset;
    float    noise_amp;         /* a, default 0.002 */
    float    _pad;
    double   bw_max_gbps;       /* clamp bound */
} OGenDesc;

int   oracle_replay(const float* D, int64_t n, int64_t stride, float w, const OPolicy* pol,
                    const OModel* m, OResult* out, uint8_t* codes, int64_t codes_stride);
float oracle_gen_trace(const OGenDesc* g, int64_t j_local, float* col, int64_t col_stride);
}
#endif
