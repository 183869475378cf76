/*
 * include/magus_replay.h -- C ABI of the B200-native MAGUS batched replay.
 *
 * MAGUS (arXiv 2502.03796) is a periodic uncore-frequency control loop: read
 * memory throughput, predict its trend from the first
 * derivative over a FIFO window (Alg. 1), log whether a change was
 * requested, detect frequent changes (Alg. 2), force the
 * maximum uncore level while changes are frequent, otherwise execute the
 * temporary decision, jumping directly to the bounds.
 * This library replays that loop for many synthetic throughput traces and
 * many policy-parameter points at once on a B200 and reports the paper's
 * metrics (performance loss, package power saving, energy saving, EDP;
 * P:297-304) against the static-max / Intel-default baselines (P:119-136,
 * P:282).  The per-tick semantics, including every reading of the paper's
 * silences, are DESIGN.md sections 2-3.
 *
 * Conventions
 *  - Every call returns magus_status (0 = MAGUS_OK).  On failure
 *    magus_replay_last_error(handle) (or magus_last_error() for calls without
 *    a handle) names the problem; for MAGUS_ERR_CONFIG it names the violated
 *    key.
 *  - Handles are single-owner and not thread-safe; distinct
 *    handles may be used concurrently from different threads.
 *  - Device pointers are borrowed: they must stay valid and unmodified until
 *    the stream passes the run's completion (magus_replay_results waits for
 *    it).  The library owns all of its scratch and its NCCL communicator.
 *  - There is no CPU fallback: without a CUDA device every compute call
 *    returns MAGUS_ERR_CUDA.
 *  - Layout of a trace set: fp32, time-major / trace-minor, element (t, j) at
 *    trace[t * trace_stride + j]; trace_stride >= n_traces, trace_stride % 4
 *    == 0 and the base 16-byte aligned (TMA 2-D tiles); w[j] fp32 is trace j's
 *    compute_weight (A18).
 */
#ifndef MAGUS_REPLAY_H
#define MAGUS_REPLAY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAGUS_ABI_VERSION 2

typedef enum {
    MAGUS_OK = 0,
    MAGUS_ERR_INVALID_ARG = 1,  /* NULL where a pointer is required, negative sizes, bad dump window */
    MAGUS_ERR_CONFIG = 2,       /* a policy/model invariant is violated; last_error names the key */
    MAGUS_ERR_ALIGN = 3,        /* trace_stride % 4 != 0 or a trace base not 16-byte aligned */
    MAGUS_ERR_TRACE = 4,        /* a sample is negative, NaN/Inf or > bw_max (err_trace/err_tick set) */
    MAGUS_ERR_STATE = 5,        /* results before any run */
    MAGUS_ERR_OOM = 6,          /* device allocation failed */
    MAGUS_ERR_CUDA = 7,         /* CUDA runtime/driver error, or no CUDA device */
    MAGUS_ERR_NCCL = 8          /* NCCL missing or a collective failed */
} magus_status;

typedef enum {
    MAGUS_POLICY_MAGUS = 0,       /* Alg. 1 + Alg. 2 + override; starts at f_min */
    MAGUS_POLICY_STATIC_MAX = 1,  /* uncore pinned at f_max; the savings baseline (DESIGN A21) */
    MAGUS_POLICY_STATIC_MIN = 2,  /* uncore pinned at f_min */
    MAGUS_POLICY_TDP_DEFAULT = 3  /* Intel default: lowered only when pkg+DRAM power nears TDP */
} magus_policy_kind;

/* One policy-parameter point (SPEC GovernorConfig). */
typedef struct {
    int32_t kind;                 /* magus_policy_kind */
    int32_t deriv_ticks;          /* k in [1, 64]: direv_length = k * sample_period_s (DESIGN A2) */
    double  inc_threshold;        /* GB/s per s, > 0 (A3-A4) */
    double  dec_threshold;        /* GB/s per s, < 0 */
    int32_t tune_log_capacity;    /* C in [1, 64]: length of uncore_tune_ls when full (A6) */
    int32_t _reserved0;
    double  high_freq_threshold;  /* (0, 1]; the paper's 0.6 */
    double  tdp_w;                /* TDP_DEFAULT only: > 0 (A24) */
    double  tdp_margin;           /* TDP_DEFAULT only: (0, 1), default 0.05 */
} magus_policy;

/* Platform / energy model (SPEC simsys S:316-323; only the two endpoint levels are ever used, A19). */
typedef struct {
    double  sample_period_s;      /* Delta > 0, default 0.1 (A1) */
    double  f_min_ghz, f_max_ghz; /* 0 < f_min < f_max; 0.8 / 2.2 */
    double  bw_max_gbps;          /* > 0, bandwidth at f_max */
    int32_t bw_shape;             /* 0 Linear, 1 Saturating */
    int32_t observe;              /* 0 closed loop: the governor observes A = min(D, bandwidth(level)) (A14);
                                     1 open loop: the trace is a recorded throughput observed as is, A = D,
                                     never throttled (NEXT-3, DESIGN A30) */
    double  bw_knee;              /* Saturating only, (0, 1] */
    double  p_pkg_idle_w, p_core_active_w, p_uncore_min_w, p_uncore_max_w; /* >= 0, max >= min */
    double  p_exponent;           /* >= 1 */
    double  p_gpu_active_w;       /* >= 0: GPU power while the trace runs */
    double  dram_w_per_gbps;      /* >= 0: DRAM power proxy, TDP predicate only (A20) */
} magus_model;

/* desc.flags */
#define MAGUS_F_PER_TRACE_STATS 0x1u  /* fill magus_results.per_trace */
#define MAGUS_F_DUMP_WORDS      0x2u  /* per-(trace,policy) 32-tick cmd/tune-flag words from the replay kernel */
#define MAGUS_F_DUMP_DECISIONS  0x4u  /* per-tick code bytes (DESIGN A27) for a window of traces, decoded from the
                                         replay kernels' own cmd / tune-flag words (magus_decode_kernel) */
#define MAGUS_F_TIMING          0x8u  /* record CUDA events around the replay kernel(s) (magus_replay_kernel_times) */
#define MAGUS_F_TIMING_DETAIL   0x10u /* with MAGUS_F_TIMING: also around the pre-pass, fix-up and totals (each
                                         event node costs a few microseconds of the run) */
#define MAGUS_F_WALLCLOCK       0x20u /* NEXT-1 time model (A32): the governor runs
                                         every Delta of WALL time while each trace entry is one Delta of work at
                                         full speed, so a throttled entry spans several governor rounds and the
                                         governor samples the entry in progress.  Records, totals, digests and
                                         counts are per round; MAGUS_F_DUMP_DECISIONS gets the first n_samples
                                         rounds (a chain runs >= n_samples rounds); MAGUS_F_DUMP_WORDS is
                                         refused; STATIC_MAX is unchanged (never throttled: one entry per
                                         round).  Default (flag clear): one governor tick per entry (A15) */
#define MAGUS_F_NCCL            0x40u /* run the cross-rank exchange (per-policy chunk sums on the device, then the
                                         NCCL allreduce of the global [n_policies_global][MAGUS_N_TOTALS]) even at
                                         world == 1, on a one-rank communicator (nccl_unique_id may be NULL then);
                                         world > 1 always runs it */

typedef struct {
    int32_t n_traces;             /* local traces in this rank's shard, >= 0 */
    int32_t n_samples;            /* ticks per trace, >= 0 */
    int64_t trace_stride;         /* floats between consecutive time rows; >= n_traces, % 4 == 0 */
    int64_t global_trace_offset;  /* global id of local trace 0 (digests are per global id) */
    int32_t n_policies;           /* >= 1 */
    int32_t _reserved0;
    const magus_policy* policies; /* [n_policies], copied at create */
    magus_model model;
    int32_t rank, world;          /* world == 1 -> no NCCL; world > 1 needs nccl_unique_id */
    const void* nccl_unique_id;   /* 128 bytes from magus_nccl_unique_id on rank 0, broadcast by the caller */
    uint32_t flags;               /* MAGUS_F_* */
    int32_t dump_first_trace, dump_n_traces;   /* MAGUS_F_DUMP_DECISIONS window (local ids) */
    int32_t tuning_segments;      /* 0 = automatic time segmentation; else the segment count (tests) */
    int32_t tuning_warmup;        /* 0 = automatic warm-up ticks; else the warm-up (multiple of 32) */
    /* Parameter-grid split (north_star "by trace and parameter grid"): this rank replays
     * its traces under the global policies [policy_offset, policy_offset + n_policies) of a policy set of
     * n_policies_global points (0 = n_policies: no split).  policy_totals and argmin_policy are then global:
     * the allreduce sums every rank's slice into the global [n_policies_global][MAGUS_N_TOTALS]; per_trace,
     * words and decisions stay local ([..][n_policies]).  With the exchange on (world > 1 or MAGUS_F_NCCL),
     * create checks across ranks that every global policy is owned by some rank, that all owners of a policy
     * passed the same parameters, and that all ranks agree on the model, n_samples and n_policies_global
     * (MAGUS_ERR_CONFIG naming the disagreement otherwise). */
    int32_t n_policies_global;
    int32_t policy_offset;
} magus_replay_desc;

/* Per-policy totals (fp64), after the cross-rank allreduce. Index with MAGUS_TOT_*. */
enum {
    MAGUS_TOT_E = 0, MAGUS_TOT_E_PKG, MAGUS_TOT_T, MAGUS_TOT_EDP, MAGUS_TOT_SLOWDOWN,
    MAGUS_TOT_ENERGY_SAVING, MAGUS_TOT_EDP_SAVING, MAGUS_TOT_N_HI, MAGUS_TOT_N_THR,
    MAGUS_TOT_TRANSITIONS, MAGUS_TOT_TUNE_EVENTS, MAGUS_TOT_LOCK_TICKS, MAGUS_TOT_N_TRACES,
    MAGUS_N_TOTALS
};

/* One (trace, policy) record; all times in s, energies in J. */
typedef struct {
    int64_t  n_hi, n_thr, transitions, tune_events, lock_ticks;
    double   T, E_pkg, E, EDP, slowdown, energy_saving, edp_saving, pkg_power_saving;
    uint64_t digest;
} magus_trace_stats;

/* Caller-owned host arrays; a NULL member is skipped. */
typedef struct {
    double*            policy_totals;  /* [n_policies_global][MAGUS_N_TOTALS]: sums over traces (and ranks) of the
                                          per-(trace, policy) records -- E, E_pkg, T, EDP, the counts, and the SUMS
                                          of the per-trace fractions slowdown / energy_saving / edp_saving (their
                                          mean is the sum / MAGUS_TOT_N_TRACES; job-level ratios from the summed
                                          energies and times: magus_active_savings with p_idle_w = 0).  Rows of
                                          global policies outside this rank's slice are 0 without the exchange */
    magus_trace_stats* per_trace;      /* [n_traces][n_policies] (needs MAGUS_F_PER_TRACE_STATS) */
    uint32_t*          words;          /* [n_policies][n_traces][n_blocks][2] = {w_cmd, w_ev}, n_blocks =
                                          ceil(n_samples/32) (needs MAGUS_F_DUMP_WORDS) */
    uint8_t*           decisions;      /* [n_samples][dump_n_traces][n_policies] (needs MAGUS_F_DUMP_DECISIONS) */
    int32_t  argmin_policy;            /* out: global index, magus_totals_argmin of policy_totals (A23) */
    int32_t  err_trace;                /* out: first local trace with an invalid sample, else -1 */
    int64_t  err_tick;                 /* out: its first invalid tick, else -1 */
    int32_t  n_segments;               /* out: time segments per trace used by the run */
    int32_t  warmup_ticks;             /* out: warm-up ticks per speculative segment */
    int64_t  n_mismatched_segments;    /* out: speculative segments whose entry state was wrong (re-run) */
    int32_t  fixup_rounds;             /* out: max rounds of the exact fix-up over all chains */
    int32_t  _reserved0;
} magus_results;

/* ---- calls ---------------------------------------------------------------------------- */

typedef struct magus_replay magus_replay_t;

/* Writes 128 bytes (an ncclUniqueId) for world > 1.  MAGUS_ERR_NCCL if NCCL cannot be loaded. */
magus_status magus_nccl_unique_id(void* out128);

/* Seeded synthetic traces: writes trace[n_samples][trace_stride] (padding
 * columns zero) and w[n_traces] on the device, stream-ordered.  Counter-based: a trace's bytes depend
 * only on (seed, global_trace_offset + j, t), so shards and strides never change them. */
typedef struct {
    uint64_t seed;
    int32_t  n_traces, class_mix;       /* 0 cfg2, 1 cfg3/4, 2 cfg5 adversarial, 3 cfg1 concatenated */
    int64_t  n_samples, trace_stride, global_trace_offset;
    float    noise_amp, _reserved0;     /* a, default 0.002 */
    double   bw_max_gbps;               /* clamp bound */
} magus_gen_desc;
magus_status magus_gen_traces(const magus_gen_desc* desc, float* d_trace, float* d_w, void* cuda_stream);

/* NEXT-3 front end ("obtaining memory throughput data"; A31): recorded
 * cumulative byte counters -> the replay's trace layout.  d_counts: device [n_rows][stride] uint64
 * (time-major, trace-minor); d_times: device [n_rows] seconds, or NULL for a uniform period_s.  Interval
 * i = rows i -> i + 1 has throughput ((double)(c[i+1] - c[i]) / dt) / 1e9 GB/s, rounded once to fp32.  An
 * interval whose counter decreased (wrap / reset) is discarded with no governor round: trace j's
 * rounds are its valid intervals in time order, written to rows [0, n_valid[j]) of its column of
 * d_trace[n_rows - 1][stride]; the rows after them (and padding columns) are 0.0 and are not rounds -- replay
 * the first min_j n_valid[j] rows, or each trace with its own count.  d_n_valid: device [n_traces] int64, or
 * NULL.  d_report: device, 2 x uint64, zeroed by the call: [0] = discarded intervals, [1] = intervals whose
 * timestamp did not increase (the caller must treat the trace as invalid).  Stream-ordered (stream-ordered
 * scratch allocation); MAGUS_ERR_INVALID_ARG on NULL pointers or bad sizes, MAGUS_ERR_CUDA without a device. */
magus_status magus_counters_to_trace(const uint64_t* d_counts, const double* d_times, int32_t n_traces,
                                     int64_t n_rows, int64_t stride, double period_s, float* d_trace,
                                     int64_t* d_n_valid, unsigned long long* d_report, void* cuda_stream);

/* Validates desc (every invariant of section "magus_policy"/"magus_model"; A17), derives the
 * exact-equivalent thresholds, allocates device scratch, creates the NCCL communicator when
 * world > 1 (collective: every rank must call it).  *out is NULL on failure. */
magus_status magus_replay_create(const magus_replay_desc* desc, magus_replay_t** out);

/* Enqueues the whole replay on cuda_stream (a cudaStream_t; NULL = legacy default stream):
 * replay kernel, exact fix-up of speculative time segments, per-trace epilogue, per-policy
 * sums, the cross-rank allreduce (world > 1) and the argmin.  d_trace/d_w are device pointers
 * in the layout above.  Asynchronous; errors in the trace content surface in results(). */
magus_status magus_replay_run(magus_replay_t* h, const float* d_trace, const float* d_w, void* cuda_stream);

/* Same, from host buffers (pinned for full speed): copies them into library-owned device memory
 * on cuda_stream, then runs.  The host buffers may be reused once results() returns. */
magus_status magus_replay_run_host(magus_replay_t* h, const float* trace, const float* w, void* cuda_stream);

/* Waits for the last run and copies its results into caller-owned host arrays.
 * Returns MAGUS_ERR_TRACE (with err_trace/err_tick) if a sample was invalid. */
magus_status magus_replay_results(magus_replay_t* h, magus_results* out);

/* Device milliseconds of the last run's kernels (needs MAGUS_F_TIMING; waits for the run), CUDA events
 * on the run's stream: out[0] replay kernel(s); with MAGUS_F_TIMING_DETAIL also out[1] fix-up, out[2]
 * totals + allreduce + argmin, out[3] whole run, out[4] pre-pass, else -1. */
magus_status magus_replay_kernel_times(magus_replay_t* h, float out_ms[5]);

/* Same intervals averaged over the last n_last runs (at most 256 are kept), e.g. the K runs of a
 * timed benchmark region.  Waits for the last run. */
magus_status magus_replay_timing_summary(magus_replay_t* h, int32_t n_last, float out_ms[5]);

void         magus_replay_destroy(magus_replay_t* h);
const char*  magus_replay_last_error(const magus_replay_t* h);
const char*  magus_last_error(void);   /* errors of calls that have no handle (create, gen, unique id) */

/* Host-only helper (no GPU needed): the exact-equivalent thresholds the kernels compare against,
 * derived by evaluating the paper's predicates on the host:
 *   out_d[0] = d*_inc  (max d with fl(d/L) <= inc_threshold:  Alg.1 returns 1  iff d > d*_inc)
 *   out_d[1] = d*_dec  (min d with fl(d/L) >= dec_threshold:  Alg.1 returns -1 iff d < d*_dec)
 *   out_d[2] = L = k * sample_period_s,  out_d[3] = P_lo,  out_d[4] = P_hi
 *   out_f[0] = B_lo, out_f[1] = B_hi,  out_f[2] = a*_lo, out_f[3] = a*_hi (TDP: cmd = f_min iff A >= a*[f])
 *   out_i[0] = s_min   (min s with fl(s/C) >= high_freq_threshold: Alg.2 true iff popcount >= s_min)  */
magus_status magus_derive_thresholds(const magus_policy* p, const magus_model* m,
                                     double out_d[5], float out_f[4], int32_t out_i[1]);

/* Host-only (no GPU needed), NEXT-4 (A29): job-level savings of policy
 * `policy` against policy `baseline` with the system's idle power p_idle_w (W) excluded, from the per-policy
 * totals of magus_replay_results (policy_totals[n_policies][MAGUS_N_TOTALS]; the job = every trace of every
 * rank).  With mean powers P = E/T and P_b = E_b/T_b of the two policies and active energies
 * E_a = E - p_idle_w*T, E_a,b = E_b - p_idle_w*T_b:
 *   out[0] = ((P_b - p_idle_w) - (P - p_idle_w)) / (P_b - p_idle_w)   active power saving
 *   out[1] = 1 - E_a / E_a,b                                          active energy saving
 *   out[2] = 1 - (E_a * T) / (E_a,b * T_b)                            active EDP saving
 * (fractions).  MAGUS_ERR_INVALID_ARG: NULL pointers, indices outside [0, n_policies), p_idle_w < 0, a
 * non-positive total time, a baseline without active power (P_b <= p_idle_w) or P < p_idle_w;
 * out is left untouched then. */
magus_status magus_active_savings(const double* policy_totals, int32_t n_policies, int32_t policy,
                                  int32_t baseline, double p_idle_w, double out[3]);

/* Host-only (no GPU needed): the argmin the library reports (A23): over the policies whose
 * MAGUS_TOT_N_TRACES total is > 0 (all policies when none is), the one with the least total EDP; ties -> the
 * lowest index.  policy_totals: [n_policies][MAGUS_N_TOTALS].  MAGUS_ERR_INVALID_ARG on NULL or n_policies < 1. */
magus_status magus_totals_argmin(const double* policy_totals, int32_t n_policies, int32_t* out);

/* Host-only (no GPU needed): the rank's share of a 2-D (trace x parameter-grid) split.
 * The world is policy_shards columns of world / policy_shards trace shards; rank r owns trace shard
 * r / policy_shards and policy slice r % policy_shards.  Traces [0, n_traces) and policies [0, n_policies) are
 * cut into contiguous ranges whose sizes differ by at most one.  out = {global_trace_offset, n_traces_local,
 * policy_offset, n_policies_local}.  MAGUS_ERR_INVALID_ARG unless 0 <= rank < world, policy_shards >= 1 divides
 * world, n_traces >= 0 and 1 <= policy_shards <= n_policies. */
magus_status magus_grid_plan(int32_t world, int32_t rank, int32_t policy_shards, int64_t n_traces,
                             int32_t n_policies, int64_t out[4]);

int32_t magus_abi_version(void);

/* Diagnostics: the current launch plan: out = {n_segments, segment_len, warmup_ticks,
 * tile_groups_per_cta, policy_warps_per_group, trace_blocks, policy_blocks, ctas, threads_per_cta,
 * smem_bytes, lane_policies, launch_groups, kernels_per_run, solo_groups, seg_long, wide_groups} (seg_long: the first
 * seg_long segments are segment_len + 32 ticks long, the rest segment_len; MAGUS_F_WALLCLOCK: ctas and
 * threads_per_cta of the wall-clock kernels, smem 0, solo_groups 0; otherwise the first launch group's CTA
 * shape; kernels_per_run = the library's kernel launches in one run, excluding the decision-dump
 * re-simulation; solo_groups = launch groups run by the one-warp-CTA kernel magus_replay_solo_kernel;
 * wide_groups = launch groups run unsegmented by magus_replay_wide_kernel, one (trace, policy) chain per lane:
 * many-policy sweeps, DESIGN.md section 9a -- then n_segments = 1 and there is no fix-up). */
magus_status magus_replay_geometry(const magus_replay_t* h, int32_t out[16]);

/* Measurement: the replay kernel's CUDA-event time of each of the last n_last runs (MAGUS_F_TIMING), oldest first,
 * into out_ms[0 .. *n_out); *n_out = min(n_last, runs so far, the timing ring's 256 slots).  Synchronises with the
 * last run.  MAGUS_ERR_STATE without a timed run; MAGUS_ERR_INVALID_ARG for NULL pointers. */
magus_status magus_replay_run_times(magus_replay_t* h, int32_t n_last, float* out_ms, int32_t* n_out);

/* Diagnostics: which replay kernels the current plan launches: out = {replay launches per run (launch groups not
 * replayed by a combined launch), fused MAGUS + TDP kernel (1/0, magus_replay_fused_kernel: one launch reads each
 * sample once for both chain kinds), open-loop fast path (1/0: the O stage and the closed-form open-loop fix-up,
 * DESIGN.md section 9b), unsegmented wide plan groups}.  MAGUS_ERR_INVALID_ARG for a NULL handle or out. */
magus_status magus_replay_plan_info(const magus_replay_t* h, int32_t out[4]);

/* Diagnostics (test infrastructure for the debug-check build): returns -1 when the library was
 * built without device-side bounds checks (the release build), else launches one thread that checks `violate == 0`
 * with the library's MAGUS_CHECK and returns 1 if the check trapped the kernel (the CUDA context is then unusable:
 * call it in a separate process), 0 if it passed.  Needs a GPU only in the debug build. */
int32_t magus_debug_check_probe(int32_t violate);

#ifdef __cplusplus
}
#endif
#endif /* MAGUS_REPLAY_H */
