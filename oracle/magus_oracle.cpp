/*
 * oracle/magus_oracle.cpp -- CPU ORACLE for the MAGUS replay.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load, link or execute anything under oracle/.  The
 * product path (paper_2502_03796_b200/, include/) never does, and this file
 * shares no code, header, table or constant generator with it.
 *
 * What it is: a plain, slow, obviously correct replay of the MAGUS uncore-
 * frequency control loop, one trace and one policy at a time, in fp64, written
 * step by step from PAPER.md (arXiv 2502.03796) in the paper's order:
 *
 *   Alg. 1  Mem_throughput_Trend_Prediction   PAPER.md:197-222  (derivative P:207,
 *           ">" P:209, "<" P:213, return 0 P:218), FIFO mem_throughput_ls P:193
 *   Alg. 2  high_freq_detection               PAPER.md:224-237  (freq = sum/len P:229,
 *           ">=" P:230), FIFO uncore_tune_ls P:243
 *   S3.1    temporary decision, not executed immediately
 *   S3.2    override to max while high-frequency; prediction keeps
 *           running and logging while locked
 *   S4      idle/initial uncore level = minimum
 *   S5.3    Intel default (TDP-triggered) baseline
 *   S5.4    metrics: perf loss, pkg power saving, energy saving
 *           (pkg + GPU), EDP
 *   S6.1    jump "directly to the lower bound"
 *   NEXT-1  wall-clock governor rounds (oracle_replay_wallclock) SPEC.md:348-362, DESIGN A32
 *
 * Where the paper is silent the readings A1-A25 of DESIGN.md section 3 apply
 * (they are cited inline as [A<n>]).  The closed-loop power/performance model
 * (achieved = min(demand, bandwidth(f)), dilation of the memory-bound
 * fraction, power law between the uncore endpoints) is SPEC.md's simsys
 * module, which SPEC itself marks as invented plumbing.
 *
 * Numerics [A22]: trace samples and achieved throughput are fp32; every
 * predicate and every energy/time quantity is fp64, IEEE round-to-nearest, in
 * exactly the operation order written below.  Build with -O2
 * -ffp-contract=off (no FMA contraction), never -ffast-math.
 *
 * Pins: tests/test_oracle_*.py check this file against the paper's worked
 * numbers, closed forms, invariants and brute force.
 */
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>
#include <atomic>
#include <algorithm>
#include "oracle.h"

extern "C" {

/* ================================ Algorithm 1 =================================
 * PAPER.md:200-220, literally.  mem_throughput_ls is the FIFO of observed
 * throughput; ls[-1] is the newest, ls[0] the oldest entry.               */
int Mem_throughput_Trend_Prediction(double inc_threshold, double dec_threshold,
                                    const std::deque<double>& mem_throughput_ls,
                                    double direv_length) {
    double derivative = (mem_throughput_ls.back() - mem_throughput_ls.front()) / direv_length;
    if (derivative > inc_threshold) {
        return 1;
    } else if (derivative < dec_threshold) {
        return -1;
    } else {
        return 0;
    }
}

/* ================================ Algorithm 2 =================================
 * PAPER.md:227-235, literally.  uncore_tune_ls holds binary flags.  */
bool high_freq_detection(double high_freq_threshold, const std::deque<int>& uncore_tune_ls) {
    double sum = 0.0;
    for (int flag : uncore_tune_ls) sum += (double)flag;
    double freq = sum / (double)uncore_tune_ls.size();
    if (freq >= high_freq_threshold) {
        return true;
    } else {
        return false;
    }
}

/* C-callable wrappers so tests can drive Alg. 1/2 directly (pins K1, K2). */
int oracle_alg1(double inc, double dec, const double* ls, int32_t n, double direv_length) {
    std::deque<double> q(ls, ls + n);
    return Mem_throughput_Trend_Prediction(inc, dec, q, direv_length);
}
int oracle_alg2(double thr, const int32_t* flags, int32_t n) {
    std::deque<int> q(flags, flags + n);
    return high_freq_detection(thr, q) ? 1 : 0;
}

/* ===================== platform model (SPEC.md simsys, endpoints only) ======== */

/* bandwidth_at: Linear bw_max*(f/f_max); Saturating
 * bw_max*min(1, (f/f_max)/knee).  Operand order is fixed by [A19]. */
double oracle_bandwidth_at(double f, const OModel* m) {
    double ratio = f / m->f_max_ghz;
    if (m->bw_shape == 0) {
        return m->bw_max_gbps * ratio;
    } else {
        double r = ratio / m->bw_knee;
        return m->bw_max_gbps * (r < 1.0 ? r : 1.0);
    }
}

/* uncore_power_at: p_min + (p_max - p_min)*((f-f_min)/(f_max-f_min))^exponent */
double oracle_uncore_power_at(double f, const OModel* m) {
    double x = (f - m->f_min_ghz) / (m->f_max_ghz - m->f_min_ghz);
    return m->p_uncore_min_w + (m->p_uncore_max_w - m->p_uncore_min_w) * std::pow(x, m->p_exponent);
}

/* package power at level f: idle + core-active + uncore */
double oracle_pkg_power_at(double f, const OModel* m) {
    return (m->p_pkg_idle_w + m->p_core_active_w) + oracle_uncore_power_at(f, m);
}

/* ============================ digest =========================== */
static uint64_t mix64(uint64_t z) {                 /* splitmix64 finaliser */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t oracle_digest(const uint8_t* cmd_hi, const uint8_t* event, int64_t n) {
    uint32_t sum_cmd = 0, sum_ev = 0;
    int64_t n_blocks = (n + 31) / 32;
    for (int64_t b = 0; b < n_blocks; ++b) {
        uint32_t w_cmd = 0, w_ev = 0;
        for (int i = 0; i < 32; ++i) {
            int64_t t = 32 * b + i;
            if (t < n) {                     /* a partial last block is zero-padded */
                w_cmd |= (uint32_t)(cmd_hi[t] ? 1u : 0u) << (31 - i);
                w_ev  |= (uint32_t)(event[t]  ? 1u : 0u) << (31 - i);
            }
        }
        uint64_t m = mix64((uint64_t)b * 0x9E3779B97F4A7C15ULL);
        uint32_t key_cmd = (uint32_t)(m >> 32) | 1u, key_ev = (uint32_t)m | 1u;   /* odd per-block keys */
        sum_cmd += w_cmd * key_cmd;                                                /* mod 2^32 */
        sum_ev += w_ev * key_ev;
    }
    return ((uint64_t)sum_cmd << 32) | (uint64_t)sum_ev;
}

/* =============================== the replay loop ==============================
 * One trace D[0..n-1] (fp32, D[t] at D[t*stride]), one policy.  Per tick, in
 * order:
 *   1 observe   A = min(D, bandwidth(level))                     [A14]
 *   2 duration  tau = thr ? Delta*(w + (1-w)*(D/A)) : Delta       [A16]
 *   3 energy    E_pkg += P*tau; E += (P + P_gpu)*tau; T += tau
 *   4 FIFO      mem_throughput_ls.push(A), capacity k+1            ([A2])
 *   5 Alg. 1    when k+1 samples: temporary decision + tune flag   ([A7])
 *   6 Alg. 2    when the tune log is full                          ([A8])
 *   7 decision  lock -> max; else 1 -> max, -1 -> min, 0 -> keep   ([A9])
 *   8 record    transition iff cmd != level                        [A25]
 *   9 actuate   the command governs the next tick                  [A15]
 * codes (optional, one byte per tick): bit0 cmd==HI, bit1 ready, bit2 tune
 * event, bit3 high-frequency, bits4-5 signal (1 = +1, 2 = -1), bit6 throttled,
 * bit7 level in effect == HI.
 */
int oracle_replay(const float* D, int64_t n, int64_t stride, float w,
                  const OPolicy* pol, const OModel* m, OResult* out,
                  uint8_t* codes, int64_t codes_stride) {
    std::memset(out, 0, sizeof(OResult));
    out->err_tick = -1;

    const double Delta = m->sample_period_s;
    /* levels are exactly {f_min, f_max} [A9] */
    const float  B_hi = (float)oracle_bandwidth_at(m->f_max_ghz, m);
    const float  B_lo = (float)oracle_bandwidth_at(m->f_min_ghz, m);
    const double P_hi = oracle_pkg_power_at(m->f_max_ghz, m);
    const double P_lo = oracle_pkg_power_at(m->f_min_ghz, m);
    const double P_gpu = m->p_gpu_active_w;
    const double wd = (double)w;

    /* validation [A17]: 0 <= D <= bw_max, finite */
    for (int64_t t = 0; t < n; ++t) {
        float d = D[t * stride];
        if (!(d >= 0.0f) || !((double)d <= m->bw_max_gbps)) {
            out->status = 2;
            out->err_tick = t;
            return 2;
        }
    }

    /* initial level [A10]: MAGUS and STATIC_MIN start at f_min;
       STATIC_MAX and the Intel default start at f_max. */
    int f = (pol->kind == O_MAGUS || pol->kind == O_STATIC_MIN) ? O_LO : O_HI;

    const int    k = pol->deriv_ticks;
    const double direv_length = (double)k * Delta;            /* [A2] */
    const int    C = pol->tune_log_capacity;
    std::deque<double> mem_throughput_ls;
    std::deque<int>    uncore_tune_ls;

    std::vector<uint8_t> cmd_bits((size_t)n), ev_bits((size_t)n);
    double E_pkg = 0.0, E = 0.0, T = 0.0;

    for (int64_t t = 0; t < n; ++t) {
        const float Dt = D[t * stride];
        /* 1 observe: closed loop, the throughput the workload attains at the level in effect [A14];
           open loop, a recorded throughput observed as is [A30] */
        const float B = (f == O_HI) ? B_hi : B_lo;
        const float A = (m->observe == 1) ? Dt : ((Dt < B) ? Dt : B);
        /* 2 duration */
        const bool thr = (A < Dt);
        double tau;
        if (thr) tau = Delta * (wd + (1.0 - wd) * ((double)Dt / (double)A));
        else     tau = Delta;
        /* 3 energy */
        const double P = (f == O_HI) ? P_hi : P_lo;
        E_pkg += P * tau;
        E += (P + P_gpu) * tau;
        T += tau;
        out->n_hi += (f == O_HI);
        out->n_thr += thr;

        int cmd = f, sig = 0, ready = 0, event = 0, hf = 0;
        if (pol->kind == O_MAGUS) {
            /* 4 FIFO of the last k+1 observations */
            mem_throughput_ls.push_back((double)A);
            if ((int64_t)mem_throughput_ls.size() > k + 1) mem_throughput_ls.pop_front();
            /* 5 Alg. 1 once the window spans k periods; the tune flag is logged
               whatever the lock state ("continues running ... log") */
            if ((int64_t)mem_throughput_ls.size() == k + 1) {
                ready = 1;
                sig = Mem_throughput_Trend_Prediction(pol->inc_threshold, pol->dec_threshold,
                                                      mem_throughput_ls, direv_length);
                event = (sig != 0) ? 1 : 0;
                uncore_tune_ls.push_back(event);
                if ((int64_t)uncore_tune_ls.size() > C) uncore_tune_ls.pop_front();
                out->tune_events += event;
            }
            /* 6 Alg. 2 on a full log only [A8] */
            if ((int64_t)uncore_tune_ls.size() == C) {
                hf = high_freq_detection(pol->high_freq_threshold, uncore_tune_ls) ? 1 : 0;
            }
            /* 7 decision: the temporary decision is overridden by the lock */
            if (hf) cmd = O_HI;
            else if (sig == 1) cmd = O_HI;       /* increase -> max [A9] */
            else if (sig == -1) cmd = O_LO;      /* decrease -> "directly to the lower bound" P:318 */
            else cmd = f;                         /* hold */
        } else if (pol->kind == O_TDP_DEFAULT) {
            /* uncore lowered only when package + DRAM power approaches TDP [A24] */
            double pkg_plus_dram = P + m->dram_w_per_gbps * (double)A;
            double bound = (1.0 - pol->tdp_margin) * pol->tdp_w;
            cmd = (pkg_plus_dram >= bound) ? O_LO : O_HI;
        } else {
            cmd = f;                              /* static governors */
        }
        out->lock_ticks += hf;

        /* 8 record */
        if (cmd != f) out->transitions += 1;
        cmd_bits[(size_t)t] = (uint8_t)(cmd == O_HI);
        ev_bits[(size_t)t] = (uint8_t)event;
        if (codes) {
            uint8_t c = 0;
            c |= (uint8_t)(cmd == O_HI);
            c |= (uint8_t)(ready << 1);
            c |= (uint8_t)(event << 2);
            c |= (uint8_t)(hf << 3);
            c |= (uint8_t)((sig == 1 ? 1 : (sig == -1 ? 2 : 0)) << 4);
            c |= (uint8_t)((thr ? 1 : 0) << 6);
            c |= (uint8_t)((f == O_HI ? 1 : 0) << 7);
            codes[t * codes_stride] = c;
        }
        /* 9 actuate */
        f = cmd;
    }

    out->T = T;
    out->E_pkg = E_pkg;
    out->E = E;
    out->EDP = E * T;
    /* static-max baseline on the same trace [A21]: never throttled, every tick lasts Delta */
    double T_b = 0.0;
    for (int64_t t = 0; t < n; ++t) T_b += Delta;
    double E_b = (P_hi + P_gpu) * T_b;
    out->T_base = T_b;
    out->E_base = E_b;
    if (n > 0) {
        out->slowdown = T / T_b - 1.0;
        out->energy_saving = 1.0 - E / E_b;
        out->edp_saving = 1.0 - (E * T) / (E_b * T_b);
        out->pkg_power_saving = 1.0 - (E_pkg / T) / P_hi;     /* P:301, time-weighted mean */
    }
    out->digest = oracle_digest(cmd_bits.data(), ev_bits.data(), n);
    return 0;
}

/* Many traces x many policies, std::thread over (trace, policy) tasks.
 * trace: [n_samples][stride] fp32 time-major; w: [n_traces]; out: [n_traces][n_policies].
 * codes (optional): [n_samples][n_traces][n_policies]. Returns the number of threads used. */
int oracle_replay_batch(const float* trace, int32_t n_traces, int64_t n_samples, int64_t stride,
                        const float* w, int32_t n_policies, const OPolicy* pols, const OModel* m,
                        OResult* out, uint8_t* codes, int32_t n_threads) {
    if (n_threads <= 0) n_threads = (int32_t)std::max(1u, std::thread::hardware_concurrency());
    const int64_t n_tasks = (int64_t)n_traces * n_policies;
    std::atomic<int64_t> next(0);
    auto worker = [&]() {
        for (;;) {
            int64_t task = next.fetch_add(1);
            if (task >= n_tasks) break;
            int32_t j = (int32_t)(task / n_policies), p = (int32_t)(task % n_policies);
            uint8_t* c = codes ? codes + (int64_t)j * n_policies + p : nullptr;
            oracle_replay(trace + j, n_samples, stride, w[j], &pols[p], m, &out[task],
                          c, (int64_t)n_traces * n_policies);
        }
    };
    std::vector<std::thread> pool;
    int32_t used = (int32_t)std::min<int64_t>(n_threads, std::max<int64_t>(1, n_tasks));
    for (int32_t i = 0; i < used; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return used;
}

/* ====================== wall-clock governor rounds (NEXT-1) ======================
 * The other reading of the time model (A32): the governor runs every Delta of wall time while
 * the workload works through its trace entries; a throttled entry spans several rounds, and the governor
 * samples the entry in progress each round.  Entry j is one Delta of work at full speed; at level f it
 * progresses at rate r = 1 / (w + (1 - w) * D_j / A) per round (the A16 dilation) when throttled, else 1.
 * Per round t (level f, entry e, remaining fraction rho of e):
 *   sample   A = min(D_e, B[f]) (A14; A = D_e in open loop, A30), throttled iff A < D_e
 *   progress u = 1 round of time: while u > 0: need = rho / r(e, f); if need > u: rho -= u * r, u = 0;
 *            else u -= need, e += 1, rho = 1 (the next entry continues at the same level); the run ends
 *            when e == n, the round lasting (1 - u) * Delta
 *   energy   E_pkg += P[f] * used * Delta, E += (P[f] + P_gpu) * used * Delta, T += used * Delta
 *   decide   the same Alg. 1 / Alg. 2 / decision / baselines as oracle_replay on this round's A
 * Counts are per round; n_thr counts rounds whose sample was throttled.  n_rounds_out = rounds run;
 * codes (optional, cap bytes) = the per-round code bytes of oracle_replay; the digest is over rounds.
 * The static-max baseline is unchanged (never throttled: one entry per round, T_b = n * Delta). */
int oracle_replay_wallclock(const float* D, int64_t n, int64_t stride, float w, const OPolicy* pol, const OModel* m,
                            OResult* out, int64_t* n_rounds_out, uint8_t* codes, int64_t codes_cap) {
    std::memset(out, 0, sizeof(OResult));
    out->err_tick = -1;
    *n_rounds_out = 0;
    const double Delta = m->sample_period_s;
    const float  B_hi = (float)oracle_bandwidth_at(m->f_max_ghz, m);
    const float  B_lo = (float)oracle_bandwidth_at(m->f_min_ghz, m);
    const double P_hi = oracle_pkg_power_at(m->f_max_ghz, m);
    const double P_lo = oracle_pkg_power_at(m->f_min_ghz, m);
    const double P_gpu = m->p_gpu_active_w;
    const double wd = (double)w;
    for (int64_t t = 0; t < n; ++t) {
        float d = D[t * stride];
        if (!(d >= 0.0f) || !((double)d <= m->bw_max_gbps)) {
            out->status = 2;
            out->err_tick = t;
            return 2;
        }
    }
    int f = (pol->kind == O_MAGUS || pol->kind == O_STATIC_MIN) ? O_LO : O_HI;
    const int    k = pol->deriv_ticks;
    const double direv_length = (double)k * Delta;
    const int    C = pol->tune_log_capacity;
    std::deque<double> mem_throughput_ls;
    std::deque<int>    uncore_tune_ls;
    std::vector<uint8_t> cmd_bits, ev_bits;
    double E_pkg = 0.0, E = 0.0, T = 0.0;

    int64_t e = 0;       /* entry in progress */
    double rho = 1.0;    /* its remaining work fraction */
    int64_t t = 0;       /* round */
    while (e < n) {
        /* sample the entry in progress */
        const float De = D[e * stride];
        const float B = (f == O_HI) ? B_hi : B_lo;
        const float A = (m->observe == 1) ? De : ((De < B) ? De : B);
        const bool thr = (A < De);
        /* progress through one round of wall time at level f */
        double u = 1.0;
        while (u > 0.0 && e < n) {
            const float Dc = D[e * stride];
            const float Ac = (m->observe == 1) ? Dc : ((Dc < B) ? Dc : B);
            double r;
            if (Ac < Dc) r = 1.0 / (wd + (1.0 - wd) * ((double)Dc / (double)Ac));
            else         r = 1.0;
            const double need = rho / r;
            if (need > u) {
                rho = rho - u * r;
                u = 0.0;
            } else {
                u = u - need;
                e += 1;
                rho = 1.0;
            }
        }
        const double used = 1.0 - u;
        const double P = (f == O_HI) ? P_hi : P_lo;
        E_pkg += P * (used * Delta);
        E += (P + P_gpu) * (used * Delta);
        T += used * Delta;
        out->n_hi += (f == O_HI);
        out->n_thr += thr;

        int cmd = f, sig = 0, ready = 0, event = 0, hf = 0;
        if (pol->kind == O_MAGUS) {
            mem_throughput_ls.push_back((double)A);
            if ((int64_t)mem_throughput_ls.size() > k + 1) mem_throughput_ls.pop_front();
            if ((int64_t)mem_throughput_ls.size() == k + 1) {
                ready = 1;
                sig = Mem_throughput_Trend_Prediction(pol->inc_threshold, pol->dec_threshold,
                                                      mem_throughput_ls, direv_length);
                event = (sig != 0) ? 1 : 0;
                uncore_tune_ls.push_back(event);
                if ((int64_t)uncore_tune_ls.size() > C) uncore_tune_ls.pop_front();
                out->tune_events += event;
            }
            if ((int64_t)uncore_tune_ls.size() == C)
                hf = high_freq_detection(pol->high_freq_threshold, uncore_tune_ls) ? 1 : 0;
            if (hf) cmd = O_HI;
            else if (sig == 1) cmd = O_HI;
            else if (sig == -1) cmd = O_LO;
            else cmd = f;
        } else if (pol->kind == O_TDP_DEFAULT) {
            double pkg_plus_dram = P + m->dram_w_per_gbps * (double)A;
            double bound = (1.0 - pol->tdp_margin) * pol->tdp_w;
            cmd = (pkg_plus_dram >= bound) ? O_LO : O_HI;
        } else {
            cmd = f;
        }
        out->lock_ticks += hf;
        if (cmd != f) out->transitions += 1;
        cmd_bits.push_back((uint8_t)(cmd == O_HI));
        ev_bits.push_back((uint8_t)event);
        if (codes && t < codes_cap) {
            uint8_t c = 0;
            c |= (uint8_t)(cmd == O_HI);
            c |= (uint8_t)(ready << 1);
            c |= (uint8_t)(event << 2);
            c |= (uint8_t)(hf << 3);
            c |= (uint8_t)((sig == 1 ? 1 : (sig == -1 ? 2 : 0)) << 4);
            c |= (uint8_t)((thr ? 1 : 0) << 6);
            c |= (uint8_t)((f == O_HI ? 1 : 0) << 7);
            codes[t] = c;
        }
        f = cmd;
        t += 1;
    }
    *n_rounds_out = t;
    out->T = T;
    out->E_pkg = E_pkg;
    out->E = E;
    out->EDP = E * T;
    double T_b = 0.0;
    for (int64_t i = 0; i < n; ++i) T_b += Delta;
    double E_b = (P_hi + P_gpu) * T_b;
    out->T_base = T_b;
    out->E_base = E_b;
    if (n > 0) {
        out->slowdown = T / T_b - 1.0;
        out->energy_saving = 1.0 - E / E_b;
        out->edp_saving = 1.0 - (E * T) / (E_b * T_b);
        out->pkg_power_saving = 1.0 - (E_pkg / T) / P_hi;
    }
    out->digest = oracle_digest(cmd_bits.data(), ev_bits.data(), t);
    return 0;
}

/* ===================== recorded byte counters -> throughput (NEXT-3) =====================
 * read_throughput: throughput = (count_now - count_prev) / (t_now - t_prev), here in GB/s
 * (1 GB/s = 1e9 B/s [A3]): ((double)(c1 - c0) / dt) / 1e9, rounded once to fp32.  A counter that decreased
 * (wrap / reset) is an error whose sample is discarded and whose baseline is re-armed; "counter
 * reset to 0 -> sample discarded, no governor round": the interval yields no round at all [A31].  So trace j's
 * rounds are its valid intervals in time order: out[0 .. n_valid[j]) of its column, the rest of the column
 * 0.0 (padding, not rounds).  A non-increasing timestamp is an error (returns -1).  Returns the number of
 * discarded intervals. */
int64_t oracle_counters_to_throughput(const uint64_t* counts, const double* times, int64_t n_rows, int32_t n_traces,
                                      int64_t stride, double period, float* out, int64_t* n_valid) {
    for (int64_t i = 0; i + 1 < n_rows; ++i) {
        double dt = times ? times[i + 1] - times[i] : period;
        if (!(dt > 0.0)) return -1;
    }
    int64_t discarded = 0;
    for (int32_t j = 0; j < n_traces; ++j) {
        int64_t k = 0;                                       /* rounds of trace j so far */
        for (int64_t i = 0; i + 1 < n_rows; ++i) {
            uint64_t c0 = counts[i * stride + j], c1 = counts[(i + 1) * stride + j];
            if (c1 < c0) {                                   /* wrap / reset: no round */
                ++discarded;
                continue;
            }
            double dt = times ? times[i + 1] - times[i] : period;
            out[k * stride + j] = (float)(((double)(c1 - c0) / dt) / 1e9);
            ++k;
        }
        n_valid[j] = k;
        for (int64_t i = k; i + 1 < n_rows; ++i) out[i * stride + j] = 0.0f;   /* padding */
    }
    return discarded;
}

/* ========================= active savings ========================
 * "we measure active power and energy savings, excluding idle power.  For instance, if MAGUS reduces
 * total power consumption from 200W to 150W on a system with 100W idle power, the active power saving
 * is (100 - 50)/100 = 50%".  Fractions (not percent), like the other savings here.
 * Returns 0, or 1 when the baseline has no active power (p_base <= p_idle) or p < p_idle. */
int oracle_active_saving(double p, double p_base, double p_idle, double* out) {
    if (!(p_base > p_idle) || p < p_idle || p_idle < 0) return 1;
    *out = ((p_base - p_idle) - (p - p_idle)) / (p_base - p_idle);
    return 0;
}

/* Job-level active savings of a policy against a baseline over the same n traces (A29):
 * mean powers P = sum(E)/sum(T), P_b = sum(E_b)/sum(T_b); active energies E_a = sum(E) - p_idle*sum(T),
 * E_a,b = sum(E_b) - p_idle*sum(T_b).  out = {active power saving, active energy saving,
 * active EDP saving} = {oracle_active_saving(P, P_b, p_idle), 1 - E_a/E_a,b,
 * 1 - (E_a*sum(T))/(E_a,b*sum(T_b))}.  Plain running sums in index order. */
int oracle_active_savings_job(const double* E, const double* T, const double* E_b, const double* T_b, int64_t n,
                              double p_idle, double out[3]) {
    double sE = 0, sT = 0, sEb = 0, sTb = 0;
    for (int64_t i = 0; i < n; ++i) {
        sE += E[i];
        sT += T[i];
        sEb += E_b[i];
        sTb += T_b[i];
    }
    if (!(sT > 0) || !(sTb > 0)) return 1;
    if (oracle_active_saving(sE / sT, sEb / sTb, p_idle, &out[0])) return 1;
    const double Ea = sE - p_idle * sT, Eab = sEb - p_idle * sTb;
    out[1] = 1.0 - Ea / Eab;
    out[2] = 1.0 - (Ea * sT) / (Eab * sTb);
    return 0;
}

} /* extern "C" */
