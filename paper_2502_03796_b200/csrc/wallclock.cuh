// wallclock.cuh -- NEXT-1: the replay with wall-clock governor rounds (A32).
//
// The governor runs every Delta of wall time while the workload works through its trace entries: entry j is
// one Delta of work at full speed and progresses at rate r = 1 / (w + (1 - w) * D_j / A) per round while
// throttled (the A16 dilation), else 1.  Round t samples the entry in progress, A = min(D_e, B[f]) (A14; the
// run's B_lo is +inf in open loop, A30), consumes one round of time across entries at its level f (rho = the
// remaining work fraction of the entry in progress, kept across a level change), and then decides exactly
// as a tick of the per-entry replay (the same tickers: Alg. 1, Alg. 2, the jump, TDP) on that sample.
//
// One thread per (lane policy, trace) chain, rounds in order: a round's work depends on the previous
// round's level, and the number of rounds per chain depends on the data, so there is neither a time
// segmentation nor a warp-uniform schedule here.  The fp64 time arithmetic uses the _rn intrinsics in the
// order A32 fixes (no FMA contraction), so entry boundaries -- hence every sample and decision -- are the
// oracle's bit for bit.  Energy is summed per round (P[f] * used * Delta), like the oracle.
#pragma once
#include "device_common.cuh"
#include "post_kernels.cuh"
#include "tickers.cuh"

namespace magus {

struct WallParams {
    TraceRec* wrec;     // [n_lane][n_traces] records of the lane chains (read by the totals kernel)
    uint8_t* codes;     // per-round codes [n_samples][n_win][P] for rounds < n_samples, or nullptr
    int32_t first, n_win;
    int32_t P;
};

// One chain's rounds.  Returns the record; codes (optional) get its first n_samples rounds.
template <class T>
__device__ void wallclock_chain(const ReplayParams& p, const EpiParams& e, const WallParams& wp, const DevPolicy& pol,
                                int64_t ci, int j, const float* __restrict__ trace) {
    typename T::State s;
    T::init(s, pol, true);
    const int64_t n = p.n_samples, stride = p.trace_stride;
    const float bw_max = __uint_as_float(p.bwbits);
    const double wd = (double)e.w[j];
    const double one_m_w = __dsub_rn(1.0, wd);
    const int k = pol.k, C = pol.C;
    const bool dump = wp.codes != nullptr && j >= wp.first && j < wp.first + wp.n_win && pol.policy_index >= 0;
    bool invalid = false;
    int64_t ei = 0;      // entry in progress
    double rho = 1.0;    // its remaining work fraction
    int64_t t = 0;       // round
    double Tw = 0.0, Epkg = 0.0, Ew = 0.0;
    uint32_t nhi = 0, nthr = 0, trans = 0, nev = 0, lock = 0;
    uint32_t wc = 0, we = 0, dc = 0, de = 0;   // 32-round digest words (round 32b + i at bit 31 - i)
    while (ei < n) {
        const float De = __ldg(trace + ei * stride + j);
        const uint32_t lvl = T::level(s);
        const float B = lvl ? p.B_hi : p.B_lo;
        // one round of wall time at level lvl
        double u = 1.0;
        while (u > 0.0 && ei < n) {
            const float Dc = __ldg(trace + ei * stride + j);
            double r = 1.0;
            if (!(Dc >= 0.0f && Dc <= bw_max)) {
                invalid = true;   // reported by the totals kernel (A17); r = 1 keeps the loop finite
            } else {
                const float Ac = fminf(Dc, B);
                if (Ac < Dc) r = __ddiv_rn(1.0, __dadd_rn(wd, __dmul_rn(one_m_w, __ddiv_rn((double)Dc, (double)Ac))));
            }
            const double need = __ddiv_rn(rho, r);
            if (need > u) {
                rho = __dsub_rn(rho, __dmul_rn(u, r));
                u = 0.0;
            } else {
                u = __dsub_rn(u, need);
                ei += 1;
                rho = 1.0;
            }
        }
        const double used = __dsub_rn(1.0, u);
        const double P = lvl ? e.P_hi : e.P_lo;
        const double dt = __dmul_rn(used, e.Delta);
        Epkg = __dadd_rn(Epkg, __dmul_rn(P, dt));
        Ew = __dadd_rn(Ew, __dmul_rn(__dadd_rn(P, e.P_gpu), dt));
        Tw = __dadd_rn(Tw, dt);
        // the governor's decision on the round's sample (the entry in progress at the round's start)
        const bool ready = t >= k, lfull = t >= k + C - 1;
        const TickOut o = T::template tick<true>(s, De, pol, p.B_lo, p.B_hi, ready, lfull);
        nhi += lvl;
        nthr += o.thr;
        trans += (o.cmd != lvl) ? 1u : 0u;
        nev += o.ev;
        lock += o.hf;
        const int bit = 31 - (int)(t & 31);
        wc |= o.cmd << bit;
        we |= o.ev << bit;
        if (bit == 0) {
            const uint2 key = digest_key((uint64_t)(t >> 5));
            dc += wc * key.x;
            de += we * key.y;
            wc = we = 0;
        }
        if (dump && t < n) {
            const uint32_t c = o.cmd | ((T::kWarmupRules && ready) ? 2u : 0u) | (o.ev << 2) | (o.hf << 3) |
                               (o.sig << 4) | (o.thr << 6) | (lvl << 7);
            wp.codes[(t * wp.n_win + (j - wp.first)) * wp.P + pol.policy_index] = (uint8_t)c;
        }
        t += 1;
    }
    if (t & 31) {   // partial last block, zero-padded
        const uint2 key = digest_key((uint64_t)(t >> 5));
        dc += wc * key.x;
        de += we * key.y;
    }
    TraceRec r;
    const double T_b = __dmul_rn((double)n, e.Delta);
    const double E_b = __dmul_rn(__dadd_rn(e.P_hi, e.P_gpu), T_b);
    r.n_hi = nhi;
    r.n_thr = nthr;
    r.transitions = trans;
    r.tune_events = nev;
    r.lock_ticks = lock;
    r.T = Tw;
    r.E_pkg = Epkg;
    r.E = Ew;
    r.EDP = Ew * Tw;
    if (n > 0) {
        r.slowdown = Tw / T_b - 1.0;
        r.energy_saving = 1.0 - Ew / E_b;
        r.edp_saving = 1.0 - (Ew * Tw) / (E_b * T_b);
        r.pkg_power_saving = 1.0 - (Epkg / Tw) / e.P_hi;
    } else {
        r.slowdown = r.energy_saving = r.edp_saving = r.pkg_power_saving = 0.0;
    }
    r.digest = digest_pack(dc, de);
    wp.wrec[ci] = r;
    p.c_vmax[ci] = invalid ? 0xFFFFFFFFu : 0u;   // the totals kernel's invalid-sample test (A17)
}

// Entry-major form of the same rounds (the default): the loop runs over trace ENTRIES, in the same order
// for every thread of a warp, so the warp's loads of an entry row are coalesced and can be issued a block of
// kWallPf entries ahead; the rounds that start inside an entry are an inner loop.  An entry takes at least
// one round (need = rho / r >= rho and r <= 1), so a round ends at most once per entry boundary and the
// round-start sample is the entry in progress when `fresh` is set.  Same operations in the same order as
// the round-major loop above and the oracle, hence the same bits.
#ifndef MAGUS_WALL_PF
#define MAGUS_WALL_PF 8
#endif
constexpr int kWallPf = MAGUS_WALL_PF;   // entries per prefetched block

template <class T>
struct WallChain {
    typename T::State s;
    double u = 1.0;          // time left in the current round
    bool fresh = true;       // the next consumption starts a round
    float De = 0.0f;         // the round's sample (entry in progress at its start)
    int64_t t = 0;           // rounds finished
    double Tw = 0.0, Epkg = 0.0, Ew = 0.0;
    uint32_t nhi = 0, nthr = 0, trans = 0, nev = 0, lock = 0;
    uint32_t wc = 0, we = 0, dc = 0, de = 0;
    bool invalid = false;

    // end of a round: its time and energy at the level in effect, then the governor's decision on De
    __device__ __forceinline__ void end_round(const ReplayParams& p, const EpiParams& e, const WallParams& wp,
                                              const DevPolicy& pol, bool dump, int j) {
        const uint32_t lvl = T::level(s);
        const double used = __dsub_rn(1.0, u);
        const double P = lvl ? e.P_hi : e.P_lo;
        const double dt = __dmul_rn(used, e.Delta);
        Epkg = __dadd_rn(Epkg, __dmul_rn(P, dt));
        Ew = __dadd_rn(Ew, __dmul_rn(__dadd_rn(P, e.P_gpu), dt));
        Tw = __dadd_rn(Tw, dt);
        const bool ready = t >= pol.k, lfull = t >= pol.k + pol.C - 1;
        const TickOut o = T::template tick<true>(s, De, pol, p.B_lo, p.B_hi, ready, lfull);
        nhi += lvl;
        nthr += o.thr;
        trans += (o.cmd != lvl) ? 1u : 0u;
        nev += o.ev;
        lock += o.hf;
        const int bit = 31 - (int)(t & 31);
        wc |= o.cmd << bit;
        we |= o.ev << bit;
        if (bit == 0) {
            const uint2 key = digest_key((uint64_t)(t >> 5));
            dc += wc * key.x;
            de += we * key.y;
            wc = we = 0;
        }
        if (dump && t < p.n_samples) {
            const uint32_t c = o.cmd | ((T::kWarmupRules && ready) ? 2u : 0u) | (o.ev << 2) | (o.hf << 3) |
                               (o.sig << 4) | (o.thr << 6) | (lvl << 7);
            wp.codes[(t * wp.n_win + (j - wp.first)) * wp.P + pol.policy_index] = (uint8_t)c;
        }
        t += 1;
        u = 1.0;
        fresh = true;
    }

    // rate of entry D at level lvl (A32): 1 unless throttled; r = 1 / (w + (1 - w) * (D / A))
    __device__ __forceinline__ static double rate(float D, uint32_t lvl, const ReplayParams& p, double wd,
                                                  double one_m_w) {
        const float A = fminf(D, lvl ? p.B_hi : p.B_lo);
        if (A < D) return __ddiv_rn(1.0, __dadd_rn(wd, __dmul_rn(one_m_w, __ddiv_rn((double)D, (double)A))));
        return 1.0;
    }

    // one whole entry, the round-end call sites apart (a round split inside the entry / a round ending with
    // it): longer code but a shorter dependent path; used by the unrolled (latency-bound) blocks
    __device__ __forceinline__ void entry_split(float Dc, const ReplayParams& p, const EpiParams& e,
                                                const WallParams& wp, const DevPolicy& pol, bool dump, int j,
                                                float bw_max, double wd, double one_m_w) {
        const bool ok = Dc >= 0.0f && Dc <= bw_max;
        invalid |= !ok;   // reported by the totals kernel (A17); r = 1 keeps the loop finite
        double r = ok ? rate(Dc, T::level(s), p, wd, one_m_w) : 1.0;
        double rho = 1.0;
        for (;;) {
            if (fresh) {
                De = Dc;
                fresh = false;
            }
            const double need = r == 1.0 ? rho : __ddiv_rn(rho, r);   // (rho / 1.0 == rho exactly)
            if (need > u) {
                rho = __dsub_rn(rho, __dmul_rn(u, r));
                u = 0.0;
                end_round(p, e, wp, pol, dump, j);
                if (ok) r = rate(Dc, T::level(s), p, wd, one_m_w);   // the next round's level
            } else {
                u = __dsub_rn(u, need);
                if (u == 0.0) end_round(p, e, wp, pol, dump, j);      // the round ends with the entry
                return;
            }
        }
    }

    // one whole entry (one copy of the round end and of the rate in the code)
    __device__ __forceinline__ void entry(float Dc, const ReplayParams& p, const EpiParams& e, const WallParams& wp,
                                          const DevPolicy& pol, bool dump, int j, float bw_max, double wd,
                                          double one_m_w) {
        const bool ok = Dc >= 0.0f && Dc <= bw_max;
        invalid |= !ok;   // reported by the totals kernel (A17); r = 1 keeps the loop finite
        double rho = 1.0, r = 1.0;
        bool need_rate = ok;
        for (;;) {
            if (fresh) {
                De = Dc;
                fresh = false;
            }
            if (need_rate) {   // at the entry's start and after a round end (the level may have changed)
                r = rate(Dc, T::level(s), p, wd, one_m_w);
                need_rate = false;
            }
            const double need = r == 1.0 ? rho : __ddiv_rn(rho, r);   // (rho / 1.0 == rho exactly)
            bool done, ends;
            if (need > u) {
                rho = __dsub_rn(rho, __dmul_rn(u, r));
                u = 0.0;
                done = false;
                ends = true;
            } else {
                u = __dsub_rn(u, need);
                done = true;
                ends = u == 0.0;   // the round ends with the entry
            }
            if (ends) {
                end_round(p, e, wp, pol, dump, j);
                need_rate = ok;
            }
            if (done) return;
        }
    }
};

template <class T, bool UNROLL>
__device__ __forceinline__ void wallclock_chain_em(const ReplayParams& p, const EpiParams& e, const WallParams& wp,
                                                   const DevPolicy& pol, int64_t ci, int j,
                                                   const float* __restrict__ trace) {
    WallChain<T> c;
    T::init(c.s, pol, true);
    const int64_t n = p.n_samples, stride = p.trace_stride;
    const float bw_max = __uint_as_float(p.bwbits);
    const double wd = (double)e.w[j];
    const double one_m_w = __dsub_rn(1.0, wd);
    const bool dump = wp.codes != nullptr && j >= wp.first && j < wp.first + wp.n_win && pol.policy_index >= 0;
    float cur[kWallPf], nxt[kWallPf];
#pragma unroll
    for (int i = 0; i < kWallPf; ++i) cur[i] = i < n ? __ldcs(trace + i * stride + j) : 0.0f;
    for (int64_t b = 0; b < n; b += kWallPf) {
#pragma unroll
        for (int i = 0; i < kWallPf; ++i) {   // the next block's rows, in flight while this block runs
            const int64_t x = b + kWallPf + i;
            nxt[i] = x < n ? __ldcs(trace + x * stride + j) : 0.0f;
        }
        if (UNROLL && b + kWallPf <= n) {
            // few chains (latency-bound): the block's entries unrolled, so independent work of neighbouring
            // entries can overlap
#pragma unroll
            for (int i = 0; i < kWallPf; ++i) c.entry_split(cur[i], p, e, wp, pol, dump, j, bw_max, wd, one_m_w);
        } else {
            // many chains (issue-bound) and the ragged tail: rolled, one copy of the entry in the code
            const int m = (int)min((int64_t)kWallPf, n - b);
#pragma unroll 1
            for (int i = 0; i < m; ++i) {
                c.entry(cur[0], p, e, wp, pol, dump, j, bw_max, wd, one_m_w);
#pragma unroll
                for (int z = 0; z < kWallPf - 1; ++z) cur[z] = cur[z + 1];
            }
        }
#pragma unroll
        for (int i = 0; i < kWallPf; ++i) cur[i] = nxt[i];
    }
    if (!c.fresh) c.end_round(p, e, wp, pol, dump, j);   // the last, partial round
    if (c.t & 31) {                                       // partial last digest block, zero-padded
        const uint2 key = digest_key((uint64_t)(c.t >> 5));
        c.dc += c.wc * key.x;
        c.de += c.we * key.y;
    }
    TraceRec r;
    const double T_b = __dmul_rn((double)n, e.Delta);
    const double E_b = __dmul_rn(__dadd_rn(e.P_hi, e.P_gpu), T_b);
    r.n_hi = c.nhi;
    r.n_thr = c.nthr;
    r.transitions = c.trans;
    r.tune_events = c.nev;
    r.lock_ticks = c.lock;
    r.T = c.Tw;
    r.E_pkg = c.Epkg;
    r.E = c.Ew;
    r.EDP = c.Ew * c.Tw;
    if (n > 0) {
        r.slowdown = c.Tw / T_b - 1.0;
        r.energy_saving = 1.0 - c.Ew / E_b;
        r.edp_saving = 1.0 - (c.Ew * c.Tw) / (E_b * T_b);
        r.pkg_power_saving = 1.0 - (c.Epkg / c.Tw) / e.P_hi;
    } else {
        r.slowdown = r.energy_saving = r.edp_saving = r.pkg_power_saving = 0.0;
    }
    r.digest = digest_pack(c.dc, c.de);
    wp.wrec[ci] = r;
    p.c_vmax[ci] = c.invalid ? 0xFFFFFFFFu : 0u;
}

// Entry-major kernel of one chain kind: grid (ceil(n_traces / 128), lanes of the launch group), 128 threads.
template <class T, bool UNROLL>
__global__ void __launch_bounds__(128) magus_wallclock_em_kernel(const ReplayParams p, const EpiParams e,
                                                                 const WallParams wp, int q_base,
                                                                 const float* __restrict__ trace) {
    ptx::pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = q_base + blockIdx.y;
    if (j >= p.n_traces) return;
    const DevPolicy pol = p.pol[q];
    wallclock_chain_em<T, UNROLL>(p, e, wp, pol, chain_idx(p, q, j), j, trace);
}

// Round-major kernel (MAGUS_WALL_ROUNDMAJOR=1; the A32 loop as written): grid (ceil(n_traces / 128), n_lane), 128 threads: thread = chain (lane q = blockIdx.y, trace j).
__global__ void __launch_bounds__(128) magus_wallclock_kernel(const ReplayParams p, const EpiParams e,
                                                              const WallParams wp, const float* __restrict__ trace) {
    ptx::pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = blockIdx.y;
    if (j >= p.n_traces) return;
    const DevPolicy pol = p.pol[q];
    const int64_t ci = chain_idx(p, q, j);
#define MAGUS_WALL(...) wallclock_chain<__VA_ARGS__>(p, e, wp, pol, ci, j, trace)
    if (pol.kind == LANE_MAGUS) {
        if (pol.C <= kMaxC32) MAGUS_WALL(MagusTicker<0, false>);
        else MAGUS_WALL(MagusTicker<0, true>);
    } else if (pol.kind == LANE_TDP) {
        MAGUS_WALL(TdpTicker);
    } else {
        MAGUS_WALL(StaticMinTicker<false>);   // also the validate-only lane: its record is never read
    }
#undef MAGUS_WALL
}

}  // namespace magus
