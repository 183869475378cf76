// post_kernels.cuh -- after the replay kernel:
//   magus_fixup_epilogue_kernel  exact fix-up of speculative time segments (one warp per chain,
//                                lanes = segments), then the per-trace epilogue (closed-form energy
//                                model from sufficient statistics)
//   magus_static_max_kernel      analytic records of STATIC_MAX policies (never throttled, A17/A21)
//   magus_totals_kernel          per-policy fixed-order sums: thread-strided, warp-shuffle tree, smem
//   magus_argmin_kernel          argmin over policies of the total EDP (ties -> lowest index, A23)
//   magus_resim_kernel           per-tick decision codes for a dump window (test diagnostics)
//   magus_scan_invalid_kernel    first invalid (trace, tick) when the replay flagged one
#pragma once
#include "device_common.cuh"
#include "tickers.cuh"

namespace magus {

// Mirrors magus_trace_stats (include/magus_replay.h) field for field.
struct TraceRec {
    int64_t n_hi, n_thr, transitions, tune_events, lock_ticks;
    double T, E_pkg, E, EDP, slowdown, energy_saving, edp_saving, pkg_power_saving;
    uint64_t digest;
};

struct EpiParams {
    int32_t n_policies;       // user policies P
    int32_t n_samples;
    double Delta, P_lo, P_hi, P_gpu;
    double B_lo_d;            // (double)B_lo
    const float* w;           // [n_traces] compute weights
    TraceRec* rec;            // [n_traces][P]
    unsigned int* flag_invalid;
    int* fix_rounds;          // max over chains
    unsigned long long* fix_segments;   // total re-run segments
};

// Closed-form energy model of one (trace, policy) from its sufficient statistics (section 8):
//   T = Delta*((N - n_thr) + w*n_thr) + Delta*(1-w)*S_thr/B_lo
//   E_pkg = P_hi*Delta*n_hi + P_lo*(T - Delta*n_hi),   E = E_pkg + P_gpu*T
__device__ __forceinline__ void finish_record(TraceRec& r, const EpiParams& e, double w, int64_t n_hi, int64_t n_thr,
                                              int64_t trans, int64_t ev, int64_t lock, double sthr, uint64_t digest) {
    const double N = (double)e.n_samples;
    const double T = e.Delta * ((N - (double)n_thr) + w * (double)n_thr) + e.Delta * (1.0 - w) * sthr / e.B_lo_d;
    const double T_hi = e.Delta * (double)n_hi;
    const double E_pkg = e.P_hi * T_hi + e.P_lo * (T - T_hi);
    const double E = E_pkg + e.P_gpu * T;
    const double T_b = N * e.Delta;
    const double E_b = (e.P_hi + e.P_gpu) * T_b;
    r.n_hi = n_hi;
    r.n_thr = n_thr;
    r.transitions = trans;
    r.tune_events = ev;
    r.lock_ticks = lock;
    r.T = T;
    r.E_pkg = E_pkg;
    r.E = E;
    r.EDP = E * T;
    if (e.n_samples > 0) {
        r.slowdown = T / T_b - 1.0;
        r.energy_saving = 1.0 - E / E_b;
        r.edp_saving = 1.0 - (E * T) / (E_b * T_b);
        r.pkg_power_saving = 1.0 - (E_pkg / T) / e.P_hi;
    } else {
        r.slowdown = r.energy_saving = r.edp_saving = r.pkg_power_saving = 0.0;
    }
    r.digest = digest;
}

// Re-run segment s of chain (q, j) from the true entry state `tru` next to the speculative one `spec`
// until they coalesce (checked at 32-tick block ends); returns true if they did.  The statistics
// delta (true - spec) over the re-run prefix is added to the stored segment statistics.
template <class T>
__device__ bool rerun_segment(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j, const float* trace,
                              typename T::State& tru, typename T::State& spec) {
    const int seg_start = s * p.seg_len;
    const int seg_end = min(seg_start + p.seg_len, p.n_samples);
    SegStats dt, dp;
    dt.zero();
    dp.zero();
    uint32_t wct = 0, wcs = 0;
    bool coalesced = false;
    for (int bt0 = seg_start; bt0 < seg_end; bt0 += 32) {
        const uint32_t fst = T::level(tru), fss = T::level(spec);
        const int n = min(32, seg_end - bt0);
        for (int i = 0; i < n; ++i) {
            const int t = bt0 + i;
            const float D = __ldg(trace + (int64_t)t * p.trace_stride + j);
            const TickOut ot = T::template tick<false>(tru, D, pol, p.B_lo, p.B_hi, true, true);
            const TickOut os = T::template tick<false>(spec, D, pol, p.B_lo, p.B_hi, true, true);
            wct = (wct << 1) | ot.cmd;
            wcs = (wcs << 1) | os.cmd;
            dt.nthr += ot.thr; dt.lock += ot.hf; if (ot.thr) dt.sthr += (double)D;
            dp.nthr += os.thr; dp.lock += os.hf; if (os.thr) dp.sthr += (double)D;
        }
        uint32_t ewt = 0, ews = 0;
        if constexpr (T::kWarmupRules) {
            ewt = (uint32_t)tru.evh;
            ews = (uint32_t)spec.evh;
        }
        const int64_t b = bt0 >> 5;
        uint32_t* wout = p.words ? p.words + (((int64_t)q * p.n_traces + j) * p.n_blocks + b) * 2 : nullptr;
        fold_block(dt, wct, ewt, fst, n, b, wout);
        fold_block(dp, wcs, ews, fss, n, b, nullptr);
        if (T::equal(tru, spec, pol)) {
            coalesced = true;
            break;
        }
    }
    const int64_t si = stat_idx(p, q, s, j);
    p.s_nhi[si] += dt.nhi - dp.nhi;
    p.s_nthr[si] += dt.nthr - dp.nthr;
    p.s_trans[si] += dt.trans - dp.trans;
    p.s_ev[si] += dt.ev - dp.ev;
    p.s_lock[si] += dt.lock - dp.lock;
    p.s_sthr[si] += dt.sthr - dp.sthr;
    p.s_digest[si] += dt.digest - dp.digest;
    return coalesced;
}

template <class T>
__device__ void fixup_and_finish(const ReplayParams& p, const EpiParams& e, const DevPolicy& pol, int q, int j,
                                 const float* trace, int lane) {
    int rounds = 0;
    unsigned long long reruns = 0;
    if (T::kStateful && p.n_seg > 1) {
        for (;;) {
            bool any = false;
            for (int base = 1; base < p.n_seg; base += 32) {
                const int s = base + lane;
                const bool need = s < p.n_seg && !T::stored_equal(p, pol, q, 0, s, 1, s - 1, j);
                const unsigned m = __ballot_sync(0xffffffffu, need);
                if (m == 0) continue;
                any = true;
                typename T::State tru, spec;
                if (need) {
                    T::load(tru, p, pol, 1, q, s - 1, j);
                    T::load(spec, p, pol, 0, q, s, j);
                }
                __syncwarp();
                if (need) {
                    const typename T::State entry = tru;   // the entry the corrected statistics belong to
                    const bool co = rerun_segment<T>(p, pol, q, s, j, trace, tru, spec);
                    T::save(entry, p, pol, 0, q, s, j);
                    if (!co) T::save(tru, p, pol, 1, q, s, j);
                    ++reruns;
                }
                __syncwarp();
            }
            if (!any) break;
            ++rounds;
        }
    }
    // sum the chain's segment statistics: lane-sequential over s = lane, lane+32, ..., then a fixed
    // xor-shuffle tree (deterministic order)
    uint64_t nhi = 0, nthr = 0, trans = 0, ev = 0, lock = 0, dig = 0;
    uint32_t vmax = 0;
    double sthr = 0.0;
    for (int s = lane; s < p.n_seg; s += 32) {
        const int64_t si = stat_idx(p, q, s, j);
        nhi += p.s_nhi[si];
        nthr += p.s_nthr[si];
        trans += p.s_trans[si];
        ev += p.s_ev[si];
        lock += p.s_lock[si];
        dig += p.s_digest[si];
        vmax = max(vmax, p.s_vmax[si]);
        sthr += p.s_sthr[si];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nhi += __shfl_xor_sync(0xffffffffu, nhi, o);
        nthr += __shfl_xor_sync(0xffffffffu, nthr, o);
        trans += __shfl_xor_sync(0xffffffffu, trans, o);
        ev += __shfl_xor_sync(0xffffffffu, ev, o);
        lock += __shfl_xor_sync(0xffffffffu, lock, o);
        dig += __shfl_xor_sync(0xffffffffu, dig, o);
        vmax = max(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        sthr += __shfl_xor_sync(0xffffffffu, sthr, o);
    }
    if (lane == 0) {
        if (pol.policy_index >= 0) {
            TraceRec& r = e.rec[(int64_t)j * e.n_policies + pol.policy_index];
            finish_record(r, e, (double)e.w[j], (int64_t)nhi, (int64_t)nthr, (int64_t)trans, (int64_t)ev,
                          (int64_t)lock, sthr, dig);
        }
        if (vmax > p.bwbits) atomicOr(e.flag_invalid, 1u);
        if (rounds) atomicMax(e.fix_rounds, rounds);
    }
    unsigned long long rr = reruns;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
    if (lane == 0 && rr) atomicAdd(e.fix_segments, rr);
}

__global__ void __launch_bounds__(256) magus_fixup_epilogue_kernel(const ReplayParams p, const EpiParams e,
                                                                   const float* __restrict__ trace) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.y;
    const int j = warp;
    if (j >= p.n_traces) return;
    const DevPolicy pol = p.pol[q];
#define MAGUS_FIX(...) fixup_and_finish<__VA_ARGS__>(p, e, pol, q, j, trace, lane)
    if (pol.kind == LANE_MAGUS) {
        if (pol.C <= 32) {
            switch (pol.k) {
                case 1: MAGUS_FIX(MagusTicker<1, false>); return;
                case 2: MAGUS_FIX(MagusTicker<2, false>); return;
                case 3: MAGUS_FIX(MagusTicker<3, false>); return;
                case 4: MAGUS_FIX(MagusTicker<4, false>); return;
                case 5: MAGUS_FIX(MagusTicker<5, false>); return;
                case 6: MAGUS_FIX(MagusTicker<6, false>); return;
                case 7: MAGUS_FIX(MagusTicker<7, false>); return;
                case 8: MAGUS_FIX(MagusTicker<8, false>); return;
                default: MAGUS_FIX(MagusTicker<0, false>); return;
            }
        } else {
            switch (pol.k) {
                case 1: MAGUS_FIX(MagusTicker<1, true>); return;
                case 2: MAGUS_FIX(MagusTicker<2, true>); return;
                case 4: MAGUS_FIX(MagusTicker<4, true>); return;
                case 8: MAGUS_FIX(MagusTicker<8, true>); return;
                default: MAGUS_FIX(MagusTicker<0, true>); return;
            }
        }
    } else if (pol.kind == LANE_TDP) {
        MAGUS_FIX(TdpTicker);
    } else if (pol.kind == LANE_STATIC_MIN) {
        MAGUS_FIX(StaticMinTicker<false>);
    } else {
        MAGUS_FIX(StaticMinTicker<true>);
    }
#undef MAGUS_FIX
}

// STATIC_MAX records: at f_max A = D <= bw_max, never throttled, never a transition or a tune flag.
__global__ void magus_static_max_kernel(const EpiParams e, int n_traces, const int* __restrict__ smax_policies,
                                        int n_smax, uint64_t digest_all_hi) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n_traces * n_smax) return;
    const int j = (int)(i / n_smax), pi = smax_policies[i % n_smax];
    TraceRec& r = e.rec[(int64_t)j * e.n_policies + pi];
    finish_record(r, e, (double)e.w[j], (int64_t)e.n_samples, 0, 0, 0, 0, 0.0, digest_all_hi);
}

constexpr int kTotThreads = 256;
constexpr int kNTot = 13;   // MAGUS_N_TOTALS

// One block per policy: fixed-order sum over traces (thread-strided, then xor-shuffle tree, then the
// 8 warp partials in order).  Deterministic for a fixed launch configuration.
__global__ void __launch_bounds__(kTotThreads) magus_totals_kernel(const TraceRec* __restrict__ rec, int n_traces,
                                                                    int n_policies, double* __restrict__ totals) {
    const int p = blockIdx.x;
    double acc[kNTot - 1];
#pragma unroll
    for (int f = 0; f < kNTot - 1; ++f) acc[f] = 0.0;
    for (int j = threadIdx.x; j < n_traces; j += kTotThreads) {
        const TraceRec& r = rec[(int64_t)j * n_policies + p];
        acc[0] += r.E;
        acc[1] += r.E_pkg;
        acc[2] += r.T;
        acc[3] += r.EDP;
        acc[4] += r.slowdown;
        acc[5] += r.energy_saving;
        acc[6] += r.edp_saving;
        acc[7] += (double)r.n_hi;
        acc[8] += (double)r.n_thr;
        acc[9] += (double)r.transitions;
        acc[10] += (double)r.tune_events;
        acc[11] += (double)r.lock_ticks;
    }
#pragma unroll
    for (int f = 0; f < kNTot - 1; ++f)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o);
    __shared__ double part[kTotThreads / 32][kNTot - 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int f = 0; f < kNTot - 1; ++f) part[warp][f] = acc[f];
    __syncthreads();
    if (threadIdx.x < kNTot - 1) {
        double s = 0.0;
        for (int w = 0; w < kTotThreads / 32; ++w) s += part[w][threadIdx.x];
        totals[p * kNTot + threadIdx.x] = s;
    }
    if (threadIdx.x == 0) totals[p * kNTot + kNTot - 1] = (double)n_traces;
}

__global__ void magus_argmin_kernel(const double* __restrict__ totals, int n_policies, int* __restrict__ argmin) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int best = 0;
    double bv = totals[3];
    for (int p = 1; p < n_policies; ++p) {
        const double v = totals[p * kNTot + 3];
        if (v < bv) {
            bv = v;
            best = p;
        }
    }
    *argmin = best;
}

// Per-tick codes (DESIGN A27) for traces [first, first + n) of every policy, re-simulated from t = 0
// with the same tick functions as the replay kernel.  codes: [n_samples][n][P].
template <class T>
__device__ void resim_chain(const ReplayParams& p, const DevPolicy& pol, int jd, int j, int n_win, int P,
                            const float* trace, uint8_t* codes) {
    typename T::State s;
    T::init(s, pol, true);
    const int k = pol.k, C = pol.C;
    for (int t = 0; t < p.n_samples; ++t) {
        const float D = trace[(int64_t)t * p.trace_stride + j];
        const uint32_t lvl = T::level(s);
        const bool ready = t >= k, lfull = t >= k + C - 1;
        const TickOut o = T::template tick<true>(s, D, pol, p.B_lo, p.B_hi, ready, lfull);
        uint32_t c = o.cmd | ((T::kWarmupRules && ready) ? 2u : 0u) | (o.ev << 2) | (o.hf << 3) | (o.sig << 4) |
                     (o.thr << 6) | (lvl << 7);
        codes[((int64_t)t * n_win + jd) * P + pol.policy_index] = (uint8_t)c;
    }
}

__global__ void magus_resim_kernel(const ReplayParams p, const float* __restrict__ trace, int first, int n_win, int P,
                                   uint8_t* codes) {
    const int jd = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = blockIdx.y;
    if (jd >= n_win) return;
    const DevPolicy pol = p.pol[q];
    if (pol.policy_index < 0) return;
    const int j = first + jd;
#define MAGUS_RESIM(...) resim_chain<__VA_ARGS__>(p, pol, jd, j, n_win, P, trace, codes)
    if (pol.kind == LANE_MAGUS) {
        if (pol.C <= 32) MAGUS_RESIM(MagusTicker<0, false>);
        else MAGUS_RESIM(MagusTicker<0, true>);
    } else if (pol.kind == LANE_TDP) {
        MAGUS_RESIM(TdpTicker);
    } else {
        MAGUS_RESIM(StaticMinTicker<false>);
    }
#undef MAGUS_RESIM
}

__global__ void magus_fill_codes_kernel(uint8_t* codes, int64_t n_rows, int P, int pi, uint8_t value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_rows) codes[i * P + pi] = value;
}

// First invalid sample (A17): valid iff bits(D) <= bits(largest fp32 <= bw_max), or D == -0.0.
__global__ void magus_scan_invalid_kernel(const float* __restrict__ trace, int n_traces, int n_samples,
                                          int64_t stride, uint32_t bwbits, unsigned long long* first_key) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_traces) return;
    for (int t = 0; t < n_samples; ++t) {
        const uint32_t b = __float_as_uint(trace[(int64_t)t * stride + j]);
        if (b > bwbits && b != 0x80000000u) {
            atomicMin(first_key, ((unsigned long long)j << 32) | (unsigned long long)(uint32_t)t);
            return;
        }
    }
}

}  // namespace magus
