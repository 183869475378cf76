// post_kernels.cuh -- the kernels around the replay kernel:
//   magus_prepass_kernel         run start: zeroes the run's scratch words, speculation aid (first_low)
//   magus_fix_mark_kernel,       exact fix-up of speculative time segments: the first wrong entry of
//   magus_fix_lockstep_kernel    every chain, then one walk per chain in time order
//   magus_totals_kernel          per-trace records (closed-form energy model from sufficient statistics,
//                                DESIGN.md section 8) and per-policy fixed-order sums
//   magus_resim_kernel           per-tick decision codes for a dump window (test diagnostics)
//   magus_scan_invalid_kernel    first invalid (trace, tick) when the replay flagged one
#pragma once
#include "device_common.cuh"
#include "ptx.cuh"
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
//   T = Delta*(N + (1-w)*X/B_lo),  X = sum over throttled ticks of (D - B_lo)  (exact in fp64)
//   E_pkg = P_hi*Delta*n_hi + P_lo*(T - Delta*n_hi),   E = E_pkg + P_gpu*T
__device__ __forceinline__ void finish_record(TraceRec& r, const EpiParams& e, double w, int64_t n_hi, int64_t n_thr,
                                              int64_t trans, int64_t ev, int64_t lock, double sexc, uint64_t digest) {
    const double N = (double)e.n_samples;
    // sum of tau over the ticks: Delta per tick, plus Delta*(1-w)*(D - B_lo)/B_lo per throttled tick
    const double T = e.Delta * (N + (1.0 - w) * sexc / e.B_lo_d);
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

// ================================================================================= exact fix-up
// Segment s >= 1 of chain (q, j) was replayed from a speculative entry E_s.
// It is exact iff E_s equals the previous segment's true exit X_{s-1}.  Where they differ, the
// segment is re-run from X_{s-1} next to the speculative trajectory from E_s until the two
// coalesce (identical state at a 32-tick block end -- from then on they are identical); the
// statistics delta (true - speculative) over the re-run prefix is added to the chain's totals.  If
// they never coalesce, the true exit is carried into the next boundary (the chain walk).

struct FixParams {
    int32_t* first_bad;       // [Q][n_traces] first wrong segment entry of a chain (INT_MAX: none)
};

template <class T>
__device__ __forceinline__ bool entry_mismatch(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j) {
    return !T::stored_equal(p, pol, q, 0, s, 1, s - 1, j);
}

__device__ __forceinline__ bool entry_mismatch_any(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j) {
    if (pol.kind == LANE_MAGUS) return entry_mismatch<MagusTicker<0, true>>(p, pol, q, s, j);
    if (pol.kind == LANE_TDP) return entry_mismatch<TdpTicker>(p, pol, q, s, j);
    return false;
}

// Chain walk, step 1: every (q, s >= 1, j) whose speculative entry differs from the previous exit lowers
// the chain's first_bad to s (first_bad is INT_MAX between runs: the walk kernel resets what it reads).
__global__ void __launch_bounds__(256) magus_fix_mark_kernel(const ReplayParams p, const FixParams f) {
    ptx::pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y + 1, q = blockIdx.z;
    if (j >= p.n_traces) return;
    const DevPolicy pol = p.pol[q];
    if (entry_mismatch_any(p, pol, q, s, j)) atomicMin(f.first_bad + (int64_t)q * p.n_traces + j, s);
}

// ------------------------------------------------------------------ the open-loop fix-up (A30)
// Open loop (magus_model.observe = 1): A = D, so Alg. 1's derivatives, the tune flags, the window count and Alg. 2's
// lock depend on the trace only, and after the warm-up (>= k + C - 1 ticks) a speculative segment's ring, log and count
// equal the true ones.  Only its entry LEVEL can be wrong, and the level is a last-writer scan of the events (lock |
// flag: cmd = lock | +1 ? f_max : -1 ? f_min : level).  So a segment replayed from the wrong entry level g (true X)
// differs only up to its first event e (recorded by the replay in st_first): the level in effect at ticks [0, e] and
// the cmd at ticks [0, e) are X instead of g, and the transition at e is [cmd_e != X] instead of [cmd_e != g]; with no
// event the whole segment is at X and so is its exit.  One thread per chain resolves the entries in segment order and
// adds these closed-form deltas (n_hi, transitions, the cmd half of the digest, the dumped cmd words) -- no chain walk.
// One warp per chain, one lane per segment (32 segments per pass): the true entry level of segment s is the
// (speculative, hence true) exit of the last earlier segment with an event, or the carried level -- a ballot and a
// shuffle, not a serial walk over the segments.
__global__ void __launch_bounds__(128) magus_fix_openloop_kernel(const ReplayParams p, const EpiParams e, int q_base) {
    ptx::pdl_wait();
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int q = q_base + blockIdx.y;
    if (j >= p.n_traces) return;   // warp-uniform
    uint32_t carry = p.st_f[st_idx(p, 1, q, 0, j)];   // segment 0 starts from the exact initial state: its exit is true
    uint32_t fixed = 0;
    for (int base = 1; base < p.n_seg; base += 32) {
        const int s = base + lane;
        const bool valid = s < p.n_seg;
        uint32_t g = 0, spec_exit = 0;
        int32_t code = -1;
        if (valid) {
            const int64_t si = st_idx(p, 0, q, s, j);
            g = p.st_f[si];                      // the speculative entry level
            code = p.st_first[si];
            spec_exit = p.st_f[st_idx(p, 1, q, s, j)];
        }
        const bool has_ev = valid && code >= 0;
        const uint32_t m = __ballot_sync(0xffffffffu, has_ev);
        const uint32_t below = m & ((1u << lane) - 1u);
        const int src = below ? 31 - __clz(below) : 0;
        const uint32_t ev_exit = __shfl_sync(0xffffffffu, spec_exit, src);
        const uint32_t x = below ? ev_exit : carry;     // the true entry level
        const uint32_t true_exit = has_ev ? spec_exit : x;
        if (valid && x != g) {
            const int seg_start = seg_begin(p, s), L = seg_finish(p, s) - seg_start;
            const int ev = has_ev ? (code & 0x3FFFFFFF) : L;   // first event (or the segment's end)
            const uint32_t tgt = ((uint32_t)code >> 30) & 1u;   // cmd at the event
            const int n_lv = has_ev ? ev + 1 : L;               // ticks whose level in effect is the entry level
            const int n_cmd = ev;                               // ticks whose cmd is the entry level
            const int32_t sg = x ? 1 : -1;
            const int32_t dtr = has_ev ? (int32_t)(tgt != x) - (int32_t)(tgt != g) : 0;
            uint32_t ddc = 0;   // cmd half of the digest: bits of ticks [seg_start, seg_start + n_cmd) flip g -> x
            for (int t0 = 0; t0 < n_cmd; t0 += 32) {
                const int r = min(32, n_cmd - t0);
                const uint32_t mask = r >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> r);   // ticks t0.. at bits 31..
                const int64_t b = (seg_start + t0) >> 5;
                ddc += (uint32_t)sg * (mask * p.dkeys[b].x);
                if (p.words) p.words[(chain_idx(p, q, j) * p.n_blocks + b) * 2] ^= mask;
            }
            add_to_chain(p, q, j, (uint32_t)(sg * n_lv), 0u, (uint32_t)dtr, 0u, 0u, 0.0, digest_pack(ddc, 0u));
            if (!has_ev) p.st_f[st_idx(p, 1, q, s, j)] = (uint8_t)x;   // no event: it ends at the true entry level
            ++fixed;
        }
        const int last = min(31, p.n_seg - 1 - base);
        carry = __shfl_sync(0xffffffffu, true_exit, last);
    }
    fixed = __reduce_add_sync(0xffffffffu, fixed);
    if (lane == 0 && fixed) {
        atomicAdd(e.fix_segments, (unsigned long long)fixed);
        atomicMax(e.fix_rounds, 1);
    }
}

// ------------------------------------------------------------------ one segment re-run (generic kinds)
template <class T>
__device__ bool rerun_segment(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j, const float* trace,
                              typename T::State& tru, typename T::State& spec) {
    const int seg_start = seg_begin(p, s);
    const int seg_end = seg_finish(p, s);
    SegStats dt, dp;
    dt.zero();
    dp.zero();
    uint32_t wct = 0, wcs = 0;
    bool coalesced = false;
    for (int bt0 = seg_start; bt0 < seg_end; bt0 += 32) {
        const uint32_t fst = T::level(tru), fss = T::level(spec);
        const int n = min(32, seg_end - bt0);
        float dv[32];   // the block's samples, loaded up front (32 loads in flight)
#pragma unroll
        for (int i = 0; i < 32; ++i) dv[i] = (i < n) ? __ldg(trace + (int64_t)(bt0 + i) * p.trace_stride + j) : 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i < n) {
                const float D = dv[i];
                const TickOut ot = T::template tick<false>(tru, D, pol, p.B_lo, p.B_hi, true, true);
                const TickOut os = T::template tick<false>(spec, D, pol, p.B_lo, p.B_hi, true, true);
                wct = (wct << 1) | ot.cmd;
                wcs = (wcs << 1) | os.cmd;
                dt.nthr += ot.thr; dt.lock += ot.hf; if (ot.thr) dt.sexc += (double)D - (double)p.B_lo;
                dp.nthr += os.thr; dp.lock += os.hf; if (os.thr) dp.sexc += (double)D - (double)p.B_lo;
            }
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
    add_to_chain(p, q, j, dt.nhi - dp.nhi, dt.nthr - dp.nthr, dt.trans - dp.trans, dt.ev - dp.ev, dt.lock - dp.lock,
                 dt.sexc - dp.sexc, digest_pack(dt.dc - dp.dc, dt.de - dp.de));
    return coalesced;
}

// ------------------------------------------------------------------ latency-optimised re-run (chain walk)
// One MAGUS tick with a short loop-carried path: everything that depends only on the sample and on the
// ring (A_{t-k}, known k ticks ahead) is computed for both levels first -- the f_min observation, both
// derivative numerators and their Alg. 1 flags -- and the level in effect only selects among them.
// The chain-to-chain dependency is then select -> log / window count -> Alg. 2 -> decision.  Same
// decisions as magus_tick (the incremental window count of tick4_asm.cuh, scaled by 2^(C-1)).
template <int K>
__device__ __forceinline__ TickOut walk_tick(MagusState<K, false>& s, float D, double dd, const DevPolicy& pol,
                                             float B_lo, double Blo_d, uint32_t bitc) {
    const double old = s.ring.oldest(pol.k);
    const bool thr_lo = D > B_lo;                     // throttled if the level in effect is f_min (A14)
    const double ad_lo = thr_lo ? Blo_d : dd;
    const double dv_lo = ad_lo - old, dv_hi = dd - old;
    const bool inc_lo = dv_lo > pol.dinc, dec_lo = dv_lo < pol.ddec;
    const bool inc_hi = dv_hi > pol.dinc, dec_hi = dv_hi < pol.ddec;
    const bool hi = s.f != 0u;
    const bool inc = hi ? inc_hi : inc_lo, dec = hi ? dec_hi : dec_lo;
    const bool ev = inc || dec;
    const uint32_t leaving = s.evh & bitc;
    s.evh = (s.evh << 1) | (ev ? 1u : 0u);
    s.cnt = s.cnt - leaving + (ev ? bitc : 0u);
    const bool hf = s.cnt >= pol.smin_sc;
    TickOut o;
    o.cmd = (hf || inc || (hi && !dec)) ? 1u : 0u;
    o.thr = (!hi && thr_lo) ? 1u : 0u;
    o.ev = ev ? 1u : 0u;
    o.hf = hf ? 1u : 0u;
    o.sig = 0;
    s.ring.push(hi ? dd : ad_lo, pol.k);
    s.f = o.cmd;
    return o;
}

// rerun_segment for the register-ring MAGUS kinds: walk_tick for the true and the speculative state side
// by side (two independent recurrences per lane), whole 32-tick blocks without per-tick predicates, and
// the samples of the next two blocks loaded while the current block is stepped (strided rows of the
// trace: one sector each; the loads, not the arithmetic, bound a lone walking warp otherwise).
template <int K, bool FULL>
__device__ __forceinline__ void walk_block(MagusState<K, false>& tru, MagusState<K, false>& spec, SegStats& dt,
                                           SegStats& dp, const float* dv, int n, const DevPolicy& pol, float B_lo,
                                           double Blo_d, uint32_t bitc, uint32_t& wct, uint32_t& wcs) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (FULL || i < n) {
            const float D = dv[i];
            const double dd = (double)D;
            const TickOut ot = walk_tick<K>(tru, D, dd, pol, B_lo, Blo_d, bitc);
            const TickOut os = walk_tick<K>(spec, D, dd, pol, B_lo, Blo_d, bitc);
            wct = (wct << 1) | ot.cmd;
            wcs = (wcs << 1) | os.cmd;
            dt.nthr += ot.thr;
            dt.lock += ot.hf;
            dt.sexc += ot.thr ? dd - Blo_d : 0.0;
            dp.nthr += os.thr;
            dp.lock += os.hf;
            dp.sexc += os.thr ? dd - Blo_d : 0.0;
        }
    }
}

template <int K>
__device__ bool rerun_segment_walk(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j,
                                   const float* trace, MagusState<K, false>& tru, MagusState<K, false>& spec) {
    const int seg_start = seg_begin(p, s);
    const int seg_end = seg_finish(p, s);
    const double Blo_d = (double)p.B_lo;
    const uint32_t bitc = 1u << (pol.C - 1);
    SegStats dt, dp;
    dt.zero();
    dp.zero();
    bool coalesced = false;
    const float* col = trace + j;
    float n1[32], n2[32];   // samples of the next two blocks
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        n1[i] = (seg_start + i < seg_end) ? __ldg(col + (int64_t)(seg_start + i) * p.trace_stride) : 0.0f;
        n2[i] = (seg_start + 32 + i < seg_end) ? __ldg(col + (int64_t)(seg_start + 32 + i) * p.trace_stride) : 0.0f;
    }
    for (int bt0 = seg_start; bt0 < seg_end; bt0 += 32) {
        float dv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            dv[i] = n1[i];
            n1[i] = n2[i];
        }
        const int nb = bt0 + 64;
        if (nb + 32 <= seg_end) {
#pragma unroll
            for (int i = 0; i < 32; ++i) n2[i] = __ldg(col + (int64_t)(nb + i) * p.trace_stride);
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) n2[i] = (nb + i < seg_end) ? __ldg(col + (int64_t)(nb + i) * p.trace_stride) : 0.f;
        }
        const uint32_t fst = tru.f, fss = spec.f;
        const int n = min(32, seg_end - bt0);
        uint32_t wct = 0, wcs = 0;
        if (n == 32) walk_block<K, true>(tru, spec, dt, dp, dv, n, pol, p.B_lo, Blo_d, bitc, wct, wcs);
        else walk_block<K, false>(tru, spec, dt, dp, dv, n, pol, p.B_lo, Blo_d, bitc, wct, wcs);
        const int64_t b = bt0 >> 5;
        uint32_t* wout = p.words ? p.words + (((int64_t)q * p.n_traces + j) * p.n_blocks + b) * 2 : nullptr;
        fold_block(dt, wct, tru.evh, fst, n, b, wout);
        fold_block(dp, wcs, spec.evh, fss, n, b, nullptr);
        if (MagusTicker<K, false>::equal(tru, spec, pol)) {
            coalesced = true;
            break;
        }
    }
    add_to_chain(p, q, j, dt.nhi - dp.nhi, dt.nthr - dp.nthr, dt.trans - dp.trans, dt.ev - dp.ev, dt.lock - dp.lock,
                 dt.sexc - dp.sexc, digest_pack(dt.dc - dp.dc, dt.de - dp.de));
    return coalesced;
}

template <class T>
struct WalkRerun {
    __device__ static bool run(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j, const float* trace,
                               typename T::State& tru, typename T::State& spec) {
        return rerun_segment<T>(p, pol, q, s, j, trace, tru, spec);
    }
};
template <int K>
struct WalkRerun<MagusTicker<K, false>> {
    __device__ static bool run(const ReplayParams& p, const DevPolicy& pol, int q, int s, int j, const float* trace,
                               MagusState<K, false>& tru, MagusState<K, false>& spec) {
        if constexpr (K >= 1) return rerun_segment_walk<K>(p, pol, q, s, j, trace, tru, spec);
        else return rerun_segment<MagusTicker<K, false>>(p, pol, q, s, j, trace, tru, spec);
    }
};

// ------------------------------------------------------------------ lockstep chain walk (k <= 3)
// A warp walks the 32 consecutive chains (traces) of its lanes in lockstep, lane = chain, each lane
// stepping its true and its speculative state over the same samples with the generated 2-chain stage
// block (MAGUS_WSTAGE_K<K>, tick4_asm.cuh).  The warp's loads are one coalesced row segment per tick.
// Segments in which no lane of the warp walks are skipped; within a segment a lane stops at the block
// end where its two states coalesce (adding the statistics delta of its prefix), and the warp leaves the
// segment when every lane has stopped.  Lanes that do not walk step garbage that is never used.
template <int K>
__device__ __forceinline__ void walk_stage(MagusState<K, false>* st, float* lock, float* nthr, uint32_t* wcmd,
                                           SegStats* ss, const float* d8, const DevPolicy& pol, double Blo_d) {
    uint32_t e0 = st[0].evh, e1 = st[1].evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define WALK_TAIL                                                                                                \
    e0, e1, st[0].cnt, st[1].cnt, ss[0].sexc, ss[1].sexc, lock[0], lock[1], nthr[0], nthr[1], wcmd[0], wcmd[1],    \
        __float_as_uint(d8[0]), __float_as_uint(d8[1]), __float_as_uint(d8[2]), __float_as_uint(d8[3]),            \
        __float_as_uint(d8[4]), __float_as_uint(d8[5]), __float_as_uint(d8[6]), __float_as_uint(d8[7]), Blo_d,      \
        pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define R0(i) st[0].ring.v[i]
#define R1(i) st[1].ring.v[i]
    if constexpr (K == 1) {
        MAGUS_WSTAGE_K1(st[0].f, st[1].f, R0(0), R1(0), WALK_TAIL);
    } else if constexpr (K == 2) {
        MAGUS_WSTAGE_K2(st[0].f, st[1].f, R0(0), R0(1), R1(0), R1(1), WALK_TAIL);
    } else if constexpr (K == 3) {
        MAGUS_WSTAGE_K3(st[0].f, st[1].f, R0(0), R0(1), R0(2), R1(0), R1(1), R1(2), WALK_TAIL);
    } else if constexpr (K == 4) {
        MAGUS_WSTAGE_K4(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R1(0), R1(1), R1(2), R1(3), WALK_TAIL);
    } else if constexpr (K == 5) {
        MAGUS_WSTAGE_K5(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R1(0), R1(1), R1(2), R1(3), R1(4),
                        WALK_TAIL);
    } else if constexpr (K == 6) {
        MAGUS_WSTAGE_K6(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R1(0), R1(1), R1(2), R1(3),
                        R1(4), R1(5), WALK_TAIL);
    } else if constexpr (K == 7) {
        MAGUS_WSTAGE_K7(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R0(6), R1(0), R1(1), R1(2),
                        R1(3), R1(4), R1(5), R1(6), WALK_TAIL);
    } else {
        MAGUS_WSTAGE_K8(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R0(6), R0(7), R1(0), R1(1),
                        R1(2), R1(3), R1(4), R1(5), R1(6), R1(7), WALK_TAIL);
    }
#undef R0
#undef R1
#undef WALK_TAIL
    st[0].evh = e0;
    st[1].evh = e1;
}

// the samples [t0, min(t0 + 32, end)) of one trace column (coalesced across the warp's lanes)
__device__ __forceinline__ void walk_load(float* v, const float* col, int t0, int end, int64_t stride) {
    const float* c = col + (int64_t)t0 * stride;
    if (t0 + 32 <= end) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __ldg(c + i * stride);
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = (t0 + i < end) ? __ldg(c + i * stride) : 0.f;
    }
}

// lockstep step of one whole 32-tick block for the pair (true, speculative) of every lane
template <class T>
struct LockstepStep;
template <int K>
struct LockstepStep<MagusTicker<K, false>> {
    __device__ __forceinline__ static void run(MagusState<K, false>* st, float* lock, float* nthr, uint32_t* wcmd,
                                               SegStats* ss, const float* dv, const DevPolicy& pol,
                                               const ReplayParams&, double Blo_d) {
#pragma unroll
        for (int g = 0; g < 4; ++g) walk_stage<K>(st, lock, nthr, wcmd, ss, dv + 8 * g, pol, Blo_d);
    }
};
template <>
struct LockstepStep<TdpTicker> {
    __device__ __forceinline__ static void run(TdpTicker::State* st, float*, float*, uint32_t* wcmd, SegStats* ss,
                                               const float* dv, const DevPolicy& pol, const ReplayParams& p,
                                               double Blo_d) {
        uint32_t vmax = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            TdpTicker::fast(st[0], dv[i], pol, p.B_lo, Blo_d, wcmd[0], ss[0], vmax);
            TdpTicker::fast(st[1], dv[i], pol, p.B_lo, Blo_d, wcmd[1], ss[1], vmax);
        }
    }
};

// one tick of the ragged last block (any chain kind)
template <class T>
__device__ __forceinline__ void lockstep_tick(typename T::State& st, float D, const DevPolicy& pol,
                                              const ReplayParams& p, double Blo_d, uint32_t& wc, SegStats& ss) {
    TickOut o;
    if constexpr (T::kWarmupRules) o = walk_tick<sizeof(st.ring.v) / sizeof(double)>(st, D, (double)D, pol, p.B_lo,
                                                                                      Blo_d, 1u << (pol.C - 1));
    else o = T::template tick<false>(st, D, pol, p.B_lo, p.B_hi, true, true);
    wc = (wc << 1) | o.cmd;
    ss.nthr += o.thr;
    ss.lock += o.hf;
    if (o.thr) ss.sexc += (double)D - Blo_d;
}

template <class T>
__global__ void __launch_bounds__(32) magus_fix_lockstep_kernel(const ReplayParams p, const EpiParams e,
                                                                const FixParams f, int q_base,
                                                                const float* __restrict__ trace) {
    ptx::pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = q_base + blockIdx.y;
    const bool valid = j < p.n_traces;
    int s0 = 0x7FFFFFFF;
    if (valid) {
        const int64_t ci = (int64_t)q * p.n_traces + j;
        s0 = f.first_bad[ci];
        if (s0 < 0x7FFFFFFF) f.first_bad[ci] = 0x7FFFFFFF;   // reset for the next run
    }
    const int ws = __reduce_min_sync(0xffffffffu, s0);
    if (ws >= p.n_seg) return;   // warp-uniform
    const DevPolicy pol = p.pol[q];
    const double Blo_d = (double)p.B_lo;
    const float* col = trace + (valid ? j : 0);
    typename T::State st[2];   // [0] true state, [1] speculative state
    bool walking = false;      // this lane's true state differs from its stored trajectory
    int walked = 0;
    for (int s = ws; s < p.n_seg; ++s) {
        if (walking) {
            T::load(st[1], p, pol, 0, q, s, j);
            if (T::equal(st[0], st[1], pol)) walking = false;
        } else if (valid && s >= s0 && !T::stored_equal(p, pol, q, 0, s, 1, s - 1, j)) {
            T::load(st[0], p, pol, 1, q, s - 1, j);
            T::load(st[1], p, pol, 0, q, s, j);
            walking = true;
        }
        if (!__any_sync(0xffffffffu, walking)) continue;
        walked += walking ? 1 : 0;
        const int seg_start = seg_begin(p, s), seg_end = seg_finish(p, s);
        SegStats ss[2];
        ss[0].zero();
        ss[1].zero();
        float lock[2] = {0.f, 0.f}, nthr[2] = {0.f, 0.f};
        bool active = walking;
        // the samples of the next two blocks are loaded while the current block is stepped
        float n1[32], n2[32];
        walk_load(n1, col, seg_start, seg_end, p.trace_stride);
        if (seg_start + 32 < seg_end) walk_load(n2, col, seg_start + 32, seg_end, p.trace_stride);
        for (int bt0 = seg_start; bt0 < seg_end; bt0 += 32) {
            if (!__any_sync(0xffffffffu, active)) break;
            const int n = min(32, seg_end - bt0);
            float dv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                dv[i] = n1[i];
                n1[i] = n2[i];
            }
            if (bt0 + 64 < seg_end) walk_load(n2, col, bt0 + 64, seg_end, p.trace_stride);
            const uint32_t fs0 = T::level(st[0]), fs1 = T::level(st[1]);
            uint32_t wcmd[2] = {0u, 0u};
            if (n == 32) {
                LockstepStep<T>::run(st, lock, nthr, wcmd, ss, dv, pol, p, Blo_d);
            } else {   // the ragged last block of a trace (static indices: dv stays in registers)
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i < n) {
                        lockstep_tick<T>(st[0], dv[i], pol, p, Blo_d, wcmd[0], ss[0]);
                        lockstep_tick<T>(st[1], dv[i], pol, p, Blo_d, wcmd[1], ss[1]);
                    }
                }
            }
            const int64_t b = bt0 >> 5;
            uint32_t* wout = (active && p.words) ? p.words + (((int64_t)q * p.n_traces + j) * p.n_blocks + b) * 2
                                                 : nullptr;
            uint32_t ew0 = 0, ew1 = 0;
            if constexpr (T::kWarmupRules) {
                ew0 = (uint32_t)st[0].evh;
                ew1 = (uint32_t)st[1].evh;
            }
            fold_block(ss[0], wcmd[0], ew0, fs0, n, b, wout);
            fold_block(ss[1], wcmd[1], ew1, fs1, n, b, nullptr);
            const bool same = T::equal(st[0], st[1], pol);
            if (active && (same || bt0 + 32 >= seg_end)) {   // coalesced (the rest is right), or segment end
                add_to_chain(p, q, j, ss[0].nhi - ss[1].nhi,
                             ss[0].nthr - ss[1].nthr + ((uint32_t)nthr[0] - (uint32_t)nthr[1]),
                             ss[0].trans - ss[1].trans, ss[0].ev - ss[1].ev,
                             ss[0].lock - ss[1].lock + ((uint32_t)lock[0] - (uint32_t)lock[1]),
                             ss[0].sexc - ss[1].sexc, digest_pack(ss[0].dc - ss[1].dc, ss[0].de - ss[1].de));
                walking = !same;   // carry the true exit into the next boundary
                active = false;
            }
        }
    }
    if (walked) {
        atomicAdd(e.fix_segments, (unsigned long long)walked);
        atomicMax(e.fix_rounds, walked);
    }
}

// ------------------------------------------------------------------ split chain walk (MAGUS, k <= 8)
// The lockstep walk with its two recurrences in two warps: warp 0 of a 64-thread CTA steps the true
// states of 32 traces, warp 1 their speculative states, each with the one-chain stage block
// (MAGUS_WSTAGE1F_K<k>).  A walking warp is alone on its SM sub-partition and issues ~0.3 instructions
// per cycle, so halving the instructions each warp issues per tick nearly halves the walk.  The warps
// meet at a named barrier at every segment boundary and every 32-tick block end: warp 1 publishes its
// state and statistics in shared memory, warp 0 compares, adds the deltas and publishes the decisions.
// MAGUS_WALK_LOOKAHEAD: the split walk's stage block with both levels' decisions evaluated ahead of the level
// (MAGUS_WSTAGE1L_K<K>: a short loop-carried dependency for the latency-bound walk), else MAGUS_WSTAGE1F_K<K>
#ifndef MAGUS_WALK_LOOKAHEAD
#define MAGUS_WALK_LOOKAHEAD 0   // measured slower (cfg 3 fix-up 9.4 vs 6.6 ms, profiles/r02_walk_ab.txt)
#endif
template <int K>
__device__ __forceinline__ void walk_stage1(MagusState<K, false>& st, float& lock, float& nthr, uint32_t& wcmd,
                                            SegStats& ss, const float* d8, const DevPolicy& pol, float B_lo,
                                            double Blo_d) {
    uint32_t e0 = st.evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define W1_TAIL                                                                                                  \
    e0, st.cnt, ss.sexc, lock, nthr, wcmd, __float_as_uint(d8[0]), __float_as_uint(d8[1]), __float_as_uint(d8[2]), \
        __float_as_uint(d8[3]), __float_as_uint(d8[4]), __float_as_uint(d8[5]), __float_as_uint(d8[6]),             \
        __float_as_uint(d8[7]), B_lo, Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define R(i) st.ring.v[i]
#if MAGUS_WALK_LOOKAHEAD
    if constexpr (K == 1) MAGUS_WSTAGE1L_K1(st.f, R(0), W1_TAIL);
    else if constexpr (K == 2) MAGUS_WSTAGE1L_K2(st.f, R(0), R(1), W1_TAIL);
    else if constexpr (K == 3) MAGUS_WSTAGE1L_K3(st.f, R(0), R(1), R(2), W1_TAIL);
    else if constexpr (K == 4) MAGUS_WSTAGE1L_K4(st.f, R(0), R(1), R(2), R(3), W1_TAIL);
    else if constexpr (K == 5) MAGUS_WSTAGE1L_K5(st.f, R(0), R(1), R(2), R(3), R(4), W1_TAIL);
    else if constexpr (K == 6) MAGUS_WSTAGE1L_K6(st.f, R(0), R(1), R(2), R(3), R(4), R(5), W1_TAIL);
    else if constexpr (K == 7) MAGUS_WSTAGE1L_K7(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), W1_TAIL);
    else MAGUS_WSTAGE1L_K8(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), W1_TAIL);
#else
    if constexpr (K == 1) MAGUS_WSTAGE1F_K1(st.f, R(0), W1_TAIL);
    else if constexpr (K == 2) MAGUS_WSTAGE1F_K2(st.f, R(0), R(1), W1_TAIL);
    else if constexpr (K == 3) MAGUS_WSTAGE1F_K3(st.f, R(0), R(1), R(2), W1_TAIL);
    else if constexpr (K == 4) MAGUS_WSTAGE1F_K4(st.f, R(0), R(1), R(2), R(3), W1_TAIL);
    else if constexpr (K == 5) MAGUS_WSTAGE1F_K5(st.f, R(0), R(1), R(2), R(3), R(4), W1_TAIL);
    else if constexpr (K == 6) MAGUS_WSTAGE1F_K6(st.f, R(0), R(1), R(2), R(3), R(4), R(5), W1_TAIL);
    else if constexpr (K == 7) MAGUS_WSTAGE1F_K7(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), W1_TAIL);
    else MAGUS_WSTAGE1F_K8(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), W1_TAIL);
#endif
#undef R
#undef W1_TAIL
    st.evh = e0;
}

template <int K>
struct SplitXchg {   // what warp 1 (speculative) publishes for warp 0 (true), per lane
    uint32_t f, evh;
    double ring[K];
    SegStats ss;
    float lock, nthr;
    int32_t s0;
    uint32_t flags;   // from warp 0: bit 0 walking, bit 1 active
};

__device__ __forceinline__ void split_bar() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

template <int K>
__global__ void __launch_bounds__(64) magus_fix_split_kernel(const ReplayParams p, const EpiParams e,
                                                             const FixParams f, int q_base,
                                                             const float* __restrict__ trace) {
    ptx::pdl_wait();
    using T = MagusTicker<K, false>;
    __shared__ SplitXchg<K> x[32];
    const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * 32 + lane;
    const int q = q_base + blockIdx.y;
    const bool valid = j < p.n_traces;
    if (role == 0) {
        int s0 = 0x7FFFFFFF;
        if (valid) {
            const int64_t ci = (int64_t)q * p.n_traces + j;
            s0 = f.first_bad[ci];
            if (s0 < 0x7FFFFFFF) f.first_bad[ci] = 0x7FFFFFFF;   // reset for the next run
        }
        x[lane].s0 = s0;
    }
    split_bar();
    const int s0 = x[lane].s0;
    const int ws = __reduce_min_sync(0xffffffffu, s0);
    if (ws >= p.n_seg) return;   // uniform over both warps
    const DevPolicy pol = p.pol[q];
    const double Blo_d = (double)p.B_lo;
    const float* col = trace + (valid ? j : 0);
    MagusState<K, false> st;   // warp 0: true state, warp 1: speculative state
    bool walking = false;
    int walked = 0;
    for (int s = ws; s < p.n_seg; ++s) {
        const bool chk = !walking && valid && s >= s0 && !T::stored_equal(p, pol, q, 0, s, 1, s - 1, j);
        if (role == 1 && (walking || chk)) T::load(st, p, pol, 0, q, s, j);
        if (role == 0 && chk) T::load(st, p, pol, 1, q, s - 1, j);
        if (role == 1) {
            x[lane].f = st.f;
            x[lane].evh = st.evh;
#pragma unroll
            for (int r = 0; r < K; ++r) x[lane].ring[r] = st.ring.v[r];
        }
        split_bar();
        if (role == 0) {
            if (walking) {
                MagusState<K, false> o;
                o.f = x[lane].f;
                o.evh = x[lane].evh;
#pragma unroll
                for (int r = 0; r < K; ++r) o.ring.v[r] = x[lane].ring[r];
                walking = !T::equal(st, o, pol);
            } else if (chk) {
                walking = true;
            }
            x[lane].flags = walking ? 1u : 0u;
        }
        split_bar();
        if (role == 1) walking = (x[lane].flags & 1u) != 0u;
        if (!__any_sync(0xffffffffu, walking)) continue;   // the same answer in both warps
        walked += walking ? 1 : 0;
        const int seg_start = seg_begin(p, s), seg_end = seg_finish(p, s);
        SegStats ss;
        ss.zero();
        float lock = 0.f, nthr = 0.f;
        bool active = walking;
        float nxt[32];
        walk_load(nxt, col, seg_start, seg_end, p.trace_stride);
        for (int bt0 = seg_start; bt0 < seg_end; bt0 += 32) {
            if (!__any_sync(0xffffffffu, active)) break;   // the same answer in both warps
            const int n = min(32, seg_end - bt0);
            float dv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) dv[i] = nxt[i];
            if (bt0 + 32 < seg_end) walk_load(nxt, col, bt0 + 32, seg_end, p.trace_stride);
            const uint32_t fs = st.f;
            uint32_t wcmd = 0u;
            if (n == 32) {
#pragma unroll
                for (int g = 0; g < 4; ++g) walk_stage1<K>(st, lock, nthr, wcmd, ss, dv + 8 * g, pol, p.B_lo, Blo_d);
            } else {   // the ragged last block (static indices keep the samples in registers)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < n) lockstep_tick<T>(st, dv[i], pol, p, Blo_d, wcmd, ss);
            }
            const int64_t b = bt0 >> 5;
            uint32_t* wout = (role == 0 && active && p.words)
                                 ? p.words + (((int64_t)q * p.n_traces + j) * p.n_blocks + b) * 2
                                 : nullptr;
            fold_block(ss, wcmd, st.evh, fs, n, b, wout);
            if (role == 1) {
                x[lane].f = st.f;
                x[lane].evh = st.evh;
#pragma unroll
                for (int r = 0; r < K; ++r) x[lane].ring[r] = st.ring.v[r];
                x[lane].ss = ss;
                x[lane].lock = lock;
                x[lane].nthr = nthr;
            }
            split_bar();
            if (role == 0) {
                MagusState<K, false> o;
                o.f = x[lane].f;
                o.evh = x[lane].evh;
#pragma unroll
                for (int r = 0; r < K; ++r) o.ring.v[r] = x[lane].ring[r];
                const bool same = T::equal(st, o, pol);
                if (active && (same || bt0 + 32 >= seg_end)) {   // coalesced (the rest is right), or segment end
                    const SegStats& c = x[lane].ss;
                    add_to_chain(p, q, j, ss.nhi - c.nhi, ss.nthr - c.nthr + ((uint32_t)nthr - (uint32_t)x[lane].nthr),
                                 ss.trans - c.trans, ss.ev - c.ev,
                                 ss.lock - c.lock + ((uint32_t)lock - (uint32_t)x[lane].lock), ss.sexc - c.sexc,
                                 digest_pack(ss.dc - c.dc, ss.de - c.de));
                    walking = !same;   // carry the true exit into the next boundary
                    active = false;
                }
                x[lane].flags = (walking ? 1u : 0u) | (active ? 2u : 0u);
            }
            split_bar();
            if (role == 1) {
                walking = (x[lane].flags & 1u) != 0u;
                active = (x[lane].flags & 2u) != 0u;
            }
        }
    }
    if (walked && role == 0) {
        atomicAdd(e.fix_segments, (unsigned long long)walked);
        atomicMax(e.fix_rounds, walked);
    }
}

// ------------------------------------------------------------------ chain walk (default fix-up, exact)
// One thread per chain (q, j): scans the segment boundaries in order; at the first entry that differs
// from the previous exit it re-runs that segment from the true state next to the speculative one
// (rerun_segment: until they coalesce at a block end, else to the segment end), and carries the true
// state on across later boundaries until it agrees with a stored entry again.  Every chain is thus
// fixed in one pass, in time order, whatever the number of consecutive wrong guesses (phase-ambiguous
// limit cycles of oscillating traces make a wrong guess persist: DESIGN.md section 9).  T: the chain
// kind of the launch group (register ring for k in {1, 2, 4, 8}).
template <class T>
__global__ void __launch_bounds__(128) magus_fix_walk_kernel(const ReplayParams p, const EpiParams e, const FixParams f,
                                                             int q_base, const float* __restrict__ trace) {
    ptx::pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = q_base + blockIdx.y;
    if (j >= p.n_traces) return;
    const int s0 = f.first_bad[(int64_t)q * p.n_traces + j];   // first wrong entry (magus_fix_mark_kernel)
    if (s0 >= p.n_seg) return;
    f.first_bad[(int64_t)q * p.n_traces + j] = 0x7FFFFFFF;       // reset for the next run
    const DevPolicy pol = p.pol[q];
    typename T::State tru, spec;
    bool carry = false;   // tru holds the true exit of segment s - 1, which the stored one is not
    int walked = 0;
    for (int s = s0; s < p.n_seg; ++s) {
        if (!carry) {
            if (T::stored_equal(p, pol, q, 0, s, 1, s - 1, j)) continue;
            T::load(tru, p, pol, 1, q, s - 1, j);
        }
        T::load(spec, p, pol, 0, q, s, j);
        if (carry && T::equal(tru, spec, pol)) {
            carry = false;
            continue;
        }
        ++walked;
        carry = !WalkRerun<T>::run(p, pol, q, s, j, trace, tru, spec);
    }
    if (walked) {
        atomicAdd(e.fix_segments, (unsigned long long)walked);
        atomicMax(e.fix_rounds, walked);
    }
}

// ================================================================================= totals
// One thread per (trace, policy): the chain's totals -> the closed-form record (section 8), STATIC_MAX
// records from their closed form (at f_max A = D <= bw_max: never throttled, never a transition or a
// tune flag, digest of an all-f_max command stream, A17 / A21); then fixed-order per-policy sums.
#ifndef MAGUS_TOT_THREADS
#define MAGUS_TOT_THREADS 256
#endif
constexpr int kTotThreads = MAGUS_TOT_THREADS;   // = traces per chunk
constexpr int kNTot = 13;              // MAGUS_N_TOTALS

// Block (p, c): the closed-form records of policy p for traces [256 c, 256 c + 256), one per thread (written
// out only when requested), then their fixed-order sum: an xor-shuffle tree per warp, the 8 warp partials
// in order -> part[p][c][0..11], part[p][c][12] = the chunk's trace count.  The host (or, across ranks,
// the allreduce and then the host) adds the chunks in order.  Reading a chain's totals zeroes them for
// the next run; a sample above bw_max (or invalid) raises the run's flag (A17).
__global__ void __launch_bounds__(kTotThreads) magus_totals_kernel(const ReplayParams rp, const EpiParams e,
                                                                    const int* __restrict__ lane_of_policy,
                                                                    int validate_lane, uint64_t digest_all_hi,
                                                                    int write_rec, const TraceRec* __restrict__ wrec,
                                                                    double* __restrict__ part) {
    ptx::pdl_wait();
    const int n_traces = rp.n_traces, n_policies = e.n_policies;
    const int p = blockIdx.x, c = blockIdx.y;
    const int q = lane_of_policy[p];
    const int j = c * kTotThreads + threadIdx.x;
    double acc[kNTot - 1];
#pragma unroll
    for (int f = 0; f < kNTot - 1; ++f) acc[f] = 0.0;
    bool invalid = false;
    if (j < n_traces) {
        TraceRec r;
        if (q < 0) {   // STATIC_MAX: never throttled, no transition or tune flag (A17, A21)
            finish_record(r, e, (double)e.w[j], (int64_t)e.n_samples, 0, 0, 0, 0, 0.0, digest_all_hi);
        } else if (wrec) {   // wall-clock rounds (A32): the chain's record as the wall-clock kernel wrote it
            const int64_t ci = chain_idx(rp, q, j);
            r = wrec[ci];
            invalid |= rp.c_vmax[ci] > rp.bwbits;
            zero_chain(rp, ci);
        } else {
            const int64_t ci = chain_idx(rp, q, j);
            finish_record(r, e, (double)e.w[j], (int64_t)rp.c_nhi[ci], (int64_t)rp.c_nthr[ci], (int64_t)rp.c_trans[ci],
                          (int64_t)rp.c_ev[ci], (int64_t)rp.c_lock[ci], rp.c_sexc[ci], (uint64_t)rp.c_digest[ci]);
            invalid |= rp.c_vmax[ci] > rp.bwbits;
            zero_chain(rp, ci);   // every chain is read exactly once per run: leave it zeroed for the next
        }
        if (p == 0 && validate_lane >= 0) {
            const int64_t ci = chain_idx(rp, validate_lane, j);
            invalid |= rp.c_vmax[ci] > rp.bwbits;
            zero_chain(rp, ci);
        }
        if (write_rec) e.rec[(int64_t)j * n_policies + p] = r;
        acc[0] = r.E;
        acc[1] = r.E_pkg;
        acc[2] = r.T;
        acc[3] = r.EDP;
        acc[4] = r.slowdown;
        acc[5] = r.energy_saving;
        acc[6] = r.edp_saving;
        acc[7] = (double)r.n_hi;
        acc[8] = (double)r.n_thr;
        acc[9] = (double)r.transitions;
        acc[10] = (double)r.tune_events;
        acc[11] = (double)r.lock_ticks;
    }
    if (__any_sync(0xffffffffu, invalid) && (threadIdx.x & 31) == 0) atomicOr(e.flag_invalid, 1u);
#pragma unroll
    for (int f = 0; f < kNTot - 1; ++f)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o);
    __shared__ double wp[kTotThreads / 32][kNTot - 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int f = 0; f < kNTot - 1; ++f) wp[warp][f] = acc[f];
    __syncthreads();
    double* out = part + ((int64_t)p * gridDim.y + c) * kNTot;
    if (threadIdx.x < kNTot - 1) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kTotThreads / 32; ++w) sum += wp[w][threadIdx.x];
        out[threadIdx.x] = sum;
    } else if (threadIdx.x == kNTot - 1) {
        out[kNTot - 1] = (double)max(0, min(kTotThreads, n_traces - c * kTotThreads));
    }
}

// world > 1: the chunk partials of policy p added in chunk order -> fin[p][0..12] (the same size on every
// rank, whatever its trace count, so the allreduce that follows is well formed).
__global__ void magus_chunk_sum_kernel(const double* __restrict__ part, int n_chunks, double* __restrict__ fin) {
    ptx::pdl_wait();
    const int p = blockIdx.x, f = threadIdx.x;
    if (f >= kNTot) return;
    double sum = 0.0;
    for (int c = 0; c < n_chunks; ++c) sum += part[((int64_t)p * n_chunks + c) * kNTot + f];
    fin[p * kNTot + f] = sum;
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
        if (pol.C <= kMaxC32) MAGUS_RESIM(MagusTicker<0, false>);
        else MAGUS_RESIM(MagusTicker<0, true>);
    } else if (pol.kind == LANE_TDP) {
        MAGUS_RESIM(TdpTicker);
    } else {
        MAGUS_RESIM(StaticMinTicker<false>);
    }
#undef MAGUS_RESIM
}

// Per-tick codes (DESIGN A27) for traces [first, first + n) of every lane policy, DECODED from the replay kernels' own
// 32-tick words (p.words: written by the replay kernel for every counted block and rewritten by the fix-up walk for
// the blocks it re-ran): the cmd and tune-flag bits are the hot kernel's; the rest follows from them and the
// samples without re-running the recurrence -- level in effect = the previous tick's cmd (f0 at t = 0); A = min(D,
// B[level]) and throttled = D > B[level] (A14); ready = t >= k (A7); signal = Alg. 1's comparison of the fp64
// difference A_t - A_{t-k} with the host thresholds; lock = Alg. 2 on the last C logged flags once the log
// is full (A8).  codes: [n_samples][n][P].  One thread per (trace, lane policy); k <= 64 (fp32 ring of A).
__global__ void magus_decode_kernel(const ReplayParams p, const float* __restrict__ trace, int first, int n_win, int P,
                                    uint8_t* codes) {
    const int jd = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = blockIdx.y;
    if (jd >= n_win) return;
    const DevPolicy pol = p.pol[q];
    if (pol.policy_index < 0) return;
    const int j = first + jd;
    const uint32_t* wq = p.words + ((int64_t)q * p.n_traces + j) * p.n_blocks * 2;
    const bool magus = pol.kind == LANE_MAGUS;
    const int k = pol.k, C = pol.C;
    float ring[KMAX_GENERIC];   // A_{t-k} .. A_{t-1}, circular by t % k
    uint64_t log = 0;
    uint32_t lvl = (uint32_t)pol.f0;
    for (int b = 0; b < p.n_blocks; ++b) {
        const uint32_t wc = wq[2 * b], we = wq[2 * b + 1];
        const int n = min(32, p.n_samples - 32 * b);
        for (int i = 0; i < n; ++i) {
            const int t = 32 * b + i;
            const uint32_t cmd = (wc >> (31 - i)) & 1u, ev = (we >> (31 - i)) & 1u;
            const float D = trace[(int64_t)t * p.trace_stride + j];
            const float B = lvl ? p.B_hi : p.B_lo;
            const float A = fminf(D, B);
            const uint32_t thr = D > B ? 1u : 0u;
            uint32_t c = cmd | (ev << 2) | (thr << 6) | (lvl << 7);
            if (magus) {
                const bool ready = t >= k;
                if (ready) {
                    const double d = (double)A - (double)ring[t % k];
                    c |= 2u | ((d > pol.dinc ? 1u : (d < pol.ddec ? 2u : 0u)) << 4);
                }
                ring[t % k] = A;
                log = (log << 1) | ev;
                const uint64_t w = log & pol.logmask;
                if (t >= k + C - 1 && (uint32_t)__popcll(w) >= (uint32_t)pol.s_min) c |= 8u;
            }
            codes[((int64_t)t * n_win + jd) * P + pol.policy_index] = (uint8_t)c;
            lvl = cmd;
        }
    }
}

__global__ void magus_fill_codes_kernel(uint8_t* codes, int64_t n_rows, int P, int pi, uint8_t value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_rows) codes[i * P + pi] = value;
}

// Start of every run.  Block 0 zeroes the run's flag and worklist words (no memset nodes).  With
// first_low != nullptr (segmented runs), the speculation aid: first_low[j] /
// first_low[n + j] = the first subsampled tick (stride `sub`) with D <= B_lo / D > B_lo, or INT_MAX.
// Block = 32 traces x 32 row slices; each thread scans its slice in increasing t, the slices are
// reduced in shared memory.  Pure performance hint: a wrong guess only costs a re-run.
#ifndef MAGUS_PREPASS_TRACES
#define MAGUS_PREPASS_TRACES 32
#endif
constexpr int kPrepassTraces = MAGUS_PREPASS_TRACES, kPrepassSlices = 1024 / MAGUS_PREPASS_TRACES;
__global__ void __launch_bounds__(kPrepassTraces * kPrepassSlices)
    magus_prepass_kernel(const float* __restrict__ trace, int n_traces, int n_samples, int64_t stride, float B_lo,
                         int sub, int* __restrict__ first_low, uint32_t* __restrict__ zero_a, int n_zero_a) {
    ptx::pdl_trigger();   // the replay kernel may start its pipeline fill; it waits before reading first_low
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < n_zero_a; i += blockDim.x) zero_a[i] = 0u;
    }
    if (first_low == nullptr) return;
    const int tx = threadIdx.x % kPrepassTraces, ty = threadIdx.x / kPrepassTraces;
    const int j = blockIdx.x * kPrepassTraces + tx;
    int lo = 0x7FFFFFFF, hi = 0x7FFFFFFF;
    if (j < n_traces) {
        const int n_sub = (n_samples + sub - 1) / sub;
        constexpr int kBatch = 16;   // loads in flight per thread: one batch covers 16 * 32 * sub ticks
        for (int i0 = ty; i0 < n_sub; i0 += kBatch * kPrepassSlices) {
            float d[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int i = i0 + u * kPrepassSlices;
                d[u] = i < n_sub ? __ldg(trace + (int64_t)i * sub * stride + j) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int i = i0 + u * kPrepassSlices;
                if (i < n_sub) {
                    if (lo == 0x7FFFFFFF && d[u] <= B_lo) lo = i * sub;
                    if (hi == 0x7FFFFFFF && d[u] > B_lo) hi = i * sub;
                }
            }
            if (lo != 0x7FFFFFFF && hi != 0x7FFFFFFF) break;
        }
    }
    __shared__ int s_lo[kPrepassSlices][kPrepassTraces], s_hi[kPrepassSlices][kPrepassTraces];
    s_lo[ty][tx] = lo;
    s_hi[ty][tx] = hi;
    __syncthreads();
    if (ty == 0 && j < n_traces) {
        for (int y = 1; y < kPrepassSlices; ++y) {
            lo = min(lo, s_lo[y][tx]);
            hi = min(hi, s_hi[y][tx]);
        }
        first_low[j] = lo;
        first_low[n_traces + j] = hi;
    }
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
