// tickers.cuh -- per-policy-kind chain adapters used by the replay, fix-up and re-simulation
// kernels: initial / speculative state, one tick, state save / load / compare.
#pragma once
#include "device_common.cuh"
#include "tick4_asm.cuh"

namespace magus {

// ----------------------------------------------------------------------------------- MAGUS
template <int K, bool LOG64>
struct MagusTicker {
    using State = MagusState<K, LOG64>;
    using LogT = typename LogWord<LOG64>::T;
    static constexpr bool kStateful = true;
    static constexpr bool kWarmupRules = true;   // Alg. 1 needs k+1 samples, Alg. 2 a full log
    static constexpr int kRingK = K;

    __device__ __forceinline__ static void init(State& s, const DevPolicy& pol, bool exact_start) {
        s.f = exact_start ? (uint32_t)pol.f0 : (uint32_t)pol.guess_f;
        s.evh = 0;
        s.cnt = 0;
        s.ring.clear(pol.k);
    }
    template <bool SLOW>
    __device__ __forceinline__ static TickOut tick(State& s, float D, const DevPolicy& pol, float B_lo, float B_hi,
                                                   bool ready, bool full) {
        return magus_tick<K, LOG64, SLOW>(s, D, pol, B_lo, B_hi, ready, full);
    }
    static constexpr bool kHasFast = true;
    static constexpr bool kHasFast4 = !LOG64;
    __device__ __forceinline__ static uint32_t window_count(const State& s, const DevPolicy& pol) {
        return popc_log<LOG64>(s.evh & (LogT)pol.logmask);
    }
    // The 4 chains of a lane in one interleaved PTX block (tick4_asm.cuh, generated).
    __device__ __forceinline__ static void fast4(State* s, const float* D, const DevPolicy& pol, float B_lo,
                                                 double Blo_d, uint32_t* wcmd, SegStats* ss, uint32_t& vmax) {
        if constexpr (!LOG64) {
            double ad0, ad1, ad2, ad3;
            uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
            const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
            MAGUS_TICK4_ASM(s[0].f, s[1].f, s[2].f, s[3].f, ad0, ad1, ad2, ad3, e0, e1, e2, e3, ss[0].sexc, ss[1].sexc,
                            ss[2].sexc, ss[3].sexc, ss[0].lock, ss[1].lock, ss[2].lock, ss[3].lock, ss[0].nthr,
                            ss[1].nthr, ss[2].nthr, ss[3].nthr, wcmd[0], wcmd[1], wcmd[2], wcmd[3], s[0].cnt, s[1].cnt,
                            s[2].cnt, s[3].cnt, vmax, D[0], D[1], D[2], D[3], s[0].ring.oldest(pol.k),
                            s[1].ring.oldest(pol.k), s[2].ring.oldest(pol.k), s[3].ring.oldest(pol.k),
                            __float_as_uint(D[0]), __float_as_uint(D[1]), __float_as_uint(D[2]), __float_as_uint(D[3]),
                            B_lo, Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone);
            s[0].evh = e0;
            s[1].evh = e1;
            s[2].evh = e2;
            s[3].evh = e3;
            s[0].ring.push(ad0, pol.k);
            s[1].ring.push(ad1, pol.k);
            s[2].ring.push(ad2, pol.k);
            s[3].ring.push(ad3, pol.k);
        }
    }
    // Warm-up ticks of the 4 chains (Alg. 1 once `ready`, Alg. 2 once `full`), same interleaved block.
    __device__ __forceinline__ static void warm4(State* s, const float* D, const DevPolicy& pol, float B_lo,
                                                 double Blo_d, uint32_t* wcmd, SegStats* ss, uint32_t& vmax,
                                                 uint32_t ready, uint32_t full) {
        if constexpr (!LOG64) {
            double ad0, ad1, ad2, ad3;
            uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
            const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
            MAGUS_TICK4W_ASM(s[0].f, s[1].f, s[2].f, s[3].f, ad0, ad1, ad2, ad3, e0, e1, e2, e3, ss[0].sexc,
                             ss[1].sexc, ss[2].sexc, ss[3].sexc, ss[0].lock, ss[1].lock, ss[2].lock, ss[3].lock,
                             ss[0].nthr, ss[1].nthr, ss[2].nthr, ss[3].nthr, wcmd[0], wcmd[1], wcmd[2], wcmd[3],
                             s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, vmax, D[0], D[1], D[2], D[3],
                             s[0].ring.oldest(pol.k), s[1].ring.oldest(pol.k), s[2].ring.oldest(pol.k),
                             s[3].ring.oldest(pol.k), __float_as_uint(D[0]), __float_as_uint(D[1]),
                             __float_as_uint(D[2]), __float_as_uint(D[3]), B_lo, Blo_d, pol.dinc, pol.ddec, bitc,
                             pol.smin_sc, pol.one, mone, ready, full);
            s[0].evh = e0;
            s[1].evh = e1;
            s[2].evh = e2;
            s[3].evh = e3;
            s[0].ring.push(ad0, pol.k);
            s[1].ring.push(ad1, pol.k);
            s[2].ring.push(ad2, pol.k);
            s[3].ring.push(ad3, pol.k);
        }
    }
    // One whole steady-state stage (8 ticks x 4 chains, the tile loads included) in one generated PTX
    // block (MAGUS_STAGE8_K<K>, tick4_asm.cuh); `tile` = this lane's float4 column of the stage's tile.
    static constexpr bool kHasStage8 = !LOG64 && K >= 1 && K <= 3;
    __device__ __forceinline__ static void stage8(State* s, uint32_t tile, const DevPolicy& pol, float B_lo,
                                                  double Blo_d, uint32_t* wcmd, SegStats* ss, uint32_t& vmax) {
        if constexpr (kHasStage8) {
            uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
            const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define MAGUS_STAGE_TAIL                                                                                        \
    e0, e1, e2, e3, ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, ss[0].lock, ss[1].lock, ss[2].lock, ss[3].lock, \
        ss[0].nthr, ss[1].nthr, ss[2].nthr, ss[3].nthr, wcmd[0], wcmd[1], wcmd[2], wcmd[3], s[0].cnt, s[1].cnt,     \
        s[2].cnt, s[3].cnt, vmax, tile, B_lo, Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
            if constexpr (K == 1) {
                MAGUS_STAGE8_K1(s[0].f, s[1].f, s[2].f, s[3].f, s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0],
                                s[3].ring.v[0], MAGUS_STAGE_TAIL);
            } else if constexpr (K == 2) {
                MAGUS_STAGE8_K2(s[0].f, s[1].f, s[2].f, s[3].f, s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0],
                                s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], s[3].ring.v[1],
                                MAGUS_STAGE_TAIL);
            } else {
                MAGUS_STAGE8_K3(s[0].f, s[1].f, s[2].f, s[3].f, s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2],
                                s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], s[2].ring.v[1],
                                s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2], MAGUS_STAGE_TAIL);
            }
#undef MAGUS_STAGE_TAIL
            s[0].evh = e0;
            s[1].evh = e1;
            s[2].evh = e2;
            s[3].evh = e3;
        }
    }
    // One steady-state tick of one chain (the 64-bit-log kinds; the 32-bit kinds use fast4).
    __device__ __forceinline__ static void fast(State& s, float D, const DevPolicy& pol, float B_lo, double Blo_d,
                                                uint32_t& wcmd, SegStats& ss, uint32_t& vmax) {
        const double old = s.ring.oldest(pol.k);
        const uint32_t f = s.f;
        const bool lo = f == 0u;
        const bool thr = lo && (D > B_lo);
        const double Dd = (double)D;
        const double Ad = thr ? Blo_d : Dd;
        const double d = Ad - old;
        ss.sexc += Dd - Ad;
        const bool inc = d > pol.dinc;
        const bool ev = inc || (d < pol.ddec);
        s.evh = (s.evh << 1) | (LogT)(ev ? 1u : 0u);
        const uint32_t cnt = popc_log<LOG64>(s.evh & (LogT)pol.logmask);
        const bool hf = cnt >= (uint32_t)pol.s_min;
        s.f = (hf || inc || (!lo && !ev)) ? 1u : 0u;
        wcmd = (wcmd << 1) | s.f;
        ss.lock += hf ? 1u : 0u;
        ss.nthr += thr ? 1u : 0u;
        vmax = max(vmax, __float_as_uint(D));
        s.ring.push(Ad, pol.k);
    }
    __device__ __forceinline__ static uint32_t level(const State& s) { return s.f; }
    __device__ __forceinline__ static void set_level(State& s, uint32_t f) { s.f = f; }
    __device__ __forceinline__ static void save(const State& s, const ReplayParams& p, const DevPolicy& pol, int e,
                                                int q, int seg, int j) {
        const int64_t i = st_idx(p, e, q, seg, j);
        p.st_f[i] = (uint8_t)s.f;
        p.st_log[i] = (uint64_t)s.evh & pol.logmask;
        s.ring.store_all(p.st_ring + ring_idx(p, e, q, seg, 0, j), pol.k, (int64_t)p.n_traces);
    }
    __device__ __forceinline__ static void load(State& s, const ReplayParams& p, const DevPolicy& pol, int e, int q,
                                                int seg, int j) {
        const int64_t i = st_idx(p, e, q, seg, j);
        s.f = p.st_f[i];
        s.evh = (LogT)p.st_log[i];
        if constexpr (!LOG64) s.cnt = popc_log<LOG64>(s.evh & (LogT)pol.logmask) << (pol.C - 1);
        s.ring.set_all(p.st_ring + ring_idx(p, e, q, seg, 0, j), pol.k, (int64_t)p.n_traces);
    }
    // exact equality of the two stored states (e0, s0) and (e1, s1): level, log bits, ring values.
    // L2-coherent loads (__ldcg): the replay kernel compares states written by other SMs in the same launch.
    __device__ __forceinline__ static bool stored_equal(const ReplayParams& p, const DevPolicy& pol, int q, int e0,
                                                        int s0, int e1, int s1, int j) {
        const int64_t a = st_idx(p, e0, q, s0, j), b = st_idx(p, e1, q, s1, j);
        if (__ldcg(p.st_f + a) != __ldcg(p.st_f + b) || __ldcg(p.st_log + a) != __ldcg(p.st_log + b)) return false;
        for (int r = 0; r < pol.k; ++r)
            if (__float_as_uint(__ldcg(p.st_ring + ring_idx(p, e0, q, s0, r, j))) !=
                __float_as_uint(__ldcg(p.st_ring + ring_idx(p, e1, q, s1, r, j))))
                return false;
        return true;
    }
    __device__ __forceinline__ static bool equal(const State& x, const State& y, const DevPolicy& pol) {
        if (x.f != y.f || (((uint64_t)(x.evh ^ y.evh)) & pol.logmask)) return false;
        return x.ring.same(y.ring, pol.k);
    }
};

// ----------------------------------------------------------------------------------- TDP default
struct TdpTicker {
    struct State { uint32_t f; };
    static constexpr bool kHasFast = true;
    static constexpr bool kHasFast4 = false;
    __device__ __forceinline__ static uint32_t window_count(const State&, const DevPolicy&) { return 0; }
    // tdp_tick + acc_tick of one tick, branch-free: A = min(D, B[f]); throttled iff D > B[f];
    // next level f_min iff A >= a*[f] (the fp32 threshold equivalent of the power predicate, A24)
    __device__ __forceinline__ static void fast(State& s, float D, const DevPolicy& pol, float B_lo, double Blo_d,
                                                uint32_t& wcmd, SegStats& ss, uint32_t& vmax) {
        const bool hi = s.f != 0u;
        const float B = hi ? pol.B_hi : B_lo;
        const bool thr = D > B;
        const float A = fminf(D, B);
        const uint32_t f = (A >= (hi ? pol.astar_hi : pol.astar_lo)) ? 0u : 1u;
        ss.nthr += thr ? 1u : 0u;
        ss.sexc += thr ? (double)D - Blo_d : 0.0;
        vmax = max(vmax, __float_as_uint(D));
        wcmd = (wcmd << 1) | f;
        s.f = f;
    }
    __device__ __forceinline__ static void fast4(State*, const float*, const DevPolicy&, float, double, uint32_t*,
                                                 SegStats*, uint32_t&) {}
    __device__ __forceinline__ static void warm4(State*, const float*, const DevPolicy&, float, double, uint32_t*,
                                                 SegStats*, uint32_t&, uint32_t, uint32_t) {}
    static constexpr bool kStateful = true;
    static constexpr bool kWarmupRules = false;
    __device__ __forceinline__ static void init(State& s, const DevPolicy& pol, bool exact_start) {
        s.f = exact_start ? (uint32_t)pol.f0 : (uint32_t)pol.guess_f;
    }
    template <bool SLOW>
    __device__ __forceinline__ static TickOut tick(State& s, float D, const DevPolicy& pol, float B_lo, float B_hi,
                                                   bool, bool) {
        return tdp_tick(s.f, D, pol, B_lo, B_hi);
    }
    __device__ __forceinline__ static uint32_t level(const State& s) { return s.f; }
    __device__ __forceinline__ static void set_level(State& s, uint32_t f) { s.f = f; }
    __device__ __forceinline__ static void save(const State& s, const ReplayParams& p, const DevPolicy&, int e, int q,
                                                int seg, int j) {
        const int64_t i = st_idx(p, e, q, seg, j);
        p.st_f[i] = (uint8_t)s.f;
        p.st_log[i] = 0;
    }
    __device__ __forceinline__ static void load(State& s, const ReplayParams& p, const DevPolicy&, int e, int q, int seg,
                                                int j) {
        s.f = p.st_f[st_idx(p, e, q, seg, j)];
    }
    __device__ __forceinline__ static bool stored_equal(const ReplayParams& p, const DevPolicy&, int q, int e0, int s0,
                                                        int e1, int s1, int j) {
        return __ldcg(p.st_f + st_idx(p, e0, q, s0, j)) == __ldcg(p.st_f + st_idx(p, e1, q, s1, j));
    }
    __device__ __forceinline__ static bool equal(const State& x, const State& y, const DevPolicy&) { return x.f == y.f; }
};

// --------------------------------------------------------------- STATIC_MIN (and validate-only)
// No state: the level is f_min every tick; only throttling statistics depend on the data.
template <bool VALIDATE_ONLY>
struct StaticMinTicker {
    struct State { uint32_t f; };
    static constexpr bool kHasFast = false;
    static constexpr bool kHasFast4 = false;
    __device__ __forceinline__ static uint32_t window_count(const State&, const DevPolicy&) { return 0; }
    __device__ __forceinline__ static void fast(State&, float, const DevPolicy&, float, double, uint32_t&, SegStats&,
                                                uint32_t&) {}
    __device__ __forceinline__ static void fast4(State*, const float*, const DevPolicy&, float, double, uint32_t*,
                                                 SegStats*, uint32_t&) {}
    __device__ __forceinline__ static void warm4(State*, const float*, const DevPolicy&, float, double, uint32_t*,
                                                 SegStats*, uint32_t&, uint32_t, uint32_t) {}
    static constexpr bool kStateful = false;
    static constexpr bool kWarmupRules = false;
    __device__ __forceinline__ static void init(State& s, const DevPolicy&, bool) { s.f = 0; }
    template <bool SLOW>
    __device__ __forceinline__ static TickOut tick(State& s, float D, const DevPolicy&, float B_lo, float, bool, bool) {
        TickOut o;
        o.thr = VALIDATE_ONLY ? 0u : (D > B_lo ? 1u : 0u);
        o.cmd = 0;
        o.ev = 0;
        o.hf = 0;
        o.sig = 0;
        return o;
    }
    __device__ __forceinline__ static uint32_t level(const State&) { return 0; }
    __device__ __forceinline__ static void set_level(State&, uint32_t) {}
    __device__ __forceinline__ static void save(const State&, const ReplayParams& p, const DevPolicy&, int e, int q,
                                                int seg, int j) {
        const int64_t i = st_idx(p, e, q, seg, j);
        p.st_f[i] = 0;
        p.st_log[i] = 0;
    }
    __device__ __forceinline__ static void load(State& s, const ReplayParams&, const DevPolicy&, int, int, int, int) {
        s.f = 0;
    }
    __device__ __forceinline__ static bool stored_equal(const ReplayParams&, const DevPolicy&, int, int, int, int, int,
                                                        int) {
        return true;
    }
    __device__ __forceinline__ static bool equal(const State&, const State&, const DevPolicy&) { return true; }
};

}  // namespace magus
