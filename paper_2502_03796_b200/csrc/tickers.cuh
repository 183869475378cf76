// tickers.cuh -- per-policy-kind chain adapters used by the replay, fix-up and re-simulation
// kernels: initial / speculative state, one tick, state save / load / compare.
#pragma once
#include "device_common.cuh"

namespace magus {

// ----------------------------------------------------------------------------------- MAGUS
template <int K, bool LOG64>
struct MagusTicker {
    using State = MagusState<K, LOG64>;
    using LogT = typename LogWord<LOG64>::T;
    static constexpr bool kStateful = true;
    static constexpr bool kWarmupRules = true;   // Alg. 1 needs k+1 samples, Alg. 2 a full log

    __device__ __forceinline__ static void init(State& s, const DevPolicy& pol, bool exact_start) {
        s.f = exact_start ? (uint32_t)pol.f0 : (uint32_t)pol.guess_f;
        s.evh = 0;
        s.ring.clear(pol.k);
    }
    template <bool SLOW>
    __device__ __forceinline__ static TickOut tick(State& s, float D, const DevPolicy& pol, float B_lo, float B_hi,
                                                   bool ready, bool full) {
        return magus_tick<K, LOG64, SLOW>(s, D, pol, B_lo, B_hi, ready, full);
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
        s.ring.set_all(p.st_ring + ring_idx(p, e, q, seg, 0, j), pol.k, (int64_t)p.n_traces);
    }
    // exact equality of the two stored states (e0, s0) and (e1, s1): level, log bits, ring values
    __device__ __forceinline__ static bool stored_equal(const ReplayParams& p, const DevPolicy& pol, int q, int e0,
                                                        int s0, int e1, int s1, int j) {
        const int64_t a = st_idx(p, e0, q, s0, j), b = st_idx(p, e1, q, s1, j);
        if (p.st_f[a] != p.st_f[b] || p.st_log[a] != p.st_log[b]) return false;
        for (int r = 0; r < pol.k; ++r)
            if (__float_as_uint(p.st_ring[ring_idx(p, e0, q, s0, r, j)]) !=
                __float_as_uint(p.st_ring[ring_idx(p, e1, q, s1, r, j)]))
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
        return p.st_f[st_idx(p, e0, q, s0, j)] == p.st_f[st_idx(p, e1, q, s1, j)];
    }
    __device__ __forceinline__ static bool equal(const State& x, const State& y, const DevPolicy&) { return x.f == y.f; }
};

// --------------------------------------------------------------- STATIC_MIN (and validate-only)
// No state: the level is f_min every tick; only throttling statistics depend on the data.
template <bool VALIDATE_ONLY>
struct StaticMinTicker {
    struct State { uint32_t f; };
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
