// device_common.cuh -- the per-tick MAGUS recurrence as device code, shared by the replay kernel
// (4 chains per lane, unrolled) and the fix-up / re-simulation kernels (scalar).
//
// One chain = one (trace, policy) recurrence.  Per tick (Alg. 1
// P:197-222, Alg. 2, S3.2 P:243, S6.1 P:318):
//   A = min(D, B[f]); thr = A < D                                          (DESIGN A14)
//   d = (double)A - (double)A_{t-k};   +1 iff d > d*_inc, -1 iff d < d*_dec  (Alg. 1, exact-equivalent
//                                       thresholds derived on the host from fl(d / (k*Delta)), section 8)
//   tune flag = signal != 0 pushed into a C-bit shift register               (A7, A12)
//   lock = log full && popcount(log) >= s_min                                (Alg. 2, s_min from fl(s/C), A8)
//   cmd = lock ? HI : +1 ? HI : -1 ? LO : f                                   (A9)
// The hot loop keeps only sufficient statistics for the energy model (section 8): ticks at HI,
// throttled ticks, the fp64 sum of throttled demand, transitions, tune flags, lock ticks and the
// 64-bit decision digest (section 5).
#pragma once
#include <cstdint>

namespace magus {

enum : int32_t { LANE_MAGUS = 0, LANE_STATIC_MIN = 2, LANE_TDP = 3, LANE_VALIDATE = 4 };
enum : int32_t { KMAX_GENERIC = 64 };

// one policy as the kernels see it (host-derived, section 8)
struct DevPolicy {
    int32_t kind;          // LANE_*
    int32_t k;             // derivative window in ticks
    int32_t C;             // tune-log capacity
    int32_t s_min;         // Alg. 2: lock iff popcount >= s_min (C+1 = never)
    uint64_t logmask;      // low C bits
    double dinc, ddec;     // Alg. 1: +1 iff d > dinc, -1 iff d < ddec
    float astar_lo, astar_hi;   // TDP: cmd = LO iff A >= astar[f]
    int32_t f0;            // initial level at t = 0 (A10)
    int32_t guess_f;       // level guessed at a speculative segment start
    int32_t policy_index;  // index in the user's policy array
    uint32_t one;          // the constant 1, as data (keeps predicated increments on the FMA pipe)
    int32_t sticky;        // k >= s_min: every edge locks Alg. 2, and after a lock Hold keeps f_max
    float B_hi;            // B[f_max] (copy of the run constant, for the TDP fast tick)
    uint32_t smin_sc;      // 32-bit-log kinds: s_min << (C-1), the lock threshold on the scaled window count
};

// Debug-check build (MAGUS_DEBUG_CHECKS=1, the library libmagus_replay_debug.so built next to the release one):
// every state / ring / chain index and every shared-memory tile or scratch access of the replay kernels is checked
// against its allocation, and a violation traps the kernel (cudaErrorLaunchFailure), so a GPU test running the
// debug build over every kernel family stands in for compute-sanitizer's memcheck where that tool is unavailable.
#ifndef MAGUS_DEBUG_CHECKS
#define MAGUS_DEBUG_CHECKS 0
#endif
#if MAGUS_DEBUG_CHECKS
#ifdef __CUDA_ARCH__
#define MAGUS_CHECK(cond)    \
    do {                     \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define MAGUS_CHECK(cond) ((void)0)
#endif
#else
#define MAGUS_CHECK(cond) ((void)0)
#endif
// a shared-memory byte range [addr, addr + bytes) lies inside the CTA's dynamic shared memory
__device__ __forceinline__ bool smem_range_ok(uint32_t addr, uint32_t bytes) {
    uint32_t size;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
    extern __shared__ __align__(16) uint8_t magus_dyn_smem_probe[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(magus_dyn_smem_probe);
    return addr >= base && addr + bytes <= base + size;
}

// run-wide constants and scratch pointers
struct ReplayParams {
    int32_t n_traces, n_samples;
    int32_t n_lane;        // Q lane policies (state / statistics arrays are indexed by lane 0..Q-1)
    int32_t q_base, nq;    // lanes covered by the current replay launch (all of one chain kind)
    int32_t q_base2, nq2;  // magus_replay_combo_kernel: the TDP group replayed next to the MAGUS group q_base / nq
    int32_t n_seg, seg_len, warmup;
    int32_t seg_long;      // the first seg_long segments are seg_len + 32 ticks long (CTA balance), the rest seg_len
    int32_t n_groups;      // ceil(n_traces / 128)
    int32_t ng, npw;       // CTA: ng tile groups x npw policy warps (+1 producer warp)
    int32_t n_tblocks, n_pblocks;
    int32_t kr;            // ring floats stored per chain state (max k over MAGUS lane policies)
    int32_t n_blocks;      // ceil(n_samples / 32)
    float B_lo, B_hi;
    uint32_t bwbits;       // bit pattern of the largest fp32 <= bw_max
    uint32_t solo_flags;   // solo replay kernel: bit 0 = speculative segments start from a synthetic full state
    int32_t solo_warm;     // warm-up ticks of the unified-stage solo kernel (multiple of 8, >= k + C - 1)
    int32_t wide_tpcu;     // wide kernel: traces per CTA (even, <= 16; the 16-trace TMA box starts at the CTA's first)
    int64_t trace_stride;
    const DevPolicy* pol;  // [n_lane]
    const int32_t* first_low;   // [2][n_traces] first subsampled tick with D <= B_lo / D > B_lo (INT32_MAX: none)
    // chain states, SoA: [e (0 entry, 1 exit)][q][s][j]
    uint8_t* st_f;
    uint64_t* st_log;
    int32_t* st_first;     // open-loop solo kernel (A30): [q][s][j] first event (lock | flag) of segment s from its start,
                           // | (the event's cmd) << 30; -1: no event in the segment
    float* st_ring;        // [e][q][s][r < kr][j]
    // per-chain totals [q][j], accumulated with atomics by every segment (and by the fix-up deltas):
    // integers add modulo 2^32 / 2^64 and the throttling excess is an exact fp64 sum, so the result
    // does not depend on the order of the additions
    uint32_t* c_nhi;
    uint32_t* c_nthr;
    uint32_t* c_trans;
    uint32_t* c_ev;
    uint32_t* c_lock;
    uint32_t* c_vmax;
    double* c_sexc;        // sum over throttled ticks of (D - B_lo)
    unsigned long long* c_digest;
    uint32_t* words;       // optional [q][j][n_blocks][2]
    const uint2* dkeys;    // [n_blocks] digest keys (digest_key), computed at create
};

__host__ __device__ __forceinline__ uint64_t fix_item(int q, int s, int j) {
    return ((uint64_t)q << 48) | ((uint64_t)(uint32_t)s << 32) | (uint64_t)(uint32_t)j;
}

// warp-aggregated append of `item` (lanes with want) to a worklist
__device__ __forceinline__ void wl_append(uint64_t* wl, uint32_t* count, bool want, uint64_t item) {
    const unsigned m = __ballot_sync(__activemask(), want);
    if (!want) return;
    const int leader = __ffs(m) - 1, lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(m));
    base = __shfl_sync(m, base, leader);
    wl[base + __popc(m & ((1u << lane) - 1u))] = item;
}

__host__ __device__ __forceinline__ int64_t st_idx(const ReplayParams& p, int e, int q, int s, int j) {
    MAGUS_CHECK(e >= 0 && e < 2 && q >= 0 && q < p.n_lane && s >= 0 && s < p.n_seg && j >= 0 && j < p.n_traces);
    return ((int64_t)(e * p.n_lane + q) * p.n_seg + s) * p.n_traces + j;
}
__host__ __device__ __forceinline__ int64_t ring_idx(const ReplayParams& p, int e, int q, int s, int r, int j) {
    MAGUS_CHECK(e >= 0 && e < 2 && q >= 0 && q < p.n_lane && s >= 0 && s < p.n_seg && r >= 0 && r < p.kr && j >= 0 &&
                j < p.n_traces);
    return (((int64_t)(e * p.n_lane + q) * p.n_seg + s) * p.kr + r) * p.n_traces + j;
}
// Time segment s covers ticks [seg_begin(s), seg_finish(s)): every boundary is a
// multiple of 32 (the digest / word blocks).
__host__ __device__ __forceinline__ int seg_begin(const ReplayParams& p, int s) {
    return s * p.seg_len + 32 * (s < p.seg_long ? s : p.seg_long);
}
__host__ __device__ __forceinline__ int seg_finish(const ReplayParams& p, int s) {
    const int e = seg_begin(p, s + 1);
    return e < p.n_samples ? e : p.n_samples;
}
__host__ __device__ __forceinline__ int64_t chain_idx(const ReplayParams& p, int q, int j) {
    MAGUS_CHECK(q >= 0 && q < p.n_lane && j >= 0 && j < p.n_traces);
    return (int64_t)q * p.n_traces + j;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {   // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ULL;
// digest keys of 32-tick block b: .x for the cmd word (high half of mix64(b * phi)),
// .y for the tune-flag word (low half), both odd, so w -> w * key is a bijection mod 2^32
__host__ __device__ __forceinline__ uint2 digest_key(uint64_t b) {
    const uint64_t m = mix64(b * kPhi);
    return make_uint2((uint32_t)(m >> 32) | 1u, (uint32_t)m | 1u);
}
// the 64-bit digest is two independent sums mod 2^32: (cmd sum << 32) | flag sum
__host__ __device__ __forceinline__ uint64_t digest_pack(uint32_t dc, uint32_t de) {
    return ((uint64_t)dc << 32) | (uint64_t)de;
}

// Chain kinds with C <= kMaxC32 keep the tune log in 32 bits and the scaled window count
// (ones << (C-1), which must not overflow: C * 2^(C-1) < 2^32); larger logs use the 64-bit kinds.
constexpr int kMaxC32 = 28;

template <bool LOG64>
struct LogWord { using T = uint32_t; };
template <>
struct LogWord<true> { using T = uint64_t; };

template <bool LOG64>
__device__ __forceinline__ uint32_t popc_log(typename LogWord<LOG64>::T v) {
    if constexpr (LOG64) return (uint32_t)__popcll(v);
    else return (uint32_t)__popc(v);
}

// Ring of the last k observations, newest first.  K > 0: fp64 registers (k <= 8, unrolled);
// K == 0: generic runtime k <= 64, fp32 circular buffer in local memory.
template <int K>
struct Ring {
    double v[K];
    __device__ __forceinline__ double oldest(int) const { return v[K - 1]; }
    __device__ __forceinline__ void push(double a, int) {
#pragma unroll
        for (int i = K - 1; i > 0; --i) v[i] = v[i - 1];
        v[0] = a;
    }
    __device__ __forceinline__ float get(int i, int) const { return (float)v[i]; }      // i = 0 newest
    // store the k values (newest first) to dst[i * stride]; compile-time indices keep v[] in registers
    __device__ __forceinline__ void store_all(float* dst, int, int64_t stride) const {
#pragma unroll
        for (int i = 0; i < K; ++i) dst[i * stride] = (float)v[i];
    }
    __device__ __forceinline__ bool same(const Ring& o, int) const {
        bool eq = true;
#pragma unroll
        for (int i = 0; i < K; ++i) eq = eq && (__double_as_longlong(v[i]) == __double_as_longlong(o.v[i]));
        return eq;
    }
    __device__ __forceinline__ void set_all(const float* src, int, int64_t stride) {
#pragma unroll
        for (int i = 0; i < K; ++i) v[i] = (double)src[i * stride];
    }
    __device__ __forceinline__ void clear(int) {
#pragma unroll
        for (int i = 0; i < K; ++i) v[i] = 0.0;
    }
};

template <>
struct Ring<0> {
    float v[KMAX_GENERIC];
    int head;   // index of the newest entry
    __device__ __forceinline__ double oldest(int k) const {
        int i = head - (k - 1);
        if (i < 0) i += k;
        return (double)v[i];
    }
    __device__ __forceinline__ void push(double a, int k) {
        head = (head + 1 == k) ? 0 : head + 1;
        v[head] = (float)a;
    }
    __device__ __forceinline__ float get(int i, int k) const {
        int x = head - i;
        if (x < 0) x += k;
        return v[x];
    }
    __device__ __forceinline__ void store_all(float* dst, int k, int64_t stride) const {
        for (int i = 0; i < k; ++i) dst[i * stride] = get(i, k);
    }
    __device__ __forceinline__ bool same(const Ring& o, int k) const {
        for (int i = 0; i < k; ++i)
            if (__float_as_uint(get(i, k)) != __float_as_uint(o.get(i, k))) return false;
        return true;
    }
    __device__ __forceinline__ void set_all(const float* src, int k, int64_t stride) {
        head = k - 1;   // newest at k-1, oldest at 0
        for (int i = 0; i < k; ++i) v[k - 1 - i] = src[i * stride];
    }
    __device__ __forceinline__ void clear(int k) {
        head = 0;
        for (int i = 0; i < k; ++i) v[i] = 0.0f;
    }
};

// State of one MAGUS chain between ticks.
template <int K, bool LOG64>
struct MagusState {
    using LogT = typename LogWord<LOG64>::T;
    uint32_t f;     // level in effect for the next tick (0 LO, 1 HI)
    LogT evh;       // tune-flag history, newest at bit 0; the log is the low C bits
    uint32_t cnt;   // 32-bit log only: (ones in the log) << (C-1), kept incrementally by the 4-chain tick
                    // (tick4_asm.cuh); derived from evh whenever a state is (re)built
    Ring<K> ring;
};

// Per-tick outputs needed by the accumulators.
struct TickOut {
    uint32_t cmd, ev, hf, thr, sig;   // sig: 1 = +1, 2 = -1, 0 = hold / not ready
};

// One MAGUS tick.  SLOW: the chain is within k + C - 1 ticks of its start, `ready` / `full` say
// whether Alg. 1 has k+1 samples and whether the log holds C flags (A7, A8); both are uniform
// across the warp because every chain of a warp starts at the same tick.
template <int K, bool LOG64, bool SLOW>
__device__ __forceinline__ TickOut magus_tick(MagusState<K, LOG64>& s, float D, const DevPolicy& pol,
                                              float B_lo, float B_hi, bool ready, bool full) {
    TickOut o;
    const float B = s.f ? B_hi : B_lo;
    const float A = fminf(D, B);
    o.thr = D > B;
    const double Ad = (double)A;
    const double d = Ad - s.ring.oldest(pol.k);
    s.ring.push(Ad, pol.k);
    bool inc = d > pol.dinc;
    bool dec = d < pol.ddec;
    if (SLOW && !ready) { inc = false; dec = false; }
    const uint32_t ev = (inc || dec) ? 1u : 0u;
    s.evh = (s.evh << 1) | (typename LogWord<LOG64>::T)ev;
    const uint32_t cnt = popc_log<LOG64>(s.evh & (typename LogWord<LOG64>::T)pol.logmask);
    if constexpr (!LOG64) s.cnt = cnt << (pol.C - 1);
    bool hf = cnt >= (uint32_t)pol.s_min;
    if (SLOW && !full) hf = false;
    const uint32_t cmd = (hf || inc || (s.f && !dec)) ? 1u : 0u;
    o.cmd = cmd;
    o.ev = ev;
    o.hf = hf ? 1u : 0u;
    o.sig = inc ? 1u : (dec ? 2u : 0u);
    s.f = cmd;
    return o;
}

// Intel default: cmd = LO iff pkg + DRAM power >= (1 - m) TDP, i.e. A >= a*[f] (section 8).
__device__ __forceinline__ TickOut tdp_tick(uint32_t& f, float D, const DevPolicy& pol, float B_lo, float B_hi) {
    TickOut o;
    const float B = f ? B_hi : B_lo;
    const float A = fminf(D, B);
    o.thr = D > B;
    const float as = f ? pol.astar_hi : pol.astar_lo;
    o.cmd = (A >= as) ? 0u : 1u;
    o.ev = 0;
    o.hf = 0;
    o.sig = 0;
    f = o.cmd;
    return o;
}

// Per-(chain, segment) statistics accumulated over the segment's own ticks.  sexc = the throttling
// excess X = sum over throttled ticks of (D - B_lo) (section 8): every term is exact in fp64, and so is
// the sum (every throttled D is an fp32 multiple of ulp32(B_lo) and N * bw_max / ulp32(B_lo) < 2^53).
struct SegStats {
    uint32_t nhi, nthr, trans, ev, lock, vmax;
    double sexc;
    uint32_t dc, de;   // digest halves (sums mod 2^32 of the cmd / tune-flag words times their block keys)
    __device__ __forceinline__ void zero() {
        nhi = nthr = trans = ev = lock = vmax = 0;
        sexc = 0.0;
        dc = de = 0;
    }
    __device__ __forceinline__ uint64_t digest() const { return digest_pack(dc, de); }
};

// Per-chain totals are zero at the start of every run: zeroed at creation, then by the totals kernel
// right after it reads them.
__device__ __forceinline__ void zero_chain(const ReplayParams& p, int64_t ci) {
    p.c_nhi[ci] = 0;
    p.c_nthr[ci] = 0;
    p.c_trans[ci] = 0;
    p.c_ev[ci] = 0;
    p.c_lock[ci] = 0;
    p.c_vmax[ci] = 0;
    p.c_sexc[ci] = 0.0;
    p.c_digest[ci] = 0;
}

// Add a segment's statistics (or a fix-up delta) to its chain's totals.
__device__ __forceinline__ void add_to_chain(const ReplayParams& p, int q, int j, uint32_t nhi, uint32_t nthr,
                                             uint32_t trans, uint32_t ev, uint32_t lock, double sexc, uint64_t digest) {
    const int64_t ci = chain_idx(p, q, j);
    if (nhi) atomicAdd(p.c_nhi + ci, nhi);
    if (nthr) atomicAdd(p.c_nthr + ci, nthr);
    if (trans) atomicAdd(p.c_trans + ci, trans);
    if (ev) atomicAdd(p.c_ev + ci, ev);
    if (lock) atomicAdd(p.c_lock + ci, lock);
    if (sexc != 0.0) atomicAdd(p.c_sexc + ci, sexc);
    // the two digest halves add independently (mod 2^32 each): no carry between them
    unsigned int* dg = reinterpret_cast<unsigned int*>(p.c_digest + ci);
    if ((uint32_t)digest) atomicAdd(dg, (unsigned int)(uint32_t)digest);
    if ((uint32_t)(digest >> 32)) atomicAdd(dg + 1, (unsigned int)(digest >> 32));
}

// Full-block fold (n == 32) with the block's digest keys (digest_key(b)) supplied by the caller.
__device__ __forceinline__ void fold_full_block(SegStats& st, uint32_t wcmd, uint32_t ew, uint32_t fstart,
                                                uint2 bkey, uint32_t* words_out) {
    const uint32_t lw = (wcmd >> 1) | (fstart << 31);   // level in effect per tick
    st.trans += __popc(wcmd ^ lw);
    st.nhi += __popc(lw);
    st.ev += __popc(ew);
    st.dc += wcmd * bkey.x;
    st.de += ew * bkey.y;
    if (words_out) {
        words_out[0] = wcmd;
        words_out[1] = ew;
    }
}

// Fold one 32-tick block [bt0, bt0 + n): `wcmd` holds the block's cmd bits (newest at bit 0, plus the
// previous tick's cmd above them), `ew` the tune flags (same alignment), fstart the level at bt0.
__device__ __forceinline__ void fold_block(SegStats& st, uint32_t wcmd, uint32_t ew, uint32_t fstart, int n,
                                           int64_t block_index, uint32_t* words_out) {
    const uint32_t mask = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    const uint32_t cw = wcmd & mask;
    const uint32_t lw = ((wcmd >> 1) & (mask >> 1)) | (fstart << (n - 1));   // level in effect per tick
    const uint32_t evw = ew & mask;
    st.trans += __popc(cw ^ lw);
    st.nhi += __popc(lw);
    st.ev += __popc(evw);
    const int sh = 32 - n;
    const uint32_t wc = cw << sh, we = evw << sh;   // tick bt0 + i at bit 31 - i; partial block zero-padded
    const uint2 key = digest_key((uint64_t)block_index);
    st.dc += wc * key.x;
    st.de += we * key.y;
    if (words_out) {
        words_out[0] = wc;
        words_out[1] = we;
    }
}

}  // namespace magus
