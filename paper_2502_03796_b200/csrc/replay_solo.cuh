// replay_solo.cuh -- the replay kernel for launch groups with one policy warp per tile group (npw == 1:
// configs 2, 4, 5) and a MAGUS chain kind with a whole-stage PTX block (k <= 3, 32-bit log).
//
// Same work unit, pipeline and segmentation as magus_replay_kernel (replay_kernel.cuh), but a CTA is ONE
// warp that consumes its own 3-deep ring of [8 ticks x 128 traces] TMA tiles.  Every pipeline address and
// counter (tile / barrier slot, phase, stage index, TMA coordinates) is then CTA-uniform, so ptxas keeps
// them in uniform registers: a stage costs its try-wait, one elected expect-tx arrive and one UTMALDG
// instead of the per-lane slot arithmetic and the elect loop of the multi-warp kernel.  Steady-state
// blocks run four calls of the generated whole-stage block (MAGUS_STAGE8_K<K>: the level carried as a
// predicate across the 8 ticks, the ring of A values in virtual registers).  DESIGN.md section 7.
#pragma once
#include <cuda.h>
#include "device_common.cuh"
#include "ptx.cuh"
#include "replay_kernel.cuh"
#include "tickers.cuh"

namespace magus {

#define K_OF(T) T::kRingK

#ifndef MAGUS_SOLO_UNROLL
#define MAGUS_SOLO_UNROLL 1
#endif

#ifndef MAGUS_SOLO_CTAS_PER_SM
#define MAGUS_SOLO_CTAS_PER_SM 16
#endif
constexpr int kSoloCtasPerSm = MAGUS_SOLO_CTAS_PER_SM;   // 16 one-warp CTAs per SM: 128 registers and ~12.3 KB smem each

template <int TC, int NSTAGE>
struct SoloSmem {
    static constexpr int kTileBytes = TC * kTracesPerWarp * 4;
    static constexpr size_t kBytes = (size_t)NSTAGE * kTileBytes + NSTAGE * sizeof(uint64_t);
};

__device__ __forceinline__ uint32_t elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}"
        : "=r"(p));
    return p;
}

// blocking parity wait on an mbarrier (try_wait loop inside one PTX block)
__device__ __forceinline__ void mbar_wait_loop(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// the elected lane arms `bar` for one tile and issues its 2-D TMA box {128 traces, TC ticks} at (x, t0)
template <int TC>
__device__ __forceinline__ void solo_issue(uint32_t tile, const CUtensorMap* tmap, uint32_t bar, int x, int t0,
                                           uint64_t cpol) {
    MAGUS_CHECK(smem_range_ok(tile, TC * kTracesPerWarp * 4) && smem_range_ok(bar, 8) && x >= 0 && t0 >= 0);
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%2], [%3, {%4, %5}], [%0], %6;\n\t}" ::"r"(bar),
        "n"(TC * kTracesPerWarp * 4), "r"(tile), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(t0),
        "l"(cpol)
        : "memory");
}


// Release a consumed ring slot.  Solo (COMBO = false): the warp owns the ring, so its elected lane refills the slot
// at once (its lanes' shared-memory reads are complete after the caller's __syncwarp).  COMBO: arrive on
// empty[slot]; the producer warp (the MAGUS warp of magus_replay_combo_kernel) waits until both consumer warps have
// arrived, then refills.  `refill` is false for the producer past the last stage and always for the other warp.
template <int TC, bool COMBO>
__device__ __forceinline__ void solo_release(uint32_t tile, const CUtensorMap* tmap, uint32_t bar0, uint32_t empty0,
                                             int slot, uint32_t phase, bool refill, int x, int t0, uint64_t cpol,
                                             int lane) {
    if constexpr (COMBO) {
        if (lane == 0) ptx::mbar_arrive_u32(empty0 + 8 * slot);
        if (refill) {
            mbar_wait_loop(empty0 + 8 * slot, phase);
            solo_issue<TC>(tile, tmap, bar0 + 8 * slot, x, t0, cpol);
        }
    } else {
        if (refill) solo_issue<TC>(tile, tmap, bar0 + 8 * slot, x, t0, cpol);
    }
}

// run constants of the pipe-balanced stage block (MAGUS_SSTAGE_K<K>, tick4_asm.cuh)
struct SoloConst {
    double Blo_d;   // B_lo as fp64
    float B_lo;
};

// One whole steady-state stage (8 ticks x 4 chains) of MAGUS chains with a register ring of K <= 3 values,
// with the 3-DSETP / 1-PLOP3 level logic: V = 3 Alg. 2 by popcount (MAGUS_PSTAGE_K<K>), V = 4 by the scaled
// incremental count (MAGUS_QSTAGE_K<K>); V = 5 / 6 the same with the chains interleaved in pairs, V = 7 / 8 one
// chain after the other (predicate-register pressure).
#ifndef MAGUS_PQ_GROUP
#define MAGUS_PQ_GROUP 4
#endif
#define PQ_CAT3(a, b, c) a##b##c
#define PQ_NAME(P, G, K) PQ_CAT3(P, G, K)
template <int K, int V>
__device__ __forceinline__ void solo_stage_pq(MagusState<K, false>* s, float* lock, float* nthr, uint32_t* wcmd,
                                              SegStats* ss, uint32_t& vmax, uint32_t tile, const SoloConst& sc,
                                              const DevPolicy& pol) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
#define PQ_F s[0].f, s[1].f, s[2].f, s[3].f
#define PQ_R1 s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0]
#define PQ_R2                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define PQ_R3                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
#define PQ_STATS                                                                                               \
    ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, lock[0], lock[1], lock[2], lock[3], nthr[0], nthr[1], nthr[2], \
        nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax, tile, sc.B_lo, sc.Blo_d, pol.dinc, pol.ddec
#define PQ_P(G, KK) PQ_NAME(MAGUS_PSTAGE, G, KK)
#define PQ_Q(G, KK) PQ_NAME(MAGUS_QSTAGE, G, KK)
#define PQ_CNT s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt
    const uint32_t maskc = (uint32_t)pol.logmask, smin = (uint32_t)pol.s_min;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define PQ_BODY(G)                                                                                             \
    if constexpr (V % 2 == 1) {                                                                                \
        if constexpr (K == 1) PQ_P(G, _K1)(PQ_F, PQ_R1, e0, e1, e2, e3, PQ_STATS, maskc, smin, pol.one);         \
        else if constexpr (K == 2) PQ_P(G, _K2)(PQ_F, PQ_R2, e0, e1, e2, e3, PQ_STATS, maskc, smin, pol.one);    \
        else PQ_P(G, _K3)(PQ_F, PQ_R3, e0, e1, e2, e3, PQ_STATS, maskc, smin, pol.one);                          \
    } else {                                                                                                   \
        if constexpr (K == 1)                                                                                  \
            PQ_Q(G, _K1)(PQ_F, PQ_R1, e0, e1, e2, e3, PQ_CNT, PQ_STATS, bitc, pol.smin_sc, pol.one, mone);       \
        else if constexpr (K == 2)                                                                             \
            PQ_Q(G, _K2)(PQ_F, PQ_R2, e0, e1, e2, e3, PQ_CNT, PQ_STATS, bitc, pol.smin_sc, pol.one, mone);       \
        else PQ_Q(G, _K3)(PQ_F, PQ_R3, e0, e1, e2, e3, PQ_CNT, PQ_STATS, bitc, pol.smin_sc, pol.one, mone);      \
    }
    if constexpr (V <= 4) { PQ_BODY() }
    else if constexpr (V <= 6) { PQ_BODY(G2) }
    else if constexpr (V <= 8) { PQ_BODY(G1) }
    else if constexpr (V <= 10) { PQ_BODY(S) }
    else if constexpr (V <= 12) { PQ_BODY(SG2) }
    else { PQ_BODY(SG1) }
#undef PQ_BODY
#undef PQ_CNT
#undef PQ_P
#undef PQ_Q
#undef PQ_F
#undef PQ_R1
#undef PQ_R2
#undef PQ_R3
#undef PQ_STATS
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

// One whole steady-state stage (8 ticks x 4 chains) of MAGUS chains with a register ring of K <= 3 values.
// BITS: the fp32 -> fp64 sample conversion by integer ops (MAGUS_SSTAGEFB_K<K>, no XU), THR32 only.
template <int K, bool THR32 = false, bool BITS = false>
__device__ __forceinline__ void solo_stage(MagusState<K, false>* s, float* lock, float* nthr,
                                           uint32_t* wcmd, SegStats* ss, uint32_t& vmax, uint32_t tile,
                                           const SoloConst& sc, const DevPolicy& pol) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define SOLO_TAIL                                                                                              \
    e0, e1, e2, e3, s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, lock[0],    \
        lock[1], lock[2], lock[3], nthr[0], nthr[1], nthr[2], nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax, \
        tile, sc.Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define SOLO_TAILF                                                                                             \
    e0, e1, e2, e3, s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, lock[0], \
        lock[1], lock[2], lock[3], nthr[0], nthr[1], nthr[2], nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax,   \
        tile, sc.B_lo, sc.Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define SOLO_F s[0].f, s[1].f, s[2].f, s[3].f
#define SOLO_R1 s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0]
#define SOLO_R2                                                                                                \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define SOLO_R3                                                                                                \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
    if constexpr (THR32 && BITS) {
        if constexpr (K == 1) MAGUS_SSTAGEFB_K1(SOLO_F, SOLO_R1, SOLO_TAILF);
        else if constexpr (K == 2) MAGUS_SSTAGEFB_K2(SOLO_F, SOLO_R2, SOLO_TAILF);
        else MAGUS_SSTAGEFB_K3(SOLO_F, SOLO_R3, SOLO_TAILF);
    } else if constexpr (THR32) {   // throttle test as an fp32 compare on the ALU pipe (less FP64 work, less power)
        if constexpr (K == 1) MAGUS_SSTAGEF_K1(SOLO_F, SOLO_R1, SOLO_TAILF);
        else if constexpr (K == 2) MAGUS_SSTAGEF_K2(SOLO_F, SOLO_R2, SOLO_TAILF);
        else MAGUS_SSTAGEF_K3(SOLO_F, SOLO_R3, SOLO_TAILF);
    } else {
        if constexpr (K == 1) MAGUS_SSTAGE_K1(SOLO_F, SOLO_R1, SOLO_TAIL);
        else if constexpr (K == 2) MAGUS_SSTAGE_K2(SOLO_F, SOLO_R2, SOLO_TAIL);
        else MAGUS_SSTAGE_K3(SOLO_F, SOLO_R3, SOLO_TAIL);
    }
#undef SOLO_TAILF
#undef SOLO_R1
#undef SOLO_R2
#undef SOLO_R3
#undef SOLO_TAIL
#undef SOLO_F
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

// One whole steady-state stage (8 ticks x 4 chains) with the level carried in the cmd word and the lock as the sign
// of the biased window count (MAGUS_LSTAGE_K<K>, BAL = 20).  The caller keeps s[c].cnt biased by -smin_sc and
// wcmd[c]'s bit 0 = the level across the steady stages; nlk[c] counts the ticks not locked.  BATCH
// (MAGUS_LB[S]STAGE_K<K>, BAL = 24 / 25, 8 <= C <= 24): the tune-flag log shifted once per stage too, the
// count scaled by 2^8 instead of 2^(C-1) (the caller converts it around the steady block).
template <int K, bool SYM, bool BATCH = false>
__device__ __forceinline__ void solo_stage_l(MagusState<K, false>* s, uint32_t* nlk, float* nthr, uint32_t* wcmd,
                                             SegStats* ss, uint32_t& vmax, uint32_t tile, const SoloConst& sc,
                                             const DevPolicy& pol) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define LS_TAIL                                                                                                \
    e0, e1, e2, e3, s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, nlk[0],  \
        nlk[1], nlk[2], nlk[3], nthr[0], nthr[1], nthr[2], nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax, tile,  \
        sc.B_lo, sc.Blo_d, pol.dinc, pol.ddec, bitc, pol.one, mone
#define LS_BTAIL LS_TAIL, (uint32_t)(pol.C - 1)
#define LS_R2                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define LS_R3                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
    if constexpr (BATCH && SYM) {
        if constexpr (K == 1) MAGUS_LBSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LS_BTAIL);
        else if constexpr (K == 2) MAGUS_LBSTAGES_K2(LS_R2, LS_BTAIL);
        else MAGUS_LBSTAGES_K3(LS_R3, LS_BTAIL);
    } else if constexpr (BATCH) {
        if constexpr (K == 1) MAGUS_LBSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LS_BTAIL);
        else if constexpr (K == 2) MAGUS_LBSTAGE_K2(LS_R2, LS_BTAIL);
        else MAGUS_LBSTAGE_K3(LS_R3, LS_BTAIL);
    } else if constexpr (SYM) {   // d*_dec == -d*_inc: the |d| tune-flag test
        if constexpr (K == 1) MAGUS_LSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LS_TAIL);
        else if constexpr (K == 2) MAGUS_LSTAGES_K2(LS_R2, LS_TAIL);
        else MAGUS_LSTAGES_K3(LS_R3, LS_TAIL);
    } else {
        if constexpr (K == 1) MAGUS_LSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LS_TAIL);
        else if constexpr (K == 2) MAGUS_LSTAGE_K2(LS_R2, LS_TAIL);
        else MAGUS_LSTAGE_K3(LS_R3, LS_TAIL);
    }
#undef LS_R2
#undef LS_R3
#undef LS_BTAIL
#undef LS_TAIL
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

// One whole steady-state stage (8 ticks x 4 chains) of the open-loop observation model (A30; MAGUS_OSTAGE[S]_K<K>,
// BAL 30 / 31): the L stage without throttling (A = D) plus the event word ewd (lock | flag per tick).  BATCH
// (MAGUS_OBSTAGE[S]_K<K>, BAL 34 / 35, 8 <= C <= 24): solo_stage_l's batched tune-flag log.
template <int K, bool SYM, bool BATCH = false>
__device__ __forceinline__ void solo_stage_o(MagusState<K, false>* s, uint32_t* nlk, uint32_t* wcmd, uint32_t* ewd,
                                             uint32_t& vmax, uint32_t tile, const DevPolicy& pol) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define OS_TAIL                                                                                                \
    e0, e1, e2, e3, s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, nlk[0], nlk[1], nlk[2], nlk[3], wcmd[0], wcmd[1],       \
        wcmd[2], wcmd[3], ewd[0], ewd[1], ewd[2], ewd[3], vmax, tile, pol.dinc, pol.ddec, bitc, pol.one, mone
#define OS_BTAIL OS_TAIL, (uint32_t)(pol.C - 1)
#define OS_R2                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define OS_R3                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
    if constexpr (BATCH && SYM) {
        if constexpr (K == 1) MAGUS_OBSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], OS_BTAIL);
        else if constexpr (K == 2) MAGUS_OBSTAGES_K2(OS_R2, OS_BTAIL);
        else MAGUS_OBSTAGES_K3(OS_R3, OS_BTAIL);
    } else if constexpr (BATCH) {
        if constexpr (K == 1) MAGUS_OBSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], OS_BTAIL);
        else if constexpr (K == 2) MAGUS_OBSTAGE_K2(OS_R2, OS_BTAIL);
        else MAGUS_OBSTAGE_K3(OS_R3, OS_BTAIL);
    } else if constexpr (SYM) {
        if constexpr (K == 1) MAGUS_OSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], OS_TAIL);
        else if constexpr (K == 2) MAGUS_OSTAGES_K2(OS_R2, OS_TAIL);
        else MAGUS_OSTAGES_K3(OS_R3, OS_TAIL);
    } else {
        if constexpr (K == 1) MAGUS_OSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], OS_TAIL);
        else if constexpr (K == 2) MAGUS_OSTAGE_K2(OS_R2, OS_TAIL);
        else MAGUS_OSTAGE_K3(OS_R3, OS_TAIL);
    }
#undef OS_R2
#undef OS_R3
#undef OS_BTAIL
#undef OS_TAIL
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

// The MAGUS solo replay of one (lane policy q, tile group, segment) by one warp, on a TMA ring that the caller has
// initialised and primed with the first NSTAGE stages.  COMBO = false: the warp owns the ring and refills a slot
// right after its own __syncwarp.  COMBO = true (magus_replay_combo_kernel): a second warp (the TDP baselines)
// consumes the same tiles; both release a slot on empty[slot] and this warp, the producer, refills it once both
// have released it.
template <class T, int TC, int NSTAGE, int BAL, bool COMBO>
__device__ __forceinline__ void solo_magus_body(const CUtensorMap* tmap, const ReplayParams& p, const uint8_t* smem,
                                                uint32_t tile0, uint32_t bar0, uint32_t empty0, int q, int tgroup,
                                                int seg, int lane) {
    static_assert(T::kHasStage8 && TC == 8, "solo kernel: whole-stage PTX block of 8 ticks");
    using State = typename T::State;
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    const SegGeom G = seg_geom<TC>(p, seg);
    const int x = tgroup * kTracesPerWarp;
    const uint64_t cpol = ptx::policy_evict_first();
    const DevPolicy pol = p.pol[q];
    const int j0 = x + lane * kChains;
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    SoloConst sc;
    sc.Blo_d = (double)B_lo;
    sc.B_lo = B_lo;
    const double Blo_d = sc.Blo_d;
    const int k = pol.k, C = pol.C;
    // ticks before Alg. 1 / 2 are fully defined (A7, A8).  Speculative segments (seg > 0) may instead start
    // from a synthetic full state (p.solo_flags bit 0): the ring filled with the first observation, the log
    // holding C zero flags.  Their warm-up ticks are not counted and only their state at s*L matters,
    // which the fix-up checks exactly, so they run the steady-state block throughout.
    const bool synth = seg > 0 && (p.solo_flags & 1u);
    const int warm_ticks = synth ? 0 : k + C - 1;
    const uint32_t lane_off = (uint32_t)lane * 16u;

    State st[kChains];
    SegStats ss[kChains];
    uint32_t wcmd[kChains], fstart[kChains];
    float lockf[kChains], nthrf[kChains];   // counts as exact fp32 integers (segment length <= 2^24)
    uint32_t nlk[kChains];   // BAL 20: ticks not locked in the counted steady blocks (lock = lockf + 32 nsb - nlk)
    uint32_t nsb = 0;        // BAL 20: counted steady blocks
    constexpr bool kOpen = BAL == 30 || BAL == 31 || BAL == 34 || BAL == 35;   // the open-loop stage (A30)
    constexpr bool kBatchLog = (BAL >= 24 && BAL < 30) || BAL == 34 || BAL == 35;   // the batched tune-flag log
    constexpr bool kL = BAL == 20 || BAL == 21 || BAL == 24 || BAL == 25;   // the L stage (24/25: batched flag log)
    uint32_t ewd[kChains];   // open loop: event word (lock | flag per tick, the cmd word's layout)
    int32_t fev[kChains];    // open loop: first event of the segment (ticks from its start) | its cmd << 30, -1: none
    uint32_t vmax = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        T::init(st[c], pol, seg == 0);
        ss[c].zero();
        wcmd[c] = 0;
        lockf[c] = nthrf[c] = 0.f;
        nlk[c] = 0;
        ewd[c] = 0;
        fev[c] = -1;
    }

    int i = 0;           // stage index (CTA-uniform)
    int slot = 0;        // i % NSTAGE
    uint32_t phase = 0;  // (i / NSTAGE) & 1
    for (int bt0 = G.tau_w; bt0 < G.seg_end; bt0 += 32) {
        if (bt0 == G.seg_start) {   // the segment's own ticks start: record the entry, reset the statistics
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if (j0 + c < p.n_traces) T::save(st[c], p, pol, 0, q, seg, j0 + c);
                ss[c].zero();
                lockf[c] = nthrf[c] = 0.f;
                nlk[c] = 0;
                fev[c] = -1;
            }
            nsb = 0;
        }
        if (bt0 == G.tau_w && seg > 0) {
            // speculative level at the warm-up start: f_max iff the trace is above B_lo
            // now and was at or below B_lo before (a high stretch entered through a rising edge that Alg. 1
            // sees even at f_min; a trace never below B_lo is never seen to rise, A14); lock-sticky policies
            // (k >= s_min) keep f_max after any low/high transition (K9)
            mbar_wait_loop(bar0 + 8 * slot, phase);
            float4 d0;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(d0.x), "=f"(d0.y), "=f"(d0.z), "=f"(d0.w)
                         : "r"(tile0 + slot * kTileBytes + lane_off)
                         : "memory");
            const float dd[4] = {d0.x, d0.y, d0.z, d0.w};
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                const int j = j0 + c;
                const int fl = j < p.n_traces ? __ldg(p.first_low + j) : 0x7FFFFFFF;
                const int fh = j < p.n_traces ? __ldg(p.first_low + p.n_traces + j) : 0x7FFFFFFF;
                const bool hi = (dd[c] > B_lo && fl < G.tau_w) || (pol.sticky && fl < G.tau_w && fh < G.tau_w);
                T::set_level(st[c], hi ? 1u : 0u);
                if (synth) {
                    const double a0 = (double)(hi ? dd[c] : fminf(dd[c], B_lo));
#pragma unroll
                    for (int r = 0; r < (int)(sizeof(st[c].ring.v) / sizeof(double)); ++r) st[c].ring.v[r] = a0;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kChains; ++c) fstart[c] = T::level(st[c]);
        const bool counting = bt0 >= G.seg_start;
        if (bt0 + 32 <= G.seg_end && bt0 - G.tau_w >= warm_ticks) {
            // steady state: four whole-stage PTX blocks
            if constexpr (kL || kOpen) {   // the count biased by -s_min << (C-1); the level in the cmd word's bit 0
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    st[c].cnt -= pol.smin_sc;
                    if constexpr (kBatchLog)   // the batched log's count scale 2^TC (exact: C - 1 >= TC - 1)
                        st[c].cnt = (uint32_t)((int32_t)st[c].cnt >> (pol.C - 1)) << TC;
                    wcmd[c] = T::level(st[c]);
                }
                if (counting) ++nsb;
            }
#if MAGUS_SOLO_UNROLL == 2
#pragma unroll 2
#else
#pragma unroll 1
#endif
            for (int sub = 0; sub < 32 / TC; ++sub) {
                const uint32_t tile = tile0 + slot * kTileBytes;
                MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
                mbar_wait_loop(bar0 + 8 * slot, phase);
                if constexpr (BAL == 1) solo_stage(st, lockf, nthrf, wcmd, ss, vmax, tile + lane_off, sc, pol);
                else if constexpr (BAL == 2)
                    solo_stage<T::kRingK, true>(st, lockf, nthrf, wcmd, ss, vmax, tile + lane_off, sc, pol);
                else if constexpr (BAL == 5)
                    solo_stage<T::kRingK, true, true>(st, lockf, nthrf, wcmd, ss, vmax, tile + lane_off, sc, pol);
                else if constexpr (BAL == 3 || BAL == 4 || (BAL >= 9 && BAL < 20))
                    solo_stage_pq<T::kRingK, BAL>(st, lockf, nthrf, wcmd, ss, vmax, tile + lane_off, sc, pol);
                else if constexpr (kL)
                    solo_stage_l<T::kRingK, BAL == 21 || BAL == 25, (BAL >= 24)>(st, nlk, nthrf, wcmd, ss, vmax,
                                                                               tile + lane_off, sc, pol);
                else if constexpr (kOpen)
                    solo_stage_o<T::kRingK, BAL == 31 || BAL == 35, (BAL >= 34)>(st, nlk, wcmd, ewd, vmax,
                                                                                 tile + lane_off, pol);
                else T::stage8(st, tile + lane_off, pol, B_lo, Blo_d, wcmd, ss, vmax);
                __syncwarp();   // every lane's tile reads are complete before the slot is refilled
                solo_release<TC, COMBO>(tile, tmap, bar0, empty0, slot, phase, i + NSTAGE < G.n_stages, x,
                                        G.tau_w + (i + NSTAGE) * TC, cpol, lane);
                ++i;
                if (++slot == NSTAGE) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
            if constexpr (kL || kOpen) {
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    if constexpr (kBatchLog) st[c].cnt = (uint32_t)((int32_t)st[c].cnt >> TC) << (pol.C - 1);
                    st[c].cnt += pol.smin_sc;
                    T::set_level(st[c], wcmd[c] & 1u);
                }
            }
        } else {
            // warm-up block (Alg. 1 / Alg. 2 gated per tick) or the ragged last block of a trace
#pragma unroll 1
            for (int sub = 0; sub < 32 / TC && i < G.n_stages; ++sub) {
                const int t0 = bt0 + sub * TC;
                const uint32_t tile = tile0 + slot * kTileBytes;
                MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
                mbar_wait_loop(bar0 + 8 * slot, phase);
                const float4* rows = reinterpret_cast<const float4*>(smem + slot * kTileBytes) + lane;
                if (t0 + TC <= G.seg_end && !kOpen) {
#pragma unroll 1   // rolled: the warm-up path runs on ~2% of the stages; its code stays small
                    for (int tt = 0; tt < TC; ++tt) {
                        const int r = t0 + tt - G.tau_w;
                        const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                        T::warm4(st, d, pol, B_lo, Blo_d, wcmd, ss, vmax, r >= k ? 1u : 0u, r >= k + C - 1 ? 1u : 0u);
                    }
                } else {
                    for (int tt = 0; tt < TC; ++tt) {
                        const int t = t0 + tt;
                        if (t >= G.seg_end) break;
                        const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                        const bool ready = (t - G.tau_w) >= k;
                        const bool lfull = (t - G.tau_w) >= k + C - 1;
#pragma unroll
                        for (int c = 0; c < kChains; ++c) {
                            const TickOut o = T::template tick<true>(st[c], d[c], pol, B_lo, B_hi, ready, lfull);
                            wcmd[c] = (wcmd[c] << 1) | o.cmd;
                            if constexpr (kOpen) ewd[c] = (ewd[c] << 1) | o.ev | o.hf;   // lock | flag
                            acc_tick(ss[c], vmax, o, d[c], B_lo);
                        }
                    }
                }
                __syncwarp();
                solo_release<TC, COMBO>(tile, tmap, bar0, empty0, slot, phase, i + NSTAGE < G.n_stages, x,
                                        G.tau_w + (i + NSTAGE) * TC, cpol, lane);
                ++i;
                if (++slot == NSTAGE) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
        if (counting) {
            const uint2 bkey = p.dkeys[bt0 >> 5];
            const int n = min(32, G.seg_end - bt0);
            if constexpr (kOpen) {   // the segment's first event (tick i of the block at bit n - 1 - i)
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    const uint32_t em = n >= 32 ? ewd[c] : (ewd[c] & ((1u << n) - 1u));
                    if (fev[c] < 0 && em != 0u) {
                        const int h = 31 - __clz(em);
                        fev[c] = (bt0 - G.seg_start + (n - 1 - h)) | (int32_t)(((wcmd[c] >> h) & 1u) << 30);
                    }
                }
            }
            if (n == 32 && p.words == nullptr) {   // the common case: a whole block, no word dump
#pragma unroll
                for (int c = 0; c < kChains; ++c)
                    fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], bkey, nullptr);
            } else {
                const int64_t bi = bt0 >> 5;
                uint32_t* wbase = p.words ? p.words + ((int64_t)q * p.n_traces * p.n_blocks + bi) * 2 : nullptr;
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    uint32_t* wout =
                        (wbase && j0 + c < p.n_traces) ? wbase + (int64_t)(j0 + c) * p.n_blocks * 2 : nullptr;
                    if (n == 32) fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], bkey, wout);
                    else fold_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], n, bi, wout);
                }
            }
        }
    }

#pragma unroll
    for (int c = 0; c < kChains; ++c)
        if (j0 + c < p.n_traces) {
            T::save(st[c], p, pol, 1, q, seg, j0 + c);
            if constexpr (kOpen) p.st_first[st_idx(p, 0, q, seg, j0 + c)] = fev[c];
        }
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const int j = j0 + c;
        if (j >= p.n_traces) continue;
        add_to_chain(p, q, j, ss[c].nhi, ss[c].nthr + (uint32_t)nthrf[c], ss[c].trans, ss[c].ev,
                     ss[c].lock + (uint32_t)lockf[c] + (kL || kOpen ? 32u * nsb - nlk[c] : 0u),
                     ss[c].sexc, ss[c].digest());
    }
    if (j0 < p.n_traces) atomicMax(p.c_vmax + chain_idx(p, q, j0), vmax);   // lane-level validation maximum
}

// BAL: 0 = the integer stage block (MAGUS_STAGE8_K<K>), 1 = the pipe-balanced one (MAGUS_SSTAGE_K<K>),
// 2 = balanced with the throttle test on the ALU pipe (MAGUS_SSTAGEF_K<K>), 3 / 4 = the 3-DSETP level logic with
// Alg. 2 by popcount / by the incremental count (MAGUS_PSTAGE_K<K> / MAGUS_QSTAGE_K<K>)
template <class T, int TC, int NSTAGE, int BAL>
__global__ void __launch_bounds__(32, kSoloCtasPerSm)
    magus_replay_solo_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x;
    // blockIdx -> (lane policy, tile group, segment); policies fastest so the CTAs of one (group,
    // segment) read the same tiles close together in time (L2 reuse when nq > 1)
    int b = blockIdx.x;
    const int qi = b % p.nq;
    b /= p.nq;
    const int tgroup = b % p.n_groups;
    const int seg = b / p.n_groups;
    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t bar0 = tile0 + NSTAGE * kTileBytes;
    if (lane == 0) {
        ptx::prefetch_tmap(&tmap);
        for (int i = 0; i < NSTAGE; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        ptx::fence_mbar_init();
    }
    __syncwarp();
    const SegGeom G = seg_geom<TC>(p, seg);
    const uint64_t cpol = ptx::policy_evict_first();
    for (int i = 0; i < NSTAGE && i < G.n_stages; ++i)
        solo_issue<TC>(tile0 + i * kTileBytes, &tmap, bar0 + 8 * i, tgroup * kTracesPerWarp, G.tau_w + i * TC, cpol);
    ptx::pdl_wait();   // first_low and the scratch words come from the pre-pass (launched just before)
    solo_magus_body<T, TC, NSTAGE, BAL, false>(&tmap, p, smem, tile0, bar0, 0u, p.q_base + qi, tgroup, seg, lane);
}

// ===================================================================================================================
// The unified-stage solo kernel: one generated stage block (MAGUS_USTAGE{S}_K<K>) for the
// warm-up and the steady state.  Alg. 1 is gated by a NaN-filled ring at the start of the chain's run, Alg. 2 by
// warp-uniform per-tick masks (zero until C flags have been logged), so the warm-up needs no per-tick path and can
// be short: speculative segments start p.solo_warm ticks (a multiple of 8, >= k + C - 1) before their first tick
// instead of a whole 32-tick block.  Only the ragged last stage of a trace uses the generic per-tick tick.
// VAR bits: 1 = symmetric thresholds (the |d| tune-flag test), 2 = Alg. 2 by the scaled incremental count (else
// by popcount), 4 = the fp32 -> fp64 sample conversion by integer ops (else F2F).  g[]: the per-tick Alg. 2 gates.
#define USTAGE_NAME(S, I, B, KK) MAGUS_USTAGE##S##I##B##_K##KK
template <int K, int VAR>
__device__ __forceinline__ void solo_ustage(MagusState<K, false>* s, float* lock, float* nthr, uint32_t* wcmd,
                                           SegStats* ss, uint32_t& vmax, uint32_t tile, const SoloConst& sc,
                                           const DevPolicy& pol, const uint32_t* g, uint32_t smin, uint32_t bitc,
                                           uint32_t mone) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
#define U_F s[0].f, s[1].f, s[2].f, s[3].f
#define U_R1 s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0]
#define U_R2                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define U_R3                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
#define U_CNT s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt,
#define U_MID                                                                                                 \
    ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, lock[0], lock[1], lock[2], lock[3], nthr[0], nthr[1], nthr[2], \
        nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax, tile, sc.B_lo, sc.Blo_d, pol.dinc, pol.ddec, g[0], g[1],  \
        g[2], g[3], g[4], g[5], g[6], g[7]
#define U_RING(KK) U_R##KK
#define U_CALLP(S, B, KK) USTAGE_NAME(S, , B, KK)(U_F, U_RING(KK), e0, e1, e2, e3, U_MID, smin, pol.one)
#define U_CALLI(S, B, KK) USTAGE_NAME(S, I, B, KK)(U_F, U_RING(KK), e0, e1, e2, e3, U_CNT U_MID, bitc, mone, pol.one)
#define U_BY_K(CALL, S, B)                                                                                     \
    if constexpr (K == 1) CALL(S, B, 1);                                                                       \
    else if constexpr (K == 2) CALL(S, B, 2);                                                                  \
    else CALL(S, B, 3);
    constexpr bool kSym = VAR & 1, kInc = VAR & 2, kBits = VAR & 4;
    if constexpr (kSym && kInc && kBits) { U_BY_K(U_CALLI, S, B) }
    else if constexpr (kSym && kInc) { U_BY_K(U_CALLI, S, ) }
    else if constexpr (kSym && kBits) { U_BY_K(U_CALLP, S, B) }
    else if constexpr (kSym) { U_BY_K(U_CALLP, S, ) }
    else if constexpr (kInc && kBits) { U_BY_K(U_CALLI, , B) }
    else if constexpr (kInc) { U_BY_K(U_CALLI, , ) }
    else if constexpr (kBits) { U_BY_K(U_CALLP, , B) }
    else { U_BY_K(U_CALLP, , ) }
#undef U_BY_K
#undef U_CALLI
#undef U_CALLP
#undef U_RING
#undef U_MID
#undef U_CNT
#undef U_F
#undef U_R1
#undef U_R2
#undef U_R3
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

template <class T, int TC, int NSTAGE, int VAR>
__global__ void __launch_bounds__(32, kSoloCtasPerSm)
    magus_replay_usolo_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    static_assert(T::kHasStage8 && TC == 8, "solo kernel: whole-stage PTX block of 8 ticks");
    using State = typename T::State;
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x;

    int b = blockIdx.x;   // -> (lane policy, tile group, segment), policies fastest
    const int qi = b % p.nq;
    b /= p.nq;
    const int tgroup = b % p.n_groups;
    const int seg = b / p.n_groups;
    const int q = p.q_base + qi;

    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t bar0 = tile0 + NSTAGE * kTileBytes;
    if (lane == 0) {
        ptx::prefetch_tmap(&tmap);
        for (int i = 0; i < NSTAGE; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        ptx::fence_mbar_init();
    }
    __syncwarp();

    const int seg_start = seg_begin(p, seg), seg_end = seg_finish(p, seg);
    const int tau_w = seg == 0 ? 0 : seg_start - p.solo_warm;
    const int n_stages = (seg_end - tau_w + TC - 1) / TC;
    const int x = tgroup * kTracesPerWarp;
    const uint64_t cpol = ptx::policy_evict_first();
    for (int i = 0; i < NSTAGE && i < n_stages; ++i)
        solo_issue<TC>(tile0 + i * kTileBytes, &tmap, bar0 + 8 * i, x, tau_w + i * TC, cpol);
    ptx::pdl_wait();   // first_low and the scratch words come from the pre-pass (launched just before)

    const DevPolicy pol = p.pol[q];
    const int j0 = x + lane * kChains;
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    SoloConst sc;
    sc.Blo_d = (double)B_lo;
    sc.B_lo = B_lo;
    const int k = pol.k, C = pol.C, kc1 = k + C - 1;
    const uint32_t smin = (uint32_t)pol.s_min, bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
    // Alg. 2 gate of a tick once the log is full / before (A8): the window mask / 0 (popcount), the scaled lock
    // threshold / never (incremental count)
    const uint32_t g_full = (VAR & 2) ? pol.smin_sc : (uint32_t)pol.logmask, g_not = (VAR & 2) ? 0xFFFFFFFFu : 0u;
    const uint32_t lane_off = (uint32_t)lane * 16u;

    State st[kChains];
    SegStats ss[kChains];
    uint32_t wcmd[kChains], fstart[kChains];
    float lockf[kChains], nthrf[kChains];   // counts as exact fp32 integers (segment length <= 2^24)
    uint32_t vmax = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        T::init(st[c], pol, seg == 0);
#pragma unroll
        for (int r = 0; r < T::kRingK; ++r) st[c].ring.v[r] = __longlong_as_double(0x7FF8000000000000LL);   // A7 gate
        ss[c].zero();
        wcmd[c] = 0;
        lockf[c] = nthrf[c] = 0.f;
    }
    // per-tick Alg. 2 gates of the next stage (A8): g_full once k + C - 1 ticks of the run have passed
    uint32_t m[TC];
    auto set_masks = [&](int r0) {
#pragma unroll
        for (int t = 0; t < TC; ++t) m[t] = (r0 + t >= kc1) ? g_full : g_not;
    };
    set_masks(0);

    if (seg > 0) {
        // speculative level at the warm-up start: f_max iff the trace is above B_lo now and
        // was at or below B_lo before; lock-sticky policies (k >= s_min) keep f_max after any low/high transition
        mbar_wait_loop(bar0, 0);
        float4 d0;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(d0.x), "=f"(d0.y), "=f"(d0.z), "=f"(d0.w)
                     : "r"(tile0 + lane_off)
                     : "memory");
        const float dd[4] = {d0.x, d0.y, d0.z, d0.w};
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            const int j = j0 + c;
            const int fl = j < p.n_traces ? __ldg(p.first_low + j) : 0x7FFFFFFF;
            const int fh = j < p.n_traces ? __ldg(p.first_low + p.n_traces + j) : 0x7FFFFFFF;
            const bool hi = (dd[c] > B_lo && fl < tau_w) || (pol.sticky && fl < tau_w && fh < tau_w);
            T::set_level(st[c], hi ? 1u : 0u);
        }
    }

    // One loop over the run's stages (one call site of the stage block: the warm-up stages, then the segment's
    // own ticks in 32-tick blocks of four stages).  All branch conditions are CTA-uniform.
    int slot = 0;        // i % NSTAGE
    uint32_t phase = 0;  // (i / NSTAGE) & 1
#pragma unroll 1
    for (int i = 0; i < n_stages; ++i) {
        const int t0 = tau_w + i * TC;
        if (t0 >= seg_start && ((t0 - seg_start) & 31) == 0) {
            if (t0 == seg_start && seg > 0) {   // the segment's own ticks start: record the entry state
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    if (j0 + c < p.n_traces) T::save(st[c], p, pol, 0, q, seg, j0 + c);
                    ss[c].zero();
                    lockf[c] = nthrf[c] = 0.f;
                }
            }
#pragma unroll
            for (int c = 0; c < kChains; ++c) fstart[c] = T::level(st[c]);
        }
        const uint32_t tile = tile0 + slot * kTileBytes;
        MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
        mbar_wait_loop(bar0 + 8 * slot, phase);
        if (t0 + TC <= seg_end) {
            solo_ustage<K_OF(T), VAR>(st, lockf, nthrf, wcmd, ss, vmax, tile + lane_off, sc, pol, m, smin, bitc, mone);
        } else {   // the ragged last stage of a trace: per tick
            const float4* rows = reinterpret_cast<const float4*>(smem + slot * kTileBytes) + lane;
#pragma unroll 1
            for (int tt = 0; tt < TC; ++tt) {
                const int t = t0 + tt;
                if (t >= seg_end) break;
                const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                const bool ready = (t - tau_w) >= k;
                const bool lfull = (t - tau_w) >= kc1;
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    const TickOut o = T::template tick<true>(st[c], d[c], pol, B_lo, B_hi, ready, lfull);
                    wcmd[c] = (wcmd[c] << 1) | o.cmd;
                    acc_tick(ss[c], vmax, o, d[c], B_lo);
                }
            }
        }
        __syncwarp();   // every lane's tile reads are complete before the slot is refilled
        if (i + NSTAGE < n_stages) solo_issue<TC>(tile, &tmap, bar0 + 8 * slot, x, tau_w + (i + NSTAGE) * TC, cpol);
        if (++slot == NSTAGE) {
            slot = 0;
            phase ^= 1u;
        }
        if ((t0 - tau_w) < kc1) set_masks(t0 + TC - tau_w);   // masks settle at maskc after the gated stages
        const int t1 = t0 + TC;
        if (t0 >= seg_start && (((t1 - seg_start) & 31) == 0 || t1 >= seg_end)) {   // a 32-tick block ends
            const int bt0 = seg_start + ((t0 - seg_start) & ~31);
            const uint2 bkey = p.dkeys[bt0 >> 5];
            const int n = min(32, seg_end - bt0);
            if (n == 32 && p.words == nullptr) {   // the common case: a whole block, no word dump
#pragma unroll
                for (int c = 0; c < kChains; ++c)
                    fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], bkey, nullptr);
            } else {
                const int64_t bi = bt0 >> 5;
                uint32_t* wbase = p.words ? p.words + ((int64_t)q * p.n_traces * p.n_blocks + bi) * 2 : nullptr;
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    uint32_t* wout =
                        (wbase && j0 + c < p.n_traces) ? wbase + (int64_t)(j0 + c) * p.n_blocks * 2 : nullptr;
                    if (n == 32) fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], bkey, wout);
                    else fold_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], n, bi, wout);
                }
            }
        }
    }

#pragma unroll
    for (int c = 0; c < kChains; ++c)
        if (j0 + c < p.n_traces) T::save(st[c], p, pol, 1, q, seg, j0 + c);
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const int j = j0 + c;
        if (j >= p.n_traces) continue;
        add_to_chain(p, q, j, ss[c].nhi, ss[c].nthr + (uint32_t)nthrf[c], ss[c].trans, ss[c].ev,
                     ss[c].lock + (uint32_t)lockf[c], ss[c].sexc, ss[c].digest());
    }
    if (j0 < p.n_traces) atomicMax(p.c_vmax + chain_idx(p, q, j0), vmax);   // lane-level validation maximum
}

// ===================================================================================================================
// The TDP_DEFAULT solo kernel (the Intel-default baseline): one-warp CTAs with the solo kernel's TMA ring;
// a warp runs NP TDP policies on the same 128 traces (4 per lane), so the samples are read once for the NP
// policies.  One generated stage block per 8 ticks (MAGUS_TSTAGE<NP>, tick4_asm.cuh).  The throttled demand is
// summed in fp64 as sum(D) (a 0/1 DFMA, exact) and turned into the excess sum(D - B_lo) = sum(D) - n_thr B_lo once
// per segment (exact: DESIGN.md section 8).  Speculative segments start p.warmup ticks early at the guessed
// level (f_max); the exact fix-up is the TDP lockstep walk.
// The TDP solo replay of one (policy pair pi, tile group, segment) by one warp on a primed TMA ring.  COMBO: the ring
// is shared with the MAGUS warp of magus_replay_combo_kernel, which refills it; this warp only releases its slots.
#ifndef MAGUS_TDP_LEAN
#define MAGUS_TDP_LEAN 0   // build switch: 1 = MAGUS_TSTAGE1L{V} (two-compare level, no select, validation only in
                           // the first group): measured slower on config 5 (0.624 vs 0.607 ms, profiles/r02_tdp_lean_ab.txt)
#endif
// VALIDATE: this launch group takes the validation maximum (A17); the other groups of a run skip it, since every
// group replays the same samples and the check is over the union of all lanes' maxima (one TDP policy per warp).
template <int NP, int TC, int NSTAGE, bool COMBO, bool VALIDATE = true>
__device__ __forceinline__ void tsolo_body(const CUtensorMap* tmap, const ReplayParams& p, const uint8_t* smem,
                                           uint32_t tile0, uint32_t bar0, uint32_t empty0, int pi, int tgroup, int seg,
                                           int lane) {
    static_assert(TC == 8, "TDP solo kernel: whole-stage PTX block of 8 ticks");
    constexpr int NC = 4 * NP;   // chains per lane
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    int qs[NP];
    bool live[NP];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
        const int qi = pi * NP + u;
        live[u] = qi < p.nq;
        qs[u] = p.q_base + (live[u] ? qi : pi * NP);   // a missing second policy repeats the first, unrecorded
    }
    const SegGeom G = seg_geom<TC>(p, seg);
    const int x = tgroup * kTracesPerWarp;
    const uint64_t cpol = ptx::policy_evict_first();
    const int j0 = x + lane * kChains;
    const float B_lo = p.B_lo;
    const double Blo_d = (double)B_lo;
    float ahi[NP], alo[NP];
    uint32_t f[NC], wcmd[NC], fstart[NC];
    double exc[NC];
    double sfac[4] = {0.0, 0.0, 0.0, 0.0};   // MAGUS_TSTAGE1L: the throttled 0/1 factors (low words stay 0)
    float nthrf[NC];
    uint32_t nhi[NC], trans[NC], dc[NC];
    uint32_t one = 1, vmax = 0;
#pragma unroll
    for (int u = 0; u < NP; ++u) {
        const DevPolicy pol = p.pol[qs[u]];
        one = pol.one;
        ahi[u] = pol.astar_hi;
        alo[u] = B_lo >= pol.astar_lo ? pol.astar_lo : __int_as_float(0x7F800000);   // A = min(D, B_lo) at f_min
#pragma unroll
        for (int c = 0; c < 4; ++c) f[u * 4 + c] = seg == 0 ? (uint32_t)pol.f0 : (uint32_t)pol.guess_f;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        wcmd[c] = 0;
        exc[c] = 0.0;
        nthrf[c] = 0.f;
        nhi[c] = trans[c] = dc[c] = 0;
    }
    const uint32_t lane_off = (uint32_t)lane * 16u;
    int i = 0, slot = 0;
    uint32_t phase = 0;
#pragma unroll 1
    for (int bt0 = G.tau_w; bt0 < G.seg_end; bt0 += 32) {
        if (bt0 == G.seg_start) {
#pragma unroll
            for (int u = 0; u < NP; ++u)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int j = j0 + c, cc = u * 4 + c;
                    if (j < p.n_traces && live[u]) {
                        const int64_t si = st_idx(p, 0, qs[u], seg, j);
                        p.st_f[si] = (uint8_t)f[cc];
                        p.st_log[si] = 0;
                    }
                    exc[cc] = 0.0;
                    nthrf[cc] = 0.f;
                    nhi[cc] = trans[cc] = dc[cc] = 0;
                }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) fstart[c] = f[c];
#pragma unroll 1
        for (int sub = 0; sub < 32 / TC && i < G.n_stages; ++sub) {
            const int t0 = bt0 + sub * TC;
            const uint32_t tile = tile0 + slot * kTileBytes;
            MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
            mbar_wait_loop(bar0 + 8 * slot, phase);
            if (t0 + TC <= G.seg_end) {
                if constexpr (NP == 1 && !MAGUS_TDP_LEAN)
                    MAGUS_TSTAGE1(f[0], f[1], f[2], f[3], exc[0], exc[1], exc[2], exc[3], nthrf[0], nthrf[1], nthrf[2],
                                  nthrf[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax, tile + lane_off, B_lo, ahi[0],
                                  alo[0], one);
                else if constexpr (NP == 1 && VALIDATE)
                    MAGUS_TSTAGE1LV(f[0], f[1], f[2], f[3], exc[0], exc[1], exc[2], exc[3], nthrf[0], nthrf[1],
                                    nthrf[2], nthrf[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], sfac[0], sfac[1], sfac[2],
                                    sfac[3], vmax, tile + lane_off, B_lo, ahi[0], alo[0], one);
                else if constexpr (NP == 1)
                    MAGUS_TSTAGE1L(f[0], f[1], f[2], f[3], exc[0], exc[1], exc[2], exc[3], nthrf[0], nthrf[1],
                                   nthrf[2], nthrf[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], sfac[0], sfac[1], sfac[2],
                                   sfac[3], tile + lane_off, B_lo, ahi[0], alo[0], one);
                else
                    MAGUS_TSTAGE2(f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], exc[0], exc[1], exc[2], exc[3],
                                  exc[4], exc[5], exc[6], exc[7], nthrf[0], nthrf[1], nthrf[2], nthrf[3], nthrf[4],
                                  nthrf[5], nthrf[6], nthrf[7], wcmd[0], wcmd[1], wcmd[2], wcmd[3], wcmd[4], wcmd[5],
                                  wcmd[6], wcmd[7], vmax, tile + lane_off, B_lo, ahi[0], ahi[1], alo[0], alo[1], one);
            } else {   // the ragged last stage of a trace: the same tick, per tick
                const float4* rows = reinterpret_cast<const float4*>(smem + slot * kTileBytes) + lane;
#pragma unroll 1
                for (int tt = 0; tt < TC; ++tt) {
                    if (t0 + tt >= G.seg_end) break;
                    const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                    const float d[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                    for (int cc = 0; cc < NC; ++cc) {
                        const float D = d[cc % 4];
                        const bool thr = f[cc] == 0u && D > B_lo;
                        const float a = f[cc] ? ahi[cc / 4] : alo[cc / 4];
                        f[cc] = D < a ? 1u : 0u;
                        exc[cc] = __fma_rn(thr ? 1.0 : 0.0, (double)D, exc[cc]);
                        nthrf[cc] += thr ? 1.f : 0.f;
                        wcmd[cc] = (wcmd[cc] << 1) | f[cc];
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) vmax = max(vmax, __float_as_uint(d[c]));
                }
            }
            __syncwarp();
            solo_release<TC, COMBO>(tile, tmap, bar0, empty0, slot, phase, !COMBO && i + NSTAGE < G.n_stages, x,
                                    G.tau_w + (i + NSTAGE) * TC, cpol, lane);
            ++i;
            if (++slot == NSTAGE) {
                slot = 0;
                phase ^= 1u;
            }
        }
        if (bt0 >= G.seg_start) {   // fold the 32-tick block: level / transition counts and the digest (no tune flags)
            const int n = min(32, G.seg_end - bt0);
            const int64_t bi = bt0 >> 5;
            const uint2 bkey = p.dkeys[bi];
#pragma unroll
            for (int u = 0; u < NP; ++u) {
                uint32_t* wbase =
                    (p.words && live[u]) ? p.words + ((int64_t)qs[u] * p.n_traces * p.n_blocks + bi) * 2 : nullptr;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int cc = u * 4 + c;
                    const uint32_t mask = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
                    const uint32_t cw = wcmd[cc] & mask;
                    const uint32_t lw = ((wcmd[cc] >> 1) & (mask >> 1)) | (fstart[cc] << (n - 1));
                    trans[cc] += __popc(cw ^ lw);
                    nhi[cc] += __popc(lw);
                    const uint32_t wc = cw << (32 - n);
                    dc[cc] += wc * (n == 32 ? bkey.x : digest_key((uint64_t)bi).x);
                    if (wbase && j0 + c < p.n_traces) {
                        uint32_t* wo = wbase + (int64_t)(j0 + c) * p.n_blocks * 2;
                        wo[0] = wc;
                        wo[1] = 0u;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < NP; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + c, cc = u * 4 + c;
            if (j >= p.n_traces || !live[u]) continue;
            const int64_t si = st_idx(p, 1, qs[u], seg, j);
            p.st_f[si] = (uint8_t)f[cc];
            p.st_log[si] = 0;
            const uint32_t nthr = (uint32_t)nthrf[cc];
            // sum(D - B_lo) over throttled ticks, exact; no throttled tick: 0 (the open-loop mode's B_lo is +inf)
            const double sexc = nthr ? exc[cc] - (double)nthr * Blo_d : 0.0;
            add_to_chain(p, qs[u], j, nhi[cc], nthr, trans[cc], 0u, 0u, sexc, digest_pack(dc[cc], 0u));
        }
    if (j0 < p.n_traces) atomicMax(p.c_vmax + chain_idx(p, qs[0], j0), vmax);
}

template <int NP, int TC, int NSTAGE, bool VALIDATE = true>
__global__ void __launch_bounds__(32, kSoloCtasPerSm)
    magus_replay_tsolo_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x;
    const int npairs = (p.nq + NP - 1) / NP;
    int b = blockIdx.x;
    const int pi = b % npairs;
    b /= npairs;
    const int tgroup = b % p.n_groups;
    const int seg = b / p.n_groups;
    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t bar0 = tile0 + NSTAGE * kTileBytes;
    if (lane == 0) {
        ptx::prefetch_tmap(&tmap);
        for (int i = 0; i < NSTAGE; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        ptx::fence_mbar_init();
    }
    __syncwarp();
    const SegGeom G = seg_geom<TC>(p, seg);
    const uint64_t cpol = ptx::policy_evict_first();
    for (int i = 0; i < NSTAGE && i < G.n_stages; ++i)
        solo_issue<TC>(tile0 + i * kTileBytes, &tmap, bar0 + 8 * i, tgroup * kTracesPerWarp, G.tau_w + i * TC, cpol);
    ptx::pdl_wait();
    tsolo_body<NP, TC, NSTAGE, false, VALIDATE>(&tmap, p, smem, tile0, bar0, 0u, pi, tgroup, seg, lane);
}

// ===================================================================================================================
// The combined kernel for a run of one MAGUS solo policy and NP TDP_DEFAULT baselines (config 5): a CTA of two warps
// shares one TMA ring, so every trace tile is read from HBM once for all of the run's replayed policies.  Warp 0
// replays MAGUS (solo_magus_body) and refills the ring; warp 1 replays the TDP pair (tsolo_body).  A slot is refilled
// once both warps released it (empty mbarrier, count 2).  p.q_base / p.nq: the MAGUS group; p.q_base2 / p.nq2: the
// TDP group.  The per-chain states, statistics and fix-up are those of the two separate kernels.
template <class T, int NP, int TC, int NSTAGE>
__global__ void __launch_bounds__(64, kSoloCtasPerSm / 2)
    magus_replay_combo_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tgroup = blockIdx.x % p.n_groups;
    const int seg = blockIdx.x / p.n_groups;
    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t bar0 = tile0 + NSTAGE * kTileBytes, empty0 = bar0 + 8 * NSTAGE;
    if (warp == 0) {
        if (lane == 0) {
            ptx::prefetch_tmap(&tmap);
            for (int i = 0; i < NSTAGE; ++i) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(empty0 + 8 * i) : "memory");
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        const SegGeom G = seg_geom<TC>(p, seg);
        const uint64_t cpol = ptx::policy_evict_first();
        for (int i = 0; i < NSTAGE && i < G.n_stages; ++i)
            solo_issue<TC>(tile0 + i * kTileBytes, &tmap, bar0 + 8 * i, tgroup * kTracesPerWarp, G.tau_w + i * TC,
                           cpol);
    }
    __syncthreads();   // the barriers are initialised before warp 1 waits on them
    ptx::pdl_wait();
    if (warp == 0) {
        solo_magus_body<T, TC, NSTAGE, 2, true>(&tmap, p, smem, tile0, bar0, empty0, p.q_base, tgroup, seg, lane);
    } else {
        ReplayParams pt = p;
        pt.q_base = p.q_base2;
        pt.nq = p.nq2;
        tsolo_body<NP, TC, NSTAGE, true, false>(&tmap, pt, smem, tile0, bar0, empty0, 0, tgroup, seg, lane);
    }
}

// ===================================================================================================================
// The fused MAGUS + TDP kernel (config 5: one MAGUS policy next to one replayed TDP_DEFAULT baseline): ONE warp per
// (tile group, segment) replays both on its own TMA ring, every lane stepping its 4 traces' MAGUS chains and TDP chains
// over the same samples (MAGUS_LTSTAGE[S]_K<K>: one tile load, one fp64 conversion and one validation maximum per
// sample for both), so every trace byte is read from HBM once.  p.q_base / p.q_base2: the MAGUS
// and the TDP policy.  MAGUS as solo_magus_body's L stage (BAL 20 / 21); TDP as tsolo_body with its level carried in
// its cmd word's bit 0.  The per-chain states, statistics and fix-up are those of the two separate kernels.
#ifndef MAGUS_FUSED_CTAS_PER_SM
#define MAGUS_FUSED_CTAS_PER_SM 12
#endif
constexpr int kFusedCtasPerSm = MAGUS_FUSED_CTAS_PER_SM;

template <int K, bool SYM, bool UP, bool LB>
__device__ __forceinline__ void fused_stage_lt(MagusState<K, false>* s, uint32_t* nlk, float* nthr, uint32_t* wcmd,
                                               SegStats* ss, uint32_t& vmax, uint32_t* wcmdT, double* excT,
                                               float* nthrT, double* sT, uint32_t tile, const SoloConst& sc,
                                               const DevPolicy& pol, float ahi, float alo) {
    uint32_t e0 = s[0].evh, e1 = s[1].evh, e2 = s[2].evh, e3 = s[3].evh;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
#define LT_TAIL                                                                                                \
    e0, e1, e2, e3, s[0].cnt, s[1].cnt, s[2].cnt, s[3].cnt, ss[0].sexc, ss[1].sexc, ss[2].sexc, ss[3].sexc, nlk[0],  \
        nlk[1], nlk[2], nlk[3], nthr[0], nthr[1], nthr[2], nthr[3], wcmd[0], wcmd[1], wcmd[2], wcmd[3], vmax,        \
        wcmdT[0], wcmdT[1], wcmdT[2], wcmdT[3], excT[0], excT[1], excT[2], excT[3], nthrT[0], nthrT[1], nthrT[2],     \
        nthrT[3], sT[0], sT[1], sT[2], sT[3], tile, sc.B_lo, sc.Blo_d, pol.dinc, pol.ddec, bitc, pol.one, mone, ahi, alo
#define LT_BTAIL LT_TAIL, (uint32_t)(pol.C - 1)
#define LT_R2                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[1].ring.v[0], s[1].ring.v[1], s[2].ring.v[0], s[2].ring.v[1], s[3].ring.v[0], \
        s[3].ring.v[1]
#define LT_R3                                                                                                  \
    s[0].ring.v[0], s[0].ring.v[1], s[0].ring.v[2], s[1].ring.v[0], s[1].ring.v[1], s[1].ring.v[2], s[2].ring.v[0], \
        s[2].ring.v[1], s[2].ring.v[2], s[3].ring.v[0], s[3].ring.v[1], s[3].ring.v[2]
    if constexpr (LB && UP && SYM) {   // LB: the batched tune-flag log (solo_stage_l's BATCH)
        if constexpr (K == 1) MAGUS_LBTUSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_BTAIL);
        else if constexpr (K == 2) MAGUS_LBTUSTAGES_K2(LT_R2, LT_BTAIL);
        else MAGUS_LBTUSTAGES_K3(LT_R3, LT_BTAIL);
    } else if constexpr (LB && UP) {
        if constexpr (K == 1) MAGUS_LBTUSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_BTAIL);
        else if constexpr (K == 2) MAGUS_LBTUSTAGE_K2(LT_R2, LT_BTAIL);
        else MAGUS_LBTUSTAGE_K3(LT_R3, LT_BTAIL);
    } else if constexpr (LB && SYM) {
        if constexpr (K == 1) MAGUS_LBTSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_BTAIL);
        else if constexpr (K == 2) MAGUS_LBTSTAGES_K2(LT_R2, LT_BTAIL);
        else MAGUS_LBTSTAGES_K3(LT_R3, LT_BTAIL);
    } else if constexpr (LB) {
        if constexpr (K == 1) MAGUS_LBTSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_BTAIL);
        else if constexpr (K == 2) MAGUS_LBTSTAGE_K2(LT_R2, LT_BTAIL);
        else MAGUS_LBTSTAGE_K3(LT_R3, LT_BTAIL);
    } else if constexpr (UP && SYM) {   // the TDP policy's f_min threshold is +inf: f_min always rises
        if constexpr (K == 1) MAGUS_LTUSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_TAIL);
        else if constexpr (K == 2) MAGUS_LTUSTAGES_K2(LT_R2, LT_TAIL);
        else MAGUS_LTUSTAGES_K3(LT_R3, LT_TAIL);
    } else if constexpr (UP) {
        if constexpr (K == 1) MAGUS_LTUSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_TAIL);
        else if constexpr (K == 2) MAGUS_LTUSTAGE_K2(LT_R2, LT_TAIL);
        else MAGUS_LTUSTAGE_K3(LT_R3, LT_TAIL);
    } else if constexpr (SYM) {
        if constexpr (K == 1) MAGUS_LTSTAGES_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_TAIL);
        else if constexpr (K == 2) MAGUS_LTSTAGES_K2(LT_R2, LT_TAIL);
        else MAGUS_LTSTAGES_K3(LT_R3, LT_TAIL);
    } else {
        if constexpr (K == 1) MAGUS_LTSTAGE_K1(s[0].ring.v[0], s[1].ring.v[0], s[2].ring.v[0], s[3].ring.v[0], LT_TAIL);
        else if constexpr (K == 2) MAGUS_LTSTAGE_K2(LT_R2, LT_TAIL);
        else MAGUS_LTSTAGE_K3(LT_R3, LT_TAIL);
    }
#undef LT_R2
#undef LT_R3
#undef LT_BTAIL
#undef LT_TAIL
    s[0].evh = e0;
    s[1].evh = e1;
    s[2].evh = e2;
    s[3].evh = e3;
}

template <class T, int TC, int NSTAGE, bool SYM, int MINB = kFusedCtasPerSm, bool UP = false, bool LB = false>
__global__ void __launch_bounds__(32, MINB)
    magus_replay_fused_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    static_assert(T::kHasStage8 && TC == 8, "fused kernel: whole-stage PTX blocks of 8 ticks");
    using State = typename T::State;
    using SM = SoloSmem<TC, NSTAGE>;
    constexpr uint32_t kTileBytes = SM::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x;
    const int tgroup = blockIdx.x % p.n_groups;
    const int seg = blockIdx.x / p.n_groups;
    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t bar0 = tile0 + NSTAGE * kTileBytes;
    if (lane == 0) {
        ptx::prefetch_tmap(&tmap);
        for (int i = 0; i < NSTAGE; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        ptx::fence_mbar_init();
    }
    __syncwarp();
    const SegGeom G = seg_geom<TC>(p, seg);
    const uint64_t cpol = ptx::policy_evict_first();
    const int x = tgroup * kTracesPerWarp;
    for (int i = 0; i < NSTAGE && i < G.n_stages; ++i) solo_issue<TC>(tile0 + i * kTileBytes, &tmap, bar0 + 8 * i, x, G.tau_w + i * TC, cpol);
    ptx::pdl_wait();   // first_low and the scratch words come from the pre-pass (launched just before)

    const int q = p.q_base, qT = p.q_base2;
    const DevPolicy pol = p.pol[q];
    const int j0 = x + lane * kChains;
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    SoloConst sc;
    sc.Blo_d = (double)B_lo;
    sc.B_lo = B_lo;
    const double Blo_d = sc.Blo_d;
    const int k = pol.k, C = pol.C;
    const bool synth = seg > 0 && (p.solo_flags & 1u);
    const int warm_ticks = synth ? 0 : k + C - 1;
    const uint32_t lane_off = (uint32_t)lane * 16u;
    // TDP (tsolo_body, NP = 1): next level f_max iff A < a*[f]; a_lo = +inf when B_lo < a*_lo (A = min(D, B_lo))
    float ahi, alo;
    uint32_t fT0;
    {
        const DevPolicy polT = p.pol[qT];
        ahi = polT.astar_hi;
        alo = B_lo >= polT.astar_lo ? polT.astar_lo : __int_as_float(0x7F800000);
        fT0 = seg == 0 ? (uint32_t)polT.f0 : (uint32_t)polT.guess_f;
    }

    State st[kChains];
    SegStats ss[kChains];
    uint32_t wcmd[kChains], fstart[kChains];
    float lockf[kChains], nthrf[kChains];
    uint32_t nlk[kChains];
    uint32_t nsb = 0;
    uint32_t vmax = 0;
    uint32_t wcmdT[kChains], fstartT[kChains], nhiT[kChains], transT[kChains], dcT[kChains];
    double excT[kChains], sT[kChains];
    float nthrT[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        T::init(st[c], pol, seg == 0);
        ss[c].zero();
        wcmd[c] = 0;
        lockf[c] = nthrf[c] = 0.f;
        nlk[c] = 0;
        wcmdT[c] = fT0;   // bit 0 = the TDP level
        excT[c] = sT[c] = 0.0;
        nthrT[c] = 0.f;
        nhiT[c] = transT[c] = dcT[c] = 0;
    }

    int i = 0, slot = 0;
    uint32_t phase = 0;
#pragma unroll 1
    for (int bt0 = G.tau_w; bt0 < G.seg_end; bt0 += 32) {
        if (bt0 == G.seg_start) {   // the segment's own ticks start: record the entries, reset the statistics
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                const int j = j0 + c;
                if (j < p.n_traces) {
                    T::save(st[c], p, pol, 0, q, seg, j);
                    const int64_t si = st_idx(p, 0, qT, seg, j);
                    p.st_f[si] = (uint8_t)(wcmdT[c] & 1u);
                    p.st_log[si] = 0;
                }
                ss[c].zero();
                lockf[c] = nthrf[c] = 0.f;
                nlk[c] = 0;
                excT[c] = 0.0;
                nthrT[c] = 0.f;
                nhiT[c] = transT[c] = dcT[c] = 0;
            }
            nsb = 0;
        }
        if (bt0 == G.tau_w && seg > 0) {   // MAGUS's speculative level at the warm-up start (solo_magus_body)
            mbar_wait_loop(bar0 + 8 * slot, phase);
            float4 d0;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(d0.x), "=f"(d0.y), "=f"(d0.z), "=f"(d0.w)
                         : "r"(tile0 + slot * kTileBytes + lane_off)
                         : "memory");
            const float dd[4] = {d0.x, d0.y, d0.z, d0.w};
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                const int j = j0 + c;
                const int fl = j < p.n_traces ? __ldg(p.first_low + j) : 0x7FFFFFFF;
                const int fh = j < p.n_traces ? __ldg(p.first_low + p.n_traces + j) : 0x7FFFFFFF;
                const bool hi = (dd[c] > B_lo && fl < G.tau_w) || (pol.sticky && fl < G.tau_w && fh < G.tau_w);
                T::set_level(st[c], hi ? 1u : 0u);
                if (synth) {
                    const double a0 = (double)(hi ? dd[c] : fminf(dd[c], B_lo));
#pragma unroll
                    for (int r = 0; r < (int)(sizeof(st[c].ring.v) / sizeof(double)); ++r) st[c].ring.v[r] = a0;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            fstart[c] = T::level(st[c]);
            fstartT[c] = wcmdT[c] & 1u;
        }
        const bool counting = bt0 >= G.seg_start;
        if (bt0 + 32 <= G.seg_end && bt0 - G.tau_w >= warm_ticks) {
            // steady state: four fused whole-stage PTX blocks
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                st[c].cnt -= pol.smin_sc;
                if constexpr (LB) st[c].cnt = (uint32_t)((int32_t)st[c].cnt >> (pol.C - 1)) << TC;   // 2^TC scale
                wcmd[c] = fstart[c];
            }
            if (counting) ++nsb;
#pragma unroll 1
            for (int sub = 0; sub < 32 / TC; ++sub) {
                const uint32_t tile = tile0 + slot * kTileBytes;
                MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
                mbar_wait_loop(bar0 + 8 * slot, phase);
                fused_stage_lt<T::kRingK, SYM, UP, LB>(st, nlk, nthrf, wcmd, ss, vmax, wcmdT, excT, nthrT, sT, tile + lane_off,
                                               sc, pol, ahi, alo);
                __syncwarp();   // every lane's tile reads are complete before the slot is refilled
                solo_release<TC, false>(tile, &tmap, bar0, 0u, slot, phase, i + NSTAGE < G.n_stages, x,
                                        G.tau_w + (i + NSTAGE) * TC, cpol, lane);
                ++i;
                if (++slot == NSTAGE) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if constexpr (LB) st[c].cnt = (uint32_t)((int32_t)st[c].cnt >> TC) << (pol.C - 1);
                st[c].cnt += pol.smin_sc;
                T::set_level(st[c], wcmd[c] & 1u);
            }
        } else {
            // warm-up block (MAGUS's Alg. 1 / Alg. 2 gated per tick) or the ragged last block of a trace
#pragma unroll 1
            for (int sub = 0; sub < 32 / TC && i < G.n_stages; ++sub) {
                const int t0 = bt0 + sub * TC;
                const uint32_t tile = tile0 + slot * kTileBytes;
                MAGUS_CHECK(slot >= 0 && slot < NSTAGE && smem_range_ok(tile + lane_off, (TC - 1) * 512 + 16));
                mbar_wait_loop(bar0 + 8 * slot, phase);
                const float4* rows = reinterpret_cast<const float4*>(smem + slot * kTileBytes) + lane;
                if (t0 + TC <= G.seg_end) {
#pragma unroll 1
                    for (int tt = 0; tt < TC; ++tt) {
                        const int r = t0 + tt - G.tau_w;
                        const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                        T::warm4(st, d, pol, B_lo, Blo_d, wcmd, ss, vmax, r >= k ? 1u : 0u, r >= k + C - 1 ? 1u : 0u);
                    }
                    MAGUS_TLSTAGE(wcmdT[0], wcmdT[1], wcmdT[2], wcmdT[3], excT[0], excT[1], excT[2], excT[3], nthrT[0],
                                  nthrT[1], nthrT[2], nthrT[3], sT[0], sT[1], sT[2], sT[3], tile + lane_off, B_lo, ahi,
                                  alo, pol.one);
                } else {
                    for (int tt = 0; tt < TC; ++tt) {
                        const int t = t0 + tt;
                        if (t >= G.seg_end) break;
                        const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                        const bool ready = (t - G.tau_w) >= k;
                        const bool lfull = (t - G.tau_w) >= k + C - 1;
#pragma unroll
                        for (int c = 0; c < kChains; ++c) {
                            const TickOut o = T::template tick<true>(st[c], d[c], pol, B_lo, B_hi, ready, lfull);
                            wcmd[c] = (wcmd[c] << 1) | o.cmd;
                            acc_tick(ss[c], vmax, o, d[c], B_lo);
                            const uint32_t fT = wcmdT[c] & 1u;   // TDP tick (tsolo_body's ragged path)
                            const bool thr = fT == 0u && d[c] > B_lo;
                            wcmdT[c] = (wcmdT[c] << 1) | ((d[c] < ahi || (fT == 0u && d[c] < alo)) ? 1u : 0u);
                            excT[c] = __fma_rn(thr ? 1.0 : 0.0, (double)d[c], excT[c]);
                            nthrT[c] += thr ? 1.f : 0.f;
                        }
                    }
                }
                __syncwarp();
                solo_release<TC, false>(tile, &tmap, bar0, 0u, slot, phase, i + NSTAGE < G.n_stages, x,
                                        G.tau_w + (i + NSTAGE) * TC, cpol, lane);
                ++i;
                if (++slot == NSTAGE) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
        if (counting) {
            const int64_t bi = bt0 >> 5;
            const uint2 bkey = p.dkeys[bi];
            const int n = min(32, G.seg_end - bt0);
            uint32_t* wbase = p.words ? p.words + ((int64_t)q * p.n_traces * p.n_blocks + bi) * 2 : nullptr;
            uint32_t* wbaseT = p.words ? p.words + ((int64_t)qT * p.n_traces * p.n_blocks + bi) * 2 : nullptr;
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                const bool live = j0 + c < p.n_traces;
                uint32_t* wout = (wbase && live) ? wbase + (int64_t)(j0 + c) * p.n_blocks * 2 : nullptr;
                if (n == 32) fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], bkey, wout);
                else fold_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], n, bi, wout);
                // TDP: level / transition counts and the cmd digest (no tune flags)
                const uint32_t mask = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
                const uint32_t cw = wcmdT[c] & mask;
                const uint32_t lw = ((wcmdT[c] >> 1) & (mask >> 1)) | (fstartT[c] << (n - 1));
                transT[c] += __popc(cw ^ lw);
                nhiT[c] += __popc(lw);
                const uint32_t wc = cw << (32 - n);
                dcT[c] += wc * (n == 32 ? bkey.x : digest_key((uint64_t)bi).x);
                if (wbaseT && live) {
                    uint32_t* wo = wbaseT + (int64_t)(j0 + c) * p.n_blocks * 2;
                    wo[0] = wc;
                    wo[1] = 0u;
                }
            }
        }
    }

#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const int j = j0 + c;
        if (j >= p.n_traces) continue;
        T::save(st[c], p, pol, 1, q, seg, j);
        add_to_chain(p, q, j, ss[c].nhi, ss[c].nthr + (uint32_t)nthrf[c], ss[c].trans, ss[c].ev,
                     ss[c].lock + (uint32_t)lockf[c] + 32u * nsb - nlk[c], ss[c].sexc, ss[c].digest());
        const int64_t si = st_idx(p, 1, qT, seg, j);
        p.st_f[si] = (uint8_t)(wcmdT[c] & 1u);
        p.st_log[si] = 0;
        const uint32_t nthr = (uint32_t)nthrT[c];
        // sum(D - B_lo) over throttled ticks, exact; no throttled tick: 0 (the open-loop mode's B_lo is +inf)
        const double sexc = nthr ? excT[c] - (double)nthr * Blo_d : 0.0;
        add_to_chain(p, qT, j, nhiT[c], nthr, transT[c], 0u, 0u, sexc, digest_pack(dcT[c], 0u));
    }
    if (j0 < p.n_traces) {
        atomicMax(p.c_vmax + chain_idx(p, q, j0), vmax);   // lane-level validation maximum
        atomicMax(p.c_vmax + chain_idx(p, qT, j0), vmax);
    }
}

}  // namespace magus
