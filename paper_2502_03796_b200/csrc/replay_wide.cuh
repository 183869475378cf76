// replay_wide.cuh -- the unsegmented replay for runs with many (trace, policy) chains: the parameter sweeps
// (config 3: 1,024 traces x 64 policy points = 65,536 MAGUS chains).  DESIGN.md section 9a.
//
// A sweep already has enough independent recurrences to fill the GPU with ONE chain per lane, so the trace is
// not cut into time segments: every chain runs from its exact initial state (A10) over all of its
// samples.  There is no speculative warm-up, no stored segment state and no fix-up chain walk -- the walk is
// what a segmented sweep pays for the chains whose speculative entries never coalesce with the true state
// (even-k aliasing on spike traces, phase-shifted limit cycles of oscillating ones).
//
// A CTA is 8 warps: 16 traces x 16 policy points of one chain kind (thread = 16 * trace + point), sharing a ring of
// [32 ticks x 16 traces] TMA tiles (64-byte box rows: a TMA box costs per row, and 16-byte rows made the TMA the
// bottleneck -- profiles/r02_wide_tma.txt).  The tile is read by the ceil(nq / 16) CTAs of each column, from L2.
// Warp 0's elected lane is the producer: it refills a stage once all 8 warps have released it (empty mbarrier).
// Per 8 ticks a lane runs the generated one-chain stage block (MAGUS_WSTAGE1F_K<K>, tick4_asm.cuh -- the same
// block as the split chain walk's); the first k + C - 1 ticks (Alg. 1 / Alg. 2 not yet defined, A7 / A8) and a
// ragged last block use the per-tick path.
#pragma once
#include <cuda.h>
#include "device_common.cuh"
#include "ptx.cuh"
#include "replay_kernel.cuh"
#include "replay_solo.cuh"
#include "tickers.cuh"

namespace magus {

constexpr int kWidePpc = 16;                  // policy points per CTA
constexpr int kWideTpc = 16;                  // traces per CTA: one 64-byte TMA box row
constexpr int kWideThreads = kWidePpc * kWideTpc;   // 256: 8 warps, one chain per thread
constexpr int kWideWarps = kWideThreads / 32;
constexpr int kWideTC = 32;                   // ticks per TMA stage = one 32-tick digest block
constexpr int kWideNStage = 6;

struct WideSmem {
    static constexpr int kTileBytes = kWideTC * kWideTpc * 4;   // 2 KB
    // + one fp64 scratch per warp: its 2 traces x 32 ticks, converted once per stage (one chain per thread)
    // (x 2 for the P stage: D and min(D, B_lo) per sample)
    static constexpr int kWarpBufBytes = 2 * 2 * kWideTC * 8;   // 1 KB
    static constexpr size_t kBarOff = (size_t)kWideNStage * kTileBytes;
    static constexpr size_t kBufOff = kBarOff + 2 * kWideNStage * sizeof(uint64_t);
    static constexpr size_t kBytes = kBufOff + (size_t)kWideWarps * kWarpBufBytes;
};

// the elected lane arms `bar` for one tile and issues the 2-D TMA box {16 traces, 32 ticks} at (x, t0); no L2
// eviction hint: the tile is read again by the other policy blocks of the column
__device__ __forceinline__ void wide_issue(uint32_t tile, const CUtensorMap* tmap, uint32_t bar, int x, int t0) {
    MAGUS_CHECK(smem_range_ok(tile, WideSmem::kTileBytes) && smem_range_ok(bar, 8) && x >= 0 && t0 >= 0);
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%2], [%3, {%4, %5}], [%0];\n\t}" ::"r"(bar),
        "n"(WideSmem::kTileBytes), "r"(tile), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(t0)
        : "memory");
}

// 8 ticks of one chain (samples in registers) by the generated one-chain stage block
template <int K>
__device__ __forceinline__ void wide_stage(MagusState<K, false>& st, float& lock, float& nthr, uint32_t& wcmd,
                                           double& sexc, const float* d8, const DevPolicy& pol, float B_lo,
                                           double Blo_d, uint32_t bitc, uint32_t mone) {
    uint32_t e0 = st.evh;
#define WD_TAIL                                                                                                  \
    e0, st.cnt, sexc, lock, nthr, wcmd, __float_as_uint(d8[0]), __float_as_uint(d8[1]), __float_as_uint(d8[2]),    \
        __float_as_uint(d8[3]), __float_as_uint(d8[4]), __float_as_uint(d8[5]), __float_as_uint(d8[6]),             \
        __float_as_uint(d8[7]), B_lo, Blo_d, pol.dinc, pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define R(i) st.ring.v[i]
    if constexpr (K == 1) MAGUS_WSTAGE1F_K1(st.f, R(0), WD_TAIL);
    else if constexpr (K == 2) MAGUS_WSTAGE1F_K2(st.f, R(0), R(1), WD_TAIL);
    else if constexpr (K == 3) MAGUS_WSTAGE1F_K3(st.f, R(0), R(1), R(2), WD_TAIL);
    else if constexpr (K == 4) MAGUS_WSTAGE1F_K4(st.f, R(0), R(1), R(2), R(3), WD_TAIL);
    else if constexpr (K == 5) MAGUS_WSTAGE1F_K5(st.f, R(0), R(1), R(2), R(3), R(4), WD_TAIL);
    else if constexpr (K == 6) MAGUS_WSTAGE1F_K6(st.f, R(0), R(1), R(2), R(3), R(4), R(5), WD_TAIL);
    else if constexpr (K == 7) MAGUS_WSTAGE1F_K7(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), WD_TAIL);
    else MAGUS_WSTAGE1F_K8(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), WD_TAIL);
#undef R
#undef WD_TAIL
    st.evh = e0;
}

// 8 ticks of one chain with the samples as fp64 values and the L-stage bookkeeping (MAGUS_WLSTAGE[S]_K<K>): the
// level in wcmd's bit 0, st.cnt biased by -smin_sc (the caller converts around the block), nlk = ticks not locked
template <int K, bool SYM>
__device__ __forceinline__ void wide_stage_l(MagusState<K, false>& st, uint32_t& nlk, float& nthr, uint32_t& wcmd,
                                             double& sexc, const double* d8, const DevPolicy& pol, double Blo_d,
                                             uint32_t bitc, uint32_t mone) {
    uint32_t e0 = st.evh;
#define WDL_TAIL                                                                                                 \
    e0, st.cnt, sexc, nlk, nthr, wcmd, d8[0], d8[1], d8[2], d8[3], d8[4], d8[5], d8[6], d8[7], Blo_d, pol.dinc,     \
        pol.ddec, bitc, pol.one, mone
#define R(i) st.ring.v[i]
#define WDL(NAME)                                                                                                \
    if constexpr (K == 1) NAME##_K1(R(0), WDL_TAIL);                                                               \
    else if constexpr (K == 2) NAME##_K2(R(0), R(1), WDL_TAIL);                                                    \
    else if constexpr (K == 3) NAME##_K3(R(0), R(1), R(2), WDL_TAIL);                                              \
    else if constexpr (K == 4) NAME##_K4(R(0), R(1), R(2), R(3), WDL_TAIL);                                        \
    else if constexpr (K == 5) NAME##_K5(R(0), R(1), R(2), R(3), R(4), WDL_TAIL);                                  \
    else if constexpr (K == 6) NAME##_K6(R(0), R(1), R(2), R(3), R(4), R(5), WDL_TAIL);                            \
    else if constexpr (K == 7) NAME##_K7(R(0), R(1), R(2), R(3), R(4), R(5), R(6), WDL_TAIL);                      \
    else NAME##_K8(R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), WDL_TAIL);
    if constexpr (SYM) {
        WDL(MAGUS_WLSTAGES)
    } else {
        WDL(MAGUS_WLSTAGE)
    }
#undef WDL
#undef R
#undef WDL_TAIL
    st.evh = e0;
}

// 8 ticks of one chain from the warp's scratch: D and min(D, B_lo) as fp64 (MAGUS_WPSTAGE[S]_K<K>: the L stage with
// A selected by the level itself; the throttled ticks are counted per block from a ballot word)
template <int K, bool SYM>
__device__ __forceinline__ void wide_stage_p(MagusState<K, false>& st, uint32_t& nlk, uint32_t& wcmd, double& sexc,
                                             const double* d8, const double* l8, const DevPolicy& pol, uint32_t bitc,
                                             uint32_t mone) {
    uint32_t e0 = st.evh;
#define WDP_TAIL                                                                                                 \
    e0, st.cnt, sexc, nlk, wcmd, d8[0], d8[1], d8[2], d8[3], d8[4], d8[5], d8[6], d8[7], l8[0], l8[1], l8[2], l8[3], \
        l8[4], l8[5], l8[6], l8[7], pol.dinc, pol.ddec, bitc, pol.one, mone
#define R(i) st.ring.v[i]
#define WDP(NAME)                                                                                                \
    if constexpr (K == 1) NAME##_K1(R(0), WDP_TAIL);                                                               \
    else if constexpr (K == 2) NAME##_K2(R(0), R(1), WDP_TAIL);                                                    \
    else if constexpr (K == 3) NAME##_K3(R(0), R(1), R(2), WDP_TAIL);                                              \
    else if constexpr (K == 4) NAME##_K4(R(0), R(1), R(2), R(3), WDP_TAIL);                                        \
    else if constexpr (K == 5) NAME##_K5(R(0), R(1), R(2), R(3), R(4), WDP_TAIL);                                  \
    else if constexpr (K == 6) NAME##_K6(R(0), R(1), R(2), R(3), R(4), R(5), WDP_TAIL);                            \
    else if constexpr (K == 7) NAME##_K7(R(0), R(1), R(2), R(3), R(4), R(5), R(6), WDP_TAIL);                      \
    else NAME##_K8(R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), WDP_TAIL);
    if constexpr (SYM) {
        WDP(MAGUS_WPSTAGES)
    } else {
        WDP(MAGUS_WPSTAGE)
    }
#undef WDP
#undef R
#undef WDP_TAIL
    st.evh = e0;
}

// 8 ticks of one chain with the samples as fp64 values (MAGUS_WSTAGE1D_K<K>: no conversion, fp64 throttle test)
template <int K>
__device__ __forceinline__ void wide_stage_d(MagusState<K, false>& st, float& lock, float& nthr, uint32_t& wcmd,
                                             double& sexc, const double* d8, const DevPolicy& pol, double Blo_d,
                                             uint32_t bitc, uint32_t mone) {
    uint32_t e0 = st.evh;
#define WDD_TAIL                                                                                                 \
    e0, st.cnt, sexc, lock, nthr, wcmd, d8[0], d8[1], d8[2], d8[3], d8[4], d8[5], d8[6], d8[7], Blo_d, pol.dinc,    \
        pol.ddec, bitc, pol.smin_sc, pol.one, mone
#define R(i) st.ring.v[i]
    if constexpr (K == 1) MAGUS_WSTAGE1D_K1(st.f, R(0), WDD_TAIL);
    else if constexpr (K == 2) MAGUS_WSTAGE1D_K2(st.f, R(0), R(1), WDD_TAIL);
    else if constexpr (K == 3) MAGUS_WSTAGE1D_K3(st.f, R(0), R(1), R(2), WDD_TAIL);
    else if constexpr (K == 4) MAGUS_WSTAGE1D_K4(st.f, R(0), R(1), R(2), R(3), WDD_TAIL);
    else if constexpr (K == 5) MAGUS_WSTAGE1D_K5(st.f, R(0), R(1), R(2), R(3), R(4), WDD_TAIL);
    else if constexpr (K == 6) MAGUS_WSTAGE1D_K6(st.f, R(0), R(1), R(2), R(3), R(4), R(5), WDD_TAIL);
    else if constexpr (K == 7) MAGUS_WSTAGE1D_K7(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), WDD_TAIL);
    else MAGUS_WSTAGE1D_K8(st.f, R(0), R(1), R(2), R(3), R(4), R(5), R(6), R(7), WDD_TAIL);
#undef R
#undef WDD_TAIL
    st.evh = e0;
}

// 8 ticks of two chains of one trace (two policy points) sharing the samples (MAGUS_WSTAGE2P_K<K>)
template <int K>
__device__ __forceinline__ void wide_stage2(MagusState<K, false>* st, float* lock, float* nthr, uint32_t* wcmd,
                                            double* sexc, const float* d8, const DevPolicy* pol, float B_lo,
                                            double Blo_d, const uint32_t* bitc, uint32_t mone) {
    uint32_t e0 = st[0].evh, e1 = st[1].evh;
#define WD2_TAIL                                                                                                 \
    e0, e1, st[0].cnt, st[1].cnt, sexc[0], sexc[1], lock[0], lock[1], nthr[0], nthr[1], wcmd[0], wcmd[1],         \
        __float_as_uint(d8[0]), __float_as_uint(d8[1]), __float_as_uint(d8[2]), __float_as_uint(d8[3]),             \
        __float_as_uint(d8[4]), __float_as_uint(d8[5]), __float_as_uint(d8[6]), __float_as_uint(d8[7]), B_lo,      \
        Blo_d, pol[0].dinc, pol[1].dinc, pol[0].ddec, pol[1].ddec, bitc[0], bitc[1], pol[0].smin_sc, pol[1].smin_sc, \
        pol[0].one, mone
#define R0(i) st[0].ring.v[i]
#define R1(i) st[1].ring.v[i]
    if constexpr (K == 1) MAGUS_WSTAGE2P_K1(st[0].f, st[1].f, R0(0), R1(0), WD2_TAIL);
    else if constexpr (K == 2) MAGUS_WSTAGE2P_K2(st[0].f, st[1].f, R0(0), R0(1), R1(0), R1(1), WD2_TAIL);
    else if constexpr (K == 3) MAGUS_WSTAGE2P_K3(st[0].f, st[1].f, R0(0), R0(1), R0(2), R1(0), R1(1), R1(2), WD2_TAIL);
    else if constexpr (K == 4)
        MAGUS_WSTAGE2P_K4(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R1(0), R1(1), R1(2), R1(3), WD2_TAIL);
    else if constexpr (K == 5)
        MAGUS_WSTAGE2P_K5(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R1(0), R1(1), R1(2), R1(3), R1(4),
                          WD2_TAIL);
    else if constexpr (K == 6)
        MAGUS_WSTAGE2P_K6(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R1(0), R1(1), R1(2), R1(3),
                          R1(4), R1(5), WD2_TAIL);
    else if constexpr (K == 7)
        MAGUS_WSTAGE2P_K7(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R0(6), R1(0), R1(1), R1(2),
                          R1(3), R1(4), R1(5), R1(6), WD2_TAIL);
    else
        MAGUS_WSTAGE2P_K8(st[0].f, st[1].f, R0(0), R0(1), R0(2), R0(3), R0(4), R0(5), R0(6), R0(7), R1(0), R1(1),
                          R1(2), R1(3), R1(4), R1(5), R1(6), R1(7), WD2_TAIL);
#undef R0
#undef R1
#undef WD2_TAIL
    st[0].evh = e0;
    st[1].evh = e1;
}

// MAGUS chains with a register ring of K <= 8 values and a 32-bit tune log (C <= 28).  NC = chains per thread: 1, or
// 2 = two policy points of the same trace sharing the samples (one shared-memory load, fp32 -> fp64 conversion and
// validation maximum per tick for both).  Launch: one (256 / NC)-thread CTA per (16-trace column, block of 16 policy
// points), policy blocks fastest; p.n_pblocks = ceil(nq / 16).  LV (NC = 1 only): 0 = the one-chain stage block
// MAGUS_WSTAGE1D_K<K>, 1 = its L form (MAGUS_WLSTAGE_K<K>: C <= 27), 2 = the L form with the |d| tune-flag test
// (every lane policy has d*_dec == -d*_inc), 3 / 4 = the P form without / with the |d| test (MAGUS_WPSTAGE[S]_K<K>:
// the warp's scratch also holds min(D, B_lo), the throttled ticks come from a ballot word per block).
template <int K, int NC, int LV>
__global__ void __launch_bounds__(kWideThreads / NC, 2)
    magus_replay_wide_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    static_assert(NC == 1 || NC == 2, "wide kernel: one or two chains per thread");
    static_assert(LV == 0 || NC == 1, "wide kernel: the L stage runs one chain per thread");
    using T = MagusTicker<K, false>;
    constexpr uint32_t kTileBytes = WideSmem::kTileBytes;
    constexpr int kPerTrace = kWidePpc / NC;   // threads per trace
    const int kWarps = (int)(blockDim.x >> 5);   // (p.wide_tpcu traces x 16 points) / NC threads
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pb = blockIdx.x % p.n_pblocks;
    // the CTA's p.wide_tpcu traces start at x; its 16-trace TMA box at xbox = x rounded down to 4 traces (16-byte
    // aligned rows), the CTA's traces at columns [xoff, xoff + tpcu) of it (tpcu <= 14 when xoff = 2; the other
    // columns are read and not replayed -- the chains per SM then balance)
    const int x = (blockIdx.x / p.n_pblocks) * p.wide_tpcu;
    const int xbox = x & ~3, xoff = x - xbox;
    const int jl = tid / kPerTrace;
    const int j = x + jl;
    int q[NC];
    bool live[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int qi = pb * kWidePpc + (tid % kPerTrace) * NC + c;
        live[c] = qi < p.nq && j < p.n_traces;
        q[c] = p.q_base + (qi < p.nq ? qi : p.nq - 1);   // idle chains replay a live point, unrecorded
    }

    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t full0 = tile0 + (uint32_t)WideSmem::kBarOff, empty0 = full0 + 8 * kWideNStage;
    double* wbuf = reinterpret_cast<double*>(smem + WideSmem::kBufOff) + warp * (WideSmem::kWarpBufBytes / 8);   // this warp's
    const int N = p.n_samples;
    const int n_st = (N + kWideTC - 1) / kWideTC;
    if (warp == 0) {
        if (lane == 0) {
            ptx::prefetch_tmap(&tmap);
            for (int i = 0; i < kWideNStage; ++i) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * i) : "memory");
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * i), "r"(kWarps) : "memory");
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        for (int i = 0; i < kWideNStage && i < n_st; ++i)
            wide_issue(tile0 + i * kTileBytes, &tmap, full0 + 8 * i, xbox, i * kWideTC);
    }
    __syncthreads();   // the barriers are initialised before any warp waits on them
    ptx::pdl_wait();   // the pre-pass zeroes the run's flag words (launched just before)

    DevPolicy pol[NC];
    uint32_t bitc[NC];
    typename T::State st[NC];
    SegStats ss[NC];
    float lockf[NC], nthrf[NC];   // per-block counts from the stage block (exact fp32 integers <= 32)
    int warm = 0;                 // ticks before Alg. 1 / Alg. 2 are defined for every chain (A7, A8): per-tick path
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        pol[c] = p.pol[q[c]];
        bitc[c] = 1u << (pol[c].C - 1);
        warm = max(warm, pol[c].k + pol[c].C - 1);
        T::init(st[c], pol[c], true);   // the exact initial state (A10): no speculation
        ss[c].zero();
        lockf[c] = nthrf[c] = 0.f;
    }
    // warp-uniform: the steady branch converts the warp's tile columns with all 32 lanes (and __syncwarp()s), so a
    // warp whose lanes' policies differ in k + C - 1 takes the per-tick path until the longest warm-up is over
    warm = __reduce_max_sync(0xffffffffu, warm);
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    const double Blo_d = (double)B_lo;
    const uint32_t mone = 0xFFFFFFFFu * pol[0].one;
    uint32_t vmax = 0;
    int slot = 0;
    uint32_t phase = 0;
#pragma unroll 1
    for (int i = 0; i < n_st; ++i) {
        const int bt0 = i * kWideTC;
        const int n = min(kWideTC, N - bt0);
        mbar_wait_loop(full0 + 8 * slot, phase);
        const float* colp = reinterpret_cast<const float*>(smem + slot * kTileBytes) + xoff + jl;   // stride 16
        uint32_t fstart[NC], wcmd[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            fstart[c] = T::level(st[c]);
            wcmd[c] = 0;
        }
        // release the stage; warp 0 refills it with stage i + NSTAGE once all warps have released it
        auto release = [&]() {
            if (lane == 0) ptx::mbar_arrive_u32(empty0 + 8 * slot);
            if (warp == 0 && i + kWideNStage < n_st) {
                ptx::mbar_wait_u32(empty0 + 8 * slot, phase);
                wide_issue(tile0 + slot * kTileBytes, &tmap, full0 + 8 * slot, xbox, (i + kWideNStage) * kWideTC);
            }
        };
        if (NC == 1 && n == kWideTC && bt0 >= warm) {
            // the warp converts its 2 traces' 32 samples to fp64 once (lane = tick) and validates them (A17), then
            // releases the fp32 slot; each thread reads its trace's values from the warp's scratch
            const float2 v = *reinterpret_cast<const float2*>(smem + slot * kTileBytes + lane * (kWideTpc * 4) +
                                                             (xoff + (tid >> 4 & ~1)) * 4);
            vmax = max(vmax, max(__float_as_uint(v.x), __float_as_uint(v.y)));
            MAGUS_CHECK(smem_range_ok(ptx::smem_u32(wbuf), WideSmem::kWarpBufBytes) && xoff + p.wide_tpcu <= kWideTpc &&
                        smem_range_ok(ptx::smem_u32(smem + slot * kTileBytes + lane * (kWideTpc * 4) +
                                                    (xoff + (tid >> 4 & ~1)) * 4), 8));
            wbuf[lane] = (double)v.x;
            wbuf[kWideTC + lane] = (double)v.y;
            uint32_t over = 0;   // LV >= 3: bit i = tick i of this thread's trace has D > B_lo
            if constexpr (LV >= 3) {
                wbuf[2 * kWideTC + lane] = fmin((double)v.x, Blo_d);   // A at f_min (A14; exact)
                wbuf[3 * kWideTC + lane] = fmin((double)v.y, Blo_d);
                const uint32_t o0 = __ballot_sync(0xffffffffu, v.x > B_lo);
                const uint32_t o1 = __ballot_sync(0xffffffffu, v.y > B_lo);
                over = ((tid >> 4) & 1) ? o1 : o0;
            }
            __syncwarp();
            release();
            const double* my = wbuf + ((tid >> 4) & 1) * kWideTC;
            if constexpr (LV >= 3) {
                uint32_t nlk = 0;
                st[0].cnt -= pol[0].smin_sc;   // biased: lock iff cnt >= 0
                wcmd[0] = fstart[0];           // bit 0 = the level
#pragma unroll
                for (int g = 0; g < kWideTC / 8; ++g) {
                    double d8[8], l8[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        d8[t] = my[8 * g + t];
                        l8[t] = my[2 * kWideTC + 8 * g + t];
                    }
                    wide_stage_p<K, LV == 4>(st[0], nlk, wcmd[0], ss[0].sexc, d8, l8, pol[0], bitc[0], mone);
                }
                st[0].cnt += pol[0].smin_sc;
                T::set_level(st[0], wcmd[0] & 1u);
                lockf[0] = (float)(kWideTC - nlk);
                // throttled ticks: f_min (the level word, tick i at bit 31 - i) and D > B_lo (the ballot, tick i at bit i)
                const uint32_t lw = (wcmd[0] >> 1) | (fstart[0] << 31);
                nthrf[0] = (float)__popc(~lw & __brev(over));
            } else if constexpr (LV != 0) {
                uint32_t nlk = 0;
                st[0].cnt -= pol[0].smin_sc;   // biased: lock iff cnt >= 0
                wcmd[0] = fstart[0];           // bit 0 = the level
#pragma unroll
                for (int g = 0; g < kWideTC / 8; ++g) {
                    double d8[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) d8[t] = my[8 * g + t];
                    wide_stage_l<K, LV == 2>(st[0], nlk, nthrf[0], wcmd[0], ss[0].sexc, d8, pol[0], Blo_d, bitc[0],
                                             mone);
                }
                st[0].cnt += pol[0].smin_sc;
                T::set_level(st[0], wcmd[0] & 1u);
                lockf[0] = (float)(kWideTC - nlk);
            } else {
#pragma unroll
                for (int g = 0; g < kWideTC / 8; ++g) {
                    double d8[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) d8[t] = my[8 * g + t];
                    wide_stage_d<K>(st[0], lockf[0], nthrf[0], wcmd[0], ss[0].sexc, d8, pol[0], Blo_d, bitc[0], mone);
                }
            }
            __syncwarp();   // every lane has read the scratch before the next stage overwrites it
        } else if (n == kWideTC && bt0 >= warm) {
#pragma unroll
            for (int g = 0; g < kWideTC / 8; ++g) {
                float d8[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) d8[t] = colp[(8 * g + t) * kWideTpc];
                vmax = max(vmax, max(max(max(__float_as_uint(d8[0]), __float_as_uint(d8[1])),
                                         max(__float_as_uint(d8[2]), __float_as_uint(d8[3]))),
                                     max(max(__float_as_uint(d8[4]), __float_as_uint(d8[5])),
                                         max(__float_as_uint(d8[6]), __float_as_uint(d8[7])))));
                if constexpr (NC == 1)
                    wide_stage<K>(st[0], lockf[0], nthrf[0], wcmd[0], ss[0].sexc, d8, pol[0], B_lo, Blo_d, bitc[0], mone);
                else {
                    double sx[2] = {ss[0].sexc, ss[1].sexc};
                    wide_stage2<K>(st, lockf, nthrf, wcmd, sx, d8, pol, B_lo, Blo_d, bitc, mone);
                    ss[0].sexc = sx[0];
                    ss[1].sexc = sx[1];
                }
            }
            __syncwarp();
            release();
        } else {
            // warm-up block (Alg. 1 / Alg. 2 gated per tick) or the ragged last block of the trace
#pragma unroll 1
            for (int tt = 0; tt < n; ++tt) {
                const float D = colp[tt * kWideTpc];
                const int t = bt0 + tt;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const TickOut o = T::template tick<true>(st[c], D, pol[c], B_lo, B_hi, t >= pol[c].k,
                                                             t >= pol[c].k + pol[c].C - 1);
                    wcmd[c] = (wcmd[c] << 1) | o.cmd;
                    acc_tick(ss[c], vmax, o, D, B_lo);
                }
            }
            __syncwarp();
            release();
        }
        if (++slot == kWideNStage) {
            slot = 0;
            phase ^= 1u;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            ss[c].lock += (uint32_t)lockf[c];
            ss[c].nthr += (uint32_t)nthrf[c];
            lockf[c] = nthrf[c] = 0.f;
            uint32_t* wout =
                (p.words && live[c]) ? p.words + ((int64_t)chain_idx(p, q[c], j) * p.n_blocks + i) * 2 : nullptr;
            if (n == kWideTC) fold_full_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], p.dkeys[i], wout);
            else fold_block(ss[c], wcmd[c], (uint32_t)st[c].evh, fstart[c], n, i, wout);
        }
    }
    // the validation maximum covers the warp's traces (the converting lanes saw both of its traces' samples); the
    // precise first invalid (trace, tick) comes from magus_scan_invalid_kernel when any maximum is out of range
    vmax = __reduce_max_sync(0xffffffffu, vmax);
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if (live[c]) {
            add_to_chain(p, q[c], j, ss[c].nhi, ss[c].nthr, ss[c].trans, ss[c].ev, ss[c].lock, ss[c].sexc,
                         ss[c].digest());
            atomicMax(p.c_vmax + chain_idx(p, q[c], j), vmax);
        }
}

}  // namespace magus
