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
    static constexpr size_t kBytes = (size_t)kWideNStage * kTileBytes + 2 * kWideNStage * sizeof(uint64_t);
};

// the elected lane arms `bar` for one tile and issues the 2-D TMA box {16 traces, 32 ticks} at (x, t0); no L2
// eviction hint: the tile is read again by the other policy blocks of the column
__device__ __forceinline__ void wide_issue(uint32_t tile, const CUtensorMap* tmap, uint32_t bar, int x, int t0) {
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

// MAGUS chains with a register ring of K <= 8 values and a 32-bit tune log (C <= 28).  Launch: one 256-thread CTA
// per (16-trace column, block of 16 policy points), policy blocks fastest; p.n_pblocks = ceil(nq / 16).
template <int K>
__global__ void __launch_bounds__(kWideThreads, 2)
    magus_replay_wide_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    using T = MagusTicker<K, false>;
    constexpr uint32_t kTileBytes = WideSmem::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pb = blockIdx.x % p.n_pblocks;
    const int x = (blockIdx.x / p.n_pblocks) * kWideTpc;
    const int qi = pb * kWidePpc + (tid % kWidePpc);
    const int jl = tid / kWidePpc;
    const int j = x + jl;
    const bool live = qi < p.nq && j < p.n_traces;
    const int q = p.q_base + (qi < p.nq ? qi : p.nq - 1);   // idle lanes replay a live point, unrecorded

    const uint32_t tile0 = ptx::smem_u32(smem);
    const uint32_t full0 = tile0 + kWideNStage * kTileBytes, empty0 = full0 + 8 * kWideNStage;
    const int N = p.n_samples;
    const int n_st = (N + kWideTC - 1) / kWideTC;
    if (warp == 0) {
        if (lane == 0) {
            ptx::prefetch_tmap(&tmap);
            for (int i = 0; i < kWideNStage; ++i) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * i) : "memory");
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * i), "r"(kWideWarps) : "memory");
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        for (int i = 0; i < kWideNStage && i < n_st; ++i)
            wide_issue(tile0 + i * kTileBytes, &tmap, full0 + 8 * i, x, i * kWideTC);
    }
    __syncthreads();   // the barriers are initialised before any warp waits on them
    ptx::pdl_wait();   // the pre-pass zeroes the run's flag words (launched just before)

    const DevPolicy pol = p.pol[q];
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    const double Blo_d = (double)B_lo;
    const uint32_t bitc = 1u << (pol.C - 1), mone = 0xFFFFFFFFu * pol.one;
    const int k = pol.k, C = pol.C;
    const int warm = k + C - 1;   // ticks before Alg. 1 / Alg. 2 are both defined (A7, A8): per-tick path

    typename T::State st;
    T::init(st, pol, true);   // the exact initial state (A10): no speculation
    SegStats ss;
    ss.zero();
    float lockf = 0.f, nthrf = 0.f;   // per-block counts from the stage block (exact fp32 integers <= 32)
    uint32_t vmax = 0;
    int slot = 0;
    uint32_t phase = 0;
#pragma unroll 1
    for (int i = 0; i < n_st; ++i) {
        const int bt0 = i * kWideTC;
        const int n = min(kWideTC, N - bt0);
        mbar_wait_loop(full0 + 8 * slot, phase);
        const float* colp = reinterpret_cast<const float*>(smem + slot * kTileBytes) + jl;   // stride 16 floats
        const uint32_t fstart = T::level(st);
        uint32_t wcmd = 0;
        if (n == kWideTC && bt0 >= warm) {
#pragma unroll
            for (int g = 0; g < kWideTC / 8; ++g) {
                float d8[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) d8[t] = colp[(8 * g + t) * kWideTpc];
                vmax = max(vmax, max(max(max(__float_as_uint(d8[0]), __float_as_uint(d8[1])),
                                         max(__float_as_uint(d8[2]), __float_as_uint(d8[3]))),
                                     max(max(__float_as_uint(d8[4]), __float_as_uint(d8[5])),
                                         max(__float_as_uint(d8[6]), __float_as_uint(d8[7])))));
                wide_stage<K>(st, lockf, nthrf, wcmd, ss.sexc, d8, pol, B_lo, Blo_d, bitc, mone);
            }
        } else {
            // warm-up block (Alg. 1 / Alg. 2 gated per tick) or the ragged last block of the trace
#pragma unroll 1
            for (int tt = 0; tt < n; ++tt) {
                const float D = colp[tt * kWideTpc];
                const int t = bt0 + tt;
                const TickOut o = T::template tick<true>(st, D, pol, B_lo, B_hi, t >= k, t >= warm);
                wcmd = (wcmd << 1) | o.cmd;
                acc_tick(ss, vmax, o, D, B_lo);
            }
        }
        // release the stage; warp 0 refills it with stage i + NSTAGE once all warps have released it
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_u32(empty0 + 8 * slot);
        if (warp == 0 && i + kWideNStage < n_st) {
            ptx::mbar_wait_u32(empty0 + 8 * slot, phase);
            wide_issue(tile0 + slot * kTileBytes, &tmap, full0 + 8 * slot, x, (i + kWideNStage) * kWideTC);
        }
        if (++slot == kWideNStage) {
            slot = 0;
            phase ^= 1u;
        }
        ss.lock += (uint32_t)lockf;
        ss.nthr += (uint32_t)nthrf;
        lockf = nthrf = 0.f;
        uint32_t* wout = (p.words && live) ? p.words + ((int64_t)chain_idx(p, q, j) * p.n_blocks + i) * 2 : nullptr;
        if (n == kWideTC) fold_full_block(ss, wcmd, (uint32_t)st.evh, fstart, p.dkeys[i], wout);
        else fold_block(ss, wcmd, (uint32_t)st.evh, fstart, n, i, wout);
    }
    if (live) {
        add_to_chain(p, q, j, ss.nhi, ss.nthr, ss.trans, ss.ev, ss.lock, ss.sexc, ss.digest());
        atomicMax(p.c_vmax + chain_idx(p, q, j), vmax);
    }
}

}  // namespace magus
