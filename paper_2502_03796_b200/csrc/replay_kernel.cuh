// replay_kernel.cuh -- the hot kernel: batched, time-segmented replay of the MAGUS loop.
//
// Work unit of one consumer warp: 128 consecutive traces (a lane owns 4, i.e. one 16-byte float4
// per time row) x one lane policy x one time segment.  A CTA = ng tile groups x npw policy warps +
// 1 producer warp.  Each tile group has an NSTAGE-deep ring of [TC ticks x 128 traces] fp32 tiles
// in shared memory, filled by 2-D TMA (cp.async.bulk.tensor, one elected producer lane) and
// consumed by the group's policy warps (full / empty mbarriers).  Every trace byte crosses HBM
// once per launch (plus the W-tick warm-up overlap of speculative segments).
//
// Time segmentation: segment s covers ticks [s*L, min((s+1)*L, N)).  s = 0
// starts from the exact initial state; s >= 1 starts speculatively W ticks early from a guessed
// state and records the state it reaches at s*L (entry) and at its end (exit).  The fix-up kernel
// compares each entry with the previous segment's exit and re-runs exactly where they differ.
#pragma once
#include <cuda.h>
#include "device_common.cuh"
#include "ptx.cuh"
#include "tickers.cuh"

namespace magus {

constexpr int kTracesPerWarp = 128;   // 32 lanes x 4 traces (one float4 per lane per time row)
constexpr int kChains = 4;
constexpr int kMaxConsumerWarps = 8;   // 256 threads: 2 warps per SM sub-partition

template <int TC, int NSTAGE>
struct ReplaySmem {
    static constexpr int kTileFloats = TC * kTracesPerWarp;
    static constexpr int kTileBytes = kTileFloats * 4;
    __host__ __device__ static size_t bytes(int ng) {
        return (size_t)ng * NSTAGE * kTileBytes + (size_t)ng * NSTAGE * 2 * sizeof(uint64_t);
    }
};

struct SegGeom {
    int seg_start, seg_end, tau_w, n_stages;
};

template <int TC>
__device__ __forceinline__ SegGeom seg_geom(const ReplayParams& p, int seg) {
    SegGeom g;
    g.seg_start = seg_begin(p, seg);
    g.seg_end = seg_finish(p, seg);
    g.tau_w = seg == 0 ? 0 : g.seg_start - p.warmup;
    g.n_stages = (g.seg_end - g.tau_w + TC - 1) / TC;
    return g;
}

// Accumulate one tick of one chain into its segment statistics (counting region only).  The
// validation maximum (A17) is kept per lane, over its 4 chains.
__device__ __forceinline__ void acc_tick(SegStats& ss, uint32_t& vmax, const TickOut& o, float D, float B_lo) {
    ss.nthr += o.thr;
    ss.lock += o.hf;
    if (o.thr) ss.sexc += (double)D - (double)B_lo;   // exact (SegStats)
    vmax = max(vmax, __float_as_uint(D));
}

// Tile producer of one group: the group's leader lane arms full[slot] and issues the 2-D TMA box
// {128 traces, TC ticks} at (first trace of the group, tick t0).
template <int TC>
__device__ __forceinline__ void issue_stage(const CUtensorMap* tmap, float* tile, uint64_t* full_bar, int x, int t0,
                                            uint64_t cpol) {
    ptx::mbar_arrive_expect_tx(full_bar, (uint32_t)(TC * kTracesPerWarp * 4));
    ptx::tma_load_2d(tile, tmap, full_bar, x, t0, cpol);
}

// SOLO: the group has one policy warp, which consumes its own tiles -- its lane 0 refills a stage as soon
// as the warp has read it (__syncwarp orders the lanes' shared-memory reads, whose values are already in
// registers, before the refill), without the empty-barrier round trip.
template <class T, int TC, int NSTAGE, bool SOLO>
__device__ __forceinline__ void consume(const CUtensorMap* tmap, const ReplayParams& p, const DevPolicy& pol, int q,
                                        int tgroup, int seg, float* tiles, uint64_t* full, uint64_t* empty, int lane,
                                        bool producer) {
    using State = typename T::State;
    static_assert(32 % TC == 0, "a 32-tick digest block must be whole stages");
    const SegGeom G = seg_geom<TC>(p, seg);
    const int x = tgroup * kTracesPerWarp;
    constexpr uint32_t kTileBytes = TC * kTracesPerWarp * 4;
    const uint32_t tile0 = ptx::smem_u32(tiles), full0 = ptx::smem_u32(full), empty0 = ptx::smem_u32(empty);
    uint64_t cpol = 0;
    if (producer) {
        cpol = ptx::policy_evict_first();
        for (int i = 0; i < NSTAGE && i < G.n_stages; ++i)
            ptx::tma_load_2d_u32(tile0 + i * kTileBytes, tmap, full0 + 8 * i, x, G.tau_w + i * TC, kTileBytes, cpol);
    }
    ptx::pdl_wait();   // first_low and the scratch words come from the pre-pass (launched just before)
    const int j0 = tgroup * kTracesPerWarp + lane * kChains;
    const float B_lo = p.B_lo, B_hi = p.B_hi;
    const double Blo_d = (double)B_lo;
    const int k = pol.k, C = pol.C;
    const int warm_ticks = T::kWarmupRules ? k + C - 1 : 0;   // ticks before Alg. 1/2 are fully defined

    State st[kChains];
    SegStats ss[kChains];
    uint32_t wcmd[kChains], fstart[kChains];
    uint32_t vmax = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        T::init(st[c], pol, seg == 0);
        ss[c].zero();
        wcmd[c] = 0;
    }

    int i = 0;           // stage index
    int slot = 0;        // i % NSTAGE
    uint32_t phase = 0;  // (i / NSTAGE) & 1
    // 32-tick digest blocks; segment starts and warm-up starts are block aligned
    for (int bt0 = G.tau_w; bt0 < G.seg_end; bt0 += 32) {
        if (bt0 == G.seg_start) {   // the segment's own ticks start: record the entry, reset the statistics
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if (j0 + c < p.n_traces) T::save(st[c], p, pol, 0, q, seg, j0 + c);
                ss[c].zero();
            }
        }
#pragma unroll
        for (int c = 0; c < kChains; ++c) fstart[c] = T::level(st[c]);
        const bool counting = bt0 >= G.seg_start;
        for (int sub = 0; sub < 32 / TC && i < G.n_stages; ++sub) {
            const int t0 = bt0 + sub * TC;
            ptx::mbar_wait_u32(full0 + 8 * slot, phase);
            const float4* rows = reinterpret_cast<const float4*>(tiles + (size_t)slot * TC * kTracesPerWarp) + lane;
            const bool fast = (t0 - G.tau_w >= warm_ticks) && (t0 + TC <= G.seg_end);
            if (fast) {
#pragma unroll
                for (int tt = 0; tt < TC; ++tt) {
                    const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                    const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                    if constexpr (T::kHasFast4) {
                        T::fast4(st, d, pol, B_lo, Blo_d, wcmd, ss, vmax);
                    } else
#pragma unroll
                    for (int c = 0; c < kChains; ++c) {
                        if constexpr (T::kHasFast) {
                            T::fast(st[c], d[c], pol, B_lo, Blo_d, wcmd[c], ss[c], vmax);
                        } else {
                            const TickOut o = T::template tick<false>(st[c], d[c], pol, B_lo, B_hi, true, true);
                            wcmd[c] = (wcmd[c] << 1) | o.cmd;
                            acc_tick(ss[c], vmax, o, d[c], B_lo);
                        }
                    }
                }
            } else {
                if (T::kWarmupRules && i == 0 && seg > 0) {
                    // speculative level at the warm-up start: f_max iff the trace is above
                    // B_lo now and was at or below B_lo before -- a high stretch entered through a rising edge
                    // that Alg. 1 sees even at f_min; a trace never below B_lo is never seen to rise (A14).
                    const float4 d0 = rows[0];
                    const float dd[4] = {d0.x, d0.y, d0.z, d0.w};
                    // Policies whose edges always lock (k >= s_min) keep f_max after any low/high transition
                    // (post-lock stickiness, K9).
#pragma unroll
                    for (int c = 0; c < kChains; ++c) {
                        const int j = j0 + c;
                        const int fl = j < p.n_traces ? __ldg(p.first_low + j) : 0x7FFFFFFF;
                        const int fh = j < p.n_traces ? __ldg(p.first_low + p.n_traces + j) : 0x7FFFFFFF;
                        const bool hi = (dd[c] > B_lo && fl < G.tau_w) || (pol.sticky && fl < G.tau_w && fh < G.tau_w);
                        T::set_level(st[c], hi ? 1u : 0u);
                        fstart[c] = T::level(st[c]);
                    }
                }
                if (T::kHasFast4 && t0 + TC <= G.seg_end) {
                    // warm-up stage: the interleaved 4-chain tick with Alg. 1 / Alg. 2 gated per tick (A7, A8)
#pragma unroll
                    for (int tt = 0; tt < TC; ++tt) {
                        const int r = t0 + tt - G.tau_w;
                        const float4 d4 = rows[tt * (kTracesPerWarp / 4)];
                        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
                        T::warm4(st, d, pol, B_lo, Blo_d, wcmd, ss, vmax, r >= k ? 1u : 0u,
                                 r >= k + C - 1 ? 1u : 0u);
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
                            acc_tick(ss[c], vmax, o, d[c], B_lo);
                        }
                    }
                }
            }
            // release the stage; the group's producer lane refills it with stage i + NSTAGE once every
            // policy warp of the group has released it
            __syncwarp();
            if constexpr (SOLO) {
                if (producer && i + NSTAGE < G.n_stages)
                    ptx::tma_load_2d_u32(tile0 + slot * kTileBytes, tmap, full0 + 8 * slot, x,
                                         G.tau_w + (i + NSTAGE) * TC, kTileBytes, cpol);
            } else {
                if (lane == 0) ptx::mbar_arrive_u32(empty0 + 8 * slot);
                if (producer && i + NSTAGE < G.n_stages) {
                    ptx::mbar_wait_u32(empty0 + 8 * slot, phase);
                    ptx::tma_load_2d_u32(tile0 + slot * kTileBytes, tmap, full0 + 8 * slot, x,
                                         G.tau_w + (i + NSTAGE) * TC, kTileBytes, cpol);
                }
            }
            ++i;
            if (++slot == NSTAGE) {
                slot = 0;
                phase ^= 1u;
            }
        }
        if (counting) {
            const uint2 bkey = p.dkeys[bt0 >> 5];
            const int n = min(32, G.seg_end - bt0);
            if (n == 32 && p.words == nullptr) {   // the common case: a whole block, no word dump
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    uint32_t ew;
                    if constexpr (T::kWarmupRules) ew = (uint32_t)st[c].evh;
                    else ew = 0u;
                    fold_full_block(ss[c], wcmd[c], ew, fstart[c], bkey, nullptr);
                }
            } else {
                const int64_t b = bt0 >> 5;
                uint32_t* wbase = p.words ? p.words + ((int64_t)q * p.n_traces * p.n_blocks + b) * 2 : nullptr;
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    uint32_t ew;
                    if constexpr (T::kWarmupRules) ew = (uint32_t)st[c].evh;
                    else ew = 0u;
                    uint32_t* wout =
                        (wbase && j0 + c < p.n_traces) ? wbase + (int64_t)(j0 + c) * p.n_blocks * 2 : nullptr;
                    if (n == 32) fold_full_block(ss[c], wcmd[c], ew, fstart[c], bkey, wout);
                    else fold_block(ss[c], wcmd[c], ew, fstart[c], n, b, wout);
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
        add_to_chain(p, q, j, ss[c].nhi, ss[c].nthr, ss[c].trans, ss[c].ev, ss[c].lock, ss[c].sexc,
                     ss[c].digest());
    }
    if (j0 < p.n_traces) atomicMax(p.c_vmax + chain_idx(p, q, j0), vmax);   // lane-level validation maximum
}

// One kernel per chain kind T (register allocation is per instantiation): a launch covers the lane
// policies [p.q_base, p.q_base + p.nq), all of kind T.  CTA = ng tile groups x npw policy warps
// (<= 8 warps = 2 per SM sub-partition, so up to 255 registers per thread); lane 0 of each group's
// first warp produces that group's tiles.
// MINB = CTAs per SM the register budget is sized for: 2 (<= 128 registers, 16 warps per SM) for the
// small-state chain kinds, 1 (<= 255 registers) for large rings / 64-bit logs, which would spill.
template <class T, int TC, int NSTAGE, int MINB>
__global__ void __launch_bounds__(kMaxConsumerWarps * 32, MINB)
    magus_replay_kernel(const __grid_constant__ CUtensorMap tmap, const ReplayParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    using SM = ReplaySmem<TC, NSTAGE>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    int b = blockIdx.x;
    const int pblock = b % p.n_pblocks;
    b /= p.n_pblocks;
    const int tblock = b % p.n_tblocks;
    const int seg = b / p.n_tblocks;

    float* tiles = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.ng * NSTAGE * SM::kTileBytes);
    uint64_t* empty = full + p.ng * NSTAGE;
    const int npw_active = min(p.npw, p.nq - pblock * p.npw);

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmap);
        for (int i = 0; i < p.ng * NSTAGE; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], (uint32_t)npw_active);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    const int g = warp / p.npw, w = warp % p.npw;
    const int tgroup = tblock * p.ng + g;
    if (g >= p.ng || tgroup >= p.n_groups || w >= npw_active) return;
    const int q = p.q_base + pblock * p.npw + w;
    const DevPolicy pol = p.pol[q];
    float* gt = tiles + (size_t)g * NSTAGE * SM::kTileFloats;
    if (npw_active == 1)
        consume<T, TC, NSTAGE, true>(&tmap, p, pol, q, tgroup, seg, gt, &full[g * NSTAGE], &empty[g * NSTAGE], lane,
                                     lane == 0);
    else
        consume<T, TC, NSTAGE, false>(&tmap, p, pol, q, tgroup, seg, gt, &full[g * NSTAGE], &empty[g * NSTAGE], lane,
                                      w == 0 && lane == 0);
}

}  // namespace magus
