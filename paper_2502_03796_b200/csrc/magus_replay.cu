// magus_replay.cu -- host side of the C ABI (include/magus_replay.h): validation, exact-equivalent
// threshold derivation, launch geometry, TMA descriptors, kernel launches, NCCL allreduce, results.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/magus_replay.h"
#include "post_kernels.cuh"
#include "replay_kernel.cuh"
#include "replay_solo.cuh"
#include "replay_wide.cuh"
#include "wallclock.cuh"

using namespace magus;

#ifndef MAGUS_TC
#define MAGUS_TC 8
#endif
#ifndef MAGUS_NSTAGE
#define MAGUS_NSTAGE 3
#endif

static_assert(sizeof(TraceRec) == sizeof(magus_trace_stats), "TraceRec must mirror magus_trace_stats");
static_assert(kNTot == MAGUS_N_TOTALS, "totals width");

namespace {

constexpr size_t kChainBytes = 8 + 8 + 6 * 4;   // sexc, digest, nhi, nthr, trans, ev, lock, vmax
constexpr int kTC = MAGUS_TC;        // ticks per TMA stage ([TC x 128] fp32 tile)
constexpr int kNStage = MAGUS_NSTAGE;  // stages per tile group
using Smem = ReplaySmem<kTC, kNStage>;
typedef void (*ReplayKernel)(CUtensorMap, ReplayParams);

// chain kind of a lane policy -> its kernel instantiation (one register allocation per kind)
int ticker_key(const DevPolicy& q) {
    if (q.kind == LANE_MAGUS) {
        const int l64 = q.C > kMaxC32 ? 1 : 0;
        int k = q.k <= 8 ? q.k : 0;
        if (l64 && (k == 3 || k == 5 || k == 6 || k == 7)) k = 0;
        return 100 * l64 + k;   // 0..8, 100..108
    }
    return 1000 + q.kind;       // TDP, STATIC_MIN, VALIDATE
}

// CTAs per SM a MAGUS chain kind's kernel is built for (register budget): 1 for K >= 4, the generic ring
// or the 64-bit log (they would spill under 128 registers), else 2 (also TDP / STATIC_MIN / VALIDATE).
int minb_for(int key) { return key < 1000 && (key == 0 || key >= 4) ? 1 : 2; }

template <class T, int MINB = 2>
ReplayKernel K() { return (ReplayKernel)magus_replay_kernel<T, kTC, kNStage, MINB>; }

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

// the lockstep walk (one-warp CTAs, lane = chain; post_kernels.cuh) covers these chain kinds
bool lockstep_walk(int key) {
    return ((key >= 1 && key <= 8) || key == 1000 + LANE_TDP) && env_int("MAGUS_WALK_LOCKSTEP", 1);
}

// the split walk (64-thread CTAs: one warp per recurrence of 32 traces) covers the register-ring MAGUS kinds
bool split_walk(int key) { return key >= 1 && key <= 8 && env_int("MAGUS_WALK_SPLIT", 1); }

// chain-walk fix-up kernel for a chain kind (nullptr: stateless kinds never mismatch)
typedef void (*WalkKernel)(ReplayParams, EpiParams, FixParams, int, const float*);
WalkKernel walk_kernel_for(int key) {
    if (split_walk(key)) {
        switch (key) {
            case 1: return magus_fix_split_kernel<1>;
            case 2: return magus_fix_split_kernel<2>;
            case 3: return magus_fix_split_kernel<3>;
            case 4: return magus_fix_split_kernel<4>;
            case 5: return magus_fix_split_kernel<5>;
            case 6: return magus_fix_split_kernel<6>;
            case 7: return magus_fix_split_kernel<7>;
            default: return magus_fix_split_kernel<8>;
        }
    }
    if (lockstep_walk(key)) {
        switch (key) {
            case 1: return magus_fix_lockstep_kernel<MagusTicker<1, false>>;
            case 2: return magus_fix_lockstep_kernel<MagusTicker<2, false>>;
            case 3: return magus_fix_lockstep_kernel<MagusTicker<3, false>>;
            case 4: return magus_fix_lockstep_kernel<MagusTicker<4, false>>;
            case 5: return magus_fix_lockstep_kernel<MagusTicker<5, false>>;
            case 6: return magus_fix_lockstep_kernel<MagusTicker<6, false>>;
            case 7: return magus_fix_lockstep_kernel<MagusTicker<7, false>>;
            case 8: return magus_fix_lockstep_kernel<MagusTicker<8, false>>;
            default: return magus_fix_lockstep_kernel<TdpTicker>;
        }
    }
    switch (key) {   // one thread per chain (the generic ring, the 64-bit logs; MAGUS_WALK_LOCKSTEP=0)
        case 1: return magus_fix_walk_kernel<MagusTicker<1, false>>;
        case 2: return magus_fix_walk_kernel<MagusTicker<2, false>>;
        case 3: return magus_fix_walk_kernel<MagusTicker<3, false>>;
        case 4: return magus_fix_walk_kernel<MagusTicker<4, false>>;
        case 5: return magus_fix_walk_kernel<MagusTicker<5, false>>;
        case 6: return magus_fix_walk_kernel<MagusTicker<6, false>>;
        case 7: return magus_fix_walk_kernel<MagusTicker<7, false>>;
        case 8: return magus_fix_walk_kernel<MagusTicker<8, false>>;
        case 1000 + LANE_TDP: return magus_fix_walk_kernel<TdpTicker>;
        case 1000 + LANE_STATIC_MIN: return nullptr;
        case 1000 + LANE_VALIDATE: return nullptr;
        default: return key >= 100 ? magus_fix_walk_kernel<MagusTicker<0, true>> : magus_fix_walk_kernel<MagusTicker<0, false>>;
    }
}

ReplayKernel replay_kernel_for(int key) {
    switch (key) {
        case 0: return K<MagusTicker<0, false>, 1>();
        case 1: return K<MagusTicker<1, false>, 2>();
        case 2: return K<MagusTicker<2, false>, 2>();
        case 3: return K<MagusTicker<3, false>, 2>();
        case 4: return K<MagusTicker<4, false>, 1>();
        case 5: return K<MagusTicker<5, false>, 1>();
        case 6: return K<MagusTicker<6, false>, 1>();
        case 7: return K<MagusTicker<7, false>, 1>();
        case 8: return K<MagusTicker<8, false>, 1>();
        case 100: return K<MagusTicker<0, true>, 1>();
        case 101: return K<MagusTicker<1, true>, 1>();
        case 102: return K<MagusTicker<2, true>, 1>();
        case 104: return K<MagusTicker<4, true>, 1>();
        case 108: return K<MagusTicker<8, true>, 1>();
        case 1000 + LANE_TDP: return K<TdpTicker>();
        case 1000 + LANE_STATIC_MIN: return K<StaticMinTicker<false>>();
        default: return K<StaticMinTicker<true>>();
    }
}

// entry-major wall-clock kernel (wallclock.cuh, A32) of a chain kind
typedef void (*WallKernel)(ReplayParams, EpiParams, WallParams, int, const float*);
template <bool U>
WallKernel wall_kernel_u(int key) {
    switch (key) {
        case 1: return magus_wallclock_em_kernel<MagusTicker<1, false>, U>;
        case 2: return magus_wallclock_em_kernel<MagusTicker<2, false>, U>;
        case 3: return magus_wallclock_em_kernel<MagusTicker<3, false>, U>;
        case 4: return magus_wallclock_em_kernel<MagusTicker<4, false>, U>;
        case 5: return magus_wallclock_em_kernel<MagusTicker<5, false>, U>;
        case 6: return magus_wallclock_em_kernel<MagusTicker<6, false>, U>;
        case 7: return magus_wallclock_em_kernel<MagusTicker<7, false>, U>;
        case 8: return magus_wallclock_em_kernel<MagusTicker<8, false>, U>;
        case 1000 + LANE_TDP: return magus_wallclock_em_kernel<TdpTicker, U>;
        case 1000 + LANE_STATIC_MIN: return magus_wallclock_em_kernel<StaticMinTicker<false>, U>;
        case 1000 + LANE_VALIDATE: return magus_wallclock_em_kernel<StaticMinTicker<false>, U>;
        default: return key >= 100 ? magus_wallclock_em_kernel<MagusTicker<0, true>, U>
                                   : magus_wallclock_em_kernel<MagusTicker<0, false>, U>;
    }
}
// unrolled entry blocks while the run has few chains per SM (latency-bound), rolled otherwise (issue-bound;
// the unrolled code also misses the instruction cache); MAGUS_WALL_UNROLL=0/1 forces one
WallKernel wall_kernel_for(int key, int64_t n_chains, int n_sm) {
    const int f = env_int("MAGUS_WALL_UNROLL", -1);
    const bool u = f >= 0 ? f != 0 : n_chains < (int64_t)n_sm * 128;
    return u ? wall_kernel_u<true>(key) : wall_kernel_u<false>(key);
}

// unsegmented one-chain-per-lane replay kernel (replay_wide.cuh) of a chain kind, or nullptr if it has none
// lv: 0 = the MAGUS_WSTAGE1D block, 1 = its L form, 2 = the L form with the |d| test (replay_wide.cuh; nc = 1 only)
ReplayKernel wide_kernel_for(int key, int nc, int lv = 0) {
#define WIDE_K(KK)                                                                                                  \
    (nc == 2    ? (ReplayKernel)magus_replay_wide_kernel<KK, 2, 0>                                                  \
     : lv == 1 ? (ReplayKernel)magus_replay_wide_kernel<KK, 1, 1>                                                   \
     : lv == 2 ? (ReplayKernel)magus_replay_wide_kernel<KK, 1, 2>                                                   \
     : lv == 3 ? (ReplayKernel)magus_replay_wide_kernel<KK, 1, 3>                                                   \
     : lv == 4 ? (ReplayKernel)magus_replay_wide_kernel<KK, 1, 4>                                                   \
               : (ReplayKernel)magus_replay_wide_kernel<KK, 1, 0>)
    switch (key) {
        case 1: return WIDE_K(1);
        case 2: return WIDE_K(2);
        case 3: return WIDE_K(3);
        case 4: return WIDE_K(4);
        case 5: return WIDE_K(5);
        case 6: return WIDE_K(6);
        case 7: return WIDE_K(7);
        case 8: return WIDE_K(8);
        default: return nullptr;
    }
#undef WIDE_K
}

// the two-warp MAGUS + TDP kernel (replay_solo.cuh) for a MAGUS chain kind with a solo stage block and np TDP policies
ReplayKernel combo_kernel_for(int key, int np) {
#define COMBO_K(KK) (np == 1 ? (ReplayKernel)magus_replay_combo_kernel<MagusTicker<KK, false>, 1, kTC, kNStage>    \
                             : (ReplayKernel)magus_replay_combo_kernel<MagusTicker<KK, false>, 2, kTC, kNStage>)
    switch (key) {
        case 1: return COMBO_K(1);
        case 2: return COMBO_K(2);
        case 3: return COMBO_K(3);
        default: return nullptr;
    }
#undef COMBO_K
}

// the fused one-warp MAGUS + TDP kernel (replay_solo.cuh) for a MAGUS chain kind with an L stage block: `sym` = the
// |d| tune-flag test (d*_dec == -d*_inc), `ctas` = resident CTAs per SM it is built for (12: 168 registers, 16: 128)
// up = the TDP policy's f_min threshold is +inf (f_min always rises: one compare fewer per TDP tick)
ReplayKernel fused_kernel_for(int key, bool sym, int ctas, bool up, bool lb) {
#define FUSED_KK(KK, S, C, U, L) (ReplayKernel)magus_replay_fused_kernel<MagusTicker<KK, false>, kTC, kNStage, S, C, U, L>
#define FUSED_K12(KK, L)                                                                                            \
    (up ? (sym ? FUSED_KK(KK, true, 12, true, L) : FUSED_KK(KK, false, 12, true, L))                               \
        : (sym ? FUSED_KK(KK, true, 12, false, L) : FUSED_KK(KK, false, 12, false, L)))
#define FUSED_K(KK)                                                                                                 \
    (ctas == 16 ? (sym ? FUSED_KK(KK, true, 16, false, false) : FUSED_KK(KK, false, 16, false, false))             \
     : lb       ? FUSED_K12(KK, true)                                                                               \
                : FUSED_K12(KK, false))
    switch (key) {
        case 1: return FUSED_K(1);
        case 2: return FUSED_K(2);
        case 3: return FUSED_K(3);
        default: return nullptr;
    }
#undef FUSED_K
#undef FUSED_K12
#undef FUSED_KK
}

// one-warp-CTA replay kernel (replay_solo.cuh) of a chain kind, or nullptr if it has none
ReplayKernel solo_kernel_for(int key, bool sym, bool bits_ok, bool lsign_ok, bool open = false,
                             bool lbatch_ok = false) {
    int v = env_int("MAGUS_SOLO_BAL", 24);   // stage block variant (replay_solo.cuh)
    // the open-loop O stage (the caller checked lsign_ok); 34 / 35 with the batched tune-flag log (8 <= C <= 24)
    if (open) v = (lbatch_ok && kTC == 8 && env_int("MAGUS_SOLO_BAL", 24) == 24 ? 34 : 30) + (sym ? 1 : 0);
    // 24: the L stage with the tune-flag log shifted once per stage (8 <= C <= 24, 8-tick stages), |d| test 25 when every
    // lane policy has d*_dec == -d*_inc; else as 20
    if (v == 24) v = (lsign_ok && lbatch_ok && kTC == 8) ? (sym ? 25 : 24) : 20;
    // 20: the L stage (level in the cmd word, lock = sign of the biased window count; needs C <= 27), with the
    // |d| tune-flag test (21) when every lane policy has d*_dec == -d*_inc; 22 forces the two-compare L stage
    if (v == 20 || v == 22) v = !lsign_ok ? 2 : (v == 20 && sym) ? 21 : 20;
    else if (v == 21 && !(sym && lsign_ok)) v = 2;
    if (v == 9) v = 2;   // PSTAGES (|d| test + popcount): slower than 2 and it failed parity on mixed-kinds (round 2)
    if (v == 5 && !bits_ok) v = 2;          // the integer sample conversion needs |d*| >= 2^-60, B_lo normal
    if (v >= 10 && v <= 17) {   // the unified-stage kernel; v - 10 = VAR bits (1 |d| test, 2 incremental count,
                                // 4 integer sample conversion)
        int var = v - 10;
        if (!sym) var &= ~1;
        if (!bits_ok) var &= ~4;
#define USOLO(KK, VV) (ReplayKernel) magus_replay_usolo_kernel<MagusTicker<KK, false>, kTC, kNStage, VV>
#define USOLO_K(KK)                                                                                             \
    switch (var) {                                                                                              \
        case 0: return USOLO(KK, 0);                                                                            \
        case 1: return USOLO(KK, 1);                                                                            \
        case 2: return USOLO(KK, 2);                                                                            \
        case 3: return USOLO(KK, 3);                                                                            \
        case 4: return USOLO(KK, 4);                                                                            \
        case 5: return USOLO(KK, 5);                                                                            \
        case 6: return USOLO(KK, 6);                                                                            \
        default: return USOLO(KK, 7);                                                                           \
    }
        switch (key) {
            case 1: USOLO_K(1)
            case 2: USOLO_K(2)
            case 3: USOLO_K(3)
            default: return nullptr;
        }
#undef USOLO_K
#undef USOLO
    }
#define SOLO_K(KK)                                                                                               \
    (v == 0   ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 0>                    \
     : v == 2 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 2>                    \
     : v == 3 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 3>                    \
     : v == 4 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 4>                    \
     : v == 5 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 5>                    \
     : v == 20 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 20>                  \
     : v == 21 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 21>                  \
     : v == 24 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 24>                  \
     : v == 25 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 25>                  \
     : v == 30 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 30>                  \
     : v == 31 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 31>                  \
     : v == 34 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 34>                  \
     : v == 35 ? (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 35>                  \
              : (ReplayKernel)magus_replay_solo_kernel<MagusTicker<KK, false>, kTC, kNStage, 1>)
    switch (key) {
        case 1: return SOLO_K(1);
        case 2: return SOLO_K(2);
        case 3: return SOLO_K(3);
        default: return nullptr;
    }
#undef SOLO_K
}

// one replay launch: the lane policies [q_base, q_base + nq) share a chain kind
struct LaunchGroup {
    ReplayKernel kernel;
    int key, q_base, nq, ng, npw, n_tblocks, n_pblocks, n_ctas, threads;
    size_t smem;
    bool solo;   // one-warp CTAs (npw == 1 and the kind has a solo kernel)
    bool wide;   // the unsegmented one-chain-per-lane kernel (replay_wide.cuh), fed by the 16-trace tensor map
    bool fused;  // replayed by the previous group's launch (magus_replay_combo_kernel): no launch of its own
};

// Kernel launch with programmatic stream serialization (PDL) when `pdl`: the kernel may be scheduled
// while its predecessor drains and waits in griddepcontrol.wait (ptx::pdl_wait) before touching the
// predecessor's outputs.  Captured into the run's graph as a programmatic edge.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

thread_local std::string g_error;

// ------------------------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool loaded = false;
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.loaded) {
        api.loaded = true;
        api.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.handle) api.handle = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (api.handle) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.handle, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.handle, "ncclCommInitRank");
            api.AllReduce = (decltype(api.AllReduce))dlsym(api.handle, "ncclAllReduce");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.handle, "ncclCommDestroy");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.handle, "ncclGetErrorString");
        }
    }
    return api;
}
bool nccl_ok() {
    NcclApi& a = nccl();
    return a.handle && a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy;
}

// ------------------------------------------------------------------------------------ TMA encode
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
        cudaGetLastError();
    }
    return fn;
}

// ------------------------------------------------------------------------------------ exact thresholds
// Ordered integer keys of doubles / floats: key order == numeric order (with -0 just below +0).
inline uint64_t dkey(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
inline double dval(uint64_t k) {
    uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    double x;
    std::memcpy(&x, &b, 8);
    return x;
}
inline float fval(uint32_t b) {
    float x;
    std::memcpy(&x, &b, 4);
    return x;
}
inline uint32_t fbits(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    return b;
}

// Alg. 1: +1 iff fl(d / L) > inc.  fl(./L) is monotone, so {d : +1} = {d > d*} with
// d* = max{d : fl(d/L) <= inc}; found by bisection over the ordered doubles, evaluating the
// predicate exactly as the oracle writes it.
double derive_dinc(double L, double inc) {
    volatile double vL = L, vi = inc;
    uint64_t lo = dkey(-INFINITY), hi = dkey(INFINITY);   // p(lo) false, p(hi) true
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        const double d = dval(mid);
        if (d / vL > vi) hi = mid;
        else lo = mid;
    }
    return dval(lo);
}
// Alg. 1: -1 iff fl(d / L) < dec  <=>  d < d*, d* = min{d : fl(d/L) >= dec}.
double derive_ddec(double L, double dec) {
    volatile double vL = L, vd = dec;
    uint64_t lo = dkey(-INFINITY), hi = dkey(INFINITY);   // q(lo) true, q(hi) false
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        const double d = dval(mid);
        if (d / vL < vd) lo = mid;
        else hi = mid;
    }
    return dval(hi);
}
// Alg. 2: true iff fl(s / C) >= thr on a full log; s_min = min such s (C+1 = never).
int derive_smin(int C, double thr) {
    for (int s = 0; s <= C; ++s)
        if ((double)s / (double)C >= thr) return s;
    return C + 1;
}

double uncore_power_at(double f, const magus_model& m) {
    const double x = (f - m.f_min_ghz) / (m.f_max_ghz - m.f_min_ghz);
    return m.p_uncore_min_w + (m.p_uncore_max_w - m.p_uncore_min_w) * std::pow(x, m.p_exponent);
}
double pkg_power_at(double f, const magus_model& m) {
    return (m.p_pkg_idle_w + m.p_core_active_w) + uncore_power_at(f, m);
}
double bandwidth_at(double f, const magus_model& m) {     // SPEC.md:333, operand order DESIGN A26
    const double ratio = f / m.f_max_ghz;
    if (m.bw_shape == 0) return m.bw_max_gbps * ratio;
    const double r = ratio / m.bw_knee;
    return m.bw_max_gbps * (r < 1.0 ? r : 1.0);
}

// TDP (A24): cmd = f_min iff fl(P + fl(c*A)) >= fl((1-m)*TDP); monotone in fp32 A >= 0, so
// it is A >= a*, a* = the smallest such fp32 (+inf if none).
float derive_astar(double P, const magus_model& m, const magus_policy& p) {
    volatile double vP = P, vc = m.dram_w_per_gbps;
    const double bound = (1.0 - p.tdp_margin) * p.tdp_w;
    auto pred = [&](uint32_t bits) { return (vP + vc * (double)fval(bits)) >= bound; };
    const uint32_t zero = 0u, inf = 0x7F800000u;
    if (pred(zero)) return 0.0f;
    if (!pred(inf)) return INFINITY;
    uint32_t lo = zero, hi = inf;
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (pred(mid)) hi = mid;
        else lo = mid;
    }
    return fval(hi);
}

bool finite(double x) { return std::isfinite(x); }

// ------------------------------------------------------------------------------------ validation
std::string validate_model(const magus_model& m) {
    if (!(finite(m.sample_period_s) && m.sample_period_s > 0)) return "sample_period_s must be finite and > 0";
    if (!(finite(m.f_min_ghz) && m.f_min_ghz > 0)) return "f_min_ghz must be finite and > 0";
    if (!(finite(m.f_max_ghz) && m.f_max_ghz > m.f_min_ghz)) return "f_max_ghz must be finite and > f_min_ghz";
    if (!(finite(m.bw_max_gbps) && m.bw_max_gbps > 0)) return "bw_max_gbps must be finite and > 0";
    if (m.bw_shape != 0 && m.bw_shape != 1) return "bw_shape must be 0 (Linear) or 1 (Saturating)";
    if (m.bw_shape == 1 && !(m.bw_knee > 0 && m.bw_knee <= 1)) return "bw_knee must be in (0, 1]";
    if (m.observe != 0 && m.observe != 1) return "observe must be 0 (closed loop) or 1 (open loop)";
    const double pw[] = {m.p_pkg_idle_w, m.p_core_active_w, m.p_uncore_min_w, m.p_uncore_max_w, m.p_gpu_active_w,
                         m.dram_w_per_gbps};
    const char* names[] = {"p_pkg_idle_w", "p_core_active_w", "p_uncore_min_w", "p_uncore_max_w",
                           "p_gpu_active_w", "dram_w_per_gbps"};
    for (int i = 0; i < 6; ++i)
        if (!(finite(pw[i]) && pw[i] >= 0)) return std::string(names[i]) + " must be finite and >= 0";
    if (!(m.p_uncore_max_w >= m.p_uncore_min_w)) return "p_uncore_max_w must be >= p_uncore_min_w";
    if (!(finite(m.p_exponent) && m.p_exponent >= 1)) return "p_exponent must be finite and >= 1";
    const float blo = (float)bandwidth_at(m.f_min_ghz, m);
    if (!(blo > 0.0f)) return "bw_max_gbps too small: bandwidth at f_min rounds to 0 in fp32";
    return "";
}

std::string validate_policy(const magus_policy& p, int i) {
    const std::string at = "policies[" + std::to_string(i) + "].";
    if (p.kind < 0 || p.kind > 3) return at + "kind must be 0..3";
    if (p.kind == MAGUS_POLICY_MAGUS) {
        if (p.deriv_ticks < 1 || p.deriv_ticks > KMAX_GENERIC) return at + "deriv_ticks must be in [1, 64]";
        if (!(finite(p.inc_threshold) && p.inc_threshold > 0)) return at + "inc_threshold must be finite and > 0";
        if (!(finite(p.dec_threshold) && p.dec_threshold < 0)) return at + "dec_threshold must be finite and < 0";
        if (p.tune_log_capacity < 1 || p.tune_log_capacity > 64) return at + "tune_log_capacity must be in [1, 64]";
        if (!(p.high_freq_threshold > 0 && p.high_freq_threshold <= 1))
            return at + "high_freq_threshold must be in (0, 1]";
    }
    if (p.kind == MAGUS_POLICY_TDP_DEFAULT) {
        if (!(finite(p.tdp_w) && p.tdp_w > 0)) return at + "tdp_w must be finite and > 0";
        if (!(p.tdp_margin > 0 && p.tdp_margin < 1)) return at + "tdp_margin must be in (0, 1)";
    }
    return "";
}

}  // namespace

// ============================================================================================ handle
struct magus_replay {
    magus_replay_desc desc{};
    std::vector<magus_policy> pols;
    std::vector<DevPolicy> lane;        // lane policies (everything but STATIC_MAX; or one validate pseudo)
    std::vector<int> smax;              // policies in the closed form of STATIC_MAX (and TDP never leaving f_max)
    float B_lo = 0, B_hi = 0;
    uint32_t bwbits = 0;
    double P_lo = 0, P_hi = 0;
    uint64_t digest_all_hi = 0;
    ReplayParams rp{};
    EpiParams ep{};
    std::vector<LaunchGroup> groups;
    FixParams fx{};
    int n_sm = 148;
    int alloc_segments = 1;           // scratch is sized for this many segments (re-plans only shrink)
    int replans = 0;
    double replan_frac = 0.25;        // re-plan above this fraction of wrong speculative entries
    int warm_extra = 0;               // adaptive warm-up: ticks added to roundup32(k + C - 1)
    int warm_replans = 0;
    bool pdl = true;           // programmatic dependent launch between the run's kernels (MAGUS_NO_PDL=1: off)
    // device memory
    std::vector<void*> allocs;
    DevPolicy* d_pol = nullptr;
    int* d_smax = nullptr;
    int* d_lane_of_policy = nullptr;  // user policy -> lane policy (-1: STATIC_MAX, analytic)
    int validate_lane = -1;           // lane of the validate-only pseudo policy, if any
    TraceRec* d_rec = nullptr;
    bool wall = false;                // MAGUS_F_WALLCLOCK: wall-clock governor rounds (A32)
    TraceRec* d_wrec = nullptr;       // wall: [n_lane][n_traces] lane-chain records
    double* d_totals = nullptr;
    uint8_t* d_out = nullptr;         // [P][chunks][13] totals partials (fp64), then the 4 run flag words: one D2H copy
    double* d_fin = nullptr;          // exchange on: [P_glob][13] per-policy totals, allreduced across ranks
    double* d_fin_local = nullptr;    // exchange on: [P_glob][13], this rank's slice rows (the rest stays 0)
    int P_glob = 1, p_off = 0;        // parameter-grid split: global policy count, global index of local policy 0
    bool xchg = false;                // the cross-rank exchange runs (world > 1 or MAGUS_F_NCCL)
    bool open_fast = false;           // open loop, every group a MAGUS solo group: the O stage + the closed-form
                                      // open-loop fix-up instead of the chain walk
    int n_chunks = 1;                 // trace chunks of the totals kernel
    int32_t* d_first_low = nullptr;   // [n_traces] speculation aid
    uint8_t* d_chain = nullptr;       // per-chain totals (ReplayParams::c_*)
    unsigned int* d_flag = nullptr;     // [0] invalid flag, [1] fix rounds, [2..3] fix segments (u64)
    unsigned long long* d_errkey = nullptr;
    uint8_t* d_codes = nullptr;
    float* d_trace_own = nullptr;
    float* d_w_own = nullptr;
    // last run
    const float* run_trace = nullptr;
    cudaStream_t run_stream = nullptr;
    bool ran = false;
    CUtensorMap tmap{};
    CUtensorMap tmap_w{};   // box {16 traces, 32 ticks}: the wide kernel's tiles
    const float* tmap_ptr = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};   // ev[4]: the run's completion
    static constexpr int kTimingRing = 256;
    std::vector<cudaEvent_t> tev;   // MAGUS_F_TIMING: 5 event slots per run, ring of kTimingRing runs
    int64_t n_runs = 0;
    ncclComm_t comm = nullptr;
    cudaGraphExec_t gexec = nullptr;  // the captured run
    cudaGraph_t graph = nullptr;
    const float* g_trace = nullptr;
    const float* g_w = nullptr;
    cudaStream_t g_stream = nullptr;
    std::vector<std::pair<cudaGraphNode_t, int>> g_events;   // event-record node -> timing slot index
    std::vector<cudaStream_t> aux;     // one per extra launch group (concurrent replay launches)
    std::vector<cudaEvent_t> join_ev;
    cudaEvent_t fork_ev = nullptr;
    std::string err;
};

static magus_status fail(magus_replay_t* h, magus_status s, const std::string& msg) {
    if (h) h->err = msg;
    g_error = msg;
    return s;
}
static magus_status cuda_fail(magus_replay_t* h, cudaError_t e, const char* where) {
    return fail(h, e == cudaErrorMemoryAllocation ? MAGUS_ERR_OOM : MAGUS_ERR_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}
#define CU(h, call)                                          \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
    } while (0)

template <class T>
static cudaError_t dalloc(magus_replay_t* h, T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, count * sizeof(T));
    if (e == cudaSuccess) {
        h->allocs.push_back(v);
        *p = (T*)v;
    }
    return e;
}

extern "C" const char* magus_set_global_error(const char* msg) {
    g_error = msg ? msg : "";
    return g_error.c_str();
}

extern "C" int32_t magus_abi_version(void) { return MAGUS_ABI_VERSION; }

extern "C" magus_status magus_replay_plan_info(const magus_replay_t* h, int32_t out[4]) {
    if (!h || !out) return MAGUS_ERR_INVALID_ARG;
    int32_t launches = 0, fused = 0, wide = 0;
    for (const LaunchGroup& g : h->groups) {
        launches += g.fused ? 0 : 1;
        fused = fused || g.fused;
        wide += g.wide ? 1 : 0;
    }
    out[0] = launches;
    out[1] = fused && h->groups.front().threads == 32 ? 1 : 0;   // the one-warp fused kernel (not the 2-warp combo)
    out[2] = h->open_fast ? 1 : 0;
    out[3] = wide;
    return MAGUS_OK;
}

__global__ void magus_debug_probe_kernel(int32_t violate) { MAGUS_CHECK(violate == 0); }

extern "C" int32_t magus_debug_check_probe(int32_t violate) {
#if MAGUS_DEBUG_CHECKS
    magus_debug_probe_kernel<<<1, 1>>>(violate);
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1;
#else
    (void)violate;
    return -1;
#endif
}
extern "C" const char* magus_last_error(void) { return g_error.c_str(); }
extern "C" const char* magus_replay_last_error(const magus_replay_t* h) {
    return h ? h->err.c_str() : g_error.c_str();
}

// NEXT-4: active savings of a policy against a baseline from the job's per-policy totals.
extern "C" magus_status magus_active_savings(const double* tot, int32_t n_policies, int32_t policy, int32_t baseline,
                                             double p_idle_w, double out[3]) {
    if (!tot || !out) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: NULL argument");
    if (policy < 0 || policy >= n_policies || baseline < 0 || baseline >= n_policies)
        return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: policy index outside [0, n_policies)");
    const double E = tot[(size_t)policy * MAGUS_N_TOTALS + MAGUS_TOT_E];
    const double T = tot[(size_t)policy * MAGUS_N_TOTALS + MAGUS_TOT_T];
    const double Eb = tot[(size_t)baseline * MAGUS_N_TOTALS + MAGUS_TOT_E];
    const double Tb = tot[(size_t)baseline * MAGUS_N_TOTALS + MAGUS_TOT_T];
    if (!(T > 0.0) || !(Tb > 0.0)) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: zero total time");
    if (!(p_idle_w >= 0.0)) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: p_idle_w must be >= 0");
    const double P = E / T, Pb = Eb / Tb;
    if (!(Pb > p_idle_w)) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: no active power in baseline");
    if (P < p_idle_w) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_active_savings: mean power below idle power");
    const double active = Pb - p_idle_w;                        // the baseline's active power
    const double Ea = E - p_idle_w * T, Eab = Eb - p_idle_w * Tb;   // active energies
    out[0] = (active - (P - p_idle_w)) / active;
    out[1] = 1.0 - Ea / Eab;
    out[2] = 1.0 - (Ea * T) / (Eab * Tb);
    return MAGUS_OK;
}

extern "C" magus_status magus_totals_argmin(const double* tot, int32_t n_policies, int32_t* out) {
    if (!tot || !out || n_policies < 1) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_totals_argmin: bad argument");
    bool any = false;
    for (int32_t p = 0; p < n_policies; ++p) any = any || tot[(size_t)p * MAGUS_N_TOTALS + MAGUS_TOT_N_TRACES] > 0.0;
    int32_t am = -1;
    for (int32_t p = 0; p < n_policies; ++p) {
        if (any && !(tot[(size_t)p * MAGUS_N_TOTALS + MAGUS_TOT_N_TRACES] > 0.0)) continue;
        if (am < 0 || tot[(size_t)p * MAGUS_N_TOTALS + MAGUS_TOT_EDP] < tot[(size_t)am * MAGUS_N_TOTALS + MAGUS_TOT_EDP])
            am = p;
    }
    *out = am;
    return MAGUS_OK;
}

extern "C" magus_status magus_grid_plan(int32_t world, int32_t rank, int32_t policy_shards, int64_t n_traces,
                                        int32_t n_policies, int64_t out[4]) {
    if (!out || world < 1 || rank < 0 || rank >= world || policy_shards < 1 || world % policy_shards != 0 ||
        n_traces < 0 || policy_shards > n_policies)
        return fail(nullptr, MAGUS_ERR_INVALID_ARG,
                    "magus_grid_plan: need 0 <= rank < world, policy_shards dividing world, "
                    "1 <= policy_shards <= n_policies, n_traces >= 0");
    const int64_t trace_shards = world / policy_shards, ts = rank / policy_shards, ps = rank % policy_shards;
    auto cut = [](int64_t n, int64_t parts, int64_t i, int64_t* off, int64_t* cnt) {   // sizes differ by <= 1
        const int64_t base = n / parts, extra = n % parts;
        *off = i * base + std::min(i, extra);
        *cnt = base + (i < extra ? 1 : 0);
    };
    cut(n_traces, trace_shards, ts, &out[0], &out[1]);
    cut(n_policies, policy_shards, ps, &out[2], &out[3]);
    return MAGUS_OK;
}

extern "C" magus_status magus_derive_thresholds(const magus_policy* p, const magus_model* m, double out_d[5],
                                                float out_f[4], int32_t out_i[1]) {
    if (!p || !m || !out_d || !out_f || !out_i) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "NULL argument");
    std::string e = validate_model(*m);
    if (e.empty()) e = validate_policy(*p, 0);
    if (!e.empty()) return fail(nullptr, MAGUS_ERR_CONFIG, e);
    const double L = (double)(p->kind == MAGUS_POLICY_MAGUS ? p->deriv_ticks : 1) * m->sample_period_s;
    const double P_lo = pkg_power_at(m->f_min_ghz, *m), P_hi = pkg_power_at(m->f_max_ghz, *m);
    out_d[0] = p->kind == MAGUS_POLICY_MAGUS ? derive_dinc(L, p->inc_threshold) : 0.0;
    out_d[1] = p->kind == MAGUS_POLICY_MAGUS ? derive_ddec(L, p->dec_threshold) : 0.0;
    out_d[2] = L;
    out_d[3] = P_lo;
    out_d[4] = P_hi;
    out_f[0] = (float)bandwidth_at(m->f_min_ghz, *m);
    out_f[1] = (float)bandwidth_at(m->f_max_ghz, *m);
    out_f[2] = p->kind == MAGUS_POLICY_TDP_DEFAULT ? derive_astar(P_lo, *m, *p) : INFINITY;
    out_f[3] = p->kind == MAGUS_POLICY_TDP_DEFAULT ? derive_astar(P_hi, *m, *p) : INFINITY;
    out_i[0] = p->kind == MAGUS_POLICY_MAGUS ? derive_smin(p->tune_log_capacity, p->high_freq_threshold) : 0;
    return MAGUS_OK;
}

extern "C" magus_status magus_nccl_unique_id(void* out128) {
    if (!out128) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "NULL argument");
    if (!nccl_ok()) return fail(nullptr, MAGUS_ERR_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, MAGUS_ERR_NCCL, nccl().GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return MAGUS_OK;
}

// ------------------------------------------------------------------------------------ geometry
// Chooses, per launch group, the CTA shape, and globally the time segmentation:
// enough independent chains to fill the SMs, whole waves of equal-work CTAs, warm-up W >= k + C - 1
// (+ margin).
static void choose_geometry(magus_replay_t* h, int n_sm, int forced_segments) {
    ReplayParams& p = h->rp;
    const magus_replay_desc& d = h->desc;
    const int Q = (int)h->lane.size();
    p.n_lane = Q;
    p.n_traces = d.n_traces;
    p.n_samples = d.n_samples;
    p.trace_stride = d.trace_stride;
    p.n_groups = (d.n_traces + kTracesPerWarp - 1) / kTracesPerWarp;
    // smem budget per CTA: 2 CTAs per SM (or 1 for the large-state kinds)
    h->groups.clear();
    for (int q = 0; q < Q;) {
        LaunchGroup g{};
        g.key = ticker_key(h->lane[q]);
        g.kernel = replay_kernel_for(g.key);
        g.q_base = q;
        while (q < Q && ticker_key(h->lane[q]) == g.key) ++q;
        g.nq = q - g.q_base;
        g.npw = std::min(g.nq, kMaxConsumerWarps);
        g.n_pblocks = (g.nq + g.npw - 1) / g.npw;
        const int ng_smem = (int)(((minb_for(g.key) == 2 ? 100 : 200) * 1024) / (kNStage * Smem::kTileBytes));
        int ng = std::min(ng_smem, kMaxConsumerWarps / g.npw);
        ng = std::min(ng, env_int("MAGUS_NG", ng));
        g.ng = std::max(1, std::min(ng, std::max(1, p.n_groups)));
        g.n_tblocks = std::max(1, (p.n_groups + g.ng - 1) / g.ng);
        g.threads = g.ng * g.npw * 32;
        g.smem = Smem::bytes(g.ng);
        h->groups.push_back(g);
    }
    int kmax = 1, cmax = 1;
    p.kr = 1;
    for (const DevPolicy& q : h->lane) {
        if (q.kind == LANE_MAGUS) {
            kmax = std::max(kmax, q.k);
            cmax = std::max(cmax, q.C);
            p.kr = std::max(p.kr, q.k);
        }
    }
    // Open loop (A30) with every launch group a MAGUS kind with a solo stage block (k <= 3, C <= 27): the O stage and
    // the closed-form open-loop fix-up (MAGUS_OPEN_FAST default 1)
    h->open_fast = d.model.observe == 1 && env_int("MAGUS_OPEN_FAST", 1) != 0 && !h->groups.empty();
    for (const LaunchGroup& g : h->groups) h->open_fast = h->open_fast && g.key >= 1 && g.key <= 3;
    for (const DevPolicy& q : h->lane) h->open_fast = h->open_fast && (q.kind != LANE_MAGUS || q.C <= 27);
    // Unsegmented plan: when every launch group is a MAGUS kind with a wide kernel and one
    // chain per lane already gives enough warps (>= MAGUS_WIDE_WARPS_PER_SM per SM, default 12; the lanes at least
    // 3/4 used), replay each chain whole -- no speculation, no fix-up.  MAGUS_WIDE = 0 never, 1 whenever possible.
    bool wide = forced_segments == 0 && d.tuning_segments == 0 && d.tuning_warmup == 0 && d.n_traces > 0;
    {
        int64_t warps = 0, lanes_used = 0, lanes_all = 0;   // lanes: policy points per trace, used / allotted
        for (const LaunchGroup& g : h->groups) {
            wide = wide && wide_kernel_for(g.key, 1) != nullptr;
            const int64_t pbs = (g.nq + kWidePpc - 1) / kWidePpc;
            warps += pbs * ((d.n_traces + kWideTpc - 1) / kWideTpc) * kWideWarps;
            lanes_used += g.nq;
            lanes_all += pbs * kWidePpc;
        }
        const int mode = env_int("MAGUS_WIDE", -1);
        if (mode == 0) wide = false;
        else if (mode != 1)
            wide = wide && warps >= (int64_t)n_sm * env_int("MAGUS_WIDE_WARPS_PER_SM", 12) && 4 * lanes_used >= 3 * lanes_all;
    }
    if (wide) {
        p.n_seg = 1;
        p.seg_len = std::max(1, d.n_samples);
        p.seg_long = 0;
        p.warmup = 0;
        p.solo_warm = 8;
        p.kr = 1;
        for (const DevPolicy& q : h->lane) p.kr = std::max(p.kr, q.k);
        p.n_blocks = (d.n_samples + 31) / 32;
        // traces per CTA: the even count <= 16 that minimises the chains on the busiest SM,
        // ceil(CTAs / SMs) x traces x 16, with every CTA resident at once (2 per SM); MAGUS_WIDE_TPC overrides
        {
            int64_t pbs_all = 0;
            for (const LaunchGroup& g : h->groups) pbs_all += (g.nq + kWidePpc - 1) / kWidePpc;
            int best = kWideTpc;
            int64_t best_load = INT64_MAX;
            for (int t = kWideTpc; t >= 8; t -= 2) {
                if (t != kWideTpc && t > kWideTpc - 2) continue;   // a box starts at a 4-trace boundary: <= 14 fit
                const int64_t ctas = pbs_all * ((d.n_traces + t - 1) / t);
                if (ctas > 2 * (int64_t)n_sm && t != kWideTpc) continue;
                const int64_t load = ((ctas + n_sm - 1) / n_sm) * t;
                if (load < best_load) {
                    best_load = load;
                    best = t;
                }
            }
            const int te = env_int("MAGUS_WIDE_TPC", 0);
            p.wide_tpcu = (te >= 2 && te <= kWideTpc - 2 && te % 2 == 0) || te == kWideTpc ? te : best;
        }
        for (LaunchGroup& g : h->groups) {
            g.wide = true;
            g.solo = false;
            // chains per thread: 1; MAGUS_WIDE_NC=2: two policy points sharing the samples (7% fewer instructions,
            // but measured slower: cfg 3 10.7 vs 7.0 ms, profiles/r02_cfg3_wide.txt)
            const int nc = env_int("MAGUS_WIDE_NC", 1) == 2 ? 2 : 1;
            // the L stage (MAGUS_WIDE_L, default 1) when every lane policy has C <= 27, with
            // the |d| tune-flag test when every one has d*_dec == -d*_inc
            bool sym = true, lsign_ok = true;
            for (int q = g.q_base; q < g.q_base + g.nq; ++q) {
                sym = sym && h->lane[q].ddec == -h->lane[q].dinc;
                lsign_ok = lsign_ok && h->lane[q].C <= 27;
            }
            // MAGUS_WIDE_L: 2 (default) = the P stage, 1 = the L stage, 0 = MAGUS_WSTAGE1D
            const int wl = env_int("MAGUS_WIDE_L", 2);
            const int lv = (wl != 0 && lsign_ok) ? (wl == 2 ? (sym ? 4 : 3) : (sym ? 2 : 1)) : 0;
            g.kernel = wide_kernel_for(g.key, nc, lv);
            g.ng = 1;
            g.npw = 1;
            g.n_pblocks = (g.nq + kWidePpc - 1) / kWidePpc;
            g.n_tblocks = (d.n_traces + p.wide_tpcu - 1) / p.wide_tpcu;
            g.threads = p.wide_tpcu * kWidePpc / nc;
            g.smem = WideSmem::kBytes;
            g.n_ctas = g.n_pblocks * g.n_tblocks;
        }
        return;
    }
    // One MAGUS solo policy next to one or two TDP_DEFAULT baselines (config 5): MAGUS_COMBO=1 runs both launch groups
    // in one two-warp kernel sharing the TMA tiles (magus_replay_combo_kernel), so each trace byte is read once.  Off
    // by default: measured slower (config 5 replay 0.84 vs 0.69 ms) -- the replay is bound by
    // instruction issue and latency, not HBM, and at 128 registers a two-warp CTA leaves MAGUS 8 warps per SM.
    const bool combo = h->groups.size() == 2 && h->groups[0].key >= 1 && h->groups[0].key <= 3 &&
                       h->groups[0].nq == 1 && h->groups[1].key == 1000 + LANE_TDP && h->groups[1].nq <= 2 &&
                       kTC == 8 && env_int("MAGUS_COMBO", 0) != 0 && env_int("MAGUS_SOLO", 1) != 0 &&
                       env_int("MAGUS_SOLO_BAL", 20) == 20 && env_int("MAGUS_TDP_SOLO", 2) == 2;
    // One MAGUS solo policy (k <= 3, C <= 27) next to ONE TDP_DEFAULT baseline (config 5): the fused kernel
    // (magus_replay_fused_kernel, MAGUS_FUSE default 1) replays both in one warp per (tile group, segment) on the same
    // samples, so each trace byte is read once and loaded / converted / validated once for both chain kinds.
    const bool fuse = !combo && h->groups.size() == 2 && h->groups[0].key >= 1 && h->groups[0].key <= 3 &&
                      h->groups[0].nq == 1 && h->lane[h->groups[0].q_base].C <= 27 &&
                      h->groups[1].key == 1000 + LANE_TDP && h->groups[1].nq == 1 && kTC == 8 &&
                      env_int("MAGUS_FUSE", 1) != 0 && env_int("MAGUS_SOLO", 1) != 0 &&
                      (env_int("MAGUS_SOLO_BAL", 24) == 24 || env_int("MAGUS_SOLO_BAL", 24) == 20) &&
                      env_int("MAGUS_TDP_SOLO", 2) != 0;
    const int fused_ctas = env_int("MAGUS_FUSED_CTAS", 12) == 16 ? 16 : 12;   // per SM (the kernel's launch bound)
    int W = d.tuning_warmup > 0 ? d.tuning_warmup
                                : ((kmax + cmax - 1 + 31) / 32) * 32 + env_int("MAGUS_WARMUP_EXTRA", 0) + h->warm_extra;
    W = ((std::max(W, kmax + cmax - 1) + 31) / 32) * 32;
    const int N = std::max(1, d.n_samples);
    int base = 0;   // CTAs per segment over all launch groups
    for (const LaunchGroup& g : h->groups) base += g.n_tblocks * g.n_pblocks;
    int S = 1;
    int S_auto = 0;   // the automatic plan's segment count before rounding to 32-tick multiples
    p.seg_long = 0;
    if (forced_segments > 0) {
        S = forced_segments;
    } else if (d.tuning_segments > 0) {
        S = d.tuning_segments;
    } else {
        // enough consumer warps for `target` per SM (each warp holds 4 chains per lane, so one warp per
        // SM sub-partition already has ILP; more warps hide more latency but need more segments, and
        // every speculative segment boundary can mismatch)
        // target: 8 warps per resident CTA (16 per SM for the 2-CTA kinds) for EACH launch group on its
        // own -- the groups run concurrently but their per-tick costs differ (a MAGUS group next to cheap
        // TDP groups must still fill the GPU: cfg 5 step 1.39 -> 1.04 ms against a warp-weighted target)
        S = 1;
        for (const LaunchGroup& g : h->groups) {
            const int64_t wps = std::max<int64_t>(1, (int64_t)p.n_groups * g.nq);   // warps per segment
            const int target = env_int("MAGUS_TARGET_WARPS_PER_SM", 8 * minb_for(g.key));
            S = (int)std::max<int64_t>(S, ((int64_t)n_sm * target) / wps);
        }
        // the combined kernel: 8 two-warp CTAs per SM (16 warps: 8 MAGUS, 8 TDP)
        if (combo) S = std::max(1, (int)(((int64_t)n_sm * env_int("MAGUS_COMBO_CTAS_PER_SM", 8)) / std::max(1, p.n_groups)));
        if (fuse) S = std::max(1, (int)(((int64_t)n_sm * fused_ctas) / std::max(1, p.n_groups)));
        const int L0 = (((N + S - 1) / S) + 31) / 32 * 32;
        if (S > 1 && L0 < 4 * W) S = std::max(1, N / (4 * W));   // segments must dwarf their warm-up
        S_auto = S;
    }
    // the solo kernel's per-segment counters are exact fp32 integers: segments of at most 2^24 ticks
    S = std::max(S, (N + (1 << 24) - 1) >> 24);
    int L = (((N + S - 1) / S) + 31) / 32 * 32;
    if (L < 32) L = 32;
    S = (N + L - 1) / L;
    if (S > 1 && L < W) {   // forced segmentation too fine for the warm-up: fall back to fewer segments
        L = ((W + 31) / 32) * 32;
        S = (N + L - 1) / L;
    }
    // CTA balance: rounding the length up to 32 ticks can drop the count below the plan (config 2: 74 ->
    // 73 segments, 2,336 CTAs on 2,368 slots, so most SMs run 16 full CTAs while the mean is 15.8).  Keep
    // the planned count with two lengths instead: the first seg_long segments 32 ticks longer.
    if (S_auto > S && S_auto <= N / 32 && env_int("MAGUS_SEG_BALANCE", 1)) {
        const int Lb = (N / S_auto) / 32 * 32;
        const int extra = (N - S_auto * Lb + 31) / 32;   // < S_auto: N / S_auto - Lb < 32
        if (Lb >= 32 && Lb >= W && Lb + 32 <= (1 << 24)) {
            S = S_auto;
            L = Lb;
            p.seg_long = extra;
        }
    }
    p.n_seg = std::max(1, S);
    p.seg_len = L;
    p.warmup = p.n_seg > 1 ? W : 0;
    // the unified-stage solo kernel's own (shorter) warm-up: a multiple of 8 ticks covering k + C - 1
    p.solo_warm = std::min(std::max(((kmax + cmax - 1 + 7) / 8) * 8, (env_int("MAGUS_SOLO_WARM", 16) + 7) / 8 * 8),
                           std::max(p.warmup, 8));
    p.n_blocks = (d.n_samples + 31) / 32;
    // Spread small launches over every SM: while the launch groups together have fewer CTAs than
    // SMs, halve the widest CTA (policy warps first, then tile groups).
    auto total_ctas = [&]() {
        int t = 0;
        for (const LaunchGroup& g : h->groups) t += p.n_seg * g.n_tblocks * g.n_pblocks;
        return t;
    };
    while (total_ctas() < n_sm) {
        LaunchGroup* wide = nullptr;
        for (LaunchGroup& g : h->groups)
            if (g.ng * g.npw > 1 && (!wide || g.ng * g.npw > wide->ng * wide->npw)) wide = &g;
        if (!wide) break;
        if (wide->npw > 1) wide->npw = (wide->npw + 1) / 2;
        else wide->ng = (wide->ng + 1) / 2;
        wide->n_pblocks = (wide->nq + wide->npw - 1) / wide->npw;
        wide->n_tblocks = std::max(1, (p.n_groups + wide->ng - 1) / wide->ng);
        wide->threads = wide->ng * wide->npw * 32;
        wide->smem = Smem::bytes(wide->ng);
    }
    for (LaunchGroup& g : h->groups) {
        g.n_ctas = p.n_seg * g.n_tblocks * g.n_pblocks;
        // one policy warp per tile group: one-warp CTAs with CTA-uniform pipeline state (replay_solo.cuh)
        bool sym = true;   // every lane policy of the group has d*_dec == -d*_inc (the |d| tune-flag test)
        // the integer fp32 -> fp64 sample conversion changes no decision when both thresholds are >= 2^-60 in
        // magnitude and B_lo is a normal fp32
        bool bits_ok = h->B_lo >= 0x1p-126f;
        bool lsign_ok = true;   // the L stage's biased scaled count stays within int32: C <= 27
        bool lbatch_ok = true;  // the batched flag log: every flag leaving during a stage logged before it, the
                                // leaving flag (bit C - 1 + 8 after the stage shift) inside the word: 8 <= C <= 24
        for (int q = g.q_base; q < g.q_base + g.nq; ++q) {
            const DevPolicy& lp = h->lane[q];
            sym = sym && lp.ddec == -lp.dinc;
            bits_ok = bits_ok && lp.dinc >= 0x1p-60 && lp.ddec <= -0x1p-60;
            lsign_ok = lsign_ok && lp.C <= 27;
            lbatch_ok = lbatch_ok && lp.C >= 8 && lp.C <= 24;
        }
        ReplayKernel sk = solo_kernel_for(g.key, sym, bits_ok, lsign_ok, h->open_fast, lbatch_ok);
        g.solo = sk && g.npw == 1 && kTC == 8 && env_int("MAGUS_SOLO", 1) != 0;
        if (g.solo) {
            g.kernel = sk;
            g.ng = 1;
            g.n_tblocks = p.n_groups;
            g.n_pblocks = g.nq;
            g.threads = 32;
            g.smem = SoloSmem<kTC, kNStage>::kBytes + env_int("MAGUS_SOLO_SMEM_PAD", 0);   // pad: occupancy probes
            g.n_ctas = p.n_seg * p.n_groups * g.nq;
        }
        // TDP_DEFAULT groups: the TDP solo kernel, NP policies per warp sharing the samples (MAGUS_TDP_SOLO = NP in
        // {1, 2}; 0: the multi-warp kernel)
        const int tnp_env = env_int("MAGUS_TDP_SOLO", 2);
        const int tnp = std::min(tnp_env, g.nq);   // one TDP policy: no idle second chain set per lane
        if (g.key == 1000 + LANE_TDP && kTC == 8 && (tnp_env == 1 || tnp_env == 2)) {
            g.solo = true;
            // the first launch group validates the samples (A17); a later TDP group skips the maximum
            const bool first = &g == &h->groups.front();
            g.kernel = tnp == 2 ? (ReplayKernel)magus_replay_tsolo_kernel<2, kTC, kNStage>
                       : first  ? (ReplayKernel)magus_replay_tsolo_kernel<1, kTC, kNStage, true>
                                : (ReplayKernel)magus_replay_tsolo_kernel<1, kTC, kNStage, false>;
            g.ng = 1;
            g.npw = 1;
            g.n_tblocks = p.n_groups;
            g.n_pblocks = (g.nq + tnp - 1) / tnp;
            g.threads = 32;
            g.smem = SoloSmem<kTC, kNStage>::kBytes;
            g.n_ctas = p.n_seg * p.n_groups * g.n_pblocks;
        }
    }
    if (fuse && h->groups[0].solo && h->groups[1].solo) {
        LaunchGroup& gm = h->groups[0];
        const DevPolicy& pt = h->lane[h->groups[1].q_base];
        const float kB_lo = d.model.observe == 1 ? __builtin_inff() : h->B_lo;   // the kernels' throttle bound
        const bool up = !(kB_lo >= pt.astar_lo) && env_int("MAGUS_FUSED_UP", 1) != 0;   // their a_lo is +inf
        // the batched tune-flag log (solo BAL 24 / 25) when 8 <= C <= 24 and MAGUS_SOLO_BAL keeps its default
        const int mc = h->lane[gm.q_base].C;
        const bool lb = mc >= 8 && mc <= 24 && env_int("MAGUS_SOLO_BAL", 24) == 24;
        gm.kernel = fused_kernel_for(gm.key, h->lane[gm.q_base].ddec == -h->lane[gm.q_base].dinc, fused_ctas, up, lb);
        gm.threads = 32;
        gm.smem = SoloSmem<kTC, kNStage>::kBytes;
        gm.n_ctas = p.n_seg * p.n_groups;
        h->groups[1].fused = true;
    }
    if (combo && h->groups[0].solo && h->groups[1].solo) {
        LaunchGroup& gm = h->groups[0];
        gm.kernel = combo_kernel_for(gm.key, h->groups[1].nq);
        gm.threads = 64;
        gm.smem = SoloSmem<kTC, kNStage>::kBytes + kNStage * sizeof(uint64_t);   // + the empty barriers
        gm.n_ctas = p.n_seg * p.n_groups;
        h->groups[1].fused = true;
    }
}

// Cross-rank consistency of a run with the exchange on (collective; called by create on every rank).  Every rank
// writes a record: a header every rank fills identically (model, n_samples, n_policies_global) and one slot per
// global policy, filled with the policy's bytes by the ranks that own it (their slice) and neutral elsewhere
// (0x00 for the MAX copy, 0xFF for the MIN copy).  After a byte-wise MAX and MIN allreduce the two copies are
// equal iff all ranks agree on the header, every owner of a policy passed the same parameters, and every
// global policy has an owner.
static magus_status check_ranks_agree(magus_replay_t* h) {
    const magus_replay_desc& d = h->desc;
    struct Header {
        magus_model model;
        int32_t n_samples, n_policies_global;
    } hd;
    std::memset(&hd, 0, sizeof(hd));
    hd.model = d.model;
    hd.n_samples = d.n_samples;
    hd.n_policies_global = h->P_glob;
    const size_t slot = sizeof(magus_policy), n_bytes = sizeof(Header) + (size_t)h->P_glob * slot;
    std::vector<uint8_t> mx(n_bytes, 0x00), mn(n_bytes, 0xFF);
    std::memcpy(mx.data(), &hd, sizeof(hd));
    std::memcpy(mn.data(), &hd, sizeof(hd));
    for (int i = 0; i < d.n_policies; ++i) {
        magus_policy p = h->pols[i];
        p._reserved0 = 0;
        uint8_t* a = mx.data() + sizeof(Header) + (size_t)(h->p_off + i) * slot;
        std::memcpy(a, &p, slot);
        std::memcpy(mn.data() + (a - mx.data()), &p, slot);
    }
    uint8_t* dbuf = nullptr;
    cudaError_t ce = cudaMalloc(&dbuf, 2 * n_bytes);
    if (ce != cudaSuccess) return cuda_fail(h, ce, "cudaMalloc rank check");
    cudaStream_t st = nullptr;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaMemcpyAsync(dbuf, mx.data(), n_bytes, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dbuf + n_bytes, mn.data(), n_bytes, cudaMemcpyHostToDevice, st);
    ncclResult_t r1 = nccl().AllReduce(dbuf, dbuf, n_bytes, ncclUint8, ncclMax, h->comm, st);
    ncclResult_t r2 = nccl().AllReduce(dbuf + n_bytes, dbuf + n_bytes, n_bytes, ncclUint8, ncclMin, h->comm, st);
    cudaMemcpyAsync(mx.data(), dbuf, n_bytes, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(mn.data(), dbuf + n_bytes, n_bytes, cudaMemcpyDeviceToHost, st);
    ce = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    cudaFree(dbuf);
    if (r1 != ncclSuccess || r2 != ncclSuccess)
        return fail(h, MAGUS_ERR_NCCL, std::string("rank check allreduce: ") +
                                           nccl().GetErrorString(r1 != ncclSuccess ? r1 : r2));
    if (ce != cudaSuccess) return cuda_fail(h, ce, "rank check");
    if (std::memcmp(mx.data(), mn.data(), sizeof(Header)) != 0)
        return fail(h, MAGUS_ERR_CONFIG, "ranks disagree on the model, n_samples or n_policies_global");
    for (int g = 0; g < h->P_glob; ++g) {
        const uint8_t* a = mx.data() + sizeof(Header) + (size_t)g * slot;
        const uint8_t* b = mn.data() + sizeof(Header) + (size_t)g * slot;
        if (std::memcmp(a, b, slot) == 0) continue;
        bool unowned = true;
        for (size_t i = 0; i < slot; ++i) unowned = unowned && a[i] == 0x00 && b[i] == 0xFF;
        return fail(h, MAGUS_ERR_CONFIG, unowned ? "global policy " + std::to_string(g) + " is owned by no rank"
                                                 : "ranks disagree on the parameters of global policy " +
                                                       std::to_string(g));
    }
    return MAGUS_OK;
}

extern "C" magus_status magus_replay_create(const magus_replay_desc* desc, magus_replay_t** out) {
    if (out) *out = nullptr;
    if (!desc || !out) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "magus_replay_create: NULL argument");
    const magus_replay_desc& d = *desc;
    if (d.n_traces < 0 || d.n_samples < 0) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "n_traces/n_samples must be >= 0");
    if (d.n_policies < 1 || !d.policies) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "n_policies must be >= 1 with a policy array");
    if (d.trace_stride < d.n_traces) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "trace_stride must be >= n_traces");
    if (d.trace_stride % 4 != 0) return fail(nullptr, MAGUS_ERR_ALIGN, "trace_stride must be a multiple of 4 floats (16 B, TMA)");
    if (d.world < 1 || d.rank < 0 || d.rank >= d.world) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "need 0 <= rank < world");
    if (d.world > 1 && !d.nccl_unique_id) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "world > 1 needs nccl_unique_id");
    if ((d.flags & MAGUS_F_DUMP_DECISIONS) &&
        (d.dump_first_trace < 0 || d.dump_n_traces < 0 || d.dump_first_trace + d.dump_n_traces > d.n_traces))
        return fail(nullptr, MAGUS_ERR_INVALID_ARG, "dump window outside [0, n_traces)");
    if ((d.flags & MAGUS_F_WALLCLOCK) && (d.flags & MAGUS_F_DUMP_WORDS))
        return fail(nullptr, MAGUS_ERR_INVALID_ARG, "MAGUS_F_DUMP_WORDS is not available with MAGUS_F_WALLCLOCK");
    if (d.tuning_warmup < 0 || d.tuning_warmup % 32 != 0)
        return fail(nullptr, MAGUS_ERR_INVALID_ARG, "tuning_warmup must be a multiple of 32");
    const int P_glob = d.n_policies_global > 0 ? d.n_policies_global : d.n_policies;
    if (d.n_policies_global < 0 || d.policy_offset < 0 || (int64_t)d.policy_offset + d.n_policies > P_glob)
        return fail(nullptr, MAGUS_ERR_INVALID_ARG,
                    "policy slice [policy_offset, policy_offset + n_policies) must lie in [0, n_policies_global)");
    std::string e = validate_model(d.model);
    if (!e.empty()) return fail(nullptr, MAGUS_ERR_CONFIG, "model." + e);
    for (int i = 0; i < d.n_policies; ++i) {
        e = validate_policy(d.policies[i], i);
        if (!e.empty()) return fail(nullptr, MAGUS_ERR_CONFIG, e);
    }
    int dev = 0, n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
        cudaGetLastError();
        return fail(nullptr, MAGUS_ERR_CUDA, "no CUDA device (there is no CPU fallback)");
    }
    cudaGetDevice(&dev);
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);

    magus_replay_t* h = new magus_replay_t();
    h->desc = d;
    h->pols.assign(d.policies, d.policies + d.n_policies);
    h->desc.policies = nullptr;
    h->desc.nccl_unique_id = nullptr;
    const magus_model& m = d.model;
    h->B_lo = (float)bandwidth_at(m.f_min_ghz, m);
    h->B_hi = (float)bandwidth_at(m.f_max_ghz, m);
    float bwf = (float)m.bw_max_gbps;
    if ((double)bwf > m.bw_max_gbps) bwf = nextafterf(bwf, 0.0f);
    h->bwbits = fbits(bwf);
    h->P_lo = pkg_power_at(m.f_min_ghz, m);
    h->P_hi = pkg_power_at(m.f_max_ghz, m);

    for (int i = 0; i < d.n_policies; ++i) {
        const magus_policy& p = h->pols[i];
        if (p.kind == MAGUS_POLICY_STATIC_MAX) {
            h->smax.push_back(i);
            continue;
        }
        DevPolicy q{};
        q.one = 1;
        q.B_hi = h->B_hi;
        q.policy_index = i;
        q.k = 1;
        q.C = 1;
        q.s_min = 0;
        q.logmask = 1;
        q.dinc = INFINITY;
        q.ddec = -INFINITY;
        q.astar_lo = q.astar_hi = INFINITY;
        if (p.kind == MAGUS_POLICY_MAGUS) {
            q.kind = LANE_MAGUS;
            q.k = p.deriv_ticks;
            q.C = p.tune_log_capacity;
            q.logmask = q.C >= 64 ? ~0ULL : ((1ULL << q.C) - 1ULL);
            const double L = (double)p.deriv_ticks * m.sample_period_s;
            q.dinc = derive_dinc(L, p.inc_threshold);
            q.ddec = derive_ddec(L, p.dec_threshold);
            q.s_min = derive_smin(q.C, p.high_freq_threshold);
            q.sticky = q.k >= q.s_min ? 1 : 0;
            q.smin_sc = q.C <= kMaxC32 ? (uint32_t)q.s_min << (q.C - 1) : 0u;
            q.f0 = 0;
            q.guess_f = 0;   // speculative segment start
        } else if (p.kind == MAGUS_POLICY_STATIC_MIN) {
            q.kind = LANE_STATIC_MIN;
            q.f0 = q.guess_f = 0;
        } else {
            q.kind = LANE_TDP;
            q.astar_lo = derive_astar(h->P_lo, m, p);
            q.astar_hi = derive_astar(h->P_hi, m, p);
            q.f0 = 1;        // the default sits at max
            q.guess_f = 1;
            // A TDP_DEFAULT policy whose budget is never reached at f_max -- a*_hi above every observable A (A =
            // min(D, B_hi) with valid D <= bw_max, A17) -- starts at f_max and never leaves it: its record
            // is STATIC_MAX's, in closed form (config 5's 270 W: 200 + 0.5 x 20 W < 256.5 W).
            // MAGUS_NO_TDP_CLOSED=1 replays it anyway.
            if (q.astar_hi > std::min(bwf, h->B_hi) && !env_int("MAGUS_NO_TDP_CLOSED", 0)) {
                h->smax.push_back(i);
                continue;
            }
        }
        h->lane.push_back(q);
    }
    if (h->lane.empty()) {   // only STATIC_MAX policies: a validate-only lane still scans the samples (A17)
        DevPolicy q{};
        q.one = 1;
        q.kind = LANE_VALIDATE;
        q.k = 1;
        q.C = 1;
        q.logmask = 1;
        q.policy_index = -1;
        h->lane.push_back(q);
    }
    // digest of an all-f_max command stream (STATIC_MAX), DESIGN.md section 5
    {
        const int64_t nb = (d.n_samples + 31) / 32;
        uint32_t dc = 0;
        for (int64_t b = 0; b < nb; ++b) {
            const int n = (int)std::min<int64_t>(32, d.n_samples - b * 32);
            const uint32_t wc = n == 32 ? 0xFFFFFFFFu : (((1u << n) - 1u) << (32 - n));
            dc += wc * digest_key((uint64_t)b).x;
        }
        h->digest_all_hi = digest_pack(dc, 0);
    }

    std::stable_sort(h->lane.begin(), h->lane.end(),
                     [](const DevPolicy& a, const DevPolicy& b) { return ticker_key(a) < ticker_key(b); });
    h->wall = (d.flags & MAGUS_F_WALLCLOCK) != 0;
    choose_geometry(h, n_sm, h->wall ? 1 : 0);   // wall-clock rounds: no time segmentation
    h->n_sm = n_sm;
    h->alloc_segments = h->rp.n_seg;
    ReplayParams& p = h->rp;
    // the kernels' throttle threshold: B_lo; +inf in open loop (A30: A = D, no tick is ever throttled).
    // The epilogue keeps the true B_lo (its throttling excess is then 0).
    p.B_lo = d.model.observe == 1 ? __builtin_inff() : h->B_lo;
    p.B_hi = h->B_hi;
    p.bwbits = h->bwbits;
    p.solo_flags = env_int("MAGUS_SOLO_SYNTH", 0) ? 1u : 0u;   // off: see DESIGN.md section 9

    const int Q = p.n_lane, S = p.n_seg;
    const size_t nst = (size_t)3 * Q * S * std::max(1, d.n_traces);   // entry, exit, staged exit
    const size_t nchain = (size_t)Q * std::max(1, d.n_traces);
    cudaError_t ce;
#define ALLOC(ptr, n)                                         \
    if ((ce = dalloc(h, &(ptr), (n))) != cudaSuccess) {       \
        magus_status s_ = cuda_fail(h, ce, "cudaMalloc " #ptr); \
        magus_replay_destroy(h);                              \
        return s_;                                            \
    }
    DevPolicy* dpol;
    ALLOC(dpol, h->lane.size());
    h->d_pol = dpol;
    ALLOC(p.st_f, nst);
    ALLOC(p.st_log, nst);
    ALLOC(p.st_first, nst);
    ALLOC(p.st_ring, nst * p.kr);
    ALLOC(h->d_chain, nchain * kChainBytes);   // per-chain totals, zeroed by every run
    p.c_sexc = (double*)h->d_chain;
    p.c_digest = (unsigned long long*)(h->d_chain + nchain * 8);
    p.c_nhi = (uint32_t*)(h->d_chain + nchain * 16);
    p.c_nthr = p.c_nhi + nchain;
    p.c_trans = p.c_nthr + nchain;
    p.c_ev = p.c_trans + nchain;
    p.c_lock = p.c_ev + nchain;
    p.c_vmax = p.c_lock + nchain;
    {   // digest keys of every 32-tick block
        std::vector<uint2> keys((size_t)std::max(1, p.n_blocks));
        for (size_t b = 0; b < keys.size(); ++b) keys[b] = digest_key((uint64_t)b);
        uint2* dk;
        ALLOC(dk, keys.size());
        ce = cudaMemcpy(dk, keys.data(), keys.size() * sizeof(uint2), cudaMemcpyHostToDevice);
        if (ce != cudaSuccess) {
            magus_status s_ = cuda_fail(h, ce, "cudaMemcpy digest keys");
            magus_replay_destroy(h);
            return s_;
        }
        p.dkeys = dk;
    }
    // the replay kernels' words: returned with MAGUS_F_DUMP_WORDS, and the source of the decision dump's codes
    // (magus_decode_kernel) with MAGUS_F_DUMP_DECISIONS
    if ((d.flags & MAGUS_F_DUMP_WORDS) || ((d.flags & MAGUS_F_DUMP_DECISIONS) && !h->wall)) {
        ALLOC(p.words, (size_t)Q * std::max(1, d.n_traces) * std::max(1, p.n_blocks) * 2);
    } else {
        p.words = nullptr;
    }
    ALLOC(h->d_rec, (size_t)std::max(1, d.n_traces) * d.n_policies);
    if (h->wall) {
        ALLOC(h->d_wrec, nchain);
    }
    h->n_chunks = std::max(1, (d.n_traces + kTotThreads - 1) / kTotThreads);
    const size_t n_part = (size_t)d.n_policies * h->n_chunks * MAGUS_N_TOTALS;
    ALLOC(h->d_out, n_part * sizeof(double) + 4 * sizeof(unsigned int));
    h->d_totals = (double*)h->d_out;
    h->d_flag = (unsigned int*)(h->d_out + n_part * sizeof(double));
    h->P_glob = P_glob;
    h->p_off = d.policy_offset;
    h->xchg = d.world > 1 || (d.flags & MAGUS_F_NCCL);
    if (h->xchg) {
        ALLOC(h->d_fin, (size_t)P_glob * MAGUS_N_TOTALS);
        ALLOC(h->d_fin_local, (size_t)P_glob * MAGUS_N_TOTALS);
        cudaMemset(h->d_fin_local, 0, (size_t)P_glob * MAGUS_N_TOTALS * sizeof(double));   // rows of other slices
    }
    ALLOC(h->d_first_low, (size_t)2 * std::max(1, d.n_traces));
    ALLOC(h->d_errkey, 1);
    if (!h->smax.empty()) {
        ALLOC(h->d_smax, h->smax.size());
    }
    ALLOC(h->d_lane_of_policy, d.n_policies);
    if ((d.flags & MAGUS_F_DUMP_DECISIONS) && d.dump_n_traces > 0 && d.n_samples > 0) {
        ALLOC(h->d_codes, (size_t)d.n_samples * d.dump_n_traces * d.n_policies);
    }
    {   // chain-walk fix-up
        ALLOC(h->fx.first_bad, (size_t)Q * std::max(1, d.n_traces));
        {   // INT_MAX ("no wrong entry") between runs: the walk kernel restores what it reads
            std::vector<int32_t> inf((size_t)Q * std::max(1, d.n_traces), 0x7FFFFFFF);
            cudaMemcpy(h->fx.first_bad, inf.data(), inf.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
        }
        h->replan_frac = env_int("MAGUS_REPLAN_PCT", 101) / 100.0;   // > 100: never (the chain walk's cost
                                                                      // does not grow with the segment count)
    }
#undef ALLOC
    p.pol = h->d_pol;
    p.first_low = h->d_first_low;
    cudaMemset(h->d_chain, 0, nchain * kChainBytes);   // zero at every run start from here on (totals kernel)
    h->pdl = !env_int("MAGUS_NO_PDL", 0);
    if ((ce = cudaMemcpy(h->d_pol, h->lane.data(), h->lane.size() * sizeof(DevPolicy), cudaMemcpyHostToDevice)) !=
        cudaSuccess) {
        magus_status s = cuda_fail(h, ce, "cudaMemcpy policies");
        magus_replay_destroy(h);
        return s;
    }
    if (!h->smax.empty())
        cudaMemcpy(h->d_smax, h->smax.data(), h->smax.size() * sizeof(int), cudaMemcpyHostToDevice);
    {
        std::vector<int> lop(d.n_policies, -1);
        for (size_t q = 0; q < h->lane.size(); ++q) {
            if (h->lane[q].policy_index >= 0) lop[h->lane[q].policy_index] = (int)q;
            else h->validate_lane = (int)q;
        }
        cudaMemcpy(h->d_lane_of_policy, lop.data(), lop.size() * sizeof(int), cudaMemcpyHostToDevice);
    }

    EpiParams& ep = h->ep;
    ep.n_policies = d.n_policies;
    ep.n_samples = d.n_samples;
    ep.Delta = m.sample_period_s;
    ep.P_lo = h->P_lo;
    ep.P_hi = h->P_hi;
    ep.P_gpu = m.p_gpu_active_w;
    ep.B_lo_d = (double)h->B_lo;
    ep.rec = h->d_rec;
    ep.flag_invalid = h->d_flag;
    ep.fix_rounds = (int*)(h->d_flag + 1);
    ep.fix_segments = (unsigned long long*)(h->d_flag + 2);

    for (int i = 0; i < 5; ++i) cudaEventCreate(&h->ev[i]);
    cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming);
    for (size_t g = 1; g < h->groups.size(); ++g) {
        cudaStream_t st;
        cudaEvent_t ev;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        h->aux.push_back(st);
        h->join_ev.push_back(ev);
    }
    if (d.flags & MAGUS_F_TIMING) {
        h->tev.resize(5 * magus_replay::kTimingRing);
        for (cudaEvent_t& e : h->tev) cudaEventCreate(&e);
    }
    for (const LaunchGroup& g : h->groups) {
        ce = cudaFuncSetAttribute((const void*)g.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
        if (ce != cudaSuccess) {
            magus_status s = cuda_fail(h, ce, "cudaFuncSetAttribute smem");
            magus_replay_destroy(h);
            return s;
        }
    }
    if (h->xchg) {
        if (!nccl_ok()) {
            magus_status s = fail(h, MAGUS_ERR_NCCL, "libnccl.so.2 could not be loaded");
            g_error = h->err;
            magus_replay_destroy(h);
            return s;
        }
        ncclUniqueId id;
        if (desc->nccl_unique_id) {
            std::memcpy(&id, desc->nccl_unique_id, sizeof(id));
        } else {   // world == 1 (MAGUS_F_NCCL): a one-rank communicator of our own
            ncclResult_t r = nccl().GetUniqueId(&id);
            if (r != ncclSuccess) {
                magus_status s = fail(h, MAGUS_ERR_NCCL, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
                magus_replay_destroy(h);
                return s;
            }
        }
        ncclResult_t r = nccl().CommInitRank(&h->comm, d.world, id, d.rank);
        if (r != ncclSuccess) {
            magus_status s = fail(h, MAGUS_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
            h->comm = nullptr;
            magus_replay_destroy(h);
            return s;
        }
        magus_status s = check_ranks_agree(h);
        if (s != MAGUS_OK) {
            g_error = h->err;
            magus_replay_destroy(h);
            return s;
        }
    }
    *out = h;
    return MAGUS_OK;
}

extern "C" void magus_replay_destroy(magus_replay_t* h) {
    if (!h) return;
    if (h->ran && h->run_stream) cudaStreamSynchronize(h->run_stream);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->graph) cudaGraphDestroy(h->graph);
    if (h->comm && nccl_ok()) nccl().CommDestroy(h->comm);
    for (void* a : h->allocs) cudaFree(a);
    for (int i = 0; i < 5; ++i)
        if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    for (cudaEvent_t e : h->tev) cudaEventDestroy(e);
    for (cudaEvent_t e : h->join_ev) cudaEventDestroy(e);
    for (cudaStream_t st : h->aux) cudaStreamDestroy(st);
    if (h->fork_ev) cudaEventDestroy(h->fork_ev);
    delete h;
}

static magus_status encode_tmap(magus_replay_t* h, const float* d_trace) {
    if (h->tmap_ptr == d_trace) return MAGUS_OK;
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(h, MAGUS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
    const magus_replay_desc& d = h->desc;
    cuuint64_t gdim[2] = {(cuuint64_t)d.n_traces, (cuuint64_t)d.n_samples};
    cuuint64_t gstride[1] = {(cuuint64_t)d.trace_stride * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)kTracesPerWarp, (cuuint32_t)kTC};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&h->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)d_trace, gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(h, MAGUS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    cuuint32_t box_w[2] = {(cuuint32_t)kWideTpc, (cuuint32_t)kWideTC};
    r = enc(&h->tmap_w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)d_trace, gdim, gstride, box_w, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(h, MAGUS_ERR_CUDA, "cuTensorMapEncodeTiled (wide) failed: " + std::to_string((int)r));
    h->tmap_ptr = d_trace;
    return MAGUS_OK;
}

// Enqueues one whole run on stream s (also used to capture the run's CUDA graph); tv = the 5 timing
// events of this run (nullptr without MAGUS_F_TIMING).
static magus_status enqueue_run(magus_replay_t* h, const float* d_trace, const float* d_w, cudaStream_t s,
                                cudaEvent_t* tv, bool capturing) {
    // inside a stream capture, only "external" records become event-record nodes of the graph
    // inside a capture, the event-record node just added is the stream's only capture dependency: keep
    // it with its timing slot so that graph replays can re-point it (launch_graph)
    auto rec = [&](int k) -> cudaError_t {
        if (!capturing) return cudaEventRecord(tv[k], s);
        cudaError_t e = cudaEventRecordWithFlags(tv[k], s, cudaEventRecordExternal);
        if (e != cudaSuccess) return e;
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        e = cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd);
        if (e == cudaSuccess && nd == 1) h->g_events.push_back({deps[0], k});
        return e;
    };
    const magus_replay_desc& d = h->desc;
    const bool has_work = d.n_traces > 0 && d.n_samples > 0;
    const bool timing = tv != nullptr;   // events around the replay kernel(s)
    const bool detail = timing && (d.flags & MAGUS_F_TIMING_DETAIL);   // ... and around every phase
    ReplayParams p = h->rp;
    EpiParams ep = h->ep;
    ep.w = d_w;
    if (detail) CU(h, rec(0));
    {
        // pre-pass: zeroes the run's flag words; for segmented runs also the speculation aid
        // (first subsampled low / high tick of every trace).  The per-chain totals are
        // already zero (creation, then the previous run's totals kernel).
        const bool seg = has_work && p.n_seg > 1;
        const int n_blk = seg ? (d.n_traces + kPrepassTraces - 1) / kPrepassTraces : 1;
        CU(h, launch_k(magus_prepass_kernel, dim3((unsigned)n_blk), dim3(kPrepassTraces * kPrepassSlices), 0, s, false,
                       d_trace, d.n_traces, d.n_samples, (int64_t)d.trace_stride, h->B_lo, 256,
                       seg ? h->d_first_low : (int*)nullptr, (uint32_t*)h->d_flag, 4));
    }
    if (timing) CU(h, rec(1));
    if (has_work && h->wall && env_int("MAGUS_WALL_ROUNDMAJOR", 0)) {
        // wall-clock governor rounds (A32), the loop as written: one thread per chain, every lane
        WallParams wp{h->d_wrec, h->d_codes, d.dump_first_trace, d.dump_n_traces, d.n_policies};
        dim3 gw((unsigned)((d.n_traces + 127) / 128), (unsigned)p.n_lane);
        CU(h, launch_k(magus_wallclock_kernel, gw, dim3(128), 0, s, h->pdl && !timing, p, ep, wp, d_trace));
    } else if (has_work && h->wall) {
        // wall-clock governor rounds (A32), entry-major: one thread per chain, one kernel per chain kind
        // (launch group), the groups concurrent; no segmentation and no fix-up
        WallParams wp{h->d_wrec, h->d_codes, d.dump_first_trace, d.dump_n_traces, d.n_policies};
        const int G = (int)h->groups.size();
        if (G > 1) {
            CU(h, cudaEventRecord(h->fork_ev, s));
            for (int g = 1; g < G; ++g) CU(h, cudaStreamWaitEvent(h->aux[g - 1], h->fork_ev, 0));
        }
        for (int gi = 0; gi < G; ++gi) {
            const LaunchGroup& g = h->groups[gi];
            dim3 gw((unsigned)((d.n_traces + 127) / 128), (unsigned)g.nq);
            CU(h, launch_k(wall_kernel_for(g.key, (int64_t)d.n_traces * p.n_lane, h->n_sm), gw, dim3(128), 0, gi == 0 ? s : h->aux[gi - 1],
                           h->pdl && G == 1 && !timing, p, ep, wp, g.q_base, d_trace));
        }
        for (int g = 1; g < G; ++g) {
            CU(h, cudaEventRecord(h->join_ev[g - 1], h->aux[g - 1]));
            CU(h, cudaStreamWaitEvent(s, h->join_ev[g - 1], 0));
        }
    } else if (has_work) {
        // launch groups (one chain kind each) run concurrently: fork onto auxiliary streams and join
        // (parallel branches when the run is captured as a graph)
        const int G = (int)h->groups.size();
        int GL = 0;   // launches: a fused group is replayed by the previous group's launch
        for (const LaunchGroup& g : h->groups) GL += g.fused ? 0 : 1;
        if (GL > 1) {
            CU(h, cudaEventRecord(h->fork_ev, s));
            for (int g = 1; g < GL; ++g) CU(h, cudaStreamWaitEvent(h->aux[g - 1], h->fork_ev, 0));
        }
        for (int gi = 0, li = 0; gi < G; ++gi) {
            const LaunchGroup& g = h->groups[gi];
            if (g.fused) continue;   // replayed by the previous group's combined launch
            cudaStream_t gs = li == 0 ? s : h->aux[li - 1];
            ++li;
            ReplayParams pg = p;
            pg.q_base = g.q_base;
            pg.nq = g.nq;
            if (gi + 1 < G && h->groups[gi + 1].fused) {
                pg.q_base2 = h->groups[gi + 1].q_base;
                pg.nq2 = h->groups[gi + 1].nq;
            }
            pg.ng = g.ng;
            pg.npw = g.npw;
            pg.n_tblocks = g.n_tblocks;
            pg.n_pblocks = g.n_pblocks;
            CU(h, launch_k(g.kernel, dim3((unsigned)g.n_ctas), dim3((unsigned)g.threads), g.smem, gs,
                           h->pdl && GL == 1 && !timing, g.wide ? h->tmap_w : h->tmap, pg));
        }
        for (int g = 1; g < GL; ++g) {
            CU(h, cudaEventRecord(h->join_ev[g - 1], h->aux[g - 1]));
            CU(h, cudaStreamWaitEvent(s, h->join_ev[g - 1], 0));
        }
    }
    if (timing) CU(h, rec(2));
    if (d.n_traces > 0) {
        bool open_fix = h->open_fast;
        for (const LaunchGroup& g : h->groups) open_fix = open_fix && g.solo;
        if (has_work && p.n_seg > 1 && open_fix) {
            // open loop: wrong entry levels corrected in closed form from each segment's first event (section 9b)
            for (const LaunchGroup& g : h->groups)
                CU(h, launch_k(magus_fix_openloop_kernel, dim3((unsigned)((d.n_traces + 3) / 4), (unsigned)g.nq),
                               dim3(128), 0, s, h->pdl && !timing, p, ep, g.q_base));
        } else if (has_work && p.n_seg > 1) {
            // exact fix-up: the first wrong entry of every chain, then one walk per
            // chain in time order from there (magus_fix_lockstep_kernel; magus_fix_walk_kernel for the rest)
            dim3 gc((unsigned)((d.n_traces + 255) / 256), (unsigned)(p.n_seg - 1), (unsigned)p.n_lane);
            CU(h, launch_k(magus_fix_mark_kernel, gc, dim3(256), 0, s, h->pdl && !timing, p, h->fx));
            // the launch groups' walks are independent (different chains): concurrent streams (parallel
            // graph branches), like the replay launches
            std::vector<const LaunchGroup*> wg;
            for (const LaunchGroup& g : h->groups)
                if (walk_kernel_for(g.key)) wg.push_back(&g);
            const int W = (int)wg.size();
            if (W > 1) {
                CU(h, cudaEventRecord(h->fork_ev, s));
                for (int i = 1; i < W; ++i) CU(h, cudaStreamWaitEvent(h->aux[i - 1], h->fork_ev, 0));
            }
            for (int i = 0; i < W; ++i) {
                const LaunchGroup& g = *wg[i];
                // split walk: 64-thread CTAs of 32 traces; lockstep walk: one-warp CTAs (a walk is latency-bound)
                const int tpb = split_walk(g.key) ? 64 : lockstep_walk(g.key) ? 32 : 128;
                const int per_cta = split_walk(g.key) ? 32 : tpb;   // traces per CTA
                dim3 gw((unsigned)((d.n_traces + per_cta - 1) / per_cta), (unsigned)g.nq);
                CU(h, launch_k(walk_kernel_for(g.key), gw, dim3(tpb), 0, i == 0 ? s : h->aux[i - 1], h->pdl && i == 0,
                               p, ep, h->fx, g.q_base, d_trace));
            }
            for (int i = 1; i < W; ++i) {
                CU(h, cudaEventRecord(h->join_ev[i - 1], h->aux[i - 1]));
                CU(h, cudaStreamWaitEvent(s, h->join_ev[i - 1], 0));
            }
        }
    }
    if (detail) CU(h, rec(3));
    {
        // per-trace records and per-(policy, trace chunk) fixed-order partial sums (the host adds the chunks)
        CU(h, launch_k(magus_totals_kernel, dim3(d.n_policies, h->n_chunks), dim3(kTotThreads), 0, s,
                       h->pdl && !detail, p, ep, (const int*)h->d_lane_of_policy, h->validate_lane, h->digest_all_hi,
                       (d.flags & MAGUS_F_PER_TRACE_STATS) ? 1 : 0, (const TraceRec*)(has_work ? h->d_wrec : nullptr),
                       h->d_totals));
    }
    if (h->xchg) {
        // this rank's per-policy sums into its slice rows of the global [P_glob][13], then one allreduce (sum)
        CU(h, launch_k(magus_chunk_sum_kernel, dim3(d.n_policies), dim3(32), 0, s, h->pdl && !detail,
                       (const double*)h->d_totals, h->n_chunks, h->d_fin_local + (size_t)h->p_off * MAGUS_N_TOTALS));
        ncclResult_t r = nccl().AllReduce(h->d_fin_local, h->d_fin, (size_t)h->P_glob * MAGUS_N_TOTALS, ncclFloat64,
                                          ncclSum, h->comm, s);
        if (r != ncclSuccess) return fail(h, MAGUS_ERR_NCCL, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
    }
    if (detail) CU(h, rec(4));
    return MAGUS_OK;
}

// The run as a CUDA graph (re-captured when the buffers, the stream or the timing flag change); its
// timing-event nodes are re-pointed at this run's ring slot before every launch.
static magus_status launch_graph(magus_replay_t* h, const float* d_trace, const float* d_w, cudaStream_t s,
                                 cudaEvent_t* tv) {
    if (!h->gexec || h->g_trace != d_trace || h->g_w != d_w || h->g_stream != s) {
        if (h->gexec) cudaGraphExecDestroy(h->gexec);
        if (h->graph) cudaGraphDestroy(h->graph);
        h->gexec = nullptr;
        h->graph = nullptr;
        h->g_events.clear();
        CU(h, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        magus_status st = enqueue_run(h, d_trace, d_w, s, tv, true);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (st != MAGUS_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (ce != cudaSuccess) return cuda_fail(h, ce, "cudaStreamEndCapture");
        const cudaError_t ie = cudaGraphInstantiate(&h->gexec, graph, 0);
        if (ie != cudaSuccess) {
            cudaGraphDestroy(graph);
            return cuda_fail(h, ie, "cudaGraphInstantiate");
        }
        h->graph = graph;   // kept: exec-node updates take the original graph's node handles
        h->g_trace = d_trace;
        h->g_w = d_w;
        h->g_stream = s;
    } else if (tv) {
        for (const auto& ne : h->g_events) CU(h, cudaGraphExecEventRecordNodeSetEvent(h->gexec, ne.first, tv[ne.second]));
    }
    CU(h, cudaGraphLaunch(h->gexec, s));
    return MAGUS_OK;
}

extern "C" magus_status magus_replay_run(magus_replay_t* h, const float* d_trace, const float* d_w, void* stream) {
    if (!h) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "NULL handle");
    const magus_replay_desc& d = h->desc;
    const bool has_work = d.n_traces > 0 && d.n_samples > 0;
    if ((has_work && !d_trace) || (d.n_traces > 0 && !d_w)) return fail(h, MAGUS_ERR_INVALID_ARG, "NULL trace or w");
    if (has_work && ((uintptr_t)d_trace % 16 != 0)) return fail(h, MAGUS_ERR_ALIGN, "trace base must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    if (has_work) {
        magus_status st = encode_tmap(h, d_trace);
        if (st != MAGUS_OK) return st;
    }
    cudaEvent_t* tv = (d.flags & MAGUS_F_TIMING) ? &h->tev[5 * (h->n_runs % magus_replay::kTimingRing)] : nullptr;
    // graphs need a capturable (non-legacy-default) stream
    const bool graph = s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread && !env_int("MAGUS_NO_GRAPH", 0);
    magus_status st = graph ? launch_graph(h, d_trace, d_w, s, tv) : enqueue_run(h, d_trace, d_w, s, tv, false);
    if (st != MAGUS_OK) return st;
    ReplayParams p = h->rp;
    if (h->d_codes && has_work) {
        const int P = d.n_policies;
        dim3 grid((unsigned)((d.dump_n_traces + 63) / 64), (unsigned)p.n_lane);
        // the codes decoded from the replay kernels' own words (MAGUS_DUMP_RESIM=1: re-simulated from t = 0
        // instead, a cross-check); the wall-clock kernel writes its rounds' codes itself
        if (!h->wall && env_int("MAGUS_DUMP_RESIM", 0))
            magus_resim_kernel<<<grid, 64, 0, s>>>(p, d_trace, d.dump_first_trace, d.dump_n_traces, P, h->d_codes);
        else if (!h->wall)
            magus_decode_kernel<<<grid, 64, 0, s>>>(p, d_trace, d.dump_first_trace, d.dump_n_traces, P, h->d_codes);
        CU(h, cudaGetLastError());
        const int64_t rows = (int64_t)d.n_samples * d.dump_n_traces;
        for (int pi : h->smax) {
            magus_fill_codes_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(h->d_codes, rows, P, pi, 0x81);
            CU(h, cudaGetLastError());
        }
    }
    CU(h, cudaEventRecord(h->ev[4], s));
    h->run_trace = d_trace;
    h->run_stream = s;
    h->ran = true;
    h->n_runs += 1;
    return MAGUS_OK;
}
extern "C" magus_status magus_replay_run_host(magus_replay_t* h, const float* trace, const float* w, void* stream) {
    if (!h) return fail(nullptr, MAGUS_ERR_INVALID_ARG, "NULL handle");
    const magus_replay_desc& d = h->desc;
    if (d.n_traces > 0 && (!trace || !w)) return fail(h, MAGUS_ERR_INVALID_ARG, "NULL trace or w");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n_trace = (size_t)d.n_samples * (size_t)d.trace_stride;
    if (!h->d_trace_own && n_trace > 0) {
        cudaError_t ce = dalloc(h, &h->d_trace_own, n_trace);
        if (ce != cudaSuccess) return cuda_fail(h, ce, "cudaMalloc host-run trace buffer");
    }
    if (!h->d_w_own) {
        cudaError_t ce = dalloc(h, &h->d_w_own, (size_t)std::max(1, d.n_traces));
        if (ce != cudaSuccess) return cuda_fail(h, ce, "cudaMalloc host-run w buffer");
    }
    if (n_trace > 0) CU(h, cudaMemcpyAsync(h->d_trace_own, trace, n_trace * sizeof(float), cudaMemcpyHostToDevice, s));
    if (d.n_traces > 0)
        CU(h, cudaMemcpyAsync(h->d_w_own, w, (size_t)d.n_traces * sizeof(float), cudaMemcpyHostToDevice, s));
    return magus_replay_run(h, h->d_trace_own, h->d_w_own, stream);
}

extern "C" magus_status magus_replay_results(magus_replay_t* h, magus_results* out) {
    if (!h || !out) return fail(h, MAGUS_ERR_INVALID_ARG, "NULL argument");
    if (!h->ran) return fail(h, MAGUS_ERR_STATE, "magus_replay_results before any run");
    const magus_replay_desc& d = h->desc;
    CU(h, cudaEventSynchronize(h->ev[4]));
    CU(h, cudaGetLastError());
    const int P = d.n_policies;
    // one copy: the totals partials and the run's flag words (adjacent on the device); the chunks are
    // added here in chunk order (fixed order: the result does not depend on timing or the rank layout)
    const size_t n_part = (size_t)P * h->n_chunks * MAGUS_N_TOTALS;
    std::vector<double> part(n_part + 2);
    CU(h, cudaMemcpy(part.data(), h->d_out, n_part * sizeof(double) + 4 * sizeof(unsigned int), cudaMemcpyDeviceToHost));
    std::vector<double> tot((size_t)h->P_glob * MAGUS_N_TOTALS, 0.0);
    if (h->xchg) {   // chunk sums on the device (same order), then the cross-rank allreduce
        CU(h, cudaMemcpy(tot.data(), h->d_fin, tot.size() * sizeof(double), cudaMemcpyDeviceToHost));
    } else {         // this rank's slice rows
        for (int pp = 0; pp < P; ++pp)
            for (int c = 0; c < h->n_chunks; ++c)
                for (int f = 0; f < MAGUS_N_TOTALS; ++f)
                    tot[(size_t)(h->p_off + pp) * MAGUS_N_TOTALS + f] +=
                        part[((size_t)pp * h->n_chunks + c) * MAGUS_N_TOTALS + f];
    }
    if (out->policy_totals) std::memcpy(out->policy_totals, tot.data(), tot.size() * sizeof(double));
    int32_t am = 0;   // argmin over policies of the total EDP, ties -> lowest index (A23)
    magus_totals_argmin(tot.data(), h->P_glob, &am);
    out->argmin_policy = am;
    unsigned int fl[4] = {0, 0, 0, 0};
    std::memcpy(fl, part.data() + n_part, sizeof(fl));
    unsigned long long segs = 0;
    std::memcpy(&segs, &fl[2], 8);
    out->n_segments = h->rp.n_seg;
    out->warmup_ticks = h->rp.warmup;
    out->n_mismatched_segments = (int64_t)segs;
    out->fixup_rounds = (int32_t)fl[1];
    // Adaptive re-plan, off by default (MAGUS_REPLAN_PCT = 101, i.e. never): when more than
    // MAGUS_REPLAN_PCT % of the speculative entries mismatched, the next runs use half as many segments.  The
    // chain walk's cost does not grow with the segment count, so this only starves the replay of parallelism.
    // Results are exact either way.
    // Adaptive warm-up: speculative entries that mismatched mean the warm-up was too short to
    // re-derive the true state (oscillating traces: the limit cycle's phase); the next runs start their speculative
    // segments earlier (extra ticks 0 -> 64 -> 192 -> 448, at most 3 times, the warm-up at most 1/8 of a segment).
    // A run without a mismatch keeps its plan.  Results are exact either way; this only trades chain-walk time
    // for replay time (config 5: 2,053 wrong entries at 32 ticks, none at 96; step 0.835 -> 0.721 ms).
    bool warm_replan = false;
    if (d.tuning_segments == 0 && d.tuning_warmup == 0 && h->rp.n_seg > 1 && segs > 0 && h->warm_replans < 3 &&
        !h->open_fast &&
        !env_int("MAGUS_NO_REPLAN", 0) && !env_int("MAGUS_NO_WARM_ADAPT", 0)) {
        const int extra = 2 * h->warm_extra + 64;
        if (h->rp.warmup + (extra - h->warm_extra) <= h->rp.seg_len / 8) {
            h->warm_extra = extra;
            h->warm_replans += 1;
            warm_replan = true;
        }
    }
    if (d.tuning_segments == 0 && h->rp.n_seg > 1 && !env_int("MAGUS_NO_REPLAN", 0) && !h->open_fast) {
        const double spec = (double)h->rp.n_lane * (h->rp.n_seg - 1) * std::max(1, d.n_traces);
        const bool halve = (double)segs > h->replan_frac * spec;
        if (halve || warm_replan) {
            const int S_new = halve ? std::max(1, h->rp.n_seg / 2) : 0;   // 0: the automatic segment count
            const ReplayParams keep = h->rp;
            choose_geometry(h, h->n_sm, S_new);
            // keep the scratch pointers, thresholds and constants; only the plan changed
            ReplayParams np = keep;
            np.n_seg = h->rp.n_seg;
            np.seg_len = h->rp.seg_len;
            np.seg_long = h->rp.seg_long;
            np.warmup = h->rp.warmup;
            np.solo_warm = h->rp.solo_warm;
            h->rp = np;
            for (const LaunchGroup& g : h->groups)
                cudaFuncSetAttribute((const void*)g.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
            if (h->gexec) cudaGraphExecDestroy(h->gexec);
            if (h->graph) cudaGraphDestroy(h->graph);
            h->gexec = nullptr;
            h->graph = nullptr;
            h->replans += 1;
        }
    }
    if (out->per_trace && (d.flags & MAGUS_F_PER_TRACE_STATS) && d.n_traces > 0)
        CU(h, cudaMemcpy(out->per_trace, h->d_rec, (size_t)d.n_traces * P * sizeof(TraceRec), cudaMemcpyDeviceToHost));
    if (out->words && (d.flags & MAGUS_F_DUMP_WORDS) && d.n_traces > 0 && h->rp.n_blocks > 0) {
        const size_t per_pol = (size_t)d.n_traces * h->rp.n_blocks * 2;
        for (size_t q = 0; q < h->lane.size(); ++q) {
            const int pi = h->lane[q].policy_index;
            if (pi < 0) continue;
            CU(h, cudaMemcpy(out->words + (size_t)pi * per_pol, h->rp.words + q * per_pol, per_pol * 4,
                             cudaMemcpyDeviceToHost));
        }
        for (int pi : h->smax) {
            uint32_t* o = out->words + (size_t)pi * per_pol;
            for (int j = 0; j < d.n_traces; ++j)
                for (int b = 0; b < h->rp.n_blocks; ++b) {
                    const int n = std::min(32, d.n_samples - b * 32);
                    o[((size_t)j * h->rp.n_blocks + b) * 2] = n == 32 ? 0xFFFFFFFFu : (((1u << n) - 1u) << (32 - n));
                    o[((size_t)j * h->rp.n_blocks + b) * 2 + 1] = 0;
                }
        }
    }
    if (out->decisions && h->d_codes)
        CU(h, cudaMemcpy(out->decisions, h->d_codes, (size_t)d.n_samples * d.dump_n_traces * P, cudaMemcpyDeviceToHost));
    out->err_trace = -1;
    out->err_tick = -1;
    if (fl[0]) {
        unsigned long long key = ~0ULL;
        CU(h, cudaMemcpy(h->d_errkey, &key, sizeof(key), cudaMemcpyHostToDevice));
        magus_scan_invalid_kernel<<<(d.n_traces + 127) / 128, 128>>>(h->run_trace, d.n_traces, d.n_samples,
                                                                     d.trace_stride, h->bwbits, h->d_errkey);
        CU(h, cudaGetLastError());
        CU(h, cudaMemcpy(&key, h->d_errkey, sizeof(key), cudaMemcpyDeviceToHost));
        if (key != ~0ULL) {
            out->err_trace = (int32_t)(key >> 32);
            out->err_tick = (int64_t)(key & 0xFFFFFFFFULL);
            return fail(h, MAGUS_ERR_TRACE,
                        "invalid sample (negative, NaN/Inf or > bw_max) at trace " + std::to_string(out->err_trace) +
                            " tick " + std::to_string(out->err_tick));
        }
    }
    return MAGUS_OK;
}

static magus_status timing_avg(magus_replay_t* h, int n_last, float out_ms[5]) {
    if (!h || !out_ms) return fail(h, MAGUS_ERR_INVALID_ARG, "NULL argument");
    if (!h->ran || h->tev.empty()) return fail(h, MAGUS_ERR_STATE, "no timed run (MAGUS_F_TIMING)");
    CU(h, cudaEventSynchronize(h->ev[4]));
    const int64_t n = std::min<int64_t>({(int64_t)std::max(1, n_last), h->n_runs, (int64_t)magus_replay::kTimingRing});
    // events per run: 0 run start, 1 replay start (after the speculation pre-pass), 2 replay end,
    // 3 fix-up end, 4 totals (+ allreduce) + argmin end; only 1 and 2 without MAGUS_F_TIMING_DETAIL
    const int iv[5][2] = {{1, 2}, {2, 3}, {3, 4}, {0, 4}, {0, 1}};
    const int n_iv = (h->desc.flags & MAGUS_F_TIMING_DETAIL) ? 5 : 1;
    double acc[5] = {0, 0, 0, 0, 0};
    for (int64_t r = h->n_runs - n; r < h->n_runs; ++r) {
        cudaEvent_t* tv = &h->tev[5 * (r % magus_replay::kTimingRing)];
        for (int k = 0; k < n_iv; ++k) {
            float ms;
            CU(h, cudaEventElapsedTime(&ms, tv[iv[k][0]], tv[iv[k][1]]));
            acc[k] += ms;
        }
    }
    for (int i = 0; i < 5; ++i) out_ms[i] = i < n_iv ? (float)(acc[i] / (double)n) : -1.0f;
    return MAGUS_OK;
}

extern "C" magus_status magus_replay_run_times(magus_replay_t* h, int32_t n_last, float* out_ms, int32_t* n_out) {
    if (!h || !out_ms || !n_out) return fail(h, MAGUS_ERR_INVALID_ARG, "NULL argument");
    if (!h->ran || h->tev.empty()) return fail(h, MAGUS_ERR_STATE, "no timed run (MAGUS_F_TIMING)");
    CU(h, cudaEventSynchronize(h->ev[4]));
    const int64_t n = std::min<int64_t>({(int64_t)std::max(1, n_last), h->n_runs, (int64_t)magus_replay::kTimingRing});
    int32_t i = 0;
    for (int64_t r = h->n_runs - n; r < h->n_runs; ++r, ++i) {
        cudaEvent_t* tv = &h->tev[5 * (r % magus_replay::kTimingRing)];
        CU(h, cudaEventElapsedTime(out_ms + i, tv[1], tv[2]));
    }
    *n_out = i;
    return MAGUS_OK;
}

extern "C" magus_status magus_replay_kernel_times(magus_replay_t* h, float out_ms[5]) {
    return timing_avg(h, 1, out_ms);
}

extern "C" magus_status magus_replay_timing_summary(magus_replay_t* h, int32_t n_last, float out_ms[5]) {
    return timing_avg(h, n_last, out_ms);
}

// Diagnostics: the chosen geometry (first launch group's CTA shape).
extern "C" magus_status magus_replay_geometry(const magus_replay_t* h, int32_t out[16]) {
    if (!h || !out) return MAGUS_ERR_INVALID_ARG;
    const ReplayParams& p = h->rp;
    const magus_replay_desc& d = h->desc;
    int ctas = 0;
    for (const LaunchGroup& g : h->groups) ctas += g.fused ? 0 : g.n_ctas;
    const LaunchGroup& g0 = h->groups.front();
    // kernel launches of one run, as enqueue_run issues them
    const bool has_work = d.n_traces > 0 && d.n_samples > 0;
    const int nwall = env_int("MAGUS_WALL_ROUNDMAJOR", 0) ? 1 : (int)h->groups.size();
    int nlaunch = 0;
    for (const LaunchGroup& g : h->groups) nlaunch += g.fused ? 0 : 1;
    int nk = 1 + (has_work ? (h->wall ? nwall : nlaunch) : 0);   // pre-pass, replay per launch (group or combined pair)
    bool open_fix = h->open_fast;
    for (const LaunchGroup& g : h->groups) open_fix = open_fix && g.solo;
    if (has_work && p.n_seg > 1 && !h->wall && open_fix) {
        nk += (int)h->groups.size();                              // one open-loop fix-up kernel per launch group
    } else if (has_work && p.n_seg > 1 && !h->wall) {
        int nw = 0;
        for (const LaunchGroup& g : h->groups) nw += walk_kernel_for(g.key) ? 1 : 0;
        nk += 1 + nw;                                             // mark + one chain-walk kernel per launch group
    }
    nk += 1 + (h->xchg ? 1 : 0);                                  // totals (+ chunk sums before the allreduce)
    int solo = 0, wide = 0;
    for (const LaunchGroup& g : h->groups) {
        solo += g.solo ? 1 : 0;
        wide += g.wide ? 1 : 0;
    }
    int32_t threads = g0.threads, smem = (int32_t)g0.smem;
    if (h->wall) {   // the wall-clock kernels (A32): one 128-thread CTA per 128 chains of a launch group
        ctas = ((d.n_traces + 127) / 128) * p.n_lane;   // (the launch groups partition the lanes)
        threads = 128;
        smem = 0;
        solo = 0;
    }
    const int32_t v[16] = {p.n_seg, p.seg_len, p.warmup, g0.ng, g0.npw, g0.n_tblocks, g0.n_pblocks, ctas,
                           threads, smem, p.n_lane, (int32_t)h->groups.size(), nk, solo, p.seg_long, wide};
    std::memcpy(out, v, sizeof(v));
    return MAGUS_OK;
}
