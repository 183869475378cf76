// SASS probe (no GPU): one instantiation of the solo replay kernel, for quick instruction-count checks of the
// generated stage blocks.  nvcc -cubin -DPROBE_V=<BAL> -DPROBE_K=<K> scripts/sass_probe.cu; scripts/solo_sass.py
#include "../paper_2502_03796_b200/csrc/post_kernels.cuh"
#include "../paper_2502_03796_b200/csrc/replay_kernel.cuh"
#include "../paper_2502_03796_b200/csrc/replay_solo.cuh"
#ifndef PROBE_K
#define PROBE_K 1
#endif
template __global__ void magus::magus_replay_solo_kernel<magus::MagusTicker<PROBE_K, false>, 8, 3, PROBE_V>(
    const __grid_constant__ CUtensorMap, const magus::ReplayParams);
#ifdef PROBE_U
template __global__ void magus::magus_replay_usolo_kernel<magus::MagusTicker<PROBE_K, false>, 8, 3, PROBE_U>(
    const __grid_constant__ CUtensorMap, const magus::ReplayParams);
#endif
#ifdef PROBE_T
template __global__ void magus::magus_replay_tsolo_kernel<PROBE_T, 8, 3>(const __grid_constant__ CUtensorMap,
                                                                         const magus::ReplayParams);
#endif
#ifdef PROBE_W
#include "../paper_2502_03796_b200/csrc/replay_wide.cuh"
template __global__ void magus::magus_replay_wide_kernel<PROBE_K, 1, PROBE_W>(const __grid_constant__ CUtensorMap,
                                                                              const magus::ReplayParams);
#endif
#ifdef PROBE_F
template __global__ void magus::magus_replay_fused_kernel<magus::MagusTicker<PROBE_K, false>, 8, 3, (PROBE_F == 2)>(
    const __grid_constant__ CUtensorMap, const magus::ReplayParams);
#endif
