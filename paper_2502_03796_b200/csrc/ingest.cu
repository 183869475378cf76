// ingest.cu -- NEXT-3 front end: recorded cumulative byte counters -> the replay's trace layout.
//
// "obtaining memory throughput data": MAGUS reads one memory-traffic counter per round; its
// throughput is the difference quotient of the cumulative byte count over the round.
// A counter that decreased (wrap / reset) gives no measurement: the interval is discarded and the baseline
// re-armed; in the one-sample-per-round replay the round repeats the last valid interval's throughput of
// its trace, 0 before any (A31).  Layouts are the replay's: time-major, trace-minor.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/magus_replay.h"

namespace magus {
namespace ingest {

constexpr int kRows = 256;   // rows (intervals) per thread: a column chunk walked in time order

// one interval's throughput in GB/s: ((double)(c1 - c0) / dt) / 1e9, rounded once to fp32
__device__ __forceinline__ float quotient(uint64_t c0, uint64_t c1, double dt) {
    return (float)(((double)(c1 - c0) / dt) / 1e9);
}

__global__ void __launch_bounds__(128) counters_kernel(const uint64_t* __restrict__ counts, const double* __restrict__ times,
                                                       int32_t n_traces, int64_t n_rows, int64_t stride, double period,
                                                       float* __restrict__ out, unsigned long long* report) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i0 = (int64_t)blockIdx.y * kRows;
    const int64_t n_int = n_rows - 1;   // intervals
    if (j >= stride || i0 >= n_int) return;
    const int64_t i1 = min(i0 + kRows, n_int);
    if (j == 0 && times) {   // timestamps must increase (one column checks them)
        unsigned long long bad = 0;
        for (int64_t i = i0; i < i1; ++i) bad += (times[i + 1] - times[i] > 0.0) ? 0ull : 1ull;
        if (bad) atomicAdd(report + 1, bad);
    }
    if (j >= n_traces) {   // padding columns
        for (int64_t i = i0; i < i1; ++i) out[i * stride + j] = 0.0f;
        return;
    }
    // the last valid interval before the chunk (usually the one just before it)
    float last = 0.0f;
    for (int64_t i = i0 - 1; i >= 0; --i) {
        const uint64_t a = counts[i * stride + j], b = counts[(i + 1) * stride + j];
        if (b >= a) {
            last = quotient(a, b, times ? times[i + 1] - times[i] : period);
            break;
        }
    }
    unsigned long long resets = 0;
    uint64_t c0 = counts[i0 * stride + j];
    for (int64_t i = i0; i < i1; ++i) {
        const uint64_t c1 = counts[(i + 1) * stride + j];
        float v;
        if (c1 < c0) {   // wrap / reset: discarded, the round repeats the last valid throughput
            v = last;
            ++resets;
        } else {
            v = quotient(c0, c1, times ? times[i + 1] - times[i] : period);
            last = v;
        }
        out[i * stride + j] = v;
        c0 = c1;
    }
    if (resets) atomicAdd(report, resets);
}

}  // namespace ingest
}  // namespace magus

extern "C" const char* magus_set_global_error(const char* msg);   // magus_replay.cu

extern "C" magus_status magus_counters_to_trace(const uint64_t* d_counts, const double* d_times, int32_t n_traces,
                                                int64_t n_rows, int64_t stride, double period_s, float* d_trace,
                                                unsigned long long* d_report, void* stream) {
    if (!d_counts || !d_trace || !d_report) {
        magus_set_global_error("magus_counters_to_trace: NULL argument");
        return MAGUS_ERR_INVALID_ARG;
    }
    if (n_traces < 0 || n_rows < 0 || stride < n_traces || (!d_times && !(period_s > 0.0))) {
        magus_set_global_error("magus_counters_to_trace: need 0 <= n_traces <= stride, n_rows >= 0, and period_s > 0 "
                               "without timestamps");
        return MAGUS_ERR_INVALID_ARG;
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        magus_set_global_error("magus_counters_to_trace: no CUDA device");
        return MAGUS_ERR_CUDA;
    }
    cudaError_t err = cudaMemsetAsync(d_report, 0, 2 * sizeof(unsigned long long), (cudaStream_t)stream);
    if (err == cudaSuccess && n_rows > 1 && stride > 0) {
        const int64_t chunks = (n_rows - 1 + magus::ingest::kRows - 1) / magus::ingest::kRows;
        dim3 grid((unsigned)((stride + 127) / 128), (unsigned)chunks);
        magus::ingest::counters_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(d_counts, d_times, n_traces, n_rows,
                                                                              stride, period_s, d_trace, d_report);
        err = cudaGetLastError();
    }
    if (err != cudaSuccess) {
        magus_set_global_error(cudaGetErrorString(err));
        return MAGUS_ERR_CUDA;
    }
    return MAGUS_OK;
}
