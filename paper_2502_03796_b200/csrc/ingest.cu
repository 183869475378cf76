// ingest.cu -- NEXT-3 front end: recorded cumulative byte counters -> the replay's trace layout.
//
// "obtaining memory throughput data": MAGUS reads one memory-traffic counter per round; its
// throughput is the difference quotient of the cumulative byte count over the round.
// A counter that decreased (wrap / reset) gives no measurement: the interval is discarded, the baseline
// re-armed and there is no governor round for it: each trace's rounds are its valid intervals in
// time order, compacted to the front of its column, with its round count in n_valid (A31).  Layouts
// are the replay's: time-major, trace-minor.
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

// grid.x = column blocks x chunks (flattened: no 65535 limit on the chunk count); a thread = one column chunk
__device__ __forceinline__ bool chunk_of(int64_t stride, int64_t n_int, int64_t& j, int64_t& i0, int64_t& i1,
                                        int64_t& chunk) {
    const int64_t cb = (stride + 127) / 128;
    chunk = (int64_t)blockIdx.x / cb;
    j = ((int64_t)blockIdx.x % cb) * 128 + threadIdx.x;
    i0 = chunk * kRows;
    i1 = min(i0 + kRows, n_int);
    return j < stride && i0 < n_int;
}

// pass 1: valid intervals (counter did not decrease) per (chunk, column); timestamps checked by column 0
__global__ void __launch_bounds__(128) count_kernel(const uint64_t* __restrict__ counts, const double* __restrict__ times,
                                                    int32_t n_traces, int64_t n_rows, int64_t stride,
                                                    int64_t* __restrict__ cnt, unsigned long long* report) {
    int64_t j, i0, i1, chunk;
    if (!chunk_of(stride, n_rows - 1, j, i0, i1, chunk)) return;
    if (j == 0 && times) {
        unsigned long long bad = 0;
        for (int64_t i = i0; i < i1; ++i) bad += (times[i + 1] - times[i] > 0.0) ? 0ull : 1ull;
        if (bad) atomicAdd(report + 1, bad);
    }
    if (j >= n_traces) return;
    int64_t v = 0;
    uint64_t c0 = counts[i0 * stride + j];
    for (int64_t i = i0; i < i1; ++i) {
        const uint64_t c1 = counts[(i + 1) * stride + j];
        v += c1 >= c0 ? 1 : 0;
        c0 = c1;
    }
    cnt[chunk * stride + j] = v;
    if (v != i1 - i0) atomicAdd(report, (unsigned long long)(i1 - i0 - v));
}

// pass 2 (one thread per column): chunk offsets (exclusive prefix in time order), the column's round count,
// and the padding rows after its last round (0.0; padding columns entirely)
__global__ void __launch_bounds__(128) scan_kernel(int32_t n_traces, int64_t n_rows, int64_t stride, int64_t chunks,
                                                   int64_t* __restrict__ cnt, int64_t* __restrict__ n_valid,
                                                   float* __restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= stride) return;
    const int64_t n_int = n_rows - 1;
    int64_t k = 0;
    if (j < n_traces) {
        for (int64_t c = 0; c < chunks; ++c) {
            const int64_t v = cnt[c * stride + j];
            cnt[c * stride + j] = k;
            k += v;
        }
        if (n_valid) n_valid[j] = k;
    }
    for (int64_t i = k; i < n_int; ++i) out[i * stride + j] = 0.0f;
}

// pass 3: each column chunk writes its valid intervals' throughputs at its offset (a discarded interval yields
// no round, A31)
__global__ void __launch_bounds__(128) write_kernel(const uint64_t* __restrict__ counts, const double* __restrict__ times,
                                                    int32_t n_traces, int64_t n_rows, int64_t stride, double period,
                                                    const int64_t* __restrict__ off, float* __restrict__ out) {
    int64_t j, i0, i1, chunk;
    if (!chunk_of(stride, n_rows - 1, j, i0, i1, chunk) || j >= n_traces) return;
    int64_t k = off[chunk * stride + j];
    uint64_t c0 = counts[i0 * stride + j];
    for (int64_t i = i0; i < i1; ++i) {
        const uint64_t c1 = counts[(i + 1) * stride + j];
        if (c1 >= c0) out[(k++) * stride + j] = quotient(c0, c1, times ? times[i + 1] - times[i] : period);
        c0 = c1;
    }
}

}  // namespace ingest
}  // namespace magus

extern "C" const char* magus_set_global_error(const char* msg);   // magus_replay.cu

extern "C" magus_status magus_counters_to_trace(const uint64_t* d_counts, const double* d_times, int32_t n_traces,
                                                int64_t n_rows, int64_t stride, double period_s, float* d_trace,
                                                int64_t* d_n_valid, unsigned long long* d_report, void* stream) {
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
    const cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err = cudaMemsetAsync(d_report, 0, 2 * sizeof(unsigned long long), st);
    if (err == cudaSuccess && d_n_valid && n_traces > 0)
        err = cudaMemsetAsync(d_n_valid, 0, (size_t)n_traces * sizeof(int64_t), st);
    const int64_t n_int = n_rows - 1;
    if (err == cudaSuccess && n_int > 0 && stride > 0) {
        using namespace magus::ingest;
        const int64_t chunks = (n_int + kRows - 1) / kRows, cb = (stride + 127) / 128;
        if (chunks * cb > 0x7FFFFFFFLL) {
            magus_set_global_error("magus_counters_to_trace: too many rows x columns for one launch");
            return MAGUS_ERR_INVALID_ARG;
        }
        int64_t* cnt = nullptr;   // [chunks][stride] round counts, then offsets (stream-ordered scratch)
        err = cudaMallocAsync((void**)&cnt, (size_t)(chunks * stride) * sizeof(int64_t), st);
        if (err == cudaSuccess) {
            count_kernel<<<(unsigned)(chunks * cb), 128, 0, st>>>(d_counts, d_times, n_traces, n_rows, stride, cnt, d_report);
            scan_kernel<<<(unsigned)cb, 128, 0, st>>>(n_traces, n_rows, stride, chunks, cnt, d_n_valid, d_trace);
            write_kernel<<<(unsigned)(chunks * cb), 128, 0, st>>>(d_counts, d_times, n_traces, n_rows, stride, period_s,
                                                                 cnt, d_trace);
            err = cudaGetLastError();
            const cudaError_t fe = cudaFreeAsync(cnt, st);
            if (err == cudaSuccess) err = fe;
        }
    }
    if (err != cudaSuccess) {
        magus_set_global_error(cudaGetErrorString(err));
        return err == cudaErrorMemoryAllocation ? MAGUS_ERR_OOM : MAGUS_ERR_CUDA;
    }
    return MAGUS_OK;
}
