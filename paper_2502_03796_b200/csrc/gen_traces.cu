// gen_traces.cu -- product-side implementation of the seeded synthetic trace generator
// (DESIGN.md section 6).  Independent of oracle/gen_oracle.cpp; a GPU test checks the two byte
// for byte.  It holds none of the method's arithmetic: it only writes the demand samples D[t][j]
// (time-major, trace-minor, the replay kernel's layout) and the compute weights w[j].
//
// Counter-based: every value depends only on (seed, global trace id, t), so any sharding or stride
// yields the same bytes.  Every fp32 operation is an explicit round-to-nearest intrinsic (no FMA
// contraction), so the device reproduces the IEEE host result exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include "../../include/magus_replay.h"

namespace magus {
namespace gen {

__device__ __constant__ int64_t kSqA[8] = {1, 21, 3, 2, 41, 5, 3, 4};
__device__ __constant__ int64_t kSqB[8] = {1, 20, 2, 1, 20, 2, 1, 1};

constexpr uint64_t PHI = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t PHI2 = 0xD1B54A32D192ED03ULL;
constexpr uint64_t PHI3 = 0x8CB92BA72F3D8DD7ULL;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float unit24(uint64_t x) {   // (x >> 40) * 2^-24, exact
    return __fmul_rn(__uint2float_rn((uint32_t)(x >> 40)), 5.9604644775390625e-08f);
}
__device__ __forceinline__ float uniform(float lo, float hi, uint64_t x) {
    return __fadd_rn(lo, __fmul_rn(__fsub_rn(hi, lo), unit24(x)));
}
__device__ __forceinline__ int64_t irange(int64_t a, int64_t b, uint64_t x) {
    return a + (int64_t)((x >> 32) % (uint64_t)(b - a + 1));
}
__device__ __forceinline__ uint64_t draw(uint64_t h, uint64_t i) { return mix(h + (i + 1) * PHI); }

struct Shape {
    int mix, cls, adv;
    float lo, hi;            // two-level classes
    int64_t a, b, c;         // class integers (phase_len / spike_len, cycle / toggle / square a,b)
};

__device__ __forceinline__ void class_params(int cls, uint64_t h, uint64_t base, Shape& s) {
    s.cls = cls;
    switch (cls) {
        case 0: s.lo = s.hi = uniform(0.5f, 4.0f, draw(h, base + 1)); break;
        case 1: s.lo = s.hi = uniform(10.0f, 19.0f, draw(h, base + 1)); break;
        case 2:
            s.lo = uniform(0.5f, 4.0f, draw(h, base + 1));
            s.hi = uniform(10.0f, 19.0f, draw(h, base + 2));
            s.a = irange(20, 2000, draw(h, base + 3));
            break;
        case 3:
            s.lo = uniform(1.0f, 3.0f, draw(h, base + 1));     // base
            s.hi = uniform(12.0f, 19.0f, draw(h, base + 2));   // spike
            s.a = irange(1, 20, draw(h, base + 3));            // spike_len
            s.b = irange(50, 500, draw(h, base + 4));          // cycle
            break;
        default:
            s.lo = uniform(0.5f, 4.0f, draw(h, base + 1));
            s.hi = uniform(10.0f, 19.0f, draw(h, base + 2));
            s.a = irange(1, 2, draw(h, base + 3));             // toggle_every
            break;
    }
}

__device__ __forceinline__ float class_level(const Shape& s, int64_t t) {
    switch (s.cls) {
        case 0:
        case 1: return s.lo;
        case 2: return ((t / s.a) & 1) ? s.hi : s.lo;
        case 3: return (t % s.b) < s.a ? s.hi : s.lo;
        default: return ((t / s.a) & 1) ? s.hi : s.lo;
    }
}

__device__ __forceinline__ float noisy(float level, uint64_t h, int64_t t, float amp, float bw) {
    const float u = unit24(mix(h ^ ((uint64_t)t * PHI2)));
    const float factor = __fadd_rn(1.0f, __fmul_rn(amp, __fsub_rn(__fmul_rn(2.0f, u), 1.0f)));
    float v = __fmul_rn(level, factor);
    if (v < 0.0f) v = 0.0f;
    if (v > bw) v = bw;
    return v;
}

// grid: x over columns j < stride (traces, then zero padding), y over tick chunks
__global__ void gen_kernel(magus_gen_desc g, float bw, int64_t chunk, float* __restrict__ trace,
                           float* __restrict__ w) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= g.trace_stride) return;
    const int64_t t_begin = (int64_t)blockIdx.y * chunk;
    const int64_t t_end = min(t_begin + chunk, g.n_samples);
    if (j >= g.n_traces) {
        for (int64_t t = t_begin; t < t_end; ++t) trace[t * g.trace_stride + j] = 0.0f;
        return;
    }
    const int64_t jg = g.global_trace_offset + j;
    const uint64_t h = mix(g.seed ^ mix((uint64_t)jg + PHI));
    if (blockIdx.y == 0) w[j] = uniform(0.5f, 0.95f, draw(h, 5));

    if (g.class_mix == 2) {   // adversarial (cfg 5): one sequential pass per trace (telegraph state)
        const int adv = (int)(jg % 11);
        const int fam = (int)(draw(h, 0) & 1);
        float lo, hi;
        if (adv >= 8 || fam == 0) {
            lo = uniform(0.5f, 4.0f, draw(h, 1));
            hi = uniform(10.0f, 19.0f, draw(h, 2));
        } else {
            lo = uniform(0.5f, 2.0f, draw(h, 1));
            hi = uniform(4.0f, 7.0f, draw(h, 2));
        }
        const float q = adv == 8 ? 0.3f : (adv == 9 ? 0.5f : 0.7f);
        int state = 0;
        for (int64_t t = 0; t < t_end; ++t) {
            float level;
            if (adv < 8) {
                level = (((2 * t * kSqB[adv]) / kSqA[adv]) & 1) ? hi : lo;
            } else {
                if (t > 0 && unit24(mix(h ^ ((uint64_t)t * PHI3))) < q) state ^= 1;
                level = state ? hi : lo;
            }
            if (t >= t_begin) trace[t * g.trace_stride + j] = noisy(level, h, t, g.noise_amp, bw);
        }
        return;
    }
    Shape s;
    if (g.class_mix == 3) {   // cfg 1: 2,000-tick segments cycling C0..C4
        int64_t cur = -1;
        for (int64_t t = t_begin; t < t_end; ++t) {
            const int64_t seg = t / 2000;
            if (seg != cur) {
                class_params((int)(seg % 5), h, (uint64_t)(16 * seg), s);
                cur = seg;
            }
            trace[t * g.trace_stride + j] = noisy(class_level(s, t - seg * 2000), h, t, g.noise_amp, bw);
        }
        return;
    }
    int cls;
    if (g.class_mix == 0) {
        cls = (int)(jg % 3);
        if (cls == 2 && (draw(h, 0) & 3) == 0) cls = 3;
    } else {
        cls = (int)(jg % 5);
    }
    class_params(cls, h, 0, s);
    for (int64_t t = t_begin; t < t_end; ++t)
        trace[t * g.trace_stride + j] = noisy(class_level(s, t), h, t, g.noise_amp, bw);
}

}  // namespace gen
}  // namespace magus

extern "C" const char* magus_set_global_error(const char* msg);   // magus_replay.cu

extern "C" magus_status magus_gen_traces(const magus_gen_desc* desc, float* d_trace, float* d_w, void* stream) {
    if (!desc || !d_trace || !d_w) {
        magus_set_global_error("magus_gen_traces: NULL argument");
        return MAGUS_ERR_INVALID_ARG;
    }
    const magus_gen_desc g = *desc;
    if (g.n_traces < 0 || g.n_samples < 0 || g.trace_stride < g.n_traces || g.class_mix < 0 || g.class_mix > 3 ||
        !(g.bw_max_gbps > 0.0) || !(g.noise_amp >= 0.0f)) {
        magus_set_global_error("magus_gen_traces: invalid descriptor (sizes, class_mix in 0..3, bw_max > 0)");
        return MAGUS_ERR_INVALID_ARG;
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        magus_set_global_error("magus_gen_traces: no CUDA device");
        return MAGUS_ERR_CUDA;
    }
    if (g.n_samples == 0 || g.trace_stride == 0) return MAGUS_OK;
    float bw = (float)g.bw_max_gbps;
    if ((double)bw > g.bw_max_gbps) bw = nextafterf(bw, 0.0f);
    // ticks per thread: 1024, more when grid.y would exceed 65535 chunks (the bytes do not depend on the chunking:
    // counter-based per (trace, tick); the adversarial class walks its trace in one sequential pass)
    const int64_t chunk = g.class_mix == 2 ? g.n_samples : std::max<int64_t>(1024, (g.n_samples + 65534) / 65535);
    const int64_t n_chunks = (g.n_samples + chunk - 1) / chunk;
    dim3 block(128), grid((unsigned)((g.trace_stride + 127) / 128), (unsigned)n_chunks);
    magus::gen::gen_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(g, bw, chunk, d_trace, d_w);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        magus_set_global_error(cudaGetErrorString(err));
        return MAGUS_ERR_CUDA;
    }
    return MAGUS_OK;
}
