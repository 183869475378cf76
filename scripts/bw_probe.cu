// bw_probe.cu -- HBM read bandwidth of the replay kernel's access pattern with trivial compute (no MAGUS
// logic): one-warp CTAs stream [TC ticks x BX traces] TMA boxes of a time-major fp32 [N][stride] array
// through an NSTAGE ring, the grid cut into (trace group, time segment) units like the solo replay kernel.
// Also a plain coalesced LDG.128 stream for reference.  Measurement aid only (not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe scripts/bw_probe.cu
//   ./bw_probe [n_traces=4096] [n_samples=100000] [segments=73]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\n\tLAB_WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra LAB_WAIT;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void issue(uint32_t tile, const CUtensorMap* m, uint32_t bar, int x, int y, uint32_t bytes) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
                 "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%2], [%3, {%4, %5}], [%0];\n\t}" ::"r"(bar), "r"(bytes), "r"(tile),
                 "l"((uint64_t)m), "r"(x), "r"(y) : "memory");
}

template <int BX, int TC, int NSTAGE>
__global__ void __launch_bounds__(32) tma_stream(const __grid_constant__ CUtensorMap tm, int n_groups, int seg_len,
                                                 int n_samples, int spin, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr uint32_t kTile = BX * TC * 4;
    const uint32_t t0s = (uint32_t)__cvta_generic_to_shared(smem), b0 = t0s + NSTAGE * kTile;
    const int g = blockIdx.x % n_groups, seg = blockIdx.x / n_groups;
    const int start = seg * seg_len, end = min(start + seg_len, n_samples);
    const int nst = (end - start + TC - 1) / TC;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * i));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    for (int i = 0; i < NSTAGE && i < nst; ++i) issue(t0s + i * kTile, &tm, b0 + 8 * i, g * BX, start + i * TC, kTile);
    float acc = 0.f;
    int slot = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
        wait_bar(b0 + 8 * slot, ph);
        const float* t = reinterpret_cast<const float*>(smem + slot * kTile);
#pragma unroll
        for (int r = 0; r < TC; ++r)
#pragma unroll
            for (int c = 0; c < BX / 32; ++c) acc += t[r * BX + c * 32 + threadIdx.x];
        for (int s = 0; s < spin; ++s) acc = acc * 0.999f + 1e-7f;   // emulated compute per stage
        __syncwarp();
        if (i + NSTAGE < nst) issue(t0s + slot * kTile, &tm, b0 + 8 * slot, g * BX, start + (i + NSTAGE) * TC, kTile);
        if (++slot == NSTAGE) { slot = 0; ph ^= 1u; }
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void ldg_stream(const float4* __restrict__ a, size_t n4, float* out) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(a + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int BX, int TC, int NSTAGE>
void run(PFN_enc enc, float* d, int nt, int ns, int S, int spin, float* out, int target_ctas) {
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)nt, (cuuint64_t)ns}, gstr[1] = {(cuuint64_t)nt * 4};
    cuuint32_t box[2] = {BX, TC}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed BX=%d TC=%d\n", BX, TC);
        return;
    }
    const int ng = nt / BX;
    int segs = S > 0 ? S : (target_ctas + ng - 1) / ng;
    const int L = ((ns + segs - 1) / segs + TC - 1) / TC * TC;
    segs = (ns + L - 1) / L;
    size_t smem = (size_t)NSTAGE * BX * TC * 4 + 64;
    cudaFuncSetAttribute(tma_stream<BX, TC, NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_stream<BX, TC, NSTAGE>, 32, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {
        cudaEventRecord(e0);
        tma_stream<BX, TC, NSTAGE><<<ng * segs, 32, smem>>>(tm, ng, L, ns, spin, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 2 && ms < best) best = ms;
    }
    const double bytes = (double)nt * ns * 4;
    printf("tma BX=%3d TC=%2d NSTAGE=%d spin=%3d ctas=%6d occ/SM=%2d : %.4f ms  %.1f GB/s  (%s)\n", BX, TC, NSTAGE,
           spin, ng * segs, occ, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int nt = argc > 1 ? atoi(argv[1]) : 4096, ns = argc > 2 ? atoi(argv[2]) : 100000;
    const int S = argc > 3 ? atoi(argv[3]) : 0;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    PFN_enc enc = (PFN_enc)p;
    float *d, *out;
    const size_t n = (size_t)nt * ns;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&out, 64);
    cudaMemset(d, 0, n * 4);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int rep = 0; rep < 12; ++rep) {
            cudaEventRecord(e0);
            ldg_stream<<<nsm * 8, 256>>>((const float4*)d, n / 4, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep >= 2 && ms < best) best = ms;
        }
        printf("ldg.128 stream            : %.4f ms  %.1f GB/s\n", best, n * 4.0 / best / 1e6);
    }
    const int T = nsm * 16;
    for (int spin : {0, 64}) {
        run<128, 8, 3>(enc, d, nt, ns, S, spin, out, T);
        run<128, 8, 2>(enc, d, nt, ns, S, spin, out, T);
        run<128, 16, 3>(enc, d, nt, ns, S, spin, out, T);
        run<128, 32, 2>(enc, d, nt, ns, S, spin, out, T);
        run<256, 8, 3>(enc, d, nt, ns, S, spin, out, T);
        run<256, 4, 3>(enc, d, nt, ns, S, spin, out, T);
        run<64, 16, 3>(enc, d, nt, ns, S, spin, out, T);
    }
    run<128, 8, 3>(enc, d, nt, ns, S, 0, out, nsm * 8);
    run<128, 8, 3>(enc, d, nt, ns, S, 0, out, nsm * 32);
    run<128, 8, 3>(enc, d, nt, ns, 1, 0, out, T);
    return 0;
}
