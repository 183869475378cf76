// Dependent-latency probe (one warp, clock64): cycles per dependent DADD, DSETP->FSEL, FSEL pair, ISETP->PLOP3,
// IMAD on sm_100a.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat scripts/lat_probe.cu && /tmp/lat
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {   // DADD chain
        asm volatile("add.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
        asm volatile("add.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
        asm volatile("add.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
        asm volatile("add.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
    }
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) {   // DSETP -> FSEL(f64) chain: y = (y > b) ? a : y+0  (compare feeds the select)
        asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %2, %0, p; }" : "+d"(y) : "d"(b), "d"(a));
        asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %2, %0, p; }" : "+d"(y) : "d"(b), "d"(a));
        asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %2, %0, p; }" : "+d"(y) : "d"(b), "d"(a));
        asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %2, %0, p; }" : "+d"(y) : "d"(b), "d"(a));
    }
    long long t2 = clock64();
    unsigned u = (unsigned)n;
    for (int i = 0; i < n; ++i) {   // ISETP -> SEL chain
        asm volatile("{ .reg .pred p; setp.gt.u32 p, %0, 7; selp.u32 %0, %0, 9, p; }" : "+r"(u));
        asm volatile("{ .reg .pred p; setp.gt.u32 p, %0, 7; selp.u32 %0, %0, 9, p; }" : "+r"(u));
        asm volatile("{ .reg .pred p; setp.gt.u32 p, %0, 7; selp.u32 %0, %0, 9, p; }" : "+r"(u));
        asm volatile("{ .reg .pred p; setp.gt.u32 p, %0, 7; selp.u32 %0, %0, 9, p; }" : "+r"(u));
    }
    long long t3 = clock64();
    float f = (float)a;
    for (int i = 0; i < n; ++i) {   // F2F f64->f32->f64 round trip chain (XU)
        double d;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f));
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(d));
    }
    long long t4 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) {   // DSETP -> predicated IMAD -> ISETP -> selp f64 (the P stage's flag -> count -> level)
        asm volatile("{ .reg .pred p, q; .reg .b32 c; setp.gt.f64 p, %0, %1; selp.u32 c, 1, 0, p; setp.ne.u32 q, c, 0; selp.f64 %0, %2, %0, q; }" : "+d"(z) : "d"(b), "d"(a));
    }
    long long t5 = clock64();
    out[threadIdx.x] = x + y + u + f + z;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = (t3 - t2); cyc[3] = (t4 - t3); cyc[4] = (t5 - t4);
    }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 32 * 8); cudaMallocManaged(&c, 8 * 8);
    const int n = 4096;
    k<<<1, 32>>>(o, c, 1.0, 0.5, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 0.5, n); cudaDeviceSynchronize();
    printf("DADD dependent: %.2f cycles\n", c[0] / (4.0 * n));
    printf("DSETP -> FSEL(f64) pair: %.2f cycles\n", c[1] / (4.0 * n));
    printf("ISETP -> SEL pair: %.2f cycles\n", c[2] / (4.0 * n));
    printf("F2F f32->f64 -> F2F f64->f32 pair: %.2f cycles\n", c[3] / (1.0 * n));
    printf("DSETP -> SEL -> ISETP -> FSEL(f64): %.2f cycles\n", c[4] / (1.0 * n));
    return 0;
}
