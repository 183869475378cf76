/*
 * oracle/gen_oracle.cpp -- the ORACLE SIDE's implementation of the seeded,
 * counter-based synthetic trace generator.  TEST INFRASTRUCTURE ONLY (see the
 * header of magus_oracle.cpp for who may load it).
 *
 * The recipe is DESIGN.md section 6 ("input recipe"); the product implements
 * the same recipe independently as a CUDA kernel
 * (paper_2502_03796_b200/csrc/gen_traces.cu) and a GPU test checks the two
 * byte for byte.  Nothing here is the method's arithmetic: it only draws the
 * demand samples D[t][j] and the compute weights w[j] that both sides replay.
 *
 * Shapes: compute-bound (C0), memory-bound (C1),
 * phase-alternating (C2), training spikes (C3,
 * SPEC.md:87-95), oscillating (C4),
 * plus the adversarial set of config 5 (square waves with periods near the
 * sampling interval, random telegraph).
 *
 * All arithmetic is integer hashing or explicit fp32 round-to-nearest
 * multiply/add with no FMA (-ffp-contract=off), so the bytes are
 * reproducible on any IEEE machine.
 */
#include <cstdint>
#include <cstring>
#include <cmath>
#include "oracle.h"

extern "C" {


static const uint64_t PHI  = 0x9E3779B97F4A7C15ULL;
static const uint64_t PHI2 = 0xD1B54A32D192ED03ULL;
static const uint64_t PHI3 = 0x8CB92BA72F3D8DD7ULL;

static uint64_t g_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* 24-bit uniform in [0,1): exact in fp32 */
static float g_u24(uint64_t x) { return (float)(uint32_t)(x >> 40) * (1.0f / 16777216.0f); }
/* fp32 uniform in [lo, hi): lo + (hi - lo) * u, two rounded fp32 ops */
static float g_unif(float lo, float hi, uint64_t x) {
    float span = hi - lo;
    float prod = span * g_u24(x);
    return lo + prod;
}
/* integer uniform in [a, b] */
static int64_t g_irange(int64_t a, int64_t b, uint64_t x) {
    return a + (int64_t)((x >> 32) % (uint64_t)(b - a + 1));
}

/* per-trace key and its i-th draw */
static uint64_t g_trace_key(uint64_t seed, int64_t j) { return g_mix64(seed ^ g_mix64((uint64_t)j + PHI)); }
static uint64_t g_draw(uint64_t h, uint64_t i) { return g_mix64(h + (i + 1) * PHI); }

/* largest fp32 <= bw_max */
static float g_clamp_bound(double bw) {
    float b = (float)bw;
    if ((double)b > bw) b = std::nextafter(b, 0.0f);
    return b;
}

/* square-wave periods p = a/b of config 5 (cfg 5) */
static const int64_t SQ_A[8] = {1, 21, 3, 2, 41, 5, 3, 4};
static const int64_t SQ_B[8] = {1, 20, 2, 1, 20, 2, 1, 1};
static const float   TELEGRAPH_Q[3] = {0.3f, 0.5f, 0.7f};

/* noise-free level of trace j (key h) at tick t for the pure classes; `base` = draw offset */
static float g_class_level(int cls, uint64_t h, uint64_t base, int64_t t) {
    switch (cls) {
    case 0:  /* C0 compute-bound: U[0.5, 4) GB/s (below B_lo) */
        return g_unif(0.5f, 4.0f, g_draw(h, base + 1));
    case 1:  /* C1 memory-bound: U[10, 19) GB/s (above B_lo) */
        return g_unif(10.0f, 19.0f, g_draw(h, base + 1));
    case 2: { /* C2 phase-alternating: low then high blocks of phase_len ticks */
        float lo = g_unif(0.5f, 4.0f, g_draw(h, base + 1));
        float hi = g_unif(10.0f, 19.0f, g_draw(h, base + 2));
        int64_t phase_len = g_irange(20, 2000, g_draw(h, base + 3));
        return ((t / phase_len) & 1) ? hi : lo;
    }
    case 3: { /* C3 training spikes: spike_len ticks of `spike` at the start of every cycle */
        float b = g_unif(1.0f, 3.0f, g_draw(h, base + 1));
        float s = g_unif(12.0f, 19.0f, g_draw(h, base + 2));
        int64_t spike_len = g_irange(1, 20, g_draw(h, base + 3));
        int64_t cycle = g_irange(50, 500, g_draw(h, base + 4));
        return (t % cycle) < spike_len ? s : b;
    }
    default: { /* C4 oscillating: toggles every 1 or 2 ticks */
        float lo = g_unif(0.5f, 4.0f, g_draw(h, base + 1));
        float hi = g_unif(10.0f, 19.0f, g_draw(h, base + 2));
        int64_t toggle = g_irange(1, 2, g_draw(h, base + 3));
        return ((t / toggle) & 1) ? hi : lo;
    }
    }
}

/* Writes trace j_local's samples to col[t * col_stride] for t in [0, n) and returns w_j. */
float oracle_gen_trace(const OGenDesc* g, int64_t j_local, float* col, int64_t col_stride) {
    const int64_t j = g->global_trace_offset + j_local;
    const uint64_t h = g_trace_key(g->seed, j);
    const float bw = g_clamp_bound(g->bw_max_gbps);
    const float amp = g->noise_amp;
    const int64_t n = g->n_samples;

    /* class and adversarial parameters */
    int cls = 0;
    int adv = 0, fam = 0;
    if (g->class_mix == 0) {
        cls = (int)(j % 3);
        if (cls == 2 && (g_draw(h, 0) & 3) == 0) cls = 3;   /* 1/4 of C2 become C3 */
    } else if (g->class_mix == 1) {
        cls = (int)(j % 5);
    } else if (g->class_mix == 2) {
        adv = (int)(j % 11);
        fam = (int)(g_draw(h, 0) & 1);
    }
    float adv_lo = 0.0f, adv_hi = 0.0f;
    if (g->class_mix == 2) {
        if (adv >= 8 || fam == 0) {   /* straddling B_lo */
            adv_lo = g_unif(0.5f, 4.0f, g_draw(h, 1));
            adv_hi = g_unif(10.0f, 19.0f, g_draw(h, 2));
        } else {                      /* both levels below B_lo */
            adv_lo = g_unif(0.5f, 2.0f, g_draw(h, 1));
            adv_hi = g_unif(4.0f, 7.0f, g_draw(h, 2));
        }
    }

    int telegraph_state = 0;
    for (int64_t t = 0; t < n; ++t) {
        float level;
        if (g->class_mix == 2) {
            if (adv < 8) {
                int64_t phase = ((2 * t * SQ_B[adv]) / SQ_A[adv]) & 1;  /* floor(2 t b / a) mod 2 */
                level = phase ? adv_hi : adv_lo;
            } else {
                if (t > 0) {
                    float u = g_u24(g_mix64(h ^ ((uint64_t)t * PHI3)));
                    if (u < TELEGRAPH_Q[adv - 8]) telegraph_state ^= 1;
                }
                level = telegraph_state ? adv_hi : adv_lo;
            }
        } else if (g->class_mix == 3) {
            int64_t seg = t / 2000;                       /* 2,000-tick segments C0..C4 */
            level = g_class_level((int)(seg % 5), h, (uint64_t)(16 * seg), t - seg * 2000);
        } else {
            level = g_class_level(cls, h, 0, t);
        }
        /* multiplicative noise: level * (1 + a*(2u - 1)), each op fp32 round-to-nearest */
        float u = g_u24(g_mix64(h ^ ((uint64_t)t * PHI2)));
        float two_u = 2.0f * u;
        float centred = two_u - 1.0f;
        float scaled = amp * centred;
        float factor = 1.0f + scaled;
        float v = level * factor;
        if (v < 0.0f) v = 0.0f;
        if (v > bw) v = bw;
        col[t * col_stride] = v;
    }
    /* compute weight: U[0.5, 0.95) (GPU-dominant) */
    return g_unif(0.5f, 0.95f, g_draw(h, 5));
}

/* Full time-major layout: trace[t * stride + j] for j < n_traces, zero padding up to stride. */
void oracle_gen_traces(const OGenDesc* g, float* trace, float* w) {
    for (int64_t t = 0; t < g->n_samples; ++t)
        for (int64_t j = g->n_traces; j < g->trace_stride; ++j) trace[t * g->trace_stride + j] = 0.0f;
    for (int64_t j = 0; j < g->n_traces; ++j)
        w[j] = oracle_gen_trace(g, j, trace + j, g->trace_stride);
}

} /* extern "C" */
