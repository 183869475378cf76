/*
 * oracle/sample_oracle.cpp -- generate-and-replay a chosen subset of traces on
 * the host without materialising the whole (possibly 262 GB) time-major array.
 * TEST INFRASTRUCTURE ONLY (see magus_oracle.cpp's header).
 *
 * Used for parity at BASELINE.json's full sizes (configs 2 and 4: the GPU runs
 * every trace, the oracle re-derives a sampled subset one by one) and for
 * bench.py's cpu_baseline timing.  It is a loop over oracle_gen_trace +
 * oracle_replay; no arithmetic of its own.
 */
#include <atomic>
#include <thread>
#include <vector>
#include <algorithm>
#include "oracle.h"

extern "C" {

/* out: [n_ids][n_policies]; w_out: [n_ids] (optional); codes: [n_ids][n_policies][n_samples] per-tick code
 * bytes (optional, the same codes oracle_replay writes).  Returns the number of threads used. */
int oracle_gen_replay_codes(const OGenDesc* g, const int64_t* j_locals, int32_t n_ids,
                            int32_t n_policies, const OPolicy* pols, const OModel* m,
                            OResult* out, float* w_out, uint8_t* codes, int32_t n_threads) {
    if (n_threads <= 0) n_threads = (int32_t)std::max(1u, std::thread::hardware_concurrency());
    std::atomic<int32_t> next(0);
    auto worker = [&]() {
        std::vector<float> col((size_t)std::max<int64_t>(1, g->n_samples));
        for (;;) {
            int32_t i = next.fetch_add(1);
            if (i >= n_ids) break;
            float w = oracle_gen_trace(g, j_locals[i], col.data(), 1);
            if (w_out) w_out[i] = w;
            for (int32_t p = 0; p < n_policies; ++p)
                oracle_replay(col.data(), g->n_samples, 1, w, &pols[p], m,
                              &out[(int64_t)i * n_policies + p],
                              codes ? codes + ((int64_t)i * n_policies + p) * g->n_samples : nullptr, 1);
        }
    };
    int32_t used = std::min<int32_t>(n_threads, std::max<int32_t>(1, n_ids));
    std::vector<std::thread> pool;
    for (int32_t t = 0; t < used; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return used;
}

int oracle_gen_replay(const OGenDesc* g, const int64_t* j_locals, int32_t n_ids,
                      int32_t n_policies, const OPolicy* pols, const OModel* m,
                      OResult* out, float* w_out, int32_t n_threads) {
    return oracle_gen_replay_codes(g, j_locals, n_ids, n_policies, pols, m, out, w_out, nullptr, n_threads);
}

} /* extern "C" */
