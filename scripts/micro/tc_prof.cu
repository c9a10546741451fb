// Debug harness (not product code): runs one c-config L2 join through the
// tensor-core kernel compiled with -DKGC_PROF_TC and prints, per barrier wait,
// the mean cycles each waiting thread spent blocked.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "kgc.h"
extern "C" void kgc_debug_tc_prof(unsigned long long* out16, int reset);
extern "C" void kgc_debug_tc2_prof(unsigned long long* out16, int reset);
int main(int argc, char** argv) {
    if (argc < 6) { printf("usage: tc_prof E.bin Rel.bin N R d eps\n"); return 1; }
    long long N = atoll(argv[3]), R = atoll(argv[4]); int d = atoi(argv[5]); float eps = atof(argv[6]);
    std::vector<float> E(N * d), Rl(R * d);
    FILE* f = fopen(argv[1], "rb"); fread(E.data(), 4, E.size(), f); fclose(f);
    f = fopen(argv[2], "rb"); fread(Rl.data(), 4, Rl.size(), f); fclose(f);
    kgc_ctx* ctx; kgc_options o; kgc_default_options(&o); const int eng = getenv("ENGINE") ? atoi(getenv("ENGINE")) : 1; o.l2_engine = eng;
    auto prof = eng == 3 ? kgc_debug_tc2_prof : kgc_debug_tc_prof; (void)0; o.pivots = getenv("PIVOTS") ? atoi(getenv("PIVOTS")) : 1;
    if (kgc_create(&ctx, &o)) { printf("create: %s\n", kgc_last_error(nullptr)); return 1; }
    for (int rep = 0; rep < 2; ++rep) {
        prof(nullptr, 1);
        if (kgc_join(ctx, E.data(), Rl.data(), N, R, d, 2, eps)) { printf("join: %s\n", kgc_last_error(ctx)); return 1; }
        unsigned long long h[16];
        prof(h, 0);
        kgc_stats_t st; kgc_stats(ctx, &st);
        const char* nm[] = {"producer b_empty", "mma a_full", "mma acc_empty", "mma b_full", "epi a_full", "epi acc_full", "builder a_empty", "relay b_full"};
        // per-CTA waiting threads; the pair kernel's MMA warp and relay thread exist in one CTA of two
        const double pr = eng == 3 ? 0.5 : 1.0;
        const double waiters[] = {1, 32 * pr, 32 * pr, 32 * pr, 256, 256, 128, pr};
        double cyc = st.ms_tiles * 1e-3 * 1.965e9;
        printf("rep %d: tiles %.3f ms (~%.3g cycles/CTA), results %lld\n", rep, st.ms_tiles, cyc, (long long)st.results);
        for (int i = 0; i < (eng == 3 ? 8 : 7); ++i) printf("  %-18s %6.1f%% of kernel time per waiting thread\n", nm[i], 100.0 * h[i] / waiters[i] / 148 / cyc);
    }
    kgc_destroy(ctx);
    return 0;
}
