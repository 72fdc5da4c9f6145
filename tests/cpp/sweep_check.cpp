// Runs the shadow-training sweep + membership attack through the C++ drop-in
// only (include/minitransfer/gpu.hpp over libmtk): BASELINE.md C1 (the
// defaults) for one paradigm, printed as one JSON line.
//   ./sweep_check model|mapping|parameter [epochs]
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "minitransfer/gpu.hpp"

int main(int argc, char** argv) {
    const char* par = argc > 1 ? argv[1] : "model";
    mt::gpu::SweepConfig cfg;  // C1: 784-256-10, 1 + 4 models, 2048 members, B 128, E 10
    if (!std::strcmp(par, "mapping")) cfg.paradigm = MTK_PARADIGM_MAPPING;
    else if (!std::strcmp(par, "parameter")) cfg.paradigm = MTK_PARADIGM_PARAMETER;
    else if (std::strcmp(par, "model")) {
        std::printf("unknown paradigm %s\n", par);
        return 2;
    }
    if (argc > 2) cfg.epochs = std::atoi(argv[2]);
    try {
        mt::gpu::Context ctx(0);
        const mt::gpu::SweepResult r = mt::gpu::run_shadow_sweep(ctx, cfg);
        std::printf("{\"paradigm\": \"%s\", \"auc\": %.17g, \"accuracy\": %.17g, \"models\": %d, "
                    "\"n_queries\": %lld, \"seconds\": %.3f, \"reference_headers\": %d}\n",
                    par, r.auc, r.accuracy, r.models, (long long)r.n_queries, r.seconds,
                    MT_GPU_HAVE_REFERENCE);
    } catch (const mt::Error& e) {  // the reference's own exception classes when present
        std::printf("mt::Error: %s\n", e.what());
        return 1;
    }
    return 0;
}
