// Drives include/minitransfer/gpu.hpp the way a reference user would.
//   ./wrapper_check        host-only checks (RNG vs reference mt::Rng, errors)
//   ./wrapper_check gpu    + one grouped bank step on cuda:0
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "minitransfer/gpu.hpp"
#if MT_GPU_HAVE_REFERENCE
#include "minitransfer/rng.hpp"
#endif

#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                              \
        }                                                          \
    } while (0)

int main(int argc, char** argv) {
    // host RNG: bit-exact with the reference mt::Rng where its headers are present
    mt::gpu::Rng r(42);
#if MT_GPU_HAVE_REFERENCE
    mt::Rng ref(42);
    for (int i = 0; i < 1000; ++i) {
        CHECK(r.next_u64() == ref.next_u64());
        CHECK(r.normal() == ref.normal());
        CHECK(r.uniform(-0.5, 0.5) == ref.uniform(-0.5, 0.5));
        CHECK(r.below(97) == ref.below(97));
    }
    auto p1 = r.permutation(500);
    auto p2 = ref.permutation(500);
    CHECK(p1 == p2);
    std::printf("rng bit-exact vs reference mt::Rng\n");
#endif
    // error mapping onto the reference classes
    bool threw = false;
    try {
        mt::gpu::Context bad(-1);
    } catch (const mt::Error& e) {
        threw = true;
    }
    CHECK(threw);
    if (argc < 2 || std::strcmp(argv[1], "gpu") != 0) {
        std::printf("host checks ok\n");
        return 0;
    }
    // one grouped step on the device
    mt::gpu::Context ctx(0);
    const int G = 3, B = 16;
    std::vector<int> dims = {64, 32, 10};
    mt::gpu::Bank bank(ctx, G, dims);
    mt::gpu::Rng init(7);
    for (int g = 0; g < G; ++g) bank.init_params(g, init);
    std::vector<float> X(G * B * dims[0]);
    std::vector<int32_t> y(G * B);
    mt::gpu::Rng data(9);
    for (auto& v : X) v = (float)data.normal();
    for (auto& v : y) v = (int32_t)data.below(10);
    float* dX = nullptr;
    int32_t* dy = nullptr;
    cudaMalloc(&dX, X.size() * 4);
    cudaMalloc(&dy, y.size() * 4);
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
    mtk_step s{};
    s.X = dX;
    s.y = dy;
    s.B = B;
    s.lr = 0.1;
    std::vector<double> l0 = bank.train_step(s);
    for (int i = 0; i < 20; ++i) bank.train_step(s);
    std::vector<double> l1 = bank.train_step(s);
    for (int g = 0; g < G; ++g) {
        CHECK(std::isfinite(l0[g]) && l1[g] < l0[g]);
        std::printf("model %d loss %.6f -> %.6f\n", g, l0[g], l1[g]);
    }
    // a bad label surfaces as the reference's ValueError
    y[5] = 11;
    cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
    threw = false;
    try {
        bank.train_step(s);
    } catch (const mt::ValueError&) {
        threw = true;
    }
    CHECK(threw);
    cudaFree(dX);
    cudaFree(dy);
    std::printf("gpu checks ok\n");
    return 0;
}
