// A small workload for compute-sanitizer (racecheck / synccheck): one bank
// step with the MMD term on the tensor-core paths (umma_kernel FWD/DX/DW,
// mmd_prep + mmd_w + V GEMM, the side stream), one fused-kernel MMD call
// (separate Xs / Xt buffers), and the attack stage in one call.
//   compute-sanitizer --tool racecheck --error-exitcode 1 ./race_check
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "minitransfer/gpu.hpp"

int main() {
    try {
        mt::gpu::Context ctx(0);
        const int G = 2, B = 128;
        const std::vector<int> dims = {64, 64, 32, 10};
        mt::gpu::Bank bank(ctx, G, dims);
        mt::gpu::Rng r(3);
        for (int g = 0; g < G; ++g) bank.init_params(g, r);
        std::vector<float> X((size_t)G * B * dims[0]);
        std::vector<int32_t> y((size_t)G * B);
        for (auto& v : X) v = (float)r.normal();
        for (auto& v : y) v = (int32_t)r.below(10);
        float *dX = nullptr, *gs = nullptr, *gt = nullptr, *logits = nullptr;
        int32_t* dy = nullptr;
        uint8_t* lab = nullptr;
        cudaMalloc(&dX, X.size() * 4);
        cudaMalloc(&dy, y.size() * 4);
        cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
        mtk_step s{};
        s.X = dX;
        s.y = dy;
        s.B = B;
        s.lr = 0.05;
        s.src_rows = B / 2;
        s.mmd_lambda = 1.0;
        std::vector<double> mmd;
        bank.train_step(s, &mmd);
        std::printf("bank step ok: mmd %.6f %.6f\n", mmd[0], mmd[1]);
        // fused pair kernel: Xs and Xt in separate buffers
        const int m = 96, n = 80, d = 64;
        cudaMalloc(&gs, (size_t)m * d * 4);
        cudaMalloc(&gt, (size_t)n * d * 4);
        const mt::gpu::MmdResult v = mt::gpu::mmd_gaussian(ctx, dX, m, dX + (size_t)B * dims[0], n, d, {}, 0.0, gs, gt);
        std::printf("mmd ok: %.6f (beta %.4f)\n", v.value, v.beta);
        // attack stage
        const int Q = 4096;
        std::vector<float> lg((size_t)Q * 10);
        std::vector<uint8_t> lb(Q);
        for (int i = 0; i < Q; ++i) {
            lb[i] = (uint8_t)(i & 1);
            for (int c = 0; c < 10; ++c) lg[(size_t)i * 10 + c] = (float)r.normal() + (lb[i] && c == 0 ? 1.f : 0.f);
        }
        cudaMalloc(&logits, lg.size() * 4);
        cudaMalloc(&lab, Q);
        cudaMemcpy(logits, lg.data(), lg.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(lab, lb.data(), Q, cudaMemcpyHostToDevice);
        mt::gpu::Bank att(ctx, 1, {3, 64, 2});
        att.init_params(0, r);
        double acc = 0.0;
        const double auc = mt::gpu::attack_auc(att, logits, Q, 10, lab, &acc);
        std::printf("attack ok: auc %.6f acc %.6f\n", auc, acc);
        ctx.synchronize();
        cudaFree(dX);
        cudaFree(dy);
        cudaFree(gs);
        cudaFree(gt);
        cudaFree(logits);
        cudaFree(lab);
    } catch (const mt::Error& e) {
        std::printf("mt::Error: %s\n", e.what());
        return 1;
    }
    std::printf("race_check done\n");
    return 0;
}
