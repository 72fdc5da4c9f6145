// k_mlp.cu -- grouped MLP kernels for the shadow-model bank (SIMT fp32 path).
//
// Replaces, for G independent models at once, the reference loops
//   detail::mm_acc    (tape.hpp:36-48)   forward  Z = H W      (+ add_bias, relu epilogue)
//   detail::mm_nt_acc (tape.hpp:50-63)   backward dH = dZ W^T  (+ relu mask epilogue)
//   detail::mm_tn_acc (tape.hpp:65-78)   backward dW = H^T dZ  (+ SGD epilogue, optim.hpp:46-48)
// and cross_entropy_weighted (tape.hpp:475-520).  Every output element is
// produced by exactly one thread with a fixed k order, so results are
// bit-deterministic run to run.
#include <cfloat>
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "ce_row.cuh"
#include "sm100.cuh"

namespace mtk {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, NT = 256;

__global__ void __launch_bounds__(NT) gemm_simt_kernel(Gemm p) {
    __shared__ float As[2][BK][BM + 4];
    __shared__ float Bs[2][BK][BN + 4];
    const int g = blockIdx.z;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const float* A = p.A + g * p.a_gs;
    const float* B = p.B + g * p.b_gs;
    const bool a_k_contig = (p.a_ks == 1);
    const bool b_n_contig = (p.b_ns == 1);

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    float ra[4], rb[4];
    auto load_regs = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = tid + i * NT;
            int mm, kk;
            if (a_k_contig) { mm = e >> 3; kk = e & 7; } else { mm = e & (BM - 1); kk = e >> 7; }
            const int gm = m0 + mm, gk = k0 + kk;
            ra[i] = (gm < p.M && gk < p.K) ? __ldg(A + gm * p.a_ms + (long long)gk * p.a_ks) : 0.f;
            int nn, kb;
            if (b_n_contig) { nn = e & (BN - 1); kb = e >> 7; } else { nn = e >> 3; kb = e & 7; }
            const int gn = n0 + nn, gkb = k0 + kb;
            rb[i] = (gn < p.N && gkb < p.K) ? __ldg(B + (long long)gkb * p.b_ks + gn * p.b_ns) : 0.f;
        }
    };
    auto store_smem = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = tid + i * NT;
            int mm, kk;
            if (a_k_contig) { mm = e >> 3; kk = e & 7; } else { mm = e & (BM - 1); kk = e >> 7; }
            As[buf][kk][mm] = ra[i];
            int nn, kb;
            if (b_n_contig) { nn = e & (BN - 1); kb = e >> 7; } else { nn = e >> 3; kb = e & 7; }
            Bs[buf][kb][nn] = rb[i];
        }
    };

    const int nk = (p.K + BK - 1) / BK;
    load_regs(0);
    store_smem(0);
    __syncthreads();
    for (int t = 0; t < nk; ++t) {
        const int buf = t & 1;
        if (t + 1 < nk) load_regs((t + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (t + 1 < nk) store_smem(buf ^ 1);
        __syncthreads();
    }

    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= p.M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= p.N) continue;
            const long long idx = g * p.c_gs + (long long)m * p.ldc + n;
            float v = acc[i][j];
            switch (p.epi) {
                case Epi::kBias:
                    v += p.bias[g * p.bias_gs + n];
                    bad |= !isfinite(v);
                    break;
                case Epi::kBiasRelu:
                    v += p.bias[g * p.bias_gs + n];
                    bad |= !isfinite(v);
                    v = v > 0.f ? v : 0.f;
                    break;
                case Epi::kMask:
                    if (p.add) v = p.add[idx] + v;
                    v = (p.mask[idx] > 0.f) ? v : 0.f;
                    break;
                case Epi::kSgd:
                    if (p.grad_out) p.grad_out[idx] = v;
                    v = sgd_update(p.C[idx], v, p.lr);
                    bad |= !isfinite(v);
                    break;
                case Epi::kStore:
                    break;
            }
            p.C[idx] = v;
        }
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

// One thread per row: softmax-CE forward + d(logits) (tape.hpp:475-520).
// Softmax-CE over one model's rows (tape.hpp:475-520): block = 256 rows of
// model blockIdx.y, one thread per row; dlogits = w_i/denom (P - onehot).
// Per warp (32 rows) it also reduces, in a fixed butterfly order, the row
// losses (fp64) into loss_part[g][blk32] and -- with colsum set -- the dlogits
// columns into colsum[g][blk32][C] (the head's bias gradient partials).
__global__ void __launch_bounds__(256) ce_kernel(CeArgs a) {
    const int g = blockIdx.y;
    const int i = blockIdx.x * 256 + threadIdx.x;  // row within the model
    const int lane = threadIdx.x & 31;
    const bool active = i < a.B;
    const long long r = (long long)g * a.B + i;
    double rl = 0.0;
    float x[32], dx[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        x[j] = (active && j < a.C) ? a.logits[r * a.C + j] : 0.f;
        dx[j] = 0.f;
    }
    if (active) {
        rl = ce_row(a, i, r, x, dx);
        float* d = a.dlogits + r * a.C;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < a.C) d[j] = dx[j];
        a.row_loss[r] = rl;
    }
    ce_warp_partials(a, g, i >> 5, lane, rl, dx);  // inactive rows contribute zeros
}

// loss[g] = sum of the 32-row partials in order
__global__ void ce_loss_kernel(const double* loss_part, int G, int nblk, double* loss, int* flags) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += loss_part[(long long)g * nblk + b];
    loss[g] = s;
    if (!isfinite(s)) atomicOr(flags, kFlagNonFinite);
}

// db = column sums of dZ, b -= lr * db.  Block = 32 columns x 32 row groups;
// each thread sums a strided row subset (loads batched 8 deep), then the 32
// partials are combined in a fixed order (deterministic, no atomics).
constexpr int BS_GROUPS = 32;
__global__ void __launch_bounds__(32 * BS_GROUPS) bias_sgd_kernel(int G, int rows, int N, const float* dZ,
                                                                  long long dz_gs, float* b, long long b_gs,
                                                                  float lr, AdamArgs adam, float* grad_out,
                                                                  int* flags) {
    __shared__ float part[BS_GROUPS][33];
    const int g = blockIdx.y;
    const int n = blockIdx.x * 32 + (threadIdx.x & 31);
    const int rg = threadIdx.x >> 5;
    float s = 0.f;
    if (n < N) {
        const float* col = dZ + g * dz_gs + n;
        for (int r = rg; r < rows; r += 8 * BS_GROUPS) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int rr = r + i * BS_GROUPS;
                v[i] = rr < rows ? __ldg(col + (long long)rr * N) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) s += v[i];
        }
    }
    part[rg][threadIdx.x & 31] = s;
    __syncthreads();
    if (rg == 0 && n < N) {
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < BS_GROUPS; ++q) t += part[q][threadIdx.x];
        if (grad_out) grad_out[g * b_gs + n] = t;
        const float v = param_update(b[g * b_gs + n], t, lr, adam, g * b_gs + n);
        if (!isfinite(v)) atomicOr(flags, kFlagNonFinite);
        b[g * b_gs + n] = v;
    }
}

}  // namespace

void launch_gemm(const Gemm& p, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0 || p.G <= 0) return;
    dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.G);
    gemm_simt_kernel<<<grid, NT, 0, s>>>(p);
    count_launch();
}

void launch_ce(const CeArgs& a, cudaStream_t s) {
    if (a.C > 32) fail(MTK_SHAPE_ERROR, "cross_entropy: more than 32 classes");
    ce_kernel<<<dim3((a.B + 255) / 256, a.G), 256, 0, s>>>(a);
    count_launch();
    launch_ce_loss(a, s);
}

void launch_ce_loss(const CeArgs& a, cudaStream_t s) {
    ce_loss_kernel<<<(a.G + 127) / 128, 128, 0, s>>>(a.loss_part, a.G, (a.B + 31) / 32, a.loss, a.flags);
    count_launch();
}

namespace {
__global__ void adam_apply_kernel(float* W, const float* grad, long long n, float lr, AdamArgs a,
                                  int* flags) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float w = param_update(W[i], grad[i], lr, a, i);
        bad |= !isfinite(w);
        W[i] = w;
    }
    if (bad && flags) atomicOr(flags, kFlagNonFinite);
}

}  // namespace

void launch_adam_apply(float* W, const float* grad, long long n, float lr, const AdamArgs& a,
                       int* flags, cudaStream_t s) {
    if (n <= 0) return;
    const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 16);
    adam_apply_kernel<<<(unsigned)blocks, 256, 0, s>>>(W, grad, n, lr, a, flags);
    count_launch();
}

namespace {
__global__ void bias_from_partials_kernel(int G, int nrb, int N, const float* partial, float* b,
                                          float lr, AdamArgs adam, float* grad_out, int* flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= G * N) return;
    const int g = t / N, n = t % N;
    float s = 0.f;
#pragma unroll 8
    for (int rb = 0; rb < nrb; ++rb) s += partial[((long long)g * nrb + rb) * N + n];
    if (grad_out) grad_out[t] = s;
    const float v = param_update(b[t], s, lr, adam, t);
    if (!isfinite(v)) atomicOr(flags, kFlagNonFinite);
    b[t] = v;
}
}  // namespace

void launch_bias_from_partials(int G, int nrb, int N, const float* partial, float* b, float lr,
                               const AdamArgs& adam, float* grad_out, int* flags, cudaStream_t s) {
    const int n = G * N;
    bias_from_partials_kernel<<<(n + 255) / 256, 256, 0, s>>>(G, nrb, N, partial, b, lr, adam, grad_out,
                                                               flags);
    count_launch();
}

void launch_bias_sgd(int G, int rows, int N, const float* dZ, long long dz_gs, float* b,
                     long long b_gs, float lr, const AdamArgs& adam, float* grad_out, int* flags,
                     cudaStream_t s) {
    dim3 grid((N + 31) / 32, G);
    bias_sgd_kernel<<<grid, 32 * BS_GROUPS, 0, s>>>(G, rows, N, dZ, dz_gs, b, b_gs, lr, adam, grad_out, flags);
    count_launch();
}

}  // namespace mtk
