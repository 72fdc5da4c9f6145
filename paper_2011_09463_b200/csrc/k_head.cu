// k_head.cu -- skinny GEMMs for narrow layers (the 10-class head, the 2-class
// attack head): out widths <= 32 do not fill a 128-wide tile, so these run
// as warp-per-row (forward) and thread-per-input-feature (dW + SGD) kernels.
//   forward  logits = H W + b          (tape.hpp:36-48 mm_acc + add_bias)
//   dW + SGD W -= lr * H^T dZ          (tape.hpp:65-78 mm_tn_acc; optim.hpp:46-48)
// Reductions run in a fixed order (bit-deterministic).
#include <cmath>

#include "internal.h"
#include "sm100.cuh"

namespace mtk {
namespace {

constexpr int MAXN = 32;

// block: 8 warps x 8 rows each; W of model g (K x N, padded stride) in smem
__global__ void __launch_bounds__(256) head_fwd_kernel(HeadFwd p) {
    extern __shared__ float sW[];
    const int g = blockIdx.y;
    const int N = p.N, K = p.K, ld = N | 1;  // odd stride: conflict-free lane-strided reads
    const float* W = p.W + g * p.w_gs;
    for (int i = threadIdx.x; i < K * N; i += blockDim.x) sW[(i / N) * ld + (i % N)] = W[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* bias = p.bias + g * p.bias_gs;
    bool bad = false;
    for (int rr = 0; rr < 8; ++rr) {
        const int r = blockIdx.x * 64 + warp * 8 + rr;
        if (r >= p.rows) break;
        const float* a = p.A + g * p.a_gs + (long long)r * p.lda;
        float acc[MAXN];
#pragma unroll
        for (int n = 0; n < MAXN; ++n) acc[n] = 0.f;
        for (int k = lane; k < K; k += 32) {
            const float av = a[k];
            const float* wr = sW + k * ld;
#pragma unroll
            for (int n = 0; n < MAXN; ++n)
                if (n < N) acc[n] = fmaf(av, wr[n], acc[n]);
        }
        float mine = 0.f;
#pragma unroll
        for (int n = 0; n < MAXN; ++n) {
            if (n >= N) break;
            float v = acc[n];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == n) mine = v;
        }
        if (lane < N) {
            float v = mine + bias[lane];
            bad |= !isfinite(v);
            if (p.relu) v = v > 0.f ? v : 0.f;
            const long long idx = g * p.c_gs + (long long)r * p.ldc + lane;
            p.C[idx] = v;
            if (p.C_hi) {
                float h, l;
                sm100::split_tf32(v, h, l);
                p.C_hi[idx] = h;
                p.C_lo[idx] = l;
            }
        }
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

// dW partials: block (p-chunk of 64 input features, model g, row split rs),
// 256 threads = 4 row groups x 64 features; partial[rs][g][p][n]
constexpr int RS = 8;
__global__ void __launch_bounds__(256) head_dw_partial_kernel(HeadDw p) {
    __shared__ float sdz[64][MAXN + 1];
    __shared__ float red[4][64][MAXN + 1];
    const int g = blockIdx.y, rs = blockIdx.z;
    const int pl = threadIdx.x & 63, rg = threadIdx.x >> 6;
    const int pp = blockIdx.x * 64 + pl;
    const int N = p.N;
    const int rbeg = (int)((long long)p.rows * rs / RS), rend = (int)((long long)p.rows * (rs + 1) / RS);
    float acc[MAXN];
#pragma unroll
    for (int n = 0; n < MAXN; ++n) acc[n] = 0.f;
    const float* A = p.A + g * p.a_gs;
    const float* dz = p.dZ + g * p.dz_gs;
    for (int r0 = rbeg; r0 < rend; r0 += 64) {
        __syncthreads();
        for (int i = threadIdx.x; i < 64 * N; i += blockDim.x) {
            const int rr = i / N, n = i % N;
            sdz[rr][n] = (r0 + rr < rend) ? dz[(long long)(r0 + rr) * p.lddz + n] : 0.f;
        }
        __syncthreads();
        if (pp < p.K) {
            for (int rr = rg; rr < 64 && r0 + rr < rend; rr += 4) {
                const float av = A[(long long)(r0 + rr) * p.lda + pp];
#pragma unroll
                for (int n = 0; n < MAXN; ++n)
                    if (n < N) acc[n] = fmaf(av, sdz[rr][n], acc[n]);
            }
        }
    }
    for (int n = 0; n < N; ++n) red[rg][pl][n] = acc[n];
    __syncthreads();
    if (rg == 0 && pp < p.K)
        for (int n = 0; n < N; ++n)
            p.partial[(((long long)rs * p.G + g) * p.K + pp) * N + n] =
                ((red[0][pl][n] + red[1][pl][n]) + red[2][pl][n]) + red[3][pl][n];
}

// dW = sum of the RS partials in fixed order; SGD + optional gradient copy
__global__ void head_dw_finish_kernel(HeadDw p) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long per = (long long)p.K * p.N;
    if (t >= per * p.G) return;
    const int g = (int)(t / per);
    const long long e = t % per;
    float gsum = 0.f;
    for (int rs = 0; rs < RS; ++rs) gsum += p.partial[((long long)rs * p.G + g) * per + e];
    const long long idx = g * p.w_gs + e;
    if (p.grad_out) p.grad_out[idx] = gsum;
    const float w = p.W[idx] - p.lr * gsum;
    if (!isfinite(w) && p.flags) atomicOr(p.flags, kFlagNonFinite);
    p.W[idx] = w;
    if (p.W_hi) {
        float h, l;
        sm100::split_tf32(w, h, l);
        p.W_hi[idx] = h;
        p.W_lo[idx] = l;
    }
}

}  // namespace

bool head_fwd_ok(int K, int N) { return N <= MAXN && (size_t)K * (N | 1) * 4 <= 96 * 1024; }
bool head_dw_ok(int N) { return N <= MAXN; }

void launch_head_fwd(const HeadFwd& p, cudaStream_t s) {
    if (p.rows <= 0) return;
    const size_t smem = (size_t)p.K * (p.N | 1) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        MTK_CUDA(cudaFuncSetAttribute(head_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      96 * 1024));
        attr = true;
    }
    dim3 grid((p.rows + 63) / 64, p.G);
    head_fwd_kernel<<<grid, 256, smem, s>>>(p);
    count_launch();
}

size_t head_dw_scratch_bytes(int G, int K, int N) { return (size_t)RS * G * K * N * sizeof(float); }

void launch_head_dw(const HeadDw& p, cudaStream_t s) {
    if (p.K <= 0) return;
    if (!p.partial) fail(MTK_ERROR, "head_dw: missing partial scratch");
    dim3 grid((p.K + 63) / 64, p.G, RS);
    head_dw_partial_kernel<<<grid, 256, 0, s>>>(p);
    count_launch();
    const long long n = (long long)p.G * p.K * p.N;
    head_dw_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p);
    count_launch();
}

}  // namespace mtk
