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

// forward: block = 64 rows of model g, 256 threads (4 per row, each owning
// outputs n = t%4, t%4+4, ...); A and W staged through smem in 64-wide k
// chunks with coalesced loads.
constexpr int FR = 64, FK = 64;
__global__ void __launch_bounds__(256) head_fwd_kernel(HeadFwd p) {
    __shared__ float sA[FR][FK + 1];
    __shared__ float sW[FK][MAXN + 1];
    const int g = blockIdx.y;
    const int r0 = blockIdx.x * FR;
    const int N = p.N;
    const int row = threadIdx.x >> 2, sub = threadIdx.x & 3;
    const float* A = p.A + g * p.a_gs;
    const float* W = p.W + g * p.w_gs;
    float acc[MAXN / 4];
#pragma unroll
    for (int i = 0; i < MAXN / 4; ++i) acc[i] = 0.f;
    for (int k0 = 0; k0 < p.K; k0 += FK) {
        const int kc = min(FK, p.K - k0);
        __syncthreads();
        for (int e = threadIdx.x; e < FR * FK; e += 256) {
            const int rr = e / FK, kk = e % FK;
            sA[rr][kk] = (r0 + rr < p.rows && kk < kc) ? A[(long long)(r0 + rr) * p.lda + k0 + kk] : 0.f;
        }
        for (int e = threadIdx.x; e < FK * N; e += 256) {
            const int kk = e / N, n = e % N;
            sW[kk][n] = kk < kc ? W[(long long)(k0 + kk) * N + n] : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < FK; ++kk) {
            const float a = sA[row][kk];
#pragma unroll
            for (int i = 0; i < MAXN / 4; ++i) {
                const int n = sub + 4 * i;
                if (n < N) acc[i] = fmaf(a, sW[kk][n], acc[i]);
            }
        }
    }
    const int r = r0 + row;
    if (r >= p.rows) return;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < MAXN / 4; ++i) {
        const int n = sub + 4 * i;
        if (n >= N) break;
        float v = acc[i] + p.bias[g * p.bias_gs + n];
        bad |= !isfinite(v);
        if (p.relu) v = v > 0.f ? v : 0.f;
        p.C[g * p.c_gs + (long long)r * p.ldc + n] = v;
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

// dX through a narrow layer: out[r, q] = (sum_j dz[r, j] W[q, j] + add[r, q]) *
// (mask[r, q] > 0), j < N <= 32.  Block = 32 rows of model g; W (K x N) and
// the dz rows in smem; threads stride q so mask/add/out are coalesced.
__global__ void __launch_bounds__(256) head_dx_kernel(HeadDx p) {
    extern __shared__ float sm[];
    const int N = p.N, ld = N | 1;
    float* sW = sm;                      // [K][ld]
    float* sdz = sm + (size_t)p.K * ld;  // [32][ld]
    const int g = blockIdx.y;
    const int r0 = blockIdx.x * 32;
    const float* W = p.W + g * p.w_gs;
    for (int e = threadIdx.x; e < p.K * N; e += blockDim.x) sW[(e / N) * ld + e % N] = W[e];
    for (int e = threadIdx.x; e < 32 * N; e += blockDim.x) {
        const int rr = e / N, j = e % N;
        sdz[rr * ld + j] = (r0 + rr < p.rows) ? p.dZ[g * p.dz_gs + (long long)(r0 + rr) * p.lddz + j] : 0.f;
    }
    __syncthreads();
    for (int rr = 0; rr < 32 && r0 + rr < p.rows; ++rr) {
        const long long rowb = g * p.c_gs + (long long)(r0 + rr) * p.ldc;
        for (int q = threadIdx.x; q < p.K; q += blockDim.x) {
            float acc = 0.f;
#pragma unroll 8
            for (int j = 0; j < N; ++j) acc = fmaf(sdz[rr * ld + j], sW[q * ld + j], acc);
            const long long idx = rowb + q;
            if (p.add) acc = p.add[idx] + acc;
            p.C[idx] = (p.mask[idx] > 0.f) ? acc : 0.f;
        }
    }
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
            const int lim = min(64, rend - r0);
#pragma unroll 4
            for (int rr = rg; rr < lim; rr += 4) {
                const float av = __ldg(A + (long long)(r0 + rr) * p.lda + pp);
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

bool head_fwd_ok(int K, int N) { return N <= MAXN && K >= 1; }
bool head_dx_ok(int K, int N) { return N <= MAXN && (size_t)(K + 32) * (N | 1) * 4 <= 96 * 1024; }
bool head_dw_ok(int N) { return N <= MAXN; }

void launch_head_fwd(const HeadFwd& p, cudaStream_t s) {
    if (p.rows <= 0) return;
    dim3 grid((p.rows + FR - 1) / FR, p.G);
    head_fwd_kernel<<<grid, 256, 0, s>>>(p);
    count_launch();
}

void launch_head_dx(const HeadDx& p, cudaStream_t s) {
    if (p.rows <= 0) return;
    const size_t smem = (size_t)(p.K + 32) * (p.N | 1) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        MTK_CUDA(cudaFuncSetAttribute(head_dx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      96 * 1024));
        attr = true;
    }
    dim3 grid((p.rows + 31) / 32, p.G);
    head_dx_kernel<<<grid, 256, smem, s>>>(p);
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
