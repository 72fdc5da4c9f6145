// k_head.cu -- skinny GEMMs for narrow layers (the 10-class head, the 2-class
// attack head): output widths <= 32 do not fill a 128-wide MMA tile, so these
// are memory-bound SIMT kernels, templated on the padded width NP (a multiple
// of 4) so every per-output loop is fully unrolled with no dead lanes.
//   forward  logits = H W + b          (tape.hpp:36-48 mm_acc + add_bias)
//   dX       dH = (dZ W^T [+ add]) * (H > 0)   (tape.hpp:50-63 mm_nt_acc, :349)
//   dW + SGD W -= lr * H^T dZ          (tape.hpp:65-78 mm_tn_acc; optim.hpp:46-48)
// Register blocking keeps the shared-memory wavefront count per FMA low: the
// narrow operand (W row or dZ row) is read as broadcast float4.
// Reductions run in a fixed order (bit-deterministic).
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <utility>

#include "internal.h"
#include "ce_row.cuh"
#include "sm100.cuh"

namespace mtk {
namespace {

constexpr int MAXN = 32;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// ---- forward: block = 64 rows x 2 k-halves (128 threads); thread owns one row
// and all NP outputs; A and W staged through smem in 64-wide k chunks, the
// next A chunk's loads in flight (registers) while the current one computes.
// With do_ce the row-owning warps (one 32-row CE block each) go on to the
// softmax-CE of their finished logits (ce_row.cuh, as ce_kernel).
constexpr int FR = 64, FK = 64;
template <int NP>
__global__ void __launch_bounds__(128, 5) head_fwd_kernel(HeadFwd p, CeArgs ce, int do_ce) {
    __shared__ float sA[FR][FK + 1];
    __shared__ __align__(16) float sW[FK][NP];
    __shared__ float red[FR][NP + 1];
    const int g = blockIdx.y;
    const int r0 = blockIdx.x * FR;
    const int N = p.N, t = threadIdx.x;
    const int row = t & (FR - 1), half = t >> 6;
    const float* A = p.A + g * p.a_gs;
    const float* W = p.W + g * p.w_gs;
    const bool vec = (p.lda % 4 == 0) && (p.K % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    float acc[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) acc[n] = 0.f;
    constexpr int PA = FR * FK / 4 / 128;
    float4 v[PA];  // the next A chunk (vec path)
    auto load_a = [&](int k0) {
        const int kc = min(FK, p.K - k0);
#pragma unroll
        for (int i = 0; i < PA; ++i) {
            const int e = t + 128 * i, rr = e / (FK / 4), c4 = e % (FK / 4);
            v[i] = (r0 + rr < p.rows && 4 * c4 < kc) ? ldg4(A + (long long)(r0 + rr) * p.lda + k0 + 4 * c4)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    if (vec) load_a(0);
    for (int k0 = 0; k0 < p.K; k0 += FK) {
        const int kc = min(FK, p.K - k0);
        __syncthreads();
        if (vec) {
#pragma unroll
            for (int i = 0; i < PA; ++i) {
                const int e = t + 128 * i, rr = e / (FK / 4), c4 = e % (FK / 4);
                sA[rr][4 * c4] = v[i].x;
                sA[rr][4 * c4 + 1] = v[i].y;
                sA[rr][4 * c4 + 2] = v[i].z;
                sA[rr][4 * c4 + 3] = v[i].w;
            }
        } else {
            for (int e = t; e < FR * FK; e += 128) {
                const int rr = e / FK, kk = e % FK;
                sA[rr][kk] = (r0 + rr < p.rows && kk < kc) ? A[(long long)(r0 + rr) * p.lda + k0 + kk] : 0.f;
            }
        }
        {
            constexpr int PER = (FK * NP + 127) / 128;
            float wv[PER];  // loads in flight together, then the smem stores
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = t + 128 * i, kk = e / NP, n = e % NP;
                wv[i] = (e < FK * NP && kk < kc && n < N) ? __ldg(W + (long long)(k0 + kk) * N + n) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = t + 128 * i;
                if (e < FK * NP) sW[e / NP][e % NP] = wv[i];
            }
        }
        __syncthreads();
        if (vec && k0 + FK < p.K) load_a(k0 + FK);  // in flight during this chunk's FMAs
#pragma unroll 4
        for (int kk = half; kk < FK; kk += 2) {
            const float a = sA[row][kk];
#pragma unroll
            for (int n4 = 0; n4 < NP / 4; ++n4) {
                const float4 w = *reinterpret_cast<const float4*>(&sW[kk][4 * n4]);
                acc[4 * n4] = fmaf(a, w.x, acc[4 * n4]);
                acc[4 * n4 + 1] = fmaf(a, w.y, acc[4 * n4 + 1]);
                acc[4 * n4 + 2] = fmaf(a, w.z, acc[4 * n4 + 2]);
                acc[4 * n4 + 3] = fmaf(a, w.w, acc[4 * n4 + 3]);
            }
        }
    }
    if (half == 1)
#pragma unroll
        for (int n = 0; n < NP; ++n) red[row][n] = acc[n];
    __syncthreads();
    if (half == 1) return;  // warps 2, 3
    const int r = r0 + row;
    const bool active = r < p.rows;
    bool bad = false;
    float x[NP];
    float* out = p.C + g * p.c_gs + (long long)r * p.ldc;
#pragma unroll
    for (int n = 0; n < NP; ++n) {
        float val = 0.f;
        if (n < N) {
            val = (acc[n] + red[row][n]) + p.bias[g * p.bias_gs + n];
            bad |= active && !isfinite(val);
            if (p.relu) val = val > 0.f ? val : 0.f;
            if (active) out[n] = val;
        }
        x[n] = val;
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
    if (do_ce) {  // rows r0 .. r0 + 63: two whole 32-row CE blocks (FR = 64)
        float dx[NP];
        double rl = 0.0;
#pragma unroll
        for (int n = 0; n < NP; ++n) dx[n] = 0.f;
        const long long rr = (long long)g * ce.B + r;
        if (active) {
            rl = ce_row(ce, r, rr, x, dx);
            float* d = ce.dlogits + rr * ce.C;
#pragma unroll
            for (int j = 0; j < NP; ++j)
                if (j < ce.C) d[j] = dx[j];
            ce.row_loss[rr] = rl;
        }
        ce_warp_partials(ce, g, r >> 5, row & 31, rl, dx);
    }
}

// ---- dX: out[r, q] = (sum_j dz[r, j] W[q, j] + add[r, q]) * (mask[r, q] > 0).
// Block = 32 rows of model g; thread owns input feature q with W[q, :] in
// registers; dz rows are broadcast float4 reads from smem; mask/add/out are
// coalesced over q.
template <int NP>
__global__ void __launch_bounds__(256) head_dx_kernel(HeadDx p) {
    __shared__ __align__(16) float sdz[32][NP];
    const int N = p.N;
    const int g = blockIdx.y;
    const int r0 = blockIdx.x * 32;
    const int nrows = min(32, p.rows - r0);
    {
        constexpr int PER = (32 * NP + 255) / 256;
        float zv[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = threadIdx.x + 256 * i, rr = e / NP, j = e % NP;
            zv[i] = (e < 32 * NP && rr < nrows && j < N)
                        ? __ldg(p.dZ + g * p.dz_gs + (long long)(r0 + rr) * p.lddz + j) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = threadIdx.x + 256 * i;
            if (e < 32 * NP) sdz[e / NP][e % NP] = zv[i];
        }
    }
    __syncthreads();
    const float* W = p.W + g * p.w_gs;
    for (int q = threadIdx.x; q < p.K; q += blockDim.x) {
        float csum = 0.f;  // column sum of this block's 32 rows (bias gradient partial)
        float w[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) w[j] = j < N ? W[(long long)q * N + j] : 0.f;
        for (int rb = 0; rb < nrows; rb += 8) {
            float mk[8], ad[8];  // all loads of the batch in flight together
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const long long idx = g * p.c_gs + (long long)(r0 + rb + i) * p.ldc + q;
                const bool ok = rb + i < nrows;
                mk[i] = ok ? __ldg(p.mask + idx) : 0.f;
                ad[i] = (ok && p.add) ? __ldg(p.add + idx) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (rb + i >= nrows) break;
                float acc = 0.f;
#pragma unroll
                for (int j4 = 0; j4 < NP / 4; ++j4) {
                    const float4 z = *reinterpret_cast<const float4*>(&sdz[rb + i][4 * j4]);
                    acc = fmaf(z.x, w[4 * j4], acc);
                    acc = fmaf(z.y, w[4 * j4 + 1], acc);
                    acc = fmaf(z.z, w[4 * j4 + 2], acc);
                    acc = fmaf(z.w, w[4 * j4 + 3], acc);
                }
                if (p.add) acc = ad[i] + acc;
                const float outv = (mk[i] > 0.f) ? acc : 0.f;
                p.C[g * p.c_gs + (long long)(r0 + rb + i) * p.ldc + q] = outv;
                csum += outv;
            }
        }
        if (p.colsum) p.colsum[((long long)g * gridDim.x + blockIdx.x) * p.K + q] = csum;
    }
}

// ---- dW partials: block (64 features p, model g, row split rs); 4 row groups
// of 64 threads; thread owns feature p with NP accumulators; dz rows are
// broadcast float4 reads from smem.
constexpr int RS = 8;
template <int NP>
__global__ void __launch_bounds__(256) head_dw_partial_kernel(HeadDw p) {
    __shared__ __align__(16) float sdz[64][NP];
    __shared__ float red[4][64][NP + 1];
    const int g = blockIdx.y, rs = blockIdx.z;
    const int pl = threadIdx.x & 63, rg = threadIdx.x >> 6;
    const int pp = blockIdx.x * 64 + pl;
    const int N = p.N;
    const int rbeg = (int)((long long)p.rows * rs / RS), rend = (int)((long long)p.rows * (rs + 1) / RS);
    float acc[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) acc[n] = 0.f;
    const float* A = p.A + g * p.a_gs;
    const float* dz = p.dZ + g * p.dz_gs;
    for (int r0 = rbeg; r0 < rend; r0 += 64) {
        __syncthreads();
        {
            constexpr int PER = (64 * NP + 255) / 256;
            float zv[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = threadIdx.x + 256 * i, rr = e / NP, n = e % NP;
                zv[i] = (e < 64 * NP && r0 + rr < rend && n < N) ? __ldg(dz + (long long)(r0 + rr) * p.lddz + n) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = threadIdx.x + 256 * i;
                if (e < 64 * NP) sdz[e / NP][e % NP] = zv[i];
            }
        }
        __syncthreads();
        if (pp < p.K) {
            const int lim = min(64, rend - r0);
            float av[16];  // this thread's 16 rows of the chunk, loads in flight together
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int rr = rg + 4 * i;
                av[i] = rr < lim ? __ldg(A + (long long)(r0 + rr) * p.lda + pp) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int rr = rg + 4 * i;
#pragma unroll
                for (int n4 = 0; n4 < NP / 4; ++n4) {
                    const float4 z = *reinterpret_cast<const float4*>(&sdz[rr][4 * n4]);
                    acc[4 * n4] = fmaf(av[i], z.x, acc[4 * n4]);
                    acc[4 * n4 + 1] = fmaf(av[i], z.y, acc[4 * n4 + 1]);
                    acc[4 * n4 + 2] = fmaf(av[i], z.z, acc[4 * n4 + 2]);
                    acc[4 * n4 + 3] = fmaf(av[i], z.w, acc[4 * n4 + 3]);
                }
            }
        }
    }
#pragma unroll
    for (int n = 0; n < NP; ++n) red[rg][pl][n] = acc[n];
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
    const long long idx = g * p.w_gs + (p.trans ? (e % p.N) * p.K + e / p.N : e);
    if (p.grad_out) p.grad_out[idx] = gsum;
    const float w = param_update(p.W[idx], gsum, p.lr, p.adam, idx);
    if (!isfinite(w) && p.flags) atomicOr(p.flags, kFlagNonFinite);
    p.W[idx] = w;
}

// Forward-only 2-layer MLP with a tiny input and output (the attack model
// k -> H -> 2): one thread per row, all weights of model g in smem, the
// hidden layer streamed through registers (never written to HBM).
// Same sums as the layered path: (x W0) + b0 -> ReLU -> (h W1) + b1.
constexpr int S2_K = 8, S2_O = 4, S2_R = 4;  // rows per thread: each smem weight read serves 4 rows
__global__ void __launch_bounds__(256) small2_forward_kernel(const float* X, int rows, int K, int H,
                                                             int O, const float* W0, const float* b0,
                                                             const float* W1, const float* b1,
                                                             float* logits) {
    extern __shared__ float sw[];
    const int g = blockIdx.y;
    float* w0 = sw;                      // [K][H]
    float* c0 = w0 + K * H;              // [H]
    float* w1 = c0 + H;                  // [H][O]
    float* c1 = w1 + H * O;              // [O]
    for (int e = threadIdx.x; e < K * H; e += blockDim.x) w0[e] = W0[(long long)g * K * H + e];
    for (int e = threadIdx.x; e < H; e += blockDim.x) c0[e] = b0[(long long)g * H + e];
    for (int e = threadIdx.x; e < H * O; e += blockDim.x) w1[e] = W1[(long long)g * H * O + e];
    for (int e = threadIdx.x; e < O; e += blockDim.x) c1[e] = b1[(long long)g * O + e];
    __syncthreads();
    // rows r0 + 256 i, i < S2_R: a warp still reads 32 consecutive rows
    const int r0 = blockIdx.x * blockDim.x * S2_R + threadIdx.x;
    float xv[S2_R][S2_K], out[S2_R][S2_O];
#pragma unroll
    for (int i = 0; i < S2_R; ++i) {
        const int r = r0 + i * blockDim.x;
        const float* x = X + ((long long)g * rows + r) * K;
#pragma unroll
        for (int k = 0; k < S2_K; ++k) xv[i][k] = (k < K && r < rows) ? __ldg(x + k) : 0.f;
#pragma unroll
        for (int o = 0; o < S2_O; ++o) out[i][o] = 0.f;
    }
#pragma unroll 2
    for (int n = 0; n < H; ++n) {
        float wk[S2_K], wo[S2_O];
#pragma unroll
        for (int k = 0; k < S2_K; ++k) wk[k] = k < K ? w0[k * H + n] : 0.f;
#pragma unroll
        for (int o = 0; o < S2_O; ++o) wo[o] = o < O ? w1[n * O + o] : 0.f;
        const float bn = c0[n];
#pragma unroll
        for (int i = 0; i < S2_R; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < S2_K; ++k)
                if (k < K) acc = fmaf(xv[i][k], wk[k], acc);
            float h = acc + bn;
            h = h > 0.f ? h : 0.f;
#pragma unroll
            for (int o = 0; o < S2_O; ++o)
                if (o < O) out[i][o] = fmaf(h, wo[o], out[i][o]);
        }
    }
#pragma unroll
    for (int i = 0; i < S2_R; ++i) {
        const int r = r0 + i * blockDim.x;
        if (r >= rows) break;
        float* y = logits + ((long long)g * rows + r) * O;
#pragma unroll
        for (int o = 0; o < S2_O; ++o)
            if (o < O) y[o] = out[i][o] + c1[o];
    }
}

template <template <int> class Launch, typename P>
void by_width(int N, const P& p, cudaStream_t s) {
    switch ((N + 3) / 4) {
        case 1: Launch<4>::run(p, s); break;
        case 2: Launch<8>::run(p, s); break;
        case 3: Launch<12>::run(p, s); break;
        case 4: Launch<16>::run(p, s); break;
        case 5: Launch<20>::run(p, s); break;
        case 6: Launch<24>::run(p, s); break;
        case 7: Launch<28>::run(p, s); break;
        case 8: Launch<32>::run(p, s); break;
        default: fail(MTK_ERROR, "head: output width above 32");
    }
}

template <int NP>
struct FwdLaunch {
    static void run(const HeadFwd& p, cudaStream_t s) {
        CeArgs ce{};
        if (p.ce) ce = *p.ce;
        head_fwd_kernel<NP><<<dim3((p.rows + FR - 1) / FR, p.G), 128, 0, s>>>(p, ce, p.ce ? 1 : 0);
    }
};
template <int NP>
struct DxLaunch {
    static void run(const HeadDx& p, cudaStream_t s) {
        head_dx_kernel<NP><<<dim3((p.rows + 31) / 32, p.G), 256, 0, s>>>(p);
    }
};
template <int NP>
struct DwLaunch {
    static void run(const HeadDw& p, cudaStream_t s) {
        head_dw_partial_kernel<NP><<<dim3((p.K + 63) / 64, p.G, RS), 256, 0, s>>>(p);
    }
};

}  // namespace

bool head_fwd_ok(int K, int N) { return N >= 1 && N <= MAXN && K >= 1; }
bool head_dx_ok(int K, int N) { return N >= 1 && N <= MAXN && K >= 1; }
bool head_dw_ok(int N) { return N >= 1 && N <= MAXN; }

void launch_head_fwd(const HeadFwd& p, cudaStream_t s) {
    if (p.rows <= 0) return;
    if (p.ce && (p.ce->B != p.rows || p.ce->C != p.N || p.ce->logits != p.C || p.c_gs != (long long)p.rows * p.N ||
                 p.ldc != p.N || p.relu))
        fail(MTK_ERROR, "head_fwd: fused CE needs the [G][rows][N] logits of a linear head");
    by_width<FwdLaunch>(p.N, p, s);
    count_launch();
}

void launch_head_dx(const HeadDx& p, cudaStream_t s) {
    if (p.rows <= 0) return;
    by_width<DxLaunch>(p.N, p, s);
    count_launch();
}

bool small2_forward_ok(int K, int H, int O) {
    return K >= 1 && K <= S2_K && O >= 1 && O <= S2_O && H >= 1 &&
           (size_t)(K * H + H + H * O + O) * 4 <= 48 * 1024;
}

void launch_small2_forward(const float* X, int G, int rows, int K, int H, int O, const float* W0,
                           const float* b0, const float* W1, const float* b1, float* logits,
                           cudaStream_t s) {
    if (rows <= 0) return;
    const size_t smem = (size_t)(K * H + H + H * O + O) * 4;
    small2_forward_kernel<<<dim3((rows + 256 * S2_R - 1) / (256 * S2_R), G), 256, smem, s>>>(
        X, rows, K, H, O, W0, b0, W1, b1, logits);
    count_launch();
}

// ---- whole SGD epochs of the attack model (k -> 64 -> 2) in one launch: one
// CTA per model keeps its 386 parameters in shared memory and runs every
// step of the epoch -- gather, forward, softmax-CE, backward, update -- with
// one thread per batch row (row sets of 256).  The per-step launch chain of the generic bank
// step (about ten small kernels) is what bounds a model this small.
// Arithmetic per row follows the generic kernels (small2_forward / ce_row /
// head_dx); the gradient sums run in a fixed order: a butterfly over each
// warp's 32 rows, then the warps in ascending order.
constexpr int E_K = 3, E_H = 64, E_O = 2;
constexpr int E_NP = E_K * E_H + E_H + E_H * E_O + E_O;  // 386 parameters
constexpr int E_NG = (E_NP + 31) / 32;                    // 13 groups of 32 per butterfly
constexpr int E_THREADS = 256;  // rows [rs * 256 + t] for row sets rs < ceil(B / 256)

// value e of a row's gradient contribution (e is a compile-time index)
template <int e>
__device__ __forceinline__ float epoch_value(const float (&x)[E_K], const float (&hv)[E_H], const float (&dh)[E_H],
                                             const float (&dlog)[E_O]) {
    if constexpr (e < E_K * E_H) return x[e / E_H] * dh[e % E_H];
    else if constexpr (e < E_K * E_H + E_H) return dh[e - E_K * E_H];
    else if constexpr (e < E_K * E_H + E_H + E_H * E_O) return hv[(e - E_K * E_H - E_H) / E_O] * dlog[(e - E_K * E_H - E_H) % E_O];
    else if constexpr (e < E_NP) return dlog[e - E_K * E_H - E_H - E_H * E_O];
    else return 0.f;
}
template <int gi, int... c>
__device__ __forceinline__ void epoch_group(float (&v)[32], const float (&x)[E_K], const float (&hv)[E_H],
                                            const float (&dh)[E_H], const float (&dlog)[E_O],
                                            std::integer_sequence<int, c...>) {
    ((v[c] = epoch_value<gi * 32 + c>(x, hv, dh, dlog)), ...);
}
// the warp's 32 rows of gradient group gi -> lane l holds the sum of value gi * 32 + l
template <int gi>
__device__ __forceinline__ float epoch_reduce(int lane, const float (&x)[E_K], const float (&hv)[E_H],
                                              const float (&dh)[E_H], const float (&dlog)[E_O]) {
    float v[32];
    epoch_group<gi>(v, x, hv, dh, dlog, std::make_integer_sequence<int, 32>{});
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
        const bool up = (lane & k) != 0;
#pragma unroll
        for (int j = 0; j < k; ++j) {
            const float send = up ? v[j] : v[j + k];
            const float keep = up ? v[j + k] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, k);
        }
    }
    return v[0];
}
template <int... gi>
__device__ __forceinline__ void epoch_reduce_all(float (&acc)[E_NG], int lane, const float (&x)[E_K],
                                                 const float (&hv)[E_H], const float (&dh)[E_H],
                                                 const float (&dlog)[E_O], std::integer_sequence<int, gi...>) {
    ((acc[gi] += epoch_reduce<gi>(lane, x, hv, dh, dlog)), ...);
}

// One thread-block cluster per model: CTA c of the cluster takes row set c
// (rows c * 256 + t) of every step, so a 1024-row step runs on four SMs
// instead of one (the kernel is latency-bound on its butterflies; one CTA
// did 4 row sets in series).  The gradient sums keep the one-CTA order
// exactly: per warp w, ((0 + B_0) + B_1) + ... over the row sets (B_c = the
// warp's butterfly over row set c, read from CTA c's shared memory), then the
// warps in ascending order -- so the parameters are bit-identical to the
// one-CTA kernel.  Every CTA applies the update to its own copy; rank 0
// writes the model back.
__global__ void __launch_bounds__(E_THREADS, 1) small2_epoch_kernel(SmallEpoch p) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ float prm[E_NG * 32];                      // W0 [K][H], b0 [H], W1 [H][O], b1 [O]
    __shared__ float part[E_THREADS / 32][E_NG * 32];     // this CTA's warp partials
    const int nsets = (int)cluster.num_blocks();          // = ceil(B / 256)
    const int rs = (int)cluster.block_rank();
    const int g = blockIdx.x / nsets, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    float* gW0 = p.W0 + (long long)g * E_K * E_H;
    float* gb0 = p.b0 + (long long)g * E_H;
    float* gW1 = p.W1 + (long long)g * E_H * E_O;
    float* gb1 = p.b1 + (long long)g * E_O;
    for (int e = t; e < E_NG * 32; e += E_THREADS) {
        float v = 0.f;
        if (e < E_K * E_H) v = gW0[e];
        else if (e < E_K * E_H + E_H) v = gb0[e - E_K * E_H];
        else if (e < E_K * E_H + E_H + E_H * E_O) v = gW1[e - E_K * E_H - E_H];
        else if (e < E_NP) v = gb1[e - E_K * E_H - E_H - E_H * E_O];
        prm[e] = v;
    }
    const float* rpart[4];  // the cluster's partial arrays (row set c in CTA c)
    float* rprm[4];         // the cluster's parameter copies
    for (int c = 0; c < 4; ++c) {
        rpart[c] = c < nsets ? cluster.map_shared_rank(&part[0][0], c) : nullptr;
        rprm[c] = c < nsets ? cluster.map_shared_rank(&prm[0], c) : nullptr;
    }
    const int per = (E_NP + nsets - 1) / nsets;  // this CTA's parameter slice
    const int pe0 = rs * per, pe1 = min(E_NP, pe0 + per);
    __syncthreads();
    const float* W0 = prm;
    const float* B0 = W0 + E_K * E_H;
    const float* W1 = B0 + E_H;
    const float* B1 = W1 + E_H * E_O;
    bool bad = false;
    unsigned long long* tr = (p.trace && blockIdx.x == 0 && t == 0) ? p.trace : nullptr;
    auto stamp = [&](int s, int k) {
        if (tr && s < 8) {
            unsigned long long v;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
            tr[s * 8 + k] = v;
        }
    };
    // this thread's row of step s (index, features, label, weight): loaded one
    // step ahead (they do not depend on the parameters)
    const int r = rs * E_THREADS + t;
    struct RowIn {
        int status;  // 0 no row, 1 row, 2 bad index
        int lab;
        float x[E_K];
        float w;
    };
    auto load_row = [&](int s2) {
        RowIn in;
        in.status = 0;
        in.lab = 0;
        in.w = 1.f;
#pragma unroll
        for (int k = 0; k < E_K; ++k) in.x[k] = 0.f;
        if (s2 < p.nsteps && r < p.B) {
            const long long q = ((long long)s2 * p.G + g) * p.B + r;
            const long long row = p.idx[q];
            if (row < 0 || row >= p.pool_rows) {
                in.status = 2;
            } else {
                in.status = 1;
                in.lab = p.y[row];
#pragma unroll
                for (int k = 0; k < E_K; ++k) in.x[k] = p.X[row * E_K + k];
                if (p.w) in.w = p.w[q];
            }
        }
        return in;
    };
    RowIn nxt = load_row(0);
    for (int s = 0; s < p.nsteps; ++s) {
        stamp(s, 0);
        const RowIn cur = nxt;
        nxt = load_row(s + 1);
        float acc[E_NG];
#pragma unroll
        for (int q = 0; q < E_NG; ++q) acc[q] = 0.f;
        const float inv = (float)(1.0 / p.denom[s]);
        {
            float x[E_K], hv[E_H], dh[E_H], dlog[E_O];
#pragma unroll
            for (int k = 0; k < E_K; ++k) x[k] = 0.f;
#pragma unroll
            for (int h = 0; h < E_H; ++h) hv[h] = 0.f;
#pragma unroll
            for (int j = 0; j < E_O; ++j) dlog[j] = 0.f;
            if (cur.status != 0) {
                if (cur.status == 2) {
                    atomicOr(p.flags, kFlagBadIndex);
                } else {
                    const int lab = cur.lab;
#pragma unroll
                    for (int k = 0; k < E_K; ++k) x[k] = cur.x[k];
                    // forward (small2_forward_kernel's order)
#pragma unroll
                    for (int h = 0; h < E_H; ++h) {
                        float a = 0.f;
#pragma unroll
                        for (int k = 0; k < E_K; ++k) a = fmaf(x[k], W0[k * E_H + h], a);
                        a = a + B0[h];
                        hv[h] = a > 0.f ? a : 0.f;
                    }
                    float o[E_O];
#pragma unroll
                    for (int j = 0; j < E_O; ++j) o[j] = 0.f;
#pragma unroll
                    for (int h = 0; h < E_H; ++h)
#pragma unroll
                        for (int j = 0; j < E_O; ++j) o[j] = fmaf(hv[h], W1[h * E_O + j], o[j]);
#pragma unroll
                    for (int j = 0; j < E_O; ++j) o[j] = o[j] + B1[j];
                    if (lab < 0 || lab >= E_O) {
                        atomicOr(p.flags, kFlagBadLabel);
                        for (int k = 0; k < E_K; ++k) x[k] = 0.f;
                    } else {  // softmax-CE row (ce_row.cuh)
                        float mx = o[0];
#pragma unroll
                        for (int j = 1; j < E_O; ++j) mx = fmaxf(mx, o[j]);
                        float z = 0.f;
#pragma unroll
                        for (int j = 0; j < E_O; ++j) z += expf(o[j] - mx);
                        const float lse = mx + logf(z);
                        const float wi = cur.w * inv;
#pragma unroll
                        for (int j = 0; j < E_O; ++j)
                            dlog[j] = wi * (expf(o[j] - lse) - (j == lab ? 1.f : 0.f));
                    }
                }
            }
            stamp(s, 1);
            // backward through the ReLU (head_dx order: j ascending from 0)
#pragma unroll
            for (int h = 0; h < E_H; ++h) {
                float a = 0.f;
#pragma unroll
                for (int j = 0; j < E_O; ++j) a = fmaf(dlog[j], W1[h * E_O + j], a);
                dh[h] = hv[h] > 0.f ? a : 0.f;
            }
            stamp(s, 2);
            epoch_reduce_all(acc, lane, x, hv, dh, dlog, std::make_integer_sequence<int, E_NG>{});
            stamp(s, 3);
        }
#pragma unroll
        for (int q = 0; q < E_NG; ++q) part[warp][q * 32 + lane] = acc[q];
        cluster.sync();  // every row set's partials written
        stamp(s, 4);
        // per warp the row sets in order, then the warps in ascending order, then
        // SGD; CTA c owns a slice of the parameters (one per thread, its
        // 8 x nsets partial loads in flight together) and writes the update
        // into every CTA's copy
        for (int e = pe0 + t; e < pe1; e += E_THREADS) {
            float v[E_THREADS / 32][4];
#pragma unroll
            for (int w2 = 0; w2 < E_THREADS / 32; ++w2)
#pragma unroll
                for (int c = 0; c < 4; ++c) v[w2][c] = c < nsets ? rpart[c][w2 * E_NG * 32 + e] : 0.f;
            float gsum = 0.f;
#pragma unroll
            for (int w2 = 0; w2 < E_THREADS / 32; ++w2) {
                float a = v[w2][0];
#pragma unroll
                for (int c = 1; c < 4; ++c)
                    if (c < nsets) a += v[w2][c];
                gsum += a;
            }
            const float nv = sgd_update(prm[e], gsum, p.lr);
            bad |= !isfinite(nv);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < nsets) rprm[c][e] = nv;
        }
        stamp(s, 5);
        cluster.sync();  // partials read everywhere (the next step rewrites them); prm updated
        stamp(s, 6);
    }
    if (bad) atomicOr(p.flags, kFlagNonFinite);
    if (rs == 0)
        for (int e = t; e < E_NP; e += E_THREADS) {
            const float v = prm[e];
            if (e < E_K * E_H) gW0[e] = v;
            else if (e < E_K * E_H + E_H) gb0[e - E_K * E_H] = v;
            else if (e < E_K * E_H + E_H + E_H * E_O) gW1[e - E_K * E_H - E_H] = v;
            else gb1[e - E_K * E_H - E_H - E_H * E_O] = v;
        }
}

bool small2_epoch_ok(int K, int H, int O, int B) { return K == E_K && H == E_H && O == E_O && B >= 1 && B <= 1024; }

void launch_small2_epoch(const SmallEpoch& p, cudaStream_t s) {
    if (!small2_epoch_ok(E_K, E_H, E_O, p.B)) fail(MTK_ERROR, "small2_epoch: unsupported shape");
    if (p.nsteps <= 0 || p.G <= 0) return;
    const int nsets = (p.B + E_THREADS - 1) / E_THREADS;  // <= 4: the cluster size
    SmallEpoch q = p;
    if (const char* t = getenv("MTK_EPOCH_TRACE")) q.trace = reinterpret_cast<unsigned long long*>(strtoull(t, nullptr, 0));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(p.G * nsets));
    cfg.blockDim = dim3(E_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)nsets;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MTK_CUDA(cudaLaunchKernelEx(&cfg, small2_epoch_kernel, q));
    count_launch();
}

size_t head_dw_scratch_bytes(int G, int K, int N) { return (size_t)RS * G * K * N * sizeof(float); }

void launch_head_dw(const HeadDw& p, cudaStream_t s) {
    if (p.K <= 0) return;
    if (!p.partial) fail(MTK_ERROR, "head_dw: missing partial scratch");
    by_width<DwLaunch>(p.N, p, s);
    count_launch();
    const long long n = (long long)p.G * p.K * p.N;
    head_dw_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p);
    count_launch();
}

}  // namespace mtk
