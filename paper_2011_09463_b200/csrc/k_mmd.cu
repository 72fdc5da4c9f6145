// k_mmd.cu -- multi-bandwidth Gaussian MMD^2 and its gradient (SIMT fp32
// pair tiles, fp64 cross-tile accumulation).
//
// The reference has no MMD; the definition
// pinned in SURVEY.md Appendix A is restated in oracle.c:orc_mmd_gaussian.
//   k(x,y)  = sum_b exp(-|x-y|^2 / s_b),  s_b = beta * mult_b, beta detached
//   MMD^2   = ss/m^2 + tt/n^2 - 2 st/(m n)      (biased V-statistic)
//   g_i     = sum_j c_ij A_ij (z_i - z_j),  A_ij = sum_b (2/s_b) k_b
//             c = -2/m^2 (S,S), -2/n^2 (T,T), +2/(m n) (cross)
// Layout: rows of the concatenated sample Z = [Xs; Xt]; a block owns TI rows
// i and streams every j tile, so each g_i is produced by one block in a fixed
// j order (deterministic, no atomics).  Per-block kernel sums are fp64.
#include <cmath>

#include "internal.h"

namespace mtk {
namespace {

constexpr int TI = 16, TJ = 64, NT = 256, MAXD = 512;

__device__ __forceinline__ const float* row_ptr(const MmdArgs& a, int g, long long r) {
    return r < a.m ? a.Xs + g * a.xs_gs + r * a.d : a.Xt + g * a.xt_gs + (r - a.m) * a.d;
}

// beta partials: block (p, g) sums rows [p*R, p*R+R) -> sum z (per dim), sum |z|^2
constexpr int BETA_ROWS = kBetaRows;
__global__ void beta_partial_kernel(MmdArgs a, double* part, int P) {
    const int g = blockIdx.y, p = blockIdx.x;
    const long long N = a.m + a.n;
    const long long r0 = (long long)p * BETA_ROWS, r1 = min(N, r0 + BETA_ROWS);
    double* out = part + ((long long)g * P + p) * (a.d + 1);
    double sq = 0.0;
    for (int k = threadIdx.x; k < a.d; k += blockDim.x) {
        double s = 0.0;
#pragma unroll 8
        for (long long r = r0; r < r1; ++r) {
            const double v = row_ptr(a, g, r)[k];
            s += v;
            sq += v * v;
        }
        out[k] = s;
    }
    __shared__ double red[NT];
    red[threadIdx.x] = sq;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[a.d] = red[0];
}

__global__ void beta_finish_kernel(MmdArgs a, const double* part, int P, double* beta) {
    const int g = blockIdx.x;
    __shared__ double red[NT];
    double ss = 0.0;
    for (int k = threadIdx.x; k < a.d; k += NT) {
        double s = 0.0;
        const double* src = part + (long long)g * P * (a.d + 1) + k;
        int p = 0;
        for (; p + 16 <= P; p += 16) {  // 16 loads in flight, then the fixed-order sum
            double v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = src[(long long)(p + q) * (a.d + 1)];
#pragma unroll
            for (int q = 0; q < 16; ++q) s += v[q];
        }
        for (; p < P; ++p) s += src[(long long)p * (a.d + 1)];
        ss += s * s;
    }
    red[threadIdx.x] = ss;
    // the row-norm partials, loaded in parallel, summed in order by thread 0
    __shared__ double np[NT];
    for (int p = threadIdx.x; p < min(P, NT); p += NT) np[p] = part[((long long)g * P + p) * (a.d + 1) + a.d];
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int p = 0; p < P; ++p) s2 += p < NT ? np[p] : part[((long long)g * P + p) * (a.d + 1) + a.d];
        const double N = (double)(a.m + a.n);
        beta[g] = (2.0 * N * s2 - 2.0 * red[0]) / (N * N - N);
    }
}

__global__ void __launch_bounds__(NT, 1) mmd_pairs_kernel(MmdArgs a, int nblk) {
    extern __shared__ float smem[];
    const int d = a.d, ld = d + 1;
    float* Zi = smem;                 // [TI][ld]
    float* Zj = Zi + TI * ld;         // [TJ][ld]
    float* Ws = Zj + TJ * ld;         // [TI][TJ]
    const int g = blockIdx.y;
    const long long N = a.m + a.n;
    const long long rb = a.row_begin, re = a.row_end < 0 ? N : a.row_end;
    const long long i0 = rb + (long long)blockIdx.x * TI;
    const int tid = threadIdx.x;
    const bool want_grad = (a.gXs != nullptr) || (a.gXt != nullptr);

    const double beta = a.beta[g];
    float inv_s[8];
    float two_inv_s[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const double s = beta * (double)a.mult[b];
        inv_s[b] = b < a.nb ? (float)(1.0 / s) : 0.f;
        two_inv_s[b] = 2.f * inv_s[b];
    }
    const float cSS = (float)(-2.0 / ((double)a.m * (double)a.m));
    const float cTT = (float)(-2.0 / ((double)a.n * (double)a.n));
    const float cST = (float)(2.0 / ((double)a.m * (double)a.n));

    for (int e = tid; e < TI * d; e += NT) {
        const int r = e / d, k = e - r * d;
        const long long gi = i0 + r;
        Zi[r * ld + k] = (gi < re) ? row_ptr(a, g, gi)[k] : 0.f;
    }

    // phase-1 mapping: rows ri0, ri0+8; cols cj0, cj0+32
    const int ri0 = tid >> 5, cj0 = tid & 31;
    // phase-2 mapping: dims k0 = tid, tid+256 ; all TI rows
    const int kq = (d + NT - 1) / NT;  // 1 or 2
    double gacc[TI][2];
    float zi_reg[TI][2];
#pragma unroll
    for (int r = 0; r < TI; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) gacc[r][q] = 0.0;
    double ksum[3] = {0.0, 0.0, 0.0};
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TI; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int k = tid + q * NT;
            zi_reg[r][q] = (q < kq && k < d) ? Zi[r * ld + k] : 0.f;
        }

    for (long long j0 = 0; j0 < N; j0 += TJ) {
        __syncthreads();
        for (int e = tid; e < TJ * d; e += NT) {
            const int r = e / d, k = e - r * d;
            const long long gj = j0 + r;
            Zj[r * ld + k] = (gj < N) ? row_ptr(a, g, gj)[k] : 0.f;
        }
        __syncthreads();
        float d00 = 0.f, d01 = 0.f, d10 = 0.f, d11 = 0.f;
        const float* zi0 = Zi + ri0 * ld;
        const float* zi1 = Zi + (ri0 + 8) * ld;
        const float* zj0 = Zj + cj0 * ld;
        const float* zj1 = Zj + (cj0 + 32) * ld;
        for (int k = 0; k < d; ++k) {
            const float a0 = zi0[k], a1 = zi1[k], b0 = zj0[k], b1 = zj1[k];
            const float t00 = a0 - b0, t01 = a0 - b1, t10 = a1 - b0, t11 = a1 - b1;
            d00 = fmaf(t00, t00, d00);
            d01 = fmaf(t01, t01, d01);
            d10 = fmaf(t10, t10, d10);
            d11 = fmaf(t11, t11, d11);
        }
        const float dd[4] = {d00, d01, d10, d11};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ri = ri0 + (q >> 1) * 8, cj = cj0 + (q & 1) * 32;
            const long long gi = i0 + ri, gj = j0 + cj;
            float wv = 0.f;
            if (gi < re && gj < N) {
                float kv = 0.f, A = 0.f;
                for (int b = 0; b < a.nb; ++b) {
                    const float e = expf(-dd[q] * inv_s[b]);
                    kv += e;
                    A = fmaf(two_inv_s[b], e, A);
                }
                const bool si = gi < a.m, sj = gj < a.m;
                if (si && sj) {
                    ksum[0] += kv;
                    wv = cSS * A;
                } else if (!si && !sj) {
                    ksum[1] += kv;
                    wv = cTT * A;
                } else {
                    if (si) ksum[2] += kv;
                    wv = cST * A;
                }
                if (gi == gj) wv = 0.f;
            }
            Ws[ri * TJ + cj] = wv;
        }
        if (!want_grad) continue;
        __syncthreads();
        float part[TI][2];
#pragma unroll
        for (int r = 0; r < TI; ++r) part[r][0] = part[r][1] = 0.f;
        for (int j = 0; j < TJ; ++j) {
            const float zj_0 = tid < d ? Zj[j * ld + tid] : 0.f;
            const float zj_1 = (kq > 1 && tid + NT < d) ? Zj[j * ld + tid + NT] : 0.f;
#pragma unroll
            for (int r = 0; r < TI; ++r) {
                const float w = Ws[r * TJ + j];
                part[r][0] = fmaf(w, zi_reg[r][0] - zj_0, part[r][0]);
                part[r][1] = fmaf(w, zi_reg[r][1] - zj_1, part[r][1]);
            }
        }
#pragma unroll
        for (int r = 0; r < TI; ++r) {
            gacc[r][0] += (double)part[r][0];
            gacc[r][1] += (double)part[r][1];
        }
    }

    if (want_grad) {
#pragma unroll
        for (int r = 0; r < TI; ++r) {
            const long long gi = i0 + r;
            if (gi >= re) break;
            float* out = gi < a.m ? (a.gXs ? a.gXs + g * a.gs_gs + gi * d : nullptr)
                                  : (a.gXt ? a.gXt + g * a.gt_gs + (gi - a.m) * d : nullptr);
            if (!out) continue;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int k = tid + q * NT;
                if (q < kq && k < d) {
                    const float v = (float)(gacc[r][q] * (double)a.grad_scale);
                    if (!isfinite(v)) atomicOr(a.flags, kFlagNonFinite);
                    out[k] = v;
                }
            }
        }
    }
    // block reduction of the three kernel sums (fixed tree order)
    __shared__ double red[3][NT];
#pragma unroll
    for (int c = 0; c < 3; ++c) red[c][tid] = ksum[c];
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (tid < w)
#pragma unroll
            for (int c = 0; c < 3; ++c) red[c][tid] += red[c][tid + w];
        __syncthreads();
    }
    if (tid < 3) a.partial[((long long)g * nblk + blockIdx.x) * 3 + tid] = red[tid][0];
}

__global__ void mmd_finish_kernel(MmdArgs a, int nblk, double* value, double* sums3) {
    const int g = blockIdx.x;
    if (threadIdx.x != 0) return;
    double s[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < nblk; ++b)
        for (int c = 0; c < 3; ++c) s[c] += a.partial[((long long)g * nblk + b) * 3 + c];
    const double m = (double)a.m, n = (double)a.n;
    if (value) {
        value[g] = s[0] / (m * m) + s[1] / (n * n) - 2.0 * s[2] / (m * n);
        if (!isfinite(value[g])) atomicOr(a.flags, kFlagNonFinite);
    }
    if (sums3)
        for (int c = 0; c < 3; ++c) sums3[g * 3 + c] = s[c];
}

}  // namespace

int mmd_blocks_per_group(const MmdArgs& a) {
    if (a.tc) return mmd_tc_blocks_per_group(a);
    const long long N = a.m + a.n;
    const long long re = a.row_end < 0 ? N : a.row_end;
    return (int)((re - a.row_begin + TI - 1) / TI);
}

size_t mmd_beta_scratch_bytes(const MmdArgs& a) {
    const long long N = a.m + a.n;
    return (size_t)a.G * ((N + BETA_ROWS - 1) / BETA_ROWS) * (a.d + 1) * sizeof(double);
}

void launch_mmd_beta(const MmdArgs& a, double* beta_out, double* scratch, cudaStream_t s) {
    const long long N = a.m + a.n;
    const int P = (int)((N + BETA_ROWS - 1) / BETA_ROWS);
    beta_partial_kernel<<<dim3(P, a.G), NT, 0, s>>>(a, scratch, P);
    count_launch();
    beta_finish_kernel<<<a.G, NT, 0, s>>>(a, scratch, P, beta_out);
    count_launch();
}

void launch_mmd_beta_finish(const MmdArgs& a, const double* part, double* beta_out, cudaStream_t s) {
    const long long N = a.m + a.n;
    const int P = (int)((N + BETA_ROWS - 1) / BETA_ROWS);
    beta_finish_kernel<<<a.G, NT, 0, s>>>(a, part, P, beta_out);
    count_launch();
}

void launch_mmd_pairs(const MmdArgs& a, cudaStream_t s) {
    if (a.d > MAXD) fail(MTK_SHAPE_ERROR, "mmd: feature dim above 512 is not supported");
    const int nblk = mmd_blocks_per_group(a);
    if (nblk <= 0) return;
    const size_t smem = (size_t)((TI + TJ) * (a.d + 1) + TI * TJ) * sizeof(float);
    ensure_smem_attr(reinterpret_cast<const void*>(mmd_pairs_kernel), (int)((TI + TJ) * (MAXD + 1) + TI * TJ) * 4);
    mmd_pairs_kernel<<<dim3(nblk, a.G), NT, smem, s>>>(a, nblk);
    count_launch();
}

void launch_mmd_finish(const MmdArgs& a, double* value, double* sums3, cudaStream_t s) {
    mmd_finish_kernel<<<a.G, 32, 0, s>>>(a, mmd_blocks_per_group(a), value, sums3);
    count_launch();
}

}  // namespace mtk
