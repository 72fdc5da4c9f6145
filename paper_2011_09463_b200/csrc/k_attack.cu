// k_attack.cu -- membership-attack stage: posteriors, top-k features, AUC.
//
// Posteriors follow Tape::softmax (tape.hpp:433-464): max-subtracted exp,
// normalised by the row sum.  Features and AUC have no reference code
// (SURVEY.md section 8(a) row a18); definitions per SURVEY.md Appendix A and
// oracle.c (orc_posterior_features, orc_auc).  These are streaming,
// HBM-bound kernels: one thread per query row, coalesced row-major output.
#include <cub/cub.cuh>

#include <cmath>

#include "internal.h"

namespace mtk {
namespace {

constexpr int MAXC = 64;

__global__ void softmax_kernel(const float* logits, long long rows, int C, float* probs) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* x = logits + r * C;
    float* p = probs + r * C;
    float mx = x[0];
    for (int j = 1; j < C; ++j) mx = fmaxf(mx, x[j]);
    float z = 0.f;
    for (int j = 0; j < C; ++j) {
        const float e = expf(x[j] - mx);
        p[j] = e;
        z += e;
    }
    const float inv = 1.f / z;
    for (int j = 0; j < C; ++j) p[j] *= inv;
}

// C <= 16 (the 10-class posteriors): everything in registers, top-k by
// unrolled insertion into a descending register list (values only, so tie
// order does not matter).
template <int CC>
__global__ void features_small_kernel(const float* logits, long long rows, int C, int k,
                                      const int32_t* labels, float* feats, int* flags) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* x = logits + r * C;
    float v[CC];
#pragma unroll
    for (int j = 0; j < CC; ++j) v[j] = j < C ? __ldg(x + j) : -INFINITY;
    float mx = v[0];
#pragma unroll
    for (int j = 1; j < CC; ++j) mx = fmaxf(mx, v[j]);
    float z = 0.f;
#pragma unroll
    for (int j = 0; j < CC; ++j) {
        v[j] = j < C ? expf(v[j] - mx) : 0.f;
        z += v[j];
    }
    const float inv = 1.f / z;
    constexpr int KM = 8;
    float top[KM];
#pragma unroll
    for (int a = 0; a < KM; ++a) top[a] = -1.f;
#pragma unroll
    for (int j = 0; j < CC; ++j) {
        if (j >= C) break;
        float t = v[j] * inv;
#pragma unroll
        for (int a = 0; a < KM; ++a) {  // insert t, keep descending
            if (a >= k) break;
            const float hi = fmaxf(top[a], t), lo = fminf(top[a], t);
            top[a] = hi;
            t = lo;
        }
    }
    const int nf = k + (labels ? 1 : 0);
    float* out = feats + r * nf;
#pragma unroll
    for (int a = 0; a < KM; ++a)
        if (a < k) out[a] = top[a];
    if (labels) {
        const int lab = labels[r];
        if (lab < 0 || lab >= C) {
            atomicOr(flags, kFlagBadLabel);
            out[k] = 0.f;
        } else {
            out[k] = mx + logf(z) - x[lab];
        }
    }
}

__global__ void features_kernel(const float* logits, long long rows, int C, int k,
                                const int32_t* labels, float* feats, int* flags) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* x = logits + r * C;
    float p[MAXC];
    float mx = x[0];
    for (int j = 1; j < C; ++j) mx = fmaxf(mx, x[j]);
    float z = 0.f;
    for (int j = 0; j < C; ++j) {
        p[j] = expf(x[j] - mx);
        z += p[j];
    }
    const float inv = 1.f / z;
    for (int j = 0; j < C; ++j) p[j] *= inv;
    const int nf = k + (labels ? 1 : 0);
    float* out = feats + r * nf;
    for (int a = 0; a < k; ++a) {
        int best = a;
        for (int j = a + 1; j < C; ++j)
            if (p[j] > p[best]) best = j;
        const float t = p[a];
        p[a] = p[best];
        p[best] = t;
        out[a] = p[a];
    }
    if (labels) {
        const int lab = labels[r];
        if (lab < 0 || lab >= C) {
            atomicOr(flags, kFlagBadLabel);
            out[k] = 0.f;
        } else {
            out[k] = mx + logf(z) - x[lab];
        }
    }
}

__global__ void column_kernel(const float* logits, long long rows, int C, int col, float* out) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* x = logits + r * C;
    float mx = x[0];
    for (int j = 1; j < C; ++j) mx = fmaxf(mx, x[j]);
    float z = 0.f;
    for (int j = 0; j < C; ++j) z += expf(x[j] - mx);
    out[r] = expf(x[col] - mx) / z;
}

// ---- AUC -------------------------------------------------------------------
// order-preserving map float -> uint32 (ascending), -0.0 == +0.0
__global__ void auc_keys_kernel(const float* s, const uint8_t* lab, long long n, uint32_t* keys,
                                uint8_t* vals, unsigned long long* counts) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long pos = 0, hit = 0;
    if (i < n) {
        float v = s[i];
        if (v == 0.f) v = 0.f;
        uint32_t u = __float_as_uint(v);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        keys[i] = u;
        const uint8_t l = lab[i] ? 1 : 0;
        vals[i] = l;
        pos = l;
        hit = ((s[i] > 0.5f) == (l != 0));
    }
    // block-aggregated integer atomics: exact and order-independent
    __shared__ unsigned long long sp[8], sh[8];
    for (int o = 16; o > 0; o >>= 1) {
        pos += __shfl_down_sync(0xffffffffu, pos, o);
        hit += __shfl_down_sync(0xffffffffu, hit, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sp[threadIdx.x >> 5] = pos;
        sh[threadIdx.x >> 5] = hit;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += sp[w];
            b += sh[w];
        }
        if (a) atomicAdd(&counts[0], a);
        if (b) atomicAdd(&counts[1], b);
    }
}

__global__ void auc_start_flags(const uint32_t* k, long long n, int* flag) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// gid = inclusive_sum(flag) - 1; record [start, end) of each tie group
__global__ void auc_group_bounds(const uint32_t* k, const int* gid1, long long n, long long* gstart,
                                 long long* gend) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int g = gid1[i] - 1;
    if (i == 0 || k[i] != k[i - 1]) gstart[g] = i;
    if (i == n - 1 || k[i] != k[i + 1]) gend[g] = i + 1;
}

// 2 * rank_sum of positives = sum over positives of (start + 1 + end) (exact int64)
__global__ void auc_rank_sum(const uint8_t* v, const int* gid1, long long n, const long long* gstart,
                             const long long* gend, unsigned long long* acc) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long t = 0;
    if (i < n && v[i]) {
        const int g = gid1[i] - 1;
        t = (unsigned long long)(gstart[g] + 1 + gend[g]);
    }
    __shared__ unsigned long long st[8];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) st[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += st[w];
        if (a) atomicAdd(acc, a);
    }
}

inline unsigned nblocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// one warp per output row: a row-contiguous copy (16-B vectors when aligned)
__global__ void gather_rows_kernel(const uint32_t* src, long long src_rows, int d, const long long* idx,
                                   int G, int nb, uint32_t* out, int out_rows, int row0, int* flags) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= (long long)G * nb) return;
    const int g = (int)(w / nb), r = (int)(w % nb);
    const long long s = idx[w];
    if (s < 0 || s >= src_rows) {
        if (lane == 0) atomicOr(flags, kFlagBadIndex);
        return;
    }
    const uint32_t* a = src + s * d;
    uint32_t* o = out + ((long long)g * out_rows + row0 + r) * d;
    if ((d & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(o)) & 15) == 0) {
        for (int k = lane; k < d / 4; k += 32)
            reinterpret_cast<uint4*>(o)[k] = __ldg(reinterpret_cast<const uint4*>(a) + k);
    } else {
        for (int k = lane; k < d; k += 32) o[k] = __ldg(a + k);
    }
}

}  // namespace

void launch_gather_rows(const uint32_t* src, long long src_rows, int d, const long long* idx, int G,
                        int nb, uint32_t* out, int out_rows, int row0, int* flags, cudaStream_t s) {
    const long long rows = (long long)G * nb;
    if (rows <= 0) return;
    gather_rows_kernel<<<nblocks(rows * 32, 256), 256, 0, s>>>(src, src_rows, d, idx, G, nb, out, out_rows,
                                                                 row0, flags);
    count_launch();
}

void launch_softmax(const float* logits, long long rows, int C, float* probs, cudaStream_t s) {
    if (rows <= 0) return;
    softmax_kernel<<<nblocks(rows, 256), 256, 0, s>>>(logits, rows, C, probs);
    count_launch();
}

void launch_features(const float* logits, long long rows, int C, int k, const int32_t* labels,
                     float* feats, int* flags, cudaStream_t s) {
    if (C > MAXC) fail(MTK_SHAPE_ERROR, "posterior_features: more than 64 classes");
    if (rows <= 0) return;
    if (C <= 16 && k <= 8)
        features_small_kernel<16><<<nblocks(rows, 256), 256, 0, s>>>(logits, rows, C, k, labels, feats,
                                                                      flags);
    else
        features_kernel<<<nblocks(rows, 256), 256, 0, s>>>(logits, rows, C, k, labels, feats, flags);
    count_launch();
}

void launch_column(const float* logits, long long rows, int C, int col, float* out,
                   cudaStream_t s) {
    if (rows <= 0) return;
    column_kernel<<<nblocks(rows, 256), 256, 0, s>>>(logits, rows, C, col, out);
    count_launch();
}

void auc_device(Ctx& ctx, const float* scores, const uint8_t* labels, long long n, double* auc,
                double* acc) {
    cudaStream_t s = ctx.stream;
    if (n > 0x7fffffffLL) fail(MTK_SHAPE_ERROR, "auc: more than 2^31 rows");
    const int ni = (int)n;
    // workspace: keys(2), vals(2), flags/gid(2 ints), gstart/gend (2 int64), counters
    size_t sort_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint8_t*)nullptr, (uint8_t*)nullptr, ni, 0, 32, s);
    cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (int*)nullptr, (int*)nullptr, ni, s);
    const size_t tmp = std::max(sort_bytes, scan_bytes);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bytes = al(4 * n) * 2 + al(n) * 2 + al(4 * n) * 2 + al(8 * n) * 2 + al(64) + al(tmp);
    char* base = static_cast<char*>(ctx.big(bytes));
    char* p = base;
    auto take = [&](size_t b) { char* r = p; p += al(b); return r; };
    uint32_t* k_in = (uint32_t*)take(4 * n);
    uint32_t* k_out = (uint32_t*)take(4 * n);
    uint8_t* v_in = (uint8_t*)take(n);
    uint8_t* v_out = (uint8_t*)take(n);
    int* flag = (int*)take(4 * n);
    int* gid = (int*)take(4 * n);
    long long* gstart = (long long*)take(8 * n);
    long long* gend = (long long*)take(8 * n);
    unsigned long long* cnt = (unsigned long long*)take(64);
    void* wk = take(tmp);
    MTK_CUDA(cudaMemsetAsync(cnt, 0, 64, s));
    auc_keys_kernel<<<nblocks(n, 256), 256, 0, s>>>(scores, labels, n, k_in, v_in, cnt);
    count_launch();
    cub::DeviceRadixSort::SortPairs(wk, sort_bytes, k_in, k_out, v_in, v_out, ni, 0, 32, s);
    auc_start_flags<<<nblocks(n, 256), 256, 0, s>>>(k_out, n, flag);
    count_launch();
    cub::DeviceScan::InclusiveSum(wk, scan_bytes, flag, gid, ni, s);
    auc_group_bounds<<<nblocks(n, 256), 256, 0, s>>>(k_out, gid, n, gstart, gend);
    count_launch();
    auc_rank_sum<<<nblocks(n, 256), 256, 0, s>>>(v_out, gid, n, gstart, gend, cnt + 2);
    count_launch();
    unsigned long long h[3];
    MTK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    MTK_CUDA(cudaStreamSynchronize(s));
    const double npos = (double)h[0], nneg = (double)n - npos;
    if (h[0] == 0 || npos == (double)n)
        fail(MTK_VALUE_ERROR, "auc: need at least one member and one non-member");
    if (auc) *auc = (0.5 * (double)h[2] - npos * (npos + 1.0) * 0.5) / (npos * nneg);
    if (acc) *acc = (double)h[1] / (double)n;
}

}  // namespace mtk
