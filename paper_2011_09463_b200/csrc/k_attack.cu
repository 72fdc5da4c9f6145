// k_attack.cu -- membership-attack stage: posteriors, top-k features, AUC.
//
// Posteriors follow Tape::softmax (tape.hpp:433-464): max-subtracted exp,
// normalised by the row sum.  Features and AUC have no reference code
// (SURVEY.md section 8(a) row a18); definitions per SURVEY.md Appendix A and
// oracle.c (orc_posterior_features, orc_auc).  These are streaming,
// HBM-bound kernels: one thread per query row, coalesced row-major output.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <mutex>

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
// Exact mid-rank AUC without a tie pass: with the non-members' keys sorted,
// each member contributes 2 * #{non-members below} + #{non-members equal}
// (lower / upper bound); U2 = the sum (exact uint64) = 2 * (R_pos - npos (npos+1) / 2).
// order-preserving map float -> uint32 (ascending), -0.0 == +0.0
__device__ __forceinline__ uint32_t auc_key(float v) {
    if (v == 0.f) v = 0.f;
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // a member's slot in the non-member key array

// block-aggregated integer atomics (exact, order-independent): cnt[0] += pos, cnt[1] += hit
__device__ __forceinline__ void add_counts(unsigned long long pos, unsigned long long hit,
                                           unsigned long long* cnt) {
    __shared__ unsigned long long sp[32], sh[32];
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
        if (a) atomicAdd(&cnt[0], a);
        if (b) atomicAdd(&cnt[1], b);
    }
}

// per query: kn = key (non-member) or the sentinel (member); kp = key (member)
__global__ void auc_keys_kernel(const float* s, const uint8_t* lab, long long n, uint32_t* kn,
                                uint32_t* kp, unsigned long long* counts) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long pos = 0, hit = 0;
    if (i < n) {
        const uint32_t u = auc_key(s[i]);
        const bool l = lab[i] != 0;
        kn[i] = l ? kSentinel : u;
        kp[i] = u;
        pos = l;
        hit = ((s[i] > 0.5f) == l);
    }
    add_counts(pos, hit, counts);
}

// members: U2 += 2 * lower_bound + (upper_bound - lower_bound) over the sorted
// non-member keys sorted[0, nneg) (nneg = n - cnt[0], read on the device).
// A block keeps every step-th sorted key in shared memory (AUC_SAMPLES of
// them), so a search touches global memory only inside one step-wide segment;
// the upper bound gallops from the lower bound (ties are usually short).
constexpr int AUC_SAMPLES = 8192, AUC_THREADS = 512;
__global__ void __launch_bounds__(AUC_THREADS) auc_member_count(const uint32_t* sorted, const uint32_t* kp,
                                                                const uint8_t* lab, long long n,
                                                                unsigned long long* cnt) {
    __shared__ uint32_t samp[AUC_SAMPLES];
    __shared__ unsigned long long st[AUC_THREADS / 32];
    const long long nneg = n - (long long)cnt[0];
    const long long step = nneg > AUC_SAMPLES ? (nneg + AUC_SAMPLES - 1) / AUC_SAMPLES : 1;
    const int ns = (int)((nneg + step - 1) / step);  // samp[s] = sorted[s * step]
    for (int i = threadIdx.x; i < ns; i += blockDim.x) samp[i] = sorted[(long long)i * step];
    __syncthreads();
    unsigned long long t = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (!lab[i]) continue;
        const uint32_t u = kp[i];
        int a = 0, b = ns;  // first sample >= u
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (samp[mid] < u) a = mid + 1;
            else b = mid;
        }
        // sorted[(a - 1) * step] < u <= sorted[a * step]: lower bound in ((a-1) step, a step]
        long long lo = a > 0 ? (long long)(a - 1) * step + 1 : 0, hi = a < ns ? (long long)a * step : nneg;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (sorted[mid] < u) lo = mid + 1;
            else hi = mid;
        }
        long long ub = lo, inc = 1;  // gallop: first index > u
        while (ub < nneg && sorted[ub] <= u) {
            ub += inc;
            inc <<= 1;
        }
        long long glo = ub - (inc >> 1), ghi = ub < nneg ? ub : nneg;  // sorted[glo - 1] <= u (or glo = lo)
        if (glo < lo) glo = lo;
        while (glo < ghi) {
            const long long mid = (glo + ghi) >> 1;
            if (sorted[mid] <= u) glo = mid + 1;
            else ghi = mid;
        }
        t += (unsigned long long)(lo + glo);  // 2 * below + equal
    }
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) st[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += st[w];
        if (acc) atomicAdd(&cnt[2], acc);
    }
}

// ---- fused attack scoring: posterior softmax -> top-KF sorted features ->
// attack MLP KF -> H (ReLU) -> 2 -> member posterior -> AUC keys, one pass
// over the logits.  Same arithmetic, in the same order, as features_small_kernel,
// small2_forward_kernel and column_kernel (bit-identical scores); the attack
// model's weights sit in constant memory (warp-uniform operands).
constexpr int ATT_K = 3, ATT_H = 64;
__constant__ float c_att[ATT_K * ATT_H + ATT_H + ATT_H * 2 + 2];  // W0 [K][H], b0 [H], W1 [H][2], b1 [2]

template <int CC>
__global__ void __launch_bounds__(256) attack_score_kernel(const float* logits, long long rows, int C,
                                                           const uint8_t* lab, float* score_out, uint32_t* kn,
                                                           uint32_t* kp, unsigned long long* cnt) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long pos = 0, hit = 0;
    if (r < rows) {
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
        float top[ATT_K];
#pragma unroll
        for (int a = 0; a < ATT_K; ++a) top[a] = -1.f;
#pragma unroll
        for (int j = 0; j < CC; ++j) {
            if (j >= C) break;
            float t = v[j] * inv;
#pragma unroll
            for (int a = 0; a < ATT_K; ++a) {
                const float hi = fmaxf(top[a], t), lo = fminf(top[a], t);
                top[a] = hi;
                t = lo;
            }
        }
        const float* W0 = c_att;
        const float* B0 = W0 + ATT_K * ATT_H;
        const float* W1 = B0 + ATT_H;
        const float* B1 = W1 + ATT_H * 2;
        float o0 = 0.f, o1 = 0.f;
#pragma unroll
        for (int h = 0; h < ATT_H; ++h) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < ATT_K; ++k) acc = fmaf(top[k], W0[k * ATT_H + h], acc);
            float hv = acc + B0[h];
            hv = hv > 0.f ? hv : 0.f;
            o0 = fmaf(hv, W1[h * 2], o0);
            o1 = fmaf(hv, W1[h * 2 + 1], o1);
        }
        o0 = o0 + B1[0];
        o1 = o1 + B1[1];
        // member posterior: column_kernel's softmax column 1
        const float m2 = fmaxf(o0, o1);
        const float z2 = expf(o0 - m2) + expf(o1 - m2);
        const float sc = expf(o1 - m2) / z2;
        if (score_out) score_out[r] = sc;
        const uint32_t u = auc_key(sc);
        const bool l = lab[r] != 0;
        kn[r] = l ? kSentinel : u;
        kp[r] = u;
        pos = l;
        hit = ((sc > 0.5f) == l);
    }
    add_counts(pos, hit, cnt);
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

namespace {
struct AucWork {
    uint32_t *kn, *kn_sorted, *kp;
    unsigned long long* cnt;  // [0] members, [1] hits at 0.5, [2] U2
    void* tmp;
    size_t tmp_bytes;
};
AucWork auc_work(Ctx& ctx, long long n) {
    if (n > 0x7fffffffLL) fail(MTK_SHAPE_ERROR, "auc: more than 2^31 rows");
    AucWork w;
    w.tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, w.tmp_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 32,
                                   ctx.stream);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    char* p = static_cast<char*>(ctx.big(al(4 * n) * 3 + al(64) + al(w.tmp_bytes)));
    auto take = [&](size_t b) { char* r = p; p += al(b); return r; };
    w.kn = (uint32_t*)take(4 * n);
    w.kn_sorted = (uint32_t*)take(4 * n);
    w.kp = (uint32_t*)take(4 * n);
    w.cnt = (unsigned long long*)take(64);
    w.tmp = take(w.tmp_bytes);
    MTK_CUDA(cudaMemsetAsync(w.cnt, 0, 64, ctx.stream));
    return w;
}
// keys written: sort the non-member keys (members' sentinels sort last), count
// members against them, read back (synchronizes)
void auc_finish(Ctx& ctx, AucWork& w, const uint8_t* labels, long long n, double* auc, double* acc) {
    cudaStream_t s = ctx.stream;
    MTK_CUDA(cub::DeviceRadixSort::SortKeys(w.tmp, w.tmp_bytes, w.kn, w.kn_sorted, (int)n, 0, 32, s));
    const int sms = device_sm_count(ctx.device);
    const long long want = (n + AUC_THREADS - 1) / AUC_THREADS;
    auc_member_count<<<(unsigned)std::min<long long>(want, 3LL * sms), AUC_THREADS, 0, s>>>(w.kn_sorted, w.kp,
                                                                                          labels, n, w.cnt);
    count_launch();
    unsigned long long* h = static_cast<unsigned long long*>(ctx.pinned_buf(64));
    MTK_CUDA(cudaMemcpyAsync(h, w.cnt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    MTK_CUDA(cudaStreamSynchronize(s));
    const double npos = (double)h[0], nneg = (double)n - npos;
    if (h[0] == 0 || npos == (double)n)
        fail(MTK_VALUE_ERROR, "auc: need at least one member and one non-member");
    if (auc) *auc = (0.5 * (double)h[2]) / (npos * nneg);
    if (acc) *acc = (double)h[1] / (double)n;
}
}  // namespace

void auc_device(Ctx& ctx, const float* scores, const uint8_t* labels, long long n, double* auc,
                double* acc) {
    AucWork w = auc_work(ctx, n);
    auc_keys_kernel<<<nblocks(n, 256), 256, 0, ctx.stream>>>(scores, labels, n, w.kn, w.kp, w.cnt);
    count_launch();
    auc_finish(ctx, w, labels, n, auc, acc);
}

namespace {
std::mutex& att_mutex() {
    static std::mutex m;
    return m;
}
cudaEvent_t& att_last_use(int device) {
    static cudaEvent_t ev[64] = {};
    if (device < 0 || device >= 64) fail(MTK_ERROR, "attack_auc: device index out of range");
    return ev[device];
}
}  // namespace

bool attack_fused_ok(int C, int K, int H, int O) { return C >= 1 && C <= 16 && K == ATT_K && H == ATT_H && O == 2; }

void attack_auc_fused(Ctx& ctx, const float* logits, long long rows, int C, const float* W0, const float* b0,
                      const float* W1, const float* b1, const uint8_t* labels, float* score_out, double* auc,
                      double* acc) {
    if (!attack_fused_ok(C, ATT_K, ATT_H, 2)) fail(MTK_ERROR, "attack_auc: unsupported shape");
    cudaStream_t s = ctx.stream;
    // c_att is one symbol per device, shared by every context on it: the copy
    // of this call must not land while another context's scoring kernel still
    // reads the previous weights (a different stream, so no implicit order).
    // Per device, the stream waits on the event recorded after the last
    // scoring launch, and records its own; the mutex orders the enqueues.
    std::lock_guard<std::mutex> lk(att_mutex());
    cudaEvent_t& last = att_last_use(ctx.device);
    if (last) MTK_CUDA(cudaStreamWaitEvent(s, last, 0));
    else MTK_CUDA(cudaEventCreateWithFlags(&last, cudaEventDisableTiming));
    // the attack model's weights -> constant memory (stream-ordered device copies)
    MTK_CUDA(cudaMemcpyToSymbolAsync(c_att, W0, ATT_K * ATT_H * 4, 0, cudaMemcpyDeviceToDevice, s));
    MTK_CUDA(cudaMemcpyToSymbolAsync(c_att, b0, ATT_H * 4, ATT_K * ATT_H * 4, cudaMemcpyDeviceToDevice, s));
    MTK_CUDA(cudaMemcpyToSymbolAsync(c_att, W1, ATT_H * 2 * 4, (ATT_K * ATT_H + ATT_H) * 4,
                                     cudaMemcpyDeviceToDevice, s));
    MTK_CUDA(cudaMemcpyToSymbolAsync(c_att, b1, 2 * 4, (ATT_K * ATT_H + ATT_H + ATT_H * 2) * 4,
                                     cudaMemcpyDeviceToDevice, s));
    AucWork w = auc_work(ctx, rows);
    attack_score_kernel<16><<<nblocks(rows, 256), 256, 0, s>>>(logits, rows, C, labels, score_out, w.kn, w.kp,
                                                               w.cnt);
    count_launch();
    MTK_CUDA(cudaEventRecord(last, s));
    auc_finish(ctx, w, labels, rows, auc, acc);
}

}  // namespace mtk
