// k_attack.cu -- membership-attack stage: posteriors, top-k features, AUC.
//
// Posteriors follow Tape::softmax (tape.hpp:433-464): max-subtracted exp,
// normalised by the row sum.  Features and AUC have no reference code
// (SURVEY.md section 8(a) row a18); definitions per SURVEY.md Appendix A and
// oracle.c (orc_posterior_features, orc_auc).  These are streaming,
// HBM-bound kernels: one thread per query row, coalesced row-major output.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <cmath>

#include "auc.cuh"
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

// ---- AUC (auc.cuh: exact mid-rank AUC from key histograms, no sort) --------
// per query: the order-preserving key; per block: the key range, member and
// hit-at-0.5 counts (auc.cuh)
__global__ void __launch_bounds__(256) auc_keys_kernel(const float* s, const uint8_t* lab, long long n, auc::Work w) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the scan kernel may launch
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long pos = 0, hit = 0;
    uint32_t kmax = 0, nkmin = 0, u = 0;
    bool l = false;
    auc::zero_next_counters(w);
    if (i < n) {
        u = auc::key_of(s[i]);
        l = lab[i] != 0;
        w.key[i] = u;
        kmax = u;
        nkmin = ~u;
        pos = l;
        hit = ((s[i] > 0.5f) == l);
    }
    if (w.win_on) auc::spec_add(w, u, l, i < n);
    auc::publish_counts(w, kmax, nkmin, pos, hit);
}

// ---- fused attack scoring: posterior softmax -> top-KF sorted features ->
// attack MLP KF -> H (ReLU) -> 2 -> member posterior -> AUC keys, one pass
// over the logits.  Same arithmetic, in the same order, as features_small_kernel,
// small2_forward_kernel and column_kernel (bit-identical scores); each CTA
// stages the attack model's weights in shared memory (warp-uniform reads).
constexpr int ATT_K = 3, ATT_H = 64;
// Two queries per thread: the attack MLP runs on packed fp32x2 (FFMA2 /
// FADD2: the same IEEE operations lane by lane, so the scores stay
// bit-identical to the one-query kernel).  The weights are read straight from
// the bank and staged per CTA, grouped per hidden unit: (W0[0][h], W0[1][h],
// W0[2][h], b0[h]) and (W1[h][0], W1[h][1]) -- one 128-bit and one 64-bit
// broadcast shared load per hidden unit, each weight broadcast into both
// lanes by FFMA2 (R.F32 operand).  No per-call weight upload, no process-wide
// symbol shared between contexts.
// EXACT: C == CC at compile time (the 10-class posteriors), no padding lanes.
static_assert(ATT_K == 3, "the per-hidden-unit record holds three input weights");
struct AttW {
    const float *W0, *b0, *W1, *b1;  // the bank's layer 0 ([ATT_K][ATT_H], [ATT_H]) and 1 ([ATT_H][2], [2])
};

template <int CC, bool EXACT>
__device__ __forceinline__ void top3_of_vals(float (&v)[CC], int C, float (&top)[ATT_K]) {
    float mx = v[0];
#pragma unroll
    for (int j = 1; j < CC; ++j) mx = fmaxf(mx, v[j]);
    float z = 0.f;
#pragma unroll
    for (int j = 0; j < CC; ++j) {
        v[j] = (EXACT || j < C) ? expf(v[j] - mx) : 0.f;
        z += v[j];
    }
    const float inv = 1.f / z;
#pragma unroll
    for (int a = 0; a < ATT_K; ++a) top[a] = -1.f;
#pragma unroll
    for (int j = 0; j < CC; ++j) {
        if (!EXACT && j >= C) break;
        float t = v[j] * inv;
#pragma unroll
        for (int a = 0; a < ATT_K; ++a) {
            const float hi = fmaxf(top[a], t), lo = fminf(top[a], t);
            top[a] = hi;
            t = lo;
        }
    }
}
template <int CC, bool EXACT>
__device__ __forceinline__ void top3_of_row(const float* x, int C, float (&top)[ATT_K]) {
    float v[CC];
#pragma unroll
    for (int j = 0; j < CC; ++j) v[j] = (EXACT || j < C) ? __ldg(x + j) : -INFINITY;
    top3_of_vals<CC, EXACT>(v, C, top);
}

template <int CC, bool EXACT, int QP>  // QP query pairs per thread
__global__ void __launch_bounds__(256) attack_score2_kernel(const float* logits, long long rows, int C,
                                                            const uint8_t* lab, float* score_out, auc::Work w,
                                                            AttW aw) {
    __shared__ float4 sa[ATT_H];  // (W0[0][h], W0[1][h], W0[2][h], b0[h])
    __shared__ float2 sb[ATT_H];  // (W1[h][0], W1[h][1])
    __shared__ float2 sc;         // (b1[0], b1[1])
    if (threadIdx.x < ATT_H) {  // issued before the posterior loads; read after them
        const int h = threadIdx.x;
        sa[h] = make_float4(__ldg(aw.W0 + h), __ldg(aw.W0 + ATT_H + h), __ldg(aw.W0 + 2 * ATT_H + h),
                            __ldg(aw.b0 + h));
        sb[h] = make_float2(__ldg(aw.W1 + 2 * h), __ldg(aw.W1 + 2 * h + 1));
        if (h == 0) sc = make_float2(__ldg(aw.b1), __ldg(aw.b1 + 1));
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the scan kernel may launch
    const long long r0 = 2LL * QP * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
    const bool vec = (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
    float2 t[QP][ATT_K];
#pragma unroll
    for (int q = 0; q < QP; ++q) {
        float ta[ATT_K], tb[ATT_K];
        const long long ra = r0 + 2 * q;
        if (CC == 10 && EXACT && vec && ra + 1 < rows) {
            // the pair's 20 posteriors are 80 contiguous, 16-B aligned bytes:
            // five 128-bit loads instead of twenty scalar ones
            const float4* p4 = reinterpret_cast<const float4*>(logits + ra * CC);
            const float4 a0 = __ldg(p4), a1 = __ldg(p4 + 1), a2 = __ldg(p4 + 2), a3 = __ldg(p4 + 3),
                         a4 = __ldg(p4 + 4);
            float va[CC] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y};
            float vb[CC] = {a2.z, a2.w, a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, a4.z, a4.w};
            top3_of_vals<CC, EXACT>(va, C, ta);
            top3_of_vals<CC, EXACT>(vb, C, tb);
#pragma unroll
            for (int a = 0; a < ATT_K; ++a) t[q][a] = make_float2(ta[a], tb[a]);
            continue;
        }
        if (ra < rows) top3_of_row<CC, EXACT>(logits + ra * C, C, ta);
        else ta[0] = ta[1] = ta[2] = 0.f;
        if (ra + 1 < rows) top3_of_row<CC, EXACT>(logits + (ra + 1) * C, C, tb);
        else tb[0] = tb[1] = tb[2] = 0.f;
#pragma unroll
        for (int a = 0; a < ATT_K; ++a) t[q][a] = make_float2(ta[a], tb[a]);
    }
    __syncthreads();  // the staged weights
    float2 o0[QP], o1[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) o0[q] = o1[q] = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int h = 0; h < ATT_H; ++h) {
        const float4 a = sa[h];
        const float2 v = sb[h];
        const float2 w0 = make_float2(a.x, a.x), w1 = make_float2(a.y, a.y), w2 = make_float2(a.z, a.z),
                     bb = make_float2(a.w, a.w);
        const float2 v0 = make_float2(v.x, v.x), v1 = make_float2(v.y, v.y);
#pragma unroll
        for (int q = 0; q < QP; ++q) {
            float2 acc = __ffma2_rn(t[q][0], w0, make_float2(0.f, 0.f));
            acc = __ffma2_rn(t[q][1], w1, acc);
            acc = __ffma2_rn(t[q][2], w2, acc);
            float2 hv = __fadd2_rn(acc, bb);
            hv.x = hv.x > 0.f ? hv.x : 0.f;
            hv.y = hv.y > 0.f ? hv.y : 0.f;
            o0[q] = __ffma2_rn(hv, v0, o0[q]);
            o1[q] = __ffma2_rn(hv, v1, o1[q]);
        }
    }
    unsigned long long pos = 0, hit = 0;
    uint32_t kmax = 0, nkmin = 0;
    auc::zero_next_counters(w);
#pragma unroll
    for (int q = 0; q < 2 * QP; ++q) {
        const long long r = r0 + q;
        const float2 a = __fadd2_rn(o0[q / 2], make_float2(sc.x, sc.x)),
                     b = __fadd2_rn(o1[q / 2], make_float2(sc.y, sc.y));
        const float p0 = (q & 1) ? a.y : a.x, p1 = (q & 1) ? b.y : b.x;
        uint32_t u = 0;
        bool l = false;
        if (r < rows) {  // member posterior: column_kernel's softmax column 1
            const float m2 = fmaxf(p0, p1);
            const float z2 = expf(p0 - m2) + expf(p1 - m2);
            const float sc = expf(p1 - m2) / z2;
            if (score_out) score_out[r] = sc;
            u = auc::key_of(sc);
            l = lab[r] != 0;
            w.key[r] = u;
            kmax = max(kmax, u);
            nkmin = max(nkmin, ~u);
            pos += l;
            hit += ((sc > 0.5f) == l);
        }
        if (w.win_on) auc::spec_add(w, u, l, r < rows);
    }
    auc::publish_counts(w, kmax, nkmin, pos, hit);
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
int auc_fast_blocks(Ctx& ctx) { return 2 * device_sm_count(ctx.device); }
// grow-only workspace from ctx.big: keys, histograms, bucket slots, the
// scattered mixed buckets, the large-bucket histograms, counters
auc::Work auc_work(Ctx& ctx, long long n) {
    if (n > 0x7fffffffLL) fail(MTK_SHAPE_ERROR, "auc: more than 2^31 rows");
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t hb = 2 * (size_t)auc::kBuckets * 4;
    char* p = static_cast<char*>(ctx.big(al(4 * n) * 2 + al(4 * auc::kBuckets) +
                                         al(16 * auc::kBuckets) + al(16 * auc::kScanBlocks) +
                                         al(3 * 8 * (size_t)auc_fast_blocks(ctx)) +
                                         al((size_t)(n / auc::kSmallMax + 1) * auc::kL2Blocks * 4)));
    auto take = [&](size_t b) { char* r = p; p += al(b); return r; };
    auc::Work w;
    w.key = (uint32_t*)take(4 * n);
    w.packed = (uint32_t*)take(4 * n);
    w.cursor = (uint32_t*)take(4 * auc::kBuckets);
    w.mixed = (uint4*)take(16 * auc::kBuckets);
    w.totals = (uint4*)take(16 * auc::kScanBlocks);
    w.big = nullptr;
    // at most n / kSmallMax buckets can be large: one level-2 slot each
    const size_t slots = (size_t)(n / auc::kSmallMax + 1);
    w.l2tot = (uint32_t*)take(slots * auc::kL2Blocks * 4);
    w.fpart = (unsigned long long*)take(3 * 8 * (size_t)auc_fast_blocks(ctx));
    // zero-invariant arena: the full-resolution bins, the block counter, the level-2 histograms
    // (the top-16 histogram too: auc_scan_kernel leaves it zeroed)
    const size_t fb = (size_t)8 << auc::kFastBits;
    char* ar = reinterpret_cast<char*>(ctx.auc_l2(fb + 512 + al(hb) + slots * 2 * auc::kBuckets * 4));
    w.fhist = reinterpret_cast<unsigned long long*>(ar);
    w.done = reinterpret_cast<unsigned int*>(ar + fb);
    // two counter blocks of 16 (counters, key range, window flag), used by
    // alternate calls; each call's first kernel zeroes the other one
    unsigned long long* cb = reinterpret_cast<unsigned long long*>(ar + fb + 256);
    w.cnt = cb + 16 * ctx.auc_parity;
    w.cnt_next = cb + 16 * (1 - ctx.auc_parity);
    ctx.auc_parity ^= 1;
    w.mm = reinterpret_cast<uint32_t*>(w.cnt + 8);
    // the speculative window: the previous call's key range (auc_finish)
    w.win_on = ctx.auc_win_valid ? 1 : 0;
    w.win_lo = ctx.auc_win_lo;
    if (!ctx.auc_mail) {
        void* hp = nullptr;
        MTK_CUDA(cudaHostAlloc(&hp, 16 * sizeof(unsigned long long), cudaHostAllocMapped));
        std::memset(hp, 0, 16 * sizeof(unsigned long long));
        ctx.auc_mail = static_cast<unsigned long long*>(hp);
        void* dp = nullptr;
        MTK_CUDA(cudaHostGetDevicePointer(&dp, hp, 0));
        ctx.auc_mail_dev = static_cast<unsigned long long*>(dp);
    }
    w.mail = ctx.auc_mail_dev;
    w.seq = ++ctx.auc_seq;
    w.flags = ctx.d_flags;
    w.hist = reinterpret_cast<uint32_t*>(ar + fb + 512);
    w.l2 = reinterpret_cast<uint32_t*>(ar + fb + 512 + al(hb));
    return w;
}
// keys and key range written: the histogram pass, then the full-resolution
// scan or (wide key ranges) the cross-bucket pass, the scatter of the mixed
// buckets and the within-bucket passes -- the kernels of the path not taken
// exit at once (device-side decision, no host round trip); read back (synchronizes)
// the general path's kernels (each exits at once when the full-resolution path applies)
void auc_general(Ctx& ctx, auc::Work& w, const uint8_t* labels, long long n) {
    cudaStream_t s = ctx.stream;
    const int sms = device_sm_count(ctx.device);
    auc::auc_scan_totals_kernel<<<auc::kScanBlocks, auc::kThreads, 0, s>>>(w);
    auc::auc_scan_kernel<<<auc::kScanBlocks, auc::kThreads, 0, s>>>(w);
    auc::auc_scatter_kernel<<<(unsigned)std::min<long long>(nblocks(n, 256), 8LL * sms), 256, 0, s>>>(w, labels, n);
    ensure_smem_attr(reinterpret_cast<const void*>(auc::auc_bucket_kernel), auc::kBucketSmem);
    auc::auc_bucket_kernel<<<8 * sms, auc::kBucketThreads, auc::kBucketSmem, s>>>(w);
    auc::auc_l2_totals_kernel<<<2 * sms, auc::kThreads, 0, s>>>(w);
    auc::auc_l2_kernel<<<2 * sms, auc::kThreads, 0, s>>>(w);
    for (int i = 0; i < 6; ++i) count_launch();
}
// keys and key range written: the histogram pass, then the full-resolution
// scan or (wide key ranges) the general path.  Which one applies is known on
// the device; the host predicts it from the context's previous call and
// launches only that path's kernels -- on a misprediction to "full
// resolution" the general kernels follow the read-back (one more round trip;
// the result does not depend on the prediction).  Reads back (synchronizes).
// flags_clear (optional): set when the result came through the mailbox with
// the context's device flags clear -- the caller's check_flags round trip is
// then redundant (every kernel of the call ran before the post)
void auc_finish(Ctx& ctx, auc::Work& w, const uint8_t* labels, long long n, double* auc, double* acc,
                bool* flags_clear = nullptr) {
    cudaStream_t s = ctx.stream;
    const int sms = device_sm_count(ctx.device);
    const unsigned hist_grid = (unsigned)std::min<long long>(nblocks(n, 256), 8LL * sms);
    auto readback = [&](unsigned long long* h) {
        MTK_CUDA(cudaMemcpyAsync(h, w.cnt, 10 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));  // counters, mm[0..2]
        MTK_CUDA(cudaStreamSynchronize(s));
    };
    // the first read-back of a call: spin on the mailbox the fast scan kernel
    // posts (counters + sequence number) once it is done, polling the stream
    // now and then so an error or a missing post falls back to the copy +
    // synchronize (either way the scan has finished when this returns)
    auto mailbox = [&](unsigned long long* h) -> bool {
        volatile unsigned long long* m = ctx.auc_mail;
        for (unsigned spins = 1;; ++spins) {
            if (m[15] == w.seq) {
                std::atomic_thread_fence(std::memory_order_acquire);
                for (int i = 0; i < 12; ++i) h[i] = m[i];
                return true;
            }
            if ((spins & 1023) == 0 && cudaStreamQuery(s) != cudaErrorNotReady) {
                if (m[15] == w.seq) continue;  // posted just now
                readback(h);                   // (raises a pending error)
                return false;
            }
        }
    };
    unsigned long long* h = static_cast<unsigned long long*>(ctx.pinned_buf(128));
    const uint32_t* mm = reinterpret_cast<const uint32_t*>(h + 8);
    bool spec_ok = false;
    if (w.win_on) {  // the keys were binned speculatively in the window
        // a programmatic dependent of the scoring / keys kernel just launched
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)auc_fast_blocks(ctx));
        cfg.blockDim = dim3(auc::kFastScanThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = umma::pdl_enabled() ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        MTK_CUDA(cudaLaunchKernelEx(&cfg, auc::auc_fast_scan_kernel, w));
        count_launch();
        const bool mailed = mailbox(h);
        spec_ok = mm[2] == 0;
        if (flags_clear) *flags_clear = mailed && spec_ok && h[11] == 0;
        w.win_on = 0;  // a re-run bins from the keys
        w.mail = nullptr;
    }
    if (!spec_ok) {
        auc::auc_hist_kernel<<<hist_grid, 256, 0, s>>>(w, labels, n);
        auc::auc_fast_scan_kernel<<<auc_fast_blocks(ctx), auc::kFastScanThreads, 0, s>>>(w);
        count_launch();
        count_launch();
        if (!ctx.auc_fast_hint) auc_general(ctx, w, labels, n);
        readback(h);
        const bool fast = mm[0] - ~mm[1] < (1u << auc::kFastBits);
        if (ctx.auc_fast_hint && !fast) {
            auc_general(ctx, w, labels, n);
            readback(h);
        }
        ctx.auc_fast_hint = fast;
    }
    // the next call's window: this key range, centred in 2^kFastBits bins
    const uint32_t kmin = ~mm[1], kmax = mm[0], range = kmax - kmin;
    const uint32_t span = (1u << auc::kFastBits) - 1u;
    ctx.auc_win_valid = range < span;
    if (ctx.auc_win_valid) {
        const uint32_t slack = (span - range) / 2;
        uint32_t lo = kmin >= slack ? kmin - slack : 0u;
        if (lo > 0xFFFFFFFFu - span) lo = 0xFFFFFFFFu - span;  // no wrap past the top key
        ctx.auc_win_lo = lo;
    }
    const double npos = (double)h[0], nneg = (double)n - npos;
    if (h[0] == 0 || npos == (double)n)
        fail(MTK_VALUE_ERROR, "auc: need at least one member and one non-member");
    if (auc) *auc = (0.5 * (double)h[2]) / (npos * nneg);
    if (acc) *acc = (double)h[1] / (double)n;
}
}  // namespace

void auc_device(Ctx& ctx, const float* scores, const uint8_t* labels, long long n, double* auc,
                double* acc, bool* flags_clear) {
    auc::Work w = auc_work(ctx, n);
    auc_keys_kernel<<<nblocks(n, 256), 256, 0, ctx.stream>>>(scores, labels, n, w);
    count_launch();
    auc_finish(ctx, w, labels, n, auc, acc, flags_clear);
}


bool attack_fused_ok(int C, int K, int H, int O) { return C >= 1 && C <= 16 && K == ATT_K && H == ATT_H && O == 2; }

void attack_auc_fused(Ctx& ctx, const float* logits, long long rows, int C, const float* W0, const float* b0,
                      const float* W1, const float* b1, const uint8_t* labels, float* score_out, double* auc,
                      double* acc, bool* flags_clear) {
    if (!attack_fused_ok(C, ATT_K, ATT_H, 2)) fail(MTK_ERROR, "attack_auc: unsupported shape");
    cudaStream_t s = ctx.stream;
    auc::Work w = auc_work(ctx, rows);
    const AttW aw{W0, b0, W1, b1};
    constexpr int QP = 1;  // one query pair per thread (QP = 2: fewer instructions, but under one wave of threads -- not faster)
    const long long thr = (rows + 2 * QP - 1) / (2 * QP);
    if (C == 10)
        attack_score2_kernel<10, true, QP><<<nblocks(thr, 256), 256, 0, s>>>(logits, rows, C, labels, score_out, w,
                                                                             aw);
    else
        attack_score2_kernel<16, false, QP><<<nblocks(thr, 256), 256, 0, s>>>(logits, rows, C, labels, score_out, w,
                                                                              aw);
    count_launch();
    auc_finish(ctx, w, labels, rows, auc, acc, flags_clear);
}

}  // namespace mtk
