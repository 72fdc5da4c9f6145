// auc.cuh -- exact mid-rank (Mann-Whitney) AUC without sorting the scores
// (AUC = (R_pos - npos (npos + 1) / 2) / (npos nneg),
// mid-ranks for ties).  With U2 = sum over members of 2 #{non-members below}
// + #{non-members equal}, AUC = (U2 / 2) / (npos nneg), all in exact integers.
//
// The scores are keyed by an order-preserving float -> uint32 map and the
// rank sums come from key histograms instead of a sort.  The kernel that
// produces the scores writes every query's key and the block-reduced key
// range [kmin, kmax].
//
// Full-resolution path (kmax - kmin < 2^kFastBits: concentrated scores, the
// attack stage's case -- bench data: a 2^20.1-key range):
//   F1. auc_hist_kernel: per query one 64-bit atomic (1 << 32 | non-member)
//       into bin key - kmin of a zero-invariant [2^kFastBits] arena (same-bin
//       lanes of a warp aggregated by match.any);
//   F2. auc_fast_scan_kernel: in bin (= key) order, every member adds
//       2 #{non-members in lower bins} + #{non-members in its bin}: per block
//       rounds of 1024 bins (block scan of the non-member counts), the
//       blocks' partials combined in block order by the last block to finish;
//       the bins are reset on the way.  Two launches after the scores.
// General path (wider ranges), on the top 16 bits of the key:
//   1. auc_hist_kernel: a per-class histogram of the key's top 16 bits
//      (warp-aggregated integer atomics);
//   2. auc_scan_totals_kernel + auc_scan_kernel (64 blocks each): in bucket
//      order, every member contributes 2 #{non-members in lower buckets} --
//      summed exactly -- and the buckets holding both classes ("mixed") get
//      a slot in a compacted, bucket-ordered array;
//   3. auc_scatter_kernel: the queries of small mixed buckets (<= 8192) go
//      to their bucket's slot as (low 16 key bits << 1 | class); those of
//      large ones into per-bucket class histograms of the low 16 bits
//      (level 2, global integer atomics over 65536 bins);
//   4. auc_bucket_kernel, one CTA per mixed bucket: within the bucket the
//      members' 2 #{below} + #{equal} over the low 16 bits -- a shared-memory
//      bitonic sort and a scan for small buckets, a scan of the level-2
//      histograms for large ones.
// Integer sums are order-independent, so the AUC is deterministic and
// bit-identical to the sort-based evaluation (and to oracle.c orc_auc's
// ranks); no library sort on the path.
#pragma once

#include <cstdint>

namespace mtk {
namespace auc {

constexpr int kFastBits = 23;  // full-resolution key histogram up to a 2^23-key range (64 MB arena)
constexpr int kBuckets = 65536;
constexpr int kSmallMax = 2048;      // bitonic-sort path up to this many queries per bucket
constexpr int kBucketThreads = 256;  // small-bucket kernel: one CTA per bucket, 8 per SM
constexpr int kThreads = 1024;       // scan / bucket kernels
constexpr uint32_t kNotMixed = 0xFFFFFFFFu;
constexpr uint32_t kLargeFlag = 0x80000000u;  // cursor / mixed-entry flag: level-2 histogram slot

// order-preserving map float -> uint32 (ascending), -0.0 == +0.0
__device__ __forceinline__ uint32_t key_of(float v) {
    if (v == 0.f) v = 0.f;
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// one query's key into the class histogram of the top 16 bits; all 32 lanes
// of the warp must call it (valid = false for lanes without a query)
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t key, bool member, bool valid) {
    const uint32_t tag = valid ? ((key >> 16) | (member ? 0x10000u : 0u)) : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, tag);
    const int lane = threadIdx.x & 31;
    if (valid && lane == __ffs(peers) - 1) atomicAdd(&hist[tag], (uint32_t)__popc(peers));
}

// block-wide exclusive scan of one u32 per thread (any multiple of 32 threads); returns
// the thread's exclusive prefix, *total the block total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0u;
        uint32_t t = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        sh[lane] = t - s;  // exclusive warp offsets
        if (lane == 31) sh[32] = t;
    }
    __syncthreads();
    const uint32_t r = sh[w] + x - v;
    *total = sh[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    __syncthreads();
    return t;  // valid on thread 0
}

struct Work {
    uint32_t* key;        // [n]
    uint32_t* hist;       // [2][kBuckets] class 0 (non-members), class 1 (members); zero on entry
    uint32_t* cursor;     // [kBuckets]
    uint32_t* packed;     // [n]
    uint4* mixed;         // [kBuckets] (bucket, offset, size, non-members)
    uint4* totals;        // [kBuckets / kThreads] per-block totals of the scan
    uint32_t* big;        // (unused)
    uint32_t* l2;         // [large slots][2][kBuckets] level-2 class histograms; zero on entry and exit
    uint32_t* l2tot;      // [large slots][kBuckets / kThreads] block totals of the non-member counts
    unsigned long long* cnt;  // [0] members, [1] hits at 0.5, [2] U2, [3] mixed, [4] large buckets
    uint32_t* mm;             // [0] max key, [1] max ~key (= ~min key), [2] a key outside the window; zero on entry
    unsigned long long* cnt_next;  // the next call's counters (ping-pong): zeroed by this call's first kernel
    uint32_t win_lo;          // speculative window [win_lo, win_lo + 2^kFastBits) of full-resolution bins
    int win_on;               // 1: the score kernel adds every in-window key to fhist[key - win_lo]
    unsigned long long* fhist;  // [2^kFastBits] (queries << 32 | non-members) per key; zero on entry and exit
    unsigned long long* fpart;  // [blocks][3] per-block (non-members, members, U2) of auc_fast_scan_kernel
    unsigned int* done;         // blocks finished in auc_fast_scan_kernel; zero on entry and exit
    unsigned long long* mail;   // mapped host mailbox (or null): [0..2] counters, [8..9] key range
                                // words, [10] 1 = U2 complete, [11] the context's device flags,
                                // [15] sequence number (written last)
    unsigned long long seq;
    const int* flags;           // the context's device flags (posted with the counters)
};

// the counters (and whether U2 is complete) to the host mailbox, then the
// sequence number (one thread; after the counters are final)
__device__ __forceinline__ void post_mail(const Work& w, bool complete) {
    if (!w.mail) return;
    __threadfence();
    for (int i = 0; i < 3; ++i) w.mail[i] = __ldcg(w.cnt + i);
    w.mail[8] = __ldcg(w.cnt + 8);
    w.mail[9] = __ldcg(w.cnt + 9);
    w.mail[10] = complete ? 1ull : 0ull;
    w.mail[11] = w.flags ? (unsigned long long)(unsigned)__ldcg(w.flags) : 0ull;
    __threadfence_system();
    w.mail[15] = w.seq;
}

// the full-resolution path applies (the key range is known once the scores are)
__device__ __forceinline__ bool fast_path(const Work& w) {
    return w.win_on ? w.mm[2] == 0 : w.mm[0] - ~w.mm[1] < (1u << kFastBits);
}

// Speculative full-resolution binning inside the kernel that produces the
// keys: the window is the previous call's key range, centred in 2^kFastBits
// bins (host side).  Every in-window key is added to its bin right away; a
// key outside sets mm[2], and the host re-runs the binning from the keys
// (the bins written are cleared by auc_fast_scan_kernel).  All 32 lanes of
// the warp call it.
__device__ __forceinline__ void spec_add(const Work& w, uint32_t key, bool member, bool valid) {
    const uint32_t b = key - w.win_lo;
    const bool in = valid && b < (1u << kFastBits);
    const uint32_t tag = in ? b : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, tag);
    const unsigned nmp = __ballot_sync(0xffffffffu, in && !member) & peers;
    const int lane = threadIdx.x & 31;
    if (in && lane == __ffs(peers) - 1)
        atomicAdd(&w.fhist[b], ((unsigned long long)__popc(peers) << 32) | (unsigned long long)__popc(nmp));
    if (__any_sync(0xffffffffu, valid && !in) && lane == 0) atomicOr(&w.mm[2], 1u);
}
// the first kernel of a call zeroes the next call's counters (this call's were
// zeroed by the previous call, whose host read-back has completed)
__device__ __forceinline__ void zero_next_counters(const Work& w) {
    if (blockIdx.x == 0 && threadIdx.x < 16) w.cnt_next[threadIdx.x] = 0ull;
}

// block-reduced key range, member and hit-at-0.5 counts -> the global counters
// (integer atomics: exact and order-independent); every thread of the block calls it
__device__ __forceinline__ void publish_counts(const Work& w, uint32_t kmax, uint32_t nkmin,
                                               unsigned long long pos, unsigned long long hit) {
    __shared__ uint32_t sa[32], sb[32];
    __shared__ unsigned long long sp[32], sq[32];
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    nkmin = __reduce_max_sync(0xffffffffu, nkmin);
    for (int o = 16; o > 0; o >>= 1) {
        pos += __shfl_down_sync(0xffffffffu, pos, o);
        hit += __shfl_down_sync(0xffffffffu, hit, o);
    }
    const int wi = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sa[wi] = kmax;
        sb[wi] = nkmin;
        sp[wi] = pos;
        sq[wi] = hit;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0, b = 0;
        unsigned long long c = 0, d = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            a = max(a, sa[i]);
            b = max(b, sb[i]);
            c += sp[i];
            d += sq[i];
        }
        if (a) atomicMax(&w.mm[0], a);
        if (b) atomicMax(&w.mm[1], b);
        if (c) atomicAdd(&w.cnt[0], c);
        if (d) atomicAdd(&w.cnt[1], d);
    }
}

// F1 / 1: per query, the full-resolution bin (fast path) or the top-16-bit
// class histogram (general path).  Grid-stride over whole warps.
__global__ void __launch_bounds__(256) auc_hist_kernel(Work w, const uint8_t* lab, long long n) {
    const bool fast = fast_path(w);
    const uint32_t kmin = ~w.mm[1];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const long long i = i0 + lane;
        const bool valid = i < n;
        const uint32_t k = valid ? w.key[i] : 0u;
        const bool nm = valid && lab[i] == 0;
        if (fast) {
            const uint32_t b = valid ? k - kmin : 0xFFFFFFFFu;
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            const unsigned nmp = __ballot_sync(0xffffffffu, nm) & peers;
            if (valid && lane == __ffs(peers) - 1)
                atomicAdd(&w.fhist[b], ((unsigned long long)__popc(peers) << 32) | (unsigned long long)__popc(nmp));
        } else {
            hist_add(w.hist, k, valid && !nm, valid);
        }
    }
}

// F2: U2 over the full-resolution bins [0, kmax - kmin].  Launched right
// behind the scoring (or keys) kernel as a programmatic dependent: its CTAs
// take the SMs that kernel's last wave frees, and wait here for its results.
constexpr int kFastScanThreads = 512;
__global__ void __launch_bounds__(kFastScanThreads) auc_fast_scan_kernel(Work w) {
    __shared__ uint32_t sh[33];
    __shared__ unsigned long long shl[32];
    __shared__ bool last;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // (a no-op without the PDL launch attribute)
    const uint32_t kmin = ~w.mm[1], kmax = w.mm[0];
    if (blockIdx.x == 0 && threadIdx.x == 0 && ((w.win_on && w.mm[2]) || !fast_path(w)))
        post_mail(w, false);  // the host continues (re-binning / the general path)
    if (w.win_on && w.mm[2]) {  // a key fell outside the window: clear the in-window bins written
        const uint32_t top = w.win_lo + ((1u << kFastBits) - 1u);
        const long long lo = (long long)(max(kmin, w.win_lo) - w.win_lo);
        const long long hi = (long long)(min(kmax, top) - w.win_lo);
        if (kmax < w.win_lo || kmin > top) return;
        for (long long b = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; b <= hi;
             b += (long long)gridDim.x * blockDim.x)
            if (w.fhist[b]) w.fhist[b] = 0ull;
        return;
    }
    if (!fast_path(w)) return;
    // bins [bin0, bin0 + nb) of fhist hold keys kmin .. kmax (bin0 aligned
    // down to 8 bins in the window: the bins below kmin are empty)
    const long long bin0 = w.win_on ? (long long)((kmin - w.win_lo) & ~7u) : 0;
    const long long nb = (w.win_on ? (long long)(kmax - w.win_lo) : (long long)(kmax - kmin)) - bin0 + 1;
    // blocks own ranges of whole 8-bin groups; a thread takes 8 consecutive
    // bins per round (four 16-B loads in flight), one block scan per round
    constexpr int kPer = 8, kRound = kPer * kFastScanThreads;
    const long long groups = (nb + kPer - 1) / kPer;
    const long long gper = (groups + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * gper * kPer, b1 = min(nb, b0 + gper * kPer);
    unsigned long long* fh = w.fhist + bin0;
    uint32_t carry = 0;  // non-members in this block's bins before the round
    unsigned long long u2 = 0, pos = 0;
    for (long long base = b0; base < b1; base += kRound) {  // block-uniform trip count
        const long long t0 = base + (long long)threadIdx.x * kPer;
        unsigned long long v[kPer];
        if (t0 + kPer <= b1) {
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(fh + t0);
#pragma unroll
            for (int j = 0; j < kPer / 2; ++j) {
                const ulonglong2 x = src[j];
                v[2 * j] = x.x;
                v[2 * j + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kPer; ++j) v[j] = t0 + j < b1 ? fh[t0 + j] : 0ull;
        }
        uint32_t nsum = 0;
        unsigned long long any = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            nsum += (uint32_t)v[j];
            any |= v[j];
        }
        uint32_t tot;
        uint32_t below = carry + block_excl_scan(nsum, sh, &tot);
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t T = (uint32_t)(v[j] >> 32), N = (uint32_t)v[j], P = T - N;
            u2 += (unsigned long long)P * (2ull * below + N);
            pos += P;
            below += N;
        }
        if (any) {  // zero-invariant arena
            if (t0 + kPer <= b1) {
                ulonglong2* dst = reinterpret_cast<ulonglong2*>(fh + t0);
#pragma unroll
                for (int j = 0; j < kPer / 2; ++j) dst[j] = make_ulonglong2(0ull, 0ull);
            } else {
                for (int j = 0; j < kPer && t0 + j < b1; ++j) fh[t0 + j] = 0ull;
            }
        }
        carry += tot;
    }
    u2 = block_sum_u64(u2, shl);
    pos = block_sum_u64(pos, shl);
    if (threadIdx.x == 0) {
        w.fpart[3 * blockIdx.x] = carry;
        w.fpart[3 * blockIdx.x + 1] = pos;
        w.fpart[3 * blockIdx.x + 2] = u2;
        __threadfence();
        last = atomicAdd(w.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {  // combine in block order: + 2 #{non-members in earlier blocks} per member (one block per thread)
        __threadfence();
        unsigned long long t = 0, carry_n = 0;
        for (unsigned k0 = 0; k0 < gridDim.x; k0 += kFastScanThreads) {
            const unsigned k = k0 + threadIdx.x;
            const bool in = k < gridDim.x;
            const uint32_t nk = in ? (uint32_t)__ldcg(w.fpart + 3 * k) : 0u;
            const unsigned long long pk = in ? __ldcg(w.fpart + 3 * k + 1) : 0ull;
            const unsigned long long uk = in ? __ldcg(w.fpart + 3 * k + 2) : 0ull;
            uint32_t tot;
            const unsigned long long before = carry_n + block_excl_scan(nk, sh, &tot);
            t += uk + 2ull * before * pk;
            carry_n += tot;
        }
        t = block_sum_u64(t, shl);
        if (threadIdx.x == 0) {
            atomicAdd(&w.cnt[2], t);
            *w.done = 0;
            post_mail(w, true);
        }
    }
}

// 2. bucket order in two fully parallel passes over kScanBlocks blocks of
// kThreads buckets (one bucket per thread, coalesced):
//   a. per block: non-members, mixed buckets, mixed-bucket queries (totals)
//   b. per block: its offsets = the totals of the blocks before it (each
//      block sums them itself), then per bucket: the exact cross-bucket U2
//      part (every member: 2 #{non-members in lower buckets}), the mixed
//      bucket's slot in the compacted array, and the histogram reset
constexpr int kScanBlocks = kBuckets / kThreads;  // 64
__device__ __forceinline__ void load_bucket(const uint32_t* hist, int b, uint32_t& N, uint32_t& P) {
    N = hist[b];
    P = hist[kBuckets + b];
}
__global__ void __launch_bounds__(kThreads) auc_scan_totals_kernel(Work w) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    __shared__ uint32_t sh[33];
    const int b = blockIdx.x * kThreads + threadIdx.x;
    uint32_t N, P;
    load_bucket(w.hist, b, N, P);
    const bool mixed = N && P, large = mixed && N + P > (uint32_t)kSmallMax;
    uint32_t t0, t1, t2, t3;
    block_excl_scan(N, sh, &t0);
    block_excl_scan(mixed ? 1u : 0u, sh, &t1);
    block_excl_scan(mixed && !large ? N + P : 0u, sh, &t2);
    block_excl_scan(large ? 1u : 0u, sh, &t3);
    if (threadIdx.x == 0) w.totals[blockIdx.x] = make_uint4(t0, t1, t2, t3);
}
__global__ void __launch_bounds__(kThreads) auc_scan_kernel(Work w) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    __shared__ uint32_t sh[33];
    __shared__ unsigned long long shl[32];
    __shared__ uint32_t base[4];
    if (threadIdx.x < 4) {
        uint32_t a = 0;
        for (int k = 0; k < (int)blockIdx.x; ++k) {
            const uint4 t = w.totals[k];
            a += threadIdx.x == 0 ? t.x : threadIdx.x == 1 ? t.y : threadIdx.x == 2 ? t.z : t.w;
        }
        base[threadIdx.x] = a;
    }
    const int b = blockIdx.x * kThreads + threadIdx.x;
    uint32_t N, P;
    load_bucket(w.hist, b, N, P);
    const bool mixed = N && P, large = mixed && N + P > (uint32_t)kSmallMax;
    uint32_t tot;
    const uint32_t eN = block_excl_scan(N, sh, &tot);
    const uint32_t eM = block_excl_scan(mixed ? 1u : 0u, sh, &tot);
    const uint32_t mtot = tot;
    const uint32_t eS = block_excl_scan(mixed && !large ? N + P : 0u, sh, &tot);  // (syncs: base visible)
    const uint32_t eL = block_excl_scan(large ? 1u : 0u, sh, &tot);
    const uint32_t ltot = tot;
    const uint32_t below = base[0] + eN;
    unsigned long long cross = (unsigned long long)P * (2ull * below);
    if (large) {  // level-2 class histograms of the low key bits, slot L
        const uint32_t L = base[3] + eL;
        w.mixed[base[1] + eM] = make_uint4((uint32_t)b | kLargeFlag, L, N + P, N);
        w.cursor[b] = kLargeFlag | L;
    } else if (mixed) {  // packed slot for the shared-memory sort
        const uint32_t off = base[2] + eS;
        w.mixed[base[1] + eM] = make_uint4((uint32_t)b, off, N + P, N);
        w.cursor[b] = off;
    } else {
        w.cursor[b] = kNotMixed;
    }
    w.hist[b] = 0;  // clean for the next call
    w.hist[kBuckets + b] = 0;
    cross = block_sum_u64(cross, shl);
    if (threadIdx.x == 0) {
        if (cross) atomicAdd(&w.cnt[2], cross);
        if (blockIdx.x == gridDim.x - 1) {
            w.cnt[3] = base[1] + mtot;
            w.cnt[4] = base[3] + ltot;
        }
    }
}

// 3. the queries of mixed buckets into their bucket's slot (order inside a
// bucket is immaterial: the bucket kernel sorts / counts it)
__global__ void auc_scatter_kernel(Work w, const uint8_t* lab, long long n) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    for (long long i0 = blockIdx.x * (long long)blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        const bool valid = i < n;
        const uint32_t k = valid ? w.key[i] : 0u;
        const uint32_t b = k >> 16;
        const uint32_t cur = valid ? w.cursor[b] : kNotMixed;
        if (cur != kNotMixed && (cur & kLargeFlag)) {  // large bucket: level-2 histogram
            const uint32_t L = cur & ~kLargeFlag;
            atomicAdd(&w.l2[((size_t)L * 2 + (lab[i] ? 1u : 0u)) * kBuckets + (k & 0xFFFFu)], 1u);
        }
        const bool mixed = cur != kNotMixed && !(cur & kLargeFlag);
        const uint32_t tag = mixed ? b : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, tag);
        const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (mixed && lane == leader) base = atomicAdd(&w.cursor[b], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (mixed) {
            const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            w.packed[base + rank] = ((k & 0xFFFFu) << 1) | (lab[i] ? 1u : 0u);
        }
    }
}

// 4. within-bucket ranks of the members against the non-members
//    small (<= kSmallMax queries): bitonic sort in shared memory + scan (here);
//    large: a grid-wide scan of the level-2 class histograms the scatter pass
//    built (auc_l2_totals_kernel, auc_l2_kernel: blocks of 1024 bins).
constexpr int kBucketSmem = 2 * kSmallMax * 4;  // the sorted bucket + its prefix counts
__global__ void __launch_bounds__(kBucketThreads) auc_bucket_kernel(Work w) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    extern __shared__ uint32_t dsm[];
    uint32_t* buf = dsm;
    uint32_t* pre = dsm + kSmallMax;
    __shared__ uint32_t sh[33];
    __shared__ unsigned long long shl[32];
    const uint32_t nmixed = (uint32_t)w.cnt[3];
    unsigned long long acc = 0;
    for (uint32_t t = blockIdx.x; t < nmixed; t += gridDim.x) {
        const uint4 mb = w.mixed[t];
        const uint32_t off = mb.y, s = mb.z;
        const uint32_t* src = w.packed + off;
        if (!(mb.x & kLargeFlag)) {
            uint32_t P = 32;
            while (P < s) P <<= 1;
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) buf[i] = i < s ? src[i] : 0xFFFFFFFFu;
            __syncthreads();
            // bitonic sort, ascending: (value, class 0 before class 1)
            for (uint32_t k = 2; k <= P; k <<= 1) {
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                        const uint32_t l = i ^ j;
                        if (l > i) {
                            const uint32_t a = buf[i], c = buf[l];
                            const bool up = (i & k) == 0;
                            if ((a > c) == up) {
                                buf[i] = c;
                                buf[l] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            // prefix count of non-members, P / blockDim elements per thread (consecutive)
            const uint32_t per = (P + blockDim.x - 1) / blockDim.x;
            const uint32_t e0 = threadIdx.x * per;
            uint32_t loc = 0;
            for (uint32_t e = e0; e < e0 + per && e < P; ++e) loc += (e < s && !(buf[e] & 1u));
            uint32_t tot;
            uint32_t run = block_excl_scan(loc, sh, &tot);
            for (uint32_t e = e0; e < e0 + per && e < P; ++e) {
                pre[e] = run;  // non-members before e
                run += (e < s && !(buf[e] & 1u));
            }
            __syncthreads();
            for (uint32_t e = threadIdx.x; e < s; e += blockDim.x) {
                const uint32_t v = buf[e];
                if (!(v & 1u)) continue;
                // members sort after the non-members of their value: pre[e]
                // counts below + equal; the value group's first element
                // (lower bound of (value << 1) in the sorted bucket) gives below
                const uint32_t first = v & ~1u;
                uint32_t lo = 0, hi = e;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (buf[mid] < first) lo = mid + 1;
                    else hi = mid;
                }
                acc += (unsigned long long)pre[lo] + pre[e];
            }
            __syncthreads();
        }
    }
    acc = block_sum_u64(acc, shl);
    if (threadIdx.x == 0 && acc) atomicAdd(&w.cnt[2], acc);
}

// 5. large buckets: members at low bits v add 2 #{non-members below v} +
// #{non-members at v}; work items (slot L, block j of kThreads bins), grid-
// stride, in two passes (block totals of the non-members, then the scan with
// the totals of the blocks before); the histograms are zeroed again
constexpr int kL2Blocks = kBuckets / kThreads;  // 64 blocks of bins per slot
__global__ void __launch_bounds__(kThreads) auc_l2_totals_kernel(Work w) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    __shared__ uint32_t sh[33];
    const uint32_t items = (uint32_t)w.cnt[4] * kL2Blocks;
    for (uint32_t it = blockIdx.x; it < items; it += gridDim.x) {
        const uint32_t L = it / kL2Blocks, j = it % kL2Blocks;
        const uint32_t nv = w.l2[(size_t)L * 2 * kBuckets + j * kThreads + threadIdx.x];
        uint32_t tot;
        block_excl_scan(nv, sh, &tot);
        if (threadIdx.x == 0) w.l2tot[it] = tot;
    }
}
__global__ void __launch_bounds__(kThreads) auc_l2_kernel(Work w) {
    if (fast_path(w)) return;  // the full-resolution path resolved the AUC
    __shared__ uint32_t sh[33];
    __shared__ unsigned long long shl[32];
    __shared__ uint32_t base;
    const uint32_t items = (uint32_t)w.cnt[4] * kL2Blocks;
    unsigned long long acc = 0;
    for (uint32_t it = blockIdx.x; it < items; it += gridDim.x) {
        const uint32_t L = it / kL2Blocks, j = it % kL2Blocks;
        if (threadIdx.x < 32) {
            uint32_t a = 0;
            for (uint32_t k = threadIdx.x; k < j; k += 32) a += w.l2tot[L * kL2Blocks + k];
            a = __reduce_add_sync(0xffffffffu, a);
            if (threadIdx.x == 0) base = a;
        }
        uint32_t* hn = w.l2 + (size_t)L * 2 * kBuckets + j * kThreads + threadIdx.x;
        uint32_t* hp = hn + kBuckets;
        const uint32_t nv = *hn, pv = *hp;
        uint32_t tot;
        const uint32_t e = block_excl_scan(nv, sh, &tot);  // (syncs: base visible)
        acc += (unsigned long long)pv * (2ull * (base + e) + nv);
        if (nv) *hn = 0;
        if (pv) *hp = 0;
    }
    acc = block_sum_u64(acc, shl);
    if (threadIdx.x == 0 && acc) atomicAdd(&w.cnt[2], acc);
}

}  // namespace auc
}  // namespace mtk
