// k_mmd_tc.cu -- multi-bandwidth Gaussian MMD^2 + gradient on the tcgen05
// tensor cores, FlashAttention-style (two chained 3xTF32 GEMMs per tile).
//
// Definition (oracle.c:orc_mmd_gaussian):
//   d2_ij = n_i + n_j - 2 z_i.z_j          (n_i = |z_i|^2)
//   k_ij  = sum_b exp(-d2_ij / s_b),   A_ij = sum_b (2/s_b) exp(-d2_ij / s_b)
//   w_ij  = c_ij A_ij  (c = -2/m^2 S-S, -2/n^2 T-T, 2/(m n) cross, 0 on i = j)
//   g_i   = sum_j w_ij (z_i - z_j) = z_i * Wsum_i - V_i,   V = W . Z
// Per CTA: 128 rows i (M) x a 256-wide slice of V's feature dims; it streams
// every 128-row j tile of Z:
//   GEMM1  S[128x128] = Z_i . Z_j^T      (TMEM cols [256,384), K = d)
//   exp    4 epilogue warps: S -> d2 -> k, A, w; fp64 kernel sums and Wsum;
//          w is split into tf32 hi/lo and written back to TMEM (hi over S,
//          lo in cols [384,512)) -- FlashAttention-4 style, no smem round trip
//   GEMM2  V[128xVD] += W[128x128] . Z_j[128xVD]  (A from TMEM; cols [0,VD))
// Operands are the tf32 hi/lo planes of Z ([G][N][d] each, written by
// mmd_prep_kernel together with the row norms); all products are 3xTF32
// (hi*hi + hi*lo + lo*hi).  TMA brings both planes, so the 128-B/clk shared
// memory port carries only TMA writes and tensor-core reads (an on-chip split
// adds a read and two writes per element and made the kernel smem-bound).
// One warp issues TMA, one issues MMAs, four run the exp epilogue.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace mtk {
namespace {

using namespace sm100;

constexpr int TI = 128, TJ = 64, KC = 32, JC = 16, VD = 256;
// Two smem plans (template RES):
//   RES = false  4-stage ring of 48 KB: G1 stages bring Z_i hi+lo and Z_j hi+lo
//   RES = true   (d <= 256) Z_i hi stays resident (128 KB, loaded once) and a
//                3-stage ring of 32 KB brings Z_i lo + Z_j hi+lo -- a quarter
//                less L2 -> smem traffic per j tile
constexpr int G1_BYTES = 2 * (TI * KC * 4) + 2 * (TJ * KC * 4);  // 48 KB (hi + lo planes)
constexpr int G1R_BYTES = (TI * KC * 4) + 2 * (TJ * KC * 4);     // 32 KB (Z_i lo + Z_j hi/lo)
constexpr int G2_BYTES = 2 * (JC * VD * 4);                       // 32 KB
constexpr int RES_BYTES = TI * VD * 4;                            // resident Z_i hi (d <= 256)
template <bool RES>
struct Plan {
    static constexpr int STAGES = RES ? 3 : 4;
    static constexpr int STAGE_BYTES = RES ? G1R_BYTES : G1_BYTES;
    static constexpr int RING_OFF = RES ? RES_BYTES : 0;
    static constexpr int SMEM_BYTES = RING_OFF + STAGES * STAGE_BYTES + 1024 + 256;
};
static_assert(Plan<true>::SMEM_BYTES <= 232448, "resident plan exceeds smem");
constexpr int NUM_THREADS = 192;
// TMEM columns: V [0,256); S / W-hi double buffer b at 256 + 64 b (S is
// overwritten in place by the hi plane of W); W-lo buffer b at 384 + 64 b.
// TMEM columns: V [0,256); S/W buffer b at 256 + 128 b.  GEMM1 runs as
//   [S_lo | S_hh] (128 cols) = Z_i_hi . [Z_j_lo | Z_j_hi]^T   (one N=128 MMA)
//   S_hh += Z_i_lo . Z_j_hi^T                                  (N=64, cols 64..127)
// so Z_i_hi is read once per k step instead of twice (GEMM1 is bound by the
// A-operand smem reads at N=64); S = S_lo + S_hh.  The epilogue then writes
// W's tf32 hi over cols [0,64) and lo over [64,128) of the same buffer.
constexpr uint32_t S_COL = 256;
constexpr uint32_t SBUF = 128;

struct MmdTcParams {
    CUtensorMap zk_hi, zk_lo;   // K-major views of the planes: (d, N, G), box (32, 64)
    CUtensorMap zm_hi, zm_lo;   // MN-major views: (d, N, G), box (32, 16), 32-B atom swizzle
    const float* zhi;           // [G][N][d] planes
    const float* zlo;
    const float* xs;            // the fp32 sample rows (z_i in the gradient epilogue)
    const float* xt;
    long long xs_gs, xt_gs;
    const float* norms;         // [G][N]
    const double* beta;         // [G]
    long long m, n;
    int d;
    int nb;
    int geo5;                   // bandwidth multipliers are {1/4, 1/2, 1, 2, 4}
    float mult[8];
    long long row_begin, row_end;
    double* partial;            // [G][nblk][3]
    int nblk;
    float* gXs;
    long long gs_gs;
    float* gXt;
    long long gt_gs;
    float grad_scale;
    int* flags;
    double* vacc;               // [G][N][d] fp64 flush buffer for V, or null (short j loops)
    unsigned long long* trace;  // diagnostics: phase timestamps of CTA (0,0,0), or null
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace layout: [0..4096) producer stage-ready times, [4096..8192) MMA stage-consumed
// times, [8192..12288) epilogue: per tile (s_full seen, w_full arrived)
#define TRACE(off, idx)                                                                   \
    do {                                                                                  \
        if (tr && (idx) < 4096) tr[(off) + (idx)] = gtime();                              \
    } while (0)

// V is accumulated in fp32 TMEM for FLUSH j tiles at a time, then drained
// into an fp64 buffer: the MMD gradient is a small difference of large
// same-domain and cross-domain sums, and fp32 tensor-core accumulation over
// tens of thousands of j would not hold 1e-5 (C4: m+n = 73728).
constexpr int FLUSH = 16;  // j tiles (1024 rows of Z) per fp32 V chunk

template <bool RES>
__global__ void __launch_bounds__(NUM_THREADS, 1) mmd_tc_kernel(const __grid_constant__ MmdTcParams p) {
    constexpr int STAGES = Plan<RES>::STAGES, STAGE_BYTES = Plan<RES>::STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* res = smem0;                          // resident Z_i hi (RES)
    uint8_t* smem = smem0 + Plan<RES>::RING_OFF;   // the stage ring
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* s_full = empty + STAGES;  // [2]
    uint64_t* w_full = s_full + 2;      // [2]
    uint64_t* v_full = w_full + 2;
    uint64_t* v_empty = v_full + 1;
    uint64_t* res_full = v_empty + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.z;
    const int dslice = blockIdx.y;
    const int v0 = dslice * VD;
    const int vd = min(VD, p.d - v0);  // feature columns of V owned here
    const long long N = p.m + p.n;
    const long long rb = p.row_begin, re = p.row_end;
    const long long i0 = rb + (long long)blockIdx.x * TI;
    const int nkc = (p.d + KC - 1) / KC;
    const int njt = (int)((N + TJ - 1) / TJ);
    const bool do_flush = p.vacc != nullptr;
    unsigned long long* tr =
        (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ? p.trace : nullptr;
    // per-CTA start / end / SM id at [12288 + 3 * cta] (diagnostics)
    const long long cta_lin = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (p.trace && threadIdx.x == 0 && cta_lin < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[12288 + 3 * cta_lin] = gtime();
        p.trace[12288 + 3 * cta_lin + 2] = smid;
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.zk_hi);
        tma_prefetch(&p.zk_lo);
        tma_prefetch(&p.zm_hi);
        tma_prefetch(&p.zm_lo);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&w_full[b], 128);
        }
        mbar_init(v_full, 1);
        mbar_init(v_empty, 128);
        mbar_init(res_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Software pipeline (MMA order == TMA order):
    //   G1(0), G1(1), G2(0), G1(2), G2(1), ..., G1(n-1), G2(n-2), G2(n-1)
    // so the exp epilogue of tile t overlaps GEMM1 of tile t+1.
    // Producer and MMA warps run their loops converged (all 32 lanes wait on
    // the barriers; lane 0 issues): a lone lane spinning while its siblings
    // sit in the final __syncthreads was observed to leave the warp
    // descheduled for ~100 us after the work was done.
    if (warp == 0) {
        {
            // ---------------- TMA producer ----------------
            if (RES && lane == 0) {  // resident Z_i hi: kc chunk at kc * 16 KB (two 64-row boxes)
                mbar_expect_tx(res_full, (uint32_t)(nkc * 2 * 8192));
                for (int kc = 0; kc < nkc; ++kc) {
                    tma_load_3d(res + kc * 16384, &p.zk_hi, res_full, kc * KC, (int)i0, g);
                    tma_load_3d(res + kc * 16384 + 8192, &p.zk_hi, res_full, kc * KC, (int)i0 + 64, g);
                }
            }
            __syncwarp();
            int st = 0;
            for (int t = 0; t <= njt; ++t) {
                if (t < njt) {
                    const int j0 = t * TJ;
                    for (int kc = 0; kc < nkc; ++kc, ++st) {
                        const int s = st % STAGES;
                        mbar_wait(&empty[s], ((st / STAGES) & 1) ^ 1);
                        if (lane == 0) TRACE(0, st);
                        uint8_t* b = smem + s * STAGE_BYTES;
                        const int k0 = kc * KC;
                        if (lane == 0) {
                            if (RES) {
                                // Z_i lo [0,16K) (two 64-row boxes), Z_j lo [16K,24K), hi [24K,32K)
                                mbar_expect_tx(&full[s], G1R_BYTES);
                                tma_load_3d(b, &p.zk_lo, &full[s], k0, (int)i0, g);
                                tma_load_3d(b + 8192, &p.zk_lo, &full[s], k0, (int)i0 + 64, g);
                                tma_load_3d(b + 16384, &p.zk_lo, &full[s], k0, j0, g);
                                tma_load_3d(b + 24576, &p.zk_hi, &full[s], k0, j0, g);
                            } else {
                                // Z_i hi [0,16K) and lo [16K,32K) (two 64-row boxes each),
                                // Z_j lo [32K,40K) and hi [40K,48K)
                                mbar_expect_tx(&full[s], G1_BYTES);
                                tma_load_3d(b, &p.zk_hi, &full[s], k0, (int)i0, g);
                                tma_load_3d(b + 8192, &p.zk_hi, &full[s], k0, (int)i0 + 64, g);
                                tma_load_3d(b + 16384, &p.zk_lo, &full[s], k0, (int)i0, g);
                                tma_load_3d(b + 24576, &p.zk_lo, &full[s], k0, (int)i0 + 64, g);
                                tma_load_3d(b + 32768, &p.zk_lo, &full[s], k0, j0, g);
                                tma_load_3d(b + 40960, &p.zk_hi, &full[s], k0, j0, g);
                            }
                        }
                        __syncwarp();
                    }
                }
                if (t >= 1) {
                    const int j0 = (t - 1) * TJ;
                    for (int jc = 0; jc < TJ / JC; ++jc, ++st) {
                        const int s = st % STAGES;
                        mbar_wait(&empty[s], ((st / STAGES) & 1) ^ 1);
                        uint8_t* b = smem + s * STAGE_BYTES;
                        if (lane == 0) {
                            TRACE(0, st);
                            mbar_expect_tx(&full[s], G2_BYTES);
                            for (int q = 0; q < VD / 32; ++q) {
                                tma_load_3d(b + q * 2048, &p.zm_hi, &full[s], v0 + 32 * q, j0 + JC * jc, g);
                                tma_load_3d(b + 16384 + q * 2048, &p.zm_lo, &full[s], v0 + 32 * q,
                                            j0 + JC * jc, g);
                            }
                        }
                        __syncwarp();
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        {
            constexpr uint32_t id1 = idesc_tf32(TI, TJ, 0, 0);
            constexpr uint32_t id1w = idesc_tf32(TI, 2 * TJ, 0, 0);
            constexpr uint32_t id2 = idesc_tf32(TI, VD, 0, 1);
            const uint32_t tV = tmem;
            const uint32_t rbase = smem_u32(res);
            if (RES) {
                mbar_wait(res_full, 0);
                tc_fence_after();
            }
            int st = 0;
            for (int t = 0; t <= njt; ++t) {
                if (t < njt) {
                    const uint32_t tS = tmem + S_COL + (t & 1) * SBUF;
                    for (int kc = 0; kc < nkc; ++kc, ++st) {
                        const int s = st % STAGES;
                        mbar_wait(&full[s], (st / STAGES) & 1);
                        tc_fence_after();
                        const uint32_t b = smem_u32(smem + s * STAGE_BYTES);
                        if (lane == 0) {
                        TRACE(4096, st);
#pragma unroll
                        for (int kk = 0; kk < KC / 8; ++kk) {
                            const uint64_t ahi = RES ? smem_desc(rbase + kc * 16384 + kk * 32, 16, 1024, 2)
                                                     : smem_desc(b + kk * 32, 16, 1024, 2);
                            const uint64_t alo = smem_desc(b + (RES ? 0 : 16384) + kk * 32, 16, 1024, 2);
                            // 128 rows: Z_j lo (64) then Z_j hi (64)
                            const uint64_t blh = smem_desc(b + (RES ? 16384 : 32768) + kk * 32, 16, 1024, 2);
                            const uint64_t bhi = smem_desc(b + (RES ? 24576 : 40960) + kk * 32, 16, 1024, 2);
                            mma_tf32(tS, ahi, blh, id1w, (kc | kk) ? 1u : 0u);
                            mma_tf32(tS + TJ, alo, bhi, id1, 1u);
                        }
                        mma_commit(&empty[s]);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) mma_commit(&s_full[t & 1]);
                    __syncwarp();
                }
                if (t >= 1) {
                    const int jt = t - 1;
                    const uint32_t tWhi = tmem + S_COL + (jt & 1) * SBUF;
                    const uint32_t tWlo = tWhi + TJ;
                    mbar_wait(&w_full[jt & 1], (jt >> 1) & 1);  // W(jt) is in TMEM
                    tc_fence_after();
                    const bool chunk_start = do_flush ? (jt % FLUSH == 0) : (jt == 0);
                    if (do_flush && jt > 0 && jt % FLUSH == 0) {
                        mbar_wait(v_empty, ((jt / FLUSH) - 1) & 1);  // previous chunk drained
                        tc_fence_after();
                    }
                    for (int jc = 0; jc < TJ / JC; ++jc, ++st) {
                        const int s = st % STAGES;
                        mbar_wait(&full[s], (st / STAGES) & 1);
                        tc_fence_after();
                        const uint32_t b = smem_u32(smem + s * STAGE_BYTES);
                        if (lane == 0) {
                        TRACE(4096, st);
#pragma unroll
                        for (int h = 0; h < JC / 8; ++h) {
                            const uint32_t kcol = (uint32_t)(jc * JC + h * 8);
                            const uint64_t bhi = smem_desc(b + h * 1024, 2048, 512, 1);
                            const uint64_t blo = smem_desc(b + 16384 + h * 1024, 2048, 512, 1);
                            const uint32_t acc0 = (!chunk_start || jc || h) ? 1u : 0u;
                            mma_tf32_ts(tV, tWlo + kcol, bhi, id2, acc0);
                            mma_tf32_ts(tV, tWhi + kcol, blo, id2, 1u);
                            mma_tf32_ts(tV, tWhi + kcol, bhi, id2, 1u);
                        }
                        mma_commit(&empty[s]);
                        }
                        __syncwarp();
                    }
                    if (lane == 0 && do_flush && (jt + 1) % FLUSH == 0 && jt + 1 < njt) mma_commit(v_full);
                    __syncwarp();
                }
            }
            if (lane == 0) mma_commit(v_full);
            __syncwarp();
            if (tr && lane == 0) tr[12282] = gtime();
        }
    } else {
        // ---------------- epilogue warps: exp + weights, then the gradient ----------------
        const int q = warp & 3;
        const int r = 32 * q + lane;  // row within the tile == TMEM lane
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const long long gi = i0 + r;
        const bool row_ok = gi < re;
        const bool si = gi < p.m;
        const double beta = p.beta[g];
        float nscale[8];  // -log2(e) / s_b
        float two_inv[8];
        for (int b = 0; b < 8; ++b) {
            const double s = beta * (double)p.mult[b];
            nscale[b] = b < p.nb ? (float)(-1.4426950408889634 / s) : 0.f;
            two_inv[b] = b < p.nb ? (float)(2.0 / s) : 0.f;
        }
        const float x1 = (float)(-1.4426950408889634 / beta);  // log2 scale for s = beta
        const float tb = (float)(2.0 / beta);
        const float cSS = (float)(-2.0 / ((double)p.m * (double)p.m));
        const float cTT = (float)(-2.0 / ((double)p.n * (double)p.n));
        const float cST = (float)(2.0 / ((double)p.m * (double)p.n));
        const float* nrm = p.norms + (long long)g * N;
        const float ni = row_ok ? nrm[gi] : 0.f;
        double ksum[3] = {0.0, 0.0, 0.0};
        double wsum = 0.0;
        int nflush = 0;
        for (int jt = 0; jt < njt; ++jt) {
            const long long j0 = (long long)jt * TJ;
            const int bsel = jt & 1;
            mbar_wait(&s_full[bsel], (jt >> 1) & 1);
            if (r == 0) TRACE(8192, 2 * jt);
            tc_fence_after();
            float kss = 0.f, ktt = 0.f, kst = 0.f, part = 0.f;
            // 8-column chunks keep the unrolled body (and the I-cache footprint) small
#pragma unroll 1
            for (int ch = 0; ch < TJ / 8; ++ch) {
                float sv[8], wlo[8];
                {
                    float sh[8];
                    tmem_ld_32x8(tmem + lane_base + S_COL + bsel * SBUF + ch * 8, sv);
                    tmem_ld_32x8(tmem + lane_base + S_COL + bsel * SBUF + TJ + ch * 8, sh);
#pragma unroll
                    for (int c = 0; c < 8; ++c) sv[c] += sh[c];  // S = S_lo + S_hh
                }
                const long long jb = j0 + ch * 8;
                // column classes are warp-uniform: all 8 j in range / same domain?
                const bool full8 = row_ok && jb + 8 <= N;
                const bool sj_all = jb + 8 <= p.m, tj_all = jb >= p.m;
                float kv8[8], A8[8];
                if (p.geo5) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const long long gj = jb + c;
                        const float nj = (gj < N) ? __ldg(nrm + gj) : 0.f;
                        const float d2 = fmaxf(ni + nj - 2.f * sv[c], 0.f);
                        // s_b = beta * {1/4,1/2,1,2,4}: two ex2, the rest by squaring
                        const float e1 = exp2f(d2 * x1);          // s = beta
                        const float e4 = exp2f(d2 * x1 * 0.25f);  // s = 4 beta
                        const float e2 = e4 * e4;                 // s = 2 beta
                        const float eh = e1 * e1;                 // s = beta/2
                        const float eq = eh * eh;                 // s = beta/4
                        kv8[c] = ((eq + eh) + (e1 + e2)) + e4;
                        A8[c] = tb * ((4.f * eq + 2.f * eh) + (e1 + 0.5f * e2) + 0.25f * e4);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const long long gj = jb + c;
                        const float nj = (gj < N) ? __ldg(nrm + gj) : 0.f;
                        const float d2 = fmaxf(ni + nj - 2.f * sv[c], 0.f);
                        float kv = 0.f, A = 0.f;
#pragma unroll 1
                        for (int b = 0; b < p.nb; ++b) {
                            const float e = exp2f(d2 * nscale[b]);
                            kv += e;
                            A = fmaf(two_inv[b], e, A);
                        }
                        kv8[c] = kv;
                        A8[c] = A;
                    }
                }
                if (full8 && (sj_all || tj_all) && !(gi >= jb && gi < jb + 8)) {
                    // fast path: one domain pair for the whole chunk, no diagonal
                    const float cw = si ? (sj_all ? cSS : cST) : (sj_all ? cST : cTT);
                    float ks = 0.f;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        ks += kv8[c];
                        const float wv = cw * A8[c];
                        part += wv;
                        split_tf32(wv, sv[c], wlo[c]);
                    }
                    if (si && sj_all) kss += ks;
                    else if (!si && tj_all) ktt += ks;
                    else if (si) kst += ks;
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const long long gj = jb + c;
                        float wv = 0.f;
                        if (row_ok && gj < N) {
                            const bool sj = gj < p.m;
                            if (si && sj) {
                                kss += kv8[c];
                                wv = cSS * A8[c];
                            } else if (!si && !sj) {
                                ktt += kv8[c];
                                wv = cTT * A8[c];
                            } else {
                                if (si) kst += kv8[c];
                                wv = cST * A8[c];
                            }
                            if (gj == gi) wv = 0.f;
                        }
                        part += wv;
                        split_tf32(wv, sv[c], wlo[c]);
                    }
                }
                tmem_st_32x8(tmem + lane_base + S_COL + bsel * SBUF + ch * 8, sv);
                tmem_st_32x8(tmem + lane_base + S_COL + bsel * SBUF + TJ + ch * 8, wlo);
            }
            ksum[0] += kss;
            ksum[1] += ktt;
            ksum[2] += kst;
            wsum += part;
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&w_full[bsel]);
            if (r == 0) TRACE(8192, 2 * jt + 1);
            // drain the previous V chunk (G2 of tile jt-1 closed it) into fp64
            if (do_flush && jt > 0 && jt % FLUSH == 0) {
                mbar_wait(v_full, nflush & 1);
                tc_fence_after();
                double* vrow = p.vacc + ((long long)g * N + (row_ok ? gi : 0)) * p.d + v0;
#pragma unroll 1
                for (int cb = 0; cb < VD / 32; ++cb) {
                    float vv[32];
                    tmem_ld_32x32(tmem + lane_base + cb * 32, vv);
                    if (!row_ok || cb * 32 >= vd) continue;
                    double2* vp = reinterpret_cast<double2*>(vrow + cb * 32);
                    if (cb * 32 + 32 <= vd) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            double2 o = nflush ? vp[c] : make_double2(0.0, 0.0);
                            o.x += (double)vv[2 * c];
                            o.y += (double)vv[2 * c + 1];
                            vp[c] = o;
                        }
                    } else {
                        for (int c = 0; cb * 32 + c < vd; ++c)
                            vrow[cb * 32 + c] = (nflush ? vrow[cb * 32 + c] : 0.0) + (double)vv[c];
                    }
                }
                tc_fence_before();
                mbar_arrive(v_empty);
                ++nflush;
            }
        }
        // gradient rows: g_i = scale * (z_i * Wsum_i - V_i) over this CTA's feature slice
        mbar_wait(v_full, nflush & 1);
        tc_fence_after();
        if (tr && r == 0) tr[12283] = gtime();  // v_full seen
        // All MMAs and TMA loads are complete, so the ring is idle.  The fp32
        // z_i tile streams into it with cp.async (every 16-B piece in flight
        // at once), each thread turns its own row into g in place (V from
        // TMEM), and the tile leaves in coalesced float4 order.
        const int t = threadIdx.x - 64;
        constexpr int VLD = VD + 4;  // float4-aligned rows, conflict-free row-wise float4
        constexpr int C4 = VD / 4;
        static_assert(TI * VLD * 4 <= Plan<true>::RING_OFF + Plan<true>::STAGES * Plan<true>::STAGE_BYTES &&
                          TI * VLD * 4 <= Plan<false>::STAGES * Plan<false>::STAGE_BYTES,
                      "finish tile exceeds the idle smem");
        const uint32_t zsb = smem_u32(smem0);
        for (int e = t; e < TI * C4; e += 128) {
            const int rr = e / C4, c4 = e % C4;
            const long long row = i0 + rr;
            if (row >= re || 4 * c4 >= vd) continue;
            const float* zr = row < p.m ? p.xs + g * p.xs_gs + row * p.d : p.xt + g * p.xt_gs + (row - p.m) * p.d;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(zsb + (uint32_t)((rr * VLD + 4 * c4) * 4)),
                         "l"(zr + v0 + 4 * c4)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tr && r == 0) tr[12284] = gtime();
        bool bad = false;
        const double scale = (double)p.grad_scale;
        const double* va = (nflush && row_ok) ? p.vacc + ((long long)g * N + gi) * p.d + v0 : nullptr;
#pragma unroll 1
        for (int cb = 0; cb < VD / 32; ++cb) {
            float vv[32];
            tmem_ld_32x32(tmem + lane_base + cb * 32, vv);
            if (!row_ok || cb * 32 >= vd) continue;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const uint32_t a4 = zsb + (uint32_t)((r * VLD + cb * 32 + c) * 4);
                const float4 z4 = lds128(a4);
                const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
                float gq[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double vt = (double)vv[c + q] + (va ? va[cb * 32 + c + q] : 0.0);
                    gq[q] = (float)(((double)zz[q] * wsum - vt) * scale);
                    bad |= !isfinite(gq[q]);
                }
                sts128(a4, make_float4(gq[0], gq[1], gq[2], gq[3]));
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tr && r == 0) tr[12285] = gtime();
        const bool vec_out = ((reinterpret_cast<uintptr_t>(p.gXs) | reinterpret_cast<uintptr_t>(p.gXt)) & 15) == 0 &&
                             (p.gs_gs | p.gt_gs) % 4 == 0;
        for (int e = t; e < TI * C4; e += 128) {
            const int rr = e / C4, c4 = e % C4;
            const long long row = i0 + rr;
            if (row >= re || 4 * c4 >= vd) continue;
            float* o = row < p.m ? (p.gXs ? p.gXs + g * p.gs_gs + row * p.d : nullptr)
                                 : (p.gXt ? p.gXt + g * p.gt_gs + (row - p.m) * p.d : nullptr);
            if (!o) continue;
            const float4 g4 = lds128(zsb + (uint32_t)((rr * VLD + 4 * c4) * 4));
            if (vec_out) {
                *reinterpret_cast<float4*>(o + v0 + 4 * c4) = g4;
            } else {
                o[v0 + 4 * c4] = g4.x;
                o[v0 + 4 * c4 + 1] = g4.y;
                o[v0 + 4 * c4 + 2] = g4.z;
                o[v0 + 4 * c4 + 3] = g4.w;
            }
        }
        if (tr && r == 0) tr[12286] = gtime();
        if (bad) atomicOr(p.flags, kFlagNonFinite);
        // fixed-order reduction of the kernel sums over the 128 rows (d-slice 0 only)
        // (dynamic smem past the finish tile: the whole ring is idle by now)
        double(*red)[128] = reinterpret_cast<double(*)[128]>(smem0 + ((TI * VLD * 4 + 1023) & ~1023));
        for (int c = 0; c < 3; ++c) red[c][t] = ksum[c];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int w = 64; w > 0; w >>= 1) {
            if (t < w)
                for (int c = 0; c < 3; ++c) red[c][t] += red[c][t + w];
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        if (t < 3 && dslice == 0) p.partial[((long long)g * p.nblk + blockIdx.x) * 3 + t] = red[t][0];
        if (tr && r == 0) tr[12287] = gtime();
    }
    tc_fence_before();
    __syncthreads();
    if (p.trace && threadIdx.x == 0 && cta_lin < 4096) p.trace[12288 + 3 * cta_lin + 1] = gtime();
    if (warp == 1) {
        if (tr && lane == 0) tr[12281] = gtime();
        tc_fence_after();
        if (tr && lane == 0) tr[12280] = gtime();
        tmem_dealloc<512>(tmem);
        if (p.trace && lane == 0 && cta_lin < 4096) p.trace[12288 + 3 * cta_lin + 2] = gtime();
    }
}

// n_i = |z_i|^2 (fp64 accumulation) and the tf32 planes hi = rna(z),
// lo = rna(z - hi) of Z = [Xs; Xt] as [G][N][d] each.  Block = kBetaRows rows
// (8 warps x 4 rows, one warp per row, float4; d % 4 == 0 on this path).
// With `part` non-null it also writes the bandwidth partials of its rows in
// beta_partial's layout: part[g][blk][c] = sum_rows z_c, part[g][blk][d] =
// sum_rows n_i (fp64, fixed order), so beta costs no second pass over Z.
constexpr int PREP_WARPS = 8;
__global__ void __launch_bounds__(256) mmd_prep_kernel(const float* Xs, long long xs_gs, const float* Xt,
                                                       long long xt_gs, long long m, long long n, int d,
                                                       float* zhi, float* zlo, float* norms,
                                                       double* part) {
    extern __shared__ double colsum[];  // [PREP_WARPS][d] when part != null
    __shared__ double nsum[PREP_WARPS];
    const int g = blockIdx.y;
    const long long N = m + n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d4 = d / 4;
    double* cs = part ? colsum + warp * d : nullptr;
    if (cs)
        for (int c = lane; c < d; c += 32) cs[c] = 0.0;
    // the warp's 4 rows advance together (their loads in flight at once);
    // per row and per column the summation order is unchanged (k ascending,
    // rows ascending)
    constexpr int R = kBetaRows / PREP_WARPS;
    const float4* src[R];
    float4* hi[R];
    float4* lo[R];
    bool ok[R];
    double acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const long long row = (long long)blockIdx.x * kBetaRows + warp * R + i;
        ok[i] = row < N;
        const long long rr = ok[i] ? row : 0;
        src[i] = reinterpret_cast<const float4*>(rr < m ? Xs + g * xs_gs + rr * d : Xt + g * xt_gs + (rr - m) * d);
        const long long o = ((long long)g * N + rr) * d;
        hi[i] = reinterpret_cast<float4*>(zhi + o);
        lo[i] = reinterpret_cast<float4*>(zlo + o);
        acc[i] = 0.0;
    }
    // two k steps per trip: all 2R row loads in flight before any store
    for (int k0 = lane; k0 < d4; k0 += 64) {
        float4 xx[2][R];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int i = 0; i < R; ++i)
                xx[u][i] = (ok[i] && k0 + 32 * u < d4) ? src[i][k0 + 32 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int k = k0 + 32 * u;
        if (k >= d4) break;
        const float4 (&x)[R] = xx[u];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (!ok[i]) continue;
            float4 h, l;
            split_tf32(x[i].x, h.x, l.x);
            split_tf32(x[i].y, h.y, l.y);
            split_tf32(x[i].z, h.z, l.z);
            split_tf32(x[i].w, h.w, l.w);
            hi[i][k] = h;
            lo[i][k] = l;
            acc[i] += (double)x[i].x * (double)x[i].x + (double)x[i].y * (double)x[i].y;
            acc[i] += (double)x[i].z * (double)x[i].z + (double)x[i].w * (double)x[i].w;
        }
        if (cs) {  // lanes own disjoint columns: no races
            double c0 = cs[4 * k], c1 = cs[4 * k + 1], c2 = cs[4 * k + 2], c3 = cs[4 * k + 3];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (!ok[i]) continue;
                c0 += (double)x[i].x;
                c1 += (double)x[i].y;
                c2 += (double)x[i].z;
                c3 += (double)x[i].w;
            }
            cs[4 * k] = c0;
            cs[4 * k + 1] = c1;
            cs[4 * k + 2] = c2;
            cs[4 * k + 3] = c3;
        }
    }
    }
    double nacc = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        double a2 = acc[i];
        for (int o2 = 16; o2 > 0; o2 >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o2);
        if (ok[i]) {
            if (lane == 0) norms[(long long)g * N + (long long)blockIdx.x * kBetaRows + warp * R + i] = (float)a2;
            nacc += a2;
        }
    }
    if (!part) return;
    if (lane == 0) nsum[warp] = nacc;
    __syncthreads();
    double* out = part + ((long long)g * gridDim.x + blockIdx.x) * (d + 1);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < PREP_WARPS; ++w) t += colsum[w * d + c];
        out[c] = t;
    }
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < PREP_WARPS; ++w) t += nsum[w];
        out[d] = t;
    }
}

// ---------------------------------------------------------------------------
// Materialised-W path (bank steps with gradients, N = m + n small enough that
// W [G][N][N] fits the scratch budget).  The kernel matrix is symmetric, so
// pass 1 visits each unordered 128 x 128 tile pair (I <= J) ONCE:
//   S_IJ = Z_I . Z_J^T      (3xTF32 on the rna planes: one N=256 MMA over
//                            [Z_J lo | Z_J hi] plus an N=128 Z_I lo . Z_J hi)
//   exp epilogue -> w_ij, written to W at (i, j) and, for I < J, at (j, i)
//   (the transposed store is coalesced: lanes are consecutive i);
//   per-tile partials: row sums of w (rows of I), column sums (rows of J),
//   the three kernel sums with the pair multiplicities of the V-statistic.
// Then V = W . Z is a plain grouped 3xTF32 GEMM (umma_kernel) whose epilogue
// forms g = scale * (z * Wsum - V) (Epi::kMmdGrad).  GEMM1 work is halved
// against the fused kernel, which evaluates every ordered pair.
constexpr int WT = 128;
constexpr int W_STAGES = 2;
constexpr int W_STAGE_BYTES = 4 * (WT * KC * 4);  // Z_I hi, Z_I lo, Z_J lo, Z_J hi: 64 KB
constexpr int W_TILE_LD = 33;  // per-warp 32 x 32 transpose tile, padded (conflict-free)
constexpr int W_MAX_G_TAB = 2048;  // per-group exp scales kept in smem
constexpr int W_SMEM_BYTES = W_STAGES * W_STAGE_BYTES + 1024 + 256 + 16 * 32 * W_TILE_LD * 4 + W_MAX_G_TAB * 8;
static_assert(W_SMEM_BYTES <= 232448, "mmd_w_kernel smem");
constexpr int W_EPI_WARPS = 16;  // 4 per TMEM lane quarter, 32 columns each
constexpr int W_THREADS = 64 + 32 * W_EPI_WARPS;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct MmdWParams {
    CUtensorMap zk_hi, zk_lo;  // K-major (d, N, G), 128-row boxes
    const float* norms;        // [G][N]
    const double* beta;        // [G]
    long long m, n;
    int d, nb, geo5;
    float mult[8];
    int T, npairs, G;
    // owned tile rows [ta, tb) (all: 0, T): the items are the tile pairs that
    // touch them -- list A, pairs (I >= ta in range, J >= I), contiguous in the
    // upper-triangle order from pair index pa; list B, pairs (I < ta, J in range)
    int ta, tb, pa, nA, nB;
    // optional explicit item order (I, J) of one group, nA entries (nB = 0):
    // the L2-blocked raster of large problems (mmd_w_order)
    const int2* order;
    float* W;                  // [G][N][ldw] (rows outside [ta, tb) * WT never written)
    long long ldw;             // row stride of W (N, or N + 32 with the head block)
    float* rpart;              // [G][T][T][4][WT]: row sums of block (I, J), per column quarter
    float* cpart;              // [G][T][T][4][WT]: column sums of block (I, J) (I < J), per row quarter
    double* kpart;             // [G][npairs][W_EPI_WARPS][3]: kernel sums per epilogue warp
    int* flags;
    int diag;                  // diagnostics (MTK_MMDW_DIAG): 1 = epilogue only arrives, 2 = no MMAs
    int no_diag_share;         // A/B (MTK_MMDW_NO_DIAG_SHARE): diagonal tiles load Z_J too
};

// unordered tile pair p -> (I, J), I <= J, row-major over the upper triangle
// (row I starts at S(I) = I*T - I*(I-1)/2): closed form + integer fix-up
__device__ __forceinline__ void pair_of(int p, int T, int& I, int& J);
// work item of one group -> (I, J, pair index) over lists A then B (above)
__device__ __forceinline__ void item_pair(const MmdWParams& p, int k, int& I, int& J, int& pidx) {
    if (p.order) {
        const int2 ij = p.order[k];
        I = ij.x;
        J = ij.y;
        pidx = (int)((long long)I * p.T - (long long)I * (I - 1) / 2) + (J - I);
        return;
    }
    if (k < p.nA) {
        pidx = p.pa + k;
        pair_of(pidx, p.T, I, J);
        return;
    }
    k -= p.nA;
    const int w = p.tb - p.ta;
    I = k / w;
    J = p.ta + k % w;
    pidx = (int)((long long)I * p.T - (long long)I * (I - 1) / 2) + (J - I);
}
__device__ __forceinline__ void pair_of(int p, int T, int& I, int& J) {
    const double b = 2.0 * T + 1.0;
    int i = (int)((b - sqrt(b * b - 8.0 * (double)p)) * 0.5);
    i = max(0, min(i, T - 1));
    auto start = [T](int r) { return (long long)r * T - (long long)r * (r - 1) / 2; };
    while (i > 0 && start(i) > p) --i;
    while (i + 1 < T && start(i + 1) <= p) ++i;
    I = i;
    J = i + (int)(p - start(i));
}

// 8 column values per lane (lane = row) -> the sum over the warp's 32 rows
// of column ((lane>>4)&1)*4 + ((lane>>3)&1)*2 + ((lane>>2)&1), complete on
// lanes with (lane & 3) == 0.  Fixed butterfly order (deterministic).
__device__ __forceinline__ float column_sums_8(const float (&v)[8], int lane) {
    float a[4], b[2];
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float send = u16 ? v[c] : v[c + 4];
        const float keep = u16 ? v[c + 4] : v[c];
        a[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const float send = u8 ? a[c] : a[c + 2];
        const float keep = u8 ? a[c + 2] : a[c];
        b[c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float x;
    {
        const float send = u4 ? b[0] : b[1];
        const float keep = u4 ? b[1] : b[0];
        x = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

__global__ void __launch_bounds__(W_THREADS, 1) mmd_w_kernel(const __grid_constant__ MmdWParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + W_STAGES * W_STAGE_BYTES);
    uint64_t* empty = full + W_STAGES;
    uint64_t* acc_full = empty + W_STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    float* wtile = reinterpret_cast<float*>(smem + W_STAGES * W_STAGE_BYTES + 256);  // [16][32][33]
    float2* gtab = reinterpret_cast<float2*>(wtile + 16 * 32 * W_TILE_LD);            // [G]: (x1, tb)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long N = p.m + p.n;
    const int nkc = (p.d + KC - 1) / KC;
    const int nloc = p.nA + p.nB;  // items per group
    const int total = p.G * nloc;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.zk_hi);
        tma_prefetch(&p.zk_lo);
        for (int s = 0; s < W_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 32 * W_EPI_WARPS);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    pdl_wait();  // the predecessors' outputs (beta, norms, planes) are read from here on
    for (int g = threadIdx.x; g < p.G && g < W_MAX_G_TAB; g += blockDim.x) {
        const double beta = p.beta[g];
        gtab[g] = make_float2((float)(-1.4426950408889634 / beta), (float)(2.0 / beta));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        int st = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const int g = item / nloc;
            int I, J, pidx_;
            item_pair(p, item % nloc, I, J, pidx_);
            const int i0 = I * WT, j0 = J * WT;
            const bool dg = I == J && !p.no_diag_share;  // a diagonal tile: Z_J is Z_I, two planes only
            for (int kc = 0; kc < nkc; ++kc, ++st) {
                const int s = st % W_STAGES;
                mbar_wait(&empty[s], ((st / W_STAGES) & 1) ^ 1);
                if (lane == 0) {
                    uint8_t* b = smem + s * W_STAGE_BYTES;
                    const int k0 = kc * KC;
                    mbar_expect_tx(&full[s], dg ? W_STAGE_BYTES / 2 : W_STAGE_BYTES);
                    tma_load_3d(b, &p.zk_hi, &full[s], k0, i0, g);  // 128-row boxes (16 KB each)
                    tma_load_3d(b + 16384, &p.zk_lo, &full[s], k0, i0, g);
                    if (!dg) {
                        tma_load_3d(b + 32768, &p.zk_lo, &full[s], k0, j0, g);
                        tma_load_3d(b + 49152, &p.zk_hi, &full[s], k0, j0, g);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idw = idesc_tf32(WT, 2 * WT, 0, 0);
        constexpr uint32_t idn = idesc_tf32(WT, WT, 0, 0);
        int st = 0, lt = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x, ++lt) {
            const int buf = lt & 1;
            const uint32_t tS = tmem + buf * 256;
            int I, J, pidx_;
            item_pair(p, item % nloc, I, J, pidx_);
            // a diagonal tile reads Z_I as both operands: B = [Z_I hi | Z_I lo] puts
            // hi.hi (+ lo.hi, second MMA) in columns [0, 128) and hi.lo in
            // [128, 256) -- the two blocks of an off-diagonal tile, swapped; the
            // epilogue adds them (commutative: the same bits)
            const bool dg = I == J && !p.no_diag_share;
            mbar_wait(&acc_empty[buf], ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            for (int kc = 0; kc < nkc; ++kc, ++st) {
                const int s = st % W_STAGES;
                mbar_wait(&full[s], (st / W_STAGES) & 1);
                tc_fence_after();
                const uint32_t b = smem_u32(smem + s * W_STAGE_BYTES);
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < KC / 8; ++kk) {
                        if (p.diag == 2) break;
                        const uint64_t ahi = smem_desc(b + kk * 32, 16, 1024, 2);
                        const uint64_t alo = smem_desc(b + 16384 + kk * 32, 16, 1024, 2);
                        if (dg) {
                            const uint64_t bhl = smem_desc(b + kk * 32, 16, 1024, 2);  // hi 128 | lo 128
                            mma_tf32(tS, ahi, bhl, idw, (kc | kk) ? 1u : 0u);
                            mma_tf32(tS, alo, ahi, idn, 1u);
                        } else {
                            const uint64_t blh = smem_desc(b + 32768 + kk * 32, 16, 1024, 2);  // lo 128 | hi 128
                            const uint64_t bhi = smem_desc(b + 49152 + kk * 32, 16, 1024, 2);
                            mma_tf32(tS, ahi, blh, idw, (kc | kk) ? 1u : 0u);
                            mma_tf32(tS + WT, alo, bhi, idn, 1u);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(&acc_full[buf]);
            __syncwarp();
        }
    } else {
        // ---------------- epilogue: exp -> w, stores, partials ----------------
        // 16 warps: warp w covers TMEM lane quarter q = w % 4 (rows 32q..32q+31)
        // and column quarter h (32 columns); four warps share each scheduler.
        // Partials go straight to global memory (no block barriers); the
        // wsum kernel combines them in a fixed order.
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int r = 32 * q + lane;
        const int ew = warp - 2;
        float* tw = wtile + ew * 32 * W_TILE_LD;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const float cSS = (float)(-2.0 / ((double)p.m * (double)p.m));
        const float cTT = (float)(-2.0 / ((double)p.n * (double)p.n));
        const float cST = (float)(2.0 / ((double)p.m * (double)p.n));
        int lt = 0;
        bool bad = false;
        for (int item = blockIdx.x; item < total; item += gridDim.x, ++lt) {
            const int g = item / nloc;
            int I, J, pidx;
            item_pair(p, item % nloc, I, J, pidx);
            const bool diag = I == J;
            // a pair whose two tiles belong to different ranks is evaluated by
            // both; each keeps only the half in its own rows (and only the
            // owner of I counts its kernel sums)
            const bool own_i = I >= p.ta && I < p.tb, own_j = J >= p.ta && J < p.tb;
            const int gi = I * WT + r;
            const bool row_ok = gi < N;
            const bool si = gi < p.m;
            float x1, tb;
            if (g < W_MAX_G_TAB) {
                const float2 xt = gtab[g];
                x1 = xt.x;
                tb = xt.y;
            } else {
                x1 = (float)(-1.4426950408889634 / p.beta[g]);
                tb = (float)(2.0 / p.beta[g]);
            }
            float nscale[8], two_inv[8];
            if (!p.geo5) {  // general bandwidth set: per-bandwidth scales
                const double beta = p.beta[g];
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const double sb = beta * (double)p.mult[b];
                    nscale[b] = b < p.nb ? (float)(-1.4426950408889634 / sb) : 0.f;
                    two_inv[b] = b < p.nb ? (float)(2.0 / sb) : 0.f;
                }
            }
            const float* nrm = p.norms + (long long)g * N;
            const float ni = row_ok ? nrm[gi] : 0.f;
            float* Wg = p.W + (long long)g * N * p.ldw;
            const long long ldw = p.ldw;
            const int buf = lt & 1;
            mbar_wait(&acc_full[buf], (lt >> 1) & 1);
            tc_fence_after();
            float kss = 0.f, ktt = 0.f, kst = 0.f, rowp = 0.f;
            const float mo = diag ? 1.f : 2.f;  // an off-diagonal unordered pair stands for two
#pragma unroll 1
            for (int ch = 4 * h; ch < 4 * h + 4; ++ch) {
                if (p.diag == 1) break;
                float sv[8];
                {
                    float sh[8];
                    tmem_ld_32x8(tmem + lane_base + buf * 256 + ch * 8, sv);
                    tmem_ld_32x8(tmem + lane_base + buf * 256 + WT + ch * 8, sh);
#pragma unroll
                    for (int c = 0; c < 8; c += 2) {
                        const float2 t2 = __fadd2_rn(make_float2(sv[c], sv[c + 1]), make_float2(sh[c], sh[c + 1]));
                        sv[c] = t2.x;
                        sv[c + 1] = t2.y;
                    }
                }
                const int jb = J * WT + ch * 8;  // N^2 < 2^31 on this path: 32-bit offsets
                const bool full8 = jb + 8 <= N;
                float nj[8];
                if (full8) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(nrm + jb));
                    const float4 b = __ldg(reinterpret_cast<const float4*>(nrm + jb + 4));
                    nj[0] = a.x; nj[1] = a.y; nj[2] = a.z; nj[3] = a.w;
                    nj[4] = b.x; nj[5] = b.y; nj[6] = b.z; nj[7] = b.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) nj[c] = jb + c < N ? __ldg(nrm + jb + c) : 0.f;
                }
                float kv8[8], A8[8];
                if (p.geo5) {
                    // packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2), two columns per op
                    const float2 ni2 = make_float2(ni, ni), m2 = make_float2(-2.f, -2.f);
                    const float2 x1v = make_float2(x1, x1), x4v = make_float2(0.25f * x1, 0.25f * x1);
                    const float2 c4 = make_float2(4.f, 4.f), c2 = make_float2(2.f, 2.f);
                    const float2 ch5 = make_float2(0.5f, 0.5f), cq = make_float2(0.25f, 0.25f);
                    const float2 tbv = make_float2(tb, tb);
#pragma unroll
                    for (int c = 0; c < 8; c += 2) {
                        float2 d = __ffma2_rn(m2, make_float2(sv[c], sv[c + 1]),
                                              __fadd2_rn(ni2, make_float2(nj[c], nj[c + 1])));
                        d.x = fmaxf(d.x, 0.f);
                        d.y = fmaxf(d.y, 0.f);
                        const float2 a1 = __fmul2_rn(d, x1v), a4 = __fmul2_rn(d, x4v);
                        const float2 e1 = make_float2(ex2_approx(a1.x), ex2_approx(a1.y));
                        const float2 e4 = make_float2(ex2_approx(a4.x), ex2_approx(a4.y));
                        const float2 e2 = __fmul2_rn(e4, e4);
                        const float2 eh = __fmul2_rn(e1, e1);
                        const float2 eq = __fmul2_rn(eh, eh);
                        const float2 kv = __fadd2_rn(__fadd2_rn(__fadd2_rn(eq, eh), __fadd2_rn(e1, e2)), e4);
                        const float2 u = __ffma2_rn(c4, eq, __fmul2_rn(c2, eh));
                        const float2 v = __ffma2_rn(ch5, e2, e1);
                        const float2 A = __fmul2_rn(tbv, __ffma2_rn(cq, e4, __fadd2_rn(u, v)));
                        kv8[c] = kv.x;
                        kv8[c + 1] = kv.y;
                        A8[c] = A.x;
                        A8[c + 1] = A.y;
                    }
                } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float d2 = fmaxf(ni + nj[c] - 2.f * sv[c], 0.f);
                    {
                        float kv = 0.f, A = 0.f;
#pragma unroll
                        for (int b = 0; b < 8; ++b) {
                            if (b >= p.nb) break;
                            const float e = exp2f(d2 * nscale[b]);
                            kv += e;
                            A = fmaf(two_inv[b], e, A);
                        }
                        kv8[c] = kv;
                        A8[c] = A;
                    }
                }
                }
                float wv[8];
                const bool sj_all = jb + 8 <= p.m, tj_all = jb >= p.m;
                if (row_ok && full8 && (sj_all || tj_all) && !(diag && gi >= jb && gi < jb + 8)) {
                    // one domain pair for the whole chunk, no diagonal element
                    const float cw = si ? (sj_all ? cSS : cST) : (sj_all ? cST : cTT);
                    const float2 cw2 = make_float2(cw, cw);
                    float2 ks2 = make_float2(0.f, 0.f), rp2 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < 8; c += 2) {
                        ks2 = __fadd2_rn(ks2, make_float2(kv8[c], kv8[c + 1]));
                        const float2 w2 = __fmul2_rn(cw2, make_float2(A8[c], A8[c + 1]));
                        wv[c] = w2.x;
                        wv[c + 1] = w2.y;
                        rp2 = __fadd2_rn(rp2, w2);
                    }
                    const float ks = ks2.x + ks2.y;
                    rowp += rp2.x + rp2.y;
                    if (si == sj_all) {  // same domain
                        if (si) kss += mo * ks;
                        else ktt += mo * ks;
                    } else if (!diag || si) {
                        kst += ks;  // a mixed unordered pair counts once, as (s, t)
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int gj = jb + c;
                        float w = 0.f;
                        if (row_ok && gj < N) {
                            const bool sj = gj < p.m;
                            if (si && sj) {
                                kss += mo * kv8[c];
                                w = cSS * A8[c];
                            } else if (!si && !sj) {
                                ktt += mo * kv8[c];
                                w = cTT * A8[c];
                            } else {
                                if (!diag || si) kst += kv8[c];
                                w = cST * A8[c];
                            }
                            if (gj == gi) w = 0.f;
                        }
                        wv[c] = w;
                        rowp += w;
                    }
                }
                // (i, j) goes through the warp's smem tile (row = lane) and leaves
                // as coalesced 128-B row segments after the last chunk
#pragma unroll
                for (int c = 0; c < 8; ++c) tw[lane * W_TILE_LD + (ch - 4 * h) * 8 + c] = wv[c];
                if (!diag && own_j) {
                    // (j, i): lanes are consecutive i -> one 128-B row segment per store
                    float* dt = Wg + ((long long)jb * ldw + gi);
                    if (p.diag == 3 || p.diag == 4) {
                    } else if (row_ok && full8) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            *dt = wv[c];
                            dt += ldw;
                        }
                    } else if (row_ok) {
                        for (int c = 0; c < 8 && jb + c < N; ++c) dt[c * ldw] = wv[c];
                    }
                    const float cs = column_sums_8(wv, lane);
                    if ((lane & 3) == 0)
                        p.cpart[((((long long)g * p.T + I) * p.T + J) * 4 + q) * WT + ch * 8 +
                                ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = cs;
                }
            }
            bad |= !isfinite(rowp);
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
            __syncwarp();
            if (p.diag != 3 && p.diag != 5 && own_i) {
                const int jc = J * WT + 32 * h + lane;
                const int r0 = I * WT + 32 * q;
                const int nr = min(32, (int)N - r0);
                if (jc < N) {
                    float* dst = Wg + ((long long)r0 * ldw + jc);
#pragma unroll 8
                    for (int rr = 0; rr < nr; ++rr) {
                        *dst = tw[rr * W_TILE_LD + lane];
                        dst += ldw;
                    }
                }
            }
            __syncwarp();

            if (!own_i) continue;  // the (j, i) half, column sums: done above
            p.rpart[((((long long)g * p.T + I) * p.T + J) * 4 + h) * WT + r] = rowp;
            // this warp's kernel sums: fixed butterfly over the 32 rows, fp64
            double kd[3] = {(double)kss, (double)ktt, (double)kst};
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) kd[c] += __shfl_xor_sync(0xffffffffu, kd[c], o);
            if (lane < 3) {
                const double v = lane == 0 ? kd[0] : (lane == 1 ? kd[1] : kd[2]);
                p.kpart[(((long long)g * p.npairs + pidx) * W_EPI_WARPS + ew) * 3 + lane] = v;
            }
        }
        if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
    }
    pdl_trigger();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// Wsum_i = sum over column blocks J of block (R, J)'s row sums, R = i / WT:
// for J >= R the four column-quarter row sums of pair (R, J), for J < R the
// four row-quarter column sums of pair (J, R) -- fixed order, fp64.  Blocks
// past the Wsum range each take one (g, I) and form the kernel-sum partials
// in the fused kernel's layout: partial[g][I][c] = sum_{J >= I} sum_w
// kpart[g][pair(I, J)][w][c] (every load in flight, then fixed-order sums).
constexpr int WSUM_THREADS = 256;
// The fused head DX (MmdArgs::hd_*) rides on the V = W.Z GEMM as 32 extra K
// columns: A = [W | dZ_head 0], B = [Z ; -W_head^T / lambda 0], so the GEMM's
// kMmdGrad epilogue lambda * (z * Wsum - acc) gives lambda * g + dZ_head W_head^T.
constexpr int kHeadK = 32;

struct WsumHead {  // the fused head DX's extra K block (hn = 0: none)
    int hn, d;
    const float* dz;   // [G][N][hn]
    long long dz_gs;
    const float* Wh;   // [G][d][hn]
    long long wh_gs;
    float scale;       // lambda
    float* W;          // [G][N][ldw]: columns N .. N + kHeadK
    long long ldw;
    float* bx;         // [G][kHeadK][d]
};
// Rows: the owned rows [r0, r0 + NR) of every group (all rows unless the
// call is tile-sharded); tile rows: [ta, ta + NT) -> blocks of the kernel sums.
__global__ void __launch_bounds__(WSUM_THREADS) mmd_wsum_kernel(const float* rpart, const float* cpart,
                                                                const double* kpart, int G, long long N,
                                                                int T, int npairs, float* wsum,
                                                                double* partial, WsumHead h, long long r0,
                                                                long long NR, int ta, int NT, float* wdiag,
                                                                long long ldw) {
    __shared__ double jsum[3][WSUM_THREADS / 3 + 1];
    const long long nbw = ((long long)G * NR + WSUM_THREADS - 1) / WSUM_THREADS;
    if (blockIdx.x >= nbw + (long long)G * NT) {  // head block B rows: -W_head^T / lambda
        const long long e = (blockIdx.x - nbw - (long long)G * T) * WSUM_THREADS + threadIdx.x;
        const long long per = (long long)kHeadK * h.d;
        if (e >= G * per) return;
        const int g = (int)(e / per), j = (int)(e % per / h.d), n = (int)(e % h.d);
        h.bx[e] = j < h.hn ? __fdiv_rn(-h.Wh[g * h.wh_gs + (long long)n * h.hn + j], h.scale) : 0.f;
        return;
    }
    if (blockIdx.x < nbw) {
        const long long tl = blockIdx.x * (long long)WSUM_THREADS + threadIdx.x;
        if (tl >= (long long)G * NR) return;
        const int g = (int)(tl / NR);
        const long long i = r0 + tl % NR;
        const long long t = (long long)g * N + i;
        if (h.hn) {  // head block A columns of row i: dZ_head[i, :], zero past hn
            const float* z = h.dz + g * h.dz_gs + i * h.hn;
            float4* dst = reinterpret_cast<float4*>(h.W + ((long long)g * N + i) * h.ldw + N);
#pragma unroll
            for (int c = 0; c < kHeadK / 4; ++c) {
                float4 v;
                v.x = 4 * c < h.hn ? z[4 * c] : 0.f;
                v.y = 4 * c + 1 < h.hn ? z[4 * c + 1] : 0.f;
                v.z = 4 * c + 2 < h.hn ? z[4 * c + 2] : 0.f;
                v.w = 4 * c + 3 < h.hn ? z[4 * c + 3] : 0.f;
                dst[c] = v;
            }
        }
        const int R = (int)(i / WT), r = (int)(i % WT);
        double s = 0.0;
#pragma unroll 4
        for (int J = 0; J < T; ++J) {
            const float* src = J >= R ? rpart + ((((long long)g * T + R) * T + J) * 4) * WT
                                      : cpart + ((((long long)g * T + J) * T + R) * 4) * WT;
            s += (double)(((src[r] + src[WT + r]) + src[2 * WT + r]) + src[3 * WT + r]);
        }
        wsum[t] = (float)s;
        // W' = W - diag(Wsum) (wdiag: the single-chunk V GEMM folds z * Wsum in)
        if (wdiag) wdiag[((long long)g * N + i) * ldw + i] = -(float)s;
        return;
    }
    const int gi = (int)(blockIdx.x - nbw), g = gi / NT, I = ta + gi % NT;
    int base = 0;
    for (int k = 0; k < I; ++k) base += T - k;
    const int nJ = T - I;
    double total[3] = {0.0, 0.0, 0.0};
    // chunks of up to WSUM_THREADS / 3 column blocks: thread (c, jj) sums the
    // 16 warp partials of pair (I, I + j0 + jj), then threads c < 3 add the
    // chunk in ascending J
    for (int j0 = 0; j0 < nJ; j0 += WSUM_THREADS / 3) {
        const int c = threadIdx.x / (WSUM_THREADS / 3), jj = threadIdx.x % (WSUM_THREADS / 3);
        if (c < 3 && j0 + jj < nJ) {
            const double* kp = kpart + ((long long)g * npairs + base + j0 + jj) * W_EPI_WARPS * 3 + c;
            double v[W_EPI_WARPS];
#pragma unroll
            for (int w = 0; w < W_EPI_WARPS; ++w) v[w] = kp[w * 3];
            double a = 0.0;
#pragma unroll
            for (int w = 0; w < W_EPI_WARPS; ++w) a += v[w];
            jsum[c][jj] = a;
        }
        __syncthreads();
        if (threadIdx.x < 3)
            for (int jj2 = 0; jj2 < WSUM_THREADS / 3 && j0 + jj2 < nJ; ++jj2) total[threadIdx.x] += jsum[threadIdx.x][jj2];
        __syncthreads();
    }
    if (threadIdx.x < 3) partial[((long long)g * T + I) * 3 + threadIdx.x] = total[threadIdx.x];
}

// Item order for large tile triangles: the tile pairs in S x S blocks (block
// rows ascending, block columns >= block row; row-major inside a block), so
// the ~148 pairs in flight at a time share ~2S tiles of Z (S = 16: 16 MB of
// tf32 planes) and Z stays in L2 while W streams out.  The row-major order
// sweeps all J for each I instead; at C4 (T = 576, 302 MB of planes) that
// re-read Z from DRAM (ncu r09: 84 GB of DRAM traffic for 21.7 GB of W).
// Only pairs touching the owned tiles [ta, tb) are listed.  Cached per
// (device, T, ta, tb); the order does not change any pair's arithmetic.
constexpr int kRasterMinT = 32, kRasterS = 16;
const int2* mmd_w_order(int T, int ta, int tb, int* count, cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, std::pair<int2*, int>> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, T, ta, tb);
    auto it = cache.find(key);
    if (it == cache.end()) {
        std::vector<int2> v;
        const int nb = (T + kRasterS - 1) / kRasterS;
        for (int bi = 0; bi < nb; ++bi)
            for (int bj = bi; bj < nb; ++bj)
                for (int I = bi * kRasterS; I < std::min(T, (bi + 1) * kRasterS); ++I)
                    for (int J = std::max(I, bj * kRasterS); J < std::min(T, (bj + 1) * kRasterS); ++J)
                        if ((I >= ta && I < tb) || (J >= ta && J < tb)) v.push_back(make_int2(I, J));
        int2* d = nullptr;
        MTK_CUDA(cudaMalloc(&d, v.size() * sizeof(int2)));
        MTK_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
        MTK_CUDA(cudaStreamSynchronize(s));
        it = cache.emplace(key, std::make_pair(d, (int)v.size())).first;
    }
    *count = it->second.second;
    return it->second.first;
}

// g = scale * (z * Wsum - sum_c V_c), the chunk partials summed in ascending
// chunk order in fp64 (the multi-chunk V = W.Z of the materialised-W path)
__global__ void mmd_vchunk_finish_kernel(const float* __restrict__ vpart, int chunks, long long per,
                                         const float* __restrict__ Z, long long z_gs,
                                         const float* __restrict__ wsum, float* __restrict__ gout,
                                         long long g_gs, int G, long long N, int d, float scale, int* flags) {
    const long long total = (long long)G * per;  // per = N * d
    bool bad = false;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int g = (int)(e / per);
        const long long o = e % per, i = o / d;
        double v = 0.0;
        for (int c = 0; c < chunks; ++c) v += (double)vpart[(long long)c * total + e];
        const double z = (double)Z[g * z_gs + o];
        const float x = (float)((double)scale * (z * (double)wsum[(long long)g * N + i] - v));
        bad |= !isfinite(x);
        gout[g * g_gs + o] = x;
    }
    if (bad) atomicOr(flags, kFlagNonFinite);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
        if (!fn) fail(MTK_ERROR, "cuTensorMapEncodeTiled unavailable");
    }
    return fn;
}

CUtensorMap zmap(const float* base, long long d, long long N, long long G, long long gs,
                 int box_outer, bool mn) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)G};
    const cuuint64_t strides[2] = {(cuuint64_t)(d * 4), (cuuint64_t)(gs * 4)};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (gs * 4) % 16)
        fail(MTK_ERROR, "mmd: sample not 16-byte aligned for TMA");
    const cuuint32_t box[3] = {32, (cuuint32_t)box_outer, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MTK_ERROR, "cuTensorMapEncodeTiled failed (mmd)");
    return m;
}

}  // namespace

bool mmd_tc_supported(const MmdArgs& a) { return a.d % 4 == 0 && a.d >= 4; }

int mmd_tc_blocks_per_group(const MmdArgs& a) {
    const long long N = a.m + a.n;
    const long long re = a.row_end < 0 ? N : a.row_end;
    return (int)((re - a.row_begin + TI - 1) / TI);
}

// the materialised-W path (mmd_w_kernel + a grouped GEMM): bank-shaped calls
// with gradients whose samples and gradients are each one contiguous
// [G][m+n][d] block and whose W fits the budget; MTK_MMD_FUSED=1 forces the
// fused kernel (A/B)
// W budget: fixed (not free-memory dependent), so the path -- and with it the
// rounding -- is the same on every box.  C4 (N = 73,728, one group) needs 21.7 GB.
constexpr double kWBudget = 48.0 * 1024 * 1024 * 1024;
static bool getenv_flag(const char* name) {  // A/B switches, read per call
    const char* e = getenv(name);
    return e && e[0] == '1';
}
static bool w_path(const MmdArgs& a) {
    const char* fe = getenv("MTK_MMD_FUSED");
    const bool fused = fe && fe[0] == '1';
    const long long N = a.m + a.n;
    if (fused || !a.gXs || !a.gXt || a.m <= 0 || a.n <= 0) return false;
    if (a.row_begin != 0 || (a.row_end >= 0 && a.row_end != N)) return false;
    if (a.tile_end >= 0) return a.G == 1 && a.d % 4 == 0 && a.d >= 32 && N % 4 == 0 &&
                                a.Xt == a.Xs + a.m * a.d && a.gXt == a.gXs + a.m * a.d;  // sharded: own rows of W
    if (a.d % 4 || a.d < 32 || N % 4) return false;
    if (a.Xt != a.Xs + a.m * a.d || a.xt_gs != a.xs_gs || a.xs_gs < N * a.d) return false;
    if (a.gXt != a.gXs + a.m * a.d || a.gt_gs != a.gs_gs || a.gs_gs != a.xs_gs) return false;
    return (double)a.G * N * N * 4.0 <= kWBudget;
}

// V = W.Z accumulates in fp32 in TMEM; past kVChunk columns of W it runs as
// kVChunk-deep GEMMs whose fp32 partials are summed in fp64 (the fused pair
// kernel's V flush interval: 16 j tiles of 64)
constexpr long long kVChunk = 1024;
static int v_chunks(const MmdArgs& a) { return (int)((a.m + a.n + kVChunk - 1) / kVChunk); }

static bool head_block(const MmdArgs& a) {
    return a.hd_n > 0 && a.hd_n <= kHeadK && (a.m + a.n) % 32 == 0 && v_chunks(a) == 1 && a.tile_end < 0;
}

// the owned tile rows [ta, tb) and rows [r0, r0 + NR) of a (tile-sharded) W path
struct WRows {
    int T, ta, tb;
    long long r0, NR;
};
static WRows w_rows(const MmdArgs& a) {
    const long long N = a.m + a.n;
    WRows w;
    w.T = (int)((N + WT - 1) / WT);
    w.ta = a.tile_end < 0 ? 0 : (int)a.tile_begin;
    w.tb = a.tile_end < 0 ? w.T : (int)a.tile_end;
    w.r0 = (long long)w.ta * WT;
    w.NR = std::min(N, (long long)w.tb * WT) - w.r0;
    return w;
}

bool mmd_head_fusable(const MmdArgs& a) { return w_path(a) && head_block(a); }
bool mmd_w_path(const MmdArgs& a) { return w_path(a); }

struct WLayout {
    long long ldw;  // row stride of W: N, or N + kHeadK with the head block
    float* bx;      // [G][kHeadK][d]: -W_head^T / lambda, zero rows past hd_n
    float* vpart;   // [chunks][G][N][d] fp32 partials of V (more than one chunk)
    float* W;
    float* rpart;
    float* cpart;
    double* kpart;
    float* wsum;
    size_t bytes;
};
static WLayout w_layout(const MmdArgs& a, uintptr_t base) {
    const long long N = a.m + a.n;
    const int T = (int)((N + WT - 1) / WT), np = T * (T + 1) / 2;
    const WRows wr = w_rows(a);
    WLayout L;
    uintptr_t cur = (base + 255) & ~uintptr_t(255);
    const uintptr_t start = cur;
    L.ldw = N + (head_block(a) ? kHeadK : 0);
    // only the owned rows of W exist (all rows unless tile-sharded, G = 1 then):
    // L.W points at row 0 of the virtual [N][ldw] matrix
    L.W = reinterpret_cast<float*>(cur) - (wr.NR < N ? wr.r0 * L.ldw : 0);
    cur = (cur + (size_t)a.G * (wr.NR < N ? wr.NR : N) * L.ldw * 4 + 255) & ~uintptr_t(255);
    L.bx = reinterpret_cast<float*>(cur);
    if (head_block(a)) cur = (cur + (size_t)a.G * kHeadK * a.d * 4 + 255) & ~uintptr_t(255);
    L.rpart = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * T * T * 4 * WT * 4 + 255) & ~uintptr_t(255);
    L.cpart = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * T * T * 4 * WT * 4 + 255) & ~uintptr_t(255);
    L.kpart = reinterpret_cast<double*>(cur);
    cur = (cur + (size_t)a.G * np * W_EPI_WARPS * 3 * 8 + 255) & ~uintptr_t(255);
    L.wsum = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * N * 4 + 255) & ~uintptr_t(255);
    L.vpart = reinterpret_cast<float*>(cur);
    if (v_chunks(a) > 1) cur = (cur + (size_t)v_chunks(a) * a.G * wr.NR * a.d * 4 + 255) & ~uintptr_t(255);
    L.bytes = cur - start + 256;
    return L;
}

static bool needs_flush(const MmdArgs& a) {
    const long long N = a.m + a.n;
    const bool grads = a.gXs || a.gXt;
    return grads && (N + TJ - 1) / TJ > FLUSH;
}

size_t mmd_tc_scratch_bytes(const MmdArgs& a) {
    const long long N = a.m + a.n;
    size_t b = (size_t)a.G * N * sizeof(float) + 1024;
    b += 2 * ((size_t)a.G * N * a.d * sizeof(float) + 256);
    if (a.beta_out) b += (size_t)a.G * ((N + kBetaRows - 1) / kBetaRows) * (a.d + 1) * sizeof(double) + 256;
    if (needs_flush(a)) b += (size_t)a.G * N * a.d * sizeof(double) + 256;
    if (w_path(a)) b += w_layout(a, 0).bytes + 256;
    return b;
}

// scratch: >= mmd_tc_scratch_bytes(a); a.partial must hold [G][blocks][3]
void launch_mmd_tc(const MmdArgs& a, void* scratch, cudaStream_t s, int stages) {
    const long long N = a.m + a.n;
    const long long re = a.row_end < 0 ? N : a.row_end;
    uintptr_t cur = (reinterpret_cast<uintptr_t>(scratch) + 255) & ~uintptr_t(255);
    float* norms = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * N * sizeof(float) + 255) & ~uintptr_t(255);
    float* zhi = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * N * a.d * sizeof(float) + 255) & ~uintptr_t(255);
    float* zlo = reinterpret_cast<float*>(cur);
    cur = (cur + (size_t)a.G * N * a.d * sizeof(float) + 255) & ~uintptr_t(255);
    double* vacc = nullptr;
    if (needs_flush(a)) {
        vacc = reinterpret_cast<double*>(cur);
        cur = (cur + (size_t)a.G * N * a.d * sizeof(double) + 255) & ~uintptr_t(255);
    }
    double* bpart = a.beta_out ? reinterpret_cast<double*>(cur) : nullptr;
    if (bpart) cur = (cur + (size_t)a.G * ((N + kBetaRows - 1) / kBetaRows) * (a.d + 1) * sizeof(double) + 255) &
                     ~uintptr_t(255);
    constexpr int kFusedBetaMaxD = 512;  // colsum smem: 8 warps x d doubles
    const bool fused_beta = bpart && a.d <= kFusedBetaMaxD;
    if (stages & kMmdPrep) {
        if (bpart && !fused_beta) launch_mmd_beta(a, a.beta_out, bpart, s);
        const dim3 pg((unsigned)((N + kBetaRows - 1) / kBetaRows), a.G);
        const size_t prep_smem = fused_beta ? (size_t)PREP_WARPS * a.d * sizeof(double) : 0;
        if ((reinterpret_cast<uintptr_t>(a.Xs) | reinterpret_cast<uintptr_t>(a.Xt)) & 15 ||
            (a.xs_gs | a.xt_gs) % 4)
            fail(MTK_ERROR, "mmd: samples not 16-byte aligned");
        mmd_prep_kernel<<<pg, 32 * PREP_WARPS, prep_smem, s>>>(a.Xs, a.xs_gs, a.Xt, a.xt_gs, a.m, a.n,
                                                                a.d, zhi, zlo, norms,
                                                                fused_beta ? bpart : nullptr);
        count_launch();
        if (fused_beta) launch_mmd_beta_finish(a, bpart, a.beta_out, s);
    }
    if (!(stages & kMmdPairs)) return;
    const long long zgs = N * a.d;
    if (w_path(a)) {
        const WLayout L = w_layout(a, cur);
        const int T = (int)((N + WT - 1) / WT), np = T * (T + 1) / 2;
        MmdWParams w;
        std::memset(&w, 0, sizeof(w));
        w.zk_hi = zmap(zhi, a.d, N, a.G, zgs, WT, false);  // whole 128-row tiles: 4 TMA ops per stage
        w.zk_lo = zmap(zlo, a.d, N, a.G, zgs, WT, false);
        w.norms = norms;
        w.beta = a.beta;
        w.m = a.m;
        w.n = a.n;
        w.d = a.d;
        w.nb = a.nb;
        for (int b = 0; b < 8; ++b) w.mult[b] = a.mult[b] > 0 ? a.mult[b] : 1.f;
        w.geo5 = a.nb == 5 && a.mult[0] == 0.25f && a.mult[1] == 0.5f && a.mult[2] == 1.f &&
                 a.mult[3] == 2.f && a.mult[4] == 4.f;
        w.T = T;
        w.npairs = np;
        w.G = a.G;
        const WRows wr = w_rows(a);
        auto S = [T](long long I) { return I * T - I * (I - 1) / 2; };  // first pair of tile row I
        w.ta = wr.ta;
        w.tb = wr.tb;
        w.pa = (int)S(wr.ta);
        w.nA = (int)(S(wr.tb) - S(wr.ta));
        w.nB = wr.ta * (wr.tb - wr.ta);
        const char* re = getenv("MTK_MMDW_ROWMAJOR");  // A/B (read per call)
        if (T >= kRasterMinT && a.G == 1 && !(re && re[0] == '1')) {
            int cnt = 0;
            w.order = mmd_w_order(T, wr.ta, wr.tb, &cnt, s);
            if (cnt != w.nA + w.nB) fail(MTK_ERROR, "mmd: tile-pair raster size mismatch");
            w.nA = cnt;
            w.nB = 0;
        }
        w.W = L.W;
        w.ldw = L.ldw;
        w.rpart = L.rpart;
        w.cpart = L.cpart;
        w.kpart = L.kpart;
        w.flags = a.flags;
        if (const char* e = getenv("MTK_MMDW_DIAG")) w.diag = atoi(e);
        w.no_diag_share = getenv_flag("MTK_MMDW_NO_DIAG_SHARE") ? 1 : 0;
        ensure_smem_attr(reinterpret_cast<const void*>(mmd_w_kernel), W_SMEM_BYTES);
        const int sms = device_sm_count(current_device());
        const int items = a.G * (w.nA + w.nB);
        {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)std::min(items, sms));
            cfg.blockDim = dim3(W_THREADS);
            cfg.dynamicSmemBytes = W_SMEM_BYTES;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (mmd_w calls pdl_wait)
            at[0].val.programmaticStreamSerializationAllowed = umma::pdl_enabled() ? 1 : 0;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            MTK_CUDA(cudaLaunchKernelEx(&cfg, mmd_w_kernel, w));
        }
        count_launch();
        const long long nbw = ((long long)a.G * wr.NR + WSUM_THREADS - 1) / WSUM_THREADS;
        const int NT = wr.tb - wr.ta;
        const bool head = head_block(a);
        WsumHead h;
        std::memset(&h, 0, sizeof(h));
        long long nbx = 0;
        if (head) {
            if (!a.hd_out || !a.hd_dz || !a.hd_W || a.grad_scale == 0.f)
                fail(MTK_ERROR, "mmd: incomplete fused head DX arguments");
            h.hn = a.hd_n;
            h.d = a.d;
            h.dz = a.hd_dz;
            h.dz_gs = a.hd_dz_gs;
            h.Wh = a.hd_W;
            h.wh_gs = a.hd_w_gs;
            h.scale = a.grad_scale;
            h.W = L.W;
            h.ldw = L.ldw;
            h.bx = L.bx;
            nbx = ((long long)a.G * kHeadK * a.d + WSUM_THREADS - 1) / WSUM_THREADS;
        }
        // single-chunk V GEMM: fold z * Wsum into it as a -Wsum diagonal of W, so
        // its epilogue needs no z (only the fused head's ReLU mask, as bits)
        const int nch = v_chunks(a);
        const bool wdiag = nch == 1 && (!head || a.hd_zbits) && !getenv_flag("MTK_MMD_NO_WDIAG");
        mmd_wsum_kernel<<<(unsigned)(nbw + (long long)a.G * NT + nbx), WSUM_THREADS, 0, s>>>(
            L.rpart, L.cpart, L.kpart, a.G, N, T, np, L.wsum, a.partial, h, wr.r0, wr.NR, wr.ta, NT,
            wdiag ? L.W : nullptr, L.ldw);
        count_launch();
        // V = W.Z over the owned rows [r0, r0 + NR) (all rows unless sharded)
        const long long r0 = wr.r0, NR = wr.NR;
        UmmaGemm u;
        u.G = a.G;
        u.M = (int)NR;
        u.N = a.d;
        u.K = (int)N;
        u.a_mn = 0;
        u.a = L.W + r0 * L.ldw;
        u.a_rs = L.ldw;
        u.a_gs = N * L.ldw;
        u.b_mn = 1;
        u.b = a.Xs;
        u.b_rs = a.d;
        u.b_gs = a.xs_gs;
        u.epi = Epi::kMmdGrad;
        u.same_sign = 1;  // W >= 0 (and Z >= 0 in bank steps): see k_umma.cu sepc
        u.sepc_share = 0;  // the gradient is a small difference: corrections separate from k = 0
        u.C = a.gXs + r0 * a.d;
        u.c_gs = a.gs_gs;
        if (head) {  // fused head DX: K gains the head block; the epilogue writes the layer's dZ
            u.K = (int)N + kHeadK;
            u.b2 = L.bx;
            u.b2_rs = a.d;
            u.b2_gs = (long long)kHeadK * a.d;
            u.ksplit = (int)N;
            u.C = a.hd_out;
            u.zmask = 1;
            u.colsum = a.hd_colsum;
        }
        u.ldc = a.d;
        u.add = a.Xs + r0 * a.d;
        u.rowvec = L.wsum + r0;  // G = 1 when sharded (the epilogue indexes g * M + m)
        u.scale = a.grad_scale;
        u.flags = a.flags;
        if (wdiag) {  // g = -scale * (W'.Z)[* mask]: no z, no Wsum in the epilogue
            u.epi = Epi::kMmdGradW;
            u.add = nullptr;
            u.rowvec = nullptr;
            // the corrections keep their own accumulator at any K: V' is a small
            // difference of the off-diagonal sum and the diagonal term
            u.same_sign = 1;
            if (head) {
                u.mbits = const_cast<uint32_t*>(a.hd_zbits) + r0 * a.hd_zbits_ld;
                u.mb_gs = a.hd_zbits_gs;
                u.mb_ld = a.hd_zbits_ld;
            }
        }
        if (nch > 1) {  // kVChunk-deep GEMMs into fp32 partials, then the fp64 finish
            const long long per = NR * a.d;
            for (int c = 0; c < nch; ++c) {
                const long long k0 = (long long)c * kVChunk;
                UmmaGemm v = u;
                v.K = (int)std::min(kVChunk, N - k0);
                v.a = L.W + r0 * L.ldw + k0;
                v.b = a.Xs + k0 * a.d;
                v.epi = Epi::kStore;
                v.sepc_share = 10;  // V partials (the difference is taken in fp64 after the chunks)
                v.C = L.vpart + (long long)c * a.G * per;
                v.c_gs = per;
                v.add = nullptr;
                v.rowvec = nullptr;
                v.colsum = nullptr;
                launch_umma(v, s);
            }
            const long long tot = (long long)a.G * per;
            mmd_vchunk_finish_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 148 * 16), 256, 0, s>>>(
                L.vpart, nch, per, a.Xs + r0 * a.d, a.xs_gs, L.wsum + r0, a.gXs + r0 * a.d, a.gs_gs, a.G, NR, a.d,
                a.grad_scale, a.flags);
            count_launch();
            return;
        }
        launch_umma(u, s);
        return;
    }
    MmdTcParams p;
    std::memset(&p, 0, sizeof(p));
    p.zk_hi = zmap(zhi, a.d, N, a.G, zgs, 64, false);  // 64-row boxes (two per 128-row tile)
    p.zk_lo = zmap(zlo, a.d, N, a.G, zgs, 64, false);
    p.zm_hi = zmap(zhi, a.d, N, a.G, zgs, JC, true);
    p.zm_lo = zmap(zlo, a.d, N, a.G, zgs, JC, true);
    p.zhi = zhi;
    p.zlo = zlo;
    p.xs = a.Xs;
    p.xt = a.Xt;
    p.xs_gs = a.xs_gs;
    p.xt_gs = a.xt_gs;
    p.norms = norms;
    p.beta = a.beta;
    p.m = a.m;
    p.n = a.n;
    p.d = a.d;
    p.nb = a.nb;
    for (int b = 0; b < 8; ++b) p.mult[b] = a.mult[b] > 0 ? a.mult[b] : 1.f;
    p.geo5 = a.nb == 5 && a.mult[0] == 0.25f && a.mult[1] == 0.5f && a.mult[2] == 1.f &&
             a.mult[3] == 2.f && a.mult[4] == 4.f;
    p.row_begin = a.row_begin;
    p.row_end = re;
    p.partial = a.partial;
    p.nblk = mmd_tc_blocks_per_group(a);
    p.gXs = a.gXs;
    p.gs_gs = a.gs_gs;
    p.gXt = a.gXt;
    p.gt_gs = a.gt_gs;
    p.grad_scale = a.grad_scale;
    p.flags = a.flags;
    p.vacc = vacc;
    p.trace = a.trace;
    ensure_smem_attr(reinterpret_cast<const void*>(mmd_tc_kernel<true>), Plan<true>::SMEM_BYTES);
    ensure_smem_attr(reinterpret_cast<const void*>(mmd_tc_kernel<false>), Plan<false>::SMEM_BYTES);
    dim3 grid(p.nblk, (a.d + VD - 1) / VD, a.G);
    // the resident-Z_i-hi plan measured ~1.5% slower than the 4-stage ring
    // (GEMM1 is bound by operand reads, not by the TMA stream); opt-in only
    static const bool use_res = getenv("MTK_MMD_RES") != nullptr;
    if (a.d <= VD && use_res)
        mmd_tc_kernel<true><<<grid, NUM_THREADS, Plan<true>::SMEM_BYTES, s>>>(p);
    else
        mmd_tc_kernel<false><<<grid, NUM_THREADS, Plan<false>::SMEM_BYTES, s>>>(p);
    count_launch();
}

}  // namespace mtk
