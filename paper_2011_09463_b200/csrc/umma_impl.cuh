// umma_impl.cuh -- grouped fp32-accurate GEMM on the 5th-gen tensor cores
// (tcgen05 + TMEM + TMA), sm_100a.
//
// C[g] (M x N) = A[g] (M x K) * B[g] (K x N) for G independent models.
// Operands live in HBM as plain fp32 and are staged into smem by TMA.
// The tf32 MMA truncates fp32 inputs (measured by tools/umma_probe.cu), so
// the staged fp32 tile itself serves as hi = trunc_tf32(x); converter warps
// add lo = rna_tf32(x - hi) (x - hi is exact) in a second tile, and three MMAs
// per k step give fp32-level products (3xTF32):
//     A*B ~= A_hi*B_lo + A_lo*B_hi + A_hi*B_hi      (dropped A_lo*B_lo < 2^-20)
// Truncated hi doubles the dropped term against rna hi (still ~1e-7 of
// max|C| on the bank's operands); it saves the in-place hi write-back, a
// seventh of the stage's shared-memory traffic, which bounds this kernel.
// (The MMD kernel keeps rna hi: its d^2 = n_i + n_j - 2 z_i.z_j cancels.)
// HBM and L2 carry 4 bytes per operand element, as for an fp32 SIMT GEMM.
//
// Replaces, for the bank's dense layers, the reference loops
//   detail::mm_acc (tape.hpp:36-48)    FWD: A = H   (K-major), B = W   (N-major)
//   detail::mm_nt_acc (tape.hpp:50-63) DX:  A = dZ  (K-major), B = W^T (K-major)
//   detail::mm_tn_acc (tape.hpp:65-78) DW:  A = H^T (M-major), B = dZ  (N-major)
// One kernel template covers both tile schemes:
//   PAIR = false  one CTA, 128 x 128 tile (small M or N)
//   PAIR = true   CTA pair (cta_group::2), 256 x 256 tile: each CTA stages
//                 128 rows of A and 128 columns of B; the leader issues
//                 M=256, N=256 MMAs over both CTAs' smem.
// Persistent: one CTA (pair) per SM (pair), static tile striding; the TMEM
// accumulator is double-buffered so the epilogue of tile t overlaps the
// mainloop of tile t+1.
// Accumulation precision (sepc): each MMA adds its 8 products into the fp32
// TMEM accumulator with the result truncated toward zero, so a long K drifts
// by ~0.5 ulp(acc) per MMA (measured, tools/gemm_precision.py: -1.9e-5 mean
// relative error at K = 1024 on same-sign operands, 8.4e-6 max on zero-mean
// ones).  Two thirds of those adds are the small hi*lo / lo*hi corrections.
// With sepc the corrections accumulate in their own TMEM accumulator (2^-10
// the magnitude, so their truncation is negligible) and the epilogue adds
// main + corr once in fp32: the drift falls to the 128 hi*hi adds of K = 1024.
// The correction accumulator takes the second TMEM buffer, so a sepc launch
// runs single-buffered (the epilogue no longer overlaps the next mainloop);
// it is used for K >= kSepcMinK and for the MMD V = W.Z GEMM (non-negative
// operands, and g = z Wsum - V cancels).
// Warp roles: w0 TMA producer, w1 MMA issuer (one elected thread), w2-w5
// epilogue (TMEM -> registers -> fused bias/ReLU | ReLU-mask | SGD -> HBM),
// w6-w13 converters.  Two rings: LS load stages (32 KB: A and B fp32 as TMA
// wrote them = the hi operands) and LO lo stages (32 KB: A lo, B lo),
// so TMA runs LS stages ahead while only LO stages hold lo planes.  128-B
// swizzle; 32-B-atom swizzle for MN-major operands (the only layout tf32
// accepts).
//
// The kernel and its launcher are templates over the operand majors, the
// CTA-pair scheme, the correction accumulator and the epilogue kind EPI (an
// Epi value, or -1 = read p.epi at run time).  The bank's launches use the
// EPI-specialised kernels: a run-time epilogue switch left all variants'
// code in the chunk loop, and the epilogue warps stalled on instruction
// fetch (ncu: stall_no_inst dominant in the epilogue).  Explicit
// instantiations live in k_umma_inst_*.cu (parallel compilation).
#pragma once

#include <cuda.h>

#include <algorithm>
#include <cmath>

#include "internal.h"
#include "sm100.cuh"

namespace mtk {
namespace umma {

using namespace sm100;


#ifndef MTK_UMMA_COAL
#define MTK_UMMA_COAL 1  // 0: no launch uses the smem-staged epilogue (A/B diagnostics)
#endif
constexpr int BK = 32, LO = 2;
constexpr int kSepcMinK = 768;  // K from which corrections get their own accumulator
constexpr int TILE_BYTES = 128 * BK * 4;     // 16 KB: 128 rows (or cols) x 32 k
constexpr int LOAD_BYTES = 2 * TILE_BYTES;   // load stage: A fp32, B fp32 (TMA bytes)
constexpr int LO_BYTES = 2 * TILE_BYTES;     // lo stage: A lo, B lo
constexpr int NUM_EPI_WARPS = 8;   // two per TMEM lane quarter, each half the columns
// Epilogue plan per epilogue kind.  The smem-staged coalesced epilogue
// (epilogue_coalesced) takes a 4 KB tile + 128 B of row words per epilogue
// warp, paid for with one load stage (LS 5 -> 4).  Measured (same box, C2
// step, the thread-per-row path as the baseline): bias / bias + ReLU (FWD)
// 239.8 -> 232 us, ReLU-mask DX without an addend 70.8 -> 62.8 us, SGD (DW,
// operands loaded in groups of 4 passes) 238.8 -> 220.5 us; the MMD-gradient
// epilogue (z and the row scale per element) spills and measured slower
// (+20 us), so it and the DX with an addend keep the thread-per-row path.
//
// Template-only epilogue kind: the ReLU-mask DX without an addend (the bank's
// DX launches).  Without the addend the coalesced epilogue loads no
// per-element operand.
constexpr int kEpiMaskNoAdd = 16;
template <int EPI>
constexpr int epi_kind() { return EPI == kEpiMaskNoAdd ? (int)Epi::kMask : EPI; }
template <int EPI>
struct EpiPlan {
#ifdef MTK_UMMA_COAL_ALL
    static constexpr bool coal = MTK_UMMA_COAL && EPI >= 0;
#else
    static constexpr bool coal = MTK_UMMA_COAL && (EPI == (int)Epi::kBias || EPI == (int)Epi::kBiasRelu ||
                                                   EPI == (int)Epi::kStore || EPI == kEpiMaskNoAdd ||
                                                   EPI == (int)Epi::kSgd || EPI == (int)Epi::kMmdGradW);
#endif
    static constexpr int ls = coal ? 4 : 5;  // load stages
    static constexpr int tile_bytes = coal ? 32 * 32 * 4 : 0;
    static constexpr int roww_bytes = coal ? 32 * 4 : 0;
    static constexpr int smem = ls * LOAD_BYTES + LO * LO_BYTES + NUM_EPI_WARPS * (tile_bytes + roww_bytes) +
                                1024 /*align*/ + 256 /*barriers*/;
    static_assert(smem <= 232448, "umma smem plan");
};
constexpr int NUM_CONV_WARPS = 4;
constexpr int EPI_W0 = 2, CONV_W0 = EPI_W0 + NUM_EPI_WARPS;
constexpr int NUM_THREADS = 32 * (CONV_W0 + NUM_CONV_WARPS);

struct UmmaParams {
    CUtensorMap a, b;  // 3-D fp32 maps, coords (inner, outer, g)
    CUtensorMap b64;   // K-major B with 64-row boxes (half tiles)
    int G, M, N, K;
    int nfull, nhalf;  // work items: nfull full tiles, then nhalf half tiles (N / 2)
    int epi;           // Epi value
    float* C;
    long long c_gs, ldc;
    const float* bias;
    long long bias_gs;
    const float* add;
    const float* mask;
    float lr;
    float* grad_out;
    float* colsum;     // kMask: per-32-row-block column sums of C, [G][ceil(M/32)][N], or null
    const float* rowvec;  // kMmdGrad: [G][M]
    float scale;          // kMmdGrad
    int zmask;            // kMmdGrad: C *= (add > 0) (the fused head DX)
    CUtensorMap b2;       // B rows k >= ksplit come from here (row k - ksplit); ksplit % 32 == 0
    int ksplit;           // K if there is no second B operand
    uint32_t* mbits;      // ReLU mask bits (kBiasRelu writes, kMask reads), [G][M][mb_ld]
    long long mb_gs, mb_ld;
    int* flags;
    unsigned long long* trace;  // diagnostics: timestamps of CTA (0,0,0)
    int ediag;                  // diagnostics (MTK_UMMA_EPI_DIAG): 1 = TMEM reads only, 2 = no global traffic
    int sepc_kf;                // SEPC: k-blocks whose corrections share the main accumulator (see below)
    int prefetch;               // A/B (MTK_UMMA_PREFETCH=1): producer-side L2 prefetch of epilogue operands
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// TMA for one operand tile of 128 (m or n) x 32 (k) into `dst`.
//   K-major: one box (32 k, 128 rows).   MN-major: four boxes (32 mn, 32 k).
template <int MN>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                             int r0, int k0, int g, int rows = 128) {
    if (MN) {
        for (int j = 0; j < rows / 32; ++j) tma_load_3d(dst + j * 4096, map, bar, r0 + 32 * j, k0, g);
    } else {
        tma_load_3d(dst, map, bar, k0, r0, g);  // the map's box carries the row count
    }
}

// work item w -> tile coordinates; items [0, nfull) are full tiles, the rest
// split the last partial wave's tiles into two N halves (half = 0 / 1)
struct Item {
    int g, mt, nt, half;  // half = -1 for a full tile
};
__device__ __forceinline__ Item decode_item(const UmmaParams& p, int w, int tiles_m, int tiles_n) {
    int t = w, half = -1;
    if (w >= p.nfull) {
        const int h = w - p.nfull;
        t = p.nfull + (h >> 1);
        half = h & 1;
    }
    Item it;
    it.nt = t % tiles_n;
    it.mt = (t / tiles_n) % tiles_m;
    it.g = t / (tiles_n * tiles_m);
    it.half = half;
    return it;
}

// lo = rna_tf32(x - trunc_tf32(x)) over the two fp32 tiles of a load stage
// (the tiles stay untouched as the hi operands).  The transform is
// elementwise, so it ignores the swizzle: lo sits at the same offset.
__device__ __forceinline__ void convert_stage(uint8_t* st, uint8_t* lo, int t) {
    constexpr int NT = 32 * NUM_CONV_WARPS;
    const uint32_t src = smem_u32(st) + 16 * t, dst = smem_u32(lo) + 16 * t;
    float4 x[2048 / NT];
#pragma unroll
    for (int j = 0; j < 2048 / NT; ++j) x[j] = lds128(src + 16 * NT * j);
#pragma unroll
    for (int j = 0; j < 2048 / NT; ++j) {
        float4 l;
        l.x = tf32_rna(x[j].x - tf32_trunc(x[j].x));
        l.y = tf32_rna(x[j].y - tf32_trunc(x[j].y));
        l.z = tf32_rna(x[j].z - tf32_trunc(x[j].z));
        l.w = tf32_rna(x[j].w - tf32_trunc(x[j].w));
        sts128(dst + 16 * NT * j, l);
    }
}

// 3 MMAs per 8-wide k step over one stage
template <int A_MN, int B_MN, bool PAIR>
__device__ __forceinline__ void mma_stage(uint32_t tmem, uint32_t tcorr, uint32_t base, uint32_t lo,
                                          uint32_t idesc, bool first) {
    constexpr uint32_t a_lbo = A_MN ? 4096 : 16, b_lbo = B_MN ? 4096 : 16;
    constexpr uint32_t a_sbo = A_MN ? 512 : 1024, b_sbo = B_MN ? 512 : 1024;
    constexpr uint32_t a_lay = A_MN ? 1 : 2, b_lay = B_MN ? 1 : 2;
#pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
        // K-major: +32 B per 8-element k step inside the 128-B swizzle row
        // MN-major: +1024 B per 8 k rows (two 32-B-atom swizzle atoms)
        const uint32_t aoff = A_MN ? kk * 1024 : kk * 32;
        const uint32_t boff = B_MN ? kk * 1024 : kk * 32;
        const uint64_t a32 = smem_desc(base + aoff, a_lbo, a_sbo, a_lay);
        const uint64_t alo = smem_desc(lo + aoff, a_lbo, a_sbo, a_lay);
        const uint64_t b32 = smem_desc(base + TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
        const uint64_t blo = smem_desc(lo + TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
        const uint32_t acc0 = (first && kk == 0) ? 0u : 1u;
        // tcorr == tmem: one accumulator; else the corrections have their own
        const uint32_t accm = tcorr == tmem ? 1u : acc0;
        if (PAIR) {
            mma_tf32_2sm(tcorr, a32, blo, idesc, acc0);
            mma_tf32_2sm(tcorr, alo, b32, idesc, 1u);
            mma_tf32_2sm(tmem, a32, b32, idesc, accm);
        } else {
            mma_tf32(tcorr, a32, blo, idesc, acc0);
            mma_tf32(tcorr, alo, b32, idesc, 1u);
            mma_tf32(tmem, a32, b32, idesc, accm);
        }
    }
}

// SEPC, separate accumulators from k-block kf on: the corrections into tcorr
// (the first of them initialising it when corr_first), the main product into
// tmem (initialising it when main_first: kf = 0)
template <int A_MN, int B_MN, bool PAIR>
__device__ __forceinline__ void mma_stage_sep(uint32_t tmem, uint32_t tcorr, uint32_t base, uint32_t lo,
                                              uint32_t idesc, bool corr_first, bool main_first) {
    constexpr uint32_t a_lbo = A_MN ? 4096 : 16, b_lbo = B_MN ? 4096 : 16;
    constexpr uint32_t a_sbo = A_MN ? 512 : 1024, b_sbo = B_MN ? 512 : 1024;
    constexpr uint32_t a_lay = A_MN ? 1 : 2, b_lay = B_MN ? 1 : 2;
#pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
        const uint32_t aoff = A_MN ? kk * 1024 : kk * 32;
        const uint32_t boff = B_MN ? kk * 1024 : kk * 32;
        const uint64_t a32 = smem_desc(base + aoff, a_lbo, a_sbo, a_lay);
        const uint64_t alo = smem_desc(lo + aoff, a_lbo, a_sbo, a_lay);
        const uint64_t b32 = smem_desc(base + TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
        const uint64_t blo = smem_desc(lo + TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
        const uint32_t accc = (corr_first && kk == 0) ? 0u : 1u;
        const uint32_t accm = (main_first && kk == 0) ? 0u : 1u;
        if (PAIR) {
            mma_tf32_2sm(tcorr, a32, blo, idesc, accc);
            mma_tf32_2sm(tcorr, alo, b32, idesc, 1u);
            mma_tf32_2sm(tmem, a32, b32, idesc, accm);
        } else {
            mma_tf32(tcorr, a32, blo, idesc, accc);
            mma_tf32(tcorr, alo, b32, idesc, 1u);
            mma_tf32(tmem, a32, b32, idesc, accm);
        }
    }
}

// SEPC phase 1 of a tile's epilogue: this warp's chunks of main += corr, in
// TMEM (the corrections' region is then free for the next tile's main)
__device__ __forceinline__ void sepc_fold(uint32_t tmain, uint32_t tcorr, int q, int c0, int c1, int n0, int N) {
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        if (n0 + c * 32 >= N) break;  // warp-uniform
        const uint32_t lq = (uint32_t)(32 * q) << 16;
        float v[32];
        tmem_ld_32x32(tmain + lq + (uint32_t)(c * 32), v);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float w[8];
            tmem_ld_32x8(tcorr + lq + (uint32_t)(c * 32 + 8 * h), w);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[8 * h + j] += w[j];
        }
        tmem_st_32x32(tmain + lq + (uint32_t)(c * 32), v);
    }
    tmem_st_wait();
}

// 32 column values per lane (lane = row) -> lane j holds the sum over the
// warp's 32 rows of column j.  Five butterfly steps, fixed order.
__device__ __forceinline__ float column_sums_32(float (&v)[32], int lane) {
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

// TMEM accumulator -> fused epilogue -> fp32 C in HBM.  Thread = row (TMEM
// lane); this warp covers the 32-column chunks [c0, c1).  Per chunk every
// global operand load (bias | mask, add | master weight) is issued before the
// TMEM read, so a chunk costs one memory round trip.  No shared memory: the
// mainloop running on the other accumulator saturates the smem port.
template <bool SEPC, int EPI>
__device__ __forceinline__ void epilogue_rows(const UmmaParams& p, uint32_t tmem, uint32_t tcorr, int q,
                                              int lane, int g, int m0, int n0, int c0, int c1,
                                              unsigned long long* etr = nullptr) {
    const int mw = m0 + 32 * q;
    const int m = mw + lane;
    const bool row_ok = m < p.M;
    const long long rowbase = (long long)g * p.c_gs + (long long)m * p.ldc;
    const int epi = EPI >= 0 ? epi_kind<EPI>() : p.epi;  // compile-time for the specialised launches
    bool bad = false;
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        const int nb = n0 + c * 32;
        if (nb >= p.N) break;  // warp-uniform
        const bool vec = row_ok && (nb + 32 <= p.N) && ((rowbase + nb) % 4 == 0);
        float4 o1[8], o2[8];  // prefetched operands of this chunk
        if (vec) {
            const float* s1 = nullptr;
            const float* s2 = nullptr;
            if (epi == (int)Epi::kBias || epi == (int)Epi::kBiasRelu) s1 = p.bias + g * p.bias_gs + nb;
            else if (epi == (int)Epi::kMask) {
                s1 = p.mbits ? nullptr : p.mask + rowbase + nb;
                s2 = p.add ? p.add + rowbase + nb : nullptr;
            }
            else if (epi == (int)Epi::kSgd) s1 = p.C + rowbase + nb;
            else if (epi == (int)Epi::kMmdGrad) s1 = p.add + rowbase + nb;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                o1[j] = s1 ? *reinterpret_cast<const float4*>(s1 + 4 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
                o2[j] = s2 ? *reinterpret_cast<const float4*>(s2 + 4 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const uint32_t mword = (p.mbits && row_ok && (epi == (int)Epi::kMask || epi == (int)Epi::kMmdGradW))
                                   ? p.mbits[(long long)g * p.mb_gs + (long long)m * p.mb_ld + nb / 32]
                                   : 0u;
        if (etr && lane == 0) etr[4 * (c - c0)] = gtime();
        float v[32];
        tmem_ld_32x32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 32), v);
        if (etr && lane == 0) etr[4 * (c - c0) + 1] = gtime();
        if (SEPC) {  // main + corrections, one fp32 add (8 columns at a time: registers)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float w[8];
                tmem_ld_32x8(tcorr + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 32 + 8 * h), w);
#pragma unroll
                for (int j = 0; j < 8; ++j) v[8 * h + j] += w[j];
            }
        }
        if (vec) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const long long idx = rowbase + nb + 4 * j;
                float4 x = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                if (epi == (int)Epi::kBias || epi == (int)Epi::kBiasRelu) {
                    x.x += o1[j].x;
                    x.y += o1[j].y;
                    x.z += o1[j].z;
                    x.w += o1[j].w;
                    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                    if (epi == (int)Epi::kBiasRelu) {
                        x.x = x.x > 0.f ? x.x : 0.f;
                        x.y = x.y > 0.f ? x.y : 0.f;
                        x.z = x.z > 0.f ? x.z : 0.f;
                        x.w = x.w > 0.f ? x.w : 0.f;
                    }
                } else if (epi == (int)Epi::kMask) {
                    if (p.add) {
                        x.x = o2[j].x + x.x;
                        x.y = o2[j].y + x.y;
                        x.z = o2[j].z + x.z;
                        x.w = o2[j].w + x.w;
                    }
                    if (p.mbits) {
                        const uint32_t mb = mword >> (4 * j);
                        x.x = (mb & 1u) ? x.x : 0.f;
                        x.y = (mb & 2u) ? x.y : 0.f;
                        x.z = (mb & 4u) ? x.z : 0.f;
                        x.w = (mb & 8u) ? x.w : 0.f;
                    } else {
                        x.x = o1[j].x > 0.f ? x.x : 0.f;
                        x.y = o1[j].y > 0.f ? x.y : 0.f;
                        x.z = o1[j].z > 0.f ? x.z : 0.f;
                        x.w = o1[j].w > 0.f ? x.w : 0.f;
                    }
                } else if (epi == (int)Epi::kMmdGradW) {  // -scale * (W'.Z), the mask bits of z
                    x.x = p.scale * -x.x;
                    x.y = p.scale * -x.y;
                    x.z = p.scale * -x.z;
                    x.w = p.scale * -x.w;
                    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                    if (p.mbits) {
                        const uint32_t mb = mword >> (4 * j);
                        x.x = (mb & 1u) ? x.x : 0.f;
                        x.y = (mb & 2u) ? x.y : 0.f;
                        x.z = (mb & 4u) ? x.z : 0.f;
                        x.w = (mb & 8u) ? x.w : 0.f;
                    }
                } else if (epi == (int)Epi::kMmdGrad) {  // o1 = z row, rowvec = Wsum
                    const float rv = p.rowvec[(long long)g * p.M + m];
                    x.x = p.scale * fmaf(o1[j].x, rv, -x.x);
                    x.y = p.scale * fmaf(o1[j].y, rv, -x.y);
                    x.z = p.scale * fmaf(o1[j].z, rv, -x.z);
                    x.w = p.scale * fmaf(o1[j].w, rv, -x.w);
                    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                    if (p.zmask) {  // fused head DX: the ReLU mask of z (= h, tape.hpp:349)
                        x.x = o1[j].x > 0.f ? x.x : 0.f;
                        x.y = o1[j].y > 0.f ? x.y : 0.f;
                        x.z = o1[j].z > 0.f ? x.z : 0.f;
                        x.w = o1[j].w > 0.f ? x.w : 0.f;
                    }
                } else if (epi == (int)Epi::kSgd) {  // C is the fp32 master weight
                    if (p.grad_out) *reinterpret_cast<float4*>(p.grad_out + idx) = x;
                    x.x = sgd_update(o1[j].x, x.x, p.lr);
                    x.y = sgd_update(o1[j].y, x.y, p.lr);
                    x.z = sgd_update(o1[j].z, x.z, p.lr);
                    x.w = sgd_update(o1[j].w, x.w, p.lr);
                    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                }
                if (epi != (int)Epi::kNone) *reinterpret_cast<float4*>(p.C + idx) = x;
                v[4 * j] = x.x;  // kept for the column sums
                v[4 * j + 1] = x.y;
                v[4 * j + 2] = x.z;
                v[4 * j + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = nb + j;
                float x = v[j];
                if (row_ok && n < p.N) {
                    const long long idx = rowbase + n;
                    if (epi == (int)Epi::kBias || epi == (int)Epi::kBiasRelu) {
                        x += p.bias[g * p.bias_gs + n];
                        bad |= !isfinite(x);
                        if (epi == (int)Epi::kBiasRelu) x = x > 0.f ? x : 0.f;
                    } else if (epi == (int)Epi::kMask) {
                        if (p.add) x = p.add[idx] + x;
                        x = (p.mbits ? ((mword >> j) & 1u) != 0 : p.mask[idx] > 0.f) ? x : 0.f;
                    } else if (epi == (int)Epi::kMmdGradW) {
                        x = p.scale * -x;
                        bad |= !isfinite(x);
                        if (p.mbits && !((mword >> j) & 1u)) x = 0.f;
                    } else if (epi == (int)Epi::kMmdGrad) {
                        const float z = p.add[idx];
                        x = p.scale * fmaf(z, p.rowvec[(long long)g * p.M + m], -x);
                        bad |= !isfinite(x);
                        if (p.zmask) x = z > 0.f ? x : 0.f;
                    } else if (epi == (int)Epi::kSgd) {
                        if (p.grad_out) p.grad_out[idx] = x;
                        x = sgd_update(p.C[idx], x, p.lr);
                        bad |= !isfinite(x);
                    }
                    if (epi != (int)Epi::kNone) p.C[idx] = x;
                } else {
                    x = 0.f;
                }
                v[j] = x;
            }
        }
        if (epi == (int)Epi::kBiasRelu && p.mbits && row_ok) {  // the ReLU mask of this chunk as bits
            uint32_t word = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) word |= (v[j] > 0.f ? 1u : 0u) << j;
            p.mbits[(long long)g * p.mb_gs + (long long)m * p.mb_ld + nb / 32] = word;
        }
        if (etr && lane == 0) etr[4 * (c - c0) + 2] = gtime();
        if (p.colsum && (epi == (int)Epi::kMask || epi == (int)Epi::kMmdGrad || epi == (int)Epi::kMmdGradW) &&
            mw < p.M) {
            // per-32-row-block column sums of the stored values (next layer's db)
            const float cs = column_sums_32(v, lane);
            if (nb + lane < p.N) {
                const int nrb = (p.M + 31) / 32;
                p.colsum[((long long)g * nrb + mw / 32) * p.N + nb + lane] = cs;
            }
        }
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

// one ragged / misaligned chunk on the thread-per-row path, out of line (its
// registers stay out of the hot loop's allocation)
template <bool SEPC, int EPI>
__device__ __noinline__ void epilogue_rows_cold(const UmmaParams& p, uint32_t tmem, uint32_t tcorr, int q, int lane,
                                                int g, int m0, int n0, int c) {
    epilogue_rows<SEPC, EPI>(p, tmem, tcorr, q, lane, g, m0, n0, c, c + 1);
}

// Operands of the coalesced epilogue (below): per pass i the float4 of row
// mw + 4i + lane/8 at columns ncol..+3 (add | master weight | z), per row
// (thread = row) the chunk's mask word or row scale, the bias columns.  They
// are loaded once the chunk's accumulator is staged, in groups of passes
// (preloading a whole chunk, the next chunk's, or the first chunk's before
// the accumulator wait spilled at 128 registers and measured slower).
template <int EPI>
__device__ __forceinline__ float4 epi_operand(const UmmaParams& p, int g, int m, int ncol) {
    const long long idx = (long long)g * p.c_gs + (long long)m * p.ldc + ncol;
    if (m < p.M && p.ediag == 0) {
        if (EPI == kEpiMaskNoAdd) {
        } else if (EPI == (int)Epi::kMask) {
            if (p.add) return *reinterpret_cast<const float4*>(p.add + idx);
        } else if (EPI == (int)Epi::kSgd) {
            return *reinterpret_cast<const float4*>(p.C + idx);
        } else if (EPI == (int)Epi::kMmdGrad) {
            return *reinterpret_cast<const float4*>(p.add + idx);
        }
    }
    return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int EPI>
__device__ __forceinline__ uint32_t epi_rowword(const UmmaParams& p, int g, int m, int nb) {
    if (m < p.M) {
        if ((epi_kind<EPI>() == (int)Epi::kMask || EPI == (int)Epi::kMmdGradW) && p.mbits) return p.mbits[(long long)g * p.mb_gs + (long long)m * p.mb_ld + nb / 32];
        if (EPI == (int)Epi::kMmdGrad) return __float_as_uint(p.rowvec[(long long)g * p.M + m]);
    }
    return 0u;
}
template <int EPI>
__device__ __forceinline__ float4 epi_bias(const UmmaParams& p, int g, int ncol) {
    if (EPI == (int)Epi::kBias || EPI == (int)Epi::kBiasRelu)
        return *reinterpret_cast<const float4*>(p.bias + g * p.bias_gs + ncol);
    return make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ bool epi_fast_chunk(const UmmaParams& p, int nb) {
    return (p.c_gs % 4 == 0) && (p.ldc % 4 == 0) && nb + 32 <= p.N;
}
// The same epilogue through a 32 x 32 shared-memory tile per warp: the TMEM
// rows (thread = row) are written to the tile, __syncwarp, and read back as
// 8 passes of 4 rows x 32 columns (lane = row 4i + lane/8, columns 4 (lane%8)
// .. +3), so every global operand load and output store of the chunk covers
// whole 128-B row segments (thread = row stores touched 32 lines per
// instruction: the L1 then processed 32 requests for 512 B, and the epilogue,
// not the MMA, paced the GEMM).  16-B granules are XOR-swizzled by row
// (granule j of row r at j ^ (r & 7)): conflict-free row writes and pass reads.
// Column sums of a 32-row block: 8 rows per lane in pass order, then lanes
// xor 8 and xor 16 (fixed order).  Ragged or misaligned chunks take the
// thread-per-row path.
template <bool SEPC, int EPI>
__device__ __forceinline__ void epilogue_coalesced(const UmmaParams& p, uint32_t tmem, uint32_t tcorr, int q,
                                                   int lane, int g, int m0, int n0, int c0, int c1, uint32_t tile,
                                                   uint32_t roww, unsigned long long* etr = nullptr) {
    constexpr int E = epi_kind<EPI>();  // the arithmetic kind (kEpiMaskNoAdd: kMask without an addend)
    constexpr bool kAdd = EPI != kEpiMaskNoAdd;
    constexpr bool kBiasE = E == (int)Epi::kBias || E == (int)Epi::kBiasRelu;
    // the mask bits applied in the row layout (no addend to add first)
    constexpr bool kRowMask = EPI == kEpiMaskNoAdd || E == (int)Epi::kMmdGradW;
    const int mw = m0 + 32 * q;
    const int gq = lane & 7, rsub = lane >> 3;
    const bool aligned = (p.c_gs % 4 == 0) && (p.ldc % 4 == 0);
    const uint32_t wrow = tile + (uint32_t)lane * 128u;
    bool bad = false;
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        const int nb = n0 + c * 32;
        if (nb >= p.N) break;  // warp-uniform
        if (!aligned || nb + 32 > p.N) {
            epilogue_rows_cold<SEPC, EPI>(p, tmem, tcorr, q, lane, g, m0, n0, c);  // (maps EPI itself)
            continue;
        }
        const int ncol = nb + 4 * gq;  // this lane's first column
        const uint32_t rw = epi_rowword<EPI>(p, g, mw + lane, nb);
        if (etr && lane == 0) etr[4 * (c - c0)] = gtime();
        {
            float v[32];
            tmem_ld_32x32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 32), v);
            if (etr && lane == 0) etr[4 * (c - c0) + 1] = gtime();
            if (SEPC) {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    float w[8];
                    tmem_ld_32x8(tcorr + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 32 + 8 * h), w);
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[8 * h + j] += w[j];
                }
            }
            if (kBiasE) {  // bias (+ ReLU) and the mask bits in the row layout: no shuffles
                const float4* bp = reinterpret_cast<const float4*>(p.bias + g * p.bias_gs + nb);
                const int m = mw + lane;
                uint32_t word = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 b4 = bp[j];  // warp-uniform: broadcast
                    v[4 * j] += b4.x;
                    v[4 * j + 1] += b4.y;
                    v[4 * j + 2] += b4.z;
                    v[4 * j + 3] += b4.w;
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (m < p.M) bad |= !isfinite(v[j]);
                    if (E == (int)Epi::kBiasRelu) v[j] = v[j] > 0.f ? v[j] : 0.f;
                    word |= (v[j] > 0.f ? 1u : 0u) << j;
                }
                if (E == (int)Epi::kBiasRelu && p.mbits && m < p.M && p.ediag == 0)
                    p.mbits[(long long)g * p.mb_gs + (long long)m * p.mb_ld + nb / 32] = word;
            }
            if (kRowMask) {  // mask (and scale) in the row layout: the row's word is this thread's
                const bool mrow = mw + lane < p.M;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (E == (int)Epi::kMmdGradW) {
                        v[j] = p.scale * -v[j];
                        if (mrow) bad |= !isfinite(v[j]);
                    }
                    if (p.mbits && !((rw >> j) & 1u)) v[j] = 0.f;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                sts128(wrow + (uint32_t)((j ^ (lane & 7)) * 16),
                       make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
            if (p.ediag == 1) {
                float t = 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j) t += v[j];
                bad |= t == 12345.f;
                continue;
            }
            if ((E == (int)Epi::kMask || E == (int)Epi::kMmdGrad) && !kRowMask) sts32(roww + 4u * lane, rw);
        }
        __syncwarp();
        // the chunk's operands, issued once the accumulator registers are free,
        // in groups of GS passes (8 preloaded float4s spilled at 128 registers)
        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
        constexpr int GS = (E == (int)Epi::kMmdGrad || E == (int)Epi::kMask) ? 2 : 4;  // passes per operand group
#pragma unroll
        for (int hp = 0; hp < 8 / GS; ++hp) {
        float4 oh[GS];
#pragma unroll
        for (int ii = 0; ii < GS; ++ii) oh[ii] = epi_operand<EPI>(p, g, mw + 4 * (GS * hp + ii) + rsub, ncol);
#pragma unroll
        for (int ii = 0; ii < GS; ++ii) {
            const int i = GS * hp + ii;
            const int r = 4 * i + rsub;
            const int m = mw + r;
            float4 x = lds128(tile + (uint32_t)(r * 128 + ((gq ^ (r & 7)) * 16)));
            const float4 op = oh[ii];
            const uint32_t rword = ((E == (int)Epi::kMask || E == (int)Epi::kMmdGrad) && !kRowMask) ? lds32(roww + 4u * r) : 0u;
            const bool ok = m < p.M && p.ediag != 2;
            const long long idx = (long long)g * p.c_gs + (long long)m * p.ldc + ncol;
            if (kBiasE) {  // applied in the row layout above
            } else if (kRowMask) {  // applied in the row layout above
            } else if (E == (int)Epi::kMask) {
                if (kAdd && p.add) {
                    x.x = op.x + x.x;
                    x.y = op.y + x.y;
                    x.z = op.z + x.z;
                    x.w = op.w + x.w;
                }
                if (p.mbits) {
                    const uint32_t mb = rword >> (4 * gq);
                    x.x = (mb & 1u) ? x.x : 0.f;
                    x.y = (mb & 2u) ? x.y : 0.f;
                    x.z = (mb & 4u) ? x.z : 0.f;
                    x.w = (mb & 8u) ? x.w : 0.f;
                } else {
                    const float4 mk = ok ? *reinterpret_cast<const float4*>(p.mask + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
                    x.x = mk.x > 0.f ? x.x : 0.f;
                    x.y = mk.y > 0.f ? x.y : 0.f;
                    x.z = mk.z > 0.f ? x.z : 0.f;
                    x.w = mk.w > 0.f ? x.w : 0.f;
                }
            } else if (E == (int)Epi::kMmdGrad) {
                const float rv = __uint_as_float(rword);
                x.x = p.scale * fmaf(op.x, rv, -x.x);
                x.y = p.scale * fmaf(op.y, rv, -x.y);
                x.z = p.scale * fmaf(op.z, rv, -x.z);
                x.w = p.scale * fmaf(op.w, rv, -x.w);
                if (ok) bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                if (p.zmask) {
                    x.x = op.x > 0.f ? x.x : 0.f;
                    x.y = op.y > 0.f ? x.y : 0.f;
                    x.z = op.z > 0.f ? x.z : 0.f;
                    x.w = op.w > 0.f ? x.w : 0.f;
                }
            } else if (E == (int)Epi::kSgd) {
                if (ok && p.grad_out) *reinterpret_cast<float4*>(p.grad_out + idx) = x;
                x.x = sgd_update(op.x, x.x, p.lr);
                x.y = sgd_update(op.y, x.y, p.lr);
                x.z = sgd_update(op.z, x.z, p.lr);
                x.w = sgd_update(op.w, x.w, p.lr);
                if (ok) bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
            }
            if (!ok) x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (E != (int)Epi::kNone && ok) *reinterpret_cast<float4*>(p.C + idx) = x;
            cs.x += x.x;
            cs.y += x.y;
            cs.z += x.z;
            cs.w += x.w;
        }
        }  // halves
        __syncwarp();  // the tile is rewritten by the next chunk
        if (etr && lane == 0) etr[4 * (c - c0) + 2] = gtime();
        if (p.colsum && (E == (int)Epi::kMask || E == (int)Epi::kMmdGrad || E == (int)Epi::kMmdGradW) && mw < p.M) {
            // per-32-row-block column sums of the stored values (next layer's db)
#pragma unroll
            for (int o = 8; o <= 16; o <<= 1) {
                cs.x += __shfl_xor_sync(0xffffffffu, cs.x, o);
                cs.y += __shfl_xor_sync(0xffffffffu, cs.y, o);
                cs.z += __shfl_xor_sync(0xffffffffu, cs.z, o);
                cs.w += __shfl_xor_sync(0xffffffffu, cs.w, o);
            }
            if (rsub == 0) {
                const int nrb = (p.M + 31) / 32;
                *reinterpret_cast<float4*>(p.colsum + ((long long)g * nrb + mw / 32) * p.N + ncol) = cs;
            }
        }
    }
    if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

// L2 prefetch of the global operands the epilogue of a tile will read (its
// 128 rows of the master weight, or the ReLU mask and addend), issued by the
// producer warp a few stages before the tile's mainloop ends.
__device__ __forceinline__ void prefetch_epilogue_rows(const UmmaParams& p, int g, int m0, int n0,
                                                       int ncols, int lane) {
    const float* src[2] = {nullptr, nullptr};
    if (p.epi == (int)Epi::kSgd) src[0] = p.C;
    else if (p.epi == (int)Epi::kMask) { src[0] = p.mask; src[1] = p.add; }
    else if (p.epi == (int)Epi::kMmdGrad) src[0] = p.add;
    if (!src[0]) return;
    const int n1 = min(n0 + ncols, p.N);
    if (n1 <= n0) return;
    const uint32_t bytes = (uint32_t)(n1 - n0) * 4;
    if (bytes % 16) return;
    for (int rr = lane; rr < 128; rr += 32) {
        const int m = m0 + rr;
        if (m >= p.M) break;
        for (int i = 0; i < 2; ++i) {
            if (!src[i]) continue;
            const float* a = src[i] + (long long)g * p.c_gs + (long long)m * p.ldc + n0;
            if (reinterpret_cast<uintptr_t>(a) & 15) continue;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
        }
    }
}

template <int A_MN, int B_MN, bool PAIR, bool SEPC, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1) umma_kernel(const __grid_constant__ UmmaParams p) {
    constexpr int TN = PAIR ? 256 : 128;  // accumulator columns per tile
    constexpr uint32_t TMEM_COLS = 2 * TN;  // double-buffered accumulator
    constexpr uint32_t NCTA = PAIR ? 2 : 1;
    constexpr int LS = EpiPlan<EPI>::ls;
    constexpr int EPI_TILE_BYTES = EpiPlan<EPI>::tile_bytes, EPI_ROWW_BYTES = EpiPlan<EPI>::roww_bytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* lo_ring = smem + LS * LOAD_BYTES;
    uint8_t* epi_tiles = lo_ring + LO * LO_BYTES;  // [NUM_EPI_WARPS][32][32] fp32
    uint8_t* epi_rowws = epi_tiles + NUM_EPI_WARPS * EPI_TILE_BYTES;  // [NUM_EPI_WARPS][32] u32
    uint64_t* full = reinterpret_cast<uint64_t*>(epi_rowws + NUM_EPI_WARPS * EPI_ROWW_BYTES);
    uint64_t* empty = full + LS;
    uint64_t* conv = empty + LS;
    uint64_t* lofree = conv + LO;
    uint64_t* acc_full = lofree + LO;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_rank() : 0;
    const int tiles_m = PAIR ? (p.M + 255) / 256 : (p.M + 127) / 128;
    const int tiles_n = (p.N + TN - 1) / TN;
    const int nitems = p.nfull + p.nhalf;
    const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ncl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int nk = (p.K + BK - 1) / BK;
    unsigned long long* tr = (p.trace && blockIdx.x == 0) ? p.trace : nullptr;
    if (p.trace && threadIdx.x == 0 && blockIdx.x < 400) p.trace[4000 + 2 * blockIdx.x] = gtime();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.a);
        tma_prefetch(&p.b);
        if (p.ksplit < p.K) tma_prefetch(&p.b2);
        if (p.nhalf && !B_MN) tma_prefetch(&p.b64);
        for (int s = 0; s < LS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < LO; ++s) {
            mbar_init(&conv[s], NCTA * NUM_CONV_WARPS);  // one arrival per converter warp
            mbar_init(&lofree[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], NCTA * NUM_EPI_WARPS);  // one arrival per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        if (PAIR) tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
        else tmem_alloc<TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    if (PAIR) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the prologue above overlapped the predecessor's tail (PDL launch); its
    // outputs are read from here on
    pdl_wait();

    // Producer and MMA warps run their loops converged (all lanes wait, lane 0
    // issues); see k_mmd_tc.cu for the divergent-lane stall this avoids.
    if (warp == 0) {
        {
            // ---------------- TMA producer ----------------
            uint32_t it = 0;
            for (int w = cid; w < nitems; w += ncl) {
                const Item im = decode_item(p, w, tiles_m, tiles_n);
                const int g = im.g;
                const int m0 = PAIR ? im.mt * 256 + (int)rank * 128 : im.mt * 128;
                const int ncols = im.half < 0 ? TN : TN / 2;
                const int n0 = im.nt * TN + (im.half > 0 ? TN / 2 : 0);
                const int brows = ncols / (int)NCTA;          // B columns staged by this CTA
                const int nb0 = n0 + (int)rank * brows;
                const uint32_t bytes = TILE_BYTES + (uint32_t)brows * BK * 4;
                const CUtensorMap* bmap = (im.half >= 0 && !B_MN) ? &p.b64 : &p.b;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % LS;
                    // optional L2 prefetch of the epilogue's per-element operands (off by
                    // default: the 128 bulk prefetches per tile queue ahead of the next
                    // tile's loads in the TMA unit -- measured ~5 us per tile boundary;
                    // without them DX 60.9 -> 48.2 us, DW 209.5 -> 202.3 us per C2 step)
                    constexpr bool kNeedsOps = EPI < 0 || EPI == (int)Epi::kSgd || EPI == (int)Epi::kMask ||
                                               EPI == (int)Epi::kMmdGrad;
                    if (kNeedsOps && p.prefetch && kb == (nk > 8 ? nk - 8 : 0))
                        prefetch_epilogue_rows(p, g, m0, n0, ncols, lane);
                    mbar_wait(&empty[s], ((it / LS) & 1) ^ 1);
                    uint8_t* st = smem + s * LOAD_BYTES;
                    if (lane == 0) {
                        if (tr && it < 1000) tr[it] = gtime();
                        mbar_expect_tx(&full[s], bytes);
                        load_operand<A_MN>(st, &p.a, &full[s], m0, kb * BK, g);
                        if (kb * BK < p.ksplit)
                            load_operand<B_MN>(st + TILE_BYTES, bmap, &full[s], nb0, kb * BK, g, brows);
                        else  // the second B operand (p.b2, N-major)
                            load_operand<B_MN>(st + TILE_BYTES, &p.b2, &full[s], nb0, kb * BK - p.ksplit, g, brows);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA, one thread) ----------------
        constexpr uint32_t idesc_full = idesc_tf32(PAIR ? 256 : 128, TN, A_MN, B_MN);
        constexpr uint32_t idesc_half = idesc_tf32(PAIR ? 256 : 128, TN / 2, A_MN, B_MN);
        if (rank == 0) {
            uint32_t it = 0, tl = 0;
            for (int w = cid; w < nitems; w += ncl, ++tl) {
                const uint32_t idesc = w < p.nfull ? idesc_full : idesc_half;
                // Non-SEPC: double-buffered accumulator (region b = tile parity,
                // freed every second tile).  SEPC: tile t's main accumulator is
                // region t & 1, its corrections region (t & 1) ^ 1; each region is
                // freed once per tile (the corrections' after the epilogue folds
                // them into main, main after the epilogue proper), so tile t
                // waits for t completions of each.  The first kf k-blocks'
                // corrections go into main (the corrections' region is still being
                // read by the previous tile's epilogue); their accumulation drift
                // is that of a small partial sum.
                const uint32_t b = tl & 1;
                const uint32_t acc = tmem + b * TN;
                const uint32_t corr = tmem + (b ^ 1) * TN;
                const int kf = p.sepc_kf;
                mbar_wait(&acc_empty[b], SEPC ? ((tl + 1) & 1) : (((tl >> 1) & 1) ^ 1));
                tc_fence_after();
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % LS, l = it % LO;
                    mbar_wait(&conv[l], (it / LO) & 1);
                    if (SEPC && kb == kf) mbar_wait(&acc_empty[b ^ 1], (tl + 1) & 1);  // corrections' region free
                    tc_fence_after();
                    if (lane == 0) {
                        if (tr && it < 1000) tr[1000 + it] = gtime();
                        if (!SEPC || kb < kf)
                            mma_stage<A_MN, B_MN, PAIR>(acc, acc, smem_u32(smem + s * LOAD_BYTES),
                                                        smem_u32(lo_ring + l * LO_BYTES), idesc, kb == 0);
                        else
                            mma_stage_sep<A_MN, B_MN, PAIR>(acc, corr, smem_u32(smem + s * LOAD_BYTES),
                                                            smem_u32(lo_ring + l * LO_BYTES), idesc, kb == kf,
                                                            kb == 0);
                        if (PAIR) {  // frees the slots in both CTAs
                            mma_commit_2sm(&empty[s], 0x3);
                            mma_commit_2sm(&lofree[l], 0x3);
                        } else {
                            mma_commit(&empty[s]);
                            mma_commit(&lofree[l]);
                        }
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    if (PAIR) mma_commit_2sm(&acc_full[b], 0x3);
                    else mma_commit(&acc_full[b]);
                }
                __syncwarp();
            }
        }
    } else if (warp < CONV_W0) {
        // ---------------- epilogue: own 128 rows x TN columns ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int hsel = (warp - EPI_W0) >> 2;  // which half of the tile's columns
        uint32_t tl = 0;
        for (int w = cid; w < nitems; w += ncl, ++tl) {
            const Item im = decode_item(p, w, tiles_m, tiles_n);
            const int g = im.g;
            const int m0 = PAIR ? im.mt * 256 + (int)rank * 128 : im.mt * 128;
            const int ncols = im.half < 0 ? TN : TN / 2;
            const int n0 = im.nt * TN + (im.half > 0 ? TN / 2 : 0);
            const uint32_t b = tl & 1;
            const int nch = ncols / 32;
            const int ec0 = hsel * (nch / 2), ec1 = (hsel + 1) * (nch / 2);
            mbar_wait(&acc_full[b], (tl >> 1) & 1);
            if (tr && threadIdx.x == 64 && tl < 16) tr[2000 + 2 * tl] = gtime();
            tc_fence_after();
            if (SEPC) {  // phase 1: fold the corrections into main, free their region
                if (p.sepc_kf < nk) sepc_fold(tmem + b * TN, tmem + (b ^ 1) * TN, q, ec0, ec1, n0, p.N);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_remote(&acc_empty[b ^ 1], 0);
                    else mbar_arrive(&acc_empty[b ^ 1]);
                }
            }
            if constexpr (EpiPlan<EPI>::coal)
                epilogue_coalesced<false, EPI>(p, tmem + b * TN, 0u, q, lane, g, m0, n0, ec0, ec1,
                                               smem_u32(epi_tiles + (warp - EPI_W0) * EPI_TILE_BYTES),
                                               smem_u32(epi_rowws + (warp - EPI_W0) * EPI_ROWW_BYTES),
                                               (tr && threadIdx.x == 64 && tl < 4) ? tr + 2100 + 32 * tl : nullptr);
            else
                epilogue_rows<false, EPI>(p, tmem + b * TN, 0u, q, lane, g, m0, n0, ec0, ec1,
                                          (tr && threadIdx.x == 64 && tl < 4) ? tr + 2100 + 32 * tl : nullptr);
            tc_fence_before();
            __syncwarp();
            if (tr && threadIdx.x == 64 && tl < 16) tr[2001 + 2 * tl] = gtime();
            if (lane == 0) {
                if (PAIR) mbar_arrive_remote(&acc_empty[b], 0);
                else mbar_arrive(&acc_empty[b]);
            }
        }
    } else {
        // ---------------- converters ----------------
        const int ct = threadIdx.x - 32 * CONV_W0;
        uint32_t it = 0;
        for (int w = cid; w < nitems; w += ncl) {
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % LS, l = it % LO;
                mbar_wait(&full[s], (it / LS) & 1);
                mbar_wait(&lofree[l], ((it / LO) & 1) ^ 1);
                if (tr && ct == 0 && it < 1000) tr[3000 + it] = gtime();
                convert_stage(smem + s * LOAD_BYTES, lo_ring + l * LO_BYTES, ct);
                fence_proxy_async_smem();  // generic-proxy stores -> tensor-core reads
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_remote(&conv[l], 0);
                    else mbar_arrive(&conv[l]);
                }
            }
        }
    }
    pdl_trigger();  // this CTA's work is issued: the next launch may start its prologue
    tc_fence_before();
    if (PAIR) cluster_sync();
    else __syncthreads();
    if (tr && threadIdx.x == 32) tr[2040] = gtime();
    if (p.trace && threadIdx.x == 32 && blockIdx.x < 400) p.trace[4001 + 2 * blockIdx.x] = gtime();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_2sm<TMEM_COLS>(tmem);
        else tmem_dealloc<TMEM_COLS>(tmem);
    }
}



bool disable_half_tiles();
bool pdl_enabled();

template <int A_MN, int B_MN, bool PAIR, bool SEPC, int EPI>
void launch_variant(UmmaParams p, int G, cudaStream_t s) {
    ensure_smem_attr(reinterpret_cast<const void*>(umma_kernel<A_MN, B_MN, PAIR, SEPC, EPI>), EpiPlan<EPI>::smem);
    const int sms = device_sm_count(current_device());
    const long long ntiles = PAIR ? (long long)((p.M + 255) / 256) * ((p.N + 255) / 256) * G
                                  : (long long)((p.M + 127) / 128) * ((p.N + 127) / 128) * G;
    const long long ncl = std::min<long long>(ntiles, PAIR ? sms / 2 : sms);
    // split the last partial wave into N halves when they fit in one wave
    p.nfull = (int)ntiles;
    p.nhalf = 0;
    const long long rem = ntiles % ncl;
    if (PAIR && ntiles > ncl && rem > 0 && 2 * rem <= ncl && !disable_half_tiles()) {
        p.nfull = (int)(ntiles - rem);
        p.nhalf = (int)(2 * rem);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(PAIR ? 2 * ncl : ncl), 1, 1);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = EpiPlan<EPI>::smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (the kernel calls pdl_wait)
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    MTK_CUDA(cudaLaunchKernelEx(&cfg, umma_kernel<A_MN, B_MN, PAIR, SEPC, EPI>, p));
    count_launch();
}


}  // namespace umma
}  // namespace mtk
