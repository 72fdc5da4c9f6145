// k_umma.cu -- grouped 3xTF32 GEMM on the 5th-gen tensor cores (tcgen05 +
// TMEM + TMA), sm_100a.
//
// C[g] (M x N) = A[g] (M x K) * B[g] (K x N) for G independent models, with
// fp32-level accuracy from three tf32 products per k step:
//     A*B ~= A_hi*B_hi + A_hi*B_lo + A_lo*B_hi        (A = A_hi + A_lo, tf32 parts)
// The hi/lo planes live in HBM next to every fp32 tensor that feeds a GEMM
// (weights, activations, gradients); producers write them in their epilogues.
//
// Replaces, for the bank's dense layers, the reference loops
//   detail::mm_acc (tape.hpp:36-48)    FWD: A = H   (K-major), B = W   (N-major)
//   detail::mm_nt_acc (tape.hpp:50-63) DX:  A = dZ  (K-major), B = W^T (K-major)
//   detail::mm_tn_acc (tape.hpp:65-78) DW:  A = H^T (M-major), B = dZ  (N-major)
// Tile 128 x 128 x 32, 3-stage TMA -> smem ring (128-byte swizzle), one
// elected thread issues tcgen05.mma into a 128x128 fp32 TMEM accumulator;
// four epilogue warps drain TMEM with tcgen05.ld and apply the fused
// epilogue (bias/ReLU, ReLU-mask, or SGD) writing fp32 + hi + lo planes.
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"
#include "sm100.cuh"

namespace mtk {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;             // 16 KB per operand plane
constexpr int STAGE_BYTES = 4 * TILE_BYTES;         // A_hi, A_lo, B_hi, B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int NUM_THREADS = 192;                    // warp0 TMA, warp1 MMA, warps2-5 epilogue
constexpr uint32_t TMEM_COLS = 128;

struct UmmaParams {
    CUtensorMap a_hi, a_lo, b_hi, b_lo;  // 3-D maps, coords (inner, outer, g)
    int M, N, K;
    int epi;                             // Epi value
    float* C;
    float* C_hi;
    float* C_lo;
    long long c_gs, ldc;
    const float* bias;
    long long bias_gs;
    const float* add;
    const float* mask;
    float lr;
    float* grad_out;
    int* flags;
    float* dbg;  // diagnostics: receives stage-0 smem (64 KB) when non-null
};

// TMEM accumulator (this warp's 32 lanes = rows m0+32q.., ncols columns) ->
// fused epilogue -> fp32 + tf32 hi/lo planes in HBM.
__device__ __forceinline__ void epilogue_rows(const UmmaParams& p, uint32_t tmem, int q, int lane,
                                              int g, int m0, int n0, int ncols) {
        const int m = m0 + 32 * q + lane;
        const bool row_ok = m < p.M;
        const long long rowbase = (long long)g * p.c_gs + (long long)m * p.ldc;
        bool bad = false;
#pragma unroll 1
        for (int c = 0; c < ncols / 32; ++c) {
            float v[32];
            tmem_ld_32x32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 32), v);
            const int nb = n0 + c * 32;
            if (!row_ok || nb >= p.N) continue;
            float xs[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = nb + j;
                const long long idx = rowbase + n;
                float x = v[j];
                if (n < p.N) {
                    if (p.epi == (int)Epi::kBias || p.epi == (int)Epi::kBiasRelu) {
                        x += p.bias[g * p.bias_gs + n];
                        bad |= !isfinite(x);
                        if (p.epi == (int)Epi::kBiasRelu) x = x > 0.f ? x : 0.f;
                    } else if (p.epi == (int)Epi::kMask) {
                        if (p.add) x = p.add[idx] + x;
                        x = (p.mask[idx] > 0.f) ? x : 0.f;
                    } else if (p.epi == (int)Epi::kSgd) {  // C is the fp32 master weight
                        if (p.grad_out) p.grad_out[idx] = x;
                        x = p.C[idx] - p.lr * x;
                        bad |= !isfinite(x);
                    }
                }
                xs[j] = x;
            }
            const bool vec = (nb + 32 <= p.N) && ((rowbase + nb) % 4 == 0);
            if (vec) {
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    float4 x4 = make_float4(xs[j], xs[j + 1], xs[j + 2], xs[j + 3]);
                    float4 h4, l4;
                    split_tf32(x4.x, h4.x, l4.x);
                    split_tf32(x4.y, h4.y, l4.y);
                    split_tf32(x4.z, h4.z, l4.z);
                    split_tf32(x4.w, h4.w, l4.w);
                    *reinterpret_cast<float4*>(p.C + rowbase + nb + j) = x4;
                    if (p.C_hi) {
                        *reinterpret_cast<float4*>(p.C_hi + rowbase + nb + j) = h4;
                        *reinterpret_cast<float4*>(p.C_lo + rowbase + nb + j) = l4;
                    }
                }
            } else {
                for (int j = 0; j < 32 && nb + j < p.N; ++j) {
                    const long long idx = rowbase + nb + j;
                    float hi, lo;
                    split_tf32(xs[j], hi, lo);
                    p.C[idx] = xs[j];
                    if (p.C_hi) {
                        p.C_hi[idx] = hi;
                        p.C_lo[idx] = lo;
                    }
                }
            }
        }
        if (bad && p.flags) atomicOr(p.flags, kFlagNonFinite);
}

template <int A_MN, int B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1) umma_gemm_kernel(const __grid_constant__ UmmaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.z;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int nk = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.a_hi);
        tma_prefetch(&p.a_lo);
        tma_prefetch(&p.b_hi);
        tma_prefetch(&p.b_lo);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                const int k0 = kb * BK;
                if (A_MN) {  // A(m,k) with m contiguous: 4 boxes of 32(m) x 32(k)
#pragma unroll
                    for (int j = 0; j < BM / 32; ++j) {
                        tma_load_3d(st + j * 4096, &p.a_hi, &full[s], m0 + 32 * j, k0, g);
                        tma_load_3d(st + TILE_BYTES + j * 4096, &p.a_lo, &full[s], m0 + 32 * j, k0, g);
                    }
                } else {     // A(m,k) with k contiguous: one box 32(k) x 128(m)
                    tma_load_3d(st, &p.a_hi, &full[s], k0, m0, g);
                    tma_load_3d(st + TILE_BYTES, &p.a_lo, &full[s], k0, m0, g);
                }
                uint8_t* sb = st + 2 * TILE_BYTES;
                if (B_MN) {  // B(k,n) with n contiguous: 4 boxes of 32(n) x 32(k)
#pragma unroll
                    for (int j = 0; j < BN / 32; ++j) {
                        tma_load_3d(sb + j * 4096, &p.b_hi, &full[s], n0 + 32 * j, k0, g);
                        tma_load_3d(sb + TILE_BYTES + j * 4096, &p.b_lo, &full[s], n0 + 32 * j, k0, g);
                    }
                } else {     // B(k,n) with k contiguous: one box 32(k) x 128(n)
                    tma_load_3d(sb, &p.b_hi, &full[s], k0, n0, g);
                    tma_load_3d(sb + TILE_BYTES, &p.b_lo, &full[s], k0, n0, g);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread) ----------------
        constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN, B_MN);
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    // K-major: +32 B per 8-element k step inside the 128-B swizzle row
                    // MN-major: +1024 B per 8 k rows (one swizzle atom)
                    const uint32_t aoff = A_MN ? kk * 1024 : kk * 32;
                    const uint32_t boff = B_MN ? kk * 1024 : kk * 32;
                    // K-major: SW128, SBO = 8 rows x 128 B.  MN-major: SW128 with
                    // 32-B atoms, LBO = 4 KB between 32-element MN boxes, SBO = 4 k
                    // rows x 128 B.
                    constexpr uint32_t a_lbo = A_MN ? 4096 : 16, b_lbo = B_MN ? 4096 : 16;
                    constexpr uint32_t a_sbo = A_MN ? 512 : 1024, b_sbo = B_MN ? 512 : 1024;
                    constexpr uint32_t a_lay = A_MN ? 1 : 2, b_lay = B_MN ? 1 : 2;
                    const uint64_t ahi = smem_desc(base + aoff, a_lbo, a_sbo, a_lay);
                    const uint64_t alo = smem_desc(base + TILE_BYTES + aoff, a_lbo, a_sbo, a_lay);
                    const uint64_t bhi = smem_desc(base + 2 * TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
                    const uint64_t blo = smem_desc(base + 3 * TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
                    const uint32_t acc0 = (kb | kk) ? 1u : 0u;
                    mma_tf32(tmem, alo, bhi, idesc, acc0);
                    mma_tf32(tmem, ahi, blo, idesc, 1u);
                    mma_tf32(tmem, ahi, bhi, idesc, 1u);
                }
                mma_commit(&empty[s]);  // frees the smem slot when these MMAs retire
            }
            mma_commit(tmem_full);
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> HBM ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        epilogue_rows(p, tmem, q, lane, g, m0, n0, BN);
        if (p.dbg) {
            const float* sf = reinterpret_cast<const float*>(smem);
            for (int i = threadIdx.x - 64; i < STAGE_BYTES / 4; i += 128) p.dbg[i] = sf[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a 2-CTA cluster computes a 256 x 256 tile.
// Each CTA stages its 128 rows of A and its 128 columns of B (hi/lo planes);
// the leader (rank 0) issues tcgen05.mma.cta_group::2 with M = 256, N = 256,
// reading both CTAs' smem; each CTA's TMEM receives its 128 rows x 256 cols.
// Per SM this halves operand bytes per MAC versus the 128 x 128 kernel.
constexpr int BN2 = 256;
constexpr uint32_t TMEM_COLS2 = 256;

template <int A_MN, int B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1) umma2_gemm_kernel(const __grid_constant__ UmmaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int g = blockIdx.z;
    const int m0 = (blockIdx.x >> 1) * 256 + (int)rank * 128;  // this CTA's rows
    const int n0 = blockIdx.y * BN2;                            // the pair's columns
    const int nb0 = n0 + (int)rank * 128;                       // this CTA's B half
    const int nk = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.a_hi);
        tma_prefetch(&p.a_lo);
        tma_prefetch(&p.b_hi);
        tma_prefetch(&p.b_lo);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 2);   // one arrival per CTA of the pair (leader's copy used)
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm<TMEM_COLS2>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs) ----------------
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                const int k0 = kb * BK;
                if (A_MN) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        tma_load_3d_2sm(st + j * 4096, &p.a_hi, &full[s], m0 + 32 * j, k0, g);
                        tma_load_3d_2sm(st + TILE_BYTES + j * 4096, &p.a_lo, &full[s], m0 + 32 * j, k0, g);
                    }
                } else {
                    tma_load_3d_2sm(st, &p.a_hi, &full[s], k0, m0, g);
                    tma_load_3d_2sm(st + TILE_BYTES, &p.a_lo, &full[s], k0, m0, g);
                }
                uint8_t* sb = st + 2 * TILE_BYTES;
                if (B_MN) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        tma_load_3d_2sm(sb + j * 4096, &p.b_hi, &full[s], nb0 + 32 * j, k0, g);
                        tma_load_3d_2sm(sb + TILE_BYTES + j * 4096, &p.b_lo, &full[s], nb0 + 32 * j, k0, g);
                    }
                } else {
                    tma_load_3d_2sm(sb, &p.b_hi, &full[s], k0, nb0, g);
                    tma_load_3d_2sm(sb + TILE_BYTES, &p.b_lo, &full[s], k0, nb0, g);
                }
                // the leader expects both CTAs' bytes; the follower only arrives
                if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
                else mbar_arrive_remote(&full[s], 0);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA, one thread) ----------------
        constexpr uint32_t idesc = idesc_tf32(256, BN2, A_MN, B_MN);
        if (rank == 0 && lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t aoff = A_MN ? kk * 1024 : kk * 32;
                    const uint32_t boff = B_MN ? kk * 1024 : kk * 32;
                    constexpr uint32_t a_lbo = A_MN ? 4096 : 16, b_lbo = B_MN ? 4096 : 16;
                    constexpr uint32_t a_sbo = A_MN ? 512 : 1024, b_sbo = B_MN ? 512 : 1024;
                    constexpr uint32_t a_lay = A_MN ? 1 : 2, b_lay = B_MN ? 1 : 2;
                    const uint64_t ahi = smem_desc(base + aoff, a_lbo, a_sbo, a_lay);
                    const uint64_t alo = smem_desc(base + TILE_BYTES + aoff, a_lbo, a_sbo, a_lay);
                    const uint64_t bhi = smem_desc(base + 2 * TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
                    const uint64_t blo = smem_desc(base + 3 * TILE_BYTES + boff, b_lbo, b_sbo, b_lay);
                    const uint32_t acc0 = (kb | kk) ? 1u : 0u;
                    mma_tf32_2sm(tmem, alo, bhi, idesc, acc0);
                    mma_tf32_2sm(tmem, ahi, blo, idesc, 1u);
                    mma_tf32_2sm(tmem, ahi, bhi, idesc, 1u);
                }
                mma_commit_2sm(&empty[s], 0x3);  // frees this slot in both CTAs
            }
            mma_commit_2sm(tmem_full, 0x3);
        }
    } else {
        // ---------------- epilogue (both CTAs: own 128 rows x 256 cols) ----------------
        const int q = warp & 3;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        epilogue_rows(p, tmem, q, lane, g, m0, n0, BN2);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<TMEM_COLS2>(tmem);
    }
}

__global__ void split_kernel(const float* __restrict__ x, float* __restrict__ hi,
                             float* __restrict__ lo, long long n) {
    const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n) {
        const float4 v = *reinterpret_cast<const float4*>(x + i);
        float4 h, l;
        split_tf32(v.x, h.x, l.x);
        split_tf32(v.y, h.y, l.y);
        split_tf32(v.z, h.z, l.z);
        split_tf32(v.w, h.w, l.w);
        *reinterpret_cast<float4*>(hi + i) = h;
        *reinterpret_cast<float4*>(lo + i) = l;
    } else {
        for (long long j = i; j < n; ++j) split_tf32(x[j], hi[j], lo[j]);
    }
}

// ---- host: tensor-map encoding through the driver entry point -------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    });
    if (!fn) fail(MTK_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 3-D fp32 map over [g][outer][inner] (inner contiguous), box (32, box_outer, 1)
CUtensorMap make_map(const float* base, long long inner, long long outer, long long G,
                     long long outer_stride, long long g_stride, int box_outer, bool mn_major) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)G};
    const cuuint64_t strides[2] = {(cuuint64_t)(outer_stride * 4), (cuuint64_t)(g_stride * 4)};
    const cuuint32_t box[3] = {32, (cuuint32_t)box_outer, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (outer_stride * 4) % 16 || (g_stride * 4) % 16)
        fail(MTK_ERROR, "umma: operand not 16-byte aligned for TMA");
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MTK_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

template <int A_MN, int B_MN>
void launch_variant(const UmmaParams& p, int G, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        MTK_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<A_MN, B_MN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr = true;
    }
    dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, G);
    umma_gemm_kernel<A_MN, B_MN><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(p);
    count_launch();
}

template <int A_MN, int B_MN>
void launch_variant2(const UmmaParams& p, int G, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        MTK_CUDA(cudaFuncSetAttribute(umma2_gemm_kernel<A_MN, B_MN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * ((p.M + 255) / 256), (p.N + BN2 - 1) / BN2, G);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MTK_CUDA(cudaLaunchKernelEx(&cfg, umma2_gemm_kernel<A_MN, B_MN>, p));
    count_launch();
}

bool use_pair_kernel(const UmmaGemm& u) {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("MTK_UMMA_PAIR");
        mode = e ? atoi(e) : 1;
    }
    return mode != 0 && u.M > 128 && u.N > 128;
}

}  // namespace

void launch_split(const float* x, float* hi, float* lo, long long n, cudaStream_t s) {
    if (n <= 0) return;
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
         reinterpret_cast<uintptr_t>(lo)) & 15)
        fail(MTK_ERROR, "split: unaligned pointer");
    const long long t = (n + 3) / 4;
    split_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(x, hi, lo, n);
    count_launch();
}

// Operand views: each operand is given as (hi, lo) planes with element
// (r, c) at base[g*gs + r*rs + c] where c is the contiguous index.
void launch_umma(const UmmaGemm& u, cudaStream_t s) {
    if (u.M <= 0 || u.N <= 0 || u.G <= 0 || u.K <= 0) return;
    UmmaParams p;
    std::memset(&p, 0, sizeof(p));
    // A: K-major -> inner = K, outer = M ; MN-major -> inner = M, outer = K
    if (u.a_mn) {
        p.a_hi = make_map(u.a_hi, u.M, u.K, u.G, u.a_rs, u.a_gs, BK, true);
        p.a_lo = make_map(u.a_lo, u.M, u.K, u.G, u.a_rs, u.a_gs, BK, true);
    } else {
        p.a_hi = make_map(u.a_hi, u.K, u.M, u.G, u.a_rs, u.a_gs, BM, false);
        p.a_lo = make_map(u.a_lo, u.K, u.M, u.G, u.a_rs, u.a_gs, BM, false);
    }
    if (u.b_mn) {
        p.b_hi = make_map(u.b_hi, u.N, u.K, u.G, u.b_rs, u.b_gs, BK, true);
        p.b_lo = make_map(u.b_lo, u.N, u.K, u.G, u.b_rs, u.b_gs, BK, true);
    } else {
        p.b_hi = make_map(u.b_hi, u.K, u.N, u.G, u.b_rs, u.b_gs, BN, false);
        p.b_lo = make_map(u.b_lo, u.K, u.N, u.G, u.b_rs, u.b_gs, BN, false);
    }
    p.M = u.M;
    p.N = u.N;
    p.K = u.K;
    p.epi = (int)u.epi;
    p.C = u.C;
    p.C_hi = u.C_hi;
    p.C_lo = u.C_lo;
    p.c_gs = u.c_gs;
    p.ldc = u.ldc;
    p.bias = u.bias;
    p.bias_gs = u.bias_gs;
    p.add = u.add;
    p.mask = u.mask;
    p.lr = u.lr;
    p.grad_out = u.grad_out;
    p.flags = u.flags;
    p.dbg = u.dbg;
    if (use_pair_kernel(u)) {
        if (!u.a_mn && u.b_mn) launch_variant2<0, 1>(p, u.G, s);
        else if (!u.a_mn && !u.b_mn) launch_variant2<0, 0>(p, u.G, s);
        else if (u.a_mn && u.b_mn) launch_variant2<1, 1>(p, u.G, s);
        else launch_variant2<1, 0>(p, u.G, s);
        return;
    }
    if (!u.a_mn && u.b_mn) launch_variant<0, 1>(p, u.G, s);
    else if (!u.a_mn && !u.b_mn) launch_variant<0, 0>(p, u.G, s);
    else if (u.a_mn && u.b_mn) launch_variant<1, 1>(p, u.G, s);
    else launch_variant<1, 0>(p, u.G, s);
}

}  // namespace mtk
