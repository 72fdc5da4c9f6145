// k_umma.cu -- host side of the grouped 3xTF32 tcgen05 GEMM (umma_impl.cuh):
// tensor-map encoding, the launch-variant dispatch (operand majors, CTA
// pair, correction accumulator, epilogue kind) and launch_umma.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "umma_impl.cuh"
#include "umma_inst.h"

namespace mtk {
namespace umma {

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
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MTK_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

// programmatic dependent launch of the GEMM (and mmd_w) launches; MTK_PDL=0 disables (A/B)
bool pdl_enabled() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("MTK_PDL");
        mode = e ? atoi(e) : 1;
    }
    return mode != 0;
}

bool disable_half_tiles() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("MTK_UMMA_NO_HALF");  // A/B diagnostics
        mode = e ? 1 : 0;
    }
    return mode == 1;
}


// Launch-variant dispatch.  The bank's (majors, epilogue) pairs run
// EPI-specialised kernels; anything else (diagnostics) the run-time one.
template <bool PAIR, bool SEPC>
void dispatch2(const UmmaParams& p, int a_mn, int b_mn, int G, cudaStream_t s) {
    const int e = p.epi;
    if (!a_mn && b_mn) {
        if (e == (int)Epi::kBias) launch_variant<0, 1, PAIR, SEPC, (int)Epi::kBias>(p, G, s);
        else if (e == (int)Epi::kBiasRelu) launch_variant<0, 1, PAIR, SEPC, (int)Epi::kBiasRelu>(p, G, s);
        else if (e == (int)Epi::kMmdGrad) launch_variant<0, 1, PAIR, SEPC, (int)Epi::kMmdGrad>(p, G, s);
        else if (e == (int)Epi::kMmdGradW) launch_variant<0, 1, PAIR, SEPC, (int)Epi::kMmdGradW>(p, G, s);
        else if (e == (int)Epi::kStore) launch_variant<0, 1, PAIR, SEPC, (int)Epi::kStore>(p, G, s);
        else launch_variant<0, 1, PAIR, SEPC, -1>(p, G, s);
    } else if (!a_mn && !b_mn) {
        if (e == (int)Epi::kMask && !p.add) launch_variant<0, 0, PAIR, SEPC, kEpiMaskNoAdd>(p, G, s);
        else if (e == (int)Epi::kMask) launch_variant<0, 0, PAIR, SEPC, (int)Epi::kMask>(p, G, s);
        else launch_variant<0, 0, PAIR, SEPC, -1>(p, G, s);
    } else if (a_mn && b_mn) {
        if (e == (int)Epi::kSgd) launch_variant<1, 1, PAIR, SEPC, (int)Epi::kSgd>(p, G, s);
        else if (e == (int)Epi::kStore) launch_variant<1, 1, PAIR, SEPC, (int)Epi::kStore>(p, G, s);
        else launch_variant<1, 1, PAIR, SEPC, -1>(p, G, s);
    } else {
        launch_variant<1, 0, PAIR, SEPC, -1>(p, G, s);
    }
}
template <bool PAIR>
void dispatch(const UmmaParams& p, int a_mn, int b_mn, int G, bool sepc, cudaStream_t s) {
    if (sepc) dispatch2<PAIR, true>(p, a_mn, b_mn, G, s);
    else dispatch2<PAIR, false>(p, a_mn, b_mn, G, s);
}

bool use_pair_kernel(const UmmaGemm& u) {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("MTK_UMMA_PAIR");
        mode = e ? atoi(e) : 1;
    }
    return mode != 0 && u.M > 128 && u.N > 128;
}

}  // namespace umma

using umma::UmmaParams;
using umma::make_map;
using umma::use_pair_kernel;
using umma::dispatch;
using umma::BK;
using umma::kSepcMinK;


// Operand views: element (r, c) of an operand sits at base[g*gs + r*rs + c],
// c the contiguous index (K-major: r = m or n, c = k; MN-major: r = k).
void launch_umma(const UmmaGemm& u, cudaStream_t s) {
    if (u.M <= 0 || u.N <= 0 || u.G <= 0 || u.K <= 0) return;
    const bool pair = use_pair_kernel(u);
    UmmaParams p;
    std::memset(&p, 0, sizeof(p));
    // A: K-major -> inner = K, outer = M ; MN-major -> inner = M, outer = K
    p.a = u.a_mn ? make_map(u.a, u.M, u.K, u.G, u.a_rs, u.a_gs, BK, true)
                 : make_map(u.a, u.K, u.M, u.G, u.a_rs, u.a_gs, 128, false);
    p.b = u.b_mn ? make_map(u.b, u.N, u.K, u.G, u.b_rs, u.b_gs, BK, true)
                 : make_map(u.b, u.K, u.N, u.G, u.b_rs, u.b_gs, 128, false);
    if (!u.b_mn) p.b64 = make_map(u.b, u.K, u.N, u.G, u.b_rs, u.b_gs, 64, false);
    p.G = u.G;
    p.M = u.M;
    p.N = u.N;
    p.K = u.K;
    p.epi = (int)u.epi;
    p.C = u.C;
    p.c_gs = u.c_gs;
    p.ldc = u.ldc;
    p.bias = u.bias;
    p.bias_gs = u.bias_gs;
    p.add = u.add;
    p.mask = u.mask;
    p.lr = u.lr;
    p.grad_out = u.grad_out;
    p.colsum = u.colsum;
    p.rowvec = u.rowvec;
    p.scale = u.scale;
    p.zmask = u.zmask;
    p.ksplit = u.K;
    p.mbits = u.mbits;
    p.mb_gs = u.mb_gs;
    p.mb_ld = u.mb_ld;
    const bool bits_epi = u.epi == Epi::kMask || u.epi == Epi::kBiasRelu || u.epi == Epi::kMmdGradW;
    if (u.mbits && bits_epi && u.mb_ld < (u.N + 31) / 32)
        fail(MTK_ERROR, "umma: mask-bit rows shorter than ceil(N / 32) words");
    if (!bits_epi) p.mbits = nullptr;
    if (u.b2) {  // K = [0, ksplit) from b, [ksplit, K) from b2 (same major-ness)
        if (u.ksplit <= 0 || u.ksplit % BK || u.ksplit >= u.K || u.b_mn != 1)
            fail(MTK_ERROR, "umma: split B needs an N-major B and ksplit % 32 == 0 inside K");
        p.ksplit = u.ksplit;
        p.b2 = make_map(u.b2, u.N, u.K - u.ksplit, u.G, u.b2_rs, u.b2_gs, BK, true);
    }
    // separate correction accumulator: long K, or operands of one sign
    // (env MTK_UMMA_SEPC: 0 never, 1 always; A/B and precision diagnostics)
    const char* se = getenv("MTK_UMMA_SEPC");  // read per call (A/B in one process)
    const int sepc_mode = se ? atoi(se) : -1;
    const bool sepc = sepc_mode >= 0 ? sepc_mode != 0 : (u.K >= kSepcMinK || u.same_sign);
    p.flags = u.flags;
    // SEPC: the first kf k-blocks' corrections share the main accumulator while
    // the previous tile's epilogue still reads the corrections' region (~the
    // epilogue's duration: up to 10 stages of ~0.9 us -- the SGD epilogue takes
    // ~8 us; at most a third of K, so the shared part's drift stays that of a
    // partial sum: FWD0 / dW0 errors 3.6e-6 / 4.7e-6 -> 4.1e-6 / 4.8e-6 at the
    // bench shape); MTK_UMMA_SEPC_KF overrides
    {
        const int nk = (u.K + BK - 1) / BK;
        int kf = std::min(u.sepc_share, nk / 3);  // <= a third of the k-blocks
        if (const char* e = getenv("MTK_UMMA_SEPC_KF")) kf = std::min(atoi(e), nk);
        p.sepc_kf = std::max(0, kf);
    }
    if (const char* e = getenv("MTK_UMMA_EPI_DIAG")) p.ediag = atoi(e);
    if (const char* e = getenv("MTK_UMMA_PREFETCH")) p.prefetch = atoi(e);
    if (const char* t = getenv("MTK_UMMA_TRACE")) {
        // diagnostics; MTK_UMMA_TRACE_SHAPE="M,N,K,epi" restricts it to matching launches
        bool match = true;
        if (const char* sh = getenv("MTK_UMMA_TRACE_SHAPE")) {
            int m = 0, n = 0, k = 0, e = 0;
            match = sscanf(sh, "%d,%d,%d,%d", &m, &n, &k, &e) == 4 && m == u.M && n == u.N && k == u.K &&
                    e == (int)u.epi;
        }
        if (match) p.trace = reinterpret_cast<unsigned long long*>(strtoull(t, nullptr, 0));
    }
    if (pair) dispatch<true>(p, u.a_mn, u.b_mn, u.G, sepc, s);
    else dispatch<false>(p, u.a_mn, u.b_mn, u.G, sepc, s);
}

}  // namespace mtk
