// umma_inst.h -- the explicit instantiations of umma::launch_variant, one
// list per k_umma_inst_<part>.cu; k_umma.cu sees them as extern templates.
#pragma once

#define MTK_UMMA_LV(X, A, B, E) \
    X template void launch_variant<A, B, false, false, E>(UmmaParams, int, cudaStream_t); \
    X template void launch_variant<A, B, false, true, E>(UmmaParams, int, cudaStream_t); \
    X template void launch_variant<A, B, true, false, E>(UmmaParams, int, cudaStream_t); \
    X template void launch_variant<A, B, true, true, E>(UmmaParams, int, cudaStream_t);

#define MTK_UMMA_PART_G(X) \
    MTK_UMMA_LV(X, 0, 0, -1) \
    MTK_UMMA_LV(X, 0, 1, -1) \
    MTK_UMMA_LV(X, 1, 0, -1) \
    MTK_UMMA_LV(X, 1, 1, -1)

#define MTK_UMMA_PART_F(X) \
    MTK_UMMA_LV(X, 0, 1, (int)Epi::kBias) \
    MTK_UMMA_LV(X, 0, 1, (int)Epi::kBiasRelu)

#define MTK_UMMA_PART_V(X) \
    MTK_UMMA_LV(X, 0, 1, (int)Epi::kMmdGrad) \
    MTK_UMMA_LV(X, 0, 1, (int)Epi::kMmdGradW) \
    MTK_UMMA_LV(X, 0, 1, (int)Epi::kStore)

#define MTK_UMMA_PART_D(X) \
    MTK_UMMA_LV(X, 0, 0, (int)Epi::kMask) \
    MTK_UMMA_LV(X, 0, 0, kEpiMaskNoAdd) \
    MTK_UMMA_LV(X, 1, 1, (int)Epi::kSgd) \
    MTK_UMMA_LV(X, 1, 1, (int)Epi::kStore)

#define MTK_UMMA_EXTERN extern
#define MTK_UMMA_NONE

#ifndef MTK_UMMA_INST_PART
namespace mtk {
namespace umma {
MTK_UMMA_PART_G(MTK_UMMA_EXTERN)
MTK_UMMA_PART_F(MTK_UMMA_EXTERN)
MTK_UMMA_PART_V(MTK_UMMA_EXTERN)
MTK_UMMA_PART_D(MTK_UMMA_EXTERN)
}  // namespace umma
}  // namespace mtk
#endif
