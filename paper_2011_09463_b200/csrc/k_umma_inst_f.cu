// k_umma_inst_f.cu -- explicit instantiations of the tcgen05 GEMM (umma_impl.cuh)
#define MTK_UMMA_INST_PART
#include "umma_impl.cuh"
#include "umma_inst.h"

namespace mtk {
namespace umma {
MTK_UMMA_PART_F(MTK_UMMA_NONE)
}  // namespace umma
}  // namespace mtk
