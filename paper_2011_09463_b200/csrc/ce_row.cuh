// ce_row.cuh -- one row of weighted softmax cross-entropy (tape.hpp:475-520)
// and its per-32-row warp partials, shared by ce_kernel (k_mlp.cu) and the
// fused head forward + CE (k_head.cu) so both round identically.
#pragma once
#include "internal.h"

namespace mtk {

// x: the row's logits (j < a.C), in registers.  Writes dlogits (dx, zero past
// C) and returns w_i (lse - x_y) / denom, the row's loss term; a label out of
// range sets kFlagBadLabel (tape.hpp:486-489) and yields zeros.
template <int NC>
__device__ __forceinline__ double ce_row(const CeArgs& a, int i, long long r, const float (&x)[NC],
                                         float (&dx)[NC]) {
#pragma unroll
    for (int j = 0; j < NC; ++j) dx[j] = 0.f;
    const int lab = a.y[r];
    if (lab < 0 || lab >= a.C) {
        atomicOr(a.flags, kFlagBadLabel);
        return 0.0;
    }
    float mx = x[0];
#pragma unroll
    for (int j = 1; j < NC; ++j)
        if (j < a.C) mx = fmaxf(mx, x[j]);
    float z = 0.f;
#pragma unroll
    for (int j = 0; j < NC; ++j)
        if (j < a.C) z += expf(x[j] - mx);
    const float lse = mx + logf(z);
    const float inv = (i < a.src_rows) ? a.inv_denom0 : a.inv_denom1;
    const float wi = (a.w ? a.w[r] : 1.f) * inv;
    float xl = x[0];
#pragma unroll
    for (int j = 1; j < NC; ++j)
        if (j == lab) xl = x[j];
    const double rl = (double)wi * ((double)lse - (double)xl);
#pragma unroll
    for (int j = 0; j < NC; ++j)
        if (j < a.C) dx[j] = wi * (expf(x[j] - lse) - (j == lab ? 1.f : 0.f));
    return rl;
}

// The warp's 32 rows (lane = row, inactive rows pass zeros) -> loss_part and,
// with a.colsum, the dlogits column partials of 32-row block blk.  Fixed
// butterfly order (deterministic).
template <int NC>
__device__ __forceinline__ void ce_warp_partials(const CeArgs& a, int g, int blk, int lane, double rl,
                                                 const float (&dx)[NC]) {
    const int nblk = (a.B + 31) / 32;
    for (int o = 16; o > 0; o >>= 1) rl += __shfl_xor_sync(0xffffffffu, rl, o);
    if (lane == 0 && blk < nblk) a.loss_part[(long long)g * nblk + blk] = rl;
    if (a.colsum) {
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            if (j >= a.C) break;
            float v = dx[j];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && blk < nblk) a.colsum[((long long)g * nblk + blk) * a.C + j] = v;
        }
    }
}

}  // namespace mtk
