// k_dp.cu -- data-parallel step kernels.
//
// A replicated bank's gradients live in one flat "arena": for every parameter
// matrix i in index order, dW_i [G, fan_in, fan_out] then db_i [G, fan_out].
// Every rank holds the same arena layout, so after an all-gather the n worker
// arenas sit part_stride floats apart in one buffer and one launch can
//   g = fp32(((p_0 + p_1) + p_2 + ...) / n)  (fp64, ascending worker order)
//   w = optimizer_step(w, g)               (SGD or Adam, optim.hpp:46-63)
// for every trainable segment.  The order of the sum is fixed per element, so
// the result is bit-identical on every rank whatever order the gradients
// arrived in ("Aggregation order is fixed").
#include <cstdint>

#include "internal.h"

namespace mtk {
namespace {

__global__ void dp_reduce_apply_kernel(DpSegments segs, const float* __restrict__ parts, int n_parts,
                                       long long part_stride, float lr, AdamArgs adam, int* flags) {
    const int si = blockIdx.y;
    const DpSegment& sg = segs.s[si];
    if (sg.frozen) return;
    AdamArgs a = adam;
    if (a.on) {
        a.m = sg.m;
        a.v = sg.v;
    }
    bool bad = false;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < sg.n;
         j += (long long)gridDim.x * blockDim.x) {
        const float* p = parts + sg.off + j;
        // fp64 accumulation: n equal fp32 values sum exactly, so identical
        // shards give back exactly the single worker's gradient
        double acc = (double)__ldg(p);
        for (int r = 1; r < n_parts; ++r) acc = __dadd_rn(acc, (double)__ldg(p + r * part_stride));
        const float g = (float)__ddiv_rn(acc, (double)n_parts);
        const float w = param_update(sg.p[j], g, lr, a, j);
        bad |= !isfinite(w);
        sg.p[j] = w;
    }
    if (bad && flags) atomicOr(flags, kFlagNonFinite);
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// order-independent 64-bit fingerprint of the parameter bits: sum (mod 2^64)
// of mix(segment, index, bits) -- integer addition commutes, so the value is
// deterministic under any block schedule.
__global__ void fingerprint_kernel(DpSegments segs, unsigned long long* out) {
    const int si = blockIdx.y;
    const DpSegment& sg = segs.s[si];
    unsigned long long h = 0;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < sg.n;
         j += (long long)gridDim.x * blockDim.x) {
        const unsigned bits = __float_as_uint(sg.p[j]);
        h += mix64(((unsigned long long)(si + 1) << 48) ^ ((unsigned long long)j << 16) ^
                   mix64(bits + 0x9e3779b97f4a7c15ULL));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

unsigned blocks_for(long long max_n) {
    long long b = (max_n + 255) / 256;
    if (b > 148LL * 4) b = 148LL * 4;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

void launch_dp_reduce_apply(const DpSegments& segs, const float* parts, int n_parts,
                            long long part_stride, float lr, const AdamArgs& adam, int* flags,
                            cudaStream_t s) {
    if (segs.count <= 0) return;
    long long mx = 0;
    for (int i = 0; i < segs.count; ++i) mx = segs.s[i].n > mx ? segs.s[i].n : mx;
    dim3 grid(blocks_for(mx), segs.count);
    dp_reduce_apply_kernel<<<grid, 256, 0, s>>>(segs, parts, n_parts, part_stride, lr, adam, flags);
    count_launch();
}

void launch_fingerprint(const DpSegments& segs, unsigned long long* out, cudaStream_t s) {
    if (segs.count <= 0) return;
    long long mx = 0;
    for (int i = 0; i < segs.count; ++i) mx = segs.s[i].n > mx ? segs.s[i].n : mx;
    dim3 grid(blocks_for(mx), segs.count);
    fingerprint_kernel<<<grid, 256, 0, s>>>(segs, out);
    count_launch();
}

}  // namespace mtk
