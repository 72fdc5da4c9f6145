// k_rng.cu -- counter-based synthetic data on the device.
//
// The host mt::Rng (rng.hpp:13-75) is sequential: 2^20 x 784 Box-Muller
// normals per pool take ~10 s on one core and are the C5 wall-clock floor.
// This generator is a pure function of (seed, stream, counter), so every
// thread computes its own slice with no state and the pools are born in HBM:
//   Philox4x64-10 (the Random123 bijection; oracle/oracle.c restates it and
//   tests pin it to the published known-answer vector and numpy's Philox),
//   key = {seed, stream};
//   normals: element e of the row-major [n, d] matrix <- counter {e/4,0,0,0};
//     words (w0,w1) -> elements 4i, 4i+1; (w2,w3) -> 4i+2, 4i+3 (Box-Muller,
//     u1 = ((wa >> 40) + 1) 2^-24, u2 = (wb >> 40) 2^-24, fp32 math here);
//   labels: row i <- word i%4 of counter {i/4,1,0,0}, y = umulhi(w, C)
//     (integer, bit-exact against the oracle);
//   X[i,k] = (mu[y_i,k] + z) (+ shift[k]).
// Parity contract: raw words and labels bit-exact; normals within a few fp32
// ulps of the oracle's f64 transform (tests/test_gpu_rng.py states the bound).
// HBM-bound: one 16-byte store per Philox block when d % 4 == 0.
#include <cstdint>

#include "internal.h"

namespace mtk {
namespace {

struct U4 {
    unsigned long long x, y, z, w;
};

__device__ __forceinline__ U4 philox4x64(unsigned long long c0, unsigned long long c1,
                                         unsigned long long c2, unsigned long long c3,
                                         unsigned long long k0, unsigned long long k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned long long hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
        const unsigned long long lo0 = 0xD2E7470EE14C6C93ULL * c0;
        const unsigned long long hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
        const unsigned long long lo1 = 0xCA5A826395121157ULL * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ void box_muller(unsigned long long wa, unsigned long long wb, float& za,
                                           float& zb) {
    const float u1 = (float)((wa >> 40) + 1ULL) * 0x1p-24f;
    const float u2 = (float)(wb >> 40) * 0x1p-24f;
    const float r = sqrtf(-2.f * logf(u1));
    float s, c;
    sincospif(2.f * u2, &s, &c);
    za = r * c;
    zb = r * s;
}

__device__ __forceinline__ float4 normals4(unsigned long long blk, unsigned long long seed,
                                           unsigned long long stream) {
    const U4 w = philox4x64(blk, 0, 0, 0, seed, stream);
    float4 z;
    box_muller(w.x, w.y, z.x, z.y);
    box_muller(w.z, w.w, z.z, z.w);
    return z;
}

__global__ void philox_fill_kernel(unsigned long long seed, unsigned long long stream,
                                   unsigned long long c0, unsigned long long c1, long long nblocks,
                                   unsigned long long* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nblocks;
         i += (long long)gridDim.x * blockDim.x) {
        const U4 w = philox4x64(c0 + (unsigned long long)i, c1, 0, 0, seed, stream);
        out[4 * i] = w.x;
        out[4 * i + 1] = w.y;
        out[4 * i + 2] = w.z;
        out[4 * i + 3] = w.w;
    }
}

__global__ void normals_kernel(unsigned long long seed, unsigned long long stream, long long first,
                               long long count, float* out) {
    const long long b0 = first / 4, b1 = (first + count + 3) / 4;
    for (long long b = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; b < b1;
         b += (long long)gridDim.x * blockDim.x) {
        const float4 z = normals4((unsigned long long)b, seed, stream);
        const float v[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long e = 4 * b + j;
            if (e >= first && e < first + count) out[e - first] = v[j];
        }
    }
}

__global__ void labels_kernel(unsigned long long seed, unsigned long long stream, int C, long long n,
                              int32_t* y) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; 4 * b < n;
         b += (long long)gridDim.x * blockDim.x) {
        const U4 w = philox4x64((unsigned long long)b, 1, 0, 0, seed, stream);
        const unsigned long long ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * b + j < n) y[4 * b + j] = (int32_t)__umul64hi(ws[j], (unsigned long long)C);
    }
}

// X[i, k] = (mu[y_i, k] + z[i*d + k]) (+ shift[k]); one Philox block per thread
template <bool VEC>
__global__ void synth_kernel(unsigned long long seed, unsigned long long stream, int d, long long n,
                             const float* __restrict__ mu, const float* __restrict__ shift,
                             const int32_t* __restrict__ y, float* __restrict__ X) {
    const long long nb = (n * d + 3) / 4;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const float4 z = normals4((unsigned long long)b, seed, stream);
        const long long e0 = 4 * b;
        if (VEC) {  // d % 4 == 0: the four elements share a row
            const long long i = e0 / d;
            const int k = (int)(e0 - i * d);
            const float4 m = *reinterpret_cast<const float4*>(mu + (long long)__ldg(y + i) * d + k);
            float4 x = make_float4(m.x + z.x, m.y + z.y, m.z + z.z, m.w + z.w);
            if (shift) {
                const float4 s = *reinterpret_cast<const float4*>(shift + k);
                x.x += s.x;
                x.y += s.y;
                x.z += s.z;
                x.w += s.w;
            }
            __stcs(reinterpret_cast<float4*>(X + e0), x);
        } else {
            const float v[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long e = e0 + j;
                if (e >= n * d) break;
                const long long i = e / d;
                const int k = (int)(e - i * d);
                float x = mu[(long long)__ldg(y + i) * d + k] + v[j];
                if (shift) x += shift[k];
                X[e] = x;
            }
        }
    }
}

unsigned grid_for(long long items) {
    long long b = (items + 255) / 256;
    const long long cap = 148LL * 16;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

void launch_philox_fill(uint64_t seed, uint64_t stream, uint64_t c0, uint64_t c1, long long nblocks,
                        uint64_t* out, cudaStream_t s) {
    if (nblocks <= 0) return;
    philox_fill_kernel<<<grid_for(nblocks), 256, 0, s>>>(seed, stream, c0, c1, nblocks,
                                                         reinterpret_cast<unsigned long long*>(out));
    count_launch();
}

void launch_counter_normals(uint64_t seed, uint64_t stream, long long first, long long count,
                            float* out, cudaStream_t s) {
    if (count <= 0) return;
    normals_kernel<<<grid_for((count + 7) / 4), 256, 0, s>>>(seed, stream, first, count, out);
    count_launch();
}

void launch_synth_counter(uint64_t seed, uint64_t stream, int C, int d, long long n,
                          const float* mu, const float* shift, float* X, int32_t* y,
                          cudaStream_t s) {
    if (n <= 0) return;
    labels_kernel<<<grid_for((n + 3) / 4), 256, 0, s>>>(seed, stream, C, n, y);
    count_launch();
    const long long nb = (n * d + 3) / 4;
    const bool vec = d % 4 == 0 && ((uintptr_t)mu & 15) == 0 && ((uintptr_t)X & 15) == 0 &&
                     (!shift || ((uintptr_t)shift & 15) == 0);
    if (vec)
        synth_kernel<true><<<grid_for(nb), 256, 0, s>>>(seed, stream, d, n, mu, shift, y, X);
    else
        synth_kernel<false><<<grid_for(nb), 256, 0, s>>>(seed, stream, d, n, mu, shift, y, X);
    count_launch();
}

}  // namespace mtk
