// umma_probe.cu -- standalone probe of the tcgen05 tf32 MMA plumbing
// (descriptor encodings, TMEM readout) on one CTA, without TMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2011_09463_b200/csrc -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstring>
#include <algorithm>

#include "sm100.cuh"

using namespace mtk::sm100;

// A: 128 x 32 (K-major), B: 128(n) x 32(k) (K-major) ; C = A * B^T (128x128)
__global__ void probe(const float* A, const float* B, float* C, int mode) {
    __shared__ __align__(1024) float sA[128 * 32];
    __shared__ __align__(1024) float sB[128 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x;
    // manual SW128 K-major fill: row r (128 B), 16-B chunk c -> c ^ (r & 7)
    for (int i = t; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32, c = k / 4, w = k % 4;
        const int pos = r * 32 + ((c ^ (r & 7)) * 4) + w;
        float a = A[i], b = B[i];
        if (mode == 2) {  // raw fp32 bits: what does the tf32 MMA do with the low 13 bits?
            sA[pos] = a;
            sB[pos] = b;
        } else {
            sA[pos] = tf32_rna(a);
            sB[pos] = tf32_rna(b);
        }
    }
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (t < 32) tmem_alloc<128>(&slot);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (t == 0) {
        uint32_t idesc = idesc_tf32(128, 128, 0, 0);
        if (mode == 1) idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128 >> 3) << 17) | ((128 >> 4) << 23);
        for (int kk = 0; kk < 4; ++kk) {
            uint64_t a = smem_desc_sw128(smem_u32(sA) + kk * 32, 16, 1024);
            uint64_t b = smem_desc_sw128(smem_u32(sB) + kk * 32, 16, 1024);
            mma_tf32(tmem, a, b, idesc, kk > 0);
        }
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int q = (t >> 5) & 3;
    for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld_32x32(tmem + ((uint32_t)(32 * q) << 16) + c * 32, v);
        for (int j = 0; j < 32; ++j) C[(32 * q + (t & 31)) * 128 + c * 32 + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

int main() {
    std::vector<float> A(128 * 32), B(128 * 32), C(128 * 128);
    for (int i = 0; i < 128 * 32; ++i) {
        A[i] = 1.0f + (float)((i * 7919) % 8191) / 8192.0f * 0.999f;   // low mantissa bits set
        B[i] = 1.0f + (float)((i * 104729) % 8191) / 8192.0f * 0.999f;
    }
    auto trunc = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return (double)y; };
    auto rna = [](float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xFFFFE000u; float y; memcpy(&y, &u, 4); return (double)y; };
    std::vector<double> ref(128 * 128, 0.0), rt(128 * 128, 0.0), rr(128 * 128, 0.0);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n)
            for (int k = 0; k < 32; ++k) {
                ref[m * 128 + n] += (double)A[m * 32 + k] * B[n * 32 + k];
                rt[m * 128 + n] += trunc(A[m * 32 + k]) * trunc(B[n * 32 + k]);
                rr[m * 128 + n] += rna(A[m * 32 + k]) * rna(B[n * 32 + k]);
            }
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode : {0, 2}) {
        cudaMemset(dC, 0, C.size() * 4);
        probe<<<1, 128>>>(dA, dB, dC, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (int i = 0; i < 128 * 128; ++i) {
            err = std::max(err, std::fabs(C[i] - ref[i]));
            mx = std::max(mx, std::fabs(ref[i]));
        }
        double et = 0, er = 0;
        for (int i = 0; i < 128 * 128; ++i) {
            et = std::max(et, std::fabs(C[i] - rt[i]));
            er = std::max(er, std::fabs(C[i] - rr[i]));
        }
        printf("mode %d: %s |C-exact| %.3g  |C-trunc| %.3g  |C-rna| %.3g  (ref max %.3g)\n", mode,
               cudaGetErrorString(e), err, et, er, mx);
    }
    return 0;
}
