// tmem_probe.cu -- cost of tcgen05.alloc / dealloc (diagnostics).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2011_09463_b200/csrc -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace mtk::sm100;

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// mode 0: alloc/dealloc only; mode 1: + tcgen05.st/ld on all lanes; mode 2: + one MMA
template <int COLS>
__global__ void probe(unsigned long long* out, int mode) {
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    unsigned long long t0 = gt();
    if (warp == 0) tmem_alloc<COLS>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    unsigned long long t1 = gt();
    if (mode == 2) {
        __shared__ __align__(1024) float sA[128 * 32];
        for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) sA[i] = 1.0f;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_barrier_init();
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 32) {
            const uint32_t idesc = idesc_tf32(128, 128, 0, 0);
            for (int it = 0; it < 64; ++it)
                for (int kk = 0; kk < 4; ++kk) {
                    uint64_t a = smem_desc_sw128(smem_u32(sA) + kk * 32, 16, 1024);
                    mma_tf32(tmem, a, a, idesc, (it | kk) > 0);
                }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        tc_fence_after();
    }
    if (mode >= 1) {
        float v[8];
        for (int i = 0; i < 8; ++i) v[i] = (float)i;
        const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
        tmem_st_32x8(tmem + lane_base, v);
        tmem_st_wait();
        tmem_ld_32x8(tmem + lane_base, v);
        if (mode == 1 && v[3] != 3.f) out[0] = 1;
    }
    tc_fence_before();
    __syncthreads();
    unsigned long long t2 = gt();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<COLS>(tmem);
    }
    unsigned long long t3 = gt();
    if (threadIdx.x == 0) {
        out[1 + 4 * blockIdx.x] = t0;
        out[2 + 4 * blockIdx.x] = t1;
        out[3 + 4 * blockIdx.x] = t2;
        out[4 + 4 * blockIdx.x] = t3;
    }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 4096);
    unsigned long long h[4096];
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, 8 * 4096);
            probe<512><<<296, 128>>>(d, mode);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, 8 * 4096, cudaMemcpyDeviceToHost);
            double al = 0, de = 0, mx = 0;
            unsigned long long mn = ~0ull, me = 0;
            for (int b = 0; b < 296; ++b) {
                unsigned long long* p = h + 1 + 4 * b;
                al += (p[1] - p[0]) / 1000.0;
                de += (p[3] - p[2]) / 1000.0;
                if ((p[3] - p[2]) / 1000.0 > mx) mx = (p[3] - p[2]) / 1000.0;
                if (p[0] < mn) mn = p[0];
                if (p[3] > me) me = p[3];
            }
            printf("mode %d rep %d (%s): 296 CTAs x 512 cols: alloc avg %.2f us, dealloc(warp0 view) avg %.2f max %.2f us, span %.2f us\n",
                   mode, rep, cudaGetErrorString(e), al / 296, de / 296, mx, (me - mn) / 1000.0);
        }
    }
    return 0;
}
