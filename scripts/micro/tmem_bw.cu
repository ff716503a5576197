// Microbenchmark (B200): TMEM read bandwidth (tcgen05.ld shapes, warps per CTA)
// and f16 UMMA issue rate (M=128, N in {64,128,256}, K=16).  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1103_2635_b200/csrc scripts/micro/tmem_bw.cu -o /tmp/tmem_bw
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace rbc;

template <int X>  // columns per load: 32x32b.x{X}
__device__ __forceinline__ uint32_t ld_cols(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld_cols<32>(uint32_t taddr) {
    uint32_t r[32];
    sm100::tmem_ld32_async(taddr, r);
    sm100::tmem_wait_ld(r);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i];
    return x;
}

template <>
__device__ __forceinline__ uint32_t ld_cols<64>(uint32_t taddr) {
    uint32_t r[32], s[32];
    sm100::tmem_ld32_async(taddr, r);
    sm100::tmem_ld32_async(taddr + 32, s);
    sm100::tmem_wait_ld(r);
    sm100::tmem_tie(s);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i] ^ s[i];
    return x;
}

template <int X>
__global__ void tmem_read_kernel(int iters, unsigned long long *cycles, uint32_t *sink) {
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) sm100::tmem_alloc<512>(&s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = s_tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const int slot = warp >> 2;  // warps sharing a quadrant read different column ranges
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) acc ^= ld_cols<X>(tmem + ((it * 64 + slot * 128) & 511));
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc<512>(s_tmem);
}

__global__ void mma_rate_kernel(int iters, int n, unsigned long long *cycles, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    sm100::fence_proxy_async_smem();
    if (warp == 0) sm100::tmem_alloc<512>(&s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (threadIdx.x == 32) {
        const uint32_t a0 = sm100::smem_u32(smem), b0 = a0 + 16384;
        const uint32_t idesc = sm100::idesc_f16_f32(128, n);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode == 1) {  // SW32 operands (one 32-byte K16 row per operand row)
                for (int kk = 0; kk < 4; ++kk)
                    sm100::umma_f16(s_tmem + (it & 1) * 256, sm100::umma_desc_sw32(a0),
                                    sm100::umma_desc_sw32(b0), idesc, kk > 0);
            } else {
                for (int kk = 0; kk < 4; ++kk)
                    sm100::umma_f16(s_tmem + (it & 1) * 256, sm100::umma_desc_sw128(a0 + kk * 32),
                                    sm100::umma_desc_sw128(b0 + kk * 32), idesc, kk > 0);
            }
            if (mode == 2) {  // 4 x SW128 + 1 x SW32 (the d = 64 chunk with the aug plane)
                sm100::umma_f16(s_tmem + (it & 1) * 256, sm100::umma_desc_sw32(a0 + 8192),
                                sm100::umma_desc_sw32(b0 + 32768), idesc, 1);
            }
        }
        sm100::umma_commit(&bar);
        sm100::mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc<512>(s_tmem);
}

// TMEM reads (warps 1..W) while warp 0 keeps the tensor core busy writing other columns
__global__ void mixed_kernel(int iters, int mma_iters, unsigned long long *cycles, uint32_t *sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    sm100::fence_proxy_async_smem();
    if (warp == 0) sm100::tmem_alloc<512>(&s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const unsigned long long t0 = clock64();
    if (warp == 0) {
        if (threadIdx.x == 0 && mma_iters > 0) {
            const uint32_t a0 = sm100::smem_u32(smem), b0 = a0 + 16384;
            const uint32_t idesc = sm100::idesc_f16_f32(128, 256);
            for (int it = 0; it < mma_iters; ++it)
                for (int kk = 0; kk < 5; ++kk)
                    sm100::umma_f16(s_tmem + 256, sm100::umma_desc_sw128(a0 + (kk & 3) * 32),
                                    sm100::umma_desc_sw128(b0 + (kk & 3) * 32), idesc, kk > 0);
            sm100::umma_commit(&bar);
            sm100::mbar_wait(&bar, 0);
            cycles[blockIdx.x * 2] = clock64() - t0;
        }
    } else {
        const uint32_t tmem = s_tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const int slot = (warp - 1) >> 2;
        uint32_t acc = 0;
        for (int it = 0; it < iters; ++it) acc ^= ld_cols<32>(tmem + ((it * 32 + slot * 64) & 255));
        sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
        if (threadIdx.x == 32) cycles[blockIdx.x * 2 + 1] = clock64() - t0;
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc<512>(s_tmem);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, 2 * sms * sizeof(unsigned long long));
    cudaMalloc(&sink, sms * 1024 * sizeof(uint32_t));
    unsigned long long h[256];
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        for (int x : {32, 64}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (x == 32) tmem_read_kernel<32><<<sms, warps * 32>>>(iters, cyc, sink);
                else tmem_read_kernel<64><<<sms, warps * 32>>>(iters, cyc, sink);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            double mean = 0;
            for (int i = 0; i < sms; ++i) mean += h[i];
            mean /= sms;
            const double bytes = double(warps) * iters * 32 * x * 4;  // per SM
            printf("tmem read: %2d warps, %d cols/wait: %.1f B/cycle/SM (%.0f cycles)\n", warps, x, bytes / mean, mean);
        }
    }
    cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int mode : {0, 1, 2})
    for (int n : {64, 128, 256}) {
        for (int rep = 0; rep < 2; ++rep) mma_rate_kernel<<<sms, 64, 80 * 1024>>>(iters, n, cyc, mode);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < sms; ++i) mean += h[i];
        mean /= sms;
        const double macs = double(iters) * 4 * 128 * n * 16;
        printf("umma f16 mode %d (0 SW128, 1 SW32, 2 4xSW128+SW32) M=128 N=%3d: %.1f cycles per group of %d MMAs\n", mode, n,
               mean / iters, mode == 2 ? 5 : 4);
    }
    cudaFuncSetAttribute(mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int warps : {8, 16}) {
        for (int mi : {0, 1}) {
            const int rd_iters = 4096, mma_iters = mi ? 3000 : 0;
            for (int rep = 0; rep < 2; ++rep) mixed_kernel<<<sms, (warps + 1) * 32, 80 * 1024>>>(rd_iters, mma_iters, cyc, sink);
            cudaDeviceSynchronize();
            unsigned long long hh[512];
            cudaMemcpy(hh, cyc, sms * 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            double mm = 0, rr = 0;
            for (int i = 0; i < sms; ++i) {
                mm += hh[2 * i];
                rr += hh[2 * i + 1];
            }
            mm /= sms;
            rr /= sms;
            const double bytes = double(warps) * rd_iters * 32 * 32 * 4;
            printf("mixed: %2d reader warps, mma %s: read %.1f B/cycle/SM over %.0f cycles; mma %.1f cycles per N=256 K=80 chunk\n",
                   warps, mi ? "on " : "off", bytes / rr, rr, mi ? mm / mma_iters : 0.0);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
