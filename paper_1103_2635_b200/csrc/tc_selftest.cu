// tc_selftest.cu -- diagnostic: one 128 x N x 64 f16 UMMA tile through the
// same descriptor / TMEM / tcgen05.ld path the stage-2 engine uses.
// Exposed as rbc_tc_selftest (tests compare it with a float64 GEMM).
#include "common.cuh"
#include "sm100.cuh"

namespace rbc {

__global__ void __launch_bounds__(128) tc_selftest_kernel(const __half *__restrict__ a, const __half *__restrict__ b,
                                                          float *__restrict__ c, int n) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms need 1 KiB alignment
    uint8_t *sa = smem;                // 128 x 128 B
    uint8_t *sb = smem + 128 * 128;    // n x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage A and B rows into the SWIZZLE_128B K-major layout
    for (int t = tid; t < 128 * 8; t += 128) {
        const int r = t >> 3, ch = t & 7;
        *reinterpret_cast<uint4 *>(sa + sm100::sw128_offset(r, ch)) = reinterpret_cast<const uint4 *>(a + r * 64)[ch];
    }
    for (int t = tid; t < n * 8; t += 128) {
        const int r = t >> 3, ch = t & 7;
        *reinterpret_cast<uint4 *>(sb + sm100::sw128_offset(r, ch)) = reinterpret_cast<const uint4 *>(b + r * 64)[ch];
    }
    sm100::fence_proxy_async_smem();
    if (tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_barrier_init();
    }
    if (warp == 0) sm100::tmem_alloc<256>(&tmem_base);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = sm100::idesc_f16_f32(128, n);
        const uint32_t a0 = sm100::smem_u32(sa), b0 = sm100::smem_u32(sb);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            sm100::umma_f16(tmem, sm100::umma_desc_sw128(a0 + kk * 32), sm100::umma_desc_sw128(b0 + kk * 32), idesc,
                            kk > 0);
        sm100::umma_commit(&bar);
    }
    __syncwarp();
    sm100::mbar_wait(&bar, 0);
    sm100::tc_fence_after();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < n; c0 += 32) {
        float v[32];
        sm100::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (c0 + j < n) c[row * n + c0 + j] = v[j];
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

}  // namespace rbc

extern "C" int rbc_tc_selftest(const void *a, const void *b, float *c, int32_t n, void *stream) {
    if (n < 16 || n > 256 || n % 16) return rbc::fail(RBC_EINVAL, "selftest: n must be a multiple of 16 in [16, 256]");
    const size_t smem = 128 * 128 + static_cast<size_t>(n) * 128 + 1024;
    cudaFuncSetAttribute(rbc::tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    rbc::tc_selftest_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const __half *>(a), reinterpret_cast<const __half *>(b), c, n);
    RBC_LAUNCHED();
    return RBC_OK;
}
