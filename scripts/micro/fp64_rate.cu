// Microbenchmark (B200): throughput of the instructions in the exact re-rank
// distance: F2F.F64.F32 conversion, DADD/DMUL, and the full per-coordinate
// step (2 cvt + dsub + dmul + dadd), per SM per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/fp64_rate.cu -o /tmp/fp64_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(const float *in, double *out, int iters, unsigned long long *cyc) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = in[(threadIdx.x + j) & 255];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE == 0) {  // conversion only
                acc[j] += 0.0;
                double x = static_cast<double>(a[j]);
                acc[j] = x;
                a[j] = __int_as_float(__float_as_int(a[j]) + 1);
            } else if (MODE == 1) {  // dadd chain x8 independent
                acc[j] = __dadd_rn(acc[j], 1.0000001);
            } else {  // full exact step with both conversions
                const double d = __dsub_rn(static_cast<double>(a[j]), static_cast<double>(a[(j + 1) & 7]));
                acc[j] = __dadd_rn(acc[j], __dmul_rn(d, d));
                a[j] = __int_as_float(__float_as_int(a[j]) ^ 1);
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// dependent-chain latency: one warp, acc = acc + x (DADD) or the full exact step
template <int MODE>
__global__ void lat(const float *in, double *out, int iters, unsigned long long *cyc) {
    float a = in[threadIdx.x], b = in[threadIdx.x + 1];
    double acc = 0.0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            acc = __dadd_rn(acc, 1.0000001);
        } else {
            const double d = __dsub_rn(static_cast<double>(a), static_cast<double>(b));
            acc = __dadd_rn(acc, __dmul_rn(d, d));
            a = __int_as_float(__float_as_int(a) ^ 1);
        }
    }
    const unsigned long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    float *in;
    double *out;
    unsigned long long *cyc;
    cudaMalloc(&in, 1024 * 4);
    cudaMemset(in, 0, 1024 * 4);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096, threads = 1024;
    const char *names[3] = {"F2F.F64.F32", "DADD", "cvt,cvt,dsub,dmul,dadd step"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) kern<0><<<148, threads>>>(in, out, iters, cyc);
            if (mode == 1) kern<1><<<148, threads>>>(in, out, iters, cyc);
            if (mode == 2) kern<2><<<148, threads>>>(in, out, iters, cyc);
            cudaDeviceSynchronize();
        }
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double m = 0;
        for (int b = 0; b < 148; ++b) m += h[b];
        m /= 148;
        const double ops = double(threads) * iters * 8;
        printf("%-32s %.1f per SM per clock (%.0f cycles)\n", names[mode], ops / m, m);
    }
    for (int mode = 0; mode < 2; ++mode) {
        if (mode == 0) lat<0><<<1, 32>>>(in, out, iters, cyc);
        else lat<1><<<1, 32>>>(in, out, iters, cyc);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        printf("latency %-20s %.1f cycles per dependent step\n", mode == 0 ? "DADD" : "exact step", double(h) / iters);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
