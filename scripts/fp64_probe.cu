// Scalar fp64 throughput / latency probe (DFMA, DMUL) on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_probe.cu -o fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void fma_tp(double *out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void mul_tp(double *out, int iters, double a) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i + 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dmul_rn(x[i], a);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int it = 20000;
    auto F8 = [&](int bl, int th) {
        double *out; cudaMalloc(&out, 8);
        fma_tp<8><<<bl, th>>>(out, 10, 1.0000001, 1e-9);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); fma_tp<8><<<bl, th>>>(out, it, 1.0000001, 1e-9); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)bl * th * it * 8;
        printf("DFMA ILP8  grid %5d x %4d: %8.3f ms  %8.1f G DFMA/s = %.1f per clk per SM (1.965 GHz)\n", bl, th, ms, ops / ms / 1e6, ops / ms / 1e6 / 1.965 / sms);
    };
    auto F1 = [&](int bl, int th) {
        double *out; cudaMalloc(&out, 8);
        fma_tp<1><<<bl, th>>>(out, 10, 1.0000001, 1e-9);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); fma_tp<1><<<bl, th>>>(out, it, 1.0000001, 1e-9); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        printf("DFMA chain grid %5d x %4d: %8.3f ms  latency %.1f cycles per dependent DFMA\n", bl, th, ms, ms * 1e-3 * 1.965e9 / it);
    };
    auto M8 = [&](int bl, int th) {
        double *out; cudaMalloc(&out, 8);
        mul_tp<8><<<bl, th>>>(out, 10, 1.0000001);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); mul_tp<8><<<bl, th>>>(out, it, 1.0000001); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)bl * th * it * 8;
        printf("DMUL ILP8  grid %5d x %4d: %8.3f ms  %8.1f G DMUL/s = %.1f per clk per SM\n", bl, th, ms, ops / ms / 1e6, ops / ms / 1e6 / 1.965 / sms);
    };
    F1(1, 32);
    F8(sms * 4, 256);
    F8(sms * 8, 256);
    M8(sms * 8, 256);
    return 0;
}
