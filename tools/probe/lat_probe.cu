// Latency / throughput probe (tool): dependent DFMA chain, LDS->DFMA chain, shfl chain, and
// named-barrier round trip, for 1..16 warps per SM.  Prints JSON lines.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x = threadIdx.x * 1e-3, y = x + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x + y;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0);
}
__global__ void k_dfma_ilp2(double* out, int iters, double a, double b) {
    double x = threadIdx.x * 1e-3, y = x + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) { x = fma(x, a, b); y = fma(y, a, b); }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x + y;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0);
}
__global__ void k_shfl(double* out, int iters) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0);
}
__global__ void k_lds(double* out, int iters) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0.0;
    __syncthreads();
    double x = 0.0;
    int idx = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) { x = fma(s[idx], 1.0, x); idx = (idx + (int)x) & 1023; }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0);
}
__global__ void k_bar(double* out, int iters) {
    __shared__ double s[2][256];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        s[i & 1][threadIdx.x] = x;
        asm volatile("bar.sync 1, 64;" ::: "memory");
        x = s[i & 1][threadIdx.x ^ 1] + 1.0;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
}
int main() {
    double* d; cudaMalloc(&d, 1 << 24);
    for (int w : {1, 4, 8, 16}) {
        double h;
        k_dfma<<<148, 32 * w>>>(d, 1000, 0.999, 1e-3); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"dfma_chain\", \"warps\": %d, \"cyc_per_op\": %.2f}\n", w, h);
        k_dfma_ilp2<<<148, 32 * w>>>(d, 1000, 0.999, 1e-3); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"dfma_ilp2\", \"warps\": %d, \"cyc_per_pair\": %.2f}\n", w, h);
        k_shfl<<<148, 32 * w>>>(d, 1000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"shfl_dadd_chain\", \"warps\": %d, \"cyc_per_op\": %.2f}\n", w, h);
        k_lds<<<148, 32 * w>>>(d, 1000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"lds_dfma_chain\", \"warps\": %d, \"cyc_per_op\": %.2f}\n", w, h);
        if (w >= 2) { k_bar<<<148, 32 * w>>>(d, 1000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"sts_bar64_lds\", \"warps\": %d, \"cyc_per_step\": %.2f}\n", w, h); }
    }
    return 0;
}
