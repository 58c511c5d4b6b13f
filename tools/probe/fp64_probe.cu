// Hardware probe: FP64 DMMA (mma.sync .f64) and DFMA issue throughput on sm_100a.
// Not part of the product path; used once to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int SHAPE> __device__ __forceinline__ void mma_step(double (&c)[8][4], const double* a, const double* b);

// m16n8k4: A 2 regs, B 1 reg, C 4 regs
template<> __device__ __forceinline__ void mma_step<4>(double (&c)[8][4], const double* a, const double* b){
#pragma unroll
  for(int t=0;t<8;t++)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[t][0]),"+d"(c[t][1]),"+d"(c[t][2]),"+d"(c[t][3]) : "d"(a[0]),"d"(a[1]),"d"(b[t&1]));
}
// m16n8k8: A 4 regs, B 2 regs
template<> __device__ __forceinline__ void mma_step<8>(double (&c)[8][4], const double* a, const double* b){
#pragma unroll
  for(int t=0;t<8;t++)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+d"(c[t][0]),"+d"(c[t][1]),"+d"(c[t][2]),"+d"(c[t][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(b[0]),"d"(b[1]));
}
// m16n8k16: A 8 regs, B 4 regs
template<> __device__ __forceinline__ void mma_step<16>(double (&c)[8][4], const double* a, const double* b){
#pragma unroll
  for(int t=0;t<8;t++)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[t][0]),"+d"(c[t][1]),"+d"(c[t][2]),"+d"(c[t][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),"d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
}
// m8n8k4: A 1 reg, B 1 reg, C 2 regs
__global__ void k_m8(double* out, int iters){
  double c[8][2]={}; double a=threadIdx.x*1e-3, b=1.0+threadIdx.x*1e-4;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int t=0;t<8;t++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[t][0]),"+d"(c[t][1]) : "d"(a),"d"(b));
  }
  double s=0; for(int t=0;t<8;t++) s+=c[t][0]+c[t][1];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int SHAPE> __global__ void k_mma(double* out, int iters){
  double c[8][4]={}; double a[8], b[4];
  for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i; for(int i=0;i<4;i++) b[i]=1.0+i*1e-4;
  for(int i=0;i<iters;i++) mma_step<SHAPE>(c,a,b);
  double s=0; for(int t=0;t<8;t++) s+=c[t][0]+c[t][1]+c[t][2]+c[t][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_dfma(double* out, int iters){
  double c[16]; double a=1.0+threadIdx.x*1e-9, b=1e-9;
  for(int i=0;i<16;i++) c[i]=i;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int t=0;t<16;t++) c[t]=fma(c[t],a,b);
  }
  double s=0; for(int t=0;t<16;t++) s+=c[t];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; CK(cudaMalloc(&out, sizeof(double)*sms*16*1024));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for(int warps : {4, 8, 16, 32}){
    int th=32*warps; int iters=20000;
    float ms;
    // DFMA: per thread 16*iters FMA
    k_dfma<<<sms*2,th>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_dfma<<<sms*2,th>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*16*iters*(double)th*sms*2; printf(", \"dfma_w%d_tflops\": %.2f", warps, fl/ms/1e9);
    // m8n8k4: 256 FMA per warp-instr
    k_m8<<<sms*2,th>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_m8<<<sms*2,th>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=2.0*8*256*iters*(double)warps*sms*2; printf(", \"m8n8k4_w%d_tflops\": %.2f", warps, fl/ms/1e9);
    k_mma<4><<<sms*2,th>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_mma<4><<<sms*2,th>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=2.0*8*512*iters*(double)warps*sms*2; printf(", \"m16n8k4_w%d_tflops\": %.2f", warps, fl/ms/1e9);
    k_mma<8><<<sms*2,th>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_mma<8><<<sms*2,th>>>(out,iters/2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=2.0*8*1024*(iters/2)*(double)warps*sms*2; printf(", \"m16n8k8_w%d_tflops\": %.2f", warps, fl/ms/1e9);
    k_mma<16><<<sms*2,th>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_mma<16><<<sms*2,th>>>(out,iters/4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=2.0*8*2048*(iters/4)*(double)warps*sms*2; printf(", \"m16n8k16_w%d_tflops\": %.2f", warps, fl/ms/1e9);
  }
  printf("}\n");
  return 0;
}
