// FP64 pipe probe for B200 (sm_100a): DFMA peak, DMMA (f64 mma.sync) peak, and
// whether the two overlap (separate pipes) when issued from the same warps.
// Also times CUDA's fp64 exp()+sqrt() per element.  Output: one line per test.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int ITERS>
__global__ void dfma_k(double* out, double s){
  double a[8];
  #pragma unroll
  for(int j=0;j<8;j++) a[j]=threadIdx.x*1e-3+j;
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int j=0;j<8;j++) a[j]=fma(a[j],s,0.5);
  }
  double t=0; for(int j=0;j<8;j++) t+=a[j];
  if(t==123.456) out[0]=t;
}
__device__ __forceinline__ void dmma(double& c0,double& c1,double a,double b){
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0),"+d"(c1) : "d"(a),"d"(b));
}
template<int ITERS>
__global__ void dmma_k(double* out, double s){
  double c[16]; double a=threadIdx.x*1e-3, b=s;
  #pragma unroll
  for(int j=0;j<16;j++) c[j]=0;
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int j=0;j<8;j++) dmma(c[2*j],c[2*j+1],a,b);
  }
  double t=0; for(int j=0;j<16;j++) t+=c[j];
  if(t==123.456) out[0]=t;
}
// both: per iteration 8 DMMA (8*256 FMA per warp) + NF DFMA per thread
template<int ITERS,int NF>
__global__ void mix_k(double* out, double s){
  double c[16]; double a=threadIdx.x*1e-3, b=s; double f[8];
  #pragma unroll
  for(int j=0;j<16;j++) c[j]=0;
  #pragma unroll
  for(int j=0;j<8;j++) f[j]=j;
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int j=0;j<8;j++) dmma(c[2*j],c[2*j+1],a,b);
    #pragma unroll
    for(int r=0;r<NF/8;r++)
    #pragma unroll
    for(int j=0;j<8;j++) f[j]=fma(f[j],s,0.5);
  }
  double t=0; for(int j=0;j<16;j++) t+=c[j]; for(int j=0;j<8;j++) t+=f[j];
  if(t==123.456) out[0]=t;
}
__global__ void expsqrt_k(double* out, const double* in, int n, int reps){
  int i=blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  double x=in[i], acc=0;
  for(int r=0;r<reps;r++){ double u=fma(-x,x,1.0); acc+=exp(18.4*(sqrt(fmax(u,0.0))-1.0)); x=x*0.999+1e-4; }
  out[i]=acc;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* d; CK(cudaMalloc(&d, 1<<26));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int SM=p.multiProcessorCount;
  for(int bpsm : {4,8,16}){
    int blocks=SM*bpsm, threads=256; const int IT=4096;
    dfma_k<IT><<<blocks,threads>>>(d,0.999); cudaEventRecord(e0);
    for(int r=0;r<5;r++) dfma_k<IT><<<blocks,threads>>>(d,0.999);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double fl=5.0*blocks*threads*(double)IT*8*2; printf("DFMA  blocks/SM=%d  %.2f TFLOP/s\n",bpsm, fl/(ms*1e-3)/1e12);
  }
  for(int bpsm : {4,8,16}){
    int blocks=SM*bpsm, threads=256; const int IT=2048;
    dmma_k<IT><<<blocks,threads>>>(d,0.999); cudaEventRecord(e0);
    for(int r=0;r<5;r++) dmma_k<IT><<<blocks,threads>>>(d,0.999);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double fl=5.0*blocks*(threads/32)*(double)IT*8*256*2; printf("DMMA  blocks/SM=%d  %.2f TFLOP/s\n",bpsm, fl/(ms*1e-3)/1e12);
  }
  {
    int blocks=SM*8, threads=256; const int IT=2048;
    #define MIX(NF) { mix_k<IT,NF><<<blocks,threads>>>(d,0.999); cudaEventRecord(e0); \
      for(int r=0;r<5;r++) mix_k<IT,NF><<<blocks,threads>>>(d,0.999); \
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); \
      double t_mma=5.0*blocks*(threads/32)*(double)IT*8*256*2, t_f=5.0*blocks*threads*(double)IT*NF*2; \
      printf("MIX NF=%d  dmma %.2f + dfma %.2f = %.2f TFLOP/s (%.3f ms)\n",NF,t_mma/(ms*1e-3)/1e12,t_f/(ms*1e-3)/1e12,(t_mma+t_f)/(ms*1e-3)/1e12, ms/5); }
    MIX(8) MIX(16) MIX(32) MIX(64)
  }
  {
    int n=SM*2048; int reps=64;
    expsqrt_k<<<(n+255)/256,256>>>(d,d,n,reps); cudaEventRecord(e0);
    for(int r=0;r<5;r++) expsqrt_k<<<(n+255)/256,256>>>(d,d+n,n,reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double ev=5.0*n*(double)reps; printf("exp+sqrt fp64: %.2f G/s  (%.2f ps each)\n", ev/(ms*1e-3)/1e9, ms*1e9/ev);
  }
  CK(cudaGetLastError());
  return 0;
}
