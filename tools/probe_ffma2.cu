// Dev probe: issue throughput of scalar FADD+FFMA vs packed FADD2+FFMA2 on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 sub2(u64 a, u64 b){u64 d; asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 fma2(u64 a, u64 c){u64 d; asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(a), "l"(c)); return d;}
template<int ACC> __global__ void scalar_k(float* out, float q0, int iters){
  float acc[ACC]; float r[ACC];
  for(int i=0;i<ACC;++i){acc[i]=0; r[i]=threadIdx.x*0.001f+i;}
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<ACC;++i){ float t=__fsub_rn(q0+it*1e-7f, r[i]); acc[i]=__fmaf_rn(t,t,acc[i]); }
  }
  float s=0; for(int i=0;i<ACC;++i) s+=acc[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int ACC> __global__ void packed_k(float* out, float q0, int iters){
  u64 acc[ACC/2]; u64 r[ACC/2];
  for(int i=0;i<ACC/2;++i){acc[i]=0; float2 v=make_float2(threadIdx.x*0.001f+2*i, threadIdx.x*0.001f+2*i+1); r[i]=*(u64*)&v;}
  for(int it=0; it<iters; ++it){
    float qq=q0+it*1e-7f; float2 qv=make_float2(qq,qq); u64 q=*(u64*)&qv;
#pragma unroll
    for(int i=0;i<ACC/2;++i){ u64 t=sub2(q, r[i]); acc[i]=fma2(t,acc[i]); }
  }
  float s=0; for(int i=0;i<ACC/2;++i){float2 v=*(float2*)&acc[i]; s+=v.x+v.y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*256*4); cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters=20000; const int blocks=148*4, th=256; float ms;
  for(int rep=0;rep<2;++rep){
  cudaEventRecord(a); scalar_k<32><<<blocks,th>>>(o,1.f,iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  double steps=double(blocks)*th*iters*32; printf("scalar: %.3f ms  %.2f Tstep/s\n", ms, steps/ms/1e9);
  cudaEventRecord(a); packed_k<32><<<blocks,th>>>(o,1.f,iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("packed: %.3f ms  %.2f Tstep/s\n", ms, steps/ms/1e9);
  }
  return 0;
}
