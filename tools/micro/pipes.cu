// Throughput microbenchmark: cycles per warp-instruction per SMSP for MUFU.EX2, F2FP pack, FFMA2, mixes.
#include <cstdio>
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned pk(float a, float b){ __half2 h=__floats2half2_rn(a,b); return *(unsigned*)&h; }
__device__ __forceinline__ float ex2(float x){ float y; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x)); return y; }
template<int MODE>
__global__ void k(float* out, long long* cyc, int iters){
  float a[8]; unsigned u[8];
  for(int i=0;i<8;i++){ a[i]=threadIdx.x*1e-3f+i*0.1f; u[i]=i; }
  __syncwarp();
  long long t0=clock64();
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;i++){
      if(MODE==0) a[i]=ex2(a[i])*0.5f;                 // MUFU (+FMUL)
      if(MODE==1) u[i]^=pk(a[i], a[(i+1)&7]);          // F2FP only
      if(MODE==2){ a[i]=ex2(a[i])*0.5f; u[i]^=pk(a[i],a[(i+3)&7]); } // both
      if(MODE==3) a[i]=a[i]*0.999f+0.5f;               // FFMA
    }
  }
  long long t1=clock64();
  float s=0; for(int i=0;i<8;i++) s+=a[i]+u[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 1<<24); cudaMalloc(&c, 1<<16);
  int iters=4096;
  for(int warps=4; warps<=16; warps*=2){
   for(int mode=0; mode<4; ++mode){
    auto f = mode==0?k<0>:mode==1?k<1>:mode==2?k<2>:k<3>;
    f<<<148, warps*32>>>(o,c,iters); cudaDeviceSynchronize();
    f<<<148, warps*32>>>(o,c,iters); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost);
    double per = (double)h/(iters*8.0); // cycles per (instr-group) per warp
    printf("warps/SM=%2d mode=%d cycles per op-group per warp=%.2f -> per SMSP per warp-instr=%.2f\n", warps, mode, per, per/(warps/4.0));
   }
  }
  return 0;
}
