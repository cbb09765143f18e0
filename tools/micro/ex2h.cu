// Throughput of MUFU.EX2 variants per SMSP: f32 vs packed f16x2 (two results per instruction?).
#include <cstdio>
#include <cuda_fp16.h>
__device__ __forceinline__ float ex2f(float x){ float y; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x)); return y; }
__device__ __forceinline__ unsigned ex2h2(unsigned x){ unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;":"=r"(y):"r"(x)); return y; }
template<int MODE>
__global__ void k(float* out, long long* cyc, int iters){
  float a[8]; unsigned u[8];
  for(int i=0;i<8;i++){ a[i]=-(threadIdx.x*1e-3f+i*0.1f); __half2 h=__floats2half2_rn(a[i], a[i]*0.5f); u[i]=*(unsigned*)&h; }
  __syncwarp();
  long long t0=clock64();
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;i++){
      if(MODE==0) a[i]=ex2f(a[i]);
      if(MODE==1) u[i]=ex2h2(u[i]) ^ 0x80008000u;   // keep inputs negative
    }
  }
  long long t1=clock64();
  float s=0; for(int i=0;i<8;i++) s+=a[i]+(float)u[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 1<<24); cudaMalloc(&c, 1<<16);
  int iters=4096;
  for(int warps=4; warps<=16; warps*=2){
   for(int mode=0; mode<2; ++mode){
    auto f = mode==0?k<0>:k<1>;
    f<<<148, warps*32>>>(o,c,iters); cudaDeviceSynchronize();
    f<<<148, warps*32>>>(o,c,iters); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost);
    double per = (double)h/(iters*8.0);
    printf("warps/SM=%2d %s: cycles per warp-instr per SMSP=%.2f (results/clk/SMSP=%.2f)\n", warps,
           mode==0?"ex2.f32  ":"ex2.f16x2", per/(warps/4.0), (mode==0?32.0:64.0)/(per/(warps/4.0)));
   }
  }
  return 0;
}
