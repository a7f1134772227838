// microbenchmark: issue cost of FADD (3-reg, |abs|) vs FADD2 vs FMUL2 per warp instruction
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b){unsigned long long r; asm volatile("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
template<int MODE>
__global__ void k(float* out, int iters, float s0){
  float a[16]; unsigned long long p[8];
  for(int i=0;i<16;i++) a[i]=s0*(threadIdx.x+i);
  for(int i=0;i<8;i++){ asm("mov.b64 %0, {%1,%2};":"=l"(p[i]):"f"(a[2*i]),"f"(a[2*i+1])); }
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++){
      if(MODE==0){ a[i] = fabsf(a[i]) + fabsf(a[(i+1)&15]); }
      else if(MODE==1){ if(i<8) p[i]=add2(p[i],p[(i+1)&7]); }
      else { a[i] = a[i] + a[(i+1)&15]; }
    }
  }
  float s=0; for(int i=0;i<16;i++) s+=a[i];
  for(int i=0;i<8;i++){float x,y; asm("mov.b64 {%0,%1}, %2;":"=f"(x),"=f"(y):"l"(p[i])); s+=x+y;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*256*4);
  int iters=20000;
  for(int mode=0;mode<3;mode++){
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0);
    if(mode==0) k<0><<<148*8,256>>>(o,iters,1e-7f);
    if(mode==1) k<1><<<148*8,256>>>(o,iters,1e-7f);
    if(mode==2) k<2><<<148*8,256>>>(o,iters,1e-7f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double warp_instr = (double)148*8*8*iters*(mode==1?8:16);
    double lanes_ops = warp_instr*32*(mode==1?2:1);
    if(rep) printf("mode %d (%s): %.3f ms, %.2f Twarp-instr/s, %.2f T fp32 adds/s\n", mode, mode==0?"FADD |a|+|b|":mode==1?"FADD2":"FADD", ms, warp_instr/ms/1e9, lanes_ops/ms/1e9);
    }
  }
  return 0;
}
