// dependent-chain latency (cycles) of FADD, FADD2, FMUL2(reg), FFMA2 on one warp
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b){unsigned long long r; asm volatile("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b){unsigned long long r; asm volatile("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
template<int MODE> __global__ void k(float* out, long long* cyc, int iters, float s0){
  float a = s0*threadIdx.x, b = s0; unsigned long long p, q;
  asm("mov.b64 %0, {%1,%2};":"=l"(p):"f"(a),"f"(b)); q = p;
  long long t0 = clock64();
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<32;i++){
      if(MODE==0){ asm volatile("add.rn.f32 %0, %0, %1;":"+f"(a):"f"(b)); }
      else if(MODE==1){ p = add2(p, q); }
      else if(MODE==2){ p = mul2(p, q); }
      else { asm volatile("mul.rn.f32 %0, %0, 0f3E800000;":"+f"(a)); }
    }
  }
  long long t1 = clock64();
  float x,y; asm("mov.b64 {%0,%1}, %2;":"=f"(x),"=f"(y):"l"(p));
  out[threadIdx.x] = a + x + y; if(threadIdx.x==0) cyc[MODE] = t1-t0;
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  int iters=1000;
  k<0><<<1,32>>>(o,c,iters,1e-7f); k<1><<<1,32>>>(o,c,iters,1e-7f); k<2><<<1,32>>>(o,c,iters,1.0f); k<3><<<1,32>>>(o,c,iters,1.0f);
  long long h[4]; cudaMemcpy(h,c,32,cudaMemcpyDeviceToHost);
  const char* nm[4]={"FADD","FADD2","FMUL2","FMUL imm"};
  for(int m=0;m<4;m++) printf("%s latency %.2f cycles\n", nm[m], (double)h[m]/(iters*32));
  return 0;
}
