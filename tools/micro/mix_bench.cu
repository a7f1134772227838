// FP32-pipe throughput of packed vs scalar ops at a given occupancy (warps per SMSP):
// mode 0 FADD2 (independent), 1 FMUL2 by a register pair, 2 FMUL2 by an immediate,
// 3 the packed half-sweep mix (2 FADD + 2 FADD2 + FMUL2, 8 independent chains),
// 4 the scalar half-sweep mix (6 FADD |.| + 2 FMUL imm, 8 chains)
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 mul2(u64 a, u64 b){u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 mul2i(u64 a){u64 r; asm("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(0x3E8000003E800000ull)); return r;}
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
template<int MODE> __global__ void k(float* out, int iters, float s0){
  u64 p[8]; float a[8], b[8]; u64 m = pk(0.25f, 0.25f);
  for(int i=0;i<8;i++){ a[i]=s0*(threadIdx.x+i); b[i]=s0*i; p[i]=pk(a[i],b[i]); }
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<8;i++){
      if(MODE==0){ p[i]=add2(p[i],p[(i+3)&7]); }
      else if(MODE==1){ p[i]=mul2(p[i],m); }
      else if(MODE==2){ p[i]=mul2i(p[i]); }
      else if(MODE==3){ float x=a[i]+b[i]; float y=b[i]+a[(i+1)&7]; u64 ew=pk(x,y); u64 ns=add2(p[i],p[(i+1)&7]); p[i]=mul2(add2(ew,ns),m); a[i]=x; }
      else { float e=fabsf(a[i])+fabsf(b[i]); float n=fabsf(a[(i+1)&7])+fabsf(b[(i+2)&7]); a[i]=0.25f*(e+n);
             float e2=fabsf(b[i])+fabsf(a[i]); float n2=fabsf(b[(i+1)&7])+fabsf(a[(i+2)&7]); b[i]=0.25f*(e2+n2); }
    }
  }
  float s=0; for(int i=0;i<8;i++){float x,y; asm("mov.b64 {%0,%1}, %2;":"=f"(x),"=f"(y):"l"(p[i])); s+=x+y+a[i]+b[i];}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int MODE> void run(const char* nm, float* o, int wps, double fp32_cycles_per_iter_per_warp){
  int iters=4000; int threads = 128; int blocks = 148*wps; // 4 warps/block = 1 warp per SMSP per block
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks,threads>>>(o,iters,1e-3f);
  cudaEventRecord(e0); k<MODE><<<blocks,threads>>>(o,iters,1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double cyc = ms*1e-3*1.9e9; double need = fp32_cycles_per_iter_per_warp*iters*wps;
  printf("%-34s warps/SMSP=%d  %.3f ms  fp32-pipe utilisation (at 2 cyc/packed, 1/scalar) %.2f\n", nm, wps, ms, need/cyc);
}
int main(){
  float* o; cudaMalloc(&o, 148*16*128*4);
  for(int w: {2,4,8}){
    run<0>("FADD2 x8", o, w, 16);
    run<1>("FMUL2 reg x8", o, w, 16);
    run<2>("FMUL2 imm x8", o, w, 16);
    run<3>("packed hs mix x8 (2F+2F2+FM2)", o, w, 8*8);
    run<4>("scalar hs mix x8 (2x(4F+1FMUL))", o, w, 8*10);
  }
  return 0;
}
