// Microbenchmark: dependent shared-memory pointer chase, cycles per step for a few loop shapes.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chase(int n, int variant, long long* out, int* sink) {
    extern __shared__ short win[];
    for (int i = threadIdx.x; i < 90112; i += blockDim.x) win[i] = (short)((1 + 256 * ((i / 7) & 1)) << 3);  // offsets 1 or 257
    __syncthreads();
    if (threadIdx.x != 0) return;
    int pos = 0, acc = 0;
    long long t0 = clock64();
    if (variant == 0) {  // plain dependent chain
        for (int k = 0; k < n; ++k) { int e = win[pos]; pos += e >> 3; if (pos > 80000) pos -= 80000; }
    } else if (variant == 1) {  // no wrap
        for (int k = 0; k < n; ++k) { int e = win[pos & 65535]; pos += e >> 3; }
    } else {  // unrolled x4 with OR
        for (int k = 0; k < n; k += 4) {
            int e0 = win[pos & 65535]; int p1 = pos + (e0 >> 3);
            int e1 = win[p1 & 65535]; int p2 = p1 + (e1 >> 3);
            int e2 = win[p2 & 65535]; int p3 = p2 + (e2 >> 3);
            int e3 = win[p3 & 65535]; pos = p3 + (e3 >> 3);
            acc |= e0 | e1 | e2 | e3;
        }
    }
    long long t1 = clock64();
    out[variant] = t1 - t0;
    sink[0] = pos + acc;
}
int main() {
    long long* d; int* s; cudaMalloc(&d, 64); cudaMalloc(&s, 4);
    cudaFuncSetAttribute(chase, cudaFuncAttributeMaxDynamicSharedMemorySize, 180224);
    for (int v = 0; v < 3; ++v) chase<<<1, 256, 180224>>>(100000, v, d, s);
    long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 3; ++v) printf("variant %d: %.1f cycles/step\n", v, h[v] / 100000.0);
    return 0;
}
