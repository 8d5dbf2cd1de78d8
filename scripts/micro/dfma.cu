#include <cstdio>
__global__ void k(double *o, double x, double y, long long *t) {
    double a = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 512; ++i) a = fma(x, y, a);
    long long t1 = clock64();
    o[threadIdx.x] = a;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k2(double *o, const float *xs, double y, long long *t) {
    double a = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < 512; ++i) a = fma((double)xs[i & 63], y, a);
    long long t1 = clock64();
    o[threadIdx.x] = a;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
    double *o; long long *t; float *xs;
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&t, 8); cudaMalloc(&xs, 256);
    cudaMemset(xs, 0, 256);
    long long h;
    for (int th : {32, 256, 1024}) {
        k<<<1, th>>>(o, 1.0000001, 0.9999999, t); cudaDeviceSynchronize();
        k<<<1, th>>>(o, 1.0000001, 0.9999999, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("threads %d: 512 dependent DFMA = %lld cycles (%.1f per DFMA)\n", th, h, h / 512.0);
        k2<<<1, th>>>(o, xs, 0.9999999, t); cudaDeviceSynchronize();
        k2<<<1, th>>>(o, xs, 0.9999999, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("threads %d: 512 dependent DFMA with F2F from global = %lld cycles (%.1f per step)\n", th, h, h / 512.0);
    }
    return 0;
}
