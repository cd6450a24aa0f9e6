// Dependent-chain latency of FP64 ops on this GPU (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ double ddiv_ieee(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double aa = fabs(a);
    const double q0 = __dmul_rn(a, rb);
    const double r = __fma_rn(-q0, b, a);
    const double q1 = __fma_rn(r, rb, q0);
    if (!(aa >= 0x1p-900 && aa <= 0x1p+900)) return ddiv_ieee(a, b);
    return q1;
}

__global__ void k(double *out, long long *cyc, double x0, double y, int n) {
    double x = x0;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
    t1 = clock64(); cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fma_rn(x, y, y);
    t1 = clock64(); cyc[2] = t1 - t0;
    // div_rn chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = div_rn(x, 1.0000001, 1.0 / 1.0000001);
    t1 = clock64(); cyc[3] = t1 - t0;
    // __ddiv_rn chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(x, 1.0000001);
    t1 = clock64(); cyc[4] = t1 - t0;
    // DSETP + select chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x > y ? x - y : x + y;
    t1 = clock64(); cyc[5] = t1 - t0;
    // shared load chain
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = x;
    __syncthreads();
    int idx = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = (int)sm[idx & 63] & 63;
    t1 = clock64(); cyc[6] = t1 - t0;
    out[0] = x + idx;
}

int main() {
    double *o; long long *c;
    cudaMalloc(&o, 8); cudaMalloc(&c, 8 * 8);
    const int n = 4096;
    k<<<1, 1>>>(o, c, 1.0, 1e-9, n);
    k<<<1, 1>>>(o, c, 1.0, 1e-9, n);
    long long h[8];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char *nm[] = {"DADD", "DMUL", "DFMA", "div_rn (Markstein)", "__ddiv_rn", "DSETP+select", "LDS dep"};
    for (int i = 0; i < 7; ++i) printf("%-20s %.1f cycles/op\n", nm[i], (double)h[i] / n);
    return 0;
}
