// Dependent-chain latency of the instructions the ray caster's traversal
// uses, measured with clock64 in one thread (development tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/ubench_latency.cu -o ubench
#include <cstdio>

__global__ void chains(double *out, long long *cyc, double seed, int iters, float fseed) {
    double a = seed, b = seed * 0.5 + 1.0;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = a + b;
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = a * b;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, b);
    t1 = clock64();
    cyc[2] = t1 - t0;
    // F2I + I2F round trip
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = (double)((int)a + 1);
    t1 = clock64();
    cyc[3] = t1 - t0;
    // floor chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = floor(a + 0.5);
    t1 = clock64();
    cyc[4] = t1 - t0;
    // DSETP -> select chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = (a < b) ? a + 1.0 : a - 1.0;
    t1 = clock64();
    cyc[5] = t1 - t0;
    // FP32 FADD chain for comparison
    float f = fseed;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) f = f + fseed;
    t1 = clock64();
    cyc[6] = t1 - t0;
    // double division chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = b / a;
    t1 = clock64();
    cyc[7] = t1 - t0;
    out[0] = a + f;
}

__global__ void pointer_chase(const long long *next, long long start, int iters, long long *cyc, long long *sink) {
    long long p = start;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = __ldg(next + p);
    long long t1 = clock64();
    cyc[0] = t1 - t0;
    *sink = p;
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMallocManaged(&cyc, 16 * 8);
    const int iters = 4096;
    chains<<<1, 1>>>(out, cyc, 1.0000001, iters, 1.0f);
    chains<<<1, 1>>>(out, cyc, 1.0000001, iters, 1.0f);
    cudaDeviceSynchronize();
    const char *names[] = {"DADD", "DMUL", "DFMA", "F2I+I2F(f64)", "DADD+floor", "DSETP+sel+DADD", "FADD", "DDIV"};
    for (int k = 0; k < 8; ++k) printf("%-16s %6.1f cycles/op\n", names[k], (double)cyc[k] / iters);
    // L1-resident and L2-resident pointer chases
    for (long long bytes : {16LL << 10, 4LL << 20, 512LL << 20}) {
        long long n = bytes / 8;
        long long *next;
        cudaMallocManaged(&next, bytes);
        long long stride = 37;  // 296 bytes: a new line every hop
        for (long long i = 0; i < n; ++i) next[i] = (i + stride) % n;
        long long *sink;
        cudaMalloc(&sink, 8);
        pointer_chase<<<1, 1>>>(next, 0, 2048, cyc, sink);
        pointer_chase<<<1, 1>>>(next, 0, 2048, cyc, sink);
        cudaDeviceSynchronize();
        printf("LDG chase over %8lld KiB: %6.1f cycles/load\n", bytes >> 10, (double)cyc[0] / 2048);
        cudaFree(next);
        cudaFree(sink);
    }
    return 0;
}
