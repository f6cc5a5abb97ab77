#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
template <int KIND>
__global__ void probe(u64 *out, int iters, uint32_t seed) {
    uint32_t a = threadIdx.x * 2654435761u + seed, b = a ^ 0x9e3779b9u;
    double f[8]; uint32_t r[8]; u64 v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) { f[j] = (a + j) * 1e-9; r[j] = b + j; v[j] = ((u64)a << 20) + j; }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (KIND == 0) f[j] = fma(f[j], 1.0000001, 1e-12 * i);            // DFMA
            else if (KIND == 1) r[j] = __umulhi(r[j], a + i) + b;             // IMAD.HI
            else if (KIND == 2) { double d = (double)(v[j] + i); v[j] = (u64)(d * 0.999999); } // I2F + DMUL + F2I
            else if (KIND == 3) { float x = __uint_as_float(r[j]); r[j] = __float_as_uint(fmaf(x, 1.0001f, 1e-7f)); } // FFMA
        }
    }
    u64 s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += (u64)f[j] + r[j] + v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    u64 *d; cudaMalloc(&d, 148 * 8 * 1024 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[] = {"DFMA", "IMAD.HI", "I2F+DMUL+F2I", "FFMA"};
    for (int kind = 0; kind < 4; kind++) {
        for (int rep = 0; rep < 2; rep++) {
            int iters = 2048, blocks = 148 * 8, threads = 256;
            cudaEventRecord(e0);
            if (kind == 0) probe<0><<<blocks, threads>>>(d, iters, rep);
            if (kind == 1) probe<1><<<blocks, threads>>>(d, iters, rep);
            if (kind == 2) probe<2><<<blocks, threads>>>(d, iters, rep);
            if (kind == 3) probe<3><<<blocks, threads>>>(d, iters, rep);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads * iters * 8;
            if (rep) printf("%-14s %.3f ms  %.2f Tops/s  %.1f ops/clk/SM @1.965GHz\n", names[kind], ms, ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
