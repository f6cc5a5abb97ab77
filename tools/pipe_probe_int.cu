// pipe throughput probe: independent chains of IMAD.WIDE.U32 / IMAD / IADD3 per thread
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
template <int KIND>
__global__ void probe(u64 *out, int iters, uint32_t seed) {
    uint32_t a = threadIdx.x * 2654435761u + seed, b = a ^ 0x9e3779b9u;
    u64 acc[8];
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) { acc[j] = a + j; r[j] = b + j; }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (KIND == 0) acc[j] = (u64)r[j] * (a + i) + acc[j];          // IMAD.WIDE.U32
            else if (KIND == 1) r[j] = r[j] * (a + i) + b;                  // IMAD
            else if (KIND == 2) r[j] = r[j] + (a ^ i) + b;                 // IADD3
            else if (KIND == 3) { acc[j] = acc[j] + (u64)(r[j] ^ i); }      // 64-bit add (IADD3 + IADD3.X)
        }
    }
    u64 s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += acc[j] + r[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    u64 *d; cudaMalloc(&d, 148 * 8 * 1024 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[] = {"IMAD.WIDE.U32", "IMAD", "IADD3", "add64"};
    for (int kind = 0; kind < 4; kind++) {
        for (int rep = 0; rep < 2; rep++) {
            int iters = 4096, blocks = 148 * 8, threads = 256;
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
