// DRAM access-pattern probe (development tool): read + write 2^16-word limbs in the column pattern of
// the NTT's strided pass (SC consecutive words from each of 256 rows 2 KB apart per CTA) versus a
// streaming copy.  Reports GB/s of (read + write) bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dram_probe tools/dram_probe.cu && /tmp/dram_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

template <int SC>
__global__ void strided(const u64 *__restrict__ in, u64 *__restrict__ out) {
    // CTA: SC columns x 256 rows of one limb; thread (cl, tau): column cl, rows tau + 16 k
    const int cl = threadIdx.x % SC, tau = threadIdx.x / SC;
    const long limb = blockIdx.y;
    const long base = limb * 65536 + blockIdx.x * SC + cl;
    u64 v[16];
#pragma unroll
    for (int k = 0; k < 16; k++) v[k] = in[base + 256L * (tau + 16 * k)];
#pragma unroll
    for (int k = 0; k < 16; k++) out[base + 256L * (tau + 16 * k)] = v[k] + 1;
}
__global__ void stream(const ulonglong2 *__restrict__ in, ulonglong2 *__restrict__ out, long n2) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
        ulonglong2 x = in[i];
        x.x += 1;
        out[i] = x;
    }
}
int main() {
    const long limbs = 2048, n = limbs * 65536;
    u64 *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto report = [&](const char *name, auto launch) {
        for (int w = 0; w < 3; w++) launch();
        cudaEventRecord(e0);
        for (int r = 0; r < 10; r++) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.1f GB/s\n", name, 2.0 * n * 8 * 10 / (ms / 1e3) / 1e9);
    };
    report("stream copy (16 B/thread)", [&] { stream<<<148 * 8, 256>>>((ulonglong2 *)a, (ulonglong2 *)b, n / 2); });
    report("strided SC=16 (128 B rows)", [&] { strided<16><<<dim3(65536 / 256 / 16, limbs), 256>>>(a, b); });
    report("strided SC=32 (256 B rows)", [&] { strided<32><<<dim3(65536 / 256 / 32, limbs), 512>>>(a, b); });
    report("strided SC=8 (64 B rows)", [&] { strided<8><<<dim3(65536 / 256 / 8, limbs), 128>>>(a, b); });
    cudaError_t err = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(err));
    return 0;
}
