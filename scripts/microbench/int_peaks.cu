// INT32 issue-rate microbenchmark: sustained LOP3 and
// IADD3 (ALU pipe) and POPC throughput of one B200, and a random dependent-load
// rate.  Each thread runs 8 independent chains so the pipes, not latency, bound it.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_ops(uint32_t *out, int iters, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    const uint32_t c = seed ^ 0x5bd1e995u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(c), "r"(a[(i + 1) & 7]));
                else if (OP == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 3) & 7]));
                else asm volatile("popc.b32 %0, %0;" : "+r"(a[i]));
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x12345678u) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    uint32_t *out;
    cudaMalloc(&out, 4);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
    const double ops = (double)blocks * threads * iters * 16 * 8;
    const char *names[3] = {"lop3", "iadd", "popc"};
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu", p.name, p.multiProcessorCount,
           p.l2CacheSize, p.sharedMemPerMultiprocessor);
    for (int op = 0; op < 3; ++op) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k_ops<0><<<blocks, threads>>>(out, iters, 7);
            else if (op == 1) k_ops<1><<<blocks, threads>>>(out, iters, 7);
            else k_ops<2><<<blocks, threads>>>(out, iters, 7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"%s_tops\": %.4f", names[op], ops / (ms * 1e-3) / 1e12);
    }
    printf("}\n");
    return 0;
}
