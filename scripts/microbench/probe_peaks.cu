// Random-probe rate microbenchmark: how many random
// 32-byte sector reads per second one B200 sustains, by working-set size --
// L2-resident (8-64 MB) and HBM (256 MB-4 GB) -- in the two forms the
// structured local-energy kernels issue them:
//   indep: every lane issues 8 independent random 32-B loads per step (the
//          hash / list / psi-hat probes of many rows in flight);
//   chain: every lane follows 8 independent dependent chains (address of the
//          next load = hash of the loaded value: Bloom word -> slot -> record).
// Grid: 148 SMs x 8 CTAs x 256 threads (the row kernels run 4 x 256 per SM;
// more warps only help the latency-bound chain form). Prints one JSON object.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <bool CHAIN>
__global__ void __launch_bounds__(256) k_probe(const ulonglong2 *buf, u64 mask_sectors, int iters, u64 *out) {
    const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    u64 s[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) s[c] = mix(tid * 8 + c + 1);
    u64 acc = 0;
    for (int it = 0; it < iters; ++it) {
        ulonglong2 v[8], w[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const u64 sec = s[c] & mask_sectors;       // one 32-B sector = 2 x 16 B
            v[c] = __ldg(buf + 2 * sec);
            w[c] = __ldg(buf + 2 * sec + 1);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const u64 x = v[c].x ^ v[c].y ^ w[c].x ^ w[c].y;
            acc += x;
            s[c] = CHAIN ? mix(x + s[c]) : mix(s[c] + 0x9E3779B97F4A7C15ULL);
        }
    }
    if (acc == 0x1234567ULL) out[0] = acc;
}

__global__ void k_fill(ulonglong2 *buf, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        buf[i] = make_ulonglong2(mix(i), mix(~i));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const u64 max_bytes = 4ULL << 30;
    ulonglong2 *buf;
    u64 *out;
    if (cudaMalloc(&buf, max_bytes) != cudaSuccess || cudaMalloc(&out, 8) != cudaSuccess) {
        printf("{\"error\": \"alloc\"}\n");
        return 1;
    }
    k_fill<<<p.multiProcessorCount * 8, 256>>>(buf, max_bytes / 16);
    cudaDeviceSynchronize();
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    const u64 sizes_mb[] = {8, 16, 32, 64, 96, 256, 1024, 4096};
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"unit\": \"random 32-B sector loads per second\"",
           p.name, p.multiProcessorCount, p.l2CacheSize);
    for (int form = 0; form < 2; ++form) {
        printf(", \"%s\": {", form ? "chain" : "indep");
        for (int si = 0; si < 8; ++si) {
            const u64 bytes = sizes_mb[si] << 20;
            const u64 mask = bytes / 32 - 1;
            const int iters = form ? 64 : 128;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0);
                if (form) k_probe<true><<<blocks, threads>>>(buf, mask, iters, out);
                else k_probe<false><<<blocks, threads>>>(buf, mask, iters, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep && ms < best) best = ms;   // rep 0 warms L2
            }
            const double probes = (double)blocks * threads * iters * 8;
            printf("%s\"%lluMB\": %.4e", si ? ", " : "", sizes_mb[si], probes / (best * 1e-3));
        }
        printf("}");
    }
    printf("}\n");
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : 1;
}
