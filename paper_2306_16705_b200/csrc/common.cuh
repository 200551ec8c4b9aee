// common.cuh -- device helpers shared by the literal (kernels.cu) and the
// structured (structured.cu) local-energy kernels of libnnqs.
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

// ------------------------------------------------ Eq. (6) chunk partials
// First pass of the count-weighted energy (weights P:226) per
// chunk of NNQS_REDUCE_CHUNK rows, in ONE fixed order shared by every producer
// (nnqs_energy_chunk_partials and the fused E_loc epilogues): lane l of a warp
// sums rows l, l + 32, l + 64, ... (ascending), then an xor butterfly
// (o = 16, 8, 4, 2, 1).  Pass 1 (mean == nullptr): (W, sum w Re E, sum w Im E);
// pass 2: (W, sum w |E - mean|^2, 0).
template <bool COHERENT>
__device__ __forceinline__ double3 chunk_partial_warp(const double2 *eloc, const int64_t *counts, int64_t base,
                                                      int len, const double *mean) {
    const int lane = threadIdx.x & 31;
    double a = 0.0, b = 0.0, c = 0.0;
    double mr = 0.0, mi = 0.0;
    if (mean) { mr = mean[0]; mi = mean[1]; }
    for (int j = lane; j < len; j += 32) {
        const double w = (double)counts[base + j];
        // fused epilogue: rows written by other warps of this grid -> bypass L1
        const double2 e = COHERENT ? __ldcg(eloc + base + j) : eloc[base + j];
        a += w;
        if (!mean) {
            b = fma(w, e.x, b);
            c = fma(w, e.y, c);
        } else {
            const double dr = e.x - mr, di = e.y - mi;
            b = fma(w, dr * dr + di * di, b);
        }
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    return make_double3(a, b, c);
}

// The same order computed by one thread (the literal kernel's epilogue runs one
// row per thread): 32 lane sums, then the butterfly on a local array.
// Bit-identical to chunk_partial_warp (IEEE addition is commutative, so every
// butterfly partner pair forms the same sum).
__device__ __forceinline__ double3 chunk_partial_serial(const double2 *eloc, const int64_t *counts, int64_t base,
                                                        int len) {
    double v[3][32];
    for (int l = 0; l < 32; ++l) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int j = l; j < len; j += 32) {
            const double w = (double)counts[base + j];
            const double2 e = __ldcg(eloc + base + j);
            a += w;
            b = fma(w, e.x, b);
            c = fma(w, e.y, c);
        }
        v[0][l] = a; v[1][l] = b; v[2][l] = c;
    }
    for (int o = 16; o; o >>= 1) {
        double t[3][32];
        for (int l = 0; l < 32; ++l)
            for (int q = 0; q < 3; ++q) t[q][l] = v[q][l] + v[q][l ^ o];
        for (int l = 0; l < 32; ++l)
            for (int q = 0; q < 3; ++q) v[q][l] = t[q][l];
    }
    return make_double3(v[0][0], v[1][0], v[2][0]);
}

// Fused epilogue, warp-wide: row r (relative to the call) has just been written
// by lane 0.  The warp that completes a chunk reduces it.
__device__ __forceinline__ void chunk_done_warp(const ChunkSink &C, const double2 *eloc, int64_t r, int64_t n_rows) {
    if (!C.partials) return;
    const int lane = threadIdx.x & 31;
    unsigned old = 0;
    const int64_t ch = r / NNQS_REDUCE_CHUNK;
    if (lane == 0) {
        __threadfence();
        old = atomicAdd(C.ctr + ch, 1u);
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    const int64_t base = ch * NNQS_REDUCE_CHUNK;
    const int len = (int)min((int64_t)NNQS_REDUCE_CHUNK, n_rows - base);
    if ((int)old == len - 1) {
        __threadfence();
        const double3 p = chunk_partial_warp<true>(eloc, C.counts, base, len, nullptr);
        if (lane == 0) {
            C.partials[3 * ch] = p.x;
            C.partials[3 * ch + 1] = p.y;
            C.partials[3 * ch + 2] = p.z;
        }
    }
}

// Fused epilogue, one thread per row (literal kernel).
__device__ __forceinline__ void chunk_done_thread(const ChunkSink &C, const double2 *eloc, int64_t r,
                                                  int64_t n_rows) {
    if (!C.partials) return;
    __threadfence();
    const int64_t ch = r / NNQS_REDUCE_CHUNK;
    const unsigned old = atomicAdd(C.ctr + ch, 1u);
    const int64_t base = ch * NNQS_REDUCE_CHUNK;
    const int len = (int)min((int64_t)NNQS_REDUCE_CHUNK, n_rows - base);
    if ((int)old == len - 1) {
        __threadfence();
        const double3 p = chunk_partial_serial(eloc, C.counts, base, len);
        C.partials[3 * ch] = p.x;
        C.partials[3 * ch + 1] = p.y;
        C.partials[3 * ch + 2] = p.z;
    }
}
