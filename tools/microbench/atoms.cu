// Shared-memory RED.ADD throughput under different address patterns
// (histogram design probe). Reports cycles per warp-RED per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096

template <int PAT>
__global__ void red_probe(unsigned* out, unsigned seed, long long* cyc) {
    __shared__ unsigned h[64 * 32 * 2];
    for (int i = threadIdx.x; i < 64 * 32 * 2; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = seed * 2654435761u + warp * 977u;           // warp-uniform stream
    unsigned xl = x ^ (lane * 0x9E3779B9u);                   // per-lane stream
    const unsigned base = (unsigned)__cvta_generic_to_shared(h);
    long long t0 = clock64();
#pragma unroll 16
    for (int it = 0; it < ITERS; ++it) {
        x = x * 1664525u + 1013904223u;
        xl = xl * 1664525u + 1013904223u;
        unsigned addr;
        if (PAT == 0) addr = base + (((xl >> 26) << 5) | lane) * 4;          // per-lane replica
        if (PAT == 1) addr = base + (xl >> 26) * 4;                          // 64 bins, random
        if (PAT == 2) addr = base + (x >> 26) * 4;                           // all lanes same bin
        if (PAT == 3) addr = base + (((xl >> 26) << 4) | (lane & 15)) * 4;   // 16x replica
        if (PAT == 4) addr = base + (((x >> 26) + (lane >> 3)) & 63) * 4;    // 4 distinct bins
        if (PAT == 5) addr = base + ((((x >> 26) + (lane >> 3)) & 63) * 32 + lane) * 4; // smooth, per-lane
        if (PAT == 6) addr = base + (((xl >> 26) << 3) | (lane & 7)) * 4;    // 8x replica
        if (PAT == 7) addr = base + ((((x >> 26) + (lane >> 3)) & 63) * 8 + (lane & 7)) * 4; // smooth, 8x
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr));
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { out[0] = h[3]; if (blockIdx.x == 0) cyc[0] = t1 - t0; }
}

template <typename K>
void run(const char* name, K k) {
    unsigned* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms * 2, 512>>>(out, 1u, cyc); cudaDeviceSynchronize();
    k<<<sms * 2, 512>>>(out, 2u, cyc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double warps = 32.0;  // 2 blocks x 16 warps resident per SM
    printf("%-34s cycles/warp-RED/SM = %.3f\n", name, (double)c / (ITERS * warps));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run("per-lane replica (conflict-free)", red_probe<0>);
    run("8x replica, random ids", red_probe<6>);
    run("16x replica, random ids", red_probe<3>);
    run("single table, random of 64", red_probe<1>);
    run("single table, all lanes same", red_probe<2>);
    run("single table, 4 distinct (smooth)", red_probe<4>);
    run("per-lane replica, smooth ids", red_probe<5>);
    run("8x replica, smooth ids", red_probe<7>);
    return 0;
}
