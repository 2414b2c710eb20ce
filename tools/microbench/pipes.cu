// Instruction-throughput probe for the ops the LDP kernel is built from.
// Each thread runs 8 independent dependency chains of one op; the kernel is
// launched with enough warps to saturate every SMSP. Prints warp-instructions
// per cycle per SM (4.0 = one per SMSP per cycle, 2.0 = half-rate pipe).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define ITERS 2048
#define CHAINS 8

template <int OP>
__device__ __forceinline__ unsigned op(unsigned a, unsigned b, unsigned c) {
    unsigned r;
    if constexpr (OP == 0) { asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
    if constexpr (OP == 1) { asm volatile("{.reg .b32 t; max.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); }
    if constexpr (OP == 2) { asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
    if constexpr (OP == 3) { asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); r += c; }
    if constexpr (OP == 4) { asm volatile("mad.lo.u32 %0, %1, 8, %2;" : "=r"(r) : "r"(a), "r"(c)); }
    if constexpr (OP == 5) { asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); }
    if constexpr (OP == 6) { asm volatile("lop3.b32 %0, %1, %2, %3, 0xe8;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); }
    if constexpr (OP == 7) { asm volatile("max.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
    if constexpr (OP == 8) { asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
    if constexpr (OP == 9) { asm volatile("{.reg .b32 t; min.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); }
    if constexpr (OP == 10) { asm volatile("{.reg .b32 t; max.f16x2 t, %1, %2; max.f16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); }
    if constexpr (OP == 11) { asm volatile("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(r) : "r"(a), "r"(b)); }
    if constexpr (OP == 12) { asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(a)); r ^= b; }
    return r;
}

template <int OP>
__global__ void probe(unsigned* out, unsigned seed, long long* cycles) {
    unsigned v[CHAINS];
    const unsigned b = seed * 0x9E3779B9u + threadIdx.x, c = seed ^ 0x5bd1e995u;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = threadIdx.x * 131u + i * 7u + seed;
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) v[i] = op<OP>(v[i], b + i, c);
    }
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc ^= v[i];
    if (acc == 0x12345678u) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

// Per-lane private shared-memory histogram (bank == lane): atomic and plain RMW.
__global__ void smem_atom(unsigned* out, unsigned seed, long long* cycles) {
    __shared__ unsigned h[56 * 32 * 4];
    for (int i = threadIdx.x; i < 56 * 32 * 4; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned* mine = h + (warp & 3) * 56 * 32 + lane;
    unsigned x = seed + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 8
    for (int it = 0; it < ITERS * 4; ++it) {
        x = x * 1664525u + 1013904223u;
        atomicAdd(mine + (((x >> 26) % 56u) << 5), 1u);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { out[1] = h[5]; if (blockIdx.x == 0) cycles[0] = t1 - t0; }
}

__global__ void smem_atom_shared_addr(unsigned* out, unsigned seed, long long* cycles) {
    __shared__ unsigned h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    unsigned x = seed + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 8
    for (int it = 0; it < ITERS * 4; ++it) {
        x = x * 1664525u + 1013904223u;
        atomicAdd(h + (x >> 26), 1u);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { out[1] = h[5]; if (blockIdx.x == 0) cycles[0] = t1 - t0; }
}

__global__ void shfl_probe(unsigned* out, unsigned seed, long long* cycles) {
    unsigned v[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = threadIdx.x * 131u + i * 7u + seed;
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) v[i] = __shfl_down_sync(0xffffffffu, v[i], 1) + 1u;
    }
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc ^= v[i];
    if (acc == 0x12345678u) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

template <typename K>
void run(const char* name, K kernel, double ops_per_thread, int threads) {
    unsigned* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    kernel<<<sms * 2, threads>>>(out, 1u, cyc);
    cudaDeviceSynchronize();
    kernel<<<sms * 2, threads>>>(out, 2u, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // two blocks per SM resident together: warps per SM = 2*threads/32
    double warps = 2.0 * threads / 32.0;
    double wi_per_cycle = warps * ops_per_thread / (double)c;
    printf("%-28s cycles=%lld  warp-instr/cycle/SM=%.3f\n", name, c, wi_per_cycle);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    const int T = 512;
    const double body = (double)ITERS / 4.0;  // loop bodies per thread
    // second argument: SASS instructions of the probed opcode per loop body (from cuobjdump)
    run("VIMNMX3.U16x2 (fused max)", probe<0>, body * 16, T);
    run("VIMNMX3.U16x2 (max3)", probe<1>, body * 32, T);
    run("VIMNMX.U16x2 (min,max)", probe<9>, body * 64, T);
    run("VHMNMX (f16 max fused)", probe<2>, body * 16, T);
    run("VHMNMX (f16 max3)", probe<10>, body * 32, T);
    run("IADD3", probe<3>, body * 32, T);
    run("IMAD-ish", probe<4>, body * 16, T);
    run("PRMT", probe<5>, body * 32, T);
    run("LOP3", probe<6>, body * 32, T);
    run("VIMNMX3.U32", probe<7>, body * 16, T);
    run("HADD2+HFMA2", probe<8>, body * 32, T);
    run("SHF", probe<11>, body * 32, T);
    run("POPC(+LOP3)", probe<12>, body * 32, T);
    run("SHFL.DOWN", shfl_probe, (double)(ITERS / 16) * 32, T);
    run("ATOMS per-lane bins (1/iter)", smem_atom, (double)ITERS * 4, T);
    run("ATOMS 64 shared bins (1/iter)", smem_atom_shared_addr, (double)ITERS * 4, T);
    return 0;
}
