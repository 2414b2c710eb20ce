// Which pipe runs VIADD (add-immediate)? Chains that cannot be folded:
// each op mixes two chains; immediates differ per op.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
template <int MODE>
__global__ void k(unsigned* out, long long* cyc) {
    unsigned v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 7u + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        unsigned t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const unsigned a = v[i], b = v[(i + 3) & 7];
            unsigned r;
            if (MODE == 0) r = a + (0x350035u + i * 0x10001u);  // VIADD?
            if (MODE == 1) asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
            if (MODE == 2) { if (i & 1) r = a + (0x350035u + i * 0x10001u);
                             else asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
            if (MODE == 3) { unsigned s = a + b;
                             r = s + (0x110011u + i); }  // IADD3 w/ imm
            if (MODE == 4) { if (i & 1) { unsigned s = a + b;
                             r = s + (0x110011u + i); }
                             else asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); }
            t[i] = r ^ (it & 1);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = t[i];
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i];
    if (acc == 1) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <typename K> void run(const char* n, K kk, double ops) {
    unsigned* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    kk<<<sms, 1024>>>(o, c); cudaDeviceSynchronize(); kk<<<sms, 1024>>>(o, c); cudaDeviceSynchronize();
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("%-22s warp-instr/clk/SM = %.2f\n", n, 32.0 * ITERS * ops / cy);
}
int main() {
    run("VIADD(imm)", k<0>, 8 + 8);      // + LOP3 for ^(it&1)
    run("VIMNMX", k<1>, 8 + 8);
    run("VIADD + VIMNMX", k<2>, 8 + 8);
    run("IADD3(imm)", k<3>, 8 + 8);
    run("IADD3 + VIMNMX", k<4>, 8 + 8);
}
