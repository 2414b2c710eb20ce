// Pipe-assignment probe: one 1024-thread CTA per SM (32 warps, verified by
// launching exactly #SM CTAs), 8 independent chains per thread. Reports
// warp-instructions per cycle per SM for single ops and for interleaved
// pairs; additive pair throughput => the two ops use different pipes.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
#define CH 8

__device__ __forceinline__ unsigned op(int k, unsigned a, unsigned b) {
    unsigned r;
    switch (k) {
    case 0: asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;          // VIMNMX
    case 1: asm volatile("mad.lo.u32 %0, %1, 3, %2;" : "=r"(r) : "r"(a), "r"(b)); break;      // IMAD
    case 2: asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;          // HMNMX2
    case 3: asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;       // HADD2
    case 4: asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;            // IADD
    case 5: asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(a), "r"(b)); break;   // PRMT
    case 6: asm volatile("lop3.b32 %0, %1, %2, 0x0f0f, 0x6a;" : "=r"(r) : "r"(a), "r"(b)); break; // LOP3
    case 7: asm volatile("max.f32 %0, %1, %2;" : "=f"(*(float*)&r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b))); break; // FMNMX
    case 8: asm volatile("add.f32 %0, %1, %2;" : "=f"(*(float*)&r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b))); break; // FADD
    case 9: asm volatile("shf.l.wrap.b32 %0, %1, %2, 6;" : "=r"(r) : "r"(a), "r"(b)); break;  // SHF
    case 10: asm volatile("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;
    case 11: asm volatile("max.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;            // IMNMX
    case 12: asm volatile("add.u32 %0, %1, 0x350035;" : "=r"(r) : "r"(a)); r ^= b & 0; break;    // VIADD imm
    case 13: { unsigned t; asm volatile("add.u32 %0, %1, %2;" : "=r"(t) : "r"(a), "r"(b)); asm volatile("add.u32 %0, %1, 0x10001;" : "=r"(r) : "r"(t)); } break; // IADD3 3-in
    case 14: asm volatile("mad.lo.u32 %0, %1, %3, %2;" : "=r"(r) : "r"(a), "r"(b), "r"(b >> 31 | 1u)); break; // IMAD x*reg+y
    case 15: asm volatile("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;             // LOP3
    case 16: asm volatile("mul.hi.u32 %0, %1, 0x40000;" : "=r"(r) : "r"(a)); r ^= b & 0; break; // IMAD.HI
    case 17: asm volatile("set.ge.f16x2.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); break;  // HSET2.BF
    case 18: asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(0x44004400u), "r"(b)); break;  // HFMA2
    case 19: asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b | 0x40000u)); break;  // IMAD.HI reg
    default: r = a;
    }
    return r;
}

template <int K1, int K2>
__global__ void probe(unsigned* out, unsigned seed, long long* cyc) {
    unsigned v[CH];
    const unsigned b = 0x3c003c01u ^ (seed * 7u);
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = 0x3c003c00u + threadIdx.x * 3u + i;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 2
    for (int it = 0; it < ITERS; ++it) {
        unsigned t[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) t[i] = op((i & 1) ? K2 : K1, v[i], v[(i + 1) % CH]);
#pragma unroll
        for (int i = 0; i < CH; ++i) v[i] = t[i] ^ (b & 0);
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc ^= v[i];
    if (acc == 0x1234567u) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename Kern>
void run(const char* name, Kern k) {
    unsigned* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 1024, 0);
    k<<<sms, 1024>>>(out, 1u, cyc); cudaDeviceSynchronize();
    k<<<sms, 1024>>>(out, 2u, cyc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-26s warp-instr/clk/SM = %.2f  (occ blocks %d)\n", name, 32.0 * ITERS * CH / (double)c, nb);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run("VIMNMX", probe<0, 0>);
    run("IMAD", probe<1, 1>);
    run("HMNMX2", probe<2, 2>);
    run("HADD2", probe<3, 3>);
    run("IADD", probe<4, 4>);
    run("PRMT", probe<5, 5>);
    run("LOP3", probe<6, 6>);
    run("FMNMX", probe<7, 7>);
    run("FADD", probe<8, 8>);
    run("SHF", probe<9, 9>);
    run("IMNMX.U32", probe<11, 11>);
    run("VIMNMX + IMAD", probe<0, 1>);
    run("VIMNMX + HMNMX2", probe<0, 2>);
    run("VIMNMX + HADD2", probe<0, 3>);
    run("VIMNMX + FMNMX", probe<0, 7>);
    run("VIMNMX + FADD", probe<0, 8>);
    run("IADD + IMAD", probe<4, 1>);
    run("PRMT + IMAD", probe<5, 1>);
    run("HMNMX2 + IMAD", probe<2, 1>);
    run("HMNMX2 + HADD2", probe<2, 3>);
    run("max+min u16x2", probe<0, 10>);
    run("VIADD imm", probe<12, 12>);
    run("VIADD + VIMNMX", probe<12, 0>);
    run("VIADD + IMAD", probe<12, 1>);
    run("IADD3 3-in", probe<13, 13>);
    run("IADD3 + VIMNMX", probe<13, 0>);
    run("IMAD reg-1", probe<14, 14>);
    run("IMAD reg-1 + VIMNMX", probe<14, 0>);
    run("IMAD.HI + VIMNMX", probe<16, 0>);
    run("XOR + IMAD", probe<15, 1>);
    run("HSET2", probe<17, 17>);
    run("HSET2 + VIMNMX", probe<17, 0>);
    run("HSET2 + IMAD", probe<17, 1>);
    run("HFMA2", probe<18, 18>);
    run("HFMA2 + VIMNMX", probe<18, 0>);
    run("HSET2 + HFMA2", probe<17, 18>);
    run("IMAD.HI", probe<16, 16>);
    run("IMAD.HI + IMAD", probe<16, 1>);
    return 0;
}
