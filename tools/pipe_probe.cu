// Microbenchmark: throughput of the instruction forms the tile kernel uses,
// as warp-instructions per cycle per SMSP (1.0 = one issue every cycle).
// Full occupancy of independent chains; kernel time by CUDA events, cycles
// from the SM clock sampled with clock64 over the same kernel.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CH = 8;
template <int K>
__global__ void __launch_bounds__(256) k(float *out, float b, int iters, long long *cyc) {
    float x[CH];
    uint32_t m[CH];
    for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 0.001f + i; m[i] = threadIdx.x + i; }
    __shared__ uint32_t sh[256];
    sh[threadIdx.x & 255] = threadIdx.x;
    __syncthreads();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sh);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (K == 0) asm volatile("{.reg .pred p; setp.ge.f32 p, %1, %2; @p or.b32 %0, %0, 16;}" : "+r"(m[i]) : "f"(x[i]), "f"(b));
            if (K == 1) asm volatile("{.reg .pred p; setp.ge.f32 p, %1, %2; @p add.u32 %0, %0, 16;}" : "+r"(m[i]) : "f"(x[i]), "f"(b));
            if (K == 2) asm volatile("{.reg .f32 s; set.ge.f32.f32 s, %1, %2; fma.rn.f32 %0, s, 0f41800000, %0;}" : "+f"(x[i]) : "f"(x[(i + 1) % CH]), "f"(b));
            if (K == 3) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F800000;" : "+f"(x[i]));
            if (K == 4) asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(x[i]) : "f"(b));
            if (K == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(m[i]) : "r"(m[(i + 1) % CH]));
            if (K == 6) asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(x[(i + 1) % CH]));
            if (K == 7) asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(m[i]) : "r"(m[(i + 1) % CH]));
            if (K == 8) asm volatile("xor.b32 %0, %0, %1;" : "+r"(m[i]) : "r"(m[(i + 1) % CH]));
            if (K == 9) asm volatile("{.reg .pred p; setp.ge.f32 p, %1, %2; selp.f32 %0, %1, %0, p;}" : "+f"(x[i]) : "f"(x[(i + 1) % CH]), "f"(b));
            if (K == 10) asm volatile("{.reg .pred p; setp.ge.f32 p, %1, %2; selp.b32 %0, 5, %0, p;}" : "+r"(m[i]) : "f"(x[i]), "f"(b));
            if (K == 11) asm volatile("add.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(x[(i + 1) % CH]));
            if (K == 12) asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(m[i]) : "r"(m[(i + 1) % CH]));
            if (K == 13) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + ((m[i] & 255u) << 2))); m[i] += v; }
            if (K == 14) { m[i] = __shfl_down_sync(0xffffffffu, m[i], 1) + 1u; }
            if (K == 15) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + ((m[i] & 255u) << 2))); m[i] = __shfl_down_sync(0xffffffffu, m[i], 1) + v; }
        }
    }
    long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < CH; ++i) acc += x[i] + float(m[i]);
    if (acc == 12345.f) out[0] = acc;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cyc, (unsigned long long)(t1 - t0));
}
template <int K>
void run(const char *name, int ops) {
    float *o;
    long long *cyc;
    cudaMalloc(&o, 8);
    cudaMalloc(&cyc, 8);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<K>, 256, 0);
    int sms = 148;
    const int iters = 2048;
    k<K><<<sms * nb, 256>>>(o, 2.f, 8, cyc);
    cudaMemset(cyc, 0, 8);
    k<K><<<sms * nb, 256>>>(o, 2.f, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warps_per_smsp = nb * 256 / 32 / 4.0;
    const double winst = warps_per_smsp * double(iters) * CH * ops;
    printf("%-34s blocks/SM %d  IPC/SMSP %.3f  (cycles per warp-instr %.2f)\n", name, nb, winst / c, c / winst);
    cudaFree(o);
    cudaFree(cyc);
}
int main() {
    run<0>("FSETP + @p LOP3(or)", 2);
    run<1>("FSETP + @p IADD", 2);
    run<2>("FSET.BF + FFMA-imm", 2);
    run<3>("FFMA imm", 1);
    run<4>("FFMA reg", 1);
    run<5>("IADD3", 1);
    run<6>("FMNMX", 1);
    run<7>("IMAD", 1);
    run<8>("LOP3", 1);
    run<9>("FSETP + FSEL", 2);
    run<10>("FSETP + SEL", 2);
    run<11>("FADD", 1);
    run<12>("SHF funnel", 1);
    run<13>("LDS (+IADD)", 2);
    run<14>("SHFL (+IADD)", 2);
    run<15>("LDS + SHFL (+IADD)", 3);
    return 0;
}
