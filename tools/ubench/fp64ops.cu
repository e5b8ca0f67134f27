// Per-opcode throughput of the FP64 / select instructions the simulator step
// uses (tuning aid, not part of the library).
#include <cstdio>
#include <cuda_runtime.h>

enum Op { DFMA_, DADD_, DMUL_, DSETP_, FSEL_, DSETP_FSEL_, DSETP_LOP_ };

template <Op OP>
__global__ void k(double* outd, int iters, double a) {
    double d[8], e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i] = threadIdx.x * 1e-3 + i; e[i] = i * 0.5; }
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (OP == DFMA_) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
            if constexpr (OP == DADD_) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(a));
            if constexpr (OP == DMUL_) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(a));
            if constexpr (OP == DSETP_) {
                unsigned r;
                asm volatile("{.reg .pred p; setp.lt.f64 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(r) : "d"(d[i]), "d"(a));
                acc += r;
            }
            if constexpr (OP == FSEL_) asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.f64 %0, %0, %1, p;}" : "+d"(d[i]) : "d"(e[i]), "r"(it & 1));
            if constexpr (OP == DSETP_FSEL_) asm volatile("{.reg .pred p; setp.lt.f64 p, %0, %1; selp.f64 %0, %0, %1, p;}" : "+d"(d[i]) : "d"(e[i]));
        }
    }
    double sd = acc;
#pragma unroll
    for (int i = 0; i < 8; ++i) sd += d[i];
    outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
}

template <Op OP>
void run(const char* name, double* od, int sms) {
    const int iters = 20000;
    dim3 g(sms * 4), b(256);
    k<OP><<<g, b>>>(od, 10, 1.0000001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<g, b>>>(od, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)g.x * b.x / 32.0;
    printf("%-14s %8.3f ms  SMSP-cycles per 8 ops per warp %.3f\n", name, ms,
           ms * 1e-3 * 1.965e9 * sms * 4 / (warps * iters));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* od;
    cudaMalloc(&od, sms * 4 * 256 * 8);
    run<DFMA_>("dfma", od, sms);
    run<DADD_>("dadd", od, sms);
    run<DMUL_>("dmul", od, sms);
    run<DSETP_>("dsetp(+sel)", od, sms);
    run<FSEL_>("fsel64", od, sms);
    run<DSETP_FSEL_>("dsetp+fsel64", od, sms);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
