// Pipe-sharing microbenchmark (tuning aid, not part of the library):
// throughput of independent DFMA / LOP3 / IMAD / FSEL streams, alone and mixed.
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NL, int NI, int NS>
__global__ void k(double* outd, unsigned* outu, int iters, double a, unsigned m) {
    double d[8];
    unsigned u[8], v[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        d[i] = threadIdx.x * 1e-3 + i;
        u[i] = threadIdx.x * 7u + i;
        v[i] = threadIdx.x * 3u + i;
        w[i] = threadIdx.x * 5u + i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ND; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
#pragma unroll
        for (int i = 0; i < NL; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(m), "r"(it));
#pragma unroll
        for (int i = 0; i < NI; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(m), "r"(it));
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.b32 %0, %0, %2, p;}" : "+r"(w[i]) : "r"(it & m), "r"(m));
        }
    }
    double sd = 0;
    unsigned su = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { sd += d[i]; su += u[i] ^ v[i] ^ w[i]; }
    outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
    outu[blockIdx.x * blockDim.x + threadIdx.x] = su;
}

template <int ND, int NL, int NI, int NS>
void run(const char* name, double* od, unsigned* ou, int sms) {
    const int iters = 20000;
    dim3 g(sms * 4), b(256);
    k<ND, NL, NI, NS><<<g, b>>>(od, ou, 10, 1.0000001, 3u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<ND, NL, NI, NS><<<g, b>>>(od, ou, iters, 1.0000001, 3u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)g.x * b.x / 32.0;
    const double clk = 1.965e9;
    const double per_smsp_clk = ms * 1e-3 * clk * sms * 4;  // SMSP-cycles
    const double wi = warps * iters;                       // warp-iterations
    printf("%-28s %8.3f ms  cycles/warp-iter/SMSP %.3f  (DFMA %d LOP3 %d IMAD %d SEL %d)\n", name, ms,
           per_smsp_clk / wi, ND, NL, NI, NS);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* od;
    unsigned* ou;
    cudaMalloc(&od, sms * 4 * 256 * 8);
    cudaMalloc(&ou, sms * 4 * 256 * 4);
    run<8, 0, 0, 0>("dfma8", od, ou, sms);
    run<0, 8, 0, 0>("lop3x8", od, ou, sms);
    run<0, 0, 8, 0>("imad8", od, ou, sms);
    run<0, 0, 0, 8>("isetp+sel8", od, ou, sms);
    run<8, 8, 0, 0>("dfma8+lop3x8", od, ou, sms);
    run<8, 0, 8, 0>("dfma8+imad8", od, ou, sms);
    run<8, 0, 0, 8>("dfma8+isetp+sel8", od, ou, sms);
    run<0, 8, 8, 0>("lop3x8+imad8", od, ou, sms);
    run<8, 8, 8, 0>("dfma8+lop3x8+imad8", od, ou, sms);
    cudaError_t e = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(e));
    return 0;
}
