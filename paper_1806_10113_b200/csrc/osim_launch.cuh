// osim_launch.cuh -- internal launcher interface between the C-ABI host code
// (osim_capi.cu) and the kernel translation units, which are compiled in
// parallel (osim_exh_*.cu, osim_batch_*.cu, osim_heur.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "osim_kernels.cuh"

namespace osim {

// Grow-only device buffer for a launcher's own temporaries (one per library
// stream; the caller holds the device lock).  Work that used it is marked by
// an event (aux_done), and the next user -- on any stream, e.g. a _dev call's
// own stream -- waits for that event first; growing waits for it and for the
// stream (the old buffer may still be read).
struct AuxBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
};
inline void* aux_get(AuxBuf* a, size_t bytes, cudaStream_t st) {
    if (!a) return nullptr;
    if (a->pending) cudaStreamWaitEvent(st, a->ev, 0);
    if (bytes > a->bytes) {
        if (a->pending) cudaEventSynchronize(a->ev);
        cudaStreamSynchronize(st);
        if (a->p) cudaFree(a->p);
        a->p = nullptr;
        a->bytes = 0;
        const size_t want = bytes + bytes / 4;
        if (cudaMalloc(&a->p, want) != cudaSuccess) {
            cudaGetLastError();  // not fatal: the caller runs without the buffer
            return nullptr;
        }
        a->bytes = want;
    }
    return a->p;
}

// the work using the buffer has been enqueued on `st`
inline void aux_done(AuxBuf* a, cudaStream_t st) {
    if (!a || !a->p) return;
    if (!a->ev && cudaEventCreateWithFlags(&a->ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(st);  // no event: finish the work instead
        return;
    }
    cudaEventRecord(a->ev, st);
    a->pending = true;
}

struct LaunchCfg {
    int sms;
    cudaStream_t st;
    AuxBuf* aux = nullptr;
};

// Per-(kernel, device, block shape) launch facts, looked up once: the
// occupancy query, the dynamic-shared-memory opt-in and the tuning env var
// cost a few microseconds per launch, which small searches (C3 shards at
// N = 8, ~40 us) would otherwise pay on every call.
struct KernelFacts {
    const void* fn;
    int dev, threads;
    size_t smem;
    int per_sm;
};

inline int cached_ctas_per_sm(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::vector<KernelFacts> facts;
    static const int cap = [] {  // OSIM_CTAS_PER_SM=<k> caps the resident CTAs per SM (tuning only)
        const char* e = std::getenv("OSIM_CTAS_PER_SM");
        return e ? std::atoi(e) : 0;
    }();
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (const KernelFacts& f : facts)
        if (f.fn == fn && f.dev == dev && f.threads == threads && f.smem == smem) return f.per_sm;
    if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    if (per_sm < 1) per_sm = 1;
    if (cap >= 1 && cap < per_sm) per_sm = cap;
    facts.push_back({fn, dev, threads, smem, per_sm});
    return per_sm;
}

template <class K>
int grid_for_sms(K kernel, int threads, size_t smem, int sms, uint64_t work_blocks) {
    const int per_sm = cached_ctas_per_sm((const void*)kernel, threads, smem);
    uint64_t g = (uint64_t)per_sm * sms;
    if (work_blocks < g) g = work_blocks;
    if (g < 1) g = 1;
    return (int)g;
}

// Suffix length L of the prefix-sharing kernels per n.
// OSIM_PFX_L=<3|4|5> overrides it for n in {8, 10, 12} (tuning only).
constexpr int default_pfx_l(int n) { return n <= 3 ? 1 : (n <= 5 ? 2 : (n <= 10 ? 3 : 4)); }
constexpr bool tunable_n(int n) { return n == 8 || n == 10 || n == 12; }

inline int pfx_l_for(int n) {
    static const int env = [] {
        const char* e = getenv("OSIM_PFX_L");
        return e ? atoi(e) : 0;
    }();
    if (env >= 3 && env <= 5 && tunable_n(n)) return env;
    return default_pfx_l(n);
}

// exhaustive, all stages non-null, prefix-sharing (returns -1: unsupported n);
// with d_out the kernel's last CTA also does the final reduction (d_done: a
// zeroed per-device counter the kernel leaves at zero)
#define OSIM_EXH_DECL(NAME)                                                                          \
    int NAME(int n, int L, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo,   \
             uint64_t hi, double thr, Part* parts, int max_parts, double* d_ms, int* grid_out,        \
             osim_summary* d_out, unsigned long long* d_below, unsigned* d_done, unsigned shard,    \
             unsigned shards);
OSIM_EXH_DECL(exh_fast_launch_d2s1)
OSIM_EXH_DECL(exh_fast_launch_d2s0)
OSIM_EXH_DECL(exh_fast_launch_d1)
#undef OSIM_EXH_DECL

int batch_fast_launch_d2(int n, int L, bool sp2, const LaunchCfg& cfg, const double* d_durs, uint64_t B,
                         double sigma, osim_summary* d_out);
int batch_fast_launch_d1(int n, int L, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
                         osim_summary* d_out);

// exhaustive search with null stages in the fast range (osim_null.cu):
// prefix sharing with the prefix-world checkpoint, L = default_pfx_l(n)
int null_pfx_launch(int n, int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo,
                    uint64_t hi, double thr, Part* parts, int max_parts, double* d_ms, int* d_err, int* g);

int null_batch_launch(int n, int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
                      osim_summary* d_out, int* d_err, int* g);

void heuristic_launch(int dma, int mode /* 0 general, 1 fast, 2 null stages */, const LaunchCfg& cfg, const double* d_durs, const uint8_t* d_idr,
                      uint64_t B, int n, double sigma, int sum_mode, uint8_t* d_order, double* d_ms,
                      uint32_t* d_ns, int* d_err);

// groups of 17..64 tasks, general path (osim_wide.cu); the eval launchers
// return the grid (= number of per-block partials in `parts`)
constexpr int kWideMaxN = 64;
void wide_timeline_launch(int dma, cudaStream_t st, const double* d_durs, int n, double sigma, const uint8_t* d_order,
                          const int8_t* d_dep, int waves, double* d_start, double* d_end, double* d_res, int* d_err);
int wide_eval_perms_launch(int dma, const LaunchCfg& cfg, const double* d_durs, int n, double sigma,
                           const uint8_t* d_perms, uint64_t cnt, double* d_ms, Part* parts, int max_parts, int* d_err);
int wide_eval_labels_launch(int dma, const LaunchCfg& cfg, const double* d_durs, int T, int N, double sigma,
                            const uint8_t* d_labels, uint64_t cnt, double* d_ms, Part* parts, int max_parts,
                            int* d_err);
void wide_heuristic_launch(int dma, const LaunchCfg& cfg, const double* d_durs, const uint8_t* d_idr, uint64_t B,
                           int n, double sigma, int sum_mode, uint8_t* d_order, double* d_ms, uint32_t* d_ns,
                           int* d_err);
void wide_harness_launch(int dma, cudaStream_t st, const double* d_durs, const uint8_t* d_idr, uint64_t S, int T,
                         int N, double sigma, int sum_mode, double* d_ms, uint8_t* d_ng, uint8_t* d_sizes,
                         double* d_start, double* d_end, int* d_err);

// groups of any size, general path (osim_big.cu): uint32 task ids, per-simulation
// workspaces in global memory carved by the caller
uint64_t big_sim_bytes(uint64_t n);
uint64_t big_heur_bytes_per_cta(uint64_t n);
uint64_t big_harness_bytes_per_thread(uint64_t T, uint64_t N);
int big_block();
void big_timeline_launch(int dma, cudaStream_t st, const double* d_durs, uint64_t n, double sigma,
                         const uint32_t* d_order, const int32_t* d_dep, int waves, uint8_t* ws, double* d_start,
                         double* d_end, double* d_res, int* d_err);
void big_eval_perms_launch(int dma, cudaStream_t st, int grid, const double* d_durs, uint64_t n, double sigma,
                           const uint32_t* d_perms, uint64_t cnt, uint8_t* ws, uint64_t wsb, double* d_ms,
                           Part* parts, int* d_err);
void big_eval_labels_launch(int dma, cudaStream_t st, int grid, const double* d_durs, uint32_t T, uint32_t N,
                            double sigma, const uint32_t* d_labels, uint64_t cnt, const int32_t* d_dep, uint8_t* ws,
                            uint64_t wsb, double* d_ms, Part* parts, int* d_err);
void big_heuristic_launch(int dma, cudaStream_t st, int grid, const double* d_durs, const uint32_t* d_idr,
                          uint64_t B, uint64_t n, double sigma, int sum_mode, uint8_t* ws, uint32_t* d_order,
                          double* d_ms, uint32_t* d_ns, int* d_err);
void big_harness_launch(int dma, cudaStream_t st, int grid, const double* d_durs, const uint32_t* d_idr, uint64_t S,
                        uint32_t T, uint32_t N, double sigma, int sum_mode, uint8_t* ws, double* d_ms, uint32_t* d_ng,
                        uint32_t* d_sizes, double* d_start, double* d_end, int* d_err);
void big_micro_timeline_launch(int dma, cudaStream_t st, const double* d_durs, uint64_t n, double sigma, double dt,
                               const uint32_t* d_order, long long max_ticks, double* d_start, double* d_end,
                               double* d_res, int* d_err);

}  // namespace osim
