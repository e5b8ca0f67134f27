// osim_big.cu -- launches of the any-size general-path kernels (osim_big.cuh)
// for the C-ABI host code.  Workspaces are carved by the caller; each
// launcher states how many threads (or CTAs) its workspace must cover.
#include "osim_big.cuh"
#include "osim_launch.cuh"

namespace osim {

uint64_t big_sim_bytes(uint64_t n) { return big_ws_bytes(n); }
uint64_t big_heur_bytes_per_cta(uint64_t n) { return big_heur_cta_bytes(n, kBigBlock); }
uint64_t big_harness_bytes_per_thread(uint64_t T, uint64_t N) { return big_harness_thread_bytes(T, N); }
int big_block() { return kBigBlock; }

void big_timeline_launch(int dma, cudaStream_t st, const double* d_durs, uint64_t n, double sigma,
                         const uint32_t* d_order, const int32_t* d_dep, int waves, uint8_t* ws, double* d_start,
                         double* d_end, double* d_res, int* d_err) {
    if (dma == 2)
        k_big_timeline<2><<<1, 32, 0, st>>>(d_durs, n, sigma, d_order, d_dep, waves, ws, d_start, d_end, d_res, d_err);
    else
        k_big_timeline<1><<<1, 32, 0, st>>>(d_durs, n, sigma, d_order, d_dep, waves, ws, d_start, d_end, d_res, d_err);
}

// `grid` CTAs of kBigBlock threads (ws: grid * kBigBlock * wsb bytes)
void big_eval_perms_launch(int dma, cudaStream_t st, int grid, const double* d_durs, uint64_t n, double sigma,
                           const uint32_t* d_perms, uint64_t cnt, uint8_t* ws, uint64_t wsb, double* d_ms,
                           Part* parts, int* d_err) {
    if (dma == 2)
        k_big_eval_perms<2><<<grid, kBigBlock, 0, st>>>(d_durs, n, sigma, d_perms, cnt, ws, wsb, d_ms, parts, d_err);
    else
        k_big_eval_perms<1><<<grid, kBigBlock, 0, st>>>(d_durs, n, sigma, d_perms, cnt, ws, wsb, d_ms, parts, d_err);
}

void big_eval_labels_launch(int dma, cudaStream_t st, int grid, const double* d_durs, uint32_t T, uint32_t N,
                            double sigma, const uint32_t* d_labels, uint64_t cnt, const int32_t* d_dep, uint8_t* ws,
                            uint64_t wsb, double* d_ms, Part* parts, int* d_err) {
    if (dma == 2)
        k_big_eval_labels<2><<<grid, kBigBlock, 0, st>>>(d_durs, T, N, sigma, d_labels, cnt, d_dep, ws, wsb, d_ms,
                                                         parts, d_err);
    else
        k_big_eval_labels<1><<<grid, kBigBlock, 0, st>>>(d_durs, T, N, sigma, d_labels, cnt, d_dep, ws, wsb, d_ms,
                                                         parts, d_err);
}

// `grid` CTAs, one group each at a time (ws: grid * big_heur_bytes_per_cta(n))
void big_heuristic_launch(int dma, cudaStream_t st, int grid, const double* d_durs, const uint32_t* d_idr,
                          uint64_t B, uint64_t n, double sigma, int sum_mode, uint8_t* ws, uint32_t* d_order,
                          double* d_ms, uint32_t* d_ns, int* d_err) {
    if (!B) return;
    if (dma == 2)
        k_big_heuristic<2><<<grid, kBigBlock, 0, st>>>(d_durs, d_idr, B, n, sigma, sum_mode, ws, d_order, d_ms, d_ns,
                                                       d_err);
    else
        k_big_heuristic<1><<<grid, kBigBlock, 0, st>>>(d_durs, d_idr, B, n, sigma, sum_mode, ws, d_order, d_ms, d_ns,
                                                       d_err);
}

// `grid` CTAs of kBigBlock threads, one scenario per thread at a time
// (ws: grid * kBigBlock * big_harness_bytes_per_thread(T, N))
void big_harness_launch(int dma, cudaStream_t st, int grid, const double* d_durs, const uint32_t* d_idr, uint64_t S,
                        uint32_t T, uint32_t N, double sigma, int sum_mode, uint8_t* ws, double* d_ms, uint32_t* d_ng,
                        uint32_t* d_sizes, double* d_start, double* d_end, int* d_err) {
    if (!S) return;
    if (dma == 2)
        k_big_harness<2><<<grid, kBigBlock, 0, st>>>(d_durs, d_idr, S, T, N, sigma, sum_mode, ws, d_ms, d_ng, d_sizes,
                                                     d_start, d_end, d_err);
    else
        k_big_harness<1><<<grid, kBigBlock, 0, st>>>(d_durs, d_idr, S, T, N, sigma, sum_mode, ws, d_ms, d_ng, d_sizes,
                                                     d_start, d_end, d_err);
}

void big_micro_timeline_launch(int dma, cudaStream_t st, const double* d_durs, uint64_t n, double sigma, double dt,
                               const uint32_t* d_order, long long max_ticks, double* d_start, double* d_end,
                               double* d_res, int* d_err) {
    if (dma == 2)
        k_big_micro_timeline<2><<<1, 32, 0, st>>>(d_durs, n, sigma, dt, d_order, max_ticks, d_start, d_end, d_res,
                                                  d_err);
    else
        k_big_micro_timeline<1><<<1, 32, 0, st>>>(d_durs, n, sigma, dt, d_order, max_ticks, d_start, d_end, d_res,
                                                  d_err);
}

}  // namespace osim
