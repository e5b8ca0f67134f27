// osim_wide.cu -- launches of the 17..64-task general-path kernels
// (osim_wide.cuh) for the C-ABI host code.
#include "osim_launch.cuh"
#include "osim_wide.cuh"

namespace osim {

void wide_timeline_launch(int dma, cudaStream_t st, const double* d_durs, int n, double sigma, const uint8_t* d_order,
                          const int8_t* d_dep, int waves, double* d_start, double* d_end, double* d_res, int* d_err) {
    if (dma == 2)
        k_wide_timeline<2><<<1, 32, 0, st>>>(d_durs, n, sigma, d_order, d_dep, waves, d_start, d_end, d_res, d_err);
    else
        k_wide_timeline<1><<<1, 32, 0, st>>>(d_durs, n, sigma, d_order, d_dep, waves, d_start, d_end, d_res, d_err);
}

int wide_eval_perms_launch(int dma, const LaunchCfg& cfg, const double* d_durs, int n, double sigma,
                           const uint8_t* d_perms, uint64_t cnt, double* d_ms, Part* parts, int max_parts, int* d_err) {
    const uint64_t blocks = (cnt + kWideBlock - 1) / kWideBlock;
    int g;
    if (dma == 2) {
        g = grid_for_sms(k_wide_eval_perms<2>, kWideBlock, 0, cfg.sms, blocks);
        if (g > max_parts) g = max_parts;
        k_wide_eval_perms<2><<<g, kWideBlock, 0, cfg.st>>>(d_durs, n, sigma, d_perms, cnt, d_ms, parts, d_err);
    } else {
        g = grid_for_sms(k_wide_eval_perms<1>, kWideBlock, 0, cfg.sms, blocks);
        if (g > max_parts) g = max_parts;
        k_wide_eval_perms<1><<<g, kWideBlock, 0, cfg.st>>>(d_durs, n, sigma, d_perms, cnt, d_ms, parts, d_err);
    }
    return g;
}

int wide_eval_labels_launch(int dma, const LaunchCfg& cfg, const double* d_durs, int T, int N, double sigma,
                            const uint8_t* d_labels, uint64_t cnt, double* d_ms, Part* parts, int max_parts,
                            int* d_err) {
    const uint64_t blocks = (cnt + kWideBlock - 1) / kWideBlock;
    int g;
    if (dma == 2) {
        g = grid_for_sms(k_wide_eval_labels<2>, kWideBlock, 0, cfg.sms, blocks);
        if (g > max_parts) g = max_parts;
        k_wide_eval_labels<2><<<g, kWideBlock, 0, cfg.st>>>(d_durs, T, N, sigma, d_labels, cnt, parts, d_ms, d_err);
    } else {
        g = grid_for_sms(k_wide_eval_labels<1>, kWideBlock, 0, cfg.sms, blocks);
        if (g > max_parts) g = max_parts;
        k_wide_eval_labels<1><<<g, kWideBlock, 0, cfg.st>>>(d_durs, T, N, sigma, d_labels, cnt, parts, d_ms, d_err);
    }
    return g;
}

void wide_heuristic_launch(int dma, const LaunchCfg& cfg, const double* d_durs, const uint8_t* d_idr, uint64_t B,
                           int n, double sigma, int sum_mode, uint8_t* d_order, double* d_ms, uint32_t* d_ns,
                           int* d_err) {
    const unsigned grid = (unsigned)((B + kWideBlock - 1) / kWideBlock);
    if (!grid) return;
    if (dma == 2)
        k_wide_heuristic<2><<<grid, kWideBlock, 0, cfg.st>>>(d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms,
                                                             d_ns, d_err);
    else
        k_wide_heuristic<1><<<grid, kWideBlock, 0, cfg.st>>>(d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms,
                                                             d_ns, d_err);
}

void wide_harness_launch(int dma, cudaStream_t st, const double* d_durs, const uint8_t* d_idr, uint64_t S, int T,
                         int N, double sigma, int sum_mode, double* d_ms, uint8_t* d_ng, uint8_t* d_sizes,
                         double* d_start, double* d_end, int* d_err) {
    const unsigned grid = (unsigned)((S + kWideBlock - 1) / kWideBlock);
    if (!grid) return;
    if (dma == 2)
        k_wide_harness<2><<<grid, kWideBlock, 0, st>>>(d_durs, d_idr, S, T, N, sigma, sum_mode, d_ms, d_ng, d_sizes,
                                                       d_start, d_end, d_err);
    else
        k_wide_harness<1><<<grid, kWideBlock, 0, st>>>(d_durs, d_idr, S, T, N, sigma, sum_mode, d_ms, d_ng, d_sizes,
                                                       d_start, d_end, d_err);
}

}  // namespace osim
