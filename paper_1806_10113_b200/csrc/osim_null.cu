// osim_null.cu -- instantiations of the null-stage prefix-sharing kernel
// (osim_null.cuh), one per (n, DMA, sigma-is-a-power-of-two).
#include "osim_launch.cuh"
#include "osim_null.cuh"

namespace osim {
namespace {

template <int N, int DMA, bool SP2>
int null_t(const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo, uint64_t hi, double thr,
           Part* parts, int max_parts, double* d_ms, int* d_err, int* g_out) {
    constexpr int L = default_pfx_l(N);
    auto k = k_exhaustive_null_pfx<N, DMA, SP2, L>;
    constexpr uint64_t LF = Fact<L>::v;
    const uint64_t prefixes = (hi + LF - 1) / LF - lo / LF;
    int g = grid_for_sms(k, kBlock, 0, cfg.sms, (prefixes + kBlock - 1) / kBlock);
    if (g > max_parts) g = max_parts;
    k<<<g, kBlock, 0, cfg.st>>>(d_durs, sigma, lo, hi, thr, parts, d_ms, d_err);
    *g_out = g;
    return 0;
}

template <int N>
int null_n(int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo, uint64_t hi,
           double thr, Part* parts, int max_parts, double* d_ms, int* d_err, int* g) {
    if (dma == 1) return null_t<N, 1, false>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, d_err, g);
    if (sp2) return null_t<N, 2, true>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, d_err, g);
    return null_t<N, 2, false>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, d_err, g);
}

template <int N, int DMA, bool SP2>
int nullb_t(const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma, osim_summary* d_out, int* d_err,
            int* g_out) {
    auto k = k_exhaustive_batch_null_pfx<N, DMA, SP2, default_pfx_l(N)>;
    const int g = grid_for_sms(k, kBlock, 0, cfg.sms, B);
    k<<<g, kBlock, 0, cfg.st>>>(d_durs, B, sigma, d_out, d_err);
    *g_out = g;
    return 0;
}

template <int N>
int nullb_n(int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
            osim_summary* d_out, int* d_err, int* g) {
    if (dma == 1) return nullb_t<N, 1, false>(cfg, d_durs, B, sigma, d_out, d_err, g);
    if (sp2) return nullb_t<N, 2, true>(cfg, d_durs, B, sigma, d_out, d_err, g);
    return nullb_t<N, 2, false>(cfg, d_durs, B, sigma, d_out, d_err, g);
}

}  // namespace

int null_batch_launch(int n, int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
                      osim_summary* d_out, int* d_err, int* g) {
    switch (n) {
#define OSIM_CASE(NN) \
    case NN: return nullb_n<NN>(dma, sp2, cfg, d_durs, B, sigma, d_out, d_err, g);
        OSIM_CASE(1) OSIM_CASE(2) OSIM_CASE(3) OSIM_CASE(4) OSIM_CASE(5) OSIM_CASE(6) OSIM_CASE(7) OSIM_CASE(8)
        OSIM_CASE(9) OSIM_CASE(10) OSIM_CASE(11) OSIM_CASE(12)
#undef OSIM_CASE
        default: return -1;
    }
}

int null_pfx_launch(int n, int dma, bool sp2, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo,
                    uint64_t hi, double thr, Part* parts, int max_parts, double* d_ms, int* d_err, int* g) {
    switch (n) {
#define OSIM_CASE(NN) \
    case NN: return null_n<NN>(dma, sp2, cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, d_err, g);
        OSIM_CASE(1) OSIM_CASE(2) OSIM_CASE(3) OSIM_CASE(4) OSIM_CASE(5) OSIM_CASE(6) OSIM_CASE(7) OSIM_CASE(8)
        OSIM_CASE(9) OSIM_CASE(10) OSIM_CASE(11) OSIM_CASE(12) OSIM_CASE(13) OSIM_CASE(14) OSIM_CASE(15)
        OSIM_CASE(16)
#undef OSIM_CASE
        default: return -1;
    }
}

}  // namespace osim
