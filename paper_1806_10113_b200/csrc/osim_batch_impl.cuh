// osim_batch_impl.cuh -- instantiations of the batched prefix-sharing
// exhaustive kernel (one CTA per group) for one DMA mode.
#include "osim_launch.cuh"

namespace osim {
namespace {

template <int N, bool SP2, int L>
int batch_t(const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma, osim_summary* d_out) {
    auto k = k_exhaustive_batch_pfx<N, OSIM_DMA, SP2, L>;
    const int g = grid_for_sms(k, kBlock, kPfxDynSmem, cfg.sms, B);
    k<<<g, kBlock, kPfxDynSmem, cfg.st>>>(d_durs, B, sigma, d_out);
    return 0;
}

template <int N, bool SP2>
int batch_n(int L, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma, osim_summary* d_out) {
    if constexpr (N == 8) {
        if (L == 4) return batch_t<N, SP2, 4>(cfg, d_durs, B, sigma, d_out);
        if (L == 5) return batch_t<N, SP2, 5>(cfg, d_durs, B, sigma, d_out);
    }
    return batch_t<N, SP2, default_pfx_l(N)>(cfg, d_durs, B, sigma, d_out);
}

template <bool SP2>
int batch_any(int n, int L, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
              osim_summary* d_out) {
    switch (n) {
#define OSIM_CASE(NN) case NN: return batch_n<NN, SP2>(L, cfg, d_durs, B, sigma, d_out);
        OSIM_CASE(1) OSIM_CASE(2) OSIM_CASE(3) OSIM_CASE(4) OSIM_CASE(5) OSIM_CASE(6)
        OSIM_CASE(7) OSIM_CASE(8) OSIM_CASE(9) OSIM_CASE(10) OSIM_CASE(11) OSIM_CASE(12)
#undef OSIM_CASE
    }
    return -1;
}

}  // namespace

#if OSIM_DMA == 2
int batch_fast_launch_d2(int n, int L, bool sp2, const LaunchCfg& cfg, const double* d_durs, uint64_t B,
                         double sigma, osim_summary* d_out) {
    return sp2 ? batch_any<true>(n, L, cfg, d_durs, B, sigma, d_out)
               : batch_any<false>(n, L, cfg, d_durs, B, sigma, d_out);
}
#else
int batch_fast_launch_d1(int n, int L, const LaunchCfg& cfg, const double* d_durs, uint64_t B, double sigma,
                         osim_summary* d_out) {
    return batch_any<false>(n, L, cfg, d_durs, B, sigma, d_out);
}
#endif

}  // namespace osim
