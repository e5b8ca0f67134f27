// osim_heur.cu -- instantiations and launch of the heuristic kernel.
#include "osim_launch.cuh"

namespace osim {

void heuristic_launch(int dma, bool fast, const LaunchCfg& cfg, const double* d_durs, const uint8_t* d_idr,
                      uint64_t B, int n, double sigma, int sum_mode, uint8_t* d_order, double* d_ms,
                      uint32_t* d_ns, int* d_err) {
    const unsigned grid = (unsigned)((B + kHG - 1) / kHG);
    const size_t sm = sizeof(HeurShared);
#define OSIM_HL(D, F) \
    k_heuristic<D, F><<<grid, kHT, sm, cfg.st>>>(d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms, d_ns, d_err)
    if (dma == 2) { if (fast) OSIM_HL(2, true); else OSIM_HL(2, false); }
    else { if (fast) OSIM_HL(1, true); else OSIM_HL(1, false); }
#undef OSIM_HL
}

}  // namespace osim
