// osim_heur.cu -- instantiations and launch of the heuristic kernel.
#include <cmath>
#include <cstdlib>

#include "osim_launch.cuh"
#include "osim_heur_lane.cuh"
#include "osim_heur_null.cuh"

namespace osim {

#ifndef OSIM_HEUR_LANE_DEFAULT
#define OSIM_HEUR_LANE_DEFAULT 1
#endif
// which all-non-null heuristic kernel runs: k_heuristic_lane (one group per
// lane) or k_heuristic_fast (8 groups per warp); OSIM_HEUR_LANE=0/1 overrides
// the default (tuning only)
static bool lane_kernel() {
    static const bool v = [] {
        const char* e = std::getenv("OSIM_HEUR_LANE");
        return e ? std::atoi(e) != 0 : (OSIM_HEUR_LANE_DEFAULT != 0);
    }();
    return v;
}

void heuristic_launch(int dma, int mode, const LaunchCfg& cfg, const double* d_durs, const uint8_t* d_idr,
                      uint64_t B, int n, double sigma, int sum_mode, uint8_t* d_order, double* d_ms,
                      uint32_t* d_ns, int* d_err) {
    const unsigned grid = (unsigned)((B + kHG - 1) / kHG);
    const size_t sm = sizeof(HeurShared);
    if (mode == 1 && lane_kernel()) {
        const unsigned gl = (unsigned)((B + kHLT - 1) / kHLT);
        const size_t sml = kHLW * kHLWarpSmem;
        int e;
        const bool sp2 = std::frexp(sigma, &e) == 0.5;
#define OSIM_HLN(D, P)                                                                               \
    do {                                                                                             \
        auto kf = k_heuristic_lane<D, P>;                                                            \
        cached_ctas_per_sm((const void*)kf, kHLT, sml); /* opts in to > 48 KB dynamic smem */        \
        kf<<<gl, kHLT, sml, cfg.st>>>(d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms, d_ns);   \
    } while (0)
        if (dma == 2) { if (sp2) OSIM_HLN(2, true); else OSIM_HLN(2, false); }
        else OSIM_HLN(1, false);
#undef OSIM_HLN
        return;
    }
    if (mode == 1) {
        const unsigned gridf = (unsigned)((B + kHGF - 1) / kHGF);
        int e;
        const bool sp2 = std::frexp(sigma, &e) == 0.5;
#define OSIM_HF(D, P)                                                                                       \
    k_heuristic_fast<D, P><<<gridf, kHTF, kWPB * sizeof(HeurWarpShared<D, P>), cfg.st>>>(d_durs, d_idr, B, n, sigma, \
                                                                                 sum_mode, d_order, d_ms, d_ns)
        if (dma == 2) { if (sp2) OSIM_HF(2, true); else OSIM_HF(2, false); }
        else OSIM_HF(1, false);
#undef OSIM_HF
        return;
    }
#define OSIM_HL(D, M) \
    k_heuristic<D, M><<<grid, kHT, sm, cfg.st>>>(d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms, d_ns, d_err)
    if (mode == 2) {  // null stages in the fast range: NullSim with prefix-world checkpoints
        const unsigned gridf = (unsigned)((B + kHGF - 1) / kHGF);
        int e;
        const bool sp2 = std::frexp(sigma, &e) == 0.5;
#define OSIM_HN(D, P)                                                                                         \
    k_heuristic_nullck<D, P><<<gridf, kHTF, kWPB * sizeof(NullHeurWarpShared<D, P>), cfg.st>>>(              \
        d_durs, d_idr, B, n, sigma, sum_mode, d_order, d_ms, d_ns, d_err)
        if (dma == 2) { if (sp2) OSIM_HN(2, true); else OSIM_HN(2, false); }
        else OSIM_HN(1, false);
#undef OSIM_HN
    } else {
        if (dma == 2) OSIM_HL(2, 0); else OSIM_HL(1, 0);
    }
#undef OSIM_HL
}

}  // namespace osim

#ifdef OSIM_HSTATS
extern "C" int osim_hstats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, osim::g_hstats, sizeof(osim::g_hstats));
    if (reset) { unsigned long long z[8] = {0}; cudaMemcpyToSymbol(osim::g_hstats, z, sizeof(z)); }
    return 0;
}
#endif
