#define OSIM_DMA 2
#define OSIM_SP2 true
#define OSIM_EXH_NAME exh_fast_launch_d2s1
#include "osim_exh_impl.cuh"

#ifdef OSIM_HSTATS
extern "C" int osim_hstats_exh(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, osim::g_hstats, sizeof(osim::g_hstats));
    if (reset) { unsigned long long z[8] = {0}; cudaMemcpyToSymbol(osim::g_hstats, z, sizeof(z)); }
    return 0;
}
#endif
