#define OSIM_DMA 2
#include "osim_batch_impl.cuh"

#ifdef OSIM_HSTATS
extern "C" int osim_hstats_batch(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, osim::g_hstats, sizeof(osim::g_hstats));
    if (reset) { unsigned long long z[8] = {0}; cudaMemcpyToSymbol(osim::g_hstats, z, sizeof(z)); }
    return 0;
}
#endif
