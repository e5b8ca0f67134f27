#define OSIM_DMA 2
#define OSIM_SP2 false
#define OSIM_EXH_NAME exh_fast_launch_d2s0
#include "osim_exh_impl.cuh"
