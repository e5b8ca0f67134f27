#define OSIM_DMA 1
#define OSIM_SP2 false
#define OSIM_EXH_NAME exh_fast_launch_d1
#include "osim_exh_impl.cuh"
