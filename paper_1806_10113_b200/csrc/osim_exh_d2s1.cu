#define OSIM_DMA 2
#define OSIM_SP2 true
#define OSIM_EXH_NAME exh_fast_launch_d2s1
#include "osim_exh_impl.cuh"
