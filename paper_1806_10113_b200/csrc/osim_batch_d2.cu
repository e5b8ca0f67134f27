#define OSIM_DMA 2
#include "osim_batch_impl.cuh"
