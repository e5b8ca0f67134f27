#define OSIM_DMA 1
#include "osim_batch_impl.cuh"
