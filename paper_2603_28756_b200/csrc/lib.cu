// Unity translation unit: the whole library is one TU so the per-device
// twiddle table (a __device__ global) is shared without relocatable device code.
#include "capi.cu"
#include "toeplitz.cu"
#include "nufft.cu"
#include "resample.cu"
#include "reduce.cu"
#include "qggmrf.cu"
