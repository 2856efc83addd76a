// MapElites device loop (qd_optimizer.cpp:12-417). Entry points are defined
// in capi.cu; the kernels live here.
#include "qd.cuh"
