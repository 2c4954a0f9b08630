// enum_plain.cu -- enumeration kernels with probe-built rows for every candidate.
#define BC_COMPACT 0
#include "enum_inst.cuh"
