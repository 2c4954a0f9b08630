// enum_compact.cu -- enumeration kernels with wedge-scattered rows for the
// level-1 survivors only (FR-shaped graphs: short opposite-layer rows).
#define BC_COMPACT 1
#include "enum_inst.cuh"
