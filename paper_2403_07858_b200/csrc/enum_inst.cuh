// enum_inst.cuh -- instantiates the enumeration kernels for one COMPACT value
// (included by enum_plain.cu / enum_compact.cu, which define BC_COMPACT) and
// defines that value's launchers declared in search_dev.cuh.
#include "search_dev.cuh"

#if BC_COMPACT
#define BC_SFX(x) x##_c1
#else
#define BC_SFX(x) x##_c0
#endif

namespace bc {
namespace sk {
namespace {

typedef void (*EnumFn)(Params, EnumArgs);
typedef void (*SubFn)(Params, EnumArgs, int64_t);

template <bool I>
EnumFn pick_enum(const EnumVariant &v) {
  constexpr bool C = BC_COMPACT != 0;
  if (v.split) return enum_kernel<I, false, true, false, C>;
  if (v.triage) return enum_kernel<I, false, false, true, C>;
  if (v.lazy) return enum_kernel<I, true, false, false, C>;
  return enum_kernel<I, false, false, false, C>;
}

EnumFn pick(const EnumVariant &v) { return v.instr ? pick_enum<true>(v) : pick_enum<false>(v); }

SubFn pick_sub(bool instr) {
  constexpr bool C = BC_COMPACT != 0;
  return instr ? sub_kernel<true, C> : sub_kernel<false, C>;
}

template <typename K>
int occupancy(K kern, size_t smem) {
  BC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ENUM_THREADS, smem));
  return per_sm < 1 ? 1 : per_sm;
}

}  // namespace

int BC_SFX(enum_blocks_per_sm)(const EnumVariant &v, size_t smem) { return occupancy(pick(v), smem); }

void BC_SFX(enum_launch)(const EnumVariant &v, unsigned blocks, size_t smem, cudaStream_t st,
                         const Params &P, const EnumArgs &A) {
  pick(v)<<<blocks, ENUM_THREADS, smem, st>>>(P, A);
  BC_CHECK_LAUNCH();
}

int BC_SFX(sub_blocks_per_sm)(bool instr, size_t smem) { return occupancy(pick_sub(instr), smem); }

void BC_SFX(sub_launch)(bool instr, unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                        const EnumArgs &A, int64_t n_sub) {
  pick_sub(instr)<<<blocks, ENUM_THREADS, smem, st>>>(P, A, n_sub);
  BC_CHECK_LAUNCH();
}

int BC_SFX(filter_blocks_per_sm)(size_t smem) {
  return occupancy(filter_kernel<BC_COMPACT != 0>, smem);
}

void BC_SFX(filter_launch)(unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                           const EnumArgs &A) {
  filter_kernel<BC_COMPACT != 0><<<blocks, ENUM_THREADS, smem, st>>>(P, A);
  BC_CHECK_LAUNCH();
}

void BC_SFX(phase_cycles)(unsigned long long *h, bool reset) {
#ifdef BC_PHASE_PROF
  BC_CUDA(cudaMemcpyFromSymbol(h, g_phase, 16 * sizeof(unsigned long long)));
  if (reset) {
    const unsigned long long z[16] = {0};
    BC_CUDA(cudaMemcpyToSymbol(g_phase, z, sizeof z));
  }
#else
  for (int i = 0; i < 16; i++) h[i] = 0;
  (void)reset;
#endif
}

}  // namespace sk
}  // namespace bc
