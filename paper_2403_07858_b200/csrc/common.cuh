// common.cuh -- shared helpers for the B200 (sm_100a) biclique counting path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/bicount_b200.h"

namespace bc {

typedef unsigned __int128 u128;

// Error carried from deep inside the host orchestration to the C-ABI edge.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define BC_CUDA(call)                                                            \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess)                                                       \
      throw ::bc::Error(_e == cudaErrorMemoryAllocation ? BC_EOOM : BC_ECUDA,    \
                        std::string(#call) + ": " + cudaGetErrorString(_e) +     \
                            " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define BC_CHECK_LAUNCH() BC_CUDA(cudaGetLastError())

constexpr int WARP = 32;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// 128-bit accumulator as two u64 limbs (lo, hi) with explicit carry.
struct Acc128 {
  unsigned long long lo, hi;
  __device__ __forceinline__ void add(unsigned long long xlo, unsigned long long xhi) {
    unsigned long long n = lo + xlo;
    hi += xhi + (n < lo ? 1ull : 0ull);
    lo = n;
  }
};

__device__ __forceinline__ Acc128 warp_sum128(Acc128 a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long l = __shfl_xor_sync(FULL, a.lo, o);
    unsigned long long h = __shfl_xor_sync(FULL, a.hi, o);
    a.add(l, h);
  }
  return a;
}

// Global 128-bit accumulation with carry; sets *overflow if the sum passes 2^128.
__device__ __forceinline__ void atomic_add128(unsigned long long *lo_hi, int *overflow,
                                              unsigned long long lo, unsigned long long hi) {
  if (lo) {
    unsigned long long old = atomicAdd(lo_hi, lo);
    if (old + lo < old) hi += 1;  // hi+1 cannot wrap unless hi == ~0: caught below
  }
  if (hi) {
    unsigned long long old = atomicAdd(lo_hi + 1, hi);
    if (old + hi < old) atomicExch(overflow, 1);
  }
}

// lower_bound over a sorted u32 array in [lo, hi).
__device__ __forceinline__ int64_t lower_bound_u32(const uint32_t *__restrict__ a, int64_t lo,
                                                   int64_t hi, uint32_t key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

}  // namespace bc
