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

// 128-bit accumulator as two u64 limbs (lo, hi) with explicit carry.  A carry out
// of hi (a partial sum of terms that each fit 128 bits passing 2^128) latches `ovf`,
// which atomic_add128 turns into the BC_EOVERFLOW flag: never a wrapped count.
struct Acc128 {
  unsigned long long lo, hi;
  unsigned ovf;
  __device__ __forceinline__ void add(unsigned long long xlo, unsigned long long xhi) {
    const unsigned long long n = lo + xlo;
    const unsigned long long h1 = hi + xhi;
    const unsigned long long h2 = h1 + (n < lo ? 1ull : 0ull);
    ovf |= (h1 < hi) | (h2 < h1);
    hi = h2;
    lo = n;
  }
  __device__ __forceinline__ void add(const Acc128 &o) {
    add(o.lo, o.hi);
    ovf |= o.ovf;
  }
};

__device__ __forceinline__ Acc128 warp_sum128(Acc128 a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long l = __shfl_xor_sync(FULL, a.lo, o);
    unsigned long long h = __shfl_xor_sync(FULL, a.hi, o);
    a.add(l, h);
  }
  a.ovf = __any_sync(FULL, a.ovf != 0) ? 1u : 0u;
  return a;
}

// Global 128-bit accumulation with carry; sets *overflow if the sum passes 2^128.
__device__ __forceinline__ void atomic_add128(unsigned long long *lo_hi, int *overflow,
                                              unsigned long long lo, unsigned long long hi) {
  unsigned long long carry = 0;
  if (lo) {
    const unsigned long long old = atomicAdd(lo_hi, lo);
    carry = old + lo < old ? 1ull : 0ull;
  }
  if (hi | carry) {
    const unsigned long long h = hi + carry;
    if (h < hi) {  // hi == ~0 and a carry in: the sum is >= 2^128
      atomicExch(overflow, 1);
      return;
    }
    const unsigned long long old = atomicAdd(lo_hi + 1, h);
    if (old + h < old) atomicExch(overflow, 1);
  }
}

__device__ __forceinline__ void atomic_add128(unsigned long long *lo_hi, int *overflow,
                                              const Acc128 &a) {
  if (a.ovf) atomicExch(overflow, 1);
  atomic_add128(lo_hi, overflow, a.lo, a.hi);
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
