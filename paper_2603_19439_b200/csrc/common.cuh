// Common device/host helpers for the B200 G-REST step (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace stg {

using i64 = long long;
using u64 = unsigned long long;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what + ":" + std::to_string(line));
}
#define STG_CUDA(x) ::stg::cuda_check((x), __FILE__, __LINE__)
#define STG_LAUNCH() ::stg::cuda_check(cudaGetLastError(), __FILE__, __LINE__)

__host__ __device__ inline i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }
__host__ __device__ inline i64 round_up(i64 a, i64 b) { return cdiv(a, b) * b; }

// Leading dimension for row-major tall-skinny blocks: multiple of 8 doubles
// (64 B) so every row starts 16 B aligned for cp.async / vector loads.
inline int ld_for(i64 cols) { return static_cast<int>(round_up(cols < 1 ? 1 : cols, 8)); }

// ---------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// Two doubles; sub-block views with odd column offsets are only 8-byte aligned.
__device__ __forceinline__ void cp_async_pair(double* smem, const double* gmem) {
  if ((reinterpret_cast<unsigned long long>(gmem) & 15ULL) == 0) {
    cp_async16(smem, gmem);
  } else {
    cp_async8(smem, gmem);
    cp_async8(smem + 1, gmem + 1);
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a): D(8x8) += A(8x4) B(4x8).
// Fragment ownership for lane l, g = l >> 2, t = l & 3:
//   a = A[g][t], b = B[t][g], {c0, c1} = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace stg
