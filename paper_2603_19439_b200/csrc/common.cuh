// Common device/host helpers for the B200 G-REST step (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

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

// ---------------------------------------------------------------- mbarrier + bulk copy
// Asynchronous bulk global->shared copies (the TMA unit's non-tensor mode)
// completing on an mbarrier with a transaction byte count.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// The spin loop is C++ around a single try_wait, so the compiler sees the
// (lane-divergent) loop and reconverges the warp after it: a branch hidden
// inside one asm block would let lanes reach the following mma.sync.aligned
// unconverged (undefined behaviour, observed as sporadically wrong tiles).
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// bytes: multiple of 16; both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 2-D TMA tile load (cp.async.bulk.tensor): box {bw columns, bh rows} at
// column x, row y of a row-major fp64 tensor map; out-of-range elements are
// zero-filled; completes on `bar` with the full box's bytes.
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(smem)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Host: tensor map of a row-major rows x cols fp64 block with leading
// dimension ld (base 16-byte aligned, ld even), box {bw, bh}.
inline CUtensorMap make_tmap_2d(const double* base, i64 rows, i64 cols, int ld, int bw, int bh) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    STG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
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
