// The RSVD test matrix Omega on the device, bit-compatible with the reference
// GaussianSampler (proj/include/spectrack/rng.hpp:27-75): std::mt19937_64
// draws, 53-bit uniforms, Box-Muller with u1 = 1 - U (cos first, sin second),
// column-major fill of an S x q matrix.
//
// The mt19937_64 sequence obeys x[j+312] = x[j+156] ^ twist(x[j], x[j+1]), so
// 156 consecutive new words depend only on the previous 312: one CTA advances
// the recurrence 156 words per barrier over a 468-slot ring in shared memory
// and writes the tempered outputs; Box-Muller then runs fully parallel.
#pragma once

#include "common.cuh"

namespace stg {

constexpr int kMtN = 312, kMtM = 156, kMtRing = 468;

__device__ __forceinline__ u64 mt_temper(u64 y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

// Generates tempered outputs [156 b_begin, 156 b_end) of the stream seeded with
// `seed`. With init the ring is seeded; otherwise it resumes from `state`
// (the 468-word ring saved by the previous launch), so a speculative prefix
// can be extended when more words turn out to be needed.
__global__ void __launch_bounds__(160) mt19937_64_kernel(u64 seed, i64 b_begin, i64 b_end, int init, u64* state,
                                                         u64* out) {
  __shared__ u64 ring[kMtRing];
  const int i = threadIdx.x;
  if (init) {
    if (i == 0) {  // std::mersenne_twister_engine::seed: x_j = f (x_{j-1} ^ (x_{j-1} >> 62)) + j
      u64 x = seed;
      ring[0] = x;
      for (int j = 1; j < kMtN; ++j) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<u64>(j);
        ring[j] = x;
      }
    }
  } else {
    for (int j = i; j < kMtRing; j += blockDim.x) ring[j] = state[j];
  }
  __syncthreads();
  for (i64 b = b_begin; b < b_end; ++b) {
    // new word J + 312 + i from x[J+i], x[J+i+1], x[J+156+i], J = 156 b
    if (i < kMtM) {
      const i64 J = b * kMtM;
      const u64 xi = ring[(J + i) % kMtRing];
      const u64 xi1 = ring[(J + i + 1) % kMtRing];
      const u64 xm = ring[(J + kMtM + i) % kMtRing];
      const u64 y = (xi & 0xFFFFFFFF80000000ULL) | (xi1 & 0x7FFFFFFFULL);
      const u64 v = xm ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
      ring[(J + kMtN + i) % kMtRing] = v;
      out[J + i] = mt_temper(v);
    }
    __syncthreads();
  }
  for (int j = i; j < kMtRing; j += blockDim.x) state[j] = ring[j];
}

// Omega(r, c) = normal #(c * S + r); normals come in (cos, sin) pairs from
// uniforms (2 p, 2 p + 1). Stored row-major S x q with leading dimension ld.
__global__ void box_muller_kernel(const u64* raw, i64 npairs, i64 S, int q, double* omega, int ld) {
  const i64 p = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  const double u1 = 1.0 - static_cast<double>(raw[2 * p] >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(raw[2 * p + 1] >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  constexpr double two_pi = 6.283185307179586476925286766559;
  double sn, cs;
  sincos(two_pi * u2, &sn, &cs);
  const i64 total = S * q;
  const i64 o0 = 2 * p, o1 = 2 * p + 1;
  if (o0 < total) omega[(o0 % S) * ld + o0 / S] = r * cs;
  if (o1 < total) omega[(o1 % S) * ld + o1 / S] = r * sn;
}

}  // namespace stg
