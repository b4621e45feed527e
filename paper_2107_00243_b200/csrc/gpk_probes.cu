// Device-side Rademacher probes: the reference draws z(i, c) = +-1/sqrt(n)
// from the low bit of consecutive outputs of ONE std::mt19937_64(seed) stream in column-major
// order (trace_estimation.hpp:27-36).  The stream is a linear recurrence of period-312 blocks:
//     mt[i] <- mt[i + 156] ^ twist(mt[i], mt[i + 1])        (indices mod 312, in place)
// whose first 156 new words depend on old words only and whose last 156 on old words and the
// first 156 new ones -- so one CTA regenerates a block in two 156-wide parallel steps, tempers
// the 312 words in parallel and stores 312 probes with coalesced 8-byte stores.  Bitwise the
// host stream (tests/test_gpu_kernels.py::test_device_probes_equal_host_stream); the n x l
// block never crosses PCIe (C5: 537 MB per optimizer step).
#include "gpk_common.cuh"
#include "gpk_internal.h"

namespace gpk {
namespace {
constexpr int kN = 312, kM = 156;
constexpr unsigned long long kA = 0xB5026F5AA96619E9ULL, kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;

GPK_DEV unsigned long long twist(unsigned long long a, unsigned long long b) {
  const unsigned long long x = (a & kUpper) | (b & kLower);
  return (x >> 1) ^ ((x & 1ULL) ? kA : 0ULL);
}
GPK_DEV unsigned long long temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  return y ^ (y >> 43);
}

__global__ void __launch_bounds__(320, 1)
    mt19937_64_probes_kernel(unsigned long long seed, long long total, double inv, double* __restrict__ out) {
  __shared__ unsigned long long mt[kN];
  const int tid = threadIdx.x;
  if (tid == 0) {  // std::mt19937_64 seeding
    unsigned long long v = seed;
    mt[0] = v;
    for (int i = 1; i < kN; ++i) {
      v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<unsigned long long>(i);
      mt[i] = v;
    }
  }
  __syncthreads();
  for (long long base = 0; base < total; base += kN) {
    unsigned long long v = 0;
    if (tid < kM) v = mt[tid + kM] ^ twist(mt[tid], mt[tid + 1]);
    __syncthreads();
    if (tid < kM) mt[tid] = v;
    __syncthreads();
    if (tid < kM) {
      const int i = kM + tid;
      v = mt[tid] ^ twist(mt[i], mt[i + 1 == kN ? 0 : i + 1]);
    }
    __syncthreads();
    if (tid < kM) mt[kM + tid] = v;
    __syncthreads();
    if (tid < kN && base + tid < total) out[base + tid] = (temper(mt[tid]) & 1ULL) ? inv : -inv;
  }
}
}  // namespace

cudaError_t launch_make_probes(long long n, int count, unsigned long long seed, double* out, cudaStream_t st) {
  mt19937_64_probes_kernel<<<1, 320, 0, st>>>(seed, n * count, 1.0 / sqrt(static_cast<double>(n)), out);
  return cudaGetLastError();
}

}  // namespace gpk
