// tcgen05.mma issue / execution cost for the shapes of the fused MVM (A operand in TMEM, B in shared
// memory, M = 128): one elected thread issues R instructions back to back, commits, waits.
//   cycles_issue = clock after the last issue - clock before the first
//   cycles_done  = clock after the commit's mbarrier phase completed - clock before the first
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_umma.bin tools/ubench_umma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

template <int KIND, int N, bool A_TMEM, int NACC = 1>
__global__ void __launch_bounds__(128, 1) k(long long* out, int reps) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = (smem_u32(raw) + 1023u) & ~1023u;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND == 0 ? idesc_f16(N) : idesc_tf32(N);
    const uint64_t bdesc = desc_sw128(base), adesc = desc_sw128(base + 32768);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tm + 256 + (r % NACC) * 64, a = tm + (r & 7) * 8;  // NACC independent accumulator chains
      if constexpr (A_TMEM) {
        if constexpr (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
      } else {
        if constexpr (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int KIND, int N, bool A_TMEM, int NACC = 1>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 16);
  auto kk = k<KIND, N, A_TMEM, NACC>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int reps : {16, 256}) {
    kk<<<1, 128, 100 * 1024>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-34s reps %4d: issue %7.1f cyc/instr, until done %7.1f cyc/instr  (%s)\n", name, reps, (double)h[0] / reps,
           (double)h[1] / reps, cudaGetErrorString(e));
  }
  cudaFree(d);
}

int main() {
  run<0, 56, true>("f16  M128 N56  K16 A=TMEM");
  run<0, 64, true>("f16  M128 N64  K16 A=TMEM");
  run<0, 72, true>("f16  M128 N72  K16 A=TMEM");
  run<0, 96, true>("f16  M128 N96  K16 A=TMEM");
  run<0, 128, true>("f16  M128 N128 K16 A=TMEM");
  run<0, 256, true>("f16  M128 N256 K16 A=TMEM");
  run<0, 56, false>("f16  M128 N56  K16 A=smem");
  run<0, 128, false>("f16  M128 N128 K16 A=smem");
  run<1, 64, true>("tf32 M128 N64  K8  A=TMEM");
  run<1, 128, true>("tf32 M128 N128 K8  A=TMEM");
  run<1, 64, false>("tf32 M128 N64  K8  A=smem");
  run<0, 16, true>("f16  M128 N16  K16 A=TMEM");
  // same instruction stream spread over 2 / 4 independent accumulators: is the floor a dependency latency?
  run<0, 56, true, 2>("f16  N56 A=TMEM, 2 accumulators");
  run<0, 56, true, 4>("f16  N56 A=TMEM, 4 accumulators");
  run<1, 64, true, 2>("tf32 N64 A=TMEM, 2 accumulators");
  run<1, 64, true, 4>("tf32 N64 A=TMEM, 4 accumulators");
  run<0, 56, false, 4>("f16  N56 A=smem, 4 accumulators");
  return 0;
}
