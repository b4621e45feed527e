// Pipe-throughput microbenchmarks for the instructions of the fused-MVM producer loop
// (MUFU.SQRT / EX2 / RSQ, F2FP pack, FHADD, FFMA2, FMNMX): thread-instructions per clock per SM
// at the kernel's own occupancy (16 warps per SM) and at 32 / 64 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_pipes.cu && /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP 64
#define ILP 8

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[ILP];
  uint32_t h[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    v[i] = 1.0f + threadIdx.x * 1e-3f + i;
    h[i] = threadIdx.x + i;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < REP / ILP; ++r) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if constexpr (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        if constexpr (OP == 1) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        if constexpr (OP == 2) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        if constexpr (OP == 3) asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h[i]) : "f"(v[i]), "r"(h[i]));
        if constexpr (OP == 4) {
          unsigned short hs = static_cast<unsigned short>(h[i]);
          asm volatile("{\n\t.reg .f16 n;\n\tneg.f16 n, %1;\n\tadd.rn.f32.f16 %0, n, %0;\n\t}" : "+f"(v[i]) : "h"(hs));
        }
        if constexpr (OP == 5) {
          // packed FFMA2
          unsigned long long a;
          asm volatile("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(v[i]));
          asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a));
          asm volatile("{.reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.f32 %0, lo;}" : "=f"(v[i]) : "l"(a));
        }
        if constexpr (OP == 6) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
        if constexpr (OP == 7) asm volatile("min.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(v[(i + 1) % ILP]));
        if constexpr (OP == 8) {  // the producer's mix per entry: sqrt, ex2, fma, mul
          float s, e;
          asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(v[i]));
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-s));
          v[i] = fmaf(s, 1.5f, 1.0f) * e + 1.0f;
        }
        if constexpr (OP == 9) {  // rsq + mul instead of sqrt
          float s, e;
          asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(v[i]));
          s *= v[i];
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-s));
          v[i] = fmaf(s, 1.5f, 1.0f) * e + 1.0f;
        }
      }
    }
  }
  long long t1 = clock64();
  float acc = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc += v[i] + __uint_as_float(h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps, double per_iter) {
  int sms = 148;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 2048 * 4);
  cudaMalloc(&cyc, sms * 8);
  int iters = 2000;
  k<OP><<<sms, warps * 32>>>(out, 10, cyc);
  k<OP><<<sms, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  double thr = (double)iters * REP * per_iter * warps * 32 / c;
  printf("%-28s warps/SM %2d: %7.2f thread-ops / clk / SM  (%.1f cycles per warp-op per SMSP-resident warp set)\n", name,
         warps, thr, c / ((double)iters * REP * per_iter));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {16, 32}) {
    run<0>("MUFU.EX2", w, 1);
    run<1>("MUFU.SQRT", w, 1);
    run<2>("MUFU.RSQ", w, 1);
    run<3>("F2FP.F16.F32.PACK_AB", w, 1);
    run<4>("FHADD (f32 = -f16 + f32)", w, 1);
    run<5>("FFMA2 (+2 movs)", w, 1);
    run<6>("FFMA", w, 1);
    run<7>("FMNMX", w, 1);
    run<8>("entry: SQRT+EX2+FMA+FMUL+FADD", w, 1);
    run<9>("entry: RSQ+MUL+EX2+FMA+..", w, 1);
  }
  return 0;
}
