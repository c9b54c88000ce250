// Pipe-throughput microbenchmark for the KSG inner-loop instruction mix on sm_100a.
// Measures warp-instructions issued per SM per cycle (clock64 per block) for
// FMNMX, FMNMX3, FADD, FADD2, FFMA, IADD3, packed f16/bf16/s16 min-max, HADD2, HSETP2, F2FP, LOP3
// and mixes. Informs DESIGN.md's ALU roofline.
// Build (the binary is not tracked): nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -o tools/pipe_microbench tools/pipe_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
template <int OP>
__global__ void __launch_bounds__(256) bench(float* out, int iters, long long* cyc) {
  float a[CH], b[CH];
  unsigned long long p[CH];
  unsigned int u[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = threadIdx.x * 0.001f + c;
    b[c] = blockIdx.x * 0.002f - c;
    float2 f = make_float2(a[c], b[c]);
    p[c] = *reinterpret_cast<unsigned long long*>(&f);
    u[c] = threadIdx.x + c;
  }
  unsigned long long q = p[0] ^ 0x1234;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      // alternating max / min on the same chain: ptxas cannot fold two of them into one FMNMX3
      // (a max-max pair on one register IS folded, which made an earlier version of this test
      // report twice the real FMNMX rate)
      if (OP == 0) {
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[(c + 1) % CH]));
      }
      if (OP == 1) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(b[c]), "f"(b[(c + 1) % CH]));
      if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
      if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(q));
      if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(b[c]), "f"(b[(c + 3) % CH]));
      if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
      if (OP == 6) {  // 1 FADD2 : 1 FMNMX
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(q));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
      }
      if (OP == 7) {  // 1 FADD2 : 3 FMNMX
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(q));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(b[c]) : "f"(a[c]));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
      }
      if (OP == 8) {  // 1 FFMA : 1 FMNMX
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(b[c]) : "f"(b[(c + 1) % CH]), "f"(b[(c + 2) % CH]));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(a[(c + 1) % CH]));
      }
      if (OP == 9) {  // FSETP + SELP-free: set.lt predicate then predicated add
        asm volatile("{.reg .pred q; setp.lt.f32 q, %0, %1; @q add.u32 %2, %2, 1;}" : "+f"(a[c]), "+f"(b[c]), "+r"(u[c]));
      }
      if (OP == 10) asm volatile("min.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
      if (OP == 12) {  // packed f16 min / max (alternating, as OP 0)
        asm volatile("max.f16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
        asm volatile("min.f16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 2) % CH]));
      }
      if (OP == 13) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
      if (OP == 14) {  // packed f16 compare feeding a predicated add
        asm volatile("{.reg .pred p, q; setp.lt.f16x2 p|q, %1, %2; @p add.u32 %0, %0, 1;}" : "+r"(u[c]) : "r"(u[(c + 1) % CH]), "r"(u[(c + 2) % CH]));
      }
      if (OP == 15) {  // f32 pair -> packed f16 (F2FP)
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(a[(c + 1) % CH]));
        asm volatile("add.f32 %0, %0, 1.0;" : "+f"(a[c]));
      }
      if (OP == 16) {  // packed bf16 min / max
        asm volatile("max.bf16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
        asm volatile("min.bf16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 2) % CH]));
      }
      if (OP == 17) {  // packed s16 min / max
        asm volatile("max.s16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
        asm volatile("min.s16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 2) % CH]));
      }
      if (OP == 18) asm volatile("lop3.b32 %0, %0, %1, %2, 0xe8;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]), "r"(u[(c + 2) % CH]));
      if (OP == 11) {  // the merge network's shape: min(l, max(l', a)) pairs
        asm volatile("max.f32 %0, %1, %2;" : "=f"(b[c]) : "f"(a[c]), "f"(a[(c + 1) % CH]));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  unsigned int us = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float2 f = *reinterpret_cast<float2*>(&p[c]);
    s += a[c] + b[c] + f.x + f.y;
    us += u[c];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + us;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_body, float* d_out, long long* d_cyc, int blocks, int threads, int iters) {
  bench<OP><<<blocks, threads>>>(d_out, iters, d_cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<blocks, threads>>>(d_out, iters, d_cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  static long long h[148 * 64];
  cudaMemcpy(h, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0; long long mx = 0;
  for (int i = 0; i < blocks; ++i) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= blocks;
  int sms = 148;
  double warp_instr_per_sm = (double)blocks / sms * (threads / 32) * (double)iters * CH * per_body;
  double ipc = warp_instr_per_sm / mx;
  double clk = mx / (ms * 1e-3) / 1e6;  // approx MHz (kernel-wide)
  printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f, \"lane_ops_per_clk_per_sm\": %.1f, \"max_cycles\": %lld, \"ms\": %.3f, \"eff_mhz\": %.0f}\n",
         name, ipc, ipc * 32, mx, ms, clk);
}

int main() {
  int blocks = 148 * 4, threads = 256, iters = 1 << 14;
  float* d_out; long long* d_cyc;
  cudaMalloc(&d_out, blocks * threads * sizeof(float));
  cudaMalloc(&d_cyc, blocks * sizeof(long long));
  run<0>("FMNMX", 2, d_out, d_cyc, blocks, threads, iters);
  run<1>("FMNMX3", 1, d_out, d_cyc, blocks, threads, iters);
  run<2>("FADD", 1, d_out, d_cyc, blocks, threads, iters);
  run<3>("FADD2", 1, d_out, d_cyc, blocks, threads, iters);
  run<4>("FFMA", 1, d_out, d_cyc, blocks, threads, iters);
  run<5>("IADD3", 1, d_out, d_cyc, blocks, threads, iters);
  run<6>("FADD2+FMNMX", 2, d_out, d_cyc, blocks, threads, iters);
  run<7>("FADD2+3FMNMX", 4, d_out, d_cyc, blocks, threads, iters);
  run<8>("FFMA+FMNMX", 2, d_out, d_cyc, blocks, threads, iters);
  run<9>("FSETP+@IADD", 2, d_out, d_cyc, blocks, threads, iters);
  run<10>("IMNMX", 1, d_out, d_cyc, blocks, threads, iters);
  run<11>("FMNMX max->min pairs", 2, d_out, d_cyc, blocks, threads, iters);
  run<12>("HMNMX2", 2, d_out, d_cyc, blocks, threads, iters);
  run<13>("HADD2", 1, d_out, d_cyc, blocks, threads, iters);
  run<14>("HSETP2+@IADD", 2, d_out, d_cyc, blocks, threads, iters);
  run<15>("F2FP.F16+FADD", 2, d_out, d_cyc, blocks, threads, iters);
  run<16>("HMNMX2.BF16", 2, d_out, d_cyc, blocks, threads, iters);
  run<17>("VIMNMX.S16x2", 2, d_out, d_cyc, blocks, threads, iters);
  run<18>("LOP3", 1, d_out, d_cyc, blocks, threads, iters);
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
