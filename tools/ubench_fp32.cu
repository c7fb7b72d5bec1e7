// Micro-benchmark: FP32 FMA issue forms on sm_100a (B200).
// Measures FMA lanes per SM clock for: FFMA reg-reg-reg, FFMA with a constant-bank
// operand, FFMA with an immediate, packed FFMA2 (reg pair operands) and FFMA2 with a
// broadcast tap.  Used to choose the inner loop of the FIR passes.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_taps[64];

#define NACC 8
#define ITERS 4096

__global__ void k_ffma_rrr(float* out, float a0, float b0, long long* cyc) {
  float acc[NACC]; float b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = threadIdx.x * 1e-3f + i; b[i] = b0 + i * 1e-4f; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], a0 + (float)0, b[i]);
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], b[(i + 1) % NACC], b[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma_const(float* out, float b0, long long* cyc) {
  float acc[NACC]; float b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = threadIdx.x * 1e-3f + i; b[i] = b0 + i * 1e-4f; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(c_taps[i], acc[i], b[i]);
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(c_taps[i + 8], acc[i], b[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma_imm(float* out, float b0, long long* cyc) {
  float acc[NACC]; float b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = threadIdx.x * 1e-3f + i; b[i] = b0 + i * 1e-4f; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], 0.999f, b[i]);
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], 1.001f, b[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return d;
}

__global__ void k_ffma2_rrr(float* out, float b0, long long* cyc) {
  float2 acc[NACC]; float2 b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = make_float2(threadIdx.x * 1e-3f + i, i); b[i] = make_float2(b0 + i * 1e-4f, b0 - i); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = ffma2(acc[i], b[(i + 3) % NACC], b[i]);
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = ffma2(acc[i], b[(i + 1) % NACC], b[i]);
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// tap broadcast from the constant bank: (k, k) pair built once per tap
__global__ void k_ffma2_tap(float* out, float b0, long long* cyc) {
  float2 acc[NACC]; float2 b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = make_float2(threadIdx.x * 1e-3f + i, i); b[i] = make_float2(b0 + i * 1e-4f, b0 - i); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 2; j++) {
      float2 k = make_float2(c_taps[j], c_taps[j]);
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = ffma2(k, b[i], acc[i]);
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  float h[64]; for (int i = 0; i < 64; i++) h[i] = 0.5f + i * 1e-3f;
  cudaMemcpyToSymbol(c_taps, h, sizeof(h));
  int blocks = p.multiProcessorCount * 4, threads = 256;
  float* out; long long* cyc; cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  long long* hc = new long long[blocks];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"ffma_rrr", "ffma_const", "ffma_imm", "ffma2_rrr", "ffma2_tap"};
  for (int which = 0; which < 5; which++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      switch (which) {
        case 0: k_ffma_rrr<<<blocks, threads>>>(out, 1.0001f, 0.5f, cyc); break;
        case 1: k_ffma_const<<<blocks, threads>>>(out, 0.5f, cyc); break;
        case 2: k_ffma_imm<<<blocks, threads>>>(out, 0.5f, cyc); break;
        case 3: k_ffma2_rrr<<<blocks, threads>>>(out, 0.5f, cyc); break;
        case 4: k_ffma2_tap<<<blocks, threads>>>(out, 0.5f, cyc); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
      double fmas_per_thread = (double)ITERS * 2 * NACC * (which >= 3 ? 2 : 1);
      double total = fmas_per_thread * blocks * threads;
      long long maxc = 0; for (int b = 0; b < blocks; b++) if (hc[b] > maxc) maxc = hc[b];
      // 4 blocks per SM resident simultaneously (256 thr, few regs): lanes/clk/SM
      double lanes_per_clk = fmas_per_thread * threads * 4 / (double)maxc;
      printf("%-11s rep%d  %.3f ms  %.2f TFMA/s  %.1f FMA lanes/clk/SM (cycles %lld)\n", names[which], rep, ms,
             total / ms / 1e9, lanes_per_clk, maxc);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
