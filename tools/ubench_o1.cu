// Microbenchmark: the O(1) exact-window recursion step (gc_o1.cu o1_update + o1_output) on
// register data only, NPG plane pairs per lane, W warps per SM — how close to the FP32 pipe
// peak can this dependency structure run?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return d;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}
__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }

struct C { float nk[6], a[6], nb[6], al[6]; };

template <int NPG>
__global__ void k(const C c, int steps, float2* out) {
  float2 S0[NPG], S[NPG][5], D[NPG][5], Ep[NPG], Lp[NPG];
  for (int q = 0; q < NPG; q++) {
    S0[q] = Ep[q] = Lp[q] = make_float2(threadIdx.x * 1e-3f, q);
    for (int t = 0; t < 5; t++) S[q][t] = D[q][t] = make_float2(t * 1e-3f, q * 1e-3f);
  }
  float2 acc = make_float2(0.f, 0.f);
  float2 pe = make_float2(threadIdx.x * 1e-4f, 1e-4f), pl = make_float2(1e-5f, threadIdx.x * 1e-5f);
#pragma unroll 1
  for (int i = 0; i < steps; i++) {
    float2 xe = pe, xl = pl;
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      float2 y = f2mul(f2s(c.al[0]), S0[q]);
#pragma unroll
      for (int t = 0; t < 5; t++) y = f2fma(f2s(c.al[t + 1]), S[q][t], y);
      acc = f2add(acc, y);
      const float2 A = f2add(xe, Lp[q]), B = f2add(Ep[q], xl);
      S0[q] = f2add(S0[q], f2add(xe, xl));
#pragma unroll
      for (int t = 0; t < 5; t++) {
        float2 d = f2fma(f2s(c.nk[t + 1]), S[q][t], D[q][t]);
        d = f2fma(f2s(c.a[t + 1]), A, d);
        d = f2fma(f2s(c.nb[t + 1]), B, d);
        D[q][t] = d;
        S[q][t] = f2add(S[q][t], d);
      }
      Ep[q] = xe;
      Lp[q] = xl;
      xe = f2mul(xe, f2s(0.999f));
      xl = f2mul(xl, f2s(0.998f));
    }
    pe = f2add(pe, f2s(1e-6f));
    pl = f2add(pl, f2s(-1e-6f));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NPG>
void run(int warps_per_sm, C c) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 128, blocks = sms * warps_per_sm / 4, steps = 4096;
  float2* out;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(float2));
  k<NPG><<<blocks, threads>>>(c, 16, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NPG><<<blocks, threads>>>(c, steps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // FP32x2 instructions per step per lane: NPG * (6 out + 1 acc + 3 A/B/box + 1 S0 + 5*4 + 2 psi) + 2
  const double ins = (double)NPG * 32 + 2;
  const double lane_flop_ops = ins * 2 * steps * (double)blocks * threads;   // FP32 lane-ops
  const double peak = (double)sms * 128 * 1.965e9 * ms * 1e-3;               // lane-ops in that time at max clock
  printf("NPG=%d warps/SM=%2d: %.3f ms, FP32 lane-ops %.1f%% of 128/clk/SM @1.965GHz\n", NPG, warps_per_sm, ms,
         100.0 * lane_flop_ops / peak);
  cudaFree(out);
}

int main() {
  C c;
  for (int i = 0; i < 6; i++) { c.nk[i] = -0.01f * i; c.a[i] = 0.5f; c.nb[i] = -0.4f; c.al[i] = 0.1f; }
  for (int w : {4, 8, 12, 16}) { run<1>(w, c); run<4>(w, c); run<7>(w, c); }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
