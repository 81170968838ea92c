// Microbenchmark: FFMA vs FFMA2 throughput and dependent-chain latency on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, bool PAIR>
__global__ void k_tp(float* out, int iters, float a, float b) {
  float x[CH]; float2 y[CH];
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = make_float2(x[c], x[c] + 1); }
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (PAIR) y[c] = __ffma2_rn(y[c], a2, b2); else x[c] = fmaf(x[c], a, b);
    }
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += PAIR ? y[c].x + y[c].y : x[c];
  if (s == 123.f) out[0] = s;
}
template <int CH, bool PAIR>
float run(int blocks, int threads, int iters) {
  float* o; cudaMalloc(&o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_tp<CH, PAIR><<<blocks, threads>>>(o, iters, 0.999f, 0.001f);
  cudaEventRecord(e0);
  k_tp<CH, PAIR><<<blocks, threads>>>(o, iters, 0.999f, 0.001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(o);
  return ms;
}
int main() {
  int iters = 20000;
  // latency: 1 warp per SM (148 blocks x 32), 1 chain
  float l1 = run<1, false>(148, 32, iters), l2 = run<1, true>(148, 32, iters);
  double clk = 1.965e9;
  printf("latency FFMA  %.2f cyc/op\n", l1 * 1e-3 * clk / iters);
  printf("latency FFMA2 %.2f cyc/op\n", l2 * 1e-3 * clk / iters);
  // throughput: 148*8 blocks x 256 threads, 8 chains
  float t1 = run<8, false>(148 * 8, 256, iters / 4), t2 = run<8, true>(148 * 8, 256, iters / 4);
  double ops = 148.0 * 8 * 256 * 8 * (iters / 4);
  printf("tp FFMA  %.1f Tfma/s  (%.3f warp-inst/clk/SM)\n", ops / (t1 * 1e-3) / 1e12, ops / 32 / (t1 * 1e-3) / clk / 148);
  printf("tp FFMA2 %.1f Tfma/s  (%.3f warp-inst/clk/SM)\n", 2 * ops / (t2 * 1e-3) / 1e12, ops / 32 / (t2 * 1e-3) / clk / 148);
  // 4 warps per SM (one per scheduler), 4 chains each
  float m1 = run<4, false>(148, 128, iters), m2 = run<4, true>(148, 128, iters);
  printf("1 warp/sched 4 chains: FFMA %.2f cyc/iter, FFMA2 %.2f cyc/iter\n", m1 * 1e-3 * clk / iters, m2 * 1e-3 * clk / iters);
  float n1 = run<8, false>(148, 128, iters), n2 = run<8, true>(148, 128, iters);
  printf("1 warp/sched 8 chains: FFMA %.2f cyc/iter, FFMA2 %.2f cyc/iter\n", n1 * 1e-3 * clk / iters, n2 * 1e-3 * clk / iters);
  return 0;
}
