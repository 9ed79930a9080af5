// Kernel-design experiments (not part of the product): times a few solve
// kernels under the code-generation knobs of the headers
//   -DNLK_COMPACT_MIN=n  -DNLK_SWEEP_MAX=w  -DNLK_INLINE_TRANS=0/1  -DNLK_MIN_BLOCKS=b
// on synthetic perturbed starts (xorshift, not the numpy streams).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_2403_16341_b200/csrc tools/variant_bench.cu -o /tmp/vb
#include <cstdio>
#include <cstdint>
#include <vector>

#include "nlk_kernel.cuh"

using namespace nlk;

static uint64_t rs = 88172645463325252ull;
static double urand() {  // [0, 1)
  rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
  return (rs >> 11) * (1.0 / 9007199254740992.0);
}

template <class P, int ALG>
void run(const char* name, const std::vector<double>& start, int64_t B) {
  constexpr int N = P::N;
  double sc = 1.0;
  for (double s : start) sc = fabs(s) > sc ? fabs(s) : sc;
  std::vector<double> h(N * B);
  for (int64_t b = 0; b < B; ++b)
    for (int i = 0; i < N; ++i) h[i * B + b] = start[i] + 0.1 * sc * (2 * urand() - 1);
  double *u0, *uo, *ro;
  int8_t* rc;
  int32_t* cnt;
  unsigned long long* counter;
  cudaMalloc(&u0, 8 * N * B); cudaMalloc(&uo, 8 * N * B); cudaMalloc(&ro, 8 * B);
  cudaMalloc(&rc, B); cudaMalloc(&cnt, 16 * B); cudaMalloc(&counter, 8);
  cudaMemcpy(u0, h.data(), 8 * N * B, cudaMemcpyHostToDevice);
  KernelArgs a{};
  a.B = B; a.u0 = u0; a.p = nullptr; a.abstol = 1e-8; a.maxiters = 1000;
  a.u_out = uo; a.resid_out = ro; a.retcode = rc;
  a.nsteps = cnt; a.nf = cnt + B; a.njac = cnt + 2 * B; a.nlinsolve = cnt + 3 * B;
  a.counter = counter;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  int grid = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(counter, 0, 8);
    cudaEventRecord(e0);
    launch_solve<P, N, double, ALG>(a, 0, &grid);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  std::vector<int32_t> steps(B);
  cudaMemcpy(steps.data(), cnt, 4 * B, cudaMemcpyDeviceToHost);
  long long tot = 0;
  for (auto s : steps) tot += s;
  cudaError_t err = cudaGetLastError();
  printf("%-28s %9.3f ms  grid %5d  mean nsteps %7.2f  %s\n", name, best, grid,
         double(tot) / B, cudaGetErrorString(err));
  cudaFree(u0); cudaFree(uo); cudaFree(ro); cudaFree(rc); cudaFree(cnt); cudaFree(counter);
}

int main() {
  const int64_t B = 262144;
  std::vector<double> trig(10, 0.1), brown(10, 0.5), msq(9, 0.0), cha(10, 1.0), gr16(16, 1.0);
  msq[0] = msq[4] = msq[8] = 1.0;
  gr16[0] = -1.2;
  run<Trigonometric, ALG_NR>("trigonometric NR", trig, B);
  run<Trigonometric, ALG_TR>("trigonometric TR", trig, B);
  run<MatrixSqrt3x3, ALG_TR>("matrix-sqrt-3x3 TR", msq, B);
  run<MatrixSqrt3x3, ALG_NR>("matrix-sqrt-3x3 NR", msq, B);
  run<BrownAlmostLinear, ALG_NR>("brown-almost-linear NR", brown, B);
  run<Chandrasekhar, ALG_TR>("chandrasekhar TR", cha, B);
  run<GeneralizedRosenbrock<16>, ALG_NR>("gen-rosenbrock16 NR", gr16, B);
  return 0;
}
