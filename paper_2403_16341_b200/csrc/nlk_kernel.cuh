// Persistent batched-solve kernel with warp-aggregated lane refill.
//
// One thread owns one system at a time and advances it one outer iteration
// per trip of the main loop.  A lane whose system terminates writes its
// result and, on the next trip, takes the next unclaimed system index from a
// global counter (one atomicAdd per warp per trip, claimed indices handed out
// by lane rank), so converged systems stop consuming issue slots while the
// heavy-tailed ones (MaxIters = 1000 iterations) keep running.  Every lane
// executes the same step() code on a different system, which keeps warps
// converged except on data-dependent branches inside one iteration.
//
// Batch layout is SoA: u0/u_out [n][B], p [m][B], scalars [B] — lanes that
// refill together claim consecutive indices, so loads/stores coalesce.
#pragma once
#include <stdint.h>
#include <cstdlib>

#include "nlk_coop.cuh"

namespace nlk {

struct KernelArgs {
  int64_t B;
  const void* u0;
  const void* p;
  double abstol;
  int maxiters;
  void* u_out;
  void* resid_out;
  int8_t* retcode;
  int32_t* nsteps;
  int32_t* nf;
  int32_t* njac;
  int32_t* nlinsolve;
  unsigned long long* counter;  // refills claimed so far (zeroed before launch)
};

constexpr int kThreads = kSmStride;
#ifndef NLK_MIN_BLOCKS
#define NLK_MIN_BLOCKS 1
#endif

template <class P, int N, class T, int ALG>
__global__ void __launch_bounds__(kThreads, NLK_MIN_BLOCKS) solve_kernel(const KernelArgs a) {
  using Solver = typename SolverOf<P, N, T, ALG>::type;
  constexpr int M = P::M;
  const T* __restrict__ u0 = static_cast<const T*>(a.u0);
  const T* __restrict__ pp = static_cast<const T*>(a.p);
  T* __restrict__ uo = static_cast<T*>(a.u_out);
  T* __restrict__ ro = static_cast<T*>(a.resid_out);
  const T abstol = static_cast<T>(a.abstol);
  const int lane = threadIdx.x & 31;
  const int64_t B = a.B;

  Solver s;
  if constexpr (Solver::kSmemElems > 0) {
    extern __shared__ __align__(16) unsigned char nlk_dyn_smem[];
    s.sm = reinterpret_cast<T*>(nlk_dyn_smem) + threadIdx.x;
  }
  // first assignment is static (one system per thread), refills are dynamic
  int64_t sys = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool fresh = true;
  for (;;) {
    const bool need = (sys < 0);
    const unsigned want = __ballot_sync(0xffffffffu, need);
    if (want) {
      const int leader = __ffs(want) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(a.counter, static_cast<unsigned long long>(__popc(want)));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const unsigned long long first = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
        sys = static_cast<int64_t>(first + base + __popc(want & ((1u << lane) - 1u)));
        fresh = true;
      }
    }
    const bool live = sys < B;
    if (!__any_sync(0xffffffffu, live)) break;
    if (!live) continue;
    int st;
    if (fresh) {
#pragma unroll
      for (int i = 0; i < N; ++i) s.u[i] = u0[i * B + sys];
#pragma unroll
      for (int i = 0; i < M; ++i) s.p[i] = pp[i * B + sys];
      st = s.init(abstol);
      fresh = false;
    } else {
      st = s.step(abstol, a.maxiters);
    }
    if (st != RUNNING) {
#pragma unroll
      for (int i = 0; i < N; ++i) uo[i * B + sys] = s.u[i];
      ro[sys] = max_abs<N>(s.f);  // resid_max_norm (core.py:101-103)
      a.retcode[sys] = static_cast<int8_t>(st);
      if (a.nsteps) a.nsteps[sys] = s.nsteps;
      if (a.nf) a.nf[sys] = s.nf;
      if (a.njac) a.njac[sys] = s.njac;
      if (a.nlinsolve) a.nlinsolve[sys] = s.nlinsolve;
      sys = -1;
    }
  }
}

// Cooperative variant (nlk_coop.cuh): a group of N lanes per system, 32/N
// systems per warp; refills are claimed per group by its row-0 lane.
template <class P, int N, class T, int ALG>
__global__ void __launch_bounds__(kThreads, NLK_MIN_BLOCKS) solve_kernel_coop(const KernelArgs a) {
  using Solver = typename CoopOf<P, N, T, ALG>::type;
  using Shape = CoopShape<N>;
  constexpr int M = P::M;
  constexpr int WARPS = kThreads / 32;
  __shared__ T tbuf[WARPS][Shape::SPW][N * Shape::LD];
  const T* __restrict__ u0 = static_cast<const T*>(a.u0);
  const T* __restrict__ pp = static_cast<const T*>(a.p);
  T* __restrict__ uo = static_cast<T*>(a.u_out);
  T* __restrict__ ro = static_cast<T*>(a.resid_out);
  const T abstol = static_cast<T>(a.abstol);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t B = a.B;
  const bool idle = lane >= Shape::LANES;
  const int grp = idle ? 0 : lane / N;

  Solver s;
  s.g.base = grp * N;
  s.g.row = lane - s.g.base;
  s.g.mask = ((1u << N) - 1u) << s.g.base;
  s.tbuf = &tbuf[warp][grp][0];
  const int64_t groups_total = static_cast<int64_t>(gridDim.x) * WARPS * Shape::SPW;
  int64_t sys = idle ? B : (static_cast<int64_t>(blockIdx.x) * WARPS + warp) * Shape::SPW + grp;
  bool fresh = true;
  for (;;) {
    const bool need = !idle && sys < 0;
    const bool leader_need = need && s.g.row == 0;
    const unsigned want = __ballot_sync(0xffffffffu, leader_need);
    if (want) {
      const int leader = __ffs(want) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(a.counter, static_cast<unsigned long long>(__popc(want)));
      base = __shfl_sync(0xffffffffu, base, leader);
      int64_t mine = static_cast<int64_t>(groups_total + base + __popc(want & ((1u << lane) - 1u)));
      mine = __shfl_sync(0xffffffffu, mine, idle ? lane : s.g.base);
      if (need) {
        sys = mine;
        fresh = true;
      }
    }
    const bool live = !idle && sys < B;
    if (!__any_sync(0xffffffffu, live)) break;
    if (!live) continue;
    int st;
    if (fresh) {
#pragma unroll
      for (int i = 0; i < N; ++i) s.u[i] = u0[i * B + sys];
#pragma unroll
      for (int i = 0; i < M; ++i) s.p[i] = pp[i * B + sys];
      st = s.init(abstol);
      fresh = false;
    } else {
      st = s.step(abstol, a.maxiters);
    }
    if (st != RUNNING) {
      // lane r writes component r; row 0 writes the scalars
      T ur = s.u[0];
#pragma unroll
      for (int i = 1; i < N; ++i)
        if (i == s.g.row) ur = s.u[i];
      uo[s.g.row * B + sys] = ur;
      if (s.g.row == 0) {
        ro[sys] = max_abs<N>(s.f);
        a.retcode[sys] = static_cast<int8_t>(st);
        if (a.nsteps) a.nsteps[sys] = s.nsteps;
        if (a.nf) a.nf[sys] = s.nf;
        if (a.njac) a.njac[sys] = s.njac;
        if (a.nlinsolve) a.nlinsolve[sys] = s.nlinsolve;
      }
      sys = -1;
    }
  }
}

// Host-side launcher: persistent grid sized from the occupancy calculator.
template <class P, int N, class T, int ALG>
cudaError_t launch_solve(const KernelArgs& a, cudaStream_t stream, int* grid_out) {
  auto kern = [] {
    if constexpr (UseCoop<N, ALG>::value) return solve_kernel_coop<P, N, T, ALG>;
    else return solve_kernel<P, N, T, ALG>;
  }();
  constexpr int per_block_systems = UseCoop<N, ALG>::value ? (kThreads / 32) * CoopShape<N>::SPW : kThreads;
  // occupancy and the smem attribute are per kernel and device: computed once
  static thread_local int cached_dev = -1, cached_sms = 0, cached_per_sm = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  size_t smem = 0;
  if constexpr (!UseCoop<N, ALG>::value)
    smem = sizeof(T) * kThreads * SolverOf<P, N, T, ALG>::type::kSmemElems;
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    // experiment knob: NLK_CARVEOUT=<percent> caps the shared-memory carve-out
    // of the smem-LU kernels (fewer blocks per SM, more L1 for spills)
    if (smem > 0) {
      static const char* co = std::getenv("NLK_CARVEOUT");
      if (co) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(co));
        if (e != cudaSuccess) return e;
      }
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    cached_dev = dev;
    cached_sms = sms;
    cached_per_sm = per_sm < 1 ? 1 : per_sm;
  }
  const int sms = cached_sms, per_sm = cached_per_sm;
  int64_t want = (a.B + per_block_systems - 1) / per_block_systems;
  int64_t grid = static_cast<int64_t>(per_sm) * sms;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = static_cast<int>(grid);
  kern<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

using Launcher = cudaError_t (*)(const KernelArgs&, cudaStream_t, int*);

}  // namespace nlk
