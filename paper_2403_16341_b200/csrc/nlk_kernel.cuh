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

#include "nlk_solvers.cuh"

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
  // Device-side poly-algorithm (run_polyalgorithm, solvers.py:570-599): 0 for
  // a plain solve; stage s = 1, 2, 3 for its s-th stage.  Stage 1 writes the
  // outputs as a plain solve does; a later stage skips every system whose
  // current best is a success, adds its counters to the running totals and
  // replaces the best (u, resid, retcode) when it succeeds or reaches a
  // strictly smaller residual -- min(results, key=(not success, resid_norm)).
  // stage_rc[(s-1)*B + b] records the stage's retcode (-1: stage not run).
  int poly_stage;
  int8_t* stage_rc;
};

// threads per block: the solver's shared-memory slice stride (128, or 64/32
// for the n >= 14 fp64 shared-memory LU)
template <class P, int N, class T, int ALG>
constexpr int block_of() { return SolverOf<P, N, T, ALG>::type::kStride; }
#ifndef NLK_MIN_BLOCKS
#define NLK_MIN_BLOCKS 1
#endif

// Result of a finished system: written as a plain solve, or merged into the
// running poly-algorithm state (KernelArgs::poly_stage).
template <int N, class T, class S>
__device__ __forceinline__ void finish(const KernelArgs& a, const S& s, int st, int64_t sys,
                                       int64_t B, T* __restrict__ uo, T* __restrict__ ro) {
  const T r = max_abs<N>(s.f);  // resid_max_norm (core.py:101-103)
  if (a.poly_stage > 1) {
    a.stage_rc[static_cast<int64_t>(a.poly_stage - 1) * B + sys] = static_cast<int8_t>(st);
    if (a.nsteps) a.nsteps[sys] += s.nsteps;
    if (a.nf) a.nf[sys] += s.nf;
    if (a.njac) a.njac[sys] += s.njac;
    if (a.nlinsolve) a.nlinsolve[sys] += s.nlinsolve;
    if (st == SUCCESS || r < ro[sys]) {  // NaN never compares smaller
#pragma unroll
      for (int i = 0; i < N; ++i) uo[i * B + sys] = s.u[i];
      ro[sys] = r;
      a.retcode[sys] = static_cast<int8_t>(st);
    }
  } else {
    if (a.poly_stage == 1) a.stage_rc[sys] = static_cast<int8_t>(st);
#pragma unroll
    for (int i = 0; i < N; ++i) uo[i * B + sys] = s.u[i];
    ro[sys] = r;
    a.retcode[sys] = static_cast<int8_t>(st);
    if (a.nsteps) a.nsteps[sys] = s.nsteps;
    if (a.nf) a.nf[sys] = s.nf;
    if (a.njac) a.njac[sys] = s.njac;
    if (a.nlinsolve) a.nlinsolve[sys] = s.nlinsolve;
  }
}

// Deferral (FAST kernels, below): a system the fast kernel cannot finish is
// marked in its retcode slot (the stage's slot for a poly-algorithm stage)
// and re-solved from its start by solve_kernel_deferred.
constexpr int8_t kDeferMark = -2;
__device__ __forceinline__ int8_t* defer_slot(const KernelArgs& a, int64_t sys) {
  return a.poly_stage > 0 ? a.stage_rc + static_cast<int64_t>(a.poly_stage - 1) * a.B + sys : a.retcode + sys;
}

template <class P, int N, class T, int ALG, bool FAST = false>
__global__ void __launch_bounds__(block_of<P, N, T, ALG>(), NLK_MIN_BLOCKS) solve_kernel(const KernelArgs a) {
  using Solver = typename SolverOf<P, N, T, ALG, FAST>::type;
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
      if (a.poly_stage > 1 && a.retcode[sys] == SUCCESS) {  // an earlier stage succeeded
        sys = -1;
        continue;
      }
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
      if (FAST && st == DEFERRED) *defer_slot(a, sys) = kDeferMark;
      else finish<N>(a, s, st, sys, B, uo, ro);
      sys = -1;
    }
  }
}

// The systems a FAST kernel deferred, each solved from its start with the
// complete solver (the dual-sweep fallback of a declined closed form inline):
// the same operations on the same inputs as a complete kernel would have
// run, so the outputs are the same bits.  Grid-stride over the marks; with
// no deferred system it only reads the B mark bytes.
template <class P, int N, class T, int ALG>
__global__ void __launch_bounds__(block_of<P, N, T, ALG>(), NLK_MIN_BLOCKS) solve_kernel_deferred(const KernelArgs a) {
  using Solver = typename SolverOf<P, N, T, ALG, false>::type;
  constexpr int M = P::M;
  const T* __restrict__ u0 = static_cast<const T*>(a.u0);
  const T* __restrict__ pp = static_cast<const T*>(a.p);
  T* __restrict__ uo = static_cast<T*>(a.u_out);
  T* __restrict__ ro = static_cast<T*>(a.resid_out);
  const T abstol = static_cast<T>(a.abstol);
  const int64_t B = a.B;
  Solver s;
  if constexpr (Solver::kSmemElems > 0) {
    extern __shared__ __align__(16) unsigned char nlk_dyn_smem[];
    s.sm = reinterpret_cast<T*>(nlk_dyn_smem) + threadIdx.x;
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t sys = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; sys < B; sys += stride) {
    if (*defer_slot(a, sys) != kDeferMark) continue;
#pragma unroll
    for (int k = 0; k < N; ++k) s.u[k] = u0[k * B + sys];
#pragma unroll
    for (int k = 0; k < M; ++k) s.p[k] = pp[k * B + sys];
    int st = s.init(abstol);
    while (st == RUNNING) st = s.step(abstol, a.maxiters);
    finish<N>(a, s, st, sys, B, uo, ro);
  }
}

// Static schedule for problem families whose iteration counts are tight
// (P::kStaticAlgs, e.g. the parametrised quadratic of C1/C5: 4-8 Newton
// steps on every system).  Each thread takes systems by grid stride and runs
// each to completion: a warp's lanes always hold consecutive systems, so
// every load and store of the SoA batch is one coalesced transaction, and
// there is no per-iteration refill bookkeeping (ballot, vote, atomics).  The
// price is that a warp runs as long as its slowest lane -- the reason the
// heavy-tailed suite problems keep the refilling kernel above.
#ifndef NLK_STATIC_PREFETCH_MAX
#define NLK_STATIC_PREFETCH_MAX 16
#endif
template <class P, int N, class T, int ALG>
__global__ void __launch_bounds__(block_of<P, N, T, ALG>(), NLK_MIN_BLOCKS) solve_kernel_static(const KernelArgs a) {
  using Solver = typename SolverOf<P, N, T, ALG>::type;
  constexpr int M = P::M;
  const T* __restrict__ u0 = static_cast<const T*>(a.u0);
  const T* __restrict__ pp = static_cast<const T*>(a.p);
  T* __restrict__ uo = static_cast<T*>(a.u_out);
  T* __restrict__ ro = static_cast<T*>(a.resid_out);
  const T abstol = static_cast<T>(a.abstol);
  const int64_t B = a.B;
  Solver s;
  if constexpr (Solver::kSmemElems > 0) {
    extern __shared__ __align__(16) unsigned char nlk_dyn_smem[];
    s.sm = reinterpret_cast<T*>(nlk_dyn_smem) + threadIdx.x;
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t sys = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // the next system's inputs are loaded before the current one is solved, so
  // their DRAM latency hides behind the solve (small N + M: registers)
  constexpr bool PF = N + M <= NLK_STATIC_PREFETCH_MAX;
  T nu[PF ? N : 1], np_[PF && M > 0 ? M : 1];
  auto load = [&](int64_t i, T* uu, T* pv) {
#pragma unroll
    for (int k = 0; k < N; ++k) uu[k] = u0[k * B + i];
#pragma unroll
    for (int k = 0; k < M; ++k) pv[k] = pp[k * B + i];
  };
  if constexpr (PF) {
    if (sys < B) load(sys, nu, np_);
  }
  for (; sys < B; sys += stride) {
    if constexpr (PF) {
#pragma unroll
      for (int k = 0; k < N; ++k) s.u[k] = nu[k];
#pragma unroll
      for (int k = 0; k < M; ++k) s.p[k] = np_[k];
      if (sys + stride < B) load(sys + stride, nu, np_);
    } else {
      load(sys, s.u, s.p);
    }
    if (a.poly_stage > 1 && a.retcode[sys] == SUCCESS) continue;  // an earlier stage succeeded
    int st = s.init(abstol);
    while (st == RUNNING) st = s.step(abstol, a.maxiters);
    finish<N>(a, s, st, sys, B, uo, ro);
  }
}

// NLK_SCHEDULE_STATIC_ALL=1 (variant builds): every kernel static
#ifndef NLK_SCHEDULE_STATIC_ALL
#define NLK_SCHEDULE_STATIC_ALL 0
#endif
#ifndef NLK_SCHEDULE_STATIC
#define NLK_SCHEDULE_STATIC 1
#endif
template <class P, int ALG> struct UseStatic {
  static constexpr bool value =
      NLK_SCHEDULE_STATIC_ALL || (NLK_SCHEDULE_STATIC && StaticSchedule<P, ALG>::value);
};
// NLK_FAST_DEFER: closed-form problems' Newton / trust-region kernels run
// without the rarely-taken dual-sweep fallback and defer the systems that
// need it (the fallback made the trigonometric trust region's kernel 1.6x
// larger and 29 % slower: profiles/r02_variants.txt r02Z/r02AB)
#ifndef NLK_FAST_DEFER
#define NLK_FAST_DEFER 1
#endif
template <class P, int ALG, class T> struct UseFast {
  static constexpr bool value = NLK_FAST_DEFER && HasJacClosedForm<P>::value && std::is_same<T, double>::value &&
                                (ALG == ALG_NR || ALG == ALG_TR || ALG == ALG_NEWTON_LS) &&
                                !UseStatic<P, ALG>::value;
};

// kernels issued by the last launch_solve on this thread (nlk_last_launches)
inline int& tl_launches() {
  static thread_local int n = 0;
  return n;
}

// Host-side launcher: persistent grid sized from the occupancy calculator.
template <class P, int N, class T, int ALG>
cudaError_t launch_solve(const KernelArgs& a, cudaStream_t stream, int* grid_out) {
  constexpr bool kFast = UseFast<P, ALG, T>::value;
  auto kern = [] {
    if constexpr (UseStatic<P, ALG>::value) return solve_kernel_static<P, N, T, ALG>;
    else return solve_kernel<P, N, T, ALG, kFast>;
  }();
  constexpr int kThreads = block_of<P, N, T, ALG>();
  constexpr int per_block_systems = kThreads;
  // occupancy and the smem attribute are per kernel and device: computed once
  // per device (per_sm_of[dev] == 0: not yet)
  static thread_local int sms_of[64], per_sm_of[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  dev &= 63;
  size_t smem = sizeof(T) * kThreads * SolverOf<P, N, T, ALG>::type::kSmemElems;
  // experiment knob: NLK_EXTRA_SMEM=<bytes> per block lowers the blocks per
  // SM (occupancy sensitivity of a kernel; results are unchanged)
  static const char* extra_smem = std::getenv("NLK_EXTRA_SMEM");
  if (extra_smem) smem += std::atoi(extra_smem);
  if (per_sm_of[dev] == 0) {
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
    sms_of[dev] = sms;
    per_sm_of[dev] = per_sm < 1 ? 1 : per_sm;
  }
  const int sms = sms_of[dev], per_sm = per_sm_of[dev];
  int64_t want = (a.B + per_block_systems - 1) / per_block_systems;
  int64_t grid = static_cast<int64_t>(per_sm) * sms;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = static_cast<int>(grid);
  kern<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(a);
  tl_launches() = kFast ? 2 : 1;
  if constexpr (kFast) {
    // the complete kernel for the deferred systems (same block and smem)
    static thread_local bool attr_set[64];
    if (!attr_set[dev] && smem > 48 * 1024) {
      e = cudaFuncSetAttribute(solve_kernel_deferred<P, N, T, ALG>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    attr_set[dev] = true;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    solve_kernel_deferred<P, N, T, ALG><<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(a);
  }
  return cudaGetLastError();
}

using Launcher = cudaError_t (*)(const KernelArgs&, cudaStream_t, int*);

}  // namespace nlk
