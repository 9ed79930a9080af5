// C-ABI entry points (include/nlk_b200.h): validation, registry lookup,
// launch of the persistent solve kernel, and the host-buffer pipeline.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nlk_b200.h"
#include "nlk_registry.cuh"
#include "nlk_ift.cuh"

namespace {

thread_local std::string g_err;
thread_local int g_grid = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(NLK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Registry {
  std::vector<const nlk::Entry*> all;
  Registry() {
    const nlk::EntryTable tables[] = {nlk::registry_suite_a(), nlk::registry_suite_b(),
                                      nlk::registry_suite_b2(), nlk::registry_suite_b3(),
                                      nlk::registry_suite_b4(),
                                      nlk::registry_suite_c(), nlk::registry_families_a(),
                                      nlk::registry_families_b(), nlk::registry_families_c(),
                                      nlk::registry_families_d(), nlk::registry_families_e()};
    for (const auto& t : tables)
      for (int i = 0; i < t.count; ++i) all.push_back(&t.entries[i]);
  }
};
const Registry& reg() {
  static Registry r;
  return r;
}

const char* kAlgNames[nlk::NUM_ALGS] = {"newton-raphson", "trust-region", "broyden",
                                        "klement", "dfsane", "newton-backtracking"};

int validate(int32_t handle, int32_t alg, int32_t dtype, int64_t B, const void* u0, const void* p,
             double abstol, int32_t maxiters, const void* u_out, const void* resid_out,
             const void* retcode_out, nlk::Launcher* launcher, const nlk::Entry** entry) {
  const auto& r = reg();
  if (handle < 0 || handle >= static_cast<int32_t>(r.all.size()))
    return fail(NLK_ERR_UNKNOWN_PROBLEM, "invalid problem handle " + std::to_string(handle));
  if (alg < 0 || alg >= nlk::NUM_ALGS)
    return fail(NLK_ERR_UNKNOWN_ALG, "invalid algorithm id " + std::to_string(alg));
  if (dtype != NLK_F64 && dtype != NLK_F32)
    return fail(NLK_ERR_BAD_ARGUMENT, "dtype must be 0 (f64) or 1 (f32)");
  if (!(abstol > 0)) return fail(NLK_ERR_BAD_OPTIONS, "abstol must be > 0");
  if (maxiters < 1) return fail(NLK_ERR_BAD_OPTIONS, "maxiters must be >= 1");
  if (B < 0) return fail(NLK_ERR_BAD_ARGUMENT, "batch size must be >= 0");
  const nlk::Entry* e = r.all[handle];
  if (B > 0) {
    if (!u0 || !u_out || !resid_out || !retcode_out)
      return fail(NLK_ERR_BAD_ARGUMENT, "u0, u_out, resid_out and retcode_out are required");
    if (e->m > 0 && !p)
      return fail(NLK_ERR_BAD_ARGUMENT, std::string(e->id) + " needs a parameter batch p");
  }
  nlk::Launcher l = e->launch[alg][dtype];
  if (!l)
    return fail(NLK_ERR_NOT_COMPILED, std::string(e->id) + " n=" + std::to_string(e->n) + " " +
                                          kAlgNames[alg] + (dtype ? " f32" : " f64") +
                                          " has no compiled kernel");
  *launcher = l;
  *entry = e;
  return NLK_OK;
}

// Calls that take a stream run on the stream's device: the occupancy query,
// the smem attribute, stream-ordered allocations and the launch all refer to
// the current device, so it is switched to the stream's for the call and
// restored after (a caller whose current device differs from the stream's
// would otherwise launch into another device's stream).
struct DeviceOfStream {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceOfStream(cudaStream_t s) {
    if (s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread) return;
    int sdev = -1, cur = -1;
    err = cudaStreamGetDevice(s, &sdev);
    if (err != cudaSuccess) return;
    err = cudaGetDevice(&cur);
    if (err != cudaSuccess || cur == sdev) return;
    err = cudaSetDevice(sdev);
    if (err == cudaSuccess) prev = cur;
  }
  ~DeviceOfStream() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Stream-ordered allocations (the 8-byte refill counter, the host path's
// staging) come from a private pool per device that keeps its memory
// (release threshold = max), so a first launch after a synchronisation pays
// no page mapping -- without changing the policy of the device's default
// pool, which other libraries in the process share.
cudaError_t pool_alloc(void** ptr, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static cudaMemPool_t pools[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev & 63]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev & 63], &props);
      if (e != cudaSuccess) return e;
      uint64_t thr = UINT64_MAX;
      e = cudaMemPoolSetAttribute(pools[dev & 63], cudaMemPoolAttrReleaseThreshold, &thr);
      if (e != cudaSuccess) return e;
    }
    pool = pools[dev & 63];
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, s);
}

int launch(nlk::Launcher l, const nlk::KernelArgs& a0, cudaStream_t s) {
  nlk::KernelArgs a = a0;
  unsigned long long* counter = nullptr;
  cudaError_t e = pool_alloc(reinterpret_cast<void**>(&counter), sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync(counter)");
  e = cudaMemsetAsync(counter, 0, sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counter)");
  a.counter = counter;
  int grid = 0;
  e = l(a, s, &grid);
  g_grid = grid;
  if (e != cudaSuccess) {
    cudaFreeAsync(counter, s);
    return cuda_fail(e, "solve kernel launch");
  }
  e = cudaFreeAsync(counter, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync(counter)");
  return NLK_OK;
}

// Per-device staging workspace for the host-buffer path: device memory and
// streams are created on first use and grown, never freed per call (a
// cudaMalloc per call would dominate small batches).  Calls on one device
// are serialised by the mutex; they are synchronous anyway.
struct Workspace {
  std::mutex mu;
  char* buf = nullptr;
  size_t cap = 0;
  std::vector<cudaStream_t> streams;
};
Workspace& workspace(int dev) {
  static Workspace ws[64];
  return ws[dev & 63];
}

}  // namespace

extern "C" {

int nlk_version(void) { return 20000; }

const char* nlk_last_error(void) { return g_err.c_str(); }

int nlk_last_grid(void) { return g_grid; }

int nlk_last_launches(void) { return nlk::tl_launches(); }

int nlk_alg_lookup(const char* name) {
  if (!name) return fail(NLK_ERR_UNKNOWN_ALG, "null algorithm name");
  for (int i = 0; i < nlk::NUM_ALGS; ++i)
    if (std::strcmp(name, kAlgNames[i]) == 0) return i;
  return fail(NLK_ERR_UNKNOWN_ALG, std::string("unknown algorithm '") + name + "'");
}

int nlk_num_problems(void) { return static_cast<int>(reg().all.size()); }

int nlk_problem_info(int32_t handle, const char** id, int32_t* n, int32_t* m) {
  const auto& r = reg();
  if (handle < 0 || handle >= static_cast<int32_t>(r.all.size()))
    return fail(NLK_ERR_UNKNOWN_PROBLEM, "invalid problem handle");
  if (id) *id = r.all[handle]->id;
  if (n) *n = r.all[handle]->n;
  if (m) *m = r.all[handle]->m;
  return NLK_OK;
}

int nlk_problem_lookup(const char* id, int32_t n, int32_t* handle, int32_t* n_out, int32_t* m_out) {
  if (!id) return fail(NLK_ERR_UNKNOWN_PROBLEM, "null problem id");
  const auto& r = reg();
  bool known = false;
  for (size_t h = 0; h < r.all.size(); ++h) {
    const nlk::Entry* e = r.all[h];
    if (std::strcmp(e->id, id) != 0) continue;
    known = true;
    if (n > 0 && e->n != n) continue;
    if (handle) *handle = static_cast<int32_t>(h);
    if (n_out) *n_out = e->n;
    if (m_out) *m_out = e->m;
    return NLK_OK;
  }
  if (known)
    return fail(NLK_ERR_BAD_SIZE, std::string(id) + " is not compiled for n=" + std::to_string(n));
  return fail(NLK_ERR_UNKNOWN_PROBLEM, std::string("unknown problem id '") + id + "'");
}

int nlk_solve_batch(int32_t handle, int32_t alg, int32_t dtype, int64_t B, const void* u0_soa,
                    const void* p_soa, double abstol, int32_t maxiters, void* u_out, void* resid_out,
                    int8_t* retcode_out, int32_t* nsteps_out, int32_t* nf_out, int32_t* njac_out,
                    int32_t* nlinsolve_out, void* stream) {
  nlk::Launcher l = nullptr;
  const nlk::Entry* e = nullptr;
  int rc = validate(handle, alg, dtype, B, u0_soa, p_soa, abstol, maxiters, u_out, resid_out,
                    retcode_out, &l, &e);
  if (rc != NLK_OK) return rc;
  if (B == 0) return NLK_OK;
  nlk::KernelArgs a{};
  a.B = B;
  a.u0 = u0_soa;
  a.p = p_soa;
  a.abstol = abstol;
  a.maxiters = maxiters;
  a.u_out = u_out;
  a.resid_out = resid_out;
  a.retcode = retcode_out;
  a.nsteps = nsteps_out;
  a.nf = nf_out;
  a.njac = njac_out;
  a.nlinsolve = nlinsolve_out;
  DeviceOfStream guard(static_cast<cudaStream_t>(stream));
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "stream device");
  return launch(l, a, static_cast<cudaStream_t>(stream));
}

int nlk_solve_batch_poly(int32_t handle, int32_t dtype, int64_t B, const void* u0_soa,
                         const void* p_soa, double abstol, int32_t maxiters, void* u_out,
                         void* resid_out, int8_t* retcode_out, int32_t* nsteps_out,
                         int32_t* nf_out, int32_t* njac_out, int32_t* nlinsolve_out,
                         int8_t* stage_retcodes_out, void* stream) {
  // run_polyalgorithm (solvers.py:570-599) for n <= QN_SKIP_THRESHOLD = 25
  // (every registered problem): the quasi-Newton stages are skipped and the
  // stages are NR -> NR + backtracking -> trust region (solvers.py:553-565).
  static const int32_t kStages[3] = {nlk::ALG_NR, nlk::ALG_NEWTON_LS, nlk::ALG_TR};
  nlk::Launcher ls[3];
  const nlk::Entry* e = nullptr;
  for (int k = 0; k < 3; ++k) {
    int rc = validate(handle, kStages[k], dtype, B, u0_soa, p_soa, abstol, maxiters, u_out,
                      resid_out, retcode_out, &ls[k], &e);
    if (rc != NLK_OK) return rc;
  }
  if (B > 0 && !stage_retcodes_out)
    return fail(NLK_ERR_BAD_ARGUMENT, "stage_retcodes_out [3][B] is required");
  if (B == 0) return NLK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceOfStream guard(st);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "stream device");
  cudaError_t ce = cudaMemsetAsync(stage_retcodes_out, 0xff, 3 * B, st);  // -1: not run
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemsetAsync(stage_retcodes)");
  for (int k = 0; k < 3; ++k) {
    nlk::KernelArgs a{};
    a.B = B;
    a.u0 = u0_soa;
    a.p = p_soa;
    a.abstol = abstol;
    a.maxiters = maxiters;
    a.u_out = u_out;
    a.resid_out = resid_out;
    a.retcode = retcode_out;
    a.nsteps = nsteps_out;
    a.nf = nf_out;
    a.njac = njac_out;
    a.nlinsolve = nlinsolve_out;
    a.poly_stage = k + 1;
    a.stage_rc = stage_retcodes_out;
    int rc = launch(ls[k], a, st);
    if (rc != NLK_OK) return rc;
  }
  return NLK_OK;
}

int nlk_solve_batch_host(int32_t handle, int32_t alg, int32_t dtype, int64_t B, const void* u0_soa,
                         const void* p_soa, double abstol, int32_t maxiters, void* u_out,
                         void* resid_out, int8_t* retcode_out, int32_t* nsteps_out, int32_t* nf_out,
                         int32_t* njac_out, int32_t* nlinsolve_out, int64_t chunk,
                         int32_t num_streams) {
  nlk::Launcher l = nullptr;
  const nlk::Entry* e = nullptr;
  int rc = validate(handle, alg, dtype, B, u0_soa, p_soa, abstol, maxiters, u_out, resid_out,
                    retcode_out, &l, &e);
  if (rc != NLK_OK) return rc;
  if (B == 0) return NLK_OK;
  if (chunk <= 0) chunk = std::max<int64_t>(1 << 16, (B + 3) / 4);
  chunk = std::min<int64_t>(chunk, B);
  if (num_streams <= 0) num_streams = 3;
  const int64_t nchunks = (B + chunk - 1) / chunk;
  num_streams = static_cast<int32_t>(std::min<int64_t>(num_streams, nchunks));
  const size_t es = dtype == NLK_F64 ? 8 : 4;
  const int n = e->n, m = e->m;
  // one device slot per stream: u0 | p | u_out | resid | counters | retcode
  const size_t slot_bytes = (chunk * es * (2 * n + m + 1) + chunk * 4 * 4 + chunk + 511) & ~size_t(255);
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGetDevice");
  Workspace& ws = workspace(dev);
  std::lock_guard<std::mutex> lock(ws.mu);
  const size_t need = slot_bytes * num_streams;
  if (ws.cap < need) {
    if (ws.buf) cudaFree(ws.buf);
    ws.buf = nullptr;
    ws.cap = 0;
    ce = cudaMalloc(&ws.buf, need);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMalloc(workspace)");
    ws.cap = need;
  }
  while (static_cast<int>(ws.streams.size()) < num_streams) {
    cudaStream_t st;
    ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamCreate");
    ws.streams.push_back(st);
  }
  std::vector<cudaStream_t> streams(ws.streams.begin(), ws.streams.begin() + num_streams);
  std::vector<char*> slots(num_streams);
  for (int s = 0; s < num_streams; ++s) slots[s] = ws.buf + s * slot_bytes;
  const char* hu0 = static_cast<const char*>(u0_soa);
  const char* hp = static_cast<const char*>(p_soa);
  char* huo = static_cast<char*>(u_out);
  char* hro = static_cast<char*>(resid_out);
  for (int64_t c = 0; c < nchunks && ce == cudaSuccess && rc == NLK_OK; ++c) {
    const int s = static_cast<int>(c % num_streams);
    cudaStream_t st = streams[s];
    const int64_t lo = c * chunk, len = std::min(chunk, B - lo);
    char* base = slots[s];
    char* du0 = base;
    char* dp = du0 + chunk * es * n;
    char* duo = dp + chunk * es * m;
    char* dro = duo + chunk * es * n;
    int32_t* dcnt = reinterpret_cast<int32_t*>(dro + chunk * es);
    int8_t* drc = reinterpret_cast<int8_t*>(dcnt + 4 * chunk);
    // H2D: n (m) strided rows of the SoA host batch into a dense [n][len] block
    ce = cudaMemcpy2DAsync(du0, len * es, hu0 + lo * es, B * es, len * es, n,
                           cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess && m > 0)
      ce = cudaMemcpy2DAsync(dp, len * es, hp + lo * es, B * es, len * es, m,
                             cudaMemcpyHostToDevice, st);
    if (ce != cudaSuccess) break;
    nlk::KernelArgs a{};
    a.B = len;
    a.u0 = du0;
    a.p = m > 0 ? dp : nullptr;
    a.abstol = abstol;
    a.maxiters = maxiters;
    a.u_out = duo;
    a.resid_out = dro;
    a.retcode = drc;
    a.nsteps = nsteps_out ? dcnt : nullptr;
    a.nf = nf_out ? dcnt + chunk : nullptr;
    a.njac = njac_out ? dcnt + 2 * chunk : nullptr;
    a.nlinsolve = nlinsolve_out ? dcnt + 3 * chunk : nullptr;
    rc = launch(l, a, st);
    if (rc != NLK_OK) break;
    ce = cudaMemcpy2DAsync(huo + lo * es, B * es, duo, len * es, len * es, n,
                           cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(hro + lo * es, dro, len * es, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(retcode_out + lo, drc, len, cudaMemcpyDeviceToHost, st);
    int32_t* outs[4] = {nsteps_out, nf_out, njac_out, nlinsolve_out};
    for (int k = 0; k < 4 && ce == cudaSuccess; ++k)
      if (outs[k]) ce = cudaMemcpyAsync(outs[k] + lo, dcnt + k * chunk, len * 4, cudaMemcpyDeviceToHost, st);
  }
  for (int s = 0; s < num_streams; ++s) {
    cudaError_t e2 = cudaStreamSynchronize(streams[s]);
    if (ce == cudaSuccess) ce = e2;
  }
  if (rc != NLK_OK) return rc;
  if (ce != cudaSuccess) return cuda_fail(ce, "nlk_solve_batch_host");
  return NLK_OK;
}

}  // extern "C"

extern "C" int nlk_solve_batch_host_async(int32_t handle, int32_t alg, int32_t dtype, int64_t B,
                                          const void* u0_soa, const void* p_soa, double abstol,
                                          int32_t maxiters, void* u_out, void* resid_out,
                                          int8_t* retcode_out, int32_t* nsteps_out,
                                          int32_t* nf_out, int32_t* njac_out,
                                          int32_t* nlinsolve_out, void* stream) {
  nlk::Launcher l = nullptr;
  const nlk::Entry* e = nullptr;
  int rc = validate(handle, alg, dtype, B, u0_soa, p_soa, abstol, maxiters, u_out, resid_out,
                    retcode_out, &l, &e);
  if (rc != NLK_OK || B == 0) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceOfStream guard(st);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "stream device");
  const size_t es = dtype == NLK_F64 ? 8 : 4;
  const int n = e->n, m = e->m;
  // staging: u0 | p | u_out | resid | counters[4] | retcode
  const size_t bytes = B * es * (2 * n + m + 1) + B * 4 * 4 + B + 256;
  char* base = nullptr;
  cudaError_t ce = pool_alloc(reinterpret_cast<void**>(&base), bytes, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMallocFromPoolAsync(staging)");
  char* du0 = base;
  char* dp = du0 + B * es * n;
  char* duo = dp + B * es * m;
  char* dro = duo + B * es * n;
  int32_t* dcnt = reinterpret_cast<int32_t*>(dro + B * es);
  int8_t* drc = reinterpret_cast<int8_t*>(dcnt + 4 * B);
  ce = cudaMemcpyAsync(du0, u0_soa, B * es * n, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess && m > 0) ce = cudaMemcpyAsync(dp, p_soa, B * es * m, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) {
    nlk::KernelArgs a{};
    a.B = B;
    a.u0 = du0;
    a.p = m > 0 ? dp : nullptr;
    a.abstol = abstol;
    a.maxiters = maxiters;
    a.u_out = duo;
    a.resid_out = dro;
    a.retcode = drc;
    a.nsteps = nsteps_out ? dcnt : nullptr;
    a.nf = nf_out ? dcnt + B : nullptr;
    a.njac = njac_out ? dcnt + 2 * B : nullptr;
    a.nlinsolve = nlinsolve_out ? dcnt + 3 * B : nullptr;
    rc = launch(l, a, st);
  }
  if (ce == cudaSuccess && rc == NLK_OK) {
    ce = cudaMemcpyAsync(u_out, duo, B * es * n, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(resid_out, dro, B * es, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(retcode_out, drc, B, cudaMemcpyDeviceToHost, st);
    int32_t* outs[4] = {nsteps_out, nf_out, njac_out, nlinsolve_out};
    for (int k = 0; k < 4 && ce == cudaSuccess; ++k)
      if (outs[k]) ce = cudaMemcpyAsync(outs[k], dcnt + k * B, B * 4, cudaMemcpyDeviceToHost, st);
  }
  cudaError_t fe = cudaFreeAsync(base, st);
  if (rc != NLK_OK) return rc;
  if (ce != cudaSuccess) return cuda_fail(ce, "nlk_solve_batch_host_async");
  if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync(staging)");
  return NLK_OK;
}

// ---- IFT sensitivities (nlk_ift.cuh) ----------------------------------------
namespace {
int ift_common(int32_t handle, int32_t dtype, int64_t B, const void* u, const void* th,
               double abstol, const void* out, const int8_t* status, bool adjoint,
               const void* gbar, nlk::IftLauncher* l) {
  const auto& r = reg();
  if (handle < 0 || handle >= static_cast<int32_t>(r.all.size()))
    return fail(NLK_ERR_UNKNOWN_PROBLEM, "invalid problem handle " + std::to_string(handle));
  if (dtype != NLK_F64) return fail(NLK_ERR_NOT_COMPILED, "sensitivities are compiled for f64 only");
  if (!(abstol > 0)) return fail(NLK_ERR_BAD_OPTIONS, "abstol must be > 0");
  if (B < 0) return fail(NLK_ERR_BAD_ARGUMENT, "batch size must be >= 0");
  const nlk::Entry* e = r.all[handle];
  if (B > 0 && (!u || !th || !out || !status || (adjoint && !gbar)))
    return fail(NLK_ERR_BAD_ARGUMENT, "u_star, theta, output and status buffers are required");
  const nlk::IftTable t = nlk::registry_ift();
  for (int i = 0; i < t.count; ++i) {
    if (std::strcmp(t.entries[i].id, e->id) == 0 && t.entries[i].n == e->n) {
      *l = adjoint ? t.entries[i].adjoint : t.entries[i].forward;
      return NLK_OK;
    }
  }
  return fail(NLK_ERR_NOT_COMPILED, std::string(e->id) + " n=" + std::to_string(e->n) +
                                        " has no sensitivity kernel (parametrised problems only)");
}
}  // namespace

extern "C" {
int nlk_ift_forward_batch(int32_t handle, int32_t dtype, int64_t B, const void* u_star_soa,
                          const void* theta_soa, double abstol, void* S_out, void* solve_resid_out,
                          int8_t* status_out, void* stream) {
  nlk::IftLauncher l = nullptr;
  int rc = ift_common(handle, dtype, B, u_star_soa, theta_soa, abstol, S_out, status_out, false,
                      nullptr, &l);
  if (rc != NLK_OK || B == 0) return rc;
  nlk::IftArgs a{B, u_star_soa, theta_soa, nullptr, abstol, S_out, solve_resid_out, status_out};
  DeviceOfStream guard(static_cast<cudaStream_t>(stream));
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "stream device");
  cudaError_t ce = l(a, static_cast<cudaStream_t>(stream));
  return ce == cudaSuccess ? NLK_OK : cuda_fail(ce, "ift kernel launch");
}

int nlk_ift_adjoint_batch(int32_t handle, int32_t dtype, int64_t B, const void* u_star_soa,
                          const void* theta_soa, const void* gbar_soa, double abstol,
                          void* grad_out, void* solve_resid_out, int8_t* status_out,
                          void* stream) {
  nlk::IftLauncher l = nullptr;
  int rc = ift_common(handle, dtype, B, u_star_soa, theta_soa, abstol, grad_out, status_out, true,
                      gbar_soa, &l);
  if (rc != NLK_OK || B == 0) return rc;
  nlk::IftArgs a{B, u_star_soa, theta_soa, gbar_soa, abstol, grad_out, solve_resid_out, status_out};
  DeviceOfStream guard(static_cast<cudaStream_t>(stream));
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "stream device");
  cudaError_t ce = l(a, static_cast<cudaStream_t>(stream));
  return ce == cudaSuccess ? NLK_OK : cuda_fail(ce, "ift kernel launch");
}
}  // extern "C"
