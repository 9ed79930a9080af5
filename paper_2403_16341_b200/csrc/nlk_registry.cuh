// Registry of compiled (problem, n) instances.  Each instance carries one
// launcher per (algorithm, dtype); a null launcher means that combination is
// not compiled and the C-ABI reports it instead of falling back.
#pragma once
#include "nlk_kernel.cuh"

namespace nlk {

struct Entry {
  const char* id;  // nlkit problem id (problems.py:353,372,386)
  int n;
  int m;
  Launcher launch[NUM_ALGS][2];  // [alg][0 = f64, 1 = f32]
};

template <class P, class T>
constexpr Launcher L(int alg) {
  return alg == ALG_NR ? &launch_solve<P, P::N, T, ALG_NR>
       : alg == ALG_TR ? &launch_solve<P, P::N, T, ALG_TR>
       : alg == ALG_BROYDEN ? &launch_solve<P, P::N, T, ALG_BROYDEN>
       : alg == ALG_KLEMENT ? &launch_solve<P, P::N, T, ALG_KLEMENT>
       : alg == ALG_DFSANE ? &launch_solve<P, P::N, T, ALG_DFSANE>
       : &launch_solve<P, P::N, T, ALG_NEWTON_LS>;
}

#define NLK_ALGS_F64(P) {{L<P, double>(0), nullptr}, {L<P, double>(1), nullptr}, \
  {L<P, double>(2), nullptr}, {L<P, double>(3), nullptr}, {L<P, double>(4), nullptr}, \
  {L<P, double>(5), nullptr}}
#define NLK_ALGS_BOTH(P) {{L<P, double>(0), L<P, float>(0)}, {L<P, double>(1), L<P, float>(1)}, \
  {L<P, double>(2), L<P, float>(2)}, {L<P, double>(3), L<P, float>(3)}, \
  {L<P, double>(4), L<P, float>(4)}, {L<P, double>(5), L<P, float>(5)}}
#define NLK_ENTRY_F64(ID, P) {ID, P::N, P::M, NLK_ALGS_F64(P)}
#define NLK_ENTRY_BOTH(ID, P) {ID, P::N, P::M, NLK_ALGS_BOTH(P)}

struct EntryTable {
  const Entry* entries;
  int count;
};

EntryTable registry_suite_a();
EntryTable registry_suite_b();
EntryTable registry_suite_b2();
EntryTable registry_suite_b3();
EntryTable registry_suite_b4();
EntryTable registry_suite_c();
EntryTable registry_families_a();
EntryTable registry_families_b();
EntryTable registry_families_c();
EntryTable registry_families_d();
EntryTable registry_families_e();

}  // namespace nlk
