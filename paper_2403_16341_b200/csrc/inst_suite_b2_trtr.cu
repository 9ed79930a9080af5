// The trigonometric trust-region kernel (registry entry in inst_suite_b2.cu),
// compiled with ptxas' register-usage level 2 instead of the default 5:
// measured 60.7 -> 58.2 ms per 1 M systems on B200 (the Newton kernel of the
// same problem is 3 % slower at that level, so it keeps the default;
// profiles/r02_variants.txt r02R/r02S).  Same code, same results.
// nlk-build: -Xptxas --register-usage-level=2
#include "nlk_registry.cuh"
namespace nlk {
template cudaError_t launch_solve<Trigonometric, 10, double, ALG_TR>(const KernelArgs&, cudaStream_t, int*);
}  // namespace nlk
