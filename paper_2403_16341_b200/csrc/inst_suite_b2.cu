// Registry instances: suite member 11 (the C2 step's most expensive instances) (problems.py:315-330), fp64.
// (Suite members 9-16 are split over four translation units so the largest
// kernels compile in parallel.)  The trust-region instance is compiled in
// inst_suite_b2_trtr.cu with its own ptxas options.
#include "nlk_registry.cuh"
namespace nlk {
extern template cudaError_t launch_solve<Trigonometric, 10, double, ALG_TR>(const KernelArgs&, cudaStream_t,
                                                                           int*);
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/trigonometric", Trigonometric),
};
EntryTable registry_suite_b2() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
